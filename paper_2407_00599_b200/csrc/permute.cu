// Token <-> slot data movement of the MoE layer, each kernel written against
// the communication layout it feeds or drains (no separate regroup passes):
//
//   dispatch_rows   slot tensor (E, S, M) built by GATHER: row (e, s) <- x[t]
//                   (zero when the slot is unfilled or padding), optionally
//                   scaled by the combine weight (backward of the combine).
//                   Reference: gate() dispatch fill, dataplane.py:101,112 and
//                   the S2 slot split + zero pad, dataplane.py:373-378.
//   combine_fwd     out[t] = sum_j w[t,j] * sum_p Y_p[e_j, s_j]  (dropped -> 0)
//                   = fused_combine's local ESP sum (collectives.py:296-310)
//                   fused with _combine (dataplane.py:131-143).
//   combine_bwd     dlogits from dOut: dw_j = <dOut[t], Y[e_j,s_j]>, softmax
//                   adjoint over all E experts (no reference).
//   dispatch_bwd    dx[t] = sum_j sum_p dR_p[e_j, s_j] + dlogits[t] . Wg^T
//   esp_sum         S2: out[e, s] = sum_p Y_p[e, s] before the MP AllGather.
//
// All rows move as 16-byte vectors, one warp per row/token; accumulation f32.
#include "common.cuh"

namespace parm {

constexpr int kRowThreads = 256;

static int row_grid(long long rows) {
    long long warps = rows;
    long long blocks = (warps * 32 + kRowThreads - 1) / kRowThreads;
    const long long cap = (long long)kNumSMs * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

__global__ void __launch_bounds__(kRowThreads) dispatch_rows_kernel(
    const bf16* __restrict__ x, long long ldx, const int* __restrict__ slot_src, const float* __restrict__ scale,
    int k, int E, int cap, int slot_lo, int slots_out, int M, bf16* __restrict__ out, long long out_stride_e,
    long long out_stride_s) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    const long long rows = (long long)E * slots_out;
    for (long long r = warp_global; r < rows; r += num_warps) {
        const int e = (int)(r / slots_out);
        const int sp = (int)(r - (long long)e * slots_out);
        const int s = slot_lo + sp;
        const int src = (s < cap) ? slot_src[(long long)e * cap + s] : -1;
        bf16* dst = out + (long long)e * out_stride_e + (long long)sp * out_stride_s;
        if (src < 0) {
            const int4 z = make_int4(0, 0, 0, 0);
            for (int c = lane * 8; c < M; c += 256) *reinterpret_cast<int4*>(dst + c) = z;
        } else {
            const int t = src / k;
            const bf16* xr = x + (long long)t * ldx;
            if (scale == nullptr) {
                for (int c = lane * 8; c < M; c += 256)
                    *reinterpret_cast<int4*>(dst + c) = __ldg(reinterpret_cast<const int4*>(xr + c));
            } else {
                const float w = scale[src];
                for (int c = lane * 8; c < M; c += 256) {
                    float f[8];
                    vec8_to_f32(ld_vec8(xr + c), f);
#pragma unroll
                    for (int u = 0; u < 8; ++u) f[u] *= w;
                    st_vec8(dst + c, f32_to_vec8(f));
                }
            }
        }
    }
}

// Sum of the n_p partial rows of (e, s) into f (8 floats at column c).
__device__ __forceinline__ void gather_slot(const SlotView& v, int e, int s, int c, float* f) {
#pragma unroll
    for (int u = 0; u < 8; ++u) f[u] = 0.0f;
    for (int p = 0; p < v.n_p; ++p) {
        float g[8];
        vec8_to_f32(ld_vec8(v.ptr + slot_offset(v, e, s, p) + c), g);
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] += g[u];
    }
}

__global__ void __launch_bounds__(kRowThreads) combine_fwd_kernel(const SlotView y, const int* __restrict__ expert_idx,
                                                                   const int* __restrict__ slot_idx,
                                                                   const float* __restrict__ combine_w, int n, int k,
                                                                   int M, bf16* __restrict__ out, long long ldo) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    for (long long t = warp_global; t < n; t += num_warps) {
        // Routing of all k picks first, so the row loads below are independent.
        int sl[8], ex[8];
        float wt[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            sl[j] = (j < k) ? slot_idx[t * k + j] : -1;
            ex[j] = (sl[j] >= 0) ? expert_idx[t * k + j] : 0;
            wt[j] = (sl[j] >= 0) ? combine_w[t * k + j] : 0.0f;
        }
        for (int c = lane * 8; c < M; c += 256) {
            float acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (sl[j] < 0) continue;
                float f[8];
                gather_slot(y, ex[j], sl[j], c, f);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = fmaf(wt[j], f[u], acc[u]);
            }
            st_vec8(out + t * ldo + c, f32_to_vec8(acc));
        }
    }
}

template <int EMAX>
__global__ void __launch_bounds__(kRowThreads) combine_bwd_kernel(const bf16* __restrict__ dout, long long ldd,
                                                                   const SlotView y, const int* __restrict__ expert_idx,
                                                                   const int* __restrict__ slot_idx,
                                                                   const float* __restrict__ probs, int n, int k, int E,
                                                                   int M, float* __restrict__ dlogits) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    for (long long t = warp_global; t < n; t += num_warps) {
        float dw[8];
        int sl[8], ex[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            dw[j] = 0.0f;
            sl[j] = (j < k) ? slot_idx[t * k + j] : -1;
            ex[j] = (sl[j] >= 0) ? expert_idx[t * k + j] : 0;
        }
        for (int c = lane * 8; c < M; c += 256) {
            float g[8];
            vec8_to_f32(ld_vec8(dout + t * ldd + c), g);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (sl[j] < 0) continue;
                float f[8];
                gather_slot(y, ex[j], sl[j], c, f);
#pragma unroll
                for (int u = 0; u < 8; ++u) dw[j] = fmaf(g[u], f[u], dw[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) dw[j] += __shfl_xor_sync(0xffffffffu, dw[j], off);
        // Softmax adjoint: dl_e = p_e * (dS_e - sum_e' p_e' dS_e'), dS nonzero on kept picks.
        if (lane < E) {
            const float pe = probs[t * E + lane];
            float dse = 0.0f, dot = 0.0f;
            for (int j = 0; j < k; ++j) {
                if (slot_idx[t * k + j] < 0) continue;
                const int e = expert_idx[t * k + j];
                float dj = 0.0f;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                    if (jj == j) dj = dw[jj];
                dot += probs[t * E + e] * dj;
                if (e == lane) dse = dj;
            }
            dlogits[t * E + lane] = pe * (dse - dot);
        }
    }
}

template <int EMAX>
__global__ void __launch_bounds__(kRowThreads) dispatch_bwd_kernel(const SlotView dr, const int* __restrict__ expert_idx,
                                                                    const int* __restrict__ slot_idx,
                                                                    const float* __restrict__ dlogits,
                                                                    const bf16* __restrict__ wgT, int n, int k, int E,
                                                                    int M, bf16* __restrict__ dx, long long ldx) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    for (long long t = warp_global; t < n; t += num_warps) {
        int sl[8], ex[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            sl[j] = (j < k) ? slot_idx[t * k + j] : -1;
            ex[j] = (sl[j] >= 0) ? expert_idx[t * k + j] : 0;
        }
        float dl[EMAX];
        if (dlogits) {
#pragma unroll
            for (int e = 0; e < EMAX; ++e) dl[e] = (e < E) ? dlogits[t * E + e] : 0.0f;
        }
        for (int c = lane * 8; c < M; c += 256) {
            float acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (sl[j] < 0) continue;
                float f[8];
                gather_slot(dr, ex[j], sl[j], c, f);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] += f[u];
            }
            if (dlogits) {   // + dlogits[t] . Wg^T with Wg stored transposed (E, M)
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    if (e < E) {
                        float w[8];
                        vec8_to_f32(ld_vec8(wgT + (long long)e * M + c), w);
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[u] = fmaf(dl[e], w[u], acc[u]);
                    }
                }
            }
            st_vec8(dx + t * ldx + c, f32_to_vec8(acc));
        }
    }
}

__global__ void __launch_bounds__(kRowThreads) esp_sum_kernel(const SlotView y, int E, int slots, int M,
                                                               bf16* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp_global = ((long long)blockIdx.x * kRowThreads + threadIdx.x) >> 5;
    const long long num_warps = ((long long)gridDim.x * kRowThreads) >> 5;
    const long long rows = (long long)E * slots;
    for (long long r = warp_global; r < rows; r += num_warps) {
        const int e = (int)(r / slots);
        const int s = (int)(r - (long long)e * slots);
        for (int c = lane * 8; c < M; c += 256) {
            float f[8];
            gather_slot(y, e, s, c, f);
            st_vec8(out + r * M + c, f32_to_vec8(f));
        }
    }
}

// ------------------------------------------------------------------ host
static int check_view(const SlotView& v, int M, const char* what) {
    PARM_CHECK_ARG(v.ptr != nullptr, "%s: null slot view", what);
    PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0, "%s: slot view base not 16-byte aligned", what);
    PARM_CHECK_ARG(v.e_local >= 1 && v.n_p >= 1 && v.slot_div >= 1, "%s: bad slot view", what);
    PARM_CHECK_ARG(M % 8 == 0, "%s: embed %d must be a multiple of 8", what, M);
    return 0;
}

int dispatch_rows(const void* x, long long ldx, const int* slot_src, const float* scale, int k, int E, int cap,
                  int slot_lo, int slots_out, int M, void* out, long long out_stride_e, long long out_stride_s,
                  cudaStream_t s) {
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0 && out_stride_s % 8 == 0 && out_stride_e % 8 == 0,
                   "dispatch_rows: rows must be 16-byte aligned (M=%d)", M);
    const long long rows = (long long)E * slots_out;
    if (rows == 0) return 0;
    dispatch_rows_kernel<<<row_grid(rows), kRowThreads, 0, s>>>(
        reinterpret_cast<const bf16*>(x), ldx, slot_src, scale, k, E, cap, slot_lo, slots_out, M,
        reinterpret_cast<bf16*>(out), out_stride_e, out_stride_s);
    PARM_CHECK_LAUNCH("dispatch_rows");
    return 0;
}

int combine_fwd(const SlotView& y, const int* expert_idx, const int* slot_idx, const float* combine_w, int n, int k,
                int M, void* out, long long ldo, cudaStream_t s) {
    if (int rc = check_view(y, M, "combine_fwd")) return rc;
    if (n == 0) return 0;
    combine_fwd_kernel<<<row_grid(n), kRowThreads, 0, s>>>(y, expert_idx, slot_idx, combine_w, n, k, M,
                                                           reinterpret_cast<bf16*>(out), ldo);
    PARM_CHECK_LAUNCH("combine_fwd");
    return 0;
}

int combine_bwd(const void* dout, long long ldd, const SlotView& y, const int* expert_idx, const int* slot_idx,
                const float* probs, int n, int k, int E, int M, float* dlogits, cudaStream_t s) {
    if (int rc = check_view(y, M, "combine_bwd")) return rc;
    PARM_CHECK_ARG(k <= 8 && E <= 32, "combine_bwd: k<=8 and E<=32 required");
    if (n == 0) return 0;
    auto D = reinterpret_cast<const bf16*>(dout);
    if (E <= 8)
        combine_bwd_kernel<8><<<row_grid(n), kRowThreads, 0, s>>>(D, ldd, y, expert_idx, slot_idx, probs, n, k, E, M,
                                                                  dlogits);
    else
        combine_bwd_kernel<32><<<row_grid(n), kRowThreads, 0, s>>>(D, ldd, y, expert_idx, slot_idx, probs, n, k, E,
                                                                   M, dlogits);
    PARM_CHECK_LAUNCH("combine_bwd");
    return 0;
}

int dispatch_bwd(const SlotView& dr, const int* expert_idx, const int* slot_idx, const float* dlogits, const void* wg,
                 int n, int k, int E, int M, void* dx, long long ldx, cudaStream_t s) {
    if (int rc = check_view(dr, M, "dispatch_bwd")) return rc;
    PARM_CHECK_ARG(E <= 32, "dispatch_bwd: E<=32 required");
    PARM_CHECK_ARG(dlogits == nullptr || wg != nullptr, "dispatch_bwd: dlogits needs gate weights");
    if (n == 0) return 0;
    auto W = reinterpret_cast<const bf16*>(wg);
    auto DX = reinterpret_cast<bf16*>(dx);
    if (E <= 8)
        dispatch_bwd_kernel<8><<<row_grid(n), kRowThreads, 0, s>>>(dr, expert_idx, slot_idx, dlogits, W, n, k, E, M,
                                                                   DX, ldx);
    else
        dispatch_bwd_kernel<32><<<row_grid(n), kRowThreads, 0, s>>>(dr, expert_idx, slot_idx, dlogits, W, n, k, E, M,
                                                                    DX, ldx);
    PARM_CHECK_LAUNCH("dispatch_bwd");
    return 0;
}

int esp_sum(const SlotView& y, int E, int slots, int M, void* out, cudaStream_t s) {
    if (int rc = check_view(y, M, "esp_sum")) return rc;
    const long long rows = (long long)E * slots;
    if (rows == 0) return 0;
    esp_sum_kernel<<<row_grid(rows), kRowThreads, 0, s>>>(y, E, slots, M, reinterpret_cast<bf16*>(out));
    PARM_CHECK_LAUNCH("esp_sum");
    return 0;
}

}  // namespace parm
