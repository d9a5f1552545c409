// Fused gate: logits -> softmax -> stable top-k -> token-major capacity slots,
// plus the gate's backward (softmax adjoint and the Wg weight gradient).
//
// Reference semantics (moesched dataplane.py:80-119):
//   scores  = softmax(X @ Wg)                       (f64)
//   ranked  = argsort(-scores, stable)[:, :k]       ties -> lower expert index
//   weights = scores[ranked]                        (raw probabilities, no renorm)
//   slots   : for t ascending, j ascending: e = ranked[t, j];
//             slot = fill[e]++ if fill[e] < capacity else dropped
//
// Routing (expert_index, slot_index) is integer work and must be bit-exact.
// Logits are therefore accumulated in f64 from the same bf16 inputs the oracle
// sees (every bf16 x bf16 product is exact in f64, so only the summation order
// differs from the oracle's BLAS f64 dot); softmax and ranking run in f64.
// The slot pass is an exact per-expert exclusive prefix count over tokens.
#include "common.cuh"

namespace parm {

constexpr int kGateThreads = 256;

// One warp handles TPW tokens at once so each Wg load is reused TPW times.
template <int EMAX, int TPW>
__global__ void __launch_bounds__(kGateThreads) gate_fwd_kernel(const bf16* __restrict__ x, long long ldx,
                                                                 const bf16* __restrict__ wg, int n, int M, int E,
                                                                 int k, int* __restrict__ expert_idx,
                                                                 float* __restrict__ combine_w,
                                                                 float* __restrict__ probs) {
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * kGateThreads + threadIdx.x) >> 5;
    const int num_warps = (gridDim.x * kGateThreads) >> 5;
    for (int t0 = warp_global * TPW; t0 < n; t0 += num_warps * TPW) {
        double acc[TPW][EMAX];
#pragma unroll
        for (int q = 0; q < TPW; ++q)
#pragma unroll
            for (int e = 0; e < EMAX; ++e) acc[q][e] = 0.0;
        for (int c = lane * 8; c < M; c += 256) {
            float xv[TPW][8];
#pragma unroll
            for (int q = 0; q < TPW; ++q) {
                if (t0 + q < n) {
                    vec8_to_f32(ld_vec8(x + (long long)(t0 + q) * ldx + c), xv[q]);
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) xv[q][u] = 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bf16* wrow = wg + (long long)(c + u) * E;
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    if (e < E) {
                        const double w = (double)bf2f(wrow[e]);
#pragma unroll
                        for (int q = 0; q < TPW; ++q) acc[q][e] = fma((double)xv[q][u], w, acc[q][e]);
                    }
                }
            }
        }
        // Butterfly all-reduce: every lane ends with every logit.
#pragma unroll
        for (int q = 0; q < TPW; ++q)
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc[q][e] += __shfl_xor_sync(0xffffffffu, acc[q][e], off);

#pragma unroll
        for (int q = 0; q < TPW; ++q) {
            const int t = t0 + q;
            if (t >= n) break;
            double mx = acc[q][0];
#pragma unroll
            for (int e = 1; e < EMAX; ++e)
                if (e < E) mx = fmax(mx, acc[q][e]);
            double ex[EMAX];
            double sum = 0.0;
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                ex[e] = (e < E) ? exp(acc[q][e] - mx) : 0.0;
                sum += ex[e];
            }
            // Lane e owns expert e: compute its stable descending rank.
            if (lane < E) {
                double mine = 0.0;
#pragma unroll
                for (int e = 0; e < EMAX; ++e)
                    if (e == lane) mine = ex[e] / sum;
                int rank = 0;
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    if (e < E) {
                        const double other = ex[e] / sum;
                        rank += (other > mine) || (other == mine && e < lane);
                    }
                }
                if (rank < k) {
                    expert_idx[(long long)t * k + rank] = lane;
                    combine_w[(long long)t * k + rank] = (float)mine;
                }
                if (probs) probs[(long long)t * E + lane] = (float)mine;
            }
        }
    }
}

// Exclusive per-expert prefix count over tokens -> slots (single CTA, exact).
constexpr int kSlotThreads = 1024;
constexpr int kMaxExperts = 64;

__global__ void __launch_bounds__(kSlotThreads) gate_slots_kernel(const int* __restrict__ expert_idx, int n, int k,
                                                                   int E, int cap, int* __restrict__ slot_idx,
                                                                   int* __restrict__ slot_src,
                                                                   int* __restrict__ fill) {
    __shared__ int warp_cnt[32][kMaxExperts];
    __shared__ int running[kMaxExperts];
    __shared__ int chunk_tot[kMaxExperts];
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    for (long long i = tid; i < (long long)E * cap; i += kSlotThreads) slot_src[i] = -1;
    if (tid < E) running[tid] = 0;
    __syncthreads();
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int base = 0; base < n; base += kSlotThreads) {
        const int t = base + tid;
        int ex[8];
        const int kk = k < 8 ? k : 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) ex[j] = (t < n && j < kk) ? expert_idx[(long long)t * k + j] : -1;
        int pre[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pre[j] = 0;
        for (int e = 0; e < E; ++e) {
            bool flag = false;
#pragma unroll
            for (int j = 0; j < 8; ++j) flag |= (ex[j] == e);
            const unsigned b = __ballot_sync(0xffffffffu, flag);
            const int p = __popc(b & lt_mask);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (ex[j] == e) pre[j] = p;
            if (lane == 0) warp_cnt[warp][e] = __popc(b);
        }
        __syncthreads();
        if (tid < E) {
            int acc = 0;
            for (int w = 0; w < 32; ++w) {
                const int c = warp_cnt[w][tid];
                warp_cnt[w][tid] = acc;
                acc += c;
            }
            chunk_tot[tid] = acc;
        }
        __syncthreads();
        if (t < n) {
            for (int j = 0; j < kk; ++j) {
                const int e = ex[j];
                const int slot = running[e] + warp_cnt[warp][e] + pre[j];
                if (slot < cap) {
                    slot_idx[(long long)t * k + j] = slot;
                    slot_src[(long long)e * cap + slot] = t * k + j;
                } else {
                    slot_idx[(long long)t * k + j] = -1;
                }
            }
        }
        __syncthreads();
        if (tid < E) running[tid] += chunk_tot[tid];
        __syncthreads();
    }
    if (tid < E) fill[tid] = running[tid] < cap ? running[tid] : cap;
}

// dWg partials: part[c][m][e] = sum_{t in chunk c} x[t][m] * dlogits[t][e].
template <int EMAX>
__global__ void __launch_bounds__(256) gate_wgrad_partial_kernel(const bf16* __restrict__ x, long long ldx,
                                                                  const float* __restrict__ dlogits, int n, int M,
                                                                  int E, int chunk, float* __restrict__ part) {
    __shared__ float dl[64][EMAX];
    const int m = blockIdx.x * 256 + threadIdx.x;
    const int c = blockIdx.y;
    const int t_begin = c * chunk;
    const int t_end = min(n, t_begin + chunk);
    float acc[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) acc[e] = 0.0f;
    for (int tb = t_begin; tb < t_end; tb += 64) {
        const int cnt = min(64, t_end - tb);
        __syncthreads();
        for (int i = threadIdx.x; i < 64 * EMAX; i += 256) {
            const int tt = i / EMAX, e = i % EMAX;
            dl[tt][e] = (tt < cnt && e < E) ? dlogits[(long long)(tb + tt) * E + e] : 0.0f;
        }
        __syncthreads();
        if (m < M) {
            for (int tt = 0; tt < cnt; ++tt) {
                const float xv = bf2f(x[(long long)(tb + tt) * ldx + m]);
#pragma unroll
                for (int e = 0; e < EMAX; ++e) acc[e] = fmaf(xv, dl[tt][e], acc[e]);
            }
        }
    }
    if (m < M)
        for (int e = 0; e < E; ++e) part[((long long)c * M + m) * E + e] = acc[e];
}

__global__ void sum_partials_kernel(const float* __restrict__ part, int chunks, long long len, float* __restrict__ out,
                                    int accumulate) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
        float s = accumulate ? out[i] : 0.0f;
        for (int c = 0; c < chunks; ++c) s += part[(long long)c * len + i];
        out[i] = s;
    }
}

// ------------------------------------------------------------------ host
template <int EMAX, int TPW>
static void launch_gate_fwd(const bf16* x, long long ldx, const bf16* wg, int n, int M, int E, int k, int* ei,
                            float* cw, float* probs, cudaStream_t s) {
    const int warps_needed = (n + TPW - 1) / TPW;
    int blocks = (warps_needed * 32 + kGateThreads - 1) / kGateThreads;
    const int max_blocks = kNumSMs * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    gate_fwd_kernel<EMAX, TPW><<<blocks, kGateThreads, 0, s>>>(x, ldx, wg, n, M, E, k, ei, cw, probs);
}

int gate_fwd(const void* x, long long ldx, const void* wg, int n, int M, int E, int k, int* expert_idx,
             float* combine_w, float* probs, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= E, "top_k (%d) exceeds number of experts (%d)", k, E);
    PARM_CHECK_ARG(E <= 32, "gate: at most 32 experts supported (got %d)", E);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate: embed (%d) and row stride must be multiples of 8", M);
    if (n == 0) return 0;
    auto X = reinterpret_cast<const bf16*>(x);
    auto W = reinterpret_cast<const bf16*>(wg);
    if (E <= 4)
        launch_gate_fwd<4, 4>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 8)
        launch_gate_fwd<8, 4>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 16)
        launch_gate_fwd<16, 2>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else
        launch_gate_fwd<32, 1>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    PARM_CHECK_LAUNCH("gate_fwd");
    return 0;
}

int gate_slots(const int* expert_idx, int n, int k, int E, int cap, int* slot_idx, int* slot_src, int* fill,
               cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= 8, "gate_slots: top_k must be in [1, 8] (got %d)", k);
    PARM_CHECK_ARG(E >= 1 && E <= kMaxExperts, "gate_slots: experts must be in [1, %d]", kMaxExperts);
    PARM_CHECK_ARG(cap >= 1, "gate_slots: capacity must be >= 1");
    gate_slots_kernel<<<1, kSlotThreads, 0, s>>>(expert_idx, n, k, E, cap, slot_idx, slot_src, fill);
    PARM_CHECK_LAUNCH("gate_slots");
    return 0;
}

size_t gate_wgrad_workspace(int n, int M, int E) {
    const int chunks = n < 64 ? 1 : (n / 64 < 128 ? n / 64 : 128);
    return (size_t)chunks * M * E * sizeof(float);
}

int gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, float* ws, size_t ws_bytes,
               float* dwg, int accumulate, cudaStream_t s) {
    PARM_CHECK_ARG(E <= 32, "gate_wgrad: at most 32 experts supported");
    const int chunks = n < 64 ? 1 : (n / 64 < 128 ? n / 64 : 128);
    PARM_CHECK_ARG(ws_bytes >= (size_t)chunks * M * E * sizeof(float), "gate_wgrad: workspace too small");
    const int chunk = (n + chunks - 1) / chunks;
    dim3 grid((M + 255) / 256, chunks);
    auto X = reinterpret_cast<const bf16*>(x);
    if (E <= 8)
        gate_wgrad_partial_kernel<8><<<grid, 256, 0, s>>>(X, ldx, dlogits, n, M, E, chunk, ws);
    else if (E <= 16)
        gate_wgrad_partial_kernel<16><<<grid, 256, 0, s>>>(X, ldx, dlogits, n, M, E, chunk, ws);
    else
        gate_wgrad_partial_kernel<32><<<grid, 256, 0, s>>>(X, ldx, dlogits, n, M, E, chunk, ws);
    PARM_CHECK_LAUNCH("gate_wgrad_partial");
    const long long len = (long long)M * E;
    int blocks = (int)((len + 255) / 256);
    if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
    sum_partials_kernel<<<blocks, 256, 0, s>>>(ws, chunks, len, dwg, accumulate);
    PARM_CHECK_LAUNCH("gate_wgrad_sum");
    return 0;
}

}  // namespace parm
