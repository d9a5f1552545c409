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
//
// Gate weights live on the device TRANSPOSED, wgT (E, M), so a lane's 8
// consecutive columns of one expert are one 16-byte load.
#include "common.cuh"

namespace parm {

constexpr int kGateThreads = 256;

// Warp-level reduce-scatter of 32 doubles: on return v[0] of lane L holds the
// warp-wide sum of input index L.  31 double shuffles instead of 5 x 32.
__device__ __forceinline__ double reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = upper ? v[i] : v[i + o];
            const double keep = upper ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// One warp handles TPW = 32 / EMAX tokens; after the reduce-scatter lane
// L = q * EMAX + e owns (token t0 + q, expert e): softmax max/sum over the
// EMAX-lane group by shuffles, one exp and one divide per lane, stable rank
// by comparing against the group's other lanes.
template <int EMAX>
__global__ void __launch_bounds__(kGateThreads) gate_fwd_kernel(const bf16* __restrict__ x, long long ldx,
                                                                 const bf16* __restrict__ wgT, int n, int M, int E,
                                                                 int k, int* __restrict__ expert_idx,
                                                                 float* __restrict__ combine_w,
                                                                 float* __restrict__ probs) {
    constexpr int TPW = 32 / EMAX;
    const int lane = threadIdx.x & 31;
    const int warp_global = (blockIdx.x * kGateThreads + threadIdx.x) >> 5;
    const int num_warps = (gridDim.x * kGateThreads) >> 5;
    for (int t0 = warp_global * TPW; t0 < n; t0 += num_warps * TPW) {
        double v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.0;
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
            for (int e = 0; e < EMAX; ++e) {
                if (e < E) {
                    float wv[8];
                    vec8_to_f32(ld_vec8(wgT + (long long)e * M + c), wv);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double w = (double)wv[u];
#pragma unroll
                        for (int q = 0; q < TPW; ++q) v[q * EMAX + e] = fma((double)xv[q][u], w, v[q * EMAX + e]);
                    }
                }
            }
        }
        const double logit = reduce_scatter32(v, lane);
        const int q = lane / EMAX;
        const int e = lane - q * EMAX;
        const int t = t0 + q;
        const bool valid = (e < E);
        double mx = valid ? logit : -INFINITY;
#pragma unroll
        for (int o = 1; o < EMAX; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double ex = valid ? exp(logit - mx) : 0.0;
        double sum = ex;
#pragma unroll
        for (int o = 1; o < EMAX; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double score = ex / sum;
        int rank = 0;
        const int base = q * EMAX;
#pragma unroll
        for (int i = 0; i < EMAX; ++i) {
            const double other = __shfl_sync(0xffffffffu, score, base + i);
            rank += (i < E) && ((other > score) || (other == score && i < e));
        }
        if (valid && t < n) {
            if (rank < k) {
                expert_idx[(long long)t * k + rank] = e;
                combine_w[(long long)t * k + rank] = (float)score;
            }
            if (probs) probs[(long long)t * E + e] = (float)score;
        }
    }
}

// Exclusive per-expert prefix count over tokens -> slots (single CTA, exact).
// Two passes: warp w owns a contiguous token range; pass 1 counts its picks
// per expert, a 32-entry scan per expert gives each warp its base, pass 2
// assigns slots in token order with ballot prefixes.
constexpr int kSlotThreads = 1024;
constexpr int kMaxExperts = 64;

template <int EMAX>
__global__ void __launch_bounds__(kSlotThreads) gate_slots_kernel(const int* __restrict__ expert_idx, int n, int k,
                                                                   int E, int cap, int* __restrict__ slot_idx,
                                                                   int* __restrict__ slot_src,
                                                                   int* __restrict__ fill) {
    __shared__ int warp_cnt[32][EMAX];
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int per = ((n + 32 * 32 - 1) / (32 * 32)) * 32;   // tokens per warp, multiple of 32
    const int t_begin = warp * per;
    const int t_end = min(n, t_begin + per);

    int cnt[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) cnt[e] = 0;
    for (int base = t_begin; base < t_end; base += 32) {
        const int t = base + lane;
        unsigned pick = 0;  // bitmask of experts picked by token t (E <= EMAX <= 32 here)
        if (t < t_end)
            for (int j = 0; j < k; ++j) pick |= 1u << expert_idx[(long long)t * k + j];
#pragma unroll
        for (int e = 0; e < EMAX; ++e) cnt[e] += __popc(__ballot_sync(0xffffffffu, (pick >> e) & 1u));
    }
    if (lane == 0)
#pragma unroll
        for (int e = 0; e < EMAX; ++e) warp_cnt[warp][e] = cnt[e];
    for (long long i = tid; i < (long long)E * cap; i += kSlotThreads) slot_src[i] = -1;
    __syncthreads();
    if (tid < E) {
        int acc = 0;
        for (int w = 0; w < 32; ++w) {
            const int c = warp_cnt[w][tid];
            warp_cnt[w][tid] = acc;
            acc += c;
        }
        fill[tid] = acc < cap ? acc : cap;
    }
    __syncthreads();
    int run[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; ++e) run[e] = warp_cnt[warp][e];
    for (int base = t_begin; base < t_end; base += 32) {
        const int t = base + lane;
        int ex[8];
        unsigned pick = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            ex[j] = (t < t_end && j < k) ? expert_idx[(long long)t * k + j] : -1;
            if (ex[j] >= 0) pick |= 1u << ex[j];
        }
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            const unsigned b = __ballot_sync(0xffffffffu, (pick >> e) & 1u);
            if ((pick >> e) & 1u) {
                const int slot = run[e] + __popc(b & lt_mask);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (ex[j] == e) {
                        if (slot < cap) {
                            slot_idx[(long long)t * k + j] = slot;
                            slot_src[(long long)e * cap + slot] = t * k + j;
                        } else {
                            slot_idx[(long long)t * k + j] = -1;
                        }
                    }
                }
            }
            run[e] += __popc(b);
        }
    }
}

// dWg^T partials: part[c][e][m] = sum_{t in chunk c} dlogits[t][e] * x[t][m].
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
        for (int e = 0; e < E; ++e) part[((long long)c * E + e) * M + m] = acc[e];
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
template <int EMAX>
static void launch_gate_fwd(const bf16* x, long long ldx, const bf16* wgT, int n, int M, int E, int k, int* ei,
                            float* cw, float* probs, cudaStream_t s) {
    constexpr int TPW = 32 / EMAX;
    const int warps_needed = (n + TPW - 1) / TPW;
    int blocks = (warps_needed * 32 + kGateThreads - 1) / kGateThreads;
    const int max_blocks = kNumSMs * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    gate_fwd_kernel<EMAX><<<blocks, kGateThreads, 0, s>>>(x, ldx, wgT, n, M, E, k, ei, cw, probs);
}

int gate_fwd(const void* x, long long ldx, const void* wgT, int n, int M, int E, int k, int* expert_idx,
             float* combine_w, float* probs, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= E, "top_k (%d) exceeds number of experts (%d)", k, E);
    PARM_CHECK_ARG(E <= 32, "gate: at most 32 experts supported (got %d)", E);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate: embed (%d) and row stride must be multiples of 8", M);
    if (n == 0) return 0;
    auto X = reinterpret_cast<const bf16*>(x);
    auto W = reinterpret_cast<const bf16*>(wgT);
    if (E <= 2)
        launch_gate_fwd<2>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 4)
        launch_gate_fwd<4>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 8)
        launch_gate_fwd<8>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else if (E <= 16)
        launch_gate_fwd<16>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    else
        launch_gate_fwd<32>(X, ldx, W, n, M, E, k, expert_idx, combine_w, probs, s);
    PARM_CHECK_LAUNCH("gate_fwd");
    return 0;
}

int gate_slots(const int* expert_idx, int n, int k, int E, int cap, int* slot_idx, int* slot_src, int* fill,
               cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= 8, "gate_slots: top_k must be in [1, 8] (got %d)", k);
    PARM_CHECK_ARG(E >= 1 && E <= 32, "gate_slots: experts must be in [1, 32]");
    PARM_CHECK_ARG(cap >= 1, "gate_slots: capacity must be >= 1");
    if (E <= 8)
        gate_slots_kernel<8><<<1, kSlotThreads, 0, s>>>(expert_idx, n, k, E, cap, slot_idx, slot_src, fill);
    else
        gate_slots_kernel<32><<<1, kSlotThreads, 0, s>>>(expert_idx, n, k, E, cap, slot_idx, slot_src, fill);
    PARM_CHECK_LAUNCH("gate_slots");
    return 0;
}

size_t gate_wgrad_workspace(int n, int M, int E) {
    const int chunks = n < 64 ? 1 : (n / 64 < 128 ? n / 64 : 128);
    return (size_t)chunks * M * E * sizeof(float);
}

int gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, float* ws, size_t ws_bytes,
               float* dwgT, int accumulate, cudaStream_t s) {
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
    sum_partials_kernel<<<blocks, 256, 0, s>>>(ws, chunks, len, dwgT, accumulate);
    PARM_CHECK_LAUNCH("gate_wgrad_sum");
    return 0;
}

}  // namespace parm
