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
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace parm {

constexpr int kGateThreads = 128;
constexpr int kGateChunks = 4;   // 16-B x chunks per lane per 1024-column group

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

// One warp handles TPW = 32 / EMAX tokens; every x load of a 1024-column group
// of all TPW tokens is issued before the f64 FMAs (memory-level parallelism),
// and each Wg^T vector is reused across the TPW tokens.  After the
// reduce-scatter lane L = q * EMAX + e owns (token t0 + q, expert e): softmax
// max/sum over the EMAX-lane group by shuffles, one exp and one divide per
// lane, stable rank against the group's other lanes.
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
        for (int g0 = 0; g0 < M; g0 += kGateChunks * 256) {
            int4 xb[TPW][kGateChunks];
#pragma unroll
            for (int q = 0; q < TPW; ++q)
#pragma unroll
                for (int i = 0; i < kGateChunks; ++i) {
                    const int c = g0 + lane * 8 + i * 256;
                    xb[q][i] = (t0 + q < n && c < M)
                                   ? __ldg(reinterpret_cast<const int4*>(x + (long long)(t0 + q) * ldx + c))
                                   : make_int4(0, 0, 0, 0);
                }
#pragma unroll
            for (int i = 0; i < kGateChunks; ++i) {
                const int c = g0 + lane * 8 + i * 256;
                if (c >= M) break;
                float xv[TPW][8];
#pragma unroll
                for (int q = 0; q < TPW; ++q) {
                    Vec8 t8;
                    *reinterpret_cast<int4*>(&t8) = xb[q][i];
                    vec8_to_f32(t8, xv[q]);
                }
#pragma unroll
                for (int u = 0; u < 8; u += 2) {
                    double xd[TPW][2];
#pragma unroll
                    for (int q = 0; q < TPW; ++q) {
                        xd[q][0] = (double)xv[q][u];
                        xd[q][1] = (double)xv[q][u + 1];
                    }
#pragma unroll
                    for (int e = 0; e < EMAX; ++e) {
                        if (e < E) {   // two bf16 gate weights, widened exactly to f64
                            const uint32_t w2 = __ldg(reinterpret_cast<const uint32_t*>(wgT + (long long)e * M + c + u));
                            const double w0 = (double)__uint_as_float(w2 << 16);
                            const double w1 = (double)__uint_as_float(w2 & 0xFFFF0000u);
#pragma unroll
                            for (int q = 0; q < TPW; ++q) {
                                v[q * EMAX + e] = fma(xd[q][0], w0, v[q * EMAX + e]);
                                v[q * EMAX + e] = fma(xd[q][1], w1, v[q * EMAX + e]);
                            }
                        }
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

// ------------------------------------------------------------------ tensor-core gate
// Logits on the tensor cores with a certified error bound (the "fp32 + tie audit" gate):
//   * mma.sync m16n8k16 bf16 -> f32: A = Wg^T (16 experts x 16 columns, from shared memory),
//     B = x^T (16 columns x 8 tokens, straight from HBM), D = 16 experts x 8 tokens.  Every
//     bf16 x bf16 product is exact; the tensor core sums a 32-column chunk (two chained MMAs
//     from a zero accumulator) in f32, and the chunk sums are added in f64.
//   * A second MMA pair over |Wg| and |x| gives S = sum_i |x_i w_ie| per (token, expert), so
//     |logit_gpu - logit_exact| <= kGateEps * S (kGateEps = 2^-17 bounds the f32 rounding of a
//     32-product chunk, 64x the one-ulp error; tools/probes/gate_err_probe.py measures the
//     observed ratio on adversarial data).
//   * Audit: a token whose picks are not separated from each other or from the best unpicked
//     expert by more than the two bounds is recomputed exactly in f64 (bf16 products exact,
//     fixed summation order -- the same semantics as the oracle's f64 dot products, so exact
//     ties still go to the lower expert), then ranked again.  Every other token's ranking is
//     certified equal to the exact one, hence to the oracle's argsort of f64 scores.
//   * k-index permutation: lane (g, q) loads 8 consecutive bf16 (one 16-byte load) of
//     x row g and of Wg^T rows g, g + 8 at column 32j + 8q; the first MMA takes words 0-1
//     (logical k = 2q, 2q+1, 2q+8, 2q+9), the second words 2-3.  A dot product only needs the
//     same permutation on both operands.
// Scores (softmax in f64 of these logits) differ from the oracle's by the logit error, ~1e-7
// relative for typical inputs.
constexpr double kGateEps = 1.0 / 131072.0;   // 2^-17
constexpr int kGmRJ = 8;                      // 32-column groups per load round (8 x 16-B loads in flight / lane)
constexpr int kGmMaxPairs = 7;                // warp pairs per CTA (448 threads: <= 146 registers)

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Per warp pair (one 8-token tile): the two column halves' partial sums, then the tile's logits,
// scores, bounds and ranks.
template <int NM>
struct GateTile {
    double part[2][8][16 * NM];
    float bpart[2][8][16 * NM];
    double lg[8][16 * NM];
    double sc[8][16 * NM];
    float bd[8][16 * NM];
    int rk[8][16 * NM];
};

// Softmax + stable top-k of the 4 tokens 4h..4h+3 of the tile: lane (t = lane / 8, r = lane % 8)
// owns experts r, r + 8, ...
//   EXACT = false (tensor-core logits): rank by the logits (ties -> lower expert) and return the
//     mask of tokens (bit t) whose picks the bounds do not separate from every other expert --
//     for the others this ranking is certified to be the exact one; scores in f32 math.
//   EXACT = true (the recomputed exact logits): f64 softmax and the stable ranking of the f64
//     scores, exactly the oracle's argsort(-scores, kind="stable").
template <int NM, bool EXACT>
__device__ __forceinline__ unsigned gate_rank4(GateTile<NM>& s, int lane, int h, int E, int k, int (&rank)[2 * NM]) {
    constexpr int EP = 16 * NM, U = EP / 8;
    const int t = 4 * h + (lane >> 3), r = lane & 7;
    double mx = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (r + 8 * u < E) mx = fmax(mx, s.lg[t][r + 8 * u]);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (EXACT) {
        double ex[U];
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ex[u] = (r + 8 * u < E) ? exp(s.lg[t][r + 8 * u] - mx) : 0.0;
            sum += ex[u];
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (r + 8 * u < E) s.sc[t][r + 8 * u] = ex[u] / sum;
    } else {
        float ex[U];
        float sum = 0.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ex[u] = (r + 8 * u < E) ? expf((float)(s.lg[t][r + 8 * u] - mx)) : 0.0f;
            sum += ex[u];
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (r + 8 * u < E) s.sc[t][r + 8 * u] = (double)(ex[u] / sum);
    }
    __syncwarp();
    bool unsure = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int e = r + 8 * u;
        rank[u] = EP;
        if (e >= E) continue;
        const double ke = EXACT ? s.sc[t][e] : s.lg[t][e];
        int rk = 0;
#pragma unroll
        for (int e2 = 0; e2 < EP; ++e2) {   // compile-time trip count: the shared loads pipeline
            if (e2 >= E) break;
            const double ko = EXACT ? s.sc[t][e2] : s.lg[t][e2];
            rk += (ko > ke) || (ko == ke && e2 < e);
        }
        rank[u] = rk;
        if (!EXACT && rk < k) {   // a pick must be separated from every other expert by the two bounds
            const double be = (double)s.bd[t][e];
#pragma unroll
            for (int e2 = 0; e2 < EP; ++e2) {   // (equal logits included: |diff| = 0)
                if (e2 >= E) break;
                unsure |= e2 != e && fabs(ke - s.lg[t][e2]) <= be + (double)s.bd[t][e2];
            }
        }
    }
    const unsigned b = __ballot_sync(0xffffffffu, unsure);
    unsigned tokens = 0;
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) tokens |= ((b >> (8 * tt)) & 0xFFu) ? (1u << tt) : 0u;
    return tokens;
}

#ifdef PARM_GATE_TRACE   // phase timestamps per CTA (tools/probes/gate_trace.py; variant builds only)
__device__ unsigned long long g_gate_trace[kNumSMs * 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GATE_MARK(i) \
    if (threadIdx.x == 0 && blockIdx.x < kNumSMs) g_gate_trace[blockIdx.x * 8 + (i)] = gtime()
#else
#define GATE_MARK(i)
#endif

__device__ __forceinline__ void pair_sync(int pw) { asm volatile("bar.sync %0, 64;" ::"r"(1 + pw) : "memory"); }

// One warp PAIR per 8-token tile: warp h of the pair sums column groups [h nj/2, (h+1) nj/2)
// (more warps in flight per SM than one warp per tile: the kernel is latency-bound), the
// partials meet in shared memory in a fixed order, and each warp ranks 4 of the tile's tokens.
template <int NM>
__global__ void __launch_bounds__(64 * kGmMaxPairs) gate_fwd_mma_kernel(const bf16* __restrict__ x, long long ldx,
                                                                        const bf16* __restrict__ wg, int n, int M,
                                                                        int E, int k, int* __restrict__ expert_idx,
                                                                        float* __restrict__ combine_w,
                                                                        float* __restrict__ probs,
                                                                        int* __restrict__ counts) {
    constexpr int EP = 16 * NM, U = EP / 8;
    extern __shared__ __align__(16) unsigned char smem[];
    const int rowb = 2 * M + 64;   // staged Wg^T row: 64-byte pad spreads the 8 g-rows over all banks
    const size_t absoff = (size_t)EP * rowb;   // |Wg^T| rows follow the Wg^T rows
    const int npairs = blockDim.x >> 6;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pw = warp >> 1, h = warp & 1;
    const int g = lane >> 2, q = lane & 3;
    GateTile<NM>& s = reinterpret_cast<GateTile<NM>*>(smem + 2 * absoff)[pw];
    const int tiles = (n + 7) / 8;
    const int nj = M / 32, nj0 = nj / 2;
    const int jb = h ? nj0 : 0, njh = h ? nj - nj0 : nj0;   // this warp's column groups
    const int rounds = (njh + kGmRJ - 1) / kGmRJ;
    int tile = blockIdx.x * npairs + pw;
    const int stride = gridDim.x * npairs;
    GATE_MARK(0);

    // x loads are unconditional (rows clamped to n - 1, groups to the half's last; the extra rows
    // and groups are never used), so no select waits on a load right after it is issued
    int4 bufA[kGmRJ], bufB[kGmRJ];
    auto load_round = [&](int4 (&dst)[kGmRJ], int tl, int rd) {
        const bf16* src = x + (long long)min(tl * 8 + g, n - 1) * ldx + 8 * q + 32 * jb;
#pragma unroll
        for (int jj = 0; jj < kGmRJ; ++jj)
            dst[jj] = __ldg(reinterpret_cast<const int4*>(src + 32 * min(rd * kGmRJ + jj, njh - 1)));
    };
    if (tile < tiles) {   // the first tile's first two rounds in flight before the Wg staging barrier
        load_round(bufA, tile, 0);
        if (rounds > 1) load_round(bufB, tile, 1);
    }

    // Wg^T (E, M) -> shared rows 0..EP-1 (rows >= E zero), and |Wg^T| at absoff (the bound's operand),
    // four 16-byte loads in flight per thread
    constexpr int kU = 4;   // (the first tile's x rounds are already live in registers)
    const int c8n = M / 8;
    const int units = EP * c8n;
    for (int u0 = 0; u0 < units; u0 += kU * blockDim.x) {
        int4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = u0 + u * blockDim.x + threadIdx.x;
            const int e = i / c8n;
            v[u] = (i < units && e < E) ? __ldg(reinterpret_cast<const int4*>(wg) + i) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int i = u0 + u * blockDim.x + threadIdx.x;
            const int e = i / c8n, c8 = i - e * c8n;
            if (i < units) {
                unsigned char* dst = smem + (size_t)e * rowb + c8 * 16;
                *reinterpret_cast<int4*>(dst) = v[u];
                *reinterpret_cast<int4*>(dst + absoff) =
                    make_int4(v[u].x & 0x7FFF7FFF, v[u].y & 0x7FFF7FFF, v[u].z & 0x7FFF7FFF, v[u].w & 0x7FFF7FFF);
            }
        }
    }
    __syncthreads();
    GATE_MARK(1);

    __shared__ int s_nflag[2];          // uncertified tokens of this round (parity double buffer)
    __shared__ int s_ftok[2 * kGmMaxPairs * 4];
    __shared__ double s_red[64][8];     // per-warp partial exact logits (<= 14 warps x 8 experts; 64 >= warps)
    if (threadIdx.x == 0) s_nflag[0] = s_nflag[1] = 0;
    __syncthreads();
    bool first_tile = true;
    int parity = 0;
    // CTA-uniform rounds (every pair of the CTA takes part in the exact-path barriers of each round)
    for (int base = blockIdx.x * npairs; base < tiles; base += stride, parity ^= 1) {
        tile = base + pw;
        const bool active = tile < tiles;
        unsigned redo = 0;
        int rank[U];
        const int t0 = tile * 8;
        if (active) {
        // two |.| accumulator chains (by group parity): the HMMA chain is the long dependency
        double acc[NM][4];
        float dab[2][NM][4];
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc[m][i] = 0.0;
                dab[0][m][i] = dab[1][m][i] = 0.0f;
            }
        auto compute = [&](const int4 (&cur)[kGmRJ], int rd) {
#pragma unroll
            for (int jj = 0; jj < kGmRJ; ++jj) {
                if (rd * kGmRJ + jj >= njh) break;
                const int j = jb + rd * kGmRJ + jj;
                const uint32_t xw[4] = {(uint32_t)cur[jj].x, (uint32_t)cur[jj].y, (uint32_t)cur[jj].z,
                                        (uint32_t)cur[jj].w};
                uint32_t xa[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) xa[w] = xw[w] & 0x7FFF7FFFu;
#pragma unroll
                for (int m = 0; m < NM; ++m) {
                    const unsigned char* ra = smem + (size_t)(16 * m + g) * rowb + 64 * j + 16 * q;
                    const unsigned char* rb = ra + 8 * (size_t)rowb;
                    const uint4 wa = *reinterpret_cast<const uint4*>(ra);
                    const uint4 wb = *reinterpret_cast<const uint4*>(rb);
                    float d[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                    mma_bf16_16816(d, wa.x, wb.x, wa.y, wb.y, xw[0], xw[1]);
                    mma_bf16_16816(d, wa.z, wb.z, wa.w, wb.w, xw[2], xw[3]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[m][i] += (double)d[i];
                    const uint4 va = *reinterpret_cast<const uint4*>(ra + absoff);
                    const uint4 vb = *reinterpret_cast<const uint4*>(rb + absoff);
                    mma_bf16_16816(dab[jj & 1][m], va.x, vb.x, va.y, vb.y, xa[0], xa[1]);
                    mma_bf16_16816(dab[jj & 1][m], va.z, vb.z, va.w, vb.w, xa[2], xa[3]);
                }
            }
        };
        if (!first_tile) {   // (the first tile's two rounds were issued before the staging barrier)
            load_round(bufA, tile, 0);
            if (rounds > 1) load_round(bufB, tile, 1);
        }
        for (int rd = 0; rd < rounds; rd += 2) {   // bufA holds round rd, bufB round rd + 1: ping-pong
            compute(bufA, rd);
            if (rd + 2 < rounds) load_round(bufA, tile, rd + 2);
            if (rd + 1 < rounds) {
                compute(bufB, rd + 1);
                if (rd + 3 < rounds) load_round(bufB, tile, rd + 3);
            }
        }
        first_tile = false;
        GATE_MARK(2);
        // D fragment: (expert 16m + g + 8 (i >> 1), token 2q + (i & 1))
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int e = 16 * m + g + 8 * (i >> 1), tl = 2 * q + (i & 1);
                s.part[h][tl][e] = acc[m][i];
                s.bpart[h][tl][e] = dab[0][m][i] + dab[1][m][i];
            }
        pair_sync(pw);
        {   // this warp's 4 tokens: halves summed in a fixed order (deterministic)
            const int tl = 4 * h + (lane >> 3), r = lane & 7;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = r + 8 * u;
                s.lg[tl][e] = s.part[0][tl][e] + s.part[1][tl][e];
                // the f32 sums of |products| are themselves rounded: 2^-10 covers it many times over
                s.bd[tl][e] = (float)(kGateEps * ((double)s.bpart[0][tl][e] + (double)s.bpart[1][tl][e]) *
                                      (1.0 + 1.0 / 1024.0));
            }
        }
        __syncwarp();
        const int live = min(8, n - t0) - 4 * h;                  // this warp's real tokens (may be <= 0)
        GATE_MARK(3);
        redo = gate_rank4<NM, false>(s, lane, h, E, k, rank);
        GATE_MARK(4);
        redo &= live >= 4 ? 0xFu : (live > 0 ? (1u << live) - 1u : 0u);
        if (lane == 0)
            for (unsigned rm = redo; rm; rm &= rm - 1) s_ftok[atomicAdd(&s_nflag[parity], 1)] = (pw << 3) | (4 * h + __ffs(rm) - 1);
        }   // active
        if (threadIdx.x == 0) s_nflag[parity ^ 1] = 0;            // next round's list (see DESIGN: parity)
        __syncthreads();
        const int nflag = s_nflag[parity];
        // Exact f64 logits of the uncertified tokens (rare), by the whole CTA: thread c handles the
        // 8-column chunks c, c + blockDim, ... in order, warps reduce by a fixed shuffle tree, then the
        // warp partials are added in warp order -- the same arithmetic for every expert, so equal gate
        // columns give equal logits (exact ties, lower expert first).
        for (int f = 0; f < nflag; ++f) {
            const int fq = s_ftok[f] >> 3, ftl = s_ftok[f] & 7;
            GateTile<NM>& fs = reinterpret_cast<GateTile<NM>*>(smem + 2 * absoff)[fq];
            const bf16* xr = x + (long long)((base + fq) * 8 + ftl) * ldx;
            for (int e0 = 0; e0 < E; e0 += 8) {
                double pe[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                for (int c = 8 * threadIdx.x; c < M; c += 8 * blockDim.x) {
                    const int4 xv = __ldg(reinterpret_cast<const int4*>(xr + c));
                    const uint32_t xs[4] = {(uint32_t)xv.x, (uint32_t)xv.y, (uint32_t)xv.z, (uint32_t)xv.w};
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (e0 + u >= E) break;
                        const int4 wv = *reinterpret_cast<const int4*>(smem + (size_t)(e0 + u) * rowb + 2 * c);
                        const uint32_t ws[4] = {(uint32_t)wv.x, (uint32_t)wv.y, (uint32_t)wv.z, (uint32_t)wv.w};
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            pe[u] = fma((double)__uint_as_float(xs[w] << 16), (double)__uint_as_float(ws[w] << 16),
                                        pe[u]);
                            pe[u] = fma((double)__uint_as_float(xs[w] & 0xFFFF0000u),
                                        (double)__uint_as_float(ws[w] & 0xFFFF0000u), pe[u]);
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
                    for (int u = 0; u < 8; ++u) pe[u] += __shfl_down_sync(0xffffffffu, pe[u], o);
                if (lane == 0)
#pragma unroll
                    for (int u = 0; u < 8; ++u) s_red[warp][u] = pe[u];
                __syncthreads();
                if (threadIdx.x < 8 && e0 + threadIdx.x < E) {
                    double v = 0.0;
                    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += s_red[w][threadIdx.x];
                    fs.lg[ftl][e0 + threadIdx.x] = v;
                }
                __syncthreads();
            }
        }
        if (active) {
        if (redo) {   // the recomputed tokens, ranked exactly (the certified ones keep their ranking)
            int rank2[U];
            gate_rank4<NM, true>(s, lane, h, E, k, rank2);
            if ((redo >> (lane >> 3)) & 1u)
#pragma unroll
                for (int u = 0; u < U; ++u) rank[u] = rank2[u];
        }
        // outputs: lane (t, r) owns experts r + 8u of token t0 + 4h + t
        const int tl = 4 * h + (lane >> 3), r = lane & 7;
        const bool tok = t0 + tl < n;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = r + 8 * u;
            s.rk[tl][e] = (tok && e < E) ? rank[u] : EP;
            if (!tok || e >= E) continue;
            const long long tt = t0 + tl;
            const float sc = (float)s.sc[tl][e];
            if (rank[u] < k) {
                expert_idx[tt * k + rank[u]] = e;
                combine_w[tt * k + rank[u]] = sc;
            }
            if (probs) probs[tt * E + e] = sc;
        }
        pair_sync(pw);
        if (counts != nullptr && h == 0 && lane < E) {   // per-tile pick counts of each expert
            int c = 0;
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) c += s.rk[tt][lane] < k;
            counts[(long long)tile * E + lane] = c;
        }
        GATE_MARK(5);
        }   // active
    }
}

#ifdef PARM_GATE_TRACE
extern "C" int parm_debug_gate_trace(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_gate_trace, sizeof(g_gate_trace));
}
#endif

namespace gring {   // bulk-copy helpers (same protocol as permute.cu's rings)
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "GATE_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GATE_WAIT;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
}  // namespace gring


// dWg^T partials: part[c][e][m] = sum_{t in token range c} dlogits[t][e] * x[t][m].
// One CTA per SM over a contiguous token range (~n/148 tokens): the range's rows stream into
// a shared-memory ring with cp.async.bulk (one copy per stage when rows are contiguous) --
// every byte of x requested at kernel start, no per-thread load latency on the critical
// path -- and the range's logit gradients sit in shared memory (broadcast reads).  Thread =
// 4 consecutive columns of a 1024-column block; f32 accumulation in token order (FFMA2); the
// partials are summed in a fixed order (deterministic) by the same launch after a grid barrier
// when every CTA is resident (cooperative launch), else by sum_partials_kernel.
constexpr int kWgThreads = 256;
constexpr int kWgBlock = kWgThreads * 4;        // columns per pass
constexpr int kWgMaxTok = 256;                  // tokens per CTA (host: grid >= n / 256)
constexpr int kWgStages = 3;
constexpr int kWgStageBytes = 64 * 1024;

// Two thread halves split each stage's rows (256 threads = 1024 columns each) and fold
// their sums through shared memory at the end: 16 warps per SM for latency hiding.
template <int EMAX, int NB>   // 4 columns x EMAX experts per thread for NB column blocks (M <= NB * 1024)
__global__ void __launch_bounds__(2 * kWgThreads) gate_wgrad_partial_kernel(const bf16* __restrict__ x, long long ldx,
                                                                        const float* __restrict__ dlogits, int n, int Mfull,
                                                                        int E, float* __restrict__ part,
                                                                        float* __restrict__ out, int accumulate,
                                                                        int* __restrict__ sync) {
    // blockIdx.y: this CTA's column slice [cbase, cbase + M) of the NB * 1024 columns it covers
    const int cbase = blockIdx.y * NB * kWgBlock;
    const int M = min(Mfull - cbase, NB * kWgBlock);
    x += cbase;
    __shared__ float sdl[kWgMaxTok * EMAX];
    __shared__ __align__(8) uint64_t bars[kWgStages];
    extern __shared__ __align__(128) unsigned char sx[];
    const int t0 = (int)((long long)n * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
    const int nt = t1 - t0;
    const int R = max(1, kWgStageBytes / (M * 2));           // token rows per stage
    const int nstage_items = (nt + R - 1) / R;
    const uint32_t bar0 = gring::saddr(bars);
    auto issue = [&](int it) {                               // thread 0: rows [it*R, ...) of the range
        const int r0 = it * R, rows = min(R, nt - r0);
        const uint32_t st = (uint32_t)(it % kWgStages);
        unsigned char* dst = sx + (size_t)st * kWgStageBytes;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        gring::bar_expect(bar0 + 8 * st, (uint32_t)(rows * M * 2));
        if (ldx == M && gridDim.y == 1) {
            gring::bulk_g2s(gring::saddr(dst), x + (long long)(t0 + r0) * ldx, rows * M * 2, bar0 + 8 * st);
        } else {
            for (int r = 0; r < rows; ++r)
                gring::bulk_g2s(gring::saddr(dst + (size_t)r * M * 2), x + (long long)(t0 + r0 + r) * ldx, M * 2,
                                bar0 + 8 * st);
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kWgStages; ++s) gring::bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int it = 0; it < min(nstage_items, kWgStages); ++it) issue(it);
    }
    for (int i = threadIdx.x; i < nt * E; i += blockDim.x) {
        const int t = i / E, e = i - t * E;
        sdl[t * EMAX + e] = __ldg(dlogits + (long long)(t0 + t) * E + e);
    }
    __syncthreads();
    const int ncb = (M + kWgBlock - 1) / kWgBlock;
    const int half = threadIdx.x / kWgThreads, ht = threadIdx.x - half * kWgThreads;
    float acc[NB][EMAX][4];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[b][e][u] = 0.0f;
    for (int it = 0; it < nstage_items; ++it) {
        const uint32_t st = (uint32_t)(it % kWgStages);
#ifndef WG_V_NOWAIT
        gring::bar_wait(bar0 + 8 * st, (uint32_t)((it / kWgStages) & 1));
#endif
        const unsigned char* base = sx + (size_t)st * kWgStageBytes;
        const int r0 = it * R, rows = min(R, nt - r0);
#ifdef WG_V_NOCOMPUTE
        if (rows > 0) continue;
#endif
        for (int r = half; r < rows; r += 2) {
            const float* d = sdl + (r0 + r) * EMAX;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (b >= ncb) break;
                const int c = b * kWgBlock + ht * 4;
                if (c >= M) continue;
                const uint2 xv = *reinterpret_cast<const uint2*>(base + ((size_t)r * M + c) * 2);
                const float f0 = __uint_as_float(xv.x << 16), f1 = __uint_as_float(xv.x & 0xFFFF0000u);
                const float f2 = __uint_as_float(xv.y << 16), f3 = __uint_as_float(xv.y & 0xFFFF0000u);
#pragma unroll
                for (int e = 0; e < EMAX; ++e) {
                    const float w = d[e];            // experts >= E: never stored below
                    ffma2(acc[b][e][0], acc[b][e][1], f0, f1, w);
                    ffma2(acc[b][e][2], acc[b][e][3], f2, f3, w);
                }
            }
        }
        __syncthreads();                                     // stage consumed by every thread
        if (threadIdx.x == 0 && it + kWgStages < nstage_items) issue(it + kWgStages);
    }
    // fold the odd-row half into the even-row half (fixed order: deterministic), through the ring
    float4* fold = reinterpret_cast<float4*>(sx);              // every stage consumed: reuse the ring
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        if (b >= ncb) break;
        if (half == 1) {
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                fold[(b * EMAX + e) * kWgThreads + ht] = make_float4(acc[b][e][0], acc[b][e][1], acc[b][e][2], acc[b][e][3]);
        }
        __syncthreads();
        const int c = b * kWgBlock + ht * 4;
        if (half == 0 && c < M) {
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                if (e >= E) break;
                const float4 o = fold[(b * EMAX + e) * kWgThreads + ht];
                *reinterpret_cast<float4*>(part + ((long long)blockIdx.x * E + e) * Mfull + cbase + c) =
                    make_float4(acc[b][e][0] + o.x, acc[b][e][1] + o.y, acc[b][e][2] + o.z, acc[b][e][3] + o.w);
            }
        }
        __syncthreads();
    }
    if (sync == nullptr) return;   // partials only: the host launches sum_partials_kernel
    // ---- every CTA's partials stored (grid barrier: cooperative launch), then CTA i sums its
    //      1/nb slice of the E x M outputs over the gridDim.x partials in a fixed order
    //      (deterministic): lanes over outputs, warps over chunks w, w + 16, ..., warp sums in order
    const int nb = gridDim.x * gridDim.y;
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(sync, 1);
        const long long t_start = clock64();
        int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(sync) : "memory");
            if (v >= nb) break;
            __nanosleep(64);
            if (clock64() - t_start > (8ll << 30)) asm volatile("trap;");
        }
    }
    __syncthreads();
    const long long len = (long long)E * Mfull;
    const long long lo = len * id / nb, hi = len * (id + 1) / nb;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kRw = 2 * kWgThreads / 32;                   // 16 warps
    constexpr int kRc = (kNumSMs + kRw - 1) / kRw;             // chunks per warp (gridDim.x <= kNumSMs here)
    float* red = reinterpret_cast<float*>(sx);                 // [kRw][64]
    const int chunks = gridDim.x;
    for (long long i0 = lo; i0 < hi; i0 += 64) {              // 64 outputs per pass, every load in flight
        float v[2][kRc];
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) {
            const long long i = i0 + 32 * g2 + lane;
#pragma unroll
            for (int r = 0; r < kRc; ++r) {
                const int c = warp + kRw * r;
                v[g2][r] = (i < hi && c < chunks) ? __ldcg(part + (long long)c * len + i) : 0.0f;
            }
        }
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) {
            float sum = 0.0f;
#pragma unroll
            for (int r = 0; r < kRc; ++r) sum += v[g2][r];
            red[warp * 64 + 32 * g2 + lane] = sum;
        }
        __syncthreads();
        if (warp < 2) {
            const long long i = i0 + 32 * warp + lane;
            if (i < hi) {
                float tot = red[32 * warp + lane];
#pragma unroll
                for (int w = 1; w < kRw; ++w) tot += red[w * 64 + 32 * warp + lane];
                out[i] = accumulate ? out[i] + tot : tot;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && atomicAdd(sync + 1, 1) == nb - 1) {   // last CTA out: counters back to zero
        sync[0] = 0;
        sync[1] = 0;
        __threadfence();
    }
}

// out[i] (+)= sum_c part[c][i]: a CTA owns 32 consecutive outputs; warp w sums
// chunks w, w + 8, ... with all its loads in flight, then the eight warp sums
// are added in a fixed order (deterministic).
__global__ void __launch_bounds__(256) sum_partials_kernel(const float* __restrict__ part, int chunks, long long len,
                                                           float* __restrict__ out, int accumulate) {
    __shared__ float ws[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * 32 + lane;
    float s = 0.0f;
    if (i < len) {   // warp w sums chunks w, w + 8, ...: 24 loads in flight per batch, added in chunk order
        for (int c0 = warp; c0 < chunks; c0 += 8 * 24) {
            float v[24];
#pragma unroll
            for (int r = 0; r < 24; ++r) {
                const int c = c0 + 8 * r;
                v[r] = c < chunks ? __ldg(part + (long long)c * len + i) : 0.0f;
            }
#pragma unroll
            for (int r = 0; r < 24; ++r) s += v[r];
        }
    }
    ws[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < len) {
        float tot = ws[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) tot += ws[w][lane];
        out[i] = accumulate ? out[i] + tot : tot;
    }
}

// Per-8-token-tile pick counts from expert_idx (the fallback gate does not emit them).
__global__ void tile_count_kernel(const int* __restrict__ expert_idx, int n, int k, int E, int* __restrict__ counts) {
    const int tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (tile * 8 >= n) return;
    int c = 0;   // lane e counts picks of expert e among the tile's tokens
    for (int i = 0; i < 8 && tile * 8 + i < n; ++i)
        for (int j = 0; j < k; ++j) c += __ldg(expert_idx + (long long)(tile * 8 + i) * k + j) == lane;
    if (lane < E) counts[(long long)tile * E + lane] = c;
}
// ------------------------------------------------------------------ host
template <int EMAX>
static void launch_gate_fwd(const bf16* x, long long ldx, const bf16* wgT, int n, int M, int E, int k, int* ei,
                            float* cw, float* probs, cudaStream_t s) {
    constexpr int TPW = 32 / EMAX;
    const int warps_needed = (n + TPW - 1) / TPW;
    int blocks = (warps_needed * 32 + kGateThreads - 1) / kGateThreads;
    const int max_blocks = kNumSMs * 16;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    launch_k(gate_fwd_kernel<EMAX>, blocks, kGateThreads, 0, s, x, ldx, wgT, n, M, E, k, ei, cw, probs);
}

size_t gate_counts_bytes(int n, int E) { return (size_t)((n + 7) / 8) * E * sizeof(int); }

// Tensor-core gate configuration for (n, M, E): warp pairs per CTA and shared memory, or false.
static bool gate_mma_config(int n, int M, int E, int& pairs, size_t& smem) {
    if (M % 64 != 0 || E > 32) return false;
    const int NM = E > 16 ? 2 : 1;
    const size_t tile = NM == 1 ? sizeof(GateTile<1>) : sizeof(GateTile<2>);
    const int tiles = (n + 7) / 8;
    // pairs per CTA (one 8-token tile each at a time): fewest tiles on the busiest SM, most pairs on ties
    pairs = kGmMaxPairs;
    long long best = -1;
    for (int w = kGmMaxPairs; w >= 2; --w) {
        const long long ctas = (tiles + w - 1) / w;
        const long long load = (ctas + kNumSMs - 1) / kNumSMs * w;
        if (best < 0 || load < best) {
            best = load;
            pairs = w;
        }
    }
    smem = (size_t)2 * 16 * NM * (2 * M + 64) + (size_t)pairs * tile;   // Wg^T, |Wg^T|, per-pair scratch
    return smem <= 227 * 1024;
}

int gate_fwd(const void* x, long long ldx, const void* wgT, int n, int M, int E, int k, int* expert_idx,
             float* combine_w, float* probs, int* counts, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= E, "top_k (%d) exceeds number of experts (%d)", k, E);
    PARM_CHECK_ARG(E <= 32, "gate: at most 32 experts supported (got %d)", E);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate: embed (%d) and row stride must be multiples of 8", M);
    if (n == 0) return 0;
    auto X = reinterpret_cast<const bf16*>(x);
    auto W = reinterpret_cast<const bf16*>(wgT);
    int pairs = 0;
    size_t smem = 0;
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(wgT) & 15) == 0 &&
        gate_mma_config(n, M, E, pairs, smem)) {
        const int tiles = (n + 7) / 8;
        const int blocks = (int)std::min<long long>((tiles + pairs - 1) / pairs, kNumSMs);
        if (E <= 16) {
            cudaFuncSetAttribute(gate_fwd_mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(gate_fwd_mma_kernel<1>, blocks, pairs * 64, smem, s, X, ldx, W, n, M, E, k, expert_idx,
                     combine_w, probs, counts);
        } else {
            cudaFuncSetAttribute(gate_fwd_mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(gate_fwd_mma_kernel<2>, blocks, pairs * 64, smem, s, X, ldx, W, n, M, E, k, expert_idx,
                     combine_w, probs, counts);
        }
        PARM_CHECK_LAUNCH("gate_fwd");
        return 0;
    }
    // shapes the tensor-core gate does not take (M % 64 != 0, unaligned rows, very wide M): f64 FMA gate
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
    if (counts != nullptr) {
        const int tiles = (n + 7) / 8;
        launch_k(tile_count_kernel, (tiles + 7) / 8, 256, 0, s, expert_idx, n, k, E, counts);
        PARM_CHECK_LAUNCH("gate_fwd(counts)");
    }
    return 0;
}

static int gate_wgrad_grid(int n) {
    int g = std::min(kNumSMs, std::max(1, (n + 31) / 32));        // >= 32 tokens per CTA when n is small
    return std::max(g, (n + kWgMaxTok - 1) / kWgMaxTok);          // <= kWgMaxTok tokens per CTA
}

// Workspace: two barrier counters (16 bytes, zero before first use; the kernel leaves them zero)
// at a fixed offset -- calls with different n share one workspace -- then the partials.
constexpr size_t kWgSyncBytes = 16;

size_t gate_wgrad_workspace(int n, int M, int E) {
    return kWgSyncBytes + (size_t)gate_wgrad_grid(n) * M * E * sizeof(float);
}

int sum_chunks(const float* src, int chunks, long long len, float* out, int accumulate, cudaStream_t s) {
    PARM_CHECK_ARG(src != nullptr && out != nullptr && chunks >= 1 && len >= 0, "sum_chunks: bad arguments");
    if (len == 0) return 0;
    launch_k(sum_partials_kernel, (int)((len + 31) / 32), 256, 0, s, src, chunks, len, out, accumulate);
    PARM_CHECK_LAUNCH("sum_chunks");
    return 0;
}

int gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, float* ws, size_t ws_bytes,
               float* dwgT, int accumulate, cudaStream_t s) {
    PARM_CHECK_ARG(E <= 32, "gate_wgrad: at most 32 experts supported");
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0,
                   "gate_wgrad: embed (%d) must be a multiple of 8, rows 16-byte aligned", M);
    PARM_CHECK_ARG(ws_bytes >= gate_wgrad_workspace(n, M, E), "gate_wgrad: workspace too small");
    const long long len = (long long)M * E;
    if (n == 0) {
        if (!accumulate) cudaMemsetAsync(dwgT, 0, len * sizeof(float), s);
        return 0;
    }
    const int grid = gate_wgrad_grid(n);
    auto X = reinterpret_cast<const bf16*>(x);
    const int smem = kWgStages * kWgStageBytes;
    const int nb = (M + kWgBlock - 1) / kWgBlock;
    int* sync = reinterpret_cast<int*>(ws);
    float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kWgSyncBytes);
    bool fused = false;   // the sum in the same launch when every CTA fits at once (1 CTA per SM)
    // column slices of NBV * 1024 columns over grid.y (one slice unless M exceeds what a thread's
    // accumulators cover: 4096 columns for E <= 8, 2048 for E <= 16, 1024 for E <= 32)
#define PARM_WG_LAUNCH(EM, NBV)                                                                              \
    do {                                                                                                     \
        static bool attr = false;                                                                            \
        if (!attr) {                                                                                         \
            cudaFuncSetAttribute(gate_wgrad_partial_kernel<EM, NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 smem);                                                                      \
            attr = true;                                                                                     \
        }                                                                                                    \
        const dim3 gr(grid, (nb + (NBV) - 1) / (NBV));                                                       \
        if ((long long)gr.x * gr.y <= kNumSMs) {                                                             \
            fused = launch_coop(gate_wgrad_partial_kernel<EM, NBV>, gr, 2 * kWgThreads, smem, s, X, ldx, dlogits, \
                                n, M, E, part, dwgT, accumulate, sync) == cudaSuccess;                       \
            if (!fused) (void)cudaGetLastError();   /* not co-resident here: the two-launch form */          \
        }                                                                                                    \
        if (!fused)                                                                                          \
            launch_k(gate_wgrad_partial_kernel<EM, NBV>, gr, 2 * kWgThreads, smem, s, X, ldx, dlogits, n, M, E, part, \
                     (float*)nullptr, 0, (int*)nullptr);                                                     \
    } while (0)
    if (E <= 8 && nb == 1)
        PARM_WG_LAUNCH(8, 1);
    else if (E <= 8)
        PARM_WG_LAUNCH(8, 4);
    else if (E <= 16 && nb == 1)
        PARM_WG_LAUNCH(16, 1);
    else if (E <= 16)
        PARM_WG_LAUNCH(16, 2);
    else
        PARM_WG_LAUNCH(32, 1);
#undef PARM_WG_LAUNCH
    PARM_CHECK_LAUNCH("gate_wgrad_partial");
    if (!fused) {
        launch_k(sum_partials_kernel, (int)((len + 31) / 32), 256, 0, s, part, grid, len, dwgT, accumulate);
        PARM_CHECK_LAUNCH("gate_wgrad_sum");
    }
    return 0;
}

}  // namespace parm
