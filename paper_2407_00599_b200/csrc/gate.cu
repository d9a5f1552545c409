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

// ------------------------------------------------------------------ FP64 tensor-core gate
// mma.m8n8k4.f64 (DMMA): one instruction = 8 tokens x 8 experts x 4 columns of
// exact-product f64 FMAs.  Lane (g, q) = (lane / 4, lane % 4) supplies A[g][q] =
// x[token g][c_q] and B[q][g] = Wg[expert g][c_q]: the k index is the quad lane,
// mapped to a lane-dependent column (the same mapping for A and B, which is all a
// dot product needs).  Step u of 32-column group j uses column c_q = 32j + 8q + u,
// so a lane's 8 consecutive bf16 of x are one 16-byte shared-memory load.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Softmax + stable top-k of one token's logits held by a lane quad: lane
// (g, q) owns experts nt * 8 + 2q + h of token t (the DMMA C-fragment layout).
// Returns, per owned expert, whether it is one of the token's k picks.
template <int NT>
__device__ __forceinline__ void gate_topk_epilogue(double (&lg)[NT][2], int g, int q, int t, bool tok, int E, int k,
                                                   int* __restrict__ expert_idx, float* __restrict__ combine_w,
                                                   float* __restrict__ probs, bool (&pick)[NT][2]) {
    double sc[NT][2];
    double mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = lg[nt][h];
            if (nt * 8 + 2 * q + h < E) mx = fmax(mx, sc[nt][h]);
        }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    double sum = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = (nt * 8 + 2 * q + h < E) ? exp(sc[nt][h] - mx) : 0.0;
            sum += sc[nt][h];
        }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    int rank[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            sc[nt][h] = sc[nt][h] / sum;
            rank[nt][h] = 0;
        }
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int nt2 = 0; nt2 < NT; ++nt2)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const double other = __shfl_sync(0xffffffffu, sc[nt2][h2], (g << 2) | qq);
                const int e2 = nt2 * 8 + 2 * qq + h2;
                if (e2 >= E) continue;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int e = nt * 8 + 2 * q + h;
                        rank[nt][h] += (other > sc[nt][h]) || (other == sc[nt][h] && e2 < e);
                    }
            }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = nt * 8 + 2 * q + h;
            pick[nt][h] = tok && e < E && rank[nt][h] < k;
            if (!tok || e >= E) continue;
            if (rank[nt][h] < k) {
                expert_idx[(long long)t * k + rank[nt][h]] = e;
                combine_w[(long long)t * k + rank[nt][h]] = (float)sc[nt][h];
            }
            if (probs) probs[(long long)t * E + e] = (float)sc[nt][h];
        }
}

__device__ __forceinline__ double bf16_to_f64(uint32_t bits16) { return (double)__uint_as_float(bits16 << 16); }

// Exact f32 -> f64 widening of a bf16-valued f32 bit pattern with integer ops (no F2F on the
// DMMA operand path): sign | (exponent + 896) << 20 | mantissa << 13 in the high word, low word
// zero.  Zero keeps its sign; subnormals, infinities and NaNs take the conversion instruction.
__device__ __forceinline__ double bf16_bits_to_f64(uint32_t f) {
    const uint32_t mag = f & 0x7FFFFFFFu;
    const uint32_t ex = mag >> 23;
    uint32_t hi = (f & 0x80000000u) | (mag ? (mag >> 3) + 0x38000000u : 0u);
    if (__builtin_expect(ex == 0u && mag != 0u, 0) || __builtin_expect(ex == 0xFFu, 0))
        return (double)__uint_as_float(f);
    return __hiloint2double((int)hi, 0);
}

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

// One CTA per SM (persistent), wpc warps, each walking its own 8-token tiles.
//   * Wg^T (bf16 (E, M) in global) is converted once per CTA to f64 in shared memory,
//     lane-major: the double2 of lane l for (group j, n-tile nt, u-pair up) sits at
//     ((j * NT + nt) * 4 + up) * 32 + l, so every B-fragment load is a conflict-free
//     contiguous 512-byte warp access and carries two steps' operands.
//   * x arrives by cp.async.bulk into a per-warp ring of S stages (8 token rows x kGateCC
//     columns each, rows padded to 576 B so the quad lanes' 16-byte loads hit distinct
//     banks), issued S-1 items ahead: all of a warp's rows are in flight at once instead
//     of one dependent round trip per chunk.
//   * Two independent DMMA accumulator chains per warp (steps u even / odd).
//   * counts (nullable): per 8-token tile, how many of its tokens picked each expert --
//     the first pass of the exact slot scan, so the slot kernel needs no count pass.
constexpr int kGateCC = 256;                        // columns per ring stage
constexpr int kGateRow = kGateCC * 2 + 64;          // bytes per staged row (bank-spreading pad)
constexpr int kGateStage = 8 * kGateRow;            // one 8-token stage

template <int NT>
__global__ void __launch_bounds__(256, 1) gate_fwd_tc_kernel(const bf16* __restrict__ x, long long ldx,
                                                             const bf16* __restrict__ wg, int n, int M, int E, int k,
                                                             int S, int* __restrict__ expert_idx,
                                                             float* __restrict__ combine_w, float* __restrict__ probs,
                                                             int* __restrict__ counts) {
    extern __shared__ __align__(128) unsigned char smem[];
#ifdef GATE_V_EMPTY
    if (threadIdx.x < 1000000) return;
#endif
    const int wpc = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int ngroups = M / 32;
    double2* sw = reinterpret_cast<double2*>(smem);
    unsigned char* ring = smem + (size_t)ngroups * NT * 4 * 32 * sizeof(double2) + (size_t)warp * S * kGateStage;
    const uint32_t bar0 = gring::saddr(smem + (size_t)ngroups * NT * 4 * 32 * sizeof(double2) +
                                       (size_t)wpc * S * kGateStage) + warp * S * 8;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) gring::bar_init(bar0 + 8 * s);
#ifndef GATE_V_NOFENCE
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
    }
    __syncwarp();

    const int tiles = (n + 7) / 8;
    const int nch = (M + kGateCC - 1) / kGateCC;
    const int first = blockIdx.x * wpc + warp, stride = gridDim.x * wpc;
    const int my_tiles = first < tiles ? (tiles - 1 - first) / stride + 1 : 0;
    const int items = my_tiles * nch;
    auto issue = [&](int it) {          // lane 0: bulk copies of item it (tile it / nch, chunk it % nch)
#ifdef GATE_V_NOCOPY
        return;
#endif
        const int ti = it / nch, ch = it - ti * nch;
        const int t0 = (first + ti * stride) * 8;
        const int c0 = ch * kGateCC;
        const int cols = min(kGateCC, M - c0);
        const int rows = min(8, n - t0);
        const uint32_t st = (uint32_t)it % S;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        gring::bar_expect(bar0 + 8 * st, (uint32_t)(rows * cols * 2));
        for (int r = 0; r < rows; ++r)
            gring::bulk_g2s(gring::saddr(ring + st * kGateStage + r * kGateRow), x + (long long)(t0 + r) * ldx + c0,
                            cols * 2, bar0 + 8 * st);
    };
    // Wg^T -> f64 lane-major shared copy; experts >= E are zero.  Unit = one expert's 8
    // consecutive columns (one 16-byte load) = lane (e % 8, q)'s four double2 of one column
    // group.  The gate-weight loads are issued FIRST (every warp waits on them), then the x
    // copies stream in behind them while the weights are converted.
#ifndef GATE_V_NOWG
    const int units = NT * 8 * (M / 8);
#else
    const int units = 0;
#endif
    constexpr int U = 8;
    const int rounds = (units + U * blockDim.x - 1) / (U * blockDim.x);
    for (int rd = 0; rd < rounds; ++rd) {
        const int u0 = rd * U * blockDim.x;
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u0 + u * blockDim.x + threadIdx.x;
            const int e = i / (M / 8), c8 = i - e * (M / 8);
            v[u] = (i < units && e < E) ? __ldg(reinterpret_cast<const int4*>(wg + (long long)e * M) + c8)
                                        : make_int4(0, 0, 0, 0);
        }
        if (rd == 0 && lane == 0)
            for (int it = 0; it < min(items, S - 1); ++it) issue(it);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u0 + u * blockDim.x + threadIdx.x;
            if (i >= units) break;
            const int e = i / (M / 8), c8 = i - e * (M / 8);
            const int nt = e >> 3, l = ((e & 7) << 2) | (c8 & 3), j = c8 >> 2;
            const uint32_t w[4] = {(uint32_t)v[u].x, (uint32_t)v[u].y, (uint32_t)v[u].z, (uint32_t)v[u].w};
#pragma unroll
            for (int up = 0; up < 4; ++up)
                sw[((j * NT + nt) * 4 + up) * 32 + l] = make_double2(bf16_to_f64(w[up] & 0xFFFFu),
                                                                    bf16_to_f64(w[up] >> 16));
        }
    }
    if (rounds == 0 && lane == 0)
        for (int it = 0; it < min(items, S - 1); ++it) issue(it);
    __syncthreads();

    int it = 0;
    for (int ti = 0; ti < my_tiles; ++ti) {
        const int tile = first + ti * stride;
        double acc[4][NT][2];   // four independent DMMA chains (DMMA latency ~28 cycles, issue ~16 per SMSP)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
        for (int ch = 0; ch < nch; ++ch, ++it) {
            if (lane == 0 && it + S - 1 < items) issue(it + S - 1);
            const uint32_t st = (uint32_t)it % S;
#ifndef GATE_V_NOWAIT
            gring::bar_wait(bar0 + 8 * st, ((uint32_t)it / S) & 1);
#endif
            const unsigned char* xs = ring + st * kGateStage + g * kGateRow;
            const int cols = min(kGateCC, M - ch * kGateCC);
            const int j0 = ch * (kGateCC / 32);
            // software-pipelined: group jj + 1's shared-memory operands load while group jj's DMMAs issue
            const int ng = cols / 32;
            int4 xv = *reinterpret_cast<const int4*>(xs + 8 * q * 2);
            double2 wv[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int up = 0; up < 4; ++up) wv[nt][up] = sw[((j0 * NT + nt) * 4 + up) * 32 + lane];
#pragma unroll 2
            for (int jj = 0; jj < ng; ++jj) {
                const int jn = jj + 1 < ng ? jj + 1 : jj;
                const int4 xn = *reinterpret_cast<const int4*>(xs + (jn * 32 + 8 * q) * 2);
                double2 wn[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int up = 0; up < 4; ++up) wn[nt][up] = sw[(((j0 + jn) * NT + nt) * 4 + up) * 32 + lane];
                const uint32_t xw[4] = {(uint32_t)xv.x, (uint32_t)xv.y, (uint32_t)xv.z, (uint32_t)xv.w};
                double a[8];
#pragma unroll
                for (int up = 0; up < 4; ++up) {
                    a[2 * up] = bf16_bits_to_f64(xw[up] << 16);
                    a[2 * up + 1] = bf16_bits_to_f64(xw[up] & 0xFFFF0000u);
                }
#ifndef GATE_V_NOMMA
#pragma unroll
                for (int up = 0; up < 4; ++up)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        dmma884(acc[(2 * up) & 3][nt][0], acc[(2 * up) & 3][nt][1], a[2 * up], wv[nt][up].x);
                        dmma884(acc[(2 * up + 1) & 3][nt][0], acc[(2 * up + 1) & 3][nt][1], a[2 * up + 1],
                                wv[nt][up].y);
                    }
#else
                acc[0][0][0] += a[0] * wv[0][0].x + a[7];
#endif
                xv = xn;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int up = 0; up < 4; ++up) wv[nt][up] = wn[nt][up];
            }
            __syncwarp();   // every lane is done with the stage before lane 0 refills it
        }
        double lg[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            lg[nt][0] = (acc[0][nt][0] + acc[1][nt][0]) + (acc[2][nt][0] + acc[3][nt][0]);
            lg[nt][1] = (acc[0][nt][1] + acc[1][nt][1]) + (acc[2][nt][1] + acc[3][nt][1]);
        }
        const int t = tile * 8 + g;
        bool pick[NT][2];
#ifndef GATE_V_NOEPI
        gate_topk_epilogue<NT>(lg, g, q, t, t < n, E, k, expert_idx, combine_w, probs, pick);
#else
        pick[0][0] = lg[0][0] > 0; pick[0][1] = false;
        if (t < n && q < k) { expert_idx[(long long)t * k + q] = q; combine_w[(long long)t * k + q] = (float)lg[0][0]; }
#endif
        if (counts != nullptr) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {   // expert nt*8 + 2qq + h: the lanes of quad index qq
                        const unsigned b = __ballot_sync(0xffffffffu, pick[nt][h] && q == qq);
                        const int e = nt * 8 + 2 * qq + h;
                        if (lane == 0 && e < E) counts[(long long)tile * E + e] = __popc(b);
                    }
        }
    }
}

// dWg^T partials: part[c][e][m] = sum_{t in token range c} dlogits[t][e] * x[t][m].
// One CTA per SM over a contiguous token range (~n/148 tokens): the range's rows stream into
// a shared-memory ring with cp.async.bulk (one copy per stage when rows are contiguous) --
// every byte of x requested at kernel start, no per-thread load latency on the critical
// path -- and the range's logit gradients sit in shared memory (broadcast reads).  Thread =
// 4 consecutive columns of a 1024-column block; f32 accumulation in token order; the
// partials are summed in a fixed order by sum_partials_kernel (deterministic).
constexpr int kWgThreads = 256;
constexpr int kWgBlock = kWgThreads * 4;        // columns per pass
constexpr int kWgMaxTok = 256;                  // tokens per CTA (host: grid >= n / 256)
constexpr int kWgStages = 3;
constexpr int kWgStageBytes = 64 * 1024;

// Two thread halves split each stage's rows (256 threads = 1024 columns each) and fold
// their sums through shared memory at the end: 16 warps per SM for latency hiding.
template <int EMAX, int NB>   // 4 columns x EMAX experts per thread for NB column blocks (M <= NB * 1024)
__global__ void __launch_bounds__(2 * kWgThreads) gate_wgrad_partial_kernel(const bf16* __restrict__ x, long long ldx,
                                                                        const float* __restrict__ dlogits, int n, int M,
                                                                        int E, float* __restrict__ part) {
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
        if (ldx == M) {
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
                    acc[b][e][0] = fmaf(w, f0, acc[b][e][0]);
                    acc[b][e][1] = fmaf(w, f1, acc[b][e][1]);
                    acc[b][e][2] = fmaf(w, f2, acc[b][e][2]);
                    acc[b][e][3] = fmaf(w, f3, acc[b][e][3]);
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
                *reinterpret_cast<float4*>(part + ((long long)blockIdx.x * E + e) * M + c) =
                    make_float4(acc[b][e][0] + o.x, acc[b][e][1] + o.y, acc[b][e][2] + o.z, acc[b][e][3] + o.w);
            }
        }
        __syncthreads();
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

// Tensor-core gate configuration for (n, M, E): warps per CTA and ring depth, or false.
static bool gate_tc_config(int n, int M, int E, int& wpc, int& stages, size_t& smem) {
    if (M % 32 != 0 || E > 16) return false;
    const int NT = E > 8 ? 2 : 1;
    const size_t wbytes = (size_t)(M / 32) * NT * 4 * 32 * 16;
    const size_t budget = 227 * 1024;
    if (wbytes + 2 * 4 * kGateStage + 1024 > budget) return false;
    const int tiles = (n + 7) / 8;
    // warps per CTA (one 8-token tile in flight each): fewest tiles on the busiest SM, most warps on ties
    wpc = 8;
    long long best = -1;
    for (int w = 8; w >= 4; --w) {
        const long long ctas = (tiles + w - 1) / w;
        const long long load = (ctas + kNumSMs - 1) / kNumSMs * w;
        if (best < 0 || load < best) {
            best = load;
            wpc = w;
        }
    }
    const int nch = (M + kGateCC - 1) / kGateCC;
    stages = (int)((budget - wbytes - 1024) / ((size_t)wpc * (kGateStage + 8)));
    const int want = nch * ((tiles + (long long)kNumSMs * wpc - 1) / ((long long)kNumSMs * wpc));   // items per warp
    stages = std::min(stages, std::max(2, std::min(want, 8)));
    if (stages < 2) return false;
    smem = wbytes + (size_t)wpc * stages * (kGateStage + 8) + 128;
    return true;
}

int gate_fwd(const void* x, long long ldx, const void* wgT, int n, int M, int E, int k, int* expert_idx,
             float* combine_w, float* probs, int* counts, cudaStream_t s) {
    PARM_CHECK_ARG(k >= 1 && k <= E, "top_k (%d) exceeds number of experts (%d)", k, E);
    PARM_CHECK_ARG(E <= 32, "gate: at most 32 experts supported (got %d)", E);
    PARM_CHECK_ARG(M % 8 == 0 && ldx % 8 == 0, "gate: embed (%d) and row stride must be multiples of 8", M);
    if (n == 0) return 0;
    auto X = reinterpret_cast<const bf16*>(x);
    auto W = reinterpret_cast<const bf16*>(wgT);
    int wpc = 0, stages = 0;
    size_t smem = 0;
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && gate_tc_config(n, M, E, wpc, stages, smem)) {
        const int tiles = (n + 7) / 8;
        const int blocks = (int)std::min<long long>((tiles + wpc - 1) / wpc, kNumSMs);
        if (E <= 8) {
            cudaFuncSetAttribute(gate_fwd_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(gate_fwd_tc_kernel<1>, blocks, wpc * 32, smem, s, X, ldx, W, n, M, E, k, stages, expert_idx,
                     combine_w, probs, counts);
        } else {
            cudaFuncSetAttribute(gate_fwd_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            launch_k(gate_fwd_tc_kernel<2>, blocks, wpc * 32, smem, s, X, ldx, W, n, M, E, k, stages, expert_idx,
                     combine_w, probs, counts);
        }
        PARM_CHECK_LAUNCH("gate_fwd");
        return 0;
    }
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

size_t gate_wgrad_workspace(int n, int M, int E) {
    return (size_t)gate_wgrad_grid(n) * M * E * sizeof(float);
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
    const int emax = E <= 8 ? 8 : (E <= 16 ? 16 : 32);
    PARM_CHECK_ARG(M % 8 == 0 && M <= (32 / emax) * kWgBlock && ldx % 8 == 0 &&
                       (reinterpret_cast<uintptr_t>(x) & 15) == 0,
                   "gate_wgrad: embed (%d) must be a multiple of 8 and <= %d for %d experts, rows 16-byte aligned", M,
                   (32 / emax) * kWgBlock, E);
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
#define PARM_WG_LAUNCH(EM, NBV)                                                                              \
    do {                                                                                                     \
        static bool attr = false;                                                                            \
        if (!attr) {                                                                                         \
            cudaFuncSetAttribute(gate_wgrad_partial_kernel<EM, NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 smem);                                                                      \
            attr = true;                                                                                     \
        }                                                                                                    \
        launch_k(gate_wgrad_partial_kernel<EM, NBV>, grid, 2 * kWgThreads, smem, s, X, ldx, dlogits, n, M, E, ws); \
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
    launch_k(sum_partials_kernel, (int)((len + 31) / 32), 256, 0, s, ws, grid, len, dwgT, accumulate);
    PARM_CHECK_LAUNCH("gate_wgrad_sum");
    return 0;
}

}  // namespace parm
