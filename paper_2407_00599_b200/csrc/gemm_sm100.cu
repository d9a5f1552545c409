// Grouped bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the expert-FFN engine of the Parm MoE layer.
//
// Every expert-row tensor of the layer lives in the AlltoAll receive layout
//     [src_hi][src_lo][expert g][row r < L][col]            ("segmented rows")
// so that each exchange is ONE message per peer; the GEMM reads and writes
// that layout directly (5-D TMA maps, OOB rows zero-filled; row-remapped
// epilogue), and skips 128-row tiles / 64-row K-blocks beyond each segment's
// fill count (capacity padding carries no work).  Two problem kinds:
//
//   ROW   D[s][g][r][n] = sum_k A[s][g][r][k] * B[g][n][k]     (B = weights,
//         K-major or MN-major)  -- fwd H = relu(R W1), Y = H W2, bwd
//         dH = (dY W2^T).[H>0], dR = dH W1^T   (reference dataplane.py:122-128)
//   WGT   D[g][m][n] = sum_{s,r} A[s][g][r][m] * B[s][g][r][n] -- dW1^T = dH^T R,
//         dW2^T = dY^T H (both operands MN-major over the segmented K)
//
// Structure (CTA pairs on a TPC, cta_group::2, persistent over 256 x BN pair tiles):
//   warp 0      TMA producer (one lane per CTA), STAGES-deep smem ring, 128B swizzle;
//               each CTA stages its 128 A rows and half of the B tile
//   warp 1      MMA issuer (leader CTA, one lane): tcgen05.mma.cta_group::2.kind::f16,
//               M=256 N=BN K=16, fp32 accumulators in TMEM (2 x BN columns,
//               double-buffered so the epilogue of tile i overlaps the MMA of i+1)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> registers -> fused op -> swizzled
//               staging -> TMA bulk-tensor store (or reduce-add)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/parm_b200.h"
#include "common.cuh"

namespace parm {
namespace gemm {

enum Major : int { kKMajor = 0, kMNMajor = 1 };
enum Kind : int { kRow = 0, kWgt = 1 };
enum Epi : int {
    kEpiBF16 = 0,
    kEpiReluBF16 = 1,
    kEpiDReluBF16 = 2,      // keep where aux (bf16, shaped like D) > 0
    kEpiF32 = 3,
    kEpiF32Acc = 4,
    kEpiReluMaskBF16 = 5,   // relu, and aux (u32 [rows][N/32]) receives the bit mask of the stored value > 0
    kEpiDMaskBF16 = 6,      // keep where the aux bit mask is set (1/16 of kEpiDReluBF16's aux bytes)
};

__device__ __forceinline__ uint32_t bf16_pos_bits(uint32_t packed) {   // bit0: low half > 0, bit1: high half > 0
    const uint32_t lo = packed & 0xFFFFu, hi = packed >> 16;
    return (uint32_t)((lo & 0x8000u) == 0 && (lo & 0x7FFFu) != 0) |
           ((uint32_t)((hi & 0x8000u) == 0 && (hi & 0x7FFFu) != 0) << 1);
}

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;

struct Params {
    int G, nhi, nlo, L;        // row space: segments (hi, lo), rows per segment
    int M, N, K;               // ROW: K = reduction, N = cols; WGT: M x N output, K from row space
    int m_tiles, n_blocks, num_tiles, k_iters;
    float alpha;
    void* D;
    long long d_ld, d_g, d_lo, d_hi;
    const bf16* aux;
    long long x_ld, x_g, x_lo, x_hi;
    const int* fill;           // [hi][lo][g] valid rows, or null
    int pairs;                 // max 256-row pair tiles per group
    int seg_peer;              // ROW: rows of segment (hi, lo) stored through SegMaps.m[hi * nlo + lo] (the
                               //   owners' receive blocks, peer memory) -- the return AlltoAll fused into the epilogue
};

// Per-segment 3-D store maps (N, rows, G) over peer destinations: the TMA-store
// epilogue writes each output tile straight into its owner's receive block.
struct SegMaps {
    CUtensorMap m[kMaxPeers];
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Spin on an mbarrier phase.  A watchdog turns a protocol bug into a trap
// (reported as a CUDA error) instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) break;
        if (clock64() - t0 > (8ll << 30)) asm volatile("trap;");  // ~4 s at 2 GHz
    }
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_load_5d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

#define PARM_TMEM_LD32(taddr, r)                                                                         \
    asm volatile(                                                                                        \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),    \
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),    \
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                             \
        : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// SM100 shared-memory matrix descriptor, 128-byte swizzle.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;   // SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::f16, A/B bf16, D f32, M=128, N=BN.
template <int BN, int MA, int MB>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)MA << 15) | ((uint32_t)MB << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// Fill counts are staged into shared memory once per CTA (kMaxFill entries): the
// single-thread producer/MMA loops must not pay a global-load latency per K block.
constexpr int kMaxFill = 2048;

__device__ __forceinline__ int seg_fill(const Params& p, const int* sfill, int g, int hi, int lo) {
    return p.fill ? sfill[(hi * p.nlo + lo) * p.G + g] : p.L;
}

// The live K blocks of one tile, in order: ROW walks k0 = 0, BK, ... K; WGT walks each
// segment's filled rows (r0 < fill) -- the (hi, lo, r0) bookkeeping is per segment, not per
// block, so the single MMA-issuing thread spends its cycles issuing MMAs.
template <int KIND, class F>
__device__ __forceinline__ void for_each_kblock(const Params& p, const int* sfill, int g, F&& body) {
    if (KIND == kRow) {
        for (int it = 0; it < p.k_iters; ++it) body(0, 0, it * BK);
    } else {
        for (int hi = 0; hi < p.nhi; ++hi)
            for (int lo = 0; lo < p.nlo; ++lo) {
                const int f = min(seg_fill(p, sfill, g, hi, lo), p.L);
                for (int r0 = 0; r0 < f; r0 += BK) body(hi, lo, r0);
            }
    }
}

// ================================================================ CTA-pair kernel
// cta_group::2: a cluster of two CTAs on a TPC computes a 256 x BN tile with one
// tcgen05.mma.cta_group::2 (UMMA M=256) issued by the even ("leader") CTA.
// Each CTA stages its own 128 A-rows and HALF of the B tile (BN/2 rows of N),
// so per-SM shared-memory traffic per FLOP drops by 1/3 versus the 1-CTA
// 128 x BN tile (the 1-CTA kernel is smem-bandwidth bound: ncu shows
// l1tex/smem ~65% busy at ~1.1 PFLOP/s).  Accumulator rows 0-127 live in the
// leader's TMEM, rows 128-255 in the peer's; each CTA's epilogue drains its own.

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}

// Arrive on the barrier at the same smem offset in CTA `rank` of the cluster.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}

// TMA load whose completion is signalled on the LEADER CTA's mbarrier (cta_group::2).
__device__ __forceinline__ void tma2_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                             int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma2_load_5d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                             int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3), "r"(c4)
        : "memory");
}

__device__ __forceinline__ void tc2_commit_both(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

__device__ __forceinline__ void tc2_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int BN, int MA, int MB>
__device__ __forceinline__ constexpr uint32_t instr_desc_pair() {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)MA << 15) | ((uint32_t)MB << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
}

// k-th live ROW tile of group g in (hi, lo, m-tile) order.
__device__ __forceinline__ bool nth_live_row_tile(const Params& p, const int* sfill, int g, int k, int& hi, int& lo,
                                                  int& m0) {
    const int nseg = p.nhi * p.nlo;
    for (int seg = 0; seg < nseg; ++seg) {
        const int h = seg / p.nlo, l = seg - h * p.nlo;
        const int f = seg_fill(p, sfill, g, h, l);
        int live = (f + BM - 1) / BM;
        if (live > p.m_tiles) live = p.m_tiles;
        if (k < live) {
            hi = h;
            lo = l;
            m0 = k * BM;
            return true;
        }
        k -= live;
    }
    return false;
}

struct PairTile {
    bool live;       // the pair has work (its first tile exists)
    int g, hi, lo, m0, n0;   // this CTA's half: rows [m0, m0+128) of segment (hi, lo); m0 >= L/M -> dummy
};

__device__ __forceinline__ PairTile decode_pair(const Params& p, const int* sfill, int tile, int kind, int bn,
                                               uint32_t rank, const int* sprefix) {
    PairTile t;
    int pj;
    t.hi = t.lo = 0;
    if (kind == kRow) {   // tile = live pair-tile index: groups' live row pairs, compacted (sprefix)
        const int pu = tile / p.n_blocks;
        t.n0 = (tile - pu * p.n_blocks) * bn;
        int g = 0;
        while (sprefix[g + 1] <= pu) ++g;
        t.g = g;
        pj = pu - sprefix[g];
    } else {
        const int per_g = p.pairs * p.n_blocks;
        t.g = tile / per_g;
        const int rem = tile - t.g * per_g;
        pj = rem / p.n_blocks;
        t.n0 = (rem % p.n_blocks) * bn;
    }
    if (kind == kRow) {
        int h0, l0, m00;
        t.live = nth_live_row_tile(p, sfill, t.g, 2 * pj, h0, l0, m00);
        if (rank == 0) {
            t.hi = h0;
            t.lo = l0;
            t.m0 = m00;
        } else if (!nth_live_row_tile(p, sfill, t.g, 2 * pj + 1, t.hi, t.lo, t.m0)) {
            t.hi = h0;
            t.lo = l0;
            t.m0 = p.L;              // dummy: fully out of bounds, zero-filled, never stored
        }
    } else {
        t.m0 = (2 * pj + (int)rank) * BM;   // >= M -> dummy rows
        t.live = true;
    }
    return t;
}

// ---------------------------------------------------------------- TMA-store epilogue (pair kernel)
// Each epilogue warp owns 32 accumulator rows.  Per 128-byte output chunk of
// its rows (64 bf16 / 32 f32 columns) it drains TMEM, applies the fused op,
// writes the chunk into a 128B-swizzled 4 KB staging buffer (conflict-free:
// 8 consecutive rows cover all banks) and issues one bulk-tensor store; two
// buffers per warp alternate so the store of chunk i overlaps chunk i+1.
// Rows past the segment (or a dummy half-tile) are clipped by the TMA unit.
constexpr int kEpiStageBytes = 32 * 128;
// One staging buffer per epilogue warp buys a sixth 32 KB pipeline stage inside
// the 227 KB opt-in shared memory: the TMA loads (not the overlapped epilogue)
// are what the MMA waits on (measured: -4% GEMM time, -5% step).
#ifndef PARM_EPI_BUFS
#define PARM_EPI_BUFS 1
#endif
constexpr int kEpiBufs = PARM_EPI_BUFS;         // staging buffers per epilogue warp
#ifndef PARM_PAIR_SMEM
#define PARM_PAIR_SMEM 232448                   // sm_100 opt-in maximum dynamic shared memory per CTA
#endif

__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

template <int BN, int KIND, int EPI>
__device__ __forceinline__ void drain_tile_tma(const Params& p, const CUtensorMap* tmap_d, uint32_t taddr, int lane,
                                               int row0, int g, int lo, int hi, int n0, bool row_ok, long long xrow,
                                               bool empty, uint8_t* stage, int& buf,
                                               const CUtensorMap* seg_map = nullptr) {
    constexpr bool F32 = (EPI == kEpiF32 || EPI == kEpiF32Acc);
    constexpr int COLS = F32 ? 32 : 64;          // output columns per 128-byte chunk
    constexpr int NCH = BN / COLS;
    uint2* mrow = reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(const_cast<bf16*>(p.aux)) + xrow + n0 / 32);
    uint2 mk_next = make_uint2(0u, 0u);
    if (EPI == kEpiDMaskBF16 && row_ok) mk_next = __ldg(mrow);
    int4 ax_next[8];
    if (EPI == kEpiDReluBF16 && row_ok) {
        const int4* src = reinterpret_cast<const int4*>(p.aux + xrow + n0);
#pragma unroll
        for (int v = 0; v < 8; ++v) ax_next[v] = __ldg(src + v);
    }
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        uint32_t pk[32];   // F32: 32 fp32 words; BF16: 32 packed bf16x2 words (64 columns)
        if (F32) {
            PARM_TMEM_LD32(taddr + ch * 32, pk);
            tmem_ld_wait();
#pragma unroll
            for (int v = 0; v < 32; ++v)
                pk[v] = empty ? 0u : __float_as_uint(p.alpha * __uint_as_float(pk[v]));
        } else {
            int4 ax_cur[8];
            if (EPI == kEpiDReluBF16) {
#pragma unroll
                for (int v = 0; v < 8; ++v) ax_cur[v] = ax_next[v];
                if (row_ok && ch + 1 < NCH) {
                    const int4* src = reinterpret_cast<const int4*>(p.aux + xrow + n0 + (ch + 1) * COLS);
#pragma unroll
                    for (int v = 0; v < 8; ++v) ax_next[v] = __ldg(src + v);
                }
            }
            uint2 mk = mk_next;
            if (EPI == kEpiDMaskBF16 && row_ok && ch + 1 < NCH) mk_next = __ldg(mrow + ch + 1);
            uint32_t r0[32], r1[32];
            PARM_TMEM_LD32(taddr + ch * 64, r0);
            PARM_TMEM_LD32(taddr + ch * 64 + 32, r1);
            tmem_ld_wait();
#pragma unroll
            for (int v = 0; v < 32; ++v) {
                float a = p.alpha * __uint_as_float(v < 16 ? r0[2 * v] : r1[2 * v - 32]);
                float b = p.alpha * __uint_as_float(v < 16 ? r0[2 * v + 1] : r1[2 * v - 31]);
                if (EPI == kEpiReluBF16) {
                    a = fmaxf(a, 0.0f);
                    b = fmaxf(b, 0.0f);
                }
                if (EPI == kEpiDReluBF16) {
                    const uint32_t m = reinterpret_cast<const uint32_t*>(ax_cur)[v];   // bf16 pair of aux
                    const float ma = __uint_as_float(m << 16), mb = __uint_as_float(m & 0xFFFF0000u);
                    a = ma > 0.0f ? a : 0.0f;
                    b = mb > 0.0f ? b : 0.0f;
                }
                if (EPI == kEpiDMaskBF16) {
                    const uint32_t w = v < 16 ? mk.x : mk.y;
                    const int bit = (2 * v) & 31;
                    a = ((w >> bit) & 1u) ? a : 0.0f;
                    b = ((w >> (bit + 1)) & 1u) ? b : 0.0f;
                }
                if (EPI == kEpiReluMaskBF16) {
                    a = fmaxf(a, 0.0f);
                    b = fmaxf(b, 0.0f);
                }
                pk[v] = pack_bf16x2(a, b);
            }
            if (EPI == kEpiReluMaskBF16 && row_ok) {   // bit per stored value > 0, two words per chunk
                uint32_t w0 = 0u, w1 = 0u;
#pragma unroll
                for (int v = 0; v < 16; ++v) w0 |= bf16_pos_bits(pk[v]) << (2 * v);
#pragma unroll
                for (int v = 0; v < 16; ++v) w1 |= bf16_pos_bits(pk[16 + v]) << (2 * v);
                mrow[ch] = make_uint2(w0, w1);
            }
        }
        uint8_t* sbuf = stage + buf * kEpiStageBytes;
        if (lane == 0) {                         // the store that last used this buffer has read it
            if (kEpiBufs == 1)
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else
                bulk_wait_read1();
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(sbuf + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            const int col = n0 + ch * COLS;
            if (KIND == kRow && seg_map != nullptr)
                tma_store_3d(seg_map, sbuf, col, row0, g);
            else if (KIND == kRow)
                tma_store_5d(tmap_d, sbuf, col, row0, g, lo, hi);
            else if (EPI == kEpiF32Acc)
                tma_reduce_add_3d(tmap_d, sbuf, col, row0, g);
            else
                tma_store_3d(tmap_d, sbuf, col, row0, g);
            bulk_commit();
        }
        buf = (buf + 1) % kEpiBufs;
    }
}

template <int BN, int KIND, int MB, int EPI>
struct CfgPair {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = (BN / 2) * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kEpiBytes = 4 * kEpiBufs * kEpiStageBytes;   // 4 epilogue warps x staging buffers
    static constexpr int kFixed = kEpiBytes + 1024 + 256 + kMaxFill * 4;
    static constexpr int kStages = (PARM_PAIR_SMEM - kFixed) / kStageBytes > 8 ? 8
                                                                               : (PARM_PAIR_SMEM - kFixed) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024 + 256 + kMaxFill * 4;
};

template <int BN, int KIND, int MB, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    moe_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                         const __grid_constant__ CUtensorMap tmap_d, const __grid_constant__ Params p,
                         const __grid_constant__ SegMaps segmaps) {
    using C = CfgPair<BN, KIND, MB, EPI>;
    constexpr int STAGES = C::kStages;
    constexpr int MA = (KIND == kRow) ? kKMajor : kMNMajor;
    constexpr int MBX = (KIND == kRow) ? MB : kMNMajor;
    constexpr int BNH = BN / 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + STAGES * C::kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    int* sfill = reinterpret_cast<int*>(smem + STAGES * C::kStageBytes + 256);
    uint8_t* smem_epi = smem + STAGES * C::kStageBytes + 256 + kMaxFill * 4;   // 1024-aligned staging
    smem_epi = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_epi) + 1023) & ~uintptr_t(1023));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair_id = blockIdx.x >> 1;
    const int num_pairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        prefetch_tmap(&tmap_d);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 2);      // leader expect_tx arrival + peer arrival
            mbar_init(&empty_bar[s], 1);     // leader's multicast commit
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull_bar[s], 1);
            mbar_init(&tempty_bar[s], 2 * 128);   // both CTAs' epilogue threads (leader's copy used)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)C::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    // everything above is independent of the previous kernel (PDL prologue); fill counts and operands are not
    if (p.fill)
        for (int i = threadIdx.x; i < p.G * p.nhi * p.nlo; i += blockDim.x) sfill[i] = __ldg(p.fill + i);
    // ROW: work list = live 256-row pair tiles only (groups' live row pairs, prefix-summed), so the
    // static round-robin over the 74 pairs balances the real work instead of an index space with
    // unfilled capacity holes (max 5 vs the ideal 4 tiles per pair measured on the second GEMM).
    int* sprefix = sfill + p.G * p.nhi * p.nlo;
    if (KIND == kRow) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            sprefix[0] = 0;
            for (int g = 0; g < p.G; ++g) {
                int lt = 0;
                for (int seg = 0; seg < p.nhi * p.nlo; ++seg) {
                    const int h = seg / p.nlo, l = seg - h * p.nlo;
                    int live = (seg_fill(p, sfill, g, h, l) + BM - 1) / BM;
                    lt += live > p.m_tiles ? p.m_tiles : live;
                }
                acc += (lt + 1) / 2;
                sprefix[g + 1] = acc;
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int ntiles = (KIND == kRow) ? sprefix[p.G] * p.n_blocks : p.num_tiles;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair_id; tile < ntiles; tile += num_pairs) {
                const PairTile t = decode_pair(p, sfill, tile, KIND, BN, rank, sprefix);
                if (!t.live) continue;
                for_each_kblock<KIND>(p, sfill, t.g, [&](int hi, int lo, int r0) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    if (leader)
                        mbar_expect_tx(&full_bar[stage], 2u * C::kStageBytes);
                    else
                        mbar_arrive_remote(&full_bar[stage], 0);
                    uint8_t* sa = smem_a + stage * C::kABytes;
                    uint8_t* sb = smem_b + stage * C::kBBytes;
                    const int nb0 = t.n0 + (int)rank * BNH;   // this CTA's half of the B tile
                    if (KIND == kRow) {
                        const int k0 = r0;
                        tma2_load_5d(&tmap_a, &full_bar[stage], sa, k0, t.m0, t.g, t.lo, t.hi);
                        if (MB == kKMajor) {
                            tma2_load_3d(&tmap_b, &full_bar[stage], sb, k0, nb0, t.g);
                        } else {
#pragma unroll
                            for (int a = 0; a < BNH / 64; ++a)
                                tma2_load_3d(&tmap_b, &full_bar[stage], sb + a * (BK * 128), nb0 + a * 64, k0, t.g);
                        }
                    } else {
#pragma unroll
                        for (int a = 0; a < BM / 64; ++a)
                            tma2_load_5d(&tmap_a, &full_bar[stage], sa + a * (BK * 128), t.m0 + a * 64, r0, t.g, lo,
                                         hi);
#pragma unroll
                        for (int a = 0; a < BNH / 64; ++a)
                            tma2_load_5d(&tmap_b, &full_bar[stage], sb + a * (BK * 128), nb0 + a * 64, r0, t.g, lo,
                                         hi);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                });
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ------------------------------------------------ MMA issuer (leader CTA only)
            constexpr uint32_t idesc = instr_desc_pair<BN, MA, MBX>();
            constexpr uint32_t a_lbo = (MA == kKMajor) ? 0 : BK * 128;
            constexpr uint32_t b_lbo = (MBX == kKMajor) ? 0 : BK * 128;
            constexpr uint32_t a_kstep = (MA == kKMajor) ? 32 : 16 * 128;
            constexpr uint32_t b_kstep = (MBX == kKMajor) ? 32 : 16 * 128;
            int stage = 0;
            uint32_t phase = 0;
            int it_tile = 0;
            for (int tile = pair_id; tile < ntiles; tile += num_pairs) {
                const PairTile t = decode_pair(p, sfill, tile, KIND, BN, rank, sprefix);
                if (!t.live) continue;
                const int as = it_tile & 1;
                const uint32_t aphase = (it_tile >> 1) & 1;
                ++it_tile;
                mbar_wait(&tempty_bar[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + as * BN;
                bool first = true;
                for_each_kblock<KIND>(p, sfill, t.g, [&](int, int, int) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem_a + stage * C::kABytes);
                    const uint32_t sb = smem_u32(smem_b + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad = smem_desc(sa + k * a_kstep, a_lbo, 1024);
                        uint64_t bd = smem_desc(sb + k * b_kstep, b_lbo, 1024);
                        tc2_mma(tmem_d, ad, bd, idesc, (first && k == 0) ? 0u : 1u);
                    }
                    first = false;
                    tc2_commit_both(&empty_bar[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                });
                tc2_commit_both(&tfull_bar[as]);
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------- epilogue (both CTAs, own TMEM rows)
        const int ew = warp & 3;
        int it_tile = 0;
        int ebuf = 0;
        uint8_t* my_stage = smem_epi + ew * kEpiBufs * kEpiStageBytes;
        for (int tile = pair_id; tile < ntiles; tile += num_pairs) {
            const PairTile t = decode_pair(p, sfill, tile, KIND, BN, rank, sprefix);
            if (!t.live) continue;
            const int as = it_tile & 1;
            const uint32_t aphase = (it_tile >> 1) & 1;
            ++it_tile;
            bool empty = false;
            if (KIND == kWgt && p.fill) {
                empty = true;
                for (int seg = 0; seg < p.nhi * p.nlo && empty; ++seg)
                    empty = seg_fill(p, sfill, t.g, seg / p.nlo, seg % p.nlo) <= 0;
            }
            mbar_wait(&tfull_bar[as], aphase);
            tc_fence_after();
            const int row = t.m0 + ew * 32 + lane;
            const bool row_ok = (KIND == kWgt) ? row < p.M : row < p.L;
            long long drow, xrow = 0;
            if (KIND == kRow) {
                drow = (long long)t.g * p.d_g + (long long)t.lo * p.d_lo + (long long)t.hi * p.d_hi +
                       (long long)row * p.d_ld;
                xrow = (long long)t.g * p.x_g + (long long)t.lo * p.x_lo + (long long)t.hi * p.x_hi +
                       (long long)row * p.x_ld;
            } else {
                drow = (long long)t.g * p.d_g + (long long)row * p.d_ld;
            }
            const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + as * BN;
            (void)drow;
            if (KIND == kRow && p.seg_peer) {   // TMA stores straight into the owner's receive block
                drain_tile_tma<BN, KIND, EPI>(p, &tmap_d, taddr, lane, t.m0 + ew * 32, t.g, t.lo, t.hi, t.n0, row_ok,
                                              xrow, empty, my_stage, ebuf, &segmaps.m[t.hi * p.nlo + t.lo]);
            } else {
                drain_tile_tma<BN, KIND, EPI>(p, &tmap_d, taddr, lane, t.m0 + ew * 32, t.g, t.lo, t.hi, t.n0, row_ok,
                                              xrow, empty, my_stage, ebuf);
            }
            tc_fence_before();
            if (leader)
                mbar_arrive(&tempty_bar[as]);
            else
                mbar_arrive_remote(&tempty_bar[as], 0);
        }
        if (lane == 0) bulk_wait_all();
    }

    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"((uint32_t)C::kTmemCols)
                     : "memory");
    }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// bf16 tensor map with 128B swizzle; dims[0] is contiguous; strides in elements for dims 1..rank-1.
static int make_tmap(CUtensorMap* map, const void* base, int rank, const long long* dims, const long long* strides,
                     int box1, int esize = 2, int box0 = 64) {
    auto enc = get_encode();
    PARM_CHECK_ARG(enc != nullptr, "gemm: cuTensorMapEncodeTiled unavailable from the driver");
    PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, "gemm: operand base not 16-byte aligned");
    cuuint64_t gd[5];
    cuuint64_t gs[4];
    cuuint32_t box[5];
    cuuint32_t es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = (cuuint64_t)(dims[i] > 0 ? dims[i] : 1);
        box[i] = i == 0 ? (cuuint32_t)box0 : (i == 1 ? (cuuint32_t)box1 : 1u);
        es[i] = 1;
    }
    for (int i = 0; i + 1 < rank; ++i) {
        long long s = strides[i] > 0 ? strides[i] : 8;
        PARM_CHECK_ARG((s * esize) % 16 == 0, "gemm: stride %lld (dim %d) not a 16-byte multiple", strides[i], i + 1);
        gs[i] = (cuuint64_t)(s * esize);
    }
    CUresult r = enc(map, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                     const_cast<void*>(base), gd, gs, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    PARM_CHECK_ARG(r == CUDA_SUCCESS, "gemm: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

static SegMaps g_segmaps;   // per-call store maps of moe_gemm_peer (host calls are stream-ordered, one thread)

template <int BN, int KIND, int MB, int EPI>
static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const Params& p,
                       cudaStream_t stream) {
    using C = CfgPair<BN, KIND, MB, EPI>;
    auto kern = moe_gemm_pair_kernel<BN, KIND, MB, EPI>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        attr_set = true;
    }
    int grid = 2 * (p.num_tiles < kNumSMs / 2 ? p.num_tiles : kNumSMs / 2);   // clusters of 2 CTAs
    if (grid < 2) grid = 2;
    launch_k(kern, grid, kThreads, C::kSmemBytes, stream, ta, tb, td, p, g_segmaps);
    PARM_CHECK_LAUNCH("moe_gemm_pair");
    return 0;
}

template <int KIND, int MB, int EPI>
static int dispatch_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const Params& p,
                       cudaStream_t s) {
    if (bn == 256) return launch_pair<256, KIND, MB, EPI>(ta, tb, td, p, s);
    return launch_pair<128, KIND, MB, EPI>(ta, tb, td, p, s);
}

}  // namespace gemm

int moe_gemm_peer(const parm_gemm_desc& q, const RowFan* seg_dst, long long sd_g, long long sd_ld, cudaStream_t stream);

int moe_gemm(const parm_gemm_desc& q, cudaStream_t stream) { return moe_gemm_peer(q, nullptr, 0, 0, stream); }

int moe_gemm_peer(const parm_gemm_desc& q, const RowFan* seg_dst, long long sd_g, long long sd_ld,
                  cudaStream_t stream) {
    using namespace gemm;
    PARM_CHECK_ARG(q.kind == kRow || q.kind == kWgt, "gemm: bad kind %d", q.kind);
    PARM_CHECK_ARG(q.groups > 0 && q.nhi > 0 && q.nlo > 0 && q.seg_len > 0, "gemm: empty row space");
    PARM_CHECK_ARG(q.N > 0 && q.N % 128 == 0, "gemm: N=%d must be a positive multiple of 128", q.N);
    PARM_CHECK_ARG(q.epi >= 0 && q.epi <= 6, "gemm: bad epilogue %d", q.epi);
    PARM_CHECK_ARG((q.epi != kEpiDReluBF16 && q.epi != kEpiReluMaskBF16 && q.epi != kEpiDMaskBF16) ||
                       q.aux.ptr != nullptr, "gemm: relu-mask epilogue needs aux");
    PARM_CHECK_ARG((q.epi != kEpiReluMaskBF16 && q.epi != kEpiDMaskBF16) ||
                       ((reinterpret_cast<uintptr_t>(q.aux.ptr) & 7) == 0 && q.N % 64 == 0 && q.aux.ld % 2 == 0),
                   "gemm: bit-mask aux must be 8-byte aligned with N %% 64 == 0");
    PARM_CHECK_ARG(q.groups * q.nhi * q.nlo + q.groups + 1 <= kMaxFill, "gemm: fill table too large");
    Params p;
    p.G = q.groups;
    p.nhi = q.nhi;
    p.nlo = q.nlo;
    p.L = q.seg_len;
    p.M = q.M;
    p.N = q.N;
    p.K = q.K;
    p.alpha = q.alpha;
    p.fill = q.fill;
    p.seg_peer = 0;
    if (seg_dst != nullptr) {
        PARM_CHECK_ARG(q.kind == kRow && (q.epi == kEpiBF16 || q.epi == kEpiReluBF16),
                       "gemm: peer segment outputs need a ROW GEMM with a bf16 epilogue");
        PARM_CHECK_ARG(seg_dst->n == q.nhi * q.nlo, "gemm: %d peer outputs for %d segments", seg_dst->n,
                       q.nhi * q.nlo);
        PARM_CHECK_ARG(sd_ld % 8 == 0 && sd_g % 8 == 0, "gemm: peer output rows must be 16-byte aligned");
        p.seg_peer = 1;
        for (int i = 0; i < seg_dst->n; ++i) {
            const long long dd[3] = {q.N, q.seg_len, q.groups};
            const long long ds[2] = {sd_ld, sd_g};
            if (int rc = make_tmap(&g_segmaps.m[i], seg_dst->ptr[i], 3, dd, ds, 32, 2, 64)) return rc;
        }
    }
    p.D = const_cast<void*>(q.d.ptr);
    p.d_ld = q.d.ld;
    p.d_g = q.d.g_stride;
    p.d_lo = q.d.lo_stride;
    p.d_hi = q.d.hi_stride;
    p.aux = reinterpret_cast<const bf16*>(q.aux.ptr);
    p.x_ld = q.aux.ld;
    p.x_g = q.aux.g_stride;
    p.x_lo = q.aux.lo_stride;
    p.x_hi = q.aux.hi_stride;
    const int bn = (q.N % 256 == 0) ? 256 : 128;
    p.n_blocks = q.N / bn;
    CUtensorMap ta, tb, td;
    int rc;
    if (q.kind == kRow) {   // D: bf16 [hi][lo][g][r][n] -> dims (N, L, G, nlo, nhi), 32-row x 128 B store boxes
        const long long dd[5] = {q.N, q.seg_len, q.groups, q.nlo, q.nhi};
        const long long ds[4] = {q.d.ld, q.d.g_stride, q.d.lo_stride, q.d.hi_stride};
        if ((rc = make_tmap(&td, q.d.ptr, 5, dd, ds, 32, 2, 64))) return rc;
    } else {                // D: f32 [g][m][n] -> dims (N, M, G)
        const long long dd[3] = {q.N, q.M, q.groups};
        const long long ds[2] = {q.d.ld, q.d.g_stride};
        if ((rc = make_tmap(&td, q.d.ptr, 3, dd, ds, 32, 4, 32))) return rc;
    }
    if (q.kind == kRow) {
        PARM_CHECK_ARG(q.K > 0 && q.K % BK == 0, "gemm: K=%d must be a positive multiple of %d", q.K, BK);
        PARM_CHECK_ARG(q.epi <= kEpiDReluBF16 || q.epi == kEpiReluMaskBF16 || q.epi == kEpiDMaskBF16,
                       "gemm: row GEMMs produce bf16");
        p.m_tiles = (q.seg_len + BM - 1) / BM;
        p.pairs = (p.nhi * p.nlo * p.m_tiles + 1) / 2;
        p.num_tiles = p.G * p.pairs * p.n_blocks;
        p.k_iters = q.K / BK;
        // A: [hi][lo][g][r][k] -> dims (K, L, G, nlo, nhi)
        const long long ad[5] = {q.K, q.seg_len, q.groups, q.nlo, q.nhi};
        const long long as[4] = {q.a.ld, q.a.g_stride, q.a.lo_stride, q.a.hi_stride};
        if ((rc = make_tmap(&ta, q.a.ptr, 5, ad, as, BM))) return rc;
        if (q.b_major == kKMajor) {   // B[g][n][k]
            const long long bd[3] = {q.K, q.N, q.groups};
            const long long bs[2] = {q.b.ld, q.b.g_stride};
            rc = make_tmap(&tb, q.b.ptr, 3, bd, bs, bn / 2);   // each CTA of the pair stages half of B
        } else {                      // B[g][k][n]
            const long long bd[3] = {q.N, q.K, q.groups};
            const long long bs[2] = {q.b.ld, q.b.g_stride};
            rc = make_tmap(&tb, q.b.ptr, 3, bd, bs, BK);
        }
        if (rc) return rc;
        const int combo = q.b_major;
        if (combo == kKMajor) {
            if (q.epi == kEpiReluBF16) return dispatch_bn<kRow, kKMajor, kEpiReluBF16>(bn, ta, tb, td, p, stream);
            if (q.epi == kEpiReluMaskBF16)
                return dispatch_bn<kRow, kKMajor, kEpiReluMaskBF16>(bn, ta, tb, td, p, stream);
            if (q.epi == kEpiBF16) return dispatch_bn<kRow, kKMajor, kEpiBF16>(bn, ta, tb, td, p, stream);
        } else {
            if (q.epi == kEpiDReluBF16) return dispatch_bn<kRow, kMNMajor, kEpiDReluBF16>(bn, ta, tb, td, p, stream);
            if (q.epi == kEpiDMaskBF16) return dispatch_bn<kRow, kMNMajor, kEpiDMaskBF16>(bn, ta, tb, td, p, stream);
            if (q.epi == kEpiBF16) return dispatch_bn<kRow, kMNMajor, kEpiBF16>(bn, ta, tb, td, p, stream);
        }
    } else {
        PARM_CHECK_ARG(q.M > 0 && q.M % BM == 0, "gemm: M=%d must be a positive multiple of %d", q.M, BM);
        PARM_CHECK_ARG(q.epi == kEpiF32 || q.epi == kEpiF32Acc, "gemm: weight GEMMs produce f32");
        p.m_tiles = q.M / BM;
        p.pairs = (p.m_tiles + 1) / 2;
        p.num_tiles = p.G * p.pairs * p.n_blocks;
        p.k_iters = p.nhi * p.nlo * ((q.seg_len + BK - 1) / BK);
        const long long ad[5] = {q.M, q.seg_len, q.groups, q.nlo, q.nhi};
        const long long as[4] = {q.a.ld, q.a.g_stride, q.a.lo_stride, q.a.hi_stride};
        if ((rc = make_tmap(&ta, q.a.ptr, 5, ad, as, BK))) return rc;
        const long long bd[5] = {q.N, q.seg_len, q.groups, q.nlo, q.nhi};
        const long long bs[4] = {q.b.ld, q.b.g_stride, q.b.lo_stride, q.b.hi_stride};
        if ((rc = make_tmap(&tb, q.b.ptr, 5, bd, bs, BK))) return rc;
        if (q.epi == kEpiF32) return dispatch_bn<kWgt, kMNMajor, kEpiF32>(bn, ta, tb, td, p, stream);
        return dispatch_bn<kWgt, kMNMajor, kEpiF32Acc>(bn, ta, tb, td, p, stream);
    }
    set_error("gemm: unsupported combination kind=%d b_major=%d epi=%d", q.kind, q.b_major, q.epi);
    return 1;
}

}  // namespace parm
