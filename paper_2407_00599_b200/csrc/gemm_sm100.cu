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
    int kind, mb, epi;         // problem kind, B operand major-ness, fused epilogue
    int dep, dep_on;           // multi-problem launch: dependency kind and the problem depended on
    int fill_off, prefix_off;  // shared-memory offsets (ints) of the fill table and the ROW live-pair prefix
    int row_ctr, col_ctr;      // completion counters (ints past ws + 2): (g, pair) and (g, n-block)
    int signal;                // a later problem depends on this one: publish tile completions
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
    int pj;                  // pair index within group g (ROW: compacted live pair; WGT: m pair)
};

__device__ __forceinline__ PairTile decode_pair(const Params& p, const int* sfill, int tile, int bn, uint32_t rank,
                                               const int* sprefix) {
    PairTile t;
    int pj;
    t.hi = t.lo = 0;
    if (p.kind == kRow) {   // tile = live pair-tile index: groups' live row pairs, compacted (sprefix)
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
    t.pj = pj;
    if (p.kind == kRow) {
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

constexpr int kBarBytes = 512;   // mbarriers, TMEM slot, tile broadcast ring, queue offsets

template <int BN>
struct CfgPair {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = (BN / 2) * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kEpiBytes = 4 * kEpiBufs * kEpiStageBytes;   // 4 epilogue warps x staging buffers
    static constexpr int kFixed = kEpiBytes + 1024 + kBarBytes + kMaxFill * 4;
    static constexpr int kStages = (PARM_PAIR_SMEM - kFixed) / kStageBytes > 8 ? 8
                                                                               : (PARM_PAIR_SMEM - kFixed) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + kFixed;
    static_assert(2 * kStages * 8 + 4 * 8 + 2 * 4 * 8 + 4 + 4 * 4 + 5 * 4 <= kBarBytes, "barrier area");
};

// ---------------------------------------------------------------- multi-problem persistent kernel
// One launch runs up to kMaxProb GEMMs (the expert FFN's forward pair or its four backward
// GEMMs) as ONE queue of 256 x BN pair tiles, problem after problem, walked round-robin by the
// persistent CTA pairs (pair p takes queue tiles p, p + pairs, ...): the partial last wave of one
// GEMM is filled by the next GEMM's tiles instead of idling (Y / dR have 256 tiles for 74 pairs:
// 3.46 waves), and the launch/drain of four kernels becomes one.  A tile of a dependent problem
// waits, before its first TMA load, for the tiles it reads:
//   kDepRowPair   ROW tile (g, pair) of problem i reads rows of the same pair of problem j
//                 over all of j's columns (Y = H W2 after H; dR = dH W1^T after dH);
//   kDepColBlock  WGT tile (g, m-pair) reads columns [256 m-pair, +256) of problem j's output
//                 for every row of group g (dW1^T = dH^T R after dH).
// Completion counters: every epilogue warp of a finished tile (8 per pair) waits for its bulk
// stores, fences, and adds 1 to the (g, pair) and (g, column block) counters of its problem --
// deferred to the start of its next drain (by then the stores are done) unless that next tile is
// itself a dependent one.
// Deadlock freedom: each pair walks its tiles in increasing queue order and a tile only waits
// on tiles of lower index, so by induction on the index every awaited tile is reached -- given
// every pair is resident, which the host guarantees with a cooperative launch whenever the
// launch has dependencies.  (A dynamic queue -- tiles claimed from a device counter and
// broadcast to the pair through shared memory -- measured ~10% slower per step than this
// static walk: tools/probes/step_ab.py.)  The last CTA to exit zeroes the counters.
constexpr int kMaxProb = 4;
enum Dep : int { kDepNone = 0, kDepRowPair = 1, kDepColBlock = 2 };

struct Multi {
    CUtensorMap ta[kMaxProb], tb[kMaxProb], td[kMaxProb];
    Params pr[kMaxProb];
    int nprob;
    int seg_prob;                  // problem whose ROW outputs go through SegMaps (-1: none)
    int* ws;                       // [0] unused, [1] exit count, [2 ...] completion counters (null: none)
    int ws_ints;                   // counters to clear at exit (from ws + 2)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void wait_counter(const int* c, int target) {
    const long long t0 = clock64();
    while (ld_acquire(c) < target) {
        __nanosleep(128);
        if (clock64() - t0 > (8ll << 30)) asm volatile("trap;");
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");   // the TMA loads that follow see the data
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Completion counter (and its target) a tile of problem p waits on, or null.
__device__ __forceinline__ int* dep_counter(const Multi& mp, const int* sfill, const Params& p, const PairTile& t,
                                            int& target) {
    if (p.dep == kDepRowPair) {
        const Params& q = mp.pr[p.dep_on];
        target = 8 * q.n_blocks;
        return mp.ws + 2 + q.row_ctr + t.g * q.pairs + t.pj;
    }
    if (p.dep == kDepColBlock) {
        const Params& q = mp.pr[p.dep_on];
        const int* qp = sfill + q.prefix_off;
        target = 8 * (qp[t.g + 1] - qp[t.g]);
        return mp.ws + 2 + q.col_ctr + t.g * q.n_blocks + t.pj;
    }
    return nullptr;
}

// (problem, local tile) of queue index `tile` (sbase: prefix of the problems' tile counts)
__device__ __forceinline__ int find_prob(const int* sbase, int nprob, int tile) {
    int pi = 0;
    while (pi + 1 < nprob && sbase[pi + 1] <= tile) ++pi;
    return pi;
}

template <int BN>
__device__ __forceinline__ void drain_any(const Params& p, const CUtensorMap* td, uint32_t taddr, int lane, int row0,
                                          const PairTile& t, bool row_ok, long long xrow, bool empty, uint8_t* stage,
                                          int& buf, const CUtensorMap* seg) {
#define PARM_DRAIN(KD, EP) \
    drain_tile_tma<BN, KD, EP>(p, td, taddr, lane, row0, t.g, t.lo, t.hi, t.n0, row_ok, xrow, empty, stage, buf, seg)
    if (p.kind == kRow) {
        switch (p.epi) {
            case kEpiReluBF16: PARM_DRAIN(kRow, kEpiReluBF16); break;
            case kEpiDReluBF16: PARM_DRAIN(kRow, kEpiDReluBF16); break;
            case kEpiReluMaskBF16: PARM_DRAIN(kRow, kEpiReluMaskBF16); break;
            case kEpiDMaskBF16: PARM_DRAIN(kRow, kEpiDMaskBF16); break;
            default: PARM_DRAIN(kRow, kEpiBF16); break;
        }
    } else if (p.epi == kEpiF32Acc) {
        PARM_DRAIN(kWgt, kEpiF32Acc);
    } else {
        PARM_DRAIN(kWgt, kEpiF32);
    }
#undef PARM_DRAIN
}


// Producer body of one pair tile: its K blocks' A rows and half B tile into the smem ring.
template <int BN, int KIND, int MB>
__device__ __forceinline__ void produce_tile(const Params& p, const int* pf, const PairTile& t, uint32_t rank,
                                             bool leader, const CUtensorMap* tma, const CUtensorMap* tmb,
                                             uint8_t* smem_a, uint8_t* smem_b, uint64_t* full_bar,
                                             uint64_t* empty_bar, int& stage, uint32_t& phase) {
    using C = CfgPair<BN>;
    constexpr int BNH = BN / 2;
    const int g = t.g;
    const int nb0 = t.n0 + (int)rank * BNH;   // this CTA's half of the B tile
    for_each_kblock<KIND>(p, pf, g, [&](int hi, int lo, int r0) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (leader)
            mbar_expect_tx(&full_bar[stage], 2u * C::kStageBytes);
        else
            mbar_arrive_remote(&full_bar[stage], 0);
        uint8_t* sa = smem_a + stage * C::kABytes;
        uint8_t* sb = smem_b + stage * C::kBBytes;
        if (KIND == kRow) {
            tma2_load_5d(tma, &full_bar[stage], sa, r0, t.m0, g, t.lo, t.hi);
            if (MB == kKMajor) {
                tma2_load_3d(tmb, &full_bar[stage], sb, r0, nb0, g);
            } else {
#pragma unroll
                for (int a = 0; a < BNH / 64; ++a)
                    tma2_load_3d(tmb, &full_bar[stage], sb + a * (BK * 128), nb0 + a * 64, r0, g);
            }
        } else {
#pragma unroll
            for (int a = 0; a < BM / 64; ++a)
                tma2_load_5d(tma, &full_bar[stage], sa + a * (BK * 128), t.m0 + a * 64, r0, g, lo, hi);
#pragma unroll
            for (int a = 0; a < BNH / 64; ++a)
                tma2_load_5d(tmb, &full_bar[stage], sb + a * (BK * 128), nb0 + a * 64, r0, g, lo, hi);
        }
        if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
        }
    });
}

// MMA body of one pair tile (leader, one thread): compile-time instruction / smem descriptors.
template <int BN, int KIND, int MA, int MBX>
__device__ __forceinline__ void mma_tile(const Params& p, const int* pf, int g, uint32_t tmem_d, uint8_t* smem_a,
                                         uint8_t* smem_b, uint64_t* full_bar, uint64_t* empty_bar, int& stage,
                                         uint32_t& phase) {
    using C = CfgPair<BN>;
    constexpr uint32_t idesc = instr_desc_pair<BN, MA, MBX>();
    constexpr uint32_t a_lbo = (MA == kKMajor) ? 0 : BK * 128;
    constexpr uint32_t b_lbo = (MBX == kKMajor) ? 0 : BK * 128;
    constexpr uint32_t a_kstep = (MA == kKMajor) ? 32 : 16 * 128;
    constexpr uint32_t b_kstep = (MBX == kKMajor) ? 32 : 16 * 128;
    bool first = true;
    for_each_kblock<KIND>(p, pf, g, [&](int, int, int) {
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
        if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
        }
    });
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    moe_gemm_pair_kernel(const __grid_constant__ Multi mp, const __grid_constant__ SegMaps segmaps) {
    using C = CfgPair<BN>;
    constexpr int STAGES = C::kStages;
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
    int* sbase = reinterpret_cast<int*>(tmem_slot + 1);          // kMaxProb + 1 queue offsets
    int* sfill = reinterpret_cast<int*>(smem + STAGES * C::kStageBytes + kBarBytes);
    uint8_t* smem_epi = smem + STAGES * C::kStageBytes + kBarBytes + kMaxFill * 4;   // 1024-aligned staging
    smem_epi = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_epi) + 1023) & ~uintptr_t(1023));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int nprob = mp.nprob;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < nprob; ++i) {
            prefetch_tmap(&mp.ta[i]);
            prefetch_tmap(&mp.tb[i]);
            prefetch_tmap(&mp.td[i]);
        }
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
    // fill tables and ROW live-pair prefixes of every problem
    for (int i = 0; i < nprob; ++i) {
        const Params& p = mp.pr[i];
        if (p.fill)
            for (int j = threadIdx.x; j < p.G * p.nhi * p.nlo; j += blockDim.x) sfill[p.fill_off + j] = __ldg(p.fill + j);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int base = 0;
        for (int i = 0; i < nprob; ++i) {
            const Params& p = mp.pr[i];
            sbase[i] = base;
            if (p.kind == kRow) {
                const int* f = sfill + p.fill_off;
                int* pre = sfill + p.prefix_off;
                int acc = 0;
                pre[0] = 0;
                for (int g = 0; g < p.G; ++g) {
                    int lt = 0;
                    for (int seg = 0; seg < p.nhi * p.nlo; ++seg) {
                        const int h = seg / p.nlo, l = seg - h * p.nlo;
                        int live = (seg_fill(p, f, g, h, l) + BM - 1) / BM;
                        lt += live > p.m_tiles ? p.m_tiles : live;
                    }
                    acc += (lt + 1) / 2;
                    pre[g + 1] = acc;
                }
                base += acc * p.n_blocks;
            } else {
                base += p.num_tiles;
            }
        }
        sbase[nprob] = base;
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total = sbase[nprob];

    // pair p takes queue tiles p, p + pairs, ... (every role computes the same sequence)
    const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;
    auto next_tile = [&](int& si) -> int {
        const int tile = pair_id + si * num_pairs;
        ++si;
        return tile < total ? tile : total;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            int si = 0;
            int pre_tile = -1, pre_val = 0;   // the next dependent tile's counter, read ahead
            while (true) {
                const int tile = next_tile(si);
                if (tile >= total) break;
                const int pi = find_prob(sbase, nprob, tile);
                const Params p = mp.pr[pi];   // by value: registers, not param-space reloads after every asm clobber
                const int* pf = sfill + p.fill_off;
                const PairTile t = decode_pair(p, pf, tile - sbase[pi], BN, rank, sfill + p.prefix_off);
                if (!t.live) continue;
#ifndef PARM_GEMM_NO_DEPS   // (measurement variant only: dependent tiles do not wait -- wrong results)
                int target = 0;
                if (const int* ctr = dep_counter(mp, sfill, p, t, target)) {
                    // the counter was read (relaxed) while the previous tile's loads were issued: when it
                    // already showed the target, a fence makes that read an acquire -- no round trip here
                    if (pre_tile == tile && pre_val >= target) {
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    } else {
                        wait_counter(ctr, target);
                    }
                }
                {   // prefetch the next tile's counter
                    const int nt = pair_id + si * num_pairs;
                    pre_tile = -1;
                    if (nt < total) {
                        const int npi = find_prob(sbase, nprob, nt);
                        const Params& np = mp.pr[npi];
                        if (np.dep != kDepNone) {
                            const PairTile ntt = decode_pair(np, sfill + np.fill_off, nt - sbase[npi], BN, rank,
                                                             sfill + np.prefix_off);
                            int nt_target = 0;
                            if (const int* nctr = dep_counter(mp, sfill, np, ntt, nt_target)) {
                                pre_val = ld_relaxed(nctr);
                                pre_tile = nt;
                            }
                        }
                    }
                }
#endif
                const CUtensorMap* tma = &mp.ta[pi];
                const CUtensorMap* tmb = &mp.tb[pi];
                // one loop per (kind, B major): compile-time TMA patterns in the per-k-block body
                if (p.kind == kWgt)
                    produce_tile<BN, kWgt, kMNMajor>(p, pf, t, rank, leader, tma, tmb, smem_a, smem_b, full_bar,
                                                     empty_bar, stage, phase);
                else if (p.mb == kKMajor)
                    produce_tile<BN, kRow, kKMajor>(p, pf, t, rank, leader, tma, tmb, smem_a, smem_b, full_bar,
                                                    empty_bar, stage, phase);
                else
                    produce_tile<BN, kRow, kMNMajor>(p, pf, t, rank, leader, tma, tmb, smem_a, smem_b, full_bar,
                                                     empty_bar, stage, phase);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ------------------------------------------------ MMA issuer (leader CTA only)
            int stage = 0;
            uint32_t phase = 0;
            int it_tile = 0;
            int si = 0;
            while (true) {
                const int tile = next_tile(si);
                if (tile >= total) break;
                const int pi = find_prob(sbase, nprob, tile);
                const Params p = mp.pr[pi];   // by value: registers, not param-space reloads after every asm clobber
                const int* pf = sfill + p.fill_off;
                const PairTile t = decode_pair(p, pf, tile - sbase[pi], BN, rank, sfill + p.prefix_off);
                if (!t.live) continue;
                const int as = it_tile & 1;
                const uint32_t aphase = (it_tile >> 1) & 1;
                ++it_tile;
                mbar_wait(&tempty_bar[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + as * BN;
                if (p.kind == kWgt)
                    mma_tile<BN, kWgt, kMNMajor, kMNMajor>(p, pf, t.g, tmem_d, smem_a, smem_b, full_bar, empty_bar,
                                                          stage, phase);
                else if (p.mb == kKMajor)
                    mma_tile<BN, kRow, kKMajor, kKMajor>(p, pf, t.g, tmem_d, smem_a, smem_b, full_bar, empty_bar,
                                                        stage, phase);
                else
                    mma_tile<BN, kRow, kKMajor, kMNMajor>(p, pf, t.g, tmem_d, smem_a, smem_b, full_bar, empty_bar,
                                                         stage, phase);
                tc2_commit_both(&tfull_bar[as]);
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------- epilogue (both CTAs, own TMEM rows)
        const int ew = warp & 3;
        int it_tile = 0;
        int ebuf = 0;
        int si = 0;
        uint8_t* my_stage = smem_epi + ew * kEpiBufs * kEpiStageBytes;
        // Completion of a depended-on tile is published one tile late -- when this warp starts its
        // next drain its stores have long completed, so the wait is free -- except before a tile
        // that itself waits on others (this warp's next tile could be waiting on this very
        // signal) and at the end.
        int* pend_row = nullptr;
        int* pend_col = nullptr;
        auto publish = [&]() {
            if (pend_row != nullptr && lane == 0) {
                bulk_wait_all();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence();
                atomicAdd(pend_row, 1);
                atomicAdd(pend_col, 1);
            }
            pend_row = pend_col = nullptr;
        };
        while (true) {
            const int tile = next_tile(si);
            if (tile >= total) break;
            const int pi = find_prob(sbase, nprob, tile);
            const Params p = mp.pr[pi];   // by value (see the producer)
            const int* pf = sfill + p.fill_off;
            const PairTile t = decode_pair(p, pf, tile - sbase[pi], BN, rank, sfill + p.prefix_off);
            if (!t.live) continue;
            if (p.dep != kDepNone) publish();
            const int as = it_tile & 1;
            const uint32_t aphase = (it_tile >> 1) & 1;
            ++it_tile;
            bool empty = false;
            if (p.kind == kWgt && p.fill) {
                empty = true;
                for (int seg = 0; seg < p.nhi * p.nlo && empty; ++seg)
                    empty = seg_fill(p, pf, t.g, seg / p.nlo, seg % p.nlo) <= 0;
            }
            mbar_wait(&tfull_bar[as], aphase);
            tc_fence_after();
            publish();
            const int row = t.m0 + ew * 32 + lane;
            const bool row_ok = (p.kind == kWgt) ? row < p.M : row < p.L;
            long long xrow = 0;
            if (p.kind == kRow)
                xrow = (long long)t.g * p.x_g + (long long)t.lo * p.x_lo + (long long)t.hi * p.x_hi +
                       (long long)row * p.x_ld;
            const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + as * BN;
            const CUtensorMap* seg = (p.kind == kRow && p.seg_peer) ? &segmaps.m[t.hi * p.nlo + t.lo] : nullptr;
            drain_any<BN>(p, &mp.td[pi], taddr, lane, t.m0 + ew * 32, t, row_ok, xrow, empty, my_stage, ebuf, seg);
            tc_fence_before();
            if (leader)
                mbar_arrive(&tempty_bar[as]);
            else
                mbar_arrive_remote(&tempty_bar[as], 0);
#ifndef PARM_GEMM_NO_DEPS
            if (p.signal) {   // this warp's rows of the tile, for dependent tiles (published later)
                pend_row = mp.ws + 2 + p.row_ctr + t.g * p.pairs + t.pj;
                pend_col = mp.ws + 2 + p.col_ctr + t.g * p.n_blocks + t.n0 / BN;
            }
#endif
        }
        publish();
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
    if (mp.ws != nullptr && threadIdx.x == 0) {   // the last CTA out resets the counters for the next launch
        __threadfence();
        if (atomicAdd(mp.ws + 1, 1) == (int)gridDim.x - 1) {
            for (int i = 0; i < mp.ws_ints; ++i) mp.ws[2 + i] = 0;
            mp.ws[0] = 0;
            __threadfence();
            mp.ws[1] = 0;
        }
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

static SegMaps g_segmaps;   // per-call store maps of the peer-output problem (host calls are stream-ordered)

// Parameters and tensor maps of one GEMM descriptor (validates it).  bn: the pair tile's width.
static int build_problem(const parm_gemm_desc& q, Params& p, CUtensorMap& ta, CUtensorMap& tb, CUtensorMap& td,
                         int& bn) {
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
    memset(&p, 0, sizeof(p));
    p.G = q.groups;
    p.nhi = q.nhi;
    p.nlo = q.nlo;
    p.L = q.seg_len;
    p.M = q.M;
    p.N = q.N;
    p.K = q.K;
    p.alpha = q.alpha;
    p.fill = q.fill;
    p.kind = q.kind;
    p.mb = q.kind == kRow ? q.b_major : kMNMajor;
    p.epi = q.epi;
    p.dep_on = -1;
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
    bn = (q.N % 256 == 0) ? 256 : 128;
    p.n_blocks = q.N / bn;
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
        return rc;
    }
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
    return make_tmap(&tb, q.b.ptr, 5, bd, bs, BK);
}

// Completion counters one problem needs when another depends on it: (g, pair) and (g, n-block).
static long long counter_ints(const Params& p) { return (long long)p.G * (p.pairs + p.n_blocks); }

static size_t multi_workspace(const parm_gemm_desc* qs, int count) {
    long long ints = 2;
    for (int i = 0; i < count; ++i) {
        const parm_gemm_desc& q = qs[i];
        const int bn = (q.N % 256 == 0) ? 256 : 128;
        const long long pairs = q.kind == kRow ? ((long long)q.nhi * q.nlo * ((q.seg_len + BM - 1) / BM) + 1) / 2
                                               : ((q.M + BM - 1) / BM + 1) / 2;
        ints += (long long)q.groups * (pairs + q.N / bn);
    }
    return (size_t)ints * sizeof(int);
}

// CTA pairs of the kernel that can be resident at once on this device (cached per instantiation).
template <int BN>
static int resident_pairs() {
    static int pairs = -1;
    if (pairs < 0) {
        using C = CfgPair<BN>;
        auto kern = moe_gemm_pair_kernel<BN>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(kNumSMs);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = C::kSmemBytes;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            clusters = 0;
        }
        pairs = clusters;
    }
    return pairs;
}

// coop: a cooperative launch (every CTA resident at once) -- required when tiles wait on others.
template <int BN>
static void launch_multi(const Multi& m, int grid, bool coop, cudaStream_t stream) {
    using C = CfgPair<BN>;
    auto kern = moe_gemm_pair_kernel<BN>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        attr_set = true;
    }
    if (!coop) {
        launch_k(kern, grid, kThreads, C::kSmemBytes, stream, m, g_segmaps);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, m, g_segmaps);
}

// count GEMMs as one persistent launch.  deps: 2 ints per problem (kind, problem depended on) or null.
// ws: null (count == 1, no dependencies: static tile order) or a zero-initialised workspace of
// multi_workspace() bytes, left zeroed by the kernel.  seg_prob >= 0: that problem's ROW outputs go
// to seg_dst (the owners' receive blocks) instead of its D.
static int run_multi(const parm_gemm_desc* qs, int count, const int* deps, int* ws, size_t ws_bytes, int seg_prob,
                     const RowFan* seg_dst, long long sd_g, long long sd_ld, cudaStream_t stream) {
    PARM_CHECK_ARG(count >= 1 && count <= kMaxProb, "gemm: %d problems (1..%d per launch)", count, kMaxProb);
    bool any_dep = false;
    for (int i = 0; deps != nullptr && i < count; ++i) any_dep |= deps[2 * i] != kDepNone;
    PARM_CHECK_ARG(ws != nullptr || !any_dep, "gemm: dependencies need a workspace (completion counters)");
    PARM_CHECK_ARG(ws == nullptr || ws_bytes >= multi_workspace(qs, count), "gemm: workspace too small");
    Multi m;
    memset(&m, 0, sizeof(m));
    int bn = 0, fill_ints = 0;
    long long ctr = 0, ub = 0;
    for (int i = 0; i < count; ++i) {
        Params& p = m.pr[i];
        int b;
        if (int rc = build_problem(qs[i], p, m.ta[i], m.tb[i], m.td[i], b)) return rc;
        PARM_CHECK_ARG(i == 0 || b == bn, "gemm: problems of one launch need the same tile width (N %% 256)");
        bn = b;
        p.fill_off = fill_ints;
        if (p.fill) fill_ints += p.G * p.nhi * p.nlo;
        p.prefix_off = fill_ints;
        if (p.kind == kRow) fill_ints += p.G + 1;
        ub += p.num_tiles;
        if (deps != nullptr && deps[2 * i] != kDepNone) {
            const int kd = deps[2 * i], on = deps[2 * i + 1];
            PARM_CHECK_ARG(on >= 0 && on < i, "gemm: problem %d depends on %d (must be an earlier problem)", i, on);
            const Params& q = m.pr[on];
            PARM_CHECK_ARG(q.kind == kRow && q.G == p.G && q.nhi == p.nhi && q.nlo == p.nlo && q.L == p.L &&
                               q.fill == p.fill,
                           "gemm: a dependency must be a ROW problem over the same rows and fill counts");
            if (kd == kDepRowPair) {
                PARM_CHECK_ARG(p.kind == kRow, "gemm: row-pair dependency of a non-ROW problem");
            } else {
                PARM_CHECK_ARG(kd == kDepColBlock && p.kind == kWgt && bn == 256 && q.N == p.M,
                               "gemm: column-block dependency needs a WGT problem with M = the ROW problem's N "
                               "and 256-wide tiles");
            }
            p.dep = kd;
            p.dep_on = on;
            m.pr[on].signal = 1;
        }
    }
    PARM_CHECK_ARG(fill_ints <= kMaxFill, "gemm: fill tables too large");
    for (int i = 0; i < count; ++i) {
        Params& p = m.pr[i];
        if (!p.signal) continue;
        p.row_ctr = (int)ctr;
        p.col_ctr = (int)(ctr + (long long)p.G * p.pairs);
        ctr += counter_ints(p);
    }
    m.seg_prob = seg_prob;
    if (seg_prob >= 0) {
        const parm_gemm_desc& q = qs[seg_prob];
        PARM_CHECK_ARG(seg_prob < count && seg_dst != nullptr, "gemm: bad peer-output problem %d", seg_prob);
        PARM_CHECK_ARG(q.kind == kRow && (q.epi == kEpiBF16 || q.epi == kEpiReluBF16),
                       "gemm: peer segment outputs need a ROW GEMM with a bf16 epilogue");
        PARM_CHECK_ARG(seg_dst->n == q.nhi * q.nlo, "gemm: %d peer outputs for %d segments", seg_dst->n,
                       q.nhi * q.nlo);
        PARM_CHECK_ARG(sd_ld % 8 == 0 && sd_g % 8 == 0, "gemm: peer output rows must be 16-byte aligned");
        PARM_CHECK_ARG(!m.pr[seg_prob].signal, "gemm: a peer-output problem cannot be depended on");
        m.pr[seg_prob].seg_peer = 1;
        for (int i = 0; i < seg_dst->n; ++i) {
            const long long dd[3] = {q.N, q.seg_len, q.groups};
            const long long ds[2] = {sd_ld, sd_g};
            if (int rc = make_tmap(&g_segmaps.m[i], seg_dst->ptr[i], 3, dd, ds, 32, 2, 64)) return rc;
        }
    }
    m.nprob = count;
    m.ws = ws;
    m.ws_ints = (int)ctr;
    long long pairs = ub < kNumSMs / 2 ? ub : kNumSMs / 2;   // clusters of 2 CTAs, one per TPC
    if (pairs < 1) pairs = 1;
    if (!any_dep) m.ws = nullptr;
    if (any_dep && pairs > (bn == 256 ? resident_pairs<256>() : resident_pairs<128>())) {
        // the dependency waits need every pair resident; where the device cannot hold the grid at
        // once, run the problems as stream-ordered single launches instead (same tiles, same results)
        for (int i = 0; i < count; ++i)
            if (int rc = run_multi(&qs[i], 1, nullptr, nullptr, 0, seg_prob == i ? 0 : -1, seg_dst, sd_g, sd_ld,
                                   stream))
                return rc;
        return 0;
    }
    if (bn == 256)
        launch_multi<256>(m, (int)(2 * pairs), any_dep, stream);
    else
        launch_multi<128>(m, (int)(2 * pairs), any_dep, stream);
    PARM_CHECK_LAUNCH("moe_gemm_pair");
    return 0;
}

}  // namespace gemm

size_t moe_gemm_multi_workspace(const parm_gemm_desc* qs, int count) { return gemm::multi_workspace(qs, count); }

int moe_gemm_multi(const parm_gemm_desc* qs, int count, const int* deps, void* ws, size_t ws_bytes, int seg_prob,
                   const RowFan* seg_dst, long long sd_g, long long sd_ld, cudaStream_t stream) {
    return gemm::run_multi(qs, count, deps, reinterpret_cast<int*>(ws), ws_bytes, seg_prob, seg_dst, sd_g, sd_ld,
                           stream);
}

int moe_gemm_peer(const parm_gemm_desc& q, const RowFan* seg_dst, long long sd_g, long long sd_ld,
                  cudaStream_t stream) {
    return gemm::run_multi(&q, 1, nullptr, nullptr, 0, seg_dst ? 0 : -1, seg_dst, sd_g, sd_ld, stream);
}

int moe_gemm(const parm_gemm_desc& q, cudaStream_t stream) { return moe_gemm_peer(q, nullptr, 0, 0, stream); }

}  // namespace parm
