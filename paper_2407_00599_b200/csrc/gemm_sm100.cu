// Grouped bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// the expert-FFN engine of the Parm MoE layer.
//
//   D_g[m][n] = sum_k A_g[m][k] * B_g[n][k]     for every group g (= local expert)
//
// A and B are each either K-major (row m / n contiguous along k) or MN-major
// (stored transposed, k rows of contiguous m / n).  That single kernel covers
// the six FFN GEMMs of one expert shard (reference dataplane.py:122-128 forward;
// the backward the reference does not have):
//   fwd  H  = relu(R W1)      A=R  (K)   B=W1t (K)   epilogue relu -> bf16
//   fwd  Y  = H W2            A=H  (K)   B=W2t (K)   epilogue bf16
//   bwd  dH = (dY W2^T).[H>0] A=dY (K)   B=W2t (MN)  epilogue relu-mask(aux=H) -> bf16
//   bwd  dR = dH W1^T         A=dH (K)   B=W1t (MN)  epilogue bf16
//   bwd dW1t = dH^T R         A=dH (MN)  B=R   (MN)  epilogue f32
//   bwd dW2t = dY^T H         A=dY (MN)  B=H   (MN)  epilogue f32
//
// Structure (one CTA per SM, persistent over tiles of 128 x BN):
//   warp 0      TMA producer (one lane), STAGES-deep smem ring, 128B swizzle
//   warp 1      MMA issuer  (one lane), tcgen05.mma.cta_group::1.kind::f16,
//               M=128 N=BN K=16, fp32 accumulators in TMEM (2 x BN columns,
//               double-buffered so the epilogue of tile i overlaps MMA of i+1)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
//
// Shape contract (enforced by the host wrapper): M % 128 == 0, N % BN == 0,
// K % 64 == 0, 16-byte aligned bases/strides.  The runtime pads rows/embed/
// hidden so every MoE shape satisfies it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace parm {
namespace gemm {

enum Major : int { kKMajor = 0, kMNMajor = 1 };
enum Epi : int { kEpiBF16 = 0, kEpiReluBF16 = 1, kEpiDReluBF16 = 2, kEpiF32 = 3, kEpiF32Acc = 4 };

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;
constexpr int kSmemBudget = 196 * 1024;

struct Params {
    int M, N, K, groups;
    int m_blocks, n_blocks, num_tiles;
    void* D;
    long long ldd, gsd;         // D row stride / group stride (elements)
    const bf16* aux;            // relu mask source for kEpiDReluBF16 (same shape as D)
    long long ld_aux, gs_aux;
    float alpha;                // D = alpha * A B^T (+ D for kEpiF32Acc)
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

// ---------------------------------------------------------------- the kernel
template <int BN, int MA, int MB, int EPI>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (kSmemBudget - 1024) / kStageBytes > 8 ? 8 : (kSmemBudget - 1024) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;
};

template <int BN, int MA, int MB, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const Params p) {
    using C = Cfg<BN, MA, MB, EPI>;
    constexpr int STAGES = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + STAGES * C::kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::kStageBytes);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmap_a);
        prefetch_tmap(&tmap_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull_bar[s], 1);
            mbar_init(&tempty_bar[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)C::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int k_blocks = p.K / BK;
    const int tiles_per_group = p.m_blocks * p.n_blocks;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
                const int g = tile / tiles_per_group;
                const int rem = tile - g * tiles_per_group;
                const int m0 = (rem / p.n_blocks) * BM;
                const int n0 = (rem % p.n_blocks) * BN;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    mbar_expect_tx(&full_bar[stage], C::kStageBytes);
                    const int k0 = kb * BK;
                    uint8_t* sa = smem_a + stage * C::kABytes;
                    uint8_t* sb = smem_b + stage * C::kBBytes;
                    if (MA == kKMajor) {
                        tma_load_3d(&tmap_a, &full_bar[stage], sa, k0, m0, g);
                    } else {
#pragma unroll
                        for (int a = 0; a < BM / 64; ++a)
                            tma_load_3d(&tmap_a, &full_bar[stage], sa + a * (BK * 128), m0 + a * 64, k0, g);
                    }
                    if (MB == kKMajor) {
                        tma_load_3d(&tmap_b, &full_bar[stage], sb, k0, n0, g);
                    } else {
#pragma unroll
                        for (int a = 0; a < BN / 64; ++a)
                            tma_load_3d(&tmap_b, &full_bar[stage], sb + a * (BK * 128), n0 + a * 64, k0, g);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = instr_desc<BN, MA, MB>();
            // K-major: 8-row core groups 1024 B apart, K advance of 16 elems = 32 B.
            // MN-major: 64-element MN atoms BK*128 B apart, K advance of 16 rows = 2048 B.
            constexpr uint32_t a_lbo = (MA == kKMajor) ? 0 : BK * 128;
            constexpr uint32_t b_lbo = (MB == kKMajor) ? 0 : BK * 128;
            constexpr uint32_t a_kstep = (MA == kKMajor) ? 32 : 16 * 128;
            constexpr uint32_t b_kstep = (MB == kKMajor) ? 32 : 16 * 128;
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
                const int as = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait(&tempty_bar[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + as * BN;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem_a + stage * C::kABytes);
                    const uint32_t sb = smem_u32(smem_b + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad = smem_desc(sa + k * a_kstep, a_lbo, 1024);
                        uint64_t bd = smem_desc(sb + k * b_kstep, b_lbo, 1024);
                        tc_mma(tmem_d, ad, bd, idesc, (kb | k) != 0);
                    }
                    tc_commit(&empty_bar[stage]);
                    if (kb == k_blocks - 1) tc_commit(&tfull_bar[as]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------- epilogue
        const int ew = warp & 3;  // TMEM lane quarter this warp may access
        int it = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
            const int g = tile / tiles_per_group;
            const int rem = tile - g * tiles_per_group;
            const int m0 = (rem / p.n_blocks) * BM;
            const int n0 = (rem % p.n_blocks) * BN;
            const int as = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            mbar_wait(&tfull_bar[as], aphase);
            tc_fence_after();
            const int row = m0 + ew * 32 + lane;
            const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + as * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                PARM_TMEM_LD32(taddr + c * 32, r);
                tmem_ld_wait();
                const int col = n0 + c * 32;
                if (EPI == kEpiF32 || EPI == kEpiF32Acc) {
                    float* dst = reinterpret_cast<float*>(p.D) + (long long)g * p.gsd + (long long)row * p.ldd + col;
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        float4 o = make_float4(p.alpha * __uint_as_float(r[4 * v]),
                                               p.alpha * __uint_as_float(r[4 * v + 1]),
                                               p.alpha * __uint_as_float(r[4 * v + 2]),
                                               p.alpha * __uint_as_float(r[4 * v + 3]));
                        if (EPI == kEpiF32Acc) {
                            float4 prev = reinterpret_cast<float4*>(dst)[v];
                            o.x += prev.x;
                            o.y += prev.y;
                            o.z += prev.z;
                            o.w += prev.w;
                        }
                        reinterpret_cast<float4*>(dst)[v] = o;
                    }
                } else {
                    bf16* dst = reinterpret_cast<bf16*>(p.D) + (long long)g * p.gsd + (long long)row * p.ldd + col;
                    float f[32];
#pragma unroll
                    for (int v = 0; v < 32; ++v) f[v] = p.alpha * __uint_as_float(r[v]);
                    if (EPI == kEpiReluBF16) {
#pragma unroll
                        for (int v = 0; v < 32; ++v) f[v] = fmaxf(f[v], 0.0f);
                    }
                    if (EPI == kEpiDReluBF16) {
                        const bf16* ax = p.aux + (long long)g * p.gs_aux + (long long)row * p.ld_aux + col;
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            float a[8];
                            vec8_to_f32(ld_vec8(ax + 8 * v), a);
#pragma unroll
                            for (int u = 0; u < 8; ++u) f[8 * v + u] = a[u] > 0.0f ? f[8 * v + u] : 0.0f;
                        }
                    }
#pragma unroll
                    for (int v = 0; v < 4; ++v) st_vec8(dst + 8 * v, f32_to_vec8(f + 8 * v));
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty_bar[as]);
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
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

// 3-D bf16 tensor map: dims {inner, outer, groups}, 128B swizzle, box {64, box_outer, 1}.
static int make_tmap(CUtensorMap* map, const void* base, long long inner, long long outer, long long groups,
                     long long ld_elems, long long gs_elems, int box_outer) {
    auto enc = get_encode();
    PARM_CHECK_ARG(enc != nullptr, "gemm: cuTensorMapEncodeTiled unavailable from the driver");
    PARM_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, "gemm: operand base not 16-byte aligned");
    PARM_CHECK_ARG((ld_elems * 2) % 16 == 0 && (gs_elems * 2) % 16 == 0, "gemm: strides not 16-byte multiples");
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)groups};
    cuuint64_t strides[2] = {(cuuint64_t)(ld_elems * 2), (cuuint64_t)((groups > 1 ? gs_elems : ld_elems * outer) * 2)};
    cuuint32_t box[3] = {64, (cuuint32_t)box_outer, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    PARM_CHECK_ARG(r == CUDA_SUCCESS, "gemm: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return 0;
}

template <int BN, int MA, int MB, int EPI>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, cudaStream_t stream) {
    using C = Cfg<BN, MA, MB, EPI>;
    auto kern = grouped_gemm_kernel<BN, MA, MB, EPI>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        attr_set = true;
    }
    int grid = p.num_tiles < kNumSMs ? p.num_tiles : kNumSMs;
    kern<<<grid, kThreads, C::kSmemBytes, stream>>>(ta, tb, p);
    PARM_CHECK_LAUNCH("grouped_gemm");
    return 0;
}

template <int MA, int MB, int EPI>
static int dispatch_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, cudaStream_t s) {
    if (bn == 256) return launch<256, MA, MB, EPI>(ta, tb, p, s);
    if (bn == 128) return launch<128, MA, MB, EPI>(ta, tb, p, s);
    return launch<64, MA, MB, EPI>(ta, tb, p, s);
}

}  // namespace gemm

// Public entry (wrapped by the C ABI in capi.cu).
int grouped_gemm(int major_a, int major_b, int epi, int M, int N, int K, int groups, const void* A, long long lda,
                 long long gsa, const void* B, long long ldb, long long gsb, void* D, long long ldd, long long gsd,
                 const void* aux, long long ld_aux, long long gs_aux, float alpha, cudaStream_t stream) {
    using namespace gemm;
    PARM_CHECK_ARG(M > 0 && N > 0 && K > 0 && groups > 0, "gemm: empty problem M=%d N=%d K=%d G=%d", M, N, K, groups);
    PARM_CHECK_ARG(M % BM == 0, "gemm: M=%d must be a multiple of %d", M, BM);
    PARM_CHECK_ARG(N % 64 == 0, "gemm: N=%d must be a multiple of 64", N);
    PARM_CHECK_ARG(K % BK == 0, "gemm: K=%d must be a multiple of %d", K, BK);
    PARM_CHECK_ARG(epi >= 0 && epi <= 4, "gemm: bad epilogue %d", epi);
    PARM_CHECK_ARG(epi != kEpiDReluBF16 || aux != nullptr, "gemm: relu-mask epilogue needs aux");
    const int bn = (N % 256 == 0) ? 256 : (N % 128 == 0 ? 128 : 64);
    CUtensorMap ta, tb;
    int rc;
    // A: K-major stored [g][m][k] (inner k); MN-major stored [g][k][m] (inner m).
    if (major_a == kKMajor)
        rc = make_tmap(&ta, A, K, M, groups, lda, gsa, BM);
    else
        rc = make_tmap(&ta, A, M, K, groups, lda, gsa, BK);
    if (rc) return rc;
    if (major_b == kKMajor)
        rc = make_tmap(&tb, B, K, N, groups, ldb, gsb, bn);
    else
        rc = make_tmap(&tb, B, N, K, groups, ldb, gsb, BK);
    if (rc) return rc;
    Params p;
    p.M = M;
    p.N = N;
    p.K = K;
    p.groups = groups;
    p.m_blocks = M / BM;
    p.n_blocks = N / bn;
    p.num_tiles = p.m_blocks * p.n_blocks * groups;
    p.D = D;
    p.ldd = ldd;
    p.gsd = gsd;
    p.aux = reinterpret_cast<const bf16*>(aux);
    p.ld_aux = ld_aux;
    p.gs_aux = gs_aux;
    p.alpha = alpha;
    const int combo = major_a * 2 + major_b;
    switch (combo) {
        case 0:  // K,K : forward GEMMs
            if (epi == kEpiReluBF16) return dispatch_bn<kKMajor, kKMajor, kEpiReluBF16>(bn, ta, tb, p, stream);
            if (epi == kEpiBF16) return dispatch_bn<kKMajor, kKMajor, kEpiBF16>(bn, ta, tb, p, stream);
            if (epi == kEpiF32) return dispatch_bn<kKMajor, kKMajor, kEpiF32>(bn, ta, tb, p, stream);
            break;
        case 1:  // K,MN : data-gradient GEMMs
            if (epi == kEpiDReluBF16) return dispatch_bn<kKMajor, kMNMajor, kEpiDReluBF16>(bn, ta, tb, p, stream);
            if (epi == kEpiBF16) return dispatch_bn<kKMajor, kMNMajor, kEpiBF16>(bn, ta, tb, p, stream);
            break;
        case 3:  // MN,MN : weight-gradient GEMMs
            if (epi == kEpiF32) return dispatch_bn<kMNMajor, kMNMajor, kEpiF32>(bn, ta, tb, p, stream);
            if (epi == kEpiF32Acc) return dispatch_bn<kMNMajor, kMNMajor, kEpiF32Acc>(bn, ta, tb, p, stream);
            break;
        default:
            break;
    }
    set_error("gemm: unsupported combination major_a=%d major_b=%d epi=%d", major_a, major_b, epi);
    return 1;
}

}  // namespace parm
