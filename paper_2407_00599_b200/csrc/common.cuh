// Shared device/host helpers for the Parm B200 MoE-layer kernels (sm_100a only).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdlib>
#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2407_00599_b200 kernels are written for sm_100a only"
#endif

namespace parm {

using bf16 = __nv_bfloat16;

// Host-side error channel behind parm_last_error(); thread-local so rank
// threads never see each other's messages.
void set_error(const char* fmt, ...);
const char* last_error();

#define PARM_CHECK_ARG(cond, ...)                 \
    do {                                          \
        if (!(cond)) {                            \
            ::parm::set_error(__VA_ARGS__);       \
            return 1;                             \
        }                                         \
    } while (0)

#define PARM_CHECK_LAUNCH(what)                                                   \
    do {                                                                          \
        cudaError_t e__ = cudaGetLastError();                                     \
        if (e__ != cudaSuccess) {                                                 \
            ::parm::set_error("%s: launch failed: %s", what, cudaGetErrorString(e__)); \
            return 2;                                                             \
        }                                                                         \
    } while (0)

constexpr int kNumSMs = 148;

// Kernel launch through cudaLaunchKernelEx (one place to attach launch attributes).
// Programmatic dependent launch was measured and left out: inside the graph-captured
// step every kernel's inputs come from the kernel before it, so only launch latency
// could overlap, and graph launches already hide that (0.764 vs 0.763 ms at N=1).
template <typename... Exp, typename... Act>
inline void launch_k(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Act&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// Cooperative launch (every CTA resident at once): for kernels with a grid-wide barrier.
template <typename... Exp, typename... Act>
inline cudaError_t launch_coop(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               Act&&... args) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// Two f32 FMAs in one FFMA2 (sm_100): (a0, a1) += (x0, x1) * w, each rounded as fmaf.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float w) {
    asm("{\n\t.reg .b64 ra, rx, rw;\n\t"
        "mov.b64 ra, {%0, %1};\n\tmov.b64 rx, {%2, %3};\n\tmov.b64 rw, {%4, %4};\n\t"
        "fma.rn.f32x2 ra, rx, rw, ra;\n\tmov.b64 {%0, %1}, ra;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(x0), "f"(x1), "f"(w));
}

__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

// 16-byte vector of 8 bf16 values.
struct alignas(16) Vec8 {
    __nv_bfloat162 h[4];
};

__device__ __forceinline__ Vec8 ld_vec8(const bf16* p) {
    Vec8 v;
    *reinterpret_cast<int4*>(&v) = __ldg(reinterpret_cast<const int4*>(p));
    return v;
}

__device__ __forceinline__ void st_vec8(bf16* p, const Vec8& v) {
    *reinterpret_cast<int4*>(p) = *reinterpret_cast<const int4*>(&v);
}

__device__ __forceinline__ void vec8_to_f32(const Vec8& v, float* f) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(v.h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

__device__ __forceinline__ Vec8 f32_to_vec8(const float* f) {
    Vec8 v;
#pragma unroll
    for (int i = 0; i < 4; ++i) v.h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// Addressing of a slot tensor that may be split across expert-parallel
// blocks, expert-sharding partial sources and MP slot shards.  Row of
// (expert e, slot s, partial p) lives at
//   ptr + (e / e_local) * stride_ep + (e % e_local) * stride_i + p * stride_p
//       + (s / slot_div) * stride_shi + (s % slot_div) * stride_slo
// (strides in elements).  Covers every receive layout the three schedules
// produce; n_p partials are summed in p order.
constexpr int kMaxPeers = 8;

struct SlotView {
    const bf16* ptr;
    int e_local;
    int n_p;
    int slot_div;
    int n_peer;                  // 0: local view.  > 0: rows live in peers' buffers (NVLink-mapped)
    long long stride_ep;
    long long stride_i;
    long long stride_p;
    long long stride_shi;
    long long stride_slo;
    const bf16* peer[kMaxPeers]; // n_peer > 0: partial (ep, p) is peer[ep * peer_ep + p * peer_p]
    int peer_ep;                 //   (+ the in-buffer offset of expert i_e, slot s); stride_ep/stride_p unused
    int peer_p;
};

// In-buffer offset of (expert e, slot s) excluding the block / partial terms.
__device__ __forceinline__ long long slot_inbuf(const SlotView& v, int e, int s, int& ep) {
    ep = e / v.e_local;
    const int i = e - ep * v.e_local;
    const int shi = s / v.slot_div;
    const int slo = s - shi * v.slot_div;
    return (long long)i * v.stride_i + (long long)shi * v.stride_shi + (long long)slo * v.stride_slo;
}

// Base of partial p of block ep (local: strides; peer view: that rank's mapped buffer).
__device__ __forceinline__ const bf16* slot_base(const SlotView& v, int ep, int p) {
    return v.n_peer ? v.peer[ep * v.peer_ep + p * v.peer_p]
                    : v.ptr + (long long)ep * v.stride_ep + (long long)p * v.stride_p;
}

__device__ __forceinline__ const bf16* slot_row(const SlotView& v, int e, int s, int p) {
    int ep;
    const long long off = slot_inbuf(v, e, s, ep);
    return slot_base(v, ep, p) + off;
}

// Output rows fanned out to up to kMaxPeers buffers with the same layout (a
// row written to every MP peer = the MP AllGather fused into the producer).
struct RowFan {
    bf16* ptr[kMaxPeers];
    int n;
    int pad_;
};

// Per-destination int tables (fill counts), indexed like SlotView::peer.
struct IntFan {
    int* ptr[kMaxPeers];
};

struct PeerSignal {
    void* pad[kMaxPeers];
    void* counter;
    int rank;
    int n;
    long long timeout_ns;
};

}  // namespace parm
