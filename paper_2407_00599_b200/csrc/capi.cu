// extern "C" boundary: plain pointers/sizes in, int status out (include/parm_b200.h).
#include <cstdarg>
#include <cstring>

#include "../../include/parm_b200.h"
#include "common.cuh"

namespace parm {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

const char* last_error() { return g_err; }

int gate_fwd(const void*, long long, const void*, int, int, int, int, int*, float*, float*, int*, cudaStream_t);
size_t gate_counts_bytes(int, int);
int route_dispatch(const void*, long long, const int*, const int*, int, int, int, int, int, int*, int*, int*, int, int,
                   void*, long long, long long, const SlotView*, const IntFan*, cudaStream_t);
size_t gate_wgrad_workspace(int, int, int);
int sum_chunks(const float*, int, long long, float*, int, cudaStream_t);
int gate_wgrad(const void*, long long, const float*, int, int, int, float*, size_t, float*, int, cudaStream_t);
int combine_fwd(const SlotView&, const int*, const int*, const float*, int, int, int, void*, long long, cudaStream_t);
int dispatch_bwd(const SlotView&, const int*, const int*, const float*, const void*, int, int, int, int, void*,
                 long long, cudaStream_t);
int combine_bwd_dispatch(const void*, long long, const SlotView&, const int*, const int*, const float*, const float*,
                         int, int, int, int, float*, int, int, const int*, void*, long long, long long, const SlotView*,
                         cudaStream_t);
int esp_sum(const SlotView&, int, int, int, void*, cudaStream_t);
int moe_gemm(const parm_gemm_desc&, cudaStream_t);
int moe_gemm_peer(const parm_gemm_desc&, const RowFan*, long long, long long, cudaStream_t);
size_t moe_gemm_multi_workspace(const parm_gemm_desc*, int);
int moe_gemm_multi(const parm_gemm_desc*, int, const int*, void*, size_t, int, const RowFan*, long long, long long,
                   cudaStream_t);
int combine_fwd_fan(const SlotView&, const int*, const int*, const float*, int, int, int, const RowFan&, long long,
                    cudaStream_t);
int dispatch_bwd_fan(const SlotView&, const int*, const int*, const float*, const void*, int, int, int, int,
                     const RowFan&, long long, cudaStream_t);
int peer_barrier(const PeerSignal*, int, cudaStream_t);
int push_rows(const void*, int, int, int, int, const int*, const RowFan&, cudaStream_t);
int fan_copy(const void*, long long, const RowFan&, cudaStream_t);

template <class A, class B>
static A abi_cast(const B* v) {
    static_assert(sizeof(A) == sizeof(B), "C ABI struct layout mismatch");
    A a;
    std::memcpy(&a, v, sizeof(a));
    return a;
}

static SlotView to_view(const parm_slot_view* v) {
    SlotView s;
    static_assert(sizeof(SlotView) == sizeof(parm_slot_view), "slot view ABI mismatch");
    std::memcpy(&s, v, sizeof(s));
    return s;
}

}  // namespace parm

using parm::to_view;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int parm_abi_version(void) { return PARM_ABI_VERSION; }

const char* parm_last_error(void) { return parm::last_error(); }

int parm_gate_fwd(const void* x, long long ldx, const void* wg, int n, int M, int E, int k, int* expert_idx,
                  float* combine_w, float* probs, int* tile_counts, void* stream) {
    return parm::gate_fwd(x, ldx, wg, n, M, E, k, expert_idx, combine_w, probs, tile_counts, S(stream));
}

size_t parm_gate_counts_bytes(int n, int E) { return parm::gate_counts_bytes(n, E); }

int parm_route_dispatch(const void* x, long long ldx, const int* expert_idx, const int* tile_counts, int n, int k,
                        int E, int cap, int M, int* slot_idx, int* slot_src, int* fill, int slot_lo, int slots_out,
                        void* out, long long out_stride_e, long long out_stride_s, const parm_slot_view* dst,
                        const parm_int_fan* fill_dst, void* stream) {
    parm::SlotView v;
    parm::IntFan f;
    if (dst) v = to_view(dst);
    if (fill_dst) f = parm::abi_cast<parm::IntFan>(fill_dst);
    return parm::route_dispatch(x, ldx, expert_idx, tile_counts, n, k, E, cap, M, slot_idx, slot_src, fill, slot_lo,
                                slots_out, out, out_stride_e, out_stride_s, dst ? &v : nullptr,
                                fill_dst ? &f : nullptr, S(stream));
}

int parm_combine_fwd(const parm_slot_view* y, const int* expert_idx, const int* slot_idx, const float* combine_w,
                     int n, int k, int M, void* out, long long ldo, void* stream) {
    if (!y) {
        parm::set_error("combine_fwd: null slot view");
        return 1;
    }
    return parm::combine_fwd(to_view(y), expert_idx, slot_idx, combine_w, n, k, M, out, ldo, S(stream));
}

int parm_combine_bwd_dispatch(const void* dout, long long ld_dout, const parm_slot_view* y, const int* expert_idx,
                              const int* slot_idx, const float* probs, const float* combine_w, int n, int k, int E,
                              int M, float* dlogits, int slot_lo, int slots_out, const int* fill, void* out,
                              long long out_stride_e, long long out_stride_s, const parm_slot_view* dst,
                              void* stream) {
    if (!y) {
        parm::set_error("combine_bwd_dispatch: null slot view");
        return 1;
    }
    parm::SlotView dv{};
    if (dst) dv = to_view(dst);
    return parm::combine_bwd_dispatch(dout, ld_dout, to_view(y), expert_idx, slot_idx, probs, combine_w, n, k, E, M,
                                      dlogits, slot_lo, slots_out, fill, out, out_stride_e, out_stride_s,
                                      dst ? &dv : nullptr, S(stream));
}

int parm_dispatch_bwd(const parm_slot_view* dr, const int* expert_idx, const int* slot_idx, const float* dlogits,
                      const void* wg, int n, int k, int E, int M, void* dx, long long ldx, void* stream) {
    if (!dr) {
        parm::set_error("dispatch_bwd: null slot view");
        return 1;
    }
    return parm::dispatch_bwd(to_view(dr), expert_idx, slot_idx, dlogits, wg, n, k, E, M, dx, ldx, S(stream));
}

int parm_esp_sum(const parm_slot_view* y, int E, int slots, int M, void* out, void* stream) {
    if (!y) {
        parm::set_error("esp_sum: null slot view");
        return 1;
    }
    return parm::esp_sum(to_view(y), E, slots, M, out, S(stream));
}

size_t parm_gate_wgrad_workspace(int n, int M, int E) { return parm::gate_wgrad_workspace(n, M, E); }

int parm_sum_chunks(const float* src, int chunks, long long len, float* out, int accumulate, void* stream) {
    return parm::sum_chunks(src, chunks, len, out, accumulate, S(stream));
}

int parm_gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, void* workspace,
                    size_t workspace_bytes, float* dwg, int accumulate, void* stream) {
    return parm::gate_wgrad(x, ldx, dlogits, n, M, E, reinterpret_cast<float*>(workspace), workspace_bytes, dwg,
                            accumulate, S(stream));
}

int parm_combine_fwd_fan(const parm_slot_view* y, const int* expert_idx, const int* slot_idx, const float* combine_w,
                         int n, int k, int M, const parm_row_fan* out, long long ldo, void* stream) {
    if (!y || !out) {
        parm::set_error("combine_fwd: null slot view or output fan");
        return 1;
    }
    return parm::combine_fwd_fan(to_view(y), expert_idx, slot_idx, combine_w, n, k, M,
                                 parm::abi_cast<parm::RowFan>(out), ldo, S(stream));
}

int parm_dispatch_bwd_fan(const parm_slot_view* dr, const int* expert_idx, const int* slot_idx, const float* dlogits,
                          const void* wg, int n, int k, int E, int M, const parm_row_fan* dx, long long ldx,
                          void* stream) {
    if (!dr || !dx) {
        parm::set_error("dispatch_bwd: null slot view or output fan");
        return 1;
    }
    return parm::dispatch_bwd_fan(to_view(dr), expert_idx, slot_idx, dlogits, wg, n, k, E, M,
                                  parm::abi_cast<parm::RowFan>(dx), ldx, S(stream));
}

int parm_push_rows(const void* src, int nseg, int e_local, int rows, int M, const int* fill, const parm_row_fan* dst,
                   void* stream) {
    if (!dst) {
        parm::set_error("push_rows: null destination fan");
        return 1;
    }
    return parm::push_rows(src, nseg, e_local, rows, M, fill, parm::abi_cast<parm::RowFan>(dst), S(stream));
}

int parm_fan_copy(const void* src, long long bytes, const parm_row_fan* dst, void* stream) {
    if (!dst) {
        parm::set_error("fan_copy: null destination fan");
        return 1;
    }
    return parm::fan_copy(src, bytes, parm::abi_cast<parm::RowFan>(dst), S(stream));
}

int parm_peer_barrier(const parm_peer_signal* sigs, int count, void* stream) {
    if (!sigs || count < 1 || count > PARM_MAX_PEERS) {
        parm::set_error("peer_barrier: need 1..%d signal descriptors (got %d)", PARM_MAX_PEERS, count);
        return 1;
    }
    parm::PeerSignal g[PARM_MAX_PEERS];
    static_assert(sizeof(parm::PeerSignal) == sizeof(parm_peer_signal), "peer signal ABI mismatch");
    std::memcpy(g, sigs, sizeof(parm_peer_signal) * count);
    return parm::peer_barrier(g, count, S(stream));
}

int parm_gemm(const parm_gemm_desc* desc, void* stream) {
    if (!desc) {
        parm::set_error("gemm: null descriptor");
        return 1;
    }
    return parm::moe_gemm(*desc, S(stream));
}

int parm_gemm_peer(const parm_gemm_desc* desc, const parm_row_fan* seg_dst, long long dst_g_stride, long long dst_ld,
                   void* stream) {
    if (!desc || !seg_dst) {
        parm::set_error("gemm_peer: null descriptor or destination fan");
        return 1;
    }
    const parm::RowFan fan = parm::abi_cast<parm::RowFan>(seg_dst);
    return parm::moe_gemm_peer(*desc, &fan, dst_g_stride, dst_ld, S(stream));
}

size_t parm_gemm_multi_workspace(const parm_gemm_desc* descs, int count) {
    if (!descs || count < 1) return 0;
    return parm::moe_gemm_multi_workspace(descs, count);
}

int parm_gemm_multi(const parm_gemm_desc* descs, int count, const int* deps, void* ws, size_t ws_bytes, int seg_prob,
                    const parm_row_fan* seg_dst, long long dst_g_stride, long long dst_ld, void* stream) {
    if (!descs) {
        parm::set_error("gemm_multi: null descriptors");
        return 1;
    }
    parm::RowFan fan{};
    if (seg_prob >= 0) {
        if (!seg_dst) {
            parm::set_error("gemm_multi: peer-output problem %d without a destination fan", seg_prob);
            return 1;
        }
        fan = parm::abi_cast<parm::RowFan>(seg_dst);
    }
    return parm::moe_gemm_multi(descs, count, deps, ws, ws_bytes, seg_prob, seg_prob >= 0 ? &fan : nullptr,
                                dst_g_stride, dst_ld, S(stream));
}

}  // extern "C"
