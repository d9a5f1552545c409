/*
 * parm_b200.h — C ABI of the B200-native Parm MoE-layer hot path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * (passed as void*), is stream-ordered, never synchronises the host and never
 * allocates: the caller (the PyTorch host layer, or any FFI binding) owns all
 * memory, including workspaces sized by the *_workspace() queries.  Status is
 * an int (0 = ok, 1 = bad argument, 2 = launch failure); the message of the
 * last failure on the calling thread is returned by parm_last_error().
 *
 * The reference (/root/reference, `moesched`) is pure Python/NumPy, so it has
 * no native FFI of its own; each function below cites the reference Python
 * interface whose work it replaces.  INTEGRATION.md shows the ctypes binding.
 */
#ifndef PARM_B200_H
#define PARM_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARM_ABI_VERSION 16

/* Addressing of a slot tensor split over expert-parallel blocks, expert-
 * sharding partials (summed in p order) and MP slot shards:
 *   row(e, s, p) = base(e / e_local, p) + (e % e_local) * stride_i
 *                + (s / slot_div) * stride_shi + (s % slot_div) * stride_slo
 * with base(ep, p) = ptr + ep * stride_ep + p * stride_p for a local view
 * (n_peer == 0), or peer[ep * peer_ep + p * peer_p] when the rows live in other
 * GPUs' buffers mapped into this process (symmetric memory over NVLink;
 * n_peer > 0).  Element strides. */
#define PARM_MAX_PEERS 8
typedef struct parm_slot_view {
    const void* ptr; /* bf16 */
    int e_local;
    int n_p;
    int slot_div;
    int n_peer;
    long long stride_ep;
    long long stride_i;
    long long stride_p;
    long long stride_shi;
    long long stride_slo;
    const void* peer[PARM_MAX_PEERS];
    int peer_ep;
    int peer_p;
} parm_slot_view;

/* Output rows written to n buffers of identical layout (fused AllGather). */
typedef struct parm_row_fan {
    void* ptr[PARM_MAX_PEERS]; /* bf16 */
    int n;
    int pad_;
} parm_row_fan;

/* Per-destination int32 tables, indexed like parm_slot_view.peer. */
typedef struct parm_int_fan {
    int* ptr[PARM_MAX_PEERS];
} parm_int_fan;

/* Device-side barrier over peers' signal pads (symmetric memory). */
typedef struct parm_peer_signal {
    void* pad[PARM_MAX_PEERS]; /* uint32 slots, this rank writes pad[j][rank] */
    void* counter;             /* uint32 on this device: epoch, advanced by every barrier */
    int rank;
    int n;
    long long timeout_ns;      /* a waiting rank traps after this long without every peer (<= 0: 300 s);
                                  host-side skew between ranks (checkpoints, eval) must stay inside it */
} parm_peer_signal;

int parm_abi_version(void);
const char* parm_last_error(void);

/* Gate, forward: logits (f64 accumulation of bf16 inputs -- every product exact,
 * FP64 tensor cores), softmax, stable top-k.  Replaces moesched.dataplane.gate
 * (dataplane.py:86-103).
 * x: (n, M) bf16 row stride ldx; wg_t: gate weights TRANSPOSED, (E, M) bf16.
 * Outputs: expert_idx (n, k) int32 in selection order, combine_w (n, k) f32
 * (= softmax score of the pick), probs (n, E) f32 (nullable), tile_counts
 * (nullable, parm_gate_counts_bytes(n, E) bytes): per 8-token tile, the number of
 * its tokens that picked each expert -- the input of parm_route_dispatch. */
int parm_gate_fwd(const void* x, long long ldx, const void* wg_t, int n, int M, int E, int k, int* expert_idx,
                  float* combine_w, float* probs, int* tile_counts, void* stream);
size_t parm_gate_counts_bytes(int n, int E);

/* Slot pass + dispatch in one kernel: token-major capacity fill (dataplane.py:104-116)
 * from the gate's tile counts -> slot_idx (n, k) int32 (-1 = dropped), slot_src (E, cap)
 * int32 (= t*k+j of the pick in (e, slot), -1 unfilled), fill (E); and every kept pick
 * with slot s in [slot_lo, slot_lo + slots_out) copies its token row to row (e, s - slot_lo)
 * of `out` (E x slots_out rows, strides in elements) -- or, with `dst` (peer view, n_p =
 * N_ESP dump copies), straight into the holders' receive buffers over NVLink, with the
 * per-segment fill counts stored into fill_dst (the EP&ESP dispatch AlltoAll fused,
 * collectives.py:256-283).  Without `dst`, fill_dst (nullable) gets the (E) per-expert fill
 * of the slot range in ptr[0]; with neither `out` nor `dst` only the slot pass runs.
 * Rows between each expert's (segment) fill and its last 128-row GEMM tile are zeroed;
 * rows beyond are not touched.  Replaces the
 * GateOutput.dispatch fill (dataplane.py:101,112) and S2's slot split + pad
 * (dataplane.py:373-378). */
int parm_route_dispatch(const void* x, long long ldx, const int* expert_idx, const int* tile_counts, int n, int k,
                        int E, int cap, int M, int* slot_idx, int* slot_src, int* fill, int slot_lo, int slots_out,
                        void* out, long long out_stride_e, long long out_stride_s, const parm_slot_view* dst,
                        const parm_int_fan* fill_dst, void* stream);

/* Combine: out[t] = sum_j combine_w[t,j] * sum_p Y_p[e_j, s_j] (dropped
 * picks contribute 0).  Fuses fused_combine's local ESP sum
 * (collectives.py:296-310) with _combine (dataplane.py:131-143). */
int parm_combine_fwd(const parm_slot_view* y, const int* expert_idx, const int* slot_idx, const float* combine_w,
                     int n, int k, int M, void* out, long long ldo, void* stream);

/* Combine backward fused with the backward dispatch of dOut: the softmax adjoint
 * dlogits[t, e] = p_e (dS_e - sum_e' p_e' dS_e') with dS_e = <dOut[t], sum_p Y_p[e, s]>
 * on the kept picks (no reference: SURVEY §8 a27), and in the same pass over dOut the
 * slot rows -- row (e, s - slot_lo) <- combine_w[t, j] * dOut[t] for each kept pick with
 * s in [slot_lo, slot_lo + slots_out), zero rows up to each expert's last 128-row GEMM
 * tile.  Rows go to out (+ e * out_stride_e + s * out_stride_s) or, when dst is
 * non-null, to the N_ESP holders through the peer view (the EP&ESP AlltoAll fused, as
 * in parm_route_dispatch).  One read of dOut, one launch. */
int parm_combine_bwd_dispatch(const void* dout, long long ld_dout, const parm_slot_view* y, const int* expert_idx,
                              const int* slot_idx, const float* probs, const float* combine_w, int n, int k, int E,
                              int M, float* dlogits, int slot_lo, int slots_out, const int* fill, void* out,
                              long long out_stride_e, long long out_stride_s, const parm_slot_view* dst,
                              void* stream);

/* Dispatch backward: dx[t] = sum_j sum_p dR_p[e_j, s_j] + dlogits[t] . Wg^T
 * (dlogits nullable; wg_t is the (E, M) bf16 gate weights, transposed).
 * Adjoint of the dump + dispatch fill. */
int parm_dispatch_bwd(const parm_slot_view* dr, const int* expert_idx, const int* slot_idx, const float* dlogits,
                      const void* wg_t, int n, int k, int E, int M, void* dx, long long ldx, void* stream);

/* S2: out (E, slots, M) = sum_p Y_p[e, s], the ESP sum of fused_combine
 * (collectives.py:302-310) materialised before the MP AllGather. */
int parm_esp_sum(const parm_slot_view* y, int E, int slots, int M, void* out, void* stream);

/* ---- peer-memory (NVLink symmetric buffers) variants: the collective fused
 * into the kernel that produces or consumes the rows.  Buffers are mapped
 * into this process (torch symmetric memory / CUDA IPC); the caller orders
 * them with parm_peer_barrier. */

/* combine_fwd reading the expert outputs through a (peer) view -- the return
 * AlltoAll + ESP sum fused into the combine -- and writing each output row to
 * out->n buffers (the MP AllGather fused into the producer). */
int parm_combine_fwd_fan(const parm_slot_view* y, const int* expert_idx, const int* slot_idx, const float* combine_w,
                         int n, int k, int M, const parm_row_fan* out, long long ldo, void* stream);

/* dispatch_bwd with the same fusions (return AlltoAll of dR + MP AllGather of dx). */
int parm_dispatch_bwd_fan(const parm_slot_view* dr, const int* expert_idx, const int* slot_idx, const float* dlogits,
                          const void* wg_t, int n, int k, int E, int M, const parm_row_fan* dx, long long ldx,
                          void* stream);

/* Return AlltoAll as a push: holder rows src[seg][i][s] (segment = source
 * rank, s < fill[seg * e_local + i]) stored into dst->ptr[seg] + (i * rows + s) * M,
 * the owner's receive block for this holder (fused_combine's exchange,
 * collectives.py:286-295). */
int parm_push_rows(const void* src, int nseg, int e_local, int rows, int M, const int* fill, const parm_row_fan* dst,
                   void* stream);

/* `bytes` of src replicated into dst->ptr[0..n) (16-byte aligned): small payloads sent to
 * every MP peer, e.g. S1's gate-weight gradient partials (replaces its MP all-reduce). */
int parm_fan_copy(const void* src, long long bytes, const parm_row_fan* dst, void* stream);

/* Device-side barrier of the n peers (one tiny kernel; graph-capturable).  sigs[0..count)
 * are the ranks this process hosts: 1 for one rank per GPU; a single-GPU emulation of
 * all n ranks passes n descriptors and gets ONE cooperative launch with a CTA per rank,
 * so ranks that wait on one another are co-resident by construction. */
int parm_peer_barrier(const parm_peer_signal* sigs, int count, void* stream);

/* Gate weight gradient, transposed: dWg^T (E, M) f32 = dlogits^T x (deterministic: per-SM
 * partials summed in a fixed order, in the same launch behind a grid barrier when every CTA is
 * resident).  accumulate != 0 adds into dwg.  workspace: parm_gate_wgrad_workspace() bytes,
 * zeroed once by the caller (it ends with barrier counters the kernel leaves zeroed; launches
 * sharing a workspace must be stream-ordered). */
size_t parm_gate_wgrad_workspace(int n, int M, int E);
/* out[i] (+)= sum_c src[c * len + i], chunks summed in a fixed order (deterministic): the S1
 * peer transport's MP gate-gradient partials, fanned out to every MP peer, reduced locally
 * (replaces the MP all-reduce of the gate gradient). */
int parm_sum_chunks(const float* src, int chunks, long long len, float* out, int accumulate, void* stream);
int parm_gate_wgrad(const void* x, long long ldx, const float* dlogits, int n, int M, int E, void* workspace,
                    size_t workspace_bytes, float* dwg_t, int accumulate, void* stream);

/* A bf16/f32 tensor addressed as [hi][lo][g][row][col]: element (hi, lo, g, r, c)
 * at ptr + hi*hi_stride + lo*lo_stride + g*g_stride + r*ld + c (element strides).
 * Plain 3-D [g][row][col] tensors set hi/lo strides to 0 (nhi = nlo = 1). */
typedef struct parm_rows {
    const void* ptr;
    long long ld;
    long long g_stride;
    long long lo_stride;
    long long hi_stride;
} parm_rows;

/* Grouped tcgen05/TMEM/TMA GEMM over the MoE layer's segmented expert rows
 * (every row tensor is the AlltoAll receive layout [src_hi][src_lo][expert][r < seg_len][col]).
 * kind 0 (ROW):  D[hi][lo][g][r][n] = alpha * sum_k A[hi][lo][g][r][k] * B[g][n][k]
 *                b_major 0: B stored [g][n][k]; 1: B stored [g][k][n].  K % 64 == 0, N % 128 == 0.
 *                epi 0 bf16, 1 relu -> bf16, 2 keep where aux > 0 -> bf16 (aux shaped like D),
 *                5 relu -> bf16 and aux (u32 rows of N/32 words) <- bit mask of the stored
 *                values > 0, 6 keep where that bit mask is set -> bf16.
 * kind 1 (WGT):  D[g][m][n] = alpha * sum_{hi,lo,r} A[hi][lo][g][r][m] * B[hi][lo][g][r][n]
 *                M % 128 == 0, N % 128 == 0; epi 3 f32, 4 f32 accumulate.
 * fill (nullable, int32 [hi][lo][g]): rows >= fill of a segment are skipped
 * (capacity padding); they must be zero in A for ROW partial tiles.
 * Replaces expert_shard_forward (dataplane.py:122-128) and its adjoints. */
typedef struct parm_gemm_desc {
    int kind;
    int epi;
    int b_major;
    int groups;
    int nhi;
    int nlo;
    int seg_len;
    int M;
    int N;
    int K;
    float alpha;
    int pad_;
    parm_rows a;
    parm_rows b;
    parm_rows d;
    parm_rows aux;
    const int* fill;
} parm_gemm_desc;

int parm_gemm(const parm_gemm_desc* desc, void* stream);

/* ROW GEMM whose output rows of segment (hi, lo) go straight to seg_dst->ptr[hi * nlo + lo]
 * + g * dst_g_stride + r * dst_ld (elements; bf16 epilogues): with peer addresses the
 * expert output is stored into every owner's receive block from the epilogue -- the
 * return AlltoAll (collectives.py:286-295) fused into the GEMM, tile by tile. */
int parm_gemm_peer(const parm_gemm_desc* desc, const parm_row_fan* seg_dst, long long dst_g_stride, long long dst_ld,
                   void* stream);

/* Several GEMMs (1..4) as ONE persistent launch over one queue of pair tiles, problem after
 * problem, walked round-robin by the resident CTA pairs: one GEMM's partial last wave is filled by
 * the next GEMM's tiles (the expert FFN's forward pair Y = relu(R W1) W2, or its backward
 * dH, dW2, dR, dW1 -- dataplane.py:122-128 and the adjoints).  deps (nullable): 2 ints per
 * problem, (kind, earlier problem):
 *   PARM_DEP_ROW_PAIR   ROW problem reads rows of the same 256-row pair of the earlier ROW
 *                       problem's output over all its columns (waits for that pair's tiles);
 *   PARM_DEP_COL_BLOCK  WGT problem reads columns [256 p, 256 p + 256) of the earlier ROW
 *                       problem's output for every row of its group (p = its 256-row block).
 * Dependent and depended-on problems must share groups, segments, seg_len and fill.  With
 * dependencies the launch is cooperative (all CTAs resident) and needs ws:
 * parm_gemm_multi_workspace() bytes, zeroed once by the caller; the kernel leaves it zeroed
 * (launches sharing a workspace must be stream-ordered).  seg_prob (-1: none): that problem's
 * outputs go to seg_dst as in parm_gemm_peer. */
#define PARM_DEP_NONE 0
#define PARM_DEP_ROW_PAIR 1
#define PARM_DEP_COL_BLOCK 2
size_t parm_gemm_multi_workspace(const parm_gemm_desc* descs, int count);
int parm_gemm_multi(const parm_gemm_desc* descs, int count, const int* deps, void* ws, size_t ws_bytes, int seg_prob,
                    const parm_row_fan* seg_dst, long long dst_g_stride, long long dst_ld, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PARM_B200_H */
