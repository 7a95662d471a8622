/*
 * smoe_b200.h — C ABI of libsmoe_b200.so, the B200 (sm_100a) implementation of
 * the ScatterMoE ParallelLinear hot path.
 *
 * Each entry point replaces one function of the reference package
 * `scattermlp` (/root/reference/pkg/src/scattermlp); the reference interface it
 * stands in for is cited above each declaration.  The reference is an
 * in-process Python/NumPy API, so the "FFI" a maintainer would bind is a
 * ctypes shim; the Python package
 * `paper_2403_08245_b200` is exactly that shim plus the reference's host logic.
 *
 * Conventions (all functions):
 *   - every pointer is a DEVICE pointer unless stated otherwise;
 *   - the library never allocates device memory: the caller passes every
 *     output and workspace buffer (reference `out=` discipline,
 *     kernels.py:186-197, parallel_linear.py:144-154);
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*) and is
 *     asynchronous; no call synchronises the host, so every call is CUDA-graph
 *     capturable;
 *   - sizes are int64; index tensors (orders, offsets, inverse) are int32
 *     (n = T*k < 2^31);
 *   - rows are dense row-major with the stated column count as the row stride;
 *   - return value is an smoe_status; on failure smoe_get_last_error() returns
 *     a thread-local message naming the offending argument / shapes.
 */
#ifndef SMOE_B200_H
#define SMOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMOE_ABI_VERSION 4

typedef enum {
  SMOE_OK = 0,
  SMOE_EINVAL = 1,  /* bad argument value  (reference: ValueError)            */
  SMOE_ESHAPE = 2,  /* shape mismatch      (reference: DimensionError, errors.py:12-19) */
  SMOE_ECUDA = 3,   /* CUDA launch / runtime failure                         */
  SMOE_ENOTSUP = 4  /* valid but unsupported combination on this build        */
} smoe_status;

/* Storage dtypes.  bf16: tcgen05 tensor cores, fp32 accumulation (the product
 * path).  F32: the check mode — SIMT kernels with 64-bit accumulation and one
 * rounding, the reference's numeric contract (core_tensor.py:1-7).  F64: the
 * reference's float64 verification dtype (its finite-difference gradient
 * checks), SIMT only.  Per-slot weights (group weights, combine weights p) and
 * dp are float32 except with SMOE_F64 storage, where they are float64. */
typedef enum { SMOE_F32 = 0, SMOE_BF16 = 1, SMOE_F64 = 2 } smoe_dtype;

/* Activations of moe_layers.py:42-72 (exact-erf GELU, ReLU, SiLU). */
typedef enum { SMOE_ACT_GELU = 0, SMOE_ACT_RELU = 1, SMOE_ACT_SILU = 2,
               /* identity: only for smoe_scatter2scatter_scaled (a routed linear with
                  combine weights; the dp partials of its input-gradient epilogue) */
               SMOE_ACT_IDENTITY = 3 } smoe_activation;

/* scatter2scatter epilogues (fusions of moe_layers.py:169-175 and :205-206). */
typedef enum {
  SMOE_EPI_NONE = 0,     /* out[dst] = acc                                          */
  SMOE_EPI_ACT = 1,      /* out[dst] = pre = acc;  out2[dst] = act(pre)             */
  SMOE_EPI_ACT_GRAD = 2, /* out[dst] = acc * act'(aux[dst])   (aux = h_pre)         */
  SMOE_EPI_ACT_ONLY = 3, /* out[dst] = act(acc)  (inference: no pre-activation kept)  */
  /* smoe_scatter2scatter_scaled only (row i's scale s = row_scale[order[i]]): */
  SMOE_EPI_ACT_SCALED = 4,     /* out = pre = acc;  out2 = s * act(pre)                      */
  SMOE_EPI_ACT_GRAD_SCALED = 5 /* out = s * acc * act'(aux);  dp_part[i, part] =
                                  sum over the part's columns of acc * act(aux)                */
} smoe_epilogue;

/* GEMM engine selection: AUTO runs bf16 on tcgen05 and the fp32 / fp64 check
 * modes on the SIMT kernels.  There is no silent fallback: a bf16 call the
 * tcgen05 engine cannot take (d_in or d_out not a multiple of 8, a buffer not
 * 16-byte aligned, more than 1024 experts, no sm_100a device) returns
 * SMOE_ENOTSUP.  SMOE_ENGINE_SIMT runs bf16 on the SIMT kernels only when
 * asked for explicitly (the tests' cross-check of the tcgen05 engine). */
typedef enum { SMOE_ENGINE_AUTO = 0, SMOE_ENGINE_SIMT = 1, SMOE_ENGINE_TCGEN05 = 2 } smoe_engine;

const char *smoe_get_last_error(void);
int smoe_abi_version(void);
/* Number of kernels this library has enqueued since load (all threads). */
uint64_t smoe_launch_count(void);

/* ---------------------------------------------------------------------------
 * Routing: replaces router.compute_grouped_order (router.py:154-164) and
 * GroupedOrder.inverse (router.py:112-116); north_star name flatten_and_sort.
 *   expert_idx            [n] int64 (the T x k routing ids, token-major)
 *   sorted_scattered_idxs [n] int32 (GroupedOrder.o: stable argsort)
 *   sorted_expert_idxs    [n] int32 (expert id at each grouped position)
 *   expert_offsets        [E+1] int32 (GroupedOrder.bin_offsets)
 *   inverse               [n] int32 or NULL (scattered slot -> grouped pos)
 * Returns SMOE_EINVAL (no device check) when ids fall outside [0,E) — ids are
 * validated on the host side of the shim, as RoutingResult.__post_init__ does.
 */
size_t smoe_route_sort_workspace_bytes(int64_t n, int32_t num_experts);
int smoe_route_sort(const int64_t *expert_idx, int64_t n, int32_t num_experts,
                    int32_t *sorted_scattered_idxs, int32_t *sorted_expert_idxs,
                    int32_t *expert_offsets, int32_t *inverse, void *workspace,
                    size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Router, the step in front of the sort.
 * smoe_router_topk replaces softmax_rows + topk_select (router.py:126-151) and,
 * with apply_softmax, gate_forward's softmax (router.py:119-123; the gate GEMM
 * itself is a plain library matmul):
 *   in        [T, E] float32 logits (apply_softmax=1) or gate probabilities
 *   gate_out  [T, E] float32 softmax output, or NULL
 *   expert_idx[T, k] int64: k largest gates, ties -> lower expert id (k <= 8)
 *   p         [T, k] float32: selected gates, renormalised in float64 if asked
 * smoe_router_backward replaces gate_backward (router.py:167-188):
 *   dlogits [T, E] float32 from grad_p [T, k] through renormalisation + softmax.
 */
int smoe_router_topk(const float *in, int64_t T, int32_t num_experts, int32_t k, int32_t apply_softmax,
                     int32_t renormalize, float *gate_out, int64_t *expert_idx, float *p, void *stream);
/* SMs the persistent tcgen05 GEMMs leave free for kernels running concurrently
 * on other streams (e.g. NCCL all-to-all chunks overlapping an expert GEMM);
 * rounded down to whole CTA pairs; default 0.  Process-wide. */
int smoe_set_sm_reserve(int32_t sms);

/* Gate GEMM fused into the router (router.py:119-151):
 * logits = x @ w_gate accumulated in float64 (never rounded), softmax in float64
 * rounded once to float32 (gate_out [T, E], may be NULL), stable top-k on the
 * float32 gates (ties -> lower id) into expert_idx [T, k] int64, p [T, k]
 * renormalised in float64 when `renormalize`.  x [T, d_model] bf16 or fp32
 * (x_dtype); w_gate [d_model, E] fp32; k <= 8.
 * The ids feed smoe_route_sort directly. */
int smoe_router_gate(const void *x, int32_t x_dtype, const float *w_gate, int64_t T, int32_t d_model,
                     int32_t num_experts, int32_t k, int32_t renormalize, float *gate_out, int64_t *expert_idx,
                     float *p, void *stream);
int smoe_router_backward(const float *gate, const int64_t *expert_idx, const float *grad_p, int64_t T,
                         int32_t num_experts, int32_t k, int32_t renormalized, float *dlogits, void *stream);

/* ---------------------------------------------------------------------------
 * scatter2scatter (kernels.py:143-220): for each grouped position i in bin e,
 *   src = grouped_in ? i : order[i] / fan_out
 *   dst = grouped_out ? i : order[i]
 *   out[dst] = x[src] @ (transpose_w ? W[e]^T : W[e])   (+ epilogue)
 *   x        [x_rows, d_in]           x_rows = n (grouped_in) or n / fan_out
 *   w        [E, w_rows, w_cols]      d_in,d_out = (w_rows,w_cols) or swapped
 *   out/out2 [n, d_out]               aux [n, d_out] (EPI_ACT_GRAD only)
 * dtype applies to x, w, out, out2, aux.  Accumulation is fp32.
 */
int smoe_scatter2scatter(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                         int64_t w_rows, int64_t w_cols, const int32_t *order,
                         const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                         int32_t grouped_in, int32_t grouped_out, int32_t transpose_w,
                         int32_t dtype, int32_t epilogue, int32_t activation, void *out,
                         void *out2, const void *aux, int32_t engine, void *stream);

/* group (kernels.py:289-326) visited by source row: out[inverse[s]] =
 * x[s / fan_out] * (weights ? weights[s] : 1) for every slot s (fan_out <= 16;
 * inverse = the grouped position of each slot, from smoe_route_sort).  Each
 * source row is read once instead of once per expert bin. */
/* MoMHA query gradient in grouped order (the query projection's backward,
 * moe_layers.py:468-473 + parallel_linear.py:208-222): row i of out is the slot
 * s = order[i] (token t = s / k, choice j = s % k) read from the attention
 * core's head layout heads[batch][hh * k + j][t % seq_len][0:d_head] for
 * hh = 0 .. heads_per_slot - 1, i.e. out[i] = the slot's d_proj-wide row.  One
 * pass replaces the head->slot permute and the grouped copy of the slot rows. */
/* scatter2scatter whose output rows go straight into the attention core's
 * head layout heads[batch][hh * k_slots + j][t % seq_len][0:d_head] (row i's
 * slot s = order[i], token t = s / k_slots, choice j = s % k_slots; bf16
 * tcgen05 only).  epilogue SMOE_EPI_NONE, or SMOE_EPI_ACT_GRAD_SCALED with its
 * act-grad operand aux_grouped read BY GROUPED ROW (row_scale, dp_part as in
 * smoe_scatter2scatter_scaled).  d_head must be a multiple of 64. */
int smoe_scatter2scatter_heads(const void *x, int64_t x_rows, const void *w, int32_t num_experts, int64_t w_rows,
                               int64_t w_cols, const int32_t *order, const int32_t *expert_offsets, int64_t n,
                               int32_t fan_out, int32_t grouped_in, int32_t transpose_w, int32_t epilogue,
                               int32_t activation, const float *row_scale, const void *aux_grouped, float *dp_part,
                               int32_t dp_parts, int64_t seq_len, int32_t k_slots, int32_t d_head, void *heads,
                               void *stream);
int smoe_heads_to_grouped(const void *heads, int64_t batch, int64_t seq_len, int32_t k, int32_t heads_per_slot,
                          int32_t d_head, const int32_t *order, int64_t n, int32_t dtype, void *out, void *stream);
/* the reverse: heads[batch][hh * k + j][t % seq_len][:] = grouped[i][hh * d_head :] for the
 * slot s = order[i] — grouped slot rows (a grouped-output GEMM's layout) to the
 * attention core's head layout. */
int smoe_grouped_to_heads(const void *grouped, int64_t batch, int64_t seq_len, int32_t k, int32_t heads_per_slot,
                          int32_t d_head, const int32_t *order, int64_t n, int32_t dtype, void *heads, void *stream);
/* out[i] = x_grouped[i] * weights[order[i]] (the routing weight of each grouped
 * row's slot), rounded once: group()'s weighting for rows already grouped. */
int smoe_scale_grouped_rows(const void *x_grouped, int64_t d, const int32_t *order, int64_t n, const void *weights,
                            int32_t dtype, void *out, void *stream);

int smoe_group_inv(const void *x, int64_t x_rows, int64_t d, const int32_t *inverse, int32_t fan_out,
                   const void *weights, int32_t dtype, void *out, void *stream);

/* ---------------------------------------------------------------------------
 * group_xty (kernels.py:329-361): dw[e] = xg[bin e]^T @ yg[bin e]; empty bin -> 0.
 *   xg [n, d_in], yg [n, d_out] (grouped order), dw [E, d_in, d_out]
 */
int smoe_group_xty(const void *xg, const void *yg, const int32_t *expert_offsets,
                   int32_t num_experts, int64_t n, int64_t d_in, int64_t d_out,
                   int32_t dtype, void *dw, int32_t engine, void *stream);

/* ---------------------------------------------------------------------------
 * group (kernels.py:289-326): out[i] = x[order[i] / fan_out] * (weights ? weights[order[i]] : 1)
 *   x [n / fan_out, d], weights [n] float32 (float64 for SMOE_F64) or NULL, out [n, d].
 */
int smoe_group(const void *x, int64_t x_rows, int64_t d, const int32_t *order, int64_t n,
               int32_t fan_out, const void *weights, int32_t dtype, void *out, void *stream);

/* _combine (parallel_linear.py:69-73): y[s] = sum_j p[s,j] * y_hat[s*J + j]
 *   y_hat [S*J, d], p [S, J] float32 (float64 for SMOE_F64), y [S, d]     */
int smoe_combine(const void *y_hat, const void *p, int64_t s_rows, int32_t j_cols, int64_t d,
                 int32_t dtype, void *y, void *stream);
/* the same combine over slot rows held in GROUPED order (a grouped-output
 * GEMM's layout): y[s] = sum_j p[s,j] * y_hat_grouped[inverse[s*J + j]]
 * (inverse = the grouped position of each slot, from smoe_route_sort).
 * Bit-identical to smoe_combine over the slot-ordered rows.              */
int smoe_combine_grouped(const void *y_hat_grouped, const int32_t *inverse, const void *p, int64_t s_rows,
                         int32_t j_cols, int64_t d, int32_t dtype, void *y, void *stream);

/* dp (parallel_linear.py:198-206): dp[s,j] = <dy[s], y_hat[s*J + j]>
 *   dy [S, d], y_hat [S*J, d], dp [S, J] float32 (float64 for SMOE_F64)   */
int smoe_combine_grad_p(const void *dy, const void *y_hat, int64_t s_rows, int32_t j_cols,
                        int64_t d, int32_t dtype, void *dp, void *stream);
/* the same over slot rows in GROUPED order: dp[s,j] = <dy[s], y_hat_grouped[inverse[s*J + j]]> */
int smoe_combine_grad_p_grouped(const void *dy, const void *y_hat_grouped, const int32_t *inverse, int64_t s_rows,
                                int32_t j_cols, int64_t d, int32_t dtype, void *dp, void *stream);

/* fan-out reduce (parallel_linear.py:259-266): dx[t] = sum_j g[t*F + j]
 *   g [T*F, d], dx [T, d]                                                 */
int smoe_fanout_reduce(const void *slot_grads, int64_t t_rows, int32_t fan_out, int64_t d,
                       int32_t dtype, void *dx, void *stream);
/* the same reduce over slot rows in GROUPED order:
 *   dx[t] = sum_j g_grouped[inverse[t*F + j]]  (bit-identical to smoe_fanout_reduce) */
int smoe_fanout_reduce_grouped(const void *slot_grads_grouped, const int32_t *inverse, int64_t t_rows,
                               int32_t fan_out, int64_t d, int32_t dtype, void *dx, void *stream);

/* elementwise activation / derivative (moe_layers.py:75-83), rounded once.
 *   apply: out = act(x);  grad: out = act'(x)                            */
int smoe_apply_activation(const void *x, int64_t numel, int32_t activation, int32_t derivative,
                    int32_t dtype, void *out, void *stream);

/* ---------------------------------------------------------------------------
 * Routing-weight-scaled epilogues of the SMoE MLP (moe_layers.py:140-211 with
 * the combine weight moved through the second GEMM, bf16, tcgen05 CTA-pair
 * engine): SMOE_EPI_ACT_SCALED writes the hidden state already multiplied by
 * its slot's routing weight, so layer 2 + an unweighted k-sum is the combine
 * (parallel_linear.py:69-73); SMOE_EPI_ACT_GRAD_SCALED produces the hidden
 * gradient and, from the same accumulators, the combine-weight gradient's
 * partial dot products (dp[s] = <dY W2^T, act(h_pre)>, parallel_linear.py:198-206)
 * without the retained layer-2 output.  dp_part is [n, dp_parts] fp32,
 * dp_parts = 2 * ceil(d_out / 256); smoe_dp_from_partials reduces it.
 */
int smoe_scatter2scatter_scaled(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                                int64_t w_rows, int64_t w_cols, const int32_t *order,
                                const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                                int32_t grouped_in, int32_t grouped_out, int32_t transpose_w,
                                int32_t epilogue, int32_t activation, const float *row_scale, void *out,
                                void *out2, const void *aux, float *dp_part, int32_t dp_parts, void *stream);
int32_t smoe_dp_parts(int64_t d_out);
/* dp[order[i]] = sum_j dp_part[i * parts + j]  (dp: n floats in slot order) */
int smoe_dp_from_partials(const float *dp_part, int64_t n, int32_t parts, const int32_t *order, float *dp,
                          void *stream);

/* ---------------------------------------------------------------------------
 * group_xty over scattered operands: the reference's group() + group_xty()
 * pair (parallel_linear.py:224-234, kernels.py:289-361) with the grouped copies
 * never materialised.  dw[e] = Xb[bin e]^T @ Yb[bin e] where grouped position i
 * of Xb is x[i] when x_grouped else x[order[i] / x_fan_out] (same for y).
 *   x [x_rows, d_in], y [y_rows, d_out]; x_rows = n (grouped) or n / x_fan_out.
 */
int smoe_group_xty_scattered(const void *x, int64_t x_rows, int32_t x_fan_out, int32_t x_grouped,
                             const void *y, int64_t y_rows, int32_t y_fan_out, int32_t y_grouped,
                             const int32_t *order, const int32_t *expert_offsets, int32_t num_experts,
                             int64_t n, int64_t d_in, int64_t d_out, int32_t dtype, void *dw,
                             int32_t engine, void *stream);

/* ---------------------------------------------------------------------------
 * scatter_combine (kernels.py:242-286), inference: y[order[i] / combine_cols] +=
 *   p_flat[order[i]] * (x[src] @ W[e]) with no T*k buffer.
 *   p_flat  [n] float32 (float64 for SMOE_F64).
 *   y_accum [n / combine_cols, d_out] float32, zeroed by this call (unused
 *           for SMOE_F64, which accumulates in y itself).
 *   y       [n / combine_cols, d_out] dtype (rounded copy of y_accum; may be
 *           the same buffer as y_accum when dtype == SMOE_F32).
 *   engine  SMOE_ENGINE_AUTO: bf16 runs the tcgen05 CTA-pair GEMM whose
 *           epilogue scales each row by p and adds it into y_accum with fp32
 *           vector reductions (order of the k additions per token is not
 *           fixed: bit-reproducible for k <= 2, within fp32 rounding above);
 *           shapes it cannot take return SMOE_ENOTSUP (no SIMT fallback for
 *           bf16).  fp32 / fp64 run the SIMT check-mode kernel.
 */
int smoe_scatter_combine(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                         int64_t d_in, int64_t d_out, const int32_t *order,
                         const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                         const void *p_flat, int32_t combine_cols, int32_t grouped_in,
                         int32_t dtype, void *y_accum, void *y, int32_t engine, void *stream);

/* ---------------------------------------------------------------------------
 * Expert parallelism over peer memory (the
 * reference has no multi-device code).  Buffers of other ranks are
 * CUDA IPC mappings (NVLink P2P across GPUs; plain device memory between
 * processes sharing one GPU).  `peer_*` arguments are DEVICE arrays of
 * world_size uint64 base addresses, one per rank (this rank's own included).
 */
size_t smoe_ipc_handle_bytes(void);
/* handle of the allocation holding dev_ptr, and dev_ptr's byte offset in it */
int smoe_ipc_get_handle(const void *dev_ptr, void *handle_out /* host, smoe_ipc_handle_bytes() */,
                        int64_t *offset_out /* host */);
/* map a peer allocation; returns its base (add the peer's offset) */
int smoe_ipc_open(const void *handle /* host */, void **dev_ptr_out /* host */);
int smoe_ipc_close(void *dev_ptr /* the base smoe_ipc_open returned */);

/* Dispatch: grouped row i of this rank in global expert e's bin (owner
 * q = e / experts_per_rank, num_experts = experts_per_rank * world) is stored at
 * row j = dstart[e] + i - bin_offsets[e] of peer_rows[q]: x[order[i] / fan_out]
 * (* weights[order[i]] if weights != NULL, the p-weighted group of
 * parallel_linear.py:213).  With peer_slot/peer_src the row's slot id and this
 * rank id are stored alongside (forward dispatch), with slot_p/peer_p its
 * routing weight slot_p[order[i]].  Experts are sent in (local expert, owner)
 * order; after each chunk of rows the sender fences at system scope and adds
 * the chunk's row count to peer_arrive[q][e % experts_per_rank] (uint64, may be
 * NULL), the owner's arrival gate.  Rows with j >= capacity are not written and
 * set bit 2 of *err (device int32). */
int smoe_ep_dispatch_rows(const void *x, int64_t x_rows, int64_t d, const int32_t *order,
                          const int32_t *bin_offsets, int32_t num_experts, int32_t fan_out, const float *weights,
                          int64_t n, const int64_t *dstart, int32_t experts_per_rank, int32_t world,
                          const uint64_t *peer_rows, const uint64_t *peer_slot, const uint64_t *peer_src, int32_t me,
                          const float *slot_p, const uint64_t *peer_p, int64_t capacity, const uint64_t *peer_arrive,
                          int32_t *err, int32_t dtype, void *stream);
/* Sets bit 2 of *err when local_offsets[experts_per_rank] (rows routed to this
 * rank) exceeds capacity (device-side; no host synchronisation). */
int smoe_ep_check_capacity(const int32_t *local_offsets, int32_t experts_per_rank, int64_t capacity, int32_t *err,
                           void *stream);
/* The owner's expert GEMM on rows delivered by peers (grouped in, grouped out,
 * bf16 tcgen05 CTA-pair engine): smoe_scatter2scatter_scaled's two epilogues
 * (row scale s_i = row_scale[order[i]]; order is the identity [0, n) for rows
 * in receive order) with each tile of local expert e started only
 * once arrive[e] (see smoe_ep_dispatch_rows) reaches the expert's bin length
 * local_offsets[e + 1] - local_offsets[e] — the dispatch overlaps the GEMM. */
int smoe_ep_expert_gemm_gated(const void *x, int64_t n, const void *w, int32_t num_experts, int64_t w_rows,
                              int64_t w_cols, const int32_t *order, const int32_t *local_offsets, int32_t transpose_w,
                              int32_t epilogue,
                              int32_t activation, const float *row_scale, void *out, void *out2, const void *aux,
                              float *dp_part, int32_t dp_parts, const uint64_t *arrive, void *stream);
/* group_xty (dw[e] = xg[bin e]^T yg[bin e]) whose yg rows are delivered by
 * peers: each tile of expert e waits for arrive_y[e] as above. */
int smoe_ep_group_xty_gated(const void *xg, const void *yg, const int32_t *local_offsets, int32_t num_experts,
                            int64_t n, int64_t d_in, int64_t d_out, void *dw, const uint64_t *arrive_y, void *stream);
/* dp of received row j < n_valid (= *n_valid, device, may be NULL for n) = sum
 * of dp_part[j, :] (smoe_scatter2scatter_scaled partials), stored at
 * peer_dp[recv_src[j]][recv_slot[j]] (float). */
int smoe_ep_dp_return(const float *dp_part, int64_t n, int32_t parts, const int32_t *recv_slot,
                      const int32_t *recv_src, const uint64_t *peer_dp, const int32_t *n_valid, void *stream);
/* Return: local row j < n_valid goes to row recv_slot[j] of peer_out[recv_src[j]]. */
int smoe_ep_return_rows(const void *y, int64_t n, int64_t d, const int32_t *recv_slot, const int32_t *recv_src,
                        const uint64_t *peer_out, const int32_t *n_valid, int32_t dtype, void *stream);
/* The return fused into the expert GEMM: out_j = x_j @ W[e] (or W[e]^T) for the
 * grouped rows x [n, d_in] (bins = expert_offsets; rows past the last bin are
 * never touched), each output row stored by the GEMM epilogue straight into row
 * recv_slot[j] of peer_out[recv_src[j]] (bf16, tcgen05 CTA-pair engine). */
int smoe_ep_gemm_return(const void *x, int64_t n, const void *w, int32_t num_experts, int64_t w_rows, int64_t w_cols,
                        const int32_t *expert_offsets, int32_t transpose_w, const int32_t *recv_slot,
                        const int32_t *recv_src, const uint64_t *peer_out, void *stream);
/* Copy `bytes` from src to every peer_dst[q] + offset_bytes. */
int smoe_ep_put(const void *src, int64_t bytes, const uint64_t *peer_dst, int64_t offset_bytes, int32_t world,
                void *stream);
/* Signal every peer (system fence, then +1 on peer q's flags[slot * world + me],
 * and +1 on this rank's my_epochs[slot]) / wait until flags[slot * world + s]
 * >= my_epochs[slot] for every source s (bit 1 of *err on timeout).  Epochs live
 * on the device, so a signal / wait sequence replays inside a CUDA graph. */
int smoe_ep_signal(const uint64_t *peer_flags, int32_t world, int32_t me, int32_t slot, uint64_t *my_epochs,
                   void *stream);
int smoe_ep_wait(const uint64_t *flags, int32_t world, int32_t slot, const uint64_t *my_epochs, int64_t timeout_ns,
                 int32_t *err, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SMOE_B200_H */
