// extern "C" entry points of libsmoe_b200.so (declared in include/smoe_b200.h).
// Argument validation mirrors the reference's checks so the Python shim can map
// status codes back onto the same exception classes (errors.py:3-19).
#include <atomic>
#include <cstdio>
#include <string>

#include "common.cuh"

namespace smoe {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int status, const std::string &msg) {
  set_error(msg);
  return status;
}
int check_launch(const char *what, int launches) {
  g_launches.fetch_add((uint64_t)launches, std::memory_order_relaxed);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(SMOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(err));
  return SMOE_OK;
}

// engines (defined in the other translation units)
size_t route_sort_workspace(int64_t n, int E);
int route_sort(const int64_t *, int64_t, int, int32_t *, int32_t *, int32_t *, int32_t *, void *, size_t, cudaStream_t);
int group(const void *, int64_t, const int32_t *, int64_t, int, const void *, int, void *, cudaStream_t);
int combine(const void *, const void *, int64_t, int, int64_t, int, void *, cudaStream_t, const int32_t *);
int combine_grad_p(const void *, const void *, int64_t, int, int64_t, int, void *, cudaStream_t, const int32_t *);
int fanout_reduce(const void *, int64_t, int, int64_t, int, void *, cudaStream_t, const int32_t *);
int dp_from_partials(const float *, int64_t, int, const int32_t *, float *, cudaStream_t);
int group_inv(const void *, int64_t, int64_t, const int32_t *, int, const void *, int, void *, cudaStream_t);
int grouped_to_heads(const void *, int64_t, int, int, int, const int32_t *, int64_t, int, void *, cudaStream_t);
int scale_grouped_rows(const void *, int64_t, const int32_t *, int64_t, const void *, int, void *, cudaStream_t);
int heads_to_grouped(const void *, int64_t, int64_t, int, int, int, const int32_t *, int64_t, int, void *,
                     cudaStream_t);
int tc_scatter2scatter_scaled(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                              const int32_t *, int64_t, int, int, int, int, int, int, const float *, void *, void *,
                              const void *, float *, int, cudaStream_t);
int activation(const void *, int64_t, int, int, int, void *, cudaStream_t);
int simt_scatter2scatter(const void *, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *, int64_t, int, int, int, int, int, int, int, void *, void *, const void *, cudaStream_t);
int simt_group_xty(const void *, const void *, const int32_t *, int, int64_t, int64_t, int, void *, cudaStream_t);
int simt_scatter_combine(const void *, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *, int64_t, int,
                         const void *, int, int, int, void *, void *, cudaStream_t);
int router_topk(const float *, int64_t, int, int, int, int, float *, int64_t *, float *, cudaStream_t);
int router_backward(const float *, const int64_t *, const float *, int64_t, int, int, int, float *, cudaStream_t);
int router_gate(const void *, int, const float *, int64_t, int, int, int, int, float *, int64_t *, float *,
                cudaStream_t);
bool tc_available();
bool tc_supports_s2s(int64_t d_in, int64_t d_out, const void *x, const void *w, const void *out);
int tc_scatter2scatter_heads(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                             const int32_t *, int64_t, int, int, int, int, int, const float *, const void *, float *, int,
                             int64_t, int, int, void *, cudaStream_t);
int tc_scatter2scatter(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *, int64_t, int, int, int, int, int, int, void *, void *, const void *, cudaStream_t);
int tc_group_xty(const void *, const void *, const int32_t *, int, int64_t, int64_t, int64_t, void *, cudaStream_t);
bool tc_supports_combine(int, int64_t, int64_t, const void *, const void *, const void *);
int tc_scatter_combine(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *,
                       int64_t, int, int, const float *, int, float *, cudaStream_t);
int round_copy(const float *, int64_t, int, void *, cudaStream_t);
bool tc_supports_xty_scattered(int, int64_t, int64_t, int64_t, int64_t, const void *, const void *, const void *);
int tc_group_xty_scattered(const void *, int64_t, int, int, const void *, int64_t, int, int, const int32_t *,
                           const int32_t *, int, int64_t, int64_t, int64_t, void *, cudaStream_t);
int simt_group_xty_scattered(const void *, int, int, const void *, int, int, const int32_t *, const int32_t *, int,
                             int64_t, int64_t, int, void *, cudaStream_t);

}  // namespace smoe

using namespace smoe;

#define REQUIRE(cond, status, msg)          \
  do {                                      \
    if (!(cond)) return fail(status, msg);  \
  } while (0)

static inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }
static inline std::string dims(int64_t a, int64_t b) {
  return "(" + std::to_string(a) + ", " + std::to_string(b) + ")";
}
static inline bool valid_dtype(int32_t d) { return d == SMOE_F32 || d == SMOE_BF16 || d == SMOE_F64; }

extern "C" {

const char *smoe_get_last_error(void) { return g_last_error.c_str(); }
int smoe_abi_version(void) { return SMOE_ABI_VERSION; }
uint64_t smoe_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

size_t smoe_route_sort_workspace_bytes(int64_t n, int32_t num_experts) {
  return route_sort_workspace(n, num_experts);
}

int smoe_route_sort(const int64_t *expert_idx, int64_t n, int32_t num_experts,
                    int32_t *sorted_scattered_idxs, int32_t *sorted_expert_idxs,
                    int32_t *expert_offsets, int32_t *inverse, void *workspace,
                    size_t workspace_bytes, void *stream) {
  REQUIRE(n == 0 || (expert_idx && sorted_scattered_idxs), SMOE_EINVAL, "route_sort: null pointer");
  REQUIRE(expert_offsets, SMOE_EINVAL, "route_sort: null expert_offsets");
  return route_sort(expert_idx, n, num_experts, sorted_scattered_idxs, sorted_expert_idxs,
                    expert_offsets, inverse, workspace, workspace_bytes, S(stream));
}

int smoe_router_topk(const float *in, int64_t T, int32_t num_experts, int32_t k, int32_t apply_softmax,
                     int32_t renormalize, float *gate_out, int64_t *expert_idx, float *p, void *stream) {
  REQUIRE(T >= 0, SMOE_EINVAL, "router_topk: T must be >= 0");
  REQUIRE(T == 0 || (in && expert_idx && p), SMOE_EINVAL, "router_topk: null pointer");
  return router_topk(in, T, num_experts, k, apply_softmax, renormalize, gate_out, expert_idx, p, S(stream));
}

int smoe_router_gate(const void *x, int32_t x_dtype, const float *w_gate, int64_t T, int32_t d_model,
                     int32_t num_experts, int32_t k, int32_t renormalize, float *gate_out, int64_t *expert_idx,
                     float *p, void *stream) {
  REQUIRE(T >= 0 && d_model >= 1, SMOE_EINVAL, "router_gate: T must be >= 0 and d_model >= 1");
  REQUIRE(T == 0 || (x && w_gate && expert_idx && p), SMOE_EINVAL, "router_gate: null pointer");
  return router_gate(x, x_dtype, w_gate, T, d_model, num_experts, k, renormalize, gate_out, expert_idx, p, S(stream));
}

int smoe_router_backward(const float *gate, const int64_t *expert_idx, const float *grad_p, int64_t T,
                         int32_t num_experts, int32_t k, int32_t renormalized, float *dlogits, void *stream) {
  REQUIRE(T >= 0, SMOE_EINVAL, "router_backward: T must be >= 0");
  REQUIRE(T == 0 || (gate && expert_idx && grad_p && dlogits), SMOE_EINVAL, "router_backward: null pointer");
  return router_backward(gate, expert_idx, grad_p, T, num_experts, k, renormalized, dlogits, S(stream));
}

int smoe_scatter2scatter(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                         int64_t w_rows, int64_t w_cols, const int32_t *order,
                         const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                         int32_t grouped_in, int32_t grouped_out, int32_t transpose_w,
                         int32_t dtype, int32_t epilogue, int32_t activation, void *out,
                         void *out2, const void *aux, int32_t engine, void *stream) {
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1, got " + std::to_string(fan_out));
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype " + std::to_string(dtype));
  REQUIRE(num_experts >= 1, SMOE_EINVAL, "num_experts must be >= 1");
  REQUIRE(epilogue >= SMOE_EPI_NONE && epilogue <= SMOE_EPI_ACT_ONLY, SMOE_EINVAL, "bad epilogue");
  REQUIRE(activation >= SMOE_ACT_GELU && activation <= SMOE_ACT_SILU, SMOE_EINVAL, "bad activation");
  if (grouped_in)
    REQUIRE(x_rows == n, SMOE_ESHAPE, "grouped input rows vs slots: " + dims(x_rows, 0) + " vs " + dims(n, 0));
  else
    REQUIRE(x_rows * fan_out == n, SMOE_EINVAL,
            "scattered input rows (" + std::to_string(x_rows) + ") * fan_out (" + std::to_string(fan_out) +
                ") must equal T*k (" + std::to_string(n) + ")");
  if (n == 0) return SMOE_OK;  // empty tensors may carry null pointers
  REQUIRE(epilogue != SMOE_EPI_ACT || out2, SMOE_EINVAL, "EPI_ACT needs out2");
  REQUIRE(epilogue != SMOE_EPI_ACT_GRAD || aux, SMOE_EINVAL, "EPI_ACT_GRAD needs aux");
  REQUIRE(x && w && order && expert_offsets && out, SMOE_EINVAL, "scatter2scatter: null pointer");
  const int64_t d_in = transpose_w ? w_cols : w_rows, d_out = transpose_w ? w_rows : w_cols;
  const bool use_tc = engine == SMOE_ENGINE_TCGEN05 || (engine == SMOE_ENGINE_AUTO && dtype == SMOE_BF16);
  if (use_tc) {
    REQUIRE(tc_available(), SMOE_ENOTSUP, "bf16 runs on the sm_100a tcgen05 engine only (no such device)");
    REQUIRE(tc_supports_s2s(d_in, d_out, x, w, out), SMOE_ENOTSUP,
            "bf16 scatter2scatter needs d_in, d_out multiples of 8 and 16-byte aligned buffers (got d_in=" +
                std::to_string(d_in) + ", d_out=" + std::to_string(d_out) + "); there is no SIMT fallback");
    REQUIRE(dtype == SMOE_BF16, SMOE_ENOTSUP, "tcgen05 engine is bf16-only (fp32 check mode runs on SIMT)");
    return tc_scatter2scatter(x, x_rows, w, num_experts, w_rows, w_cols, order, expert_offsets, n, fan_out,
                              grouped_in, grouped_out, transpose_w, epilogue, activation, out, out2, aux, S(stream));
  }
  return simt_scatter2scatter(x, w, num_experts, w_rows, w_cols, order, expert_offsets, n, fan_out, grouped_in,
                              grouped_out, transpose_w, dtype, epilogue, activation, out, out2, aux, S(stream));
}

int smoe_scatter2scatter_heads(const void *x, int64_t x_rows, const void *w, int32_t num_experts, int64_t w_rows,
                               int64_t w_cols, const int32_t *order, const int32_t *expert_offsets, int64_t n,
                               int32_t fan_out, int32_t grouped_in, int32_t transpose_w, int32_t epilogue,
                               int32_t activation, const float *row_scale, const void *aux_grouped, float *dp_part,
                               int32_t dp_parts, int64_t seq_len, int32_t k_slots, int32_t d_head, void *heads,
                               void *stream) {
  REQUIRE(epilogue == SMOE_EPI_NONE || epilogue == SMOE_EPI_ACT_GRAD_SCALED, SMOE_EINVAL,
          "scatter2scatter_heads takes SMOE_EPI_NONE or SMOE_EPI_ACT_GRAD_SCALED");
  REQUIRE(activation >= SMOE_ACT_GELU && activation <= SMOE_ACT_IDENTITY, SMOE_EINVAL, "bad activation");
  REQUIRE(fan_out >= 1 && k_slots >= 1 && seq_len >= 1 && d_head >= 1, SMOE_EINVAL, "bad dimensions");
  REQUIRE(n % ((int64_t)k_slots * seq_len) == 0, SMOE_ESHAPE, "slots must be batch * seq_len * k_slots");
  if (grouped_in)
    REQUIRE(x_rows == n, SMOE_ESHAPE, "grouped input rows vs slots");
  else
    REQUIRE(x_rows * fan_out == n, SMOE_EINVAL, "scattered input rows * fan_out must equal T*k");
  const int64_t d_out = transpose_w ? w_rows : w_cols;
  REQUIRE(!dp_part || dp_parts == smoe_dp_parts(d_out), SMOE_EINVAL, "dp_parts must be smoe_dp_parts(d_out)");
  if (n == 0) return SMOE_OK;
  REQUIRE(epilogue != SMOE_EPI_ACT_GRAD_SCALED || (aux_grouped && row_scale), SMOE_EINVAL,
          "EPI_ACT_GRAD_SCALED needs the grouped act-grad operand and row scales");
  REQUIRE(x && w && order && expert_offsets && heads, SMOE_EINVAL, "scatter2scatter_heads: null pointer");
  REQUIRE(tc_available(), SMOE_ENOTSUP, "head-layout output runs on the tcgen05 engine");
  return tc_scatter2scatter_heads(x, x_rows, w, num_experts, w_rows, w_cols, order, expert_offsets, n, fan_out,
                                  grouped_in, transpose_w, epilogue, activation, row_scale, aux_grouped, dp_part,
                                  dp_parts, seq_len, k_slots, d_head, heads, S(stream));
}

int smoe_group_xty_scattered(const void *x, int64_t x_rows, int32_t x_fan_out, int32_t x_grouped, const void *y,
                             int64_t y_rows, int32_t y_fan_out, int32_t y_grouped, const int32_t *order,
                             const int32_t *expert_offsets, int32_t num_experts, int64_t n, int64_t d_in,
                             int64_t d_out, int32_t dtype, void *dw, int32_t engine, void *stream) {
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype " + std::to_string(dtype));
  REQUIRE(num_experts >= 1, SMOE_EINVAL, "num_experts must be >= 1");
  REQUIRE(x_fan_out >= 1 && y_fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1");
  REQUIRE(dw && expert_offsets, SMOE_EINVAL, "group_xty_scattered: null pointer");
  REQUIRE(n == 0 || (x && y && order), SMOE_EINVAL, "group_xty_scattered: null pointer");
  REQUIRE(x_grouped ? x_rows == n : x_rows * x_fan_out == n, SMOE_ESHAPE,
          "x rows (" + std::to_string(x_rows) + ") do not cover the " + std::to_string(n) + " slots");
  REQUIRE(y_grouped ? y_rows == n : y_rows * y_fan_out == n, SMOE_ESHAPE,
          "y rows (" + std::to_string(y_rows) + ") do not cover the " + std::to_string(n) + " slots");
  if (n == 0) return simt_group_xty_scattered(x, x_fan_out, x_grouped, y, y_fan_out, y_grouped, order,
                                              expert_offsets, num_experts, d_in, d_out, dtype, dw, S(stream));
  const bool use_tc = engine == SMOE_ENGINE_TCGEN05 || (engine == SMOE_ENGINE_AUTO && dtype == SMOE_BF16);
  if (use_tc) {
    REQUIRE(tc_available(), SMOE_ENOTSUP, "bf16 runs on the sm_100a tcgen05 engine only (no such device)");
    REQUIRE(tc_supports_xty_scattered(num_experts, x_rows, d_in, y_rows, d_out, x, y, dw), SMOE_ENOTSUP,
            "bf16 group_xty over scattered operands needs d_in, d_out multiples of 8, 16-byte aligned buffers and "
            "at most 1024 experts; there is no SIMT fallback");
    REQUIRE(dtype == SMOE_BF16, SMOE_ENOTSUP, "tcgen05 engine is bf16-only (fp32 check mode runs on SIMT)");
    return tc_group_xty_scattered(x, x_rows, x_fan_out, x_grouped, y, y_rows, y_fan_out, y_grouped, order,
                                  expert_offsets, num_experts, n, d_in, d_out, dw, S(stream));
  }
  return simt_group_xty_scattered(x, x_fan_out, x_grouped, y, y_fan_out, y_grouped, order, expert_offsets,
                                  num_experts, d_in, d_out, dtype, dw, S(stream));
}

int smoe_group_xty(const void *xg, const void *yg, const int32_t *expert_offsets,
                   int32_t num_experts, int64_t n, int64_t d_in, int64_t d_out, int32_t dtype,
                   void *dw, int32_t engine, void *stream) {
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype " + std::to_string(dtype));
  REQUIRE(num_experts >= 1, SMOE_EINVAL, "num_experts must be >= 1");
  REQUIRE(dw && expert_offsets, SMOE_EINVAL, "group_xty: null pointer");
  REQUIRE(n == 0 || (xg && yg), SMOE_EINVAL, "group_xty: null pointer");
  if (n == 0) return simt_group_xty(xg, yg, expert_offsets, num_experts, d_in, d_out, dtype, dw, S(stream));
  const bool use_tc = engine == SMOE_ENGINE_TCGEN05 || (engine == SMOE_ENGINE_AUTO && dtype == SMOE_BF16);
  if (use_tc) {
    REQUIRE(tc_available(), SMOE_ENOTSUP, "bf16 runs on the sm_100a tcgen05 engine only (no such device)");
    REQUIRE(tc_supports_s2s(d_in, d_out, xg, yg, dw), SMOE_ENOTSUP,
            "bf16 group_xty needs d_in, d_out multiples of 8 and 16-byte aligned buffers; there is no SIMT fallback");
    REQUIRE(dtype == SMOE_BF16, SMOE_ENOTSUP, "tcgen05 engine is bf16-only");
    return tc_group_xty(xg, yg, expert_offsets, num_experts, n, d_in, d_out, dw, S(stream));
  }
  return simt_group_xty(xg, yg, expert_offsets, num_experts, d_in, d_out, dtype, dw, S(stream));
}

int smoe_group(const void *x, int64_t x_rows, int64_t d, const int32_t *order, int64_t n,
               int32_t fan_out, const void *weights, int32_t dtype, void *out, void *stream) {
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1, got " + std::to_string(fan_out));
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  REQUIRE(x_rows * fan_out == n, SMOE_EINVAL,
          "input rows (" + std::to_string(x_rows) + ") * fan_out (" + std::to_string(fan_out) +
              ") must equal T*k (" + std::to_string(n) + ")");
  if (n == 0) return SMOE_OK;
  REQUIRE(x && order && out, SMOE_EINVAL, "group: null pointer");
  return group(x, d, order, n, fan_out, weights, dtype, out, S(stream));
}

int smoe_heads_to_grouped(const void *heads, int64_t batch, int64_t seq_len, int32_t k, int32_t heads_per_slot,
                          int32_t d_head, const int32_t *order, int64_t n, int32_t dtype, void *out, void *stream) {
  REQUIRE(dtype == SMOE_F32 || dtype == SMOE_BF16, SMOE_EINVAL, "heads_to_grouped: bf16 or fp32 only");
  REQUIRE(batch >= 0 && seq_len >= 1 && k >= 1 && heads_per_slot >= 1 && d_head >= 1, SMOE_EINVAL,
          "heads_to_grouped: bad dimensions");
  REQUIRE(n == batch * seq_len * k, SMOE_ESHAPE, "heads_to_grouped: n must equal batch * seq_len * k");
  if (n == 0) return SMOE_OK;
  REQUIRE(heads && order && out, SMOE_EINVAL, "heads_to_grouped: null pointer");
  return heads_to_grouped(heads, batch, seq_len, k, heads_per_slot, d_head, order, n, dtype, out, S(stream));
}

int smoe_grouped_to_heads(const void *grouped, int64_t batch, int64_t seq_len, int32_t k, int32_t h, int32_t d_head,
                          const int32_t *order, int64_t n, int32_t dtype, void *heads, void *stream) {
  REQUIRE(k >= 1 && h >= 1 && d_head >= 1 && seq_len >= 1, SMOE_EINVAL, "grouped_to_heads: bad dimensions");
  REQUIRE(n == batch * seq_len * k, SMOE_ESHAPE, "grouped_to_heads: n must equal batch * seq_len * k");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (n == 0) return SMOE_OK;
  REQUIRE(grouped && order && heads, SMOE_EINVAL, "grouped_to_heads: null pointer");
  return grouped_to_heads(grouped, seq_len, k, h, d_head, order, n, dtype, heads, S(stream));
}

int smoe_scale_grouped_rows(const void *x_grouped, int64_t d, const int32_t *order, int64_t n, const void *weights,
                            int32_t dtype, void *out, void *stream) {
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (n == 0) return SMOE_OK;
  REQUIRE(x_grouped && order && weights && out, SMOE_EINVAL, "scale_grouped_rows: null pointer");
  return scale_grouped_rows(x_grouped, d, order, n, weights, dtype, out, S(stream));
}

int smoe_group_inv(const void *x, int64_t x_rows, int64_t d, const int32_t *inverse, int32_t fan_out,
                   const void *weights, int32_t dtype, void *out, void *stream) {
  REQUIRE(fan_out >= 1 && fan_out <= 16, SMOE_EINVAL, "group_inv: fan_out must be in [1, 16]");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (x_rows == 0) return SMOE_OK;
  REQUIRE(x && inverse && out, SMOE_EINVAL, "group_inv: null pointer");
  return group_inv(x, x_rows, d, inverse, fan_out, weights, dtype, out, S(stream));
}

int smoe_combine(const void *y_hat, const void *p, int64_t s_rows, int32_t j_cols, int64_t d,
                 int32_t dtype, void *y, void *stream) {
  REQUIRE(j_cols >= 1, SMOE_EINVAL, "combine: J must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (s_rows == 0) return SMOE_OK;
  REQUIRE(y_hat && p && y, SMOE_EINVAL, "combine: null pointer");
  return combine(y_hat, p, s_rows, j_cols, d, dtype, y, S(stream), nullptr);
}

int smoe_combine_grouped(const void *y_hat_grouped, const int32_t *inverse, const void *p, int64_t s_rows,
                         int32_t j_cols, int64_t d, int32_t dtype, void *y, void *stream) {
  REQUIRE(j_cols >= 1, SMOE_EINVAL, "combine_grouped: J must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (s_rows == 0) return SMOE_OK;
  REQUIRE(y_hat_grouped && inverse && p && y, SMOE_EINVAL, "combine_grouped: null pointer");
  return combine(y_hat_grouped, p, s_rows, j_cols, d, dtype, y, S(stream), inverse);
}

int smoe_combine_grad_p(const void *dy, const void *y_hat, int64_t s_rows, int32_t j_cols,
                        int64_t d, int32_t dtype, void *dp, void *stream) {
  REQUIRE(j_cols >= 1, SMOE_EINVAL, "combine_grad_p: J must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (s_rows == 0) return SMOE_OK;
  REQUIRE(dy && y_hat && dp, SMOE_EINVAL, "combine_grad_p: null pointer");
  return combine_grad_p(dy, y_hat, s_rows, j_cols, d, dtype, dp, S(stream), nullptr);
}

int smoe_combine_grad_p_grouped(const void *dy, const void *y_hat_grouped, const int32_t *inverse, int64_t s_rows,
                                int32_t j_cols, int64_t d, int32_t dtype, void *dp, void *stream) {
  REQUIRE(j_cols >= 1, SMOE_EINVAL, "combine_grad_p_grouped: J must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (s_rows == 0) return SMOE_OK;
  REQUIRE(dy && y_hat_grouped && inverse && dp, SMOE_EINVAL, "combine_grad_p_grouped: null pointer");
  return combine_grad_p(dy, y_hat_grouped, s_rows, j_cols, d, dtype, dp, S(stream), inverse);
}

int32_t smoe_dp_parts(int64_t d_out) { return (int32_t)(2 * ((d_out + 255) / 256)); }

int smoe_dp_from_partials(const float *dp_part, int64_t n, int32_t parts, const int32_t *order, float *dp,
                          void *stream) {
  REQUIRE(parts >= 1, SMOE_EINVAL, "dp_from_partials: parts must be >= 1");
  if (n == 0) return SMOE_OK;
  REQUIRE(dp_part && order && dp, SMOE_EINVAL, "dp_from_partials: null pointer");
  return dp_from_partials(dp_part, n, parts, order, dp, S(stream));
}

int smoe_scatter2scatter_scaled(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                                int64_t w_rows, int64_t w_cols, const int32_t *order,
                                const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                                int32_t grouped_in, int32_t grouped_out, int32_t transpose_w,
                                int32_t epilogue, int32_t activation, const float *row_scale, void *out,
                                void *out2, const void *aux, float *dp_part, int32_t dp_parts, void *stream) {
  REQUIRE(epilogue == SMOE_EPI_ACT_SCALED || epilogue == SMOE_EPI_ACT_GRAD_SCALED, SMOE_EINVAL,
          "scatter2scatter_scaled takes SMOE_EPI_ACT_SCALED or SMOE_EPI_ACT_GRAD_SCALED");
  REQUIRE(activation >= SMOE_ACT_GELU && activation <= SMOE_ACT_IDENTITY, SMOE_EINVAL, "bad activation");
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1");
  if (grouped_in)
    REQUIRE(x_rows == n, SMOE_ESHAPE, "grouped input rows vs slots");
  else
    REQUIRE(x_rows * fan_out == n, SMOE_EINVAL, "scattered input rows * fan_out must equal T*k");
  const int64_t d_out = transpose_w ? w_rows : w_cols;
  REQUIRE(!dp_part || dp_parts == smoe_dp_parts(d_out), SMOE_EINVAL, "dp_parts must be smoe_dp_parts(d_out)");
  if (n == 0) return SMOE_OK;  // empty tensors may carry null pointers
  REQUIRE(epilogue != SMOE_EPI_ACT_SCALED || out2, SMOE_EINVAL, "EPI_ACT_SCALED needs out2");
  REQUIRE(epilogue != SMOE_EPI_ACT_GRAD_SCALED || aux, SMOE_EINVAL, "EPI_ACT_GRAD_SCALED needs aux");
  REQUIRE(x && w && order && expert_offsets && out && row_scale, SMOE_EINVAL, "scatter2scatter_scaled: null pointer");
  REQUIRE(tc_available(), SMOE_ENOTSUP, "scaled epilogues run on the tcgen05 engine");
  return tc_scatter2scatter_scaled(x, x_rows, w, num_experts, w_rows, w_cols, order, expert_offsets, n, fan_out,
                                   grouped_in, grouped_out, transpose_w, epilogue, activation, row_scale, out, out2,
                                   aux, dp_part, dp_parts, S(stream));
}

int smoe_fanout_reduce(const void *slot_grads, int64_t t_rows, int32_t fan_out, int64_t d,
                       int32_t dtype, void *dx, void *stream) {
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (t_rows == 0) return SMOE_OK;
  REQUIRE(slot_grads && dx, SMOE_EINVAL, "fanout_reduce: null pointer");
  return fanout_reduce(slot_grads, t_rows, fan_out, d, dtype, dx, S(stream), nullptr);
}

int smoe_fanout_reduce_grouped(const void *slot_grads_grouped, const int32_t *inverse, int64_t t_rows,
                               int32_t fan_out, int64_t d, int32_t dtype, void *dx, void *stream) {
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (t_rows == 0) return SMOE_OK;
  REQUIRE(slot_grads_grouped && inverse && dx, SMOE_EINVAL, "fanout_reduce_grouped: null pointer");
  return fanout_reduce(slot_grads_grouped, t_rows, fan_out, d, dtype, dx, S(stream), inverse);
}

int smoe_apply_activation(const void *x, int64_t numel, int32_t act, int32_t derivative, int32_t dtype,
                    void *out, void *stream) {
  REQUIRE(act >= SMOE_ACT_GELU && act <= SMOE_ACT_SILU, SMOE_EINVAL, "bad activation");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (numel == 0) return SMOE_OK;
  REQUIRE(x && out, SMOE_EINVAL, "activation: null pointer");
  return activation(x, numel, act, derivative, dtype, out, S(stream));
}

int smoe_scatter_combine(const void *x, int64_t x_rows, const void *w, int32_t num_experts,
                         int64_t d_in, int64_t d_out, const int32_t *order,
                         const int32_t *expert_offsets, int64_t n, int32_t fan_out,
                         const void *p_flat, int32_t combine_cols, int32_t grouped_in,
                         int32_t dtype, void *y_accum, void *y, int32_t engine, void *stream) {
  REQUIRE(fan_out >= 1, SMOE_EINVAL, "fan_out must be >= 1");
  REQUIRE(combine_cols >= 1 && n % combine_cols == 0, SMOE_EINVAL,
          "combine width " + std::to_string(combine_cols) + " must divide T*k (" + std::to_string(n) + ")");
  REQUIRE(valid_dtype(dtype), SMOE_EINVAL, "unsupported dtype");
  if (grouped_in)
    REQUIRE(x_rows == n, SMOE_ESHAPE, "grouped input rows vs slots");
  else
    REQUIRE(x_rows * fan_out == n, SMOE_EINVAL, "scattered input rows * fan_out must equal T*k");
  if (n == 0) return SMOE_OK;  // empty tensors may carry null pointers
  if (dtype == SMOE_F64) y_accum = y;  // float64 storage accumulates in y itself
  REQUIRE(y_accum && y, SMOE_EINVAL, "scatter_combine: null output");
  if (d_out == 0) return simt_scatter_combine(x, w, num_experts, d_in, d_out, order, expert_offsets, n,
                                                        fan_out, p_flat, combine_cols, grouped_in, dtype, y_accum, y,
                                                        S(stream));
  REQUIRE(x && w && order && expert_offsets && p_flat, SMOE_EINVAL, "scatter_combine: null pointer");
  const bool use_tc = engine == SMOE_ENGINE_TCGEN05 || (engine == SMOE_ENGINE_AUTO && dtype == SMOE_BF16);
  if (use_tc) {
    REQUIRE(tc_available(), SMOE_ENOTSUP, "bf16 runs on the sm_100a tcgen05 engine only (no such device)");
    REQUIRE(tc_supports_combine(num_experts, d_in, d_out, x, w, (const void *)y_accum), SMOE_ENOTSUP,
            "bf16 scatter_combine needs d_in, d_out multiples of 8, 16-byte aligned buffers and at most 1024 "
            "experts; there is no SIMT fallback");
    REQUIRE(dtype == SMOE_BF16, SMOE_ENOTSUP, "tcgen05 engine is bf16-only (fp32 check mode runs on SIMT)");
    int st = tc_scatter_combine(x, x_rows, w, num_experts, d_in, d_out, order, expert_offsets, n, fan_out, grouped_in,
                                (const float *)p_flat, combine_cols, (float *)y_accum, S(stream));
    if (st != SMOE_OK) return st;
    return round_copy((const float *)y_accum, (n / combine_cols) * d_out, dtype, y, S(stream));
  }
  return simt_scatter_combine(x, w, num_experts, d_in, d_out, order, expert_offsets, n, fan_out, p_flat,
                              combine_cols, grouped_in, dtype, y_accum, y, S(stream));
}

}  // extern "C"
