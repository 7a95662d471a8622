// Router: softmax + stable top-k + renormalisation, and the gate backward
// (the step in front of the K1 sort).
//
// Reference: router.py:119-151 (gate_forward / softmax_rows / topk_select) and
// router.py:167-188 (gate_backward).  One warp per token; lane l holds experts
// l, l+32, ... (PER per lane, a compile-time bound so the row stays in
// registers).  Softmax runs in float64 and is rounded once to float32, as the
// reference does; top-k selects on the float32 gate values with ties going to
// the lower expert id (numpy's stable argsort of -g); p is renormalised in
// float64.  Given identical logits the indices are bit-identical to the
// reference and p matches to float32 rounding.
#include "common.cuh"

namespace smoe {

constexpr int kRouterThreads = 256;
constexpr int kRouterWarps = kRouterThreads / 32;
constexpr int kRouterMaxK = 8;

// descending value, then ascending index: the larger key wins
__device__ __forceinline__ unsigned long long topk_key(float v, int idx) {
  uint32_t b = __float_as_uint(v);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving float -> uint
  return ((unsigned long long)b << 32) | (uint32_t)(0xFFFFFFFFu - (uint32_t)idx);
}

template <int PER>
__global__ void __launch_bounds__(kRouterThreads) router_topk_kernel(const float *__restrict__ in, int64_t T, int E,
                                                                     int k, int apply_softmax, int renormalize,
                                                                     float *__restrict__ gate_out,
                                                                     int64_t *__restrict__ idx_out,
                                                                     float *__restrict__ p_out) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kRouterWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  const float *row = in + t * E;
  float g[PER];
  if (apply_softmax) {
    double x[PER];
    double m = -INFINITY;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      x[j] = e < E ? (double)row[e] : -INFINITY;
      m = fmax(m, x[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      x[j] = (lane + 32 * j < E) ? exp(x[j] - m) : 0.0;
      s += x[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
    for (int j = 0; j < PER; ++j) g[j] = (float)(x[j] / s);
  } else {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      g[j] = e < E ? row[e] : 0.0f;
    }
  }
  if (gate_out) {
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      if (e < E) gate_out[t * E + e] = g[j];
    }
  }
  // k rounds of a warp arg-max over (value desc, index asc); winners are masked out.
  uint32_t taken = 0u;
  double sel_sum = 0.0;
  float sel_val[kRouterMaxK];
#pragma unroll
  for (int r = 0; r < kRouterMaxK; ++r) {
    if (r >= k) break;
    unsigned long long best = 0ull;
    float best_v = 0.0f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      if (e < E && !((taken >> j) & 1u)) {
        const unsigned long long key = topk_key(g[j], e);
        if (key > best) { best = key; best_v = g[j]; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, best, o);
      const float ov = __shfl_xor_sync(0xffffffffu, best_v, o);
      if (ok > best) { best = ok; best_v = ov; }
    }
    const int e_win = (int)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFull));
    if ((e_win & 31) == lane) taken |= 1u << (e_win >> 5);
    sel_val[r] = best_v;
    sel_sum += (double)best_v;
    if (lane == 0) idx_out[t * k + r] = e_win;
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < kRouterMaxK; ++r) {
      if (r >= k) break;
      p_out[t * k + r] = renormalize ? (float)((double)sel_val[r] / sel_sum) : sel_val[r];
    }
  }
}

// gate_backward (router.py:167-188): d logits from d p, float64 inside.
template <int PER>
__global__ void __launch_bounds__(kRouterThreads) router_backward_kernel(const float *__restrict__ gate,
                                                                         const int64_t *__restrict__ idx,
                                                                         const float *__restrict__ grad_p, int64_t T,
                                                                         int E, int k, int renormalized,
                                                                         float *__restrict__ dlogits) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kRouterWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  const float *g = gate + t * E;
  double s = 0.0, dotp = 0.0;
  if (renormalized) {
    for (int r = 0; r < k; ++r) s += (double)g[idx[t * k + r]];
    for (int r = 0; r < k; ++r) dotp += (double)grad_p[t * k + r] * ((double)g[idx[t * k + r]] / s);
  }
  double dg[PER];
  double gdot = 0.0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane + 32 * j;
    double v = 0.0;
    if (e < E) {
      for (int r = 0; r < k; ++r)
        if (idx[t * k + r] == e) v = renormalized ? ((double)grad_p[t * k + r] - dotp) / s : (double)grad_p[t * k + r];
      gdot += v * (double)g[e];
    }
    dg[j] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gdot += __shfl_xor_sync(0xffffffffu, gdot, o);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane + 32 * j;
    if (e < E) dlogits[t * E + e] = (float)((double)g[e] * (dg[j] - gdot));
  }
}

#define SMOE_ROUTER_DISPATCH(KERNEL, ...)                                            \
  do {                                                                               \
    const int per = (E + 31) / 32;                                                   \
    const unsigned blocks = (unsigned)((T + kRouterWarps - 1) / kRouterWarps);      \
    if (per <= 1) KERNEL<1><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);         \
    else if (per <= 2) KERNEL<2><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);    \
    else if (per <= 4) KERNEL<4><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);    \
    else if (per <= 8) KERNEL<8><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);    \
    else if (per <= 16) KERNEL<16><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);  \
    else KERNEL<32><<<blocks, kRouterThreads, 0, st>>>(__VA_ARGS__);                 \
  } while (0)

int router_topk(const float *in, int64_t T, int E, int k, int apply_softmax, int renormalize, float *gate_out,
                int64_t *idx_out, float *p_out, cudaStream_t st) {
  if (E < 1 || E > 1024) return fail(SMOE_EINVAL, "router: E must be in [1, 1024], got " + std::to_string(E));
  if (k < 1 || k > E || k > kRouterMaxK)
    return fail(SMOE_EINVAL, "router: k must be in [1, min(E, 8)], got " + std::to_string(k));
  if (T == 0) return SMOE_OK;
  SMOE_ROUTER_DISPATCH(router_topk_kernel, in, T, E, k, apply_softmax, renormalize, gate_out, idx_out, p_out);
  return check_launch("router_topk");
}

int router_backward(const float *gate, const int64_t *idx, const float *grad_p, int64_t T, int E, int k,
                    int renormalized, float *dlogits, cudaStream_t st) {
  if (E < 1 || E > 1024) return fail(SMOE_EINVAL, "router: E must be in [1, 1024]");
  if (k < 1 || k > E) return fail(SMOE_EINVAL, "router: k must be in [1, E]");
  if (T == 0) return SMOE_OK;
  SMOE_ROUTER_DISPATCH(router_backward_kernel, gate, idx, grad_p, T, E, k, renormalized, dlogits);
  return check_launch("router_backward");
}

}  // namespace smoe
