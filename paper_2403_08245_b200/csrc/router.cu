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

// ---- gate GEMM fused into the router ----------------------
// router.py:119-151: logits = x @ W_g accumulated in float64 (the reference
// upcasts both operands, :121-122), softmax in float64 rounded once to float32,
// stable top-k on the float32 gates, p renormalised in float64.  One block
// owns kGateTokens tokens, one lane per token: W_g is staged in shared memory
// as float64 in chunks of kGateChunk rows and read by broadcast (every lane of
// a warp reads the same W_g element), each lane streams its token's x row
// (16-byte vectors, L1-resident across the 8 elements of a vector) and keeps
// up to kGateEG float64 accumulators; the logits tile then goes through shared
// memory so each lane finishes its token's softmax / top-k / renormalisation
// and writes gate, expert ids and p — the ids feed the K1 sort directly.
constexpr int kGateTokens = 128;   // tokens per block (4 warps)
constexpr int kGateChunk = 128;    // W_g rows staged per pass
// experts accumulated per pass over x: EG = 8 (E <= 8) or 16

template <typename XT>
__device__ __forceinline__ void load8(const XT *p, double (&v)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16 *p, double (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = (double)__uint_as_float(w[i] << 16);
    v[2 * i + 1] = (double)__uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float *p, double (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <typename XT, int kGateEG, bool VEC>
__global__ void __launch_bounds__(kGateTokens) router_gate_kernel(const void *__restrict__ x_raw,
                                                                  const float *__restrict__ wg,
                                                                  int64_t T, int D, int E, int k, int renormalize,
                                                                  float *__restrict__ gate_out,
                                                                  int64_t *__restrict__ idx_out,
                                                                  float *__restrict__ p_out) {
  extern __shared__ double g_sm[];
  const XT *x = static_cast<const XT *>(x_raw);
  double *s_w = g_sm;                                  // [kGateChunk][kGateEG]
  double *s_logit = g_sm + kGateChunk * kGateEG;       // [kGateTokens][E + 1]
  const int ldl = E + 1;
  const int64_t t = (int64_t)blockIdx.x * kGateTokens + threadIdx.x;
  const bool live = t < T;
  const XT *xrow = x + (live ? t : 0) * (int64_t)D;
  for (int e0 = 0; e0 < E; e0 += kGateEG) {
    const int eg = min(kGateEG, E - e0);
    double acc[kGateEG];
#pragma unroll
    for (int j = 0; j < kGateEG; ++j) acc[j] = 0.0;
    for (int d0 = 0; d0 < D; d0 += kGateChunk) {
      const int dc = min(kGateChunk, D - d0);
      __syncthreads();
      for (int i = threadIdx.x; i < kGateChunk * kGateEG; i += kGateTokens) {
        const int r = i / kGateEG, c = i - r * kGateEG;
        s_w[i] = (r < dc && c < eg) ? (double)wg[(int64_t)(d0 + r) * E + e0 + c] : 0.0;
      }
      __syncthreads();
      if (VEC) {
        for (int r = 0; r < dc; r += 8) {
          double xv[8];
          load8<XT>(xrow + d0 + r, xv);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double *wr = s_w + (r + i) * kGateEG;
#pragma unroll
            for (int j = 0; j < kGateEG; ++j) acc[j] = fma(xv[i], wr[j], acc[j]);
          }
        }
      } else {
        for (int r = 0; r < dc; ++r) {
          const double xv = (double)Conv<XT>::to_acc(xrow[d0 + r]);
          const double *wr = s_w + r * kGateEG;
#pragma unroll
          for (int j = 0; j < kGateEG; ++j) acc[j] = fma(xv, wr[j], acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kGateEG; ++j)
      if (j < eg) s_logit[threadIdx.x * ldl + e0 + j] = acc[j];
  }
  if (!live) return;
  // softmax over the token's row (float64), rounded once; stable top-k on the rounded gates
  const double *z = s_logit + threadIdx.x * ldl;
  double m = -INFINITY;
  for (int e = 0; e < E; ++e) m = fmax(m, z[e]);
  double ssum = 0.0;
  for (int e = 0; e < E; ++e) ssum += exp(z[e] - m);
  int sel[kRouterMaxK];
  float selv[kRouterMaxK];
  int have = 0;
  for (int e = 0; e < E; ++e) {
    const float g = (float)(exp(z[e] - m) / ssum);
    if (gate_out) gate_out[t * E + e] = g;
    // insertion into the running top-k: strictly larger value wins, ties keep the lower id
    int pos = have < k ? have : k;
    while (pos > 0 && g > selv[pos - 1]) --pos;
    if (pos < k) {
      for (int q = (have < k ? have : k - 1); q > pos; --q) { sel[q] = sel[q - 1]; selv[q] = selv[q - 1]; }
      sel[pos] = e;
      selv[pos] = g;
      if (have < k) ++have;
    }
  }
  double s = 0.0;
  for (int r = 0; r < k; ++r) s += (double)selv[r];
  for (int r = 0; r < k; ++r) {
    idx_out[t * k + r] = sel[r];
    p_out[t * k + r] = renormalize ? (float)((double)selv[r] / s) : selv[r];
  }
}

int router_gate(const void *x, int x_dtype, const float *wg, int64_t T, int D, int E, int k, int renormalize,
                float *gate_out, int64_t *idx_out, float *p_out, cudaStream_t st) {
  if (E < 1 || E > 1024) return fail(SMOE_EINVAL, "router_gate: E must be in [1, 1024], got " + std::to_string(E));
  if (k < 1 || k > E || k > kRouterMaxK)
    return fail(SMOE_EINVAL, "router_gate: k must be in [1, min(E, 8)], got " + std::to_string(k));
  if (x_dtype != SMOE_BF16 && x_dtype != SMOE_F32) return fail(SMOE_EINVAL, "router_gate: x must be bf16 or fp32");
  // 16-byte row vectors when every row starts aligned; element loads otherwise
  const bool vec = D % 8 == 0 && ((uintptr_t)x & 15) == 0;
  if (T == 0) return SMOE_OK;
  const int eg = E <= 8 ? 8 : 16;
  const size_t smem = sizeof(double) * ((size_t)kGateChunk * eg + (size_t)kGateTokens * (E + 1));
  if (smem > 227 * 1024) return fail(SMOE_ENOTSUP, "router_gate: too many experts for the shared logits tile");
  const unsigned blocks = (unsigned)((T + kGateTokens - 1) / kGateTokens);
  using GateFn = void (*)(const void *, const float *, int64_t, int, int, int, int, float *, int64_t *, float *);
  GateFn kern = nullptr;
  if (x_dtype == SMOE_BF16)
    kern = eg == 8 ? (vec ? router_gate_kernel<__nv_bfloat16, 8, true> : router_gate_kernel<__nv_bfloat16, 8, false>)
                   : (vec ? router_gate_kernel<__nv_bfloat16, 16, true> : router_gate_kernel<__nv_bfloat16, 16, false>);
  else
    kern = eg == 8 ? (vec ? router_gate_kernel<float, 8, true> : router_gate_kernel<float, 8, false>)
                   : (vec ? router_gate_kernel<float, 16, true> : router_gate_kernel<float, 16, false>);
  if (smem > 48 * 1024 && cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem) != cudaSuccess)
    return check_launch("router_gate: smem attribute", 0);
  kern<<<blocks, kGateTokens, smem, st>>>(x, wg, T, D, E, k, renormalize, gate_out, idx_out, p_out);
  return check_launch("router_gate");
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
