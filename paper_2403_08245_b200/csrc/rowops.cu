// HBM-bound row kernels of the ParallelLinear path (K5/K9 and the combine /
// fan-out reductions of SURVEY.md §2.3).  One warp owns one output row and
// moves it with 16-byte vectors; sums accumulate in fp32 for bf16 storage and
// in 64-bit for the fp32 check mode, are rounded once and written once, so the
// results are deterministic (no atomics anywhere).
//
//   group            kernels.py:289-326       out[i] = x[o[i]/F] * w[o[i]]
//   combine          parallel_linear.py:69-73 y[s]  = sum_j p[s,j] y_hat[s*J+j]
//   combine_grad_p   parallel_linear.py:198-206  dp[s,j] = <dy[s], y_hat[s*J+j]>
//   fanout_reduce    parallel_linear.py:259-266  dx[t] = sum_j g[t*F+j]
//   activation       moe_layers.py:75-83      act(x) / act'(x)
#include "common.cuh"

namespace smoe {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;

// Launch `launch` (which names the template constant FKC) with the fan-out as
// a compile-time constant for the common k = 1, 2, 4, 8, dynamic otherwise.
#define SMOE_FANOUT_DISPATCH(fan, launch)       \
  do {                                          \
    switch (fan) {                              \
      case 1: { constexpr int FKC = 1; launch; } break; \
      case 2: { constexpr int FKC = 2; launch; } break; \
      case 4: { constexpr int FKC = 4; launch; } break; \
      case 8: { constexpr int FKC = 8; launch; } break; \
      default: { constexpr int FKC = 0; launch; } break; \
    }                                           \
  } while (0)

template <typename T> struct alignas(16) Vec {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

template <typename T> __device__ __forceinline__ Vec<T> ldv(const T *p) {
  Vec<T> r;
  *reinterpret_cast<uint4 *>(&r) = __ldg(reinterpret_cast<const uint4 *>(p));
  return r;
}
template <typename T> __device__ __forceinline__ void stv(T *p, const Vec<T> &v) {
  *reinterpret_cast<uint4 *>(p) = *reinterpret_cast<const uint4 *>(&v);
}

static inline bool vec_ok(const void *p, int64_t d, size_t esz) {
  return ((uintptr_t)p % 16 == 0) && ((d * (int64_t)esz) % 16 == 0);
}

// ---- group -----------------------------------------------------------------
template <typename T, bool VEC>
__global__ void __launch_bounds__(kRowThreads) group_kernel(const T *__restrict__ x, int64_t d,
                                                             const int32_t *__restrict__ order,
                                                             int64_t n, int fan_out,
                                                             const typename WOf<T>::type *__restrict__ weights,
                                                             T *__restrict__ out) {
  using A = typename AccOf<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const int32_t slot = order[i];
  const T *src = x + (int64_t)(slot / fan_out) * d;
  T *dst = out + i * d;
  // the product is rounded to the storage dtype (kernels.py:323-325)
  const A wgt = weights ? (A)weights[slot] : A(1);
  if (VEC) {
    constexpr int N = Vec<T>::N;
    for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
      Vec<T> v = ldv(src + c);
      if (weights) {
#pragma unroll
        for (int q = 0; q < N; ++q) v.v[q] = Conv<T>::from_acc(Conv<T>::to_acc(v.v[q]) * wgt);
      }
      stv(dst + c, v);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      T v = src[c];
      dst[c] = weights ? Conv<T>::from_acc(Conv<T>::to_acc(v) * wgt) : v;
    }
  }
}

// ---- group, token-major (fan-out > 1) ---------------------------------------
// Same result as group_kernel, visited by source row: one warp loads x[t] once
// and writes it (times w[s]) to the k grouped positions inv[s], s = t*F + j.
// group_kernel's grouped-order visit re-reads each source row once per bin
// (k times, from DRAM when x exceeds L2); this reads it once.
// FK > 0: the fan-out is a compile-time constant (1, 2, 4, 8: destinations and
// weights stay in registers and the k stores of a chunk issue back to back).
template <typename T, bool VEC, int FK>
__global__ void __launch_bounds__(kRowThreads) group_inv_kernel(const T *__restrict__ x, int64_t d,
                                                                const int32_t *__restrict__ inv, int64_t t_rows,
                                                                int fan_out,
                                                                const typename WOf<T>::type *__restrict__ weights,
                                                                T *__restrict__ out) {
  using A = typename AccOf<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (t >= t_rows) return;
  const T *src = x + t * d;
  constexpr int MAXF = FK > 0 ? FK : 16;
  int64_t dst[MAXF];
  A wgt[MAXF];
  const int F = FK > 0 ? FK : (fan_out < MAXF ? fan_out : MAXF);
#pragma unroll
  for (int j = 0; j < MAXF; ++j) {
    if (j >= F) break;
    const int64_t s = t * fan_out + j;
    dst[j] = (int64_t)inv[s] * d;
    wgt[j] = weights ? (A)weights[s] : A(1);
  }
  if (VEC) {
    constexpr int N = Vec<T>::N;
    for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
      const Vec<T> v = ldv(src + c);
#pragma unroll
      for (int j = 0; j < MAXF; ++j) {
        if (j >= F) break;
        Vec<T> o = v;
        if (weights) {
#pragma unroll
          for (int q = 0; q < N; ++q) o.v[q] = Conv<T>::from_acc(Conv<T>::to_acc(v.v[q]) * wgt[j]);
        }
        stv(out + dst[j] + c, o);
      }
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      const T v = src[c];
#pragma unroll
      for (int j = 0; j < MAXF; ++j) {
        if (j >= F) break;
        out[dst[j] + c] = weights ? Conv<T>::from_acc(Conv<T>::to_acc(v) * wgt[j]) : v;
      }
    }
  }
}

// ---- MoMHA: attention-core head layout -> grouped slot rows ----------------
// One warp per grouped row i: slot s = order[i], token t = s / k, choice j;
// the row's d_proj = h * d_head values come from head hh * k + j of t's
// sequence position, d_head contiguous elements per head (16-byte chunks).
template <typename T>
__global__ void __launch_bounds__(kRowThreads) heads_to_grouped_kernel(const T *__restrict__ heads, int64_t seq_len,
                                                                       int k, int h, int dh,
                                                                       const int32_t *__restrict__ order, int64_t n,
                                                                       T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const int64_t s = order[i];
  const int64_t t = s / k;
  const int j = (int)(s - t * k);
  const int64_t b = t / seq_len, pos = t - b * seq_len;
  constexpr int N = 16 / sizeof(T);           // elements per 16-byte chunk
  const int cph = dh / N;                     // chunks per head
  T *dst = out + i * (int64_t)h * dh;
  for (int c = lane; c < h * cph; c += 32) {
    const int hh = c / cph, q = c - hh * cph;
    const T *src = heads + (((b * h + hh) * k + j) * seq_len + pos) * (int64_t)dh + q * N;
    *reinterpret_cast<uint4 *>(dst + hh * dh + q * N) = __ldg(reinterpret_cast<const uint4 *>(src));
  }
}

static inline unsigned row_blocks(int64_t rows);

int heads_to_grouped(const void *heads, int64_t batch, int64_t seq_len, int k, int h, int dh, const int32_t *order,
                     int64_t n, int dtype, void *out, cudaStream_t st) {
  (void)batch;
  if (dtype == SMOE_F64) return fail(SMOE_ENOTSUP, "heads_to_grouped: bf16 / fp32 only");
  const int esz = dtype == SMOE_BF16 ? 2 : 4;
  if ((dh * esz) % 16 || (reinterpret_cast<uintptr_t>(heads) | reinterpret_cast<uintptr_t>(out)) % 16)
    return fail(SMOE_ENOTSUP, "heads_to_grouped: d_head * element size must be a multiple of 16 bytes (aligned)");
  if (dtype == SMOE_BF16)
    heads_to_grouped_kernel<__nv_bfloat16><<<row_blocks(n), kRowThreads, 0, st>>>(
        (const __nv_bfloat16 *)heads, seq_len, k, h, dh, order, n, (__nv_bfloat16 *)out);
  else
    heads_to_grouped_kernel<float><<<row_blocks(n), kRowThreads, 0, st>>>((const float *)heads, seq_len, k, h, dh,
                                                                         order, n, (float *)out);
  return check_launch("heads_to_grouped");
}

// ---- combine ---------------------------------------------------------------
// inv (optional): y_hat holds the slot rows in GROUPED order and slot s*J+j is
// row inv[s*J+j] (the grouped-output GEMM's layout); null = slot order.
template <typename T, bool VEC, int JK>
__global__ void __launch_bounds__(kRowThreads) combine_kernel(const T *__restrict__ y_hat,
                                                               const typename WOf<T>::type *__restrict__ p,
                                                               int64_t S, int J_, int64_t d,
                                                               T *__restrict__ y, const int32_t *__restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (s >= S) return;
  using A = typename AccOf<T>::type;
  const int J = JK > 0 ? JK : J_;   // JK > 0: compile-time k (weights in registers, all k loads in flight)
  A pw[JK > 0 ? JK : 1];
  if (JK > 0) {
#pragma unroll
    for (int j = 0; j < (JK > 0 ? JK : 1); ++j) pw[j] = p[s * J + j];
  }
  const T *src = y_hat + s * J * d;
  T *dst = y + s * d;
  // row of slot s*J+j: (JK > 0) offsets in registers, all k loads in flight
  int64_t roff[JK > 0 ? JK : 1];
  if (JK > 0) {
#pragma unroll
    for (int j = 0; j < (JK > 0 ? JK : 1); ++j) roff[j] = (inv ? (int64_t)inv[s * J + j] - s * J : j) * d;
  }
  if (VEC) {
    constexpr int N = Vec<T>::N;
    for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
      A acc[N];
#pragma unroll
      for (int q = 0; q < N; ++q) acc[q] = 0;
#pragma unroll
      for (int j = 0; j < (JK > 0 ? JK : J); ++j) {
        const A pj = JK > 0 ? pw[j] : (A)p[s * J + j];
        const int64_t ro = JK > 0 ? roff[j] : (inv ? (int64_t)inv[s * J + j] - s * J : j) * d;
        Vec<T> v = ldv(src + ro + c);
#pragma unroll
        for (int q = 0; q < N; ++q) acc[q] = fma(pj, Conv<T>::to_acc(v.v[q]), acc[q]);
      }
      Vec<T> o;
#pragma unroll
      for (int q = 0; q < N; ++q) o.v[q] = Conv<T>::from_acc(acc[q]);
      stv(dst + c, o);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      A acc = 0;
      for (int j = 0; j < J; ++j) {
        const int64_t ro = (inv ? (int64_t)inv[s * J + j] - s * J : j) * d;
        acc = fma((A)p[s * J + j], Conv<T>::to_acc(src[ro + c]), acc);
      }
      dst[c] = Conv<T>::from_acc(acc);
    }
  }
}

// ---- dp --------------------------------------------------------------------
// One warp per combine row s; J partial dot products reduced with shuffles.
// inv (optional): y_hat in grouped order, slot s*J+j is row inv[s*J+j].
template <typename T, bool VEC>
__global__ void __launch_bounds__(kRowThreads) combine_grad_p_kernel(const T *__restrict__ dy,
                                                                      const T *__restrict__ y_hat,
                                                                      int64_t S, int J, int64_t d,
                                                                      typename WOf<T>::type *__restrict__ dp,
                                                                      const int32_t *__restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (s >= S) return;
  using A = typename AccOf<T>::type;
  const T *g = dy + s * d;
  for (int j = 0; j < J; ++j) {
    const T *yh = y_hat + (inv ? (int64_t)inv[s * J + j] : s * J + j) * d;
    A acc = 0;
    if (VEC) {
      constexpr int N = Vec<T>::N;
      for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
        Vec<T> a = ldv(g + c), b = ldv(yh + c);
#pragma unroll
        for (int q = 0; q < N; ++q) acc = fma(Conv<T>::to_acc(a.v[q]), Conv<T>::to_acc(b.v[q]), acc);
      }
    } else {
      for (int64_t c = lane; c < d; c += 32) acc = fma(Conv<T>::to_acc(g[c]), Conv<T>::to_acc(yh[c]), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) dp[s * J + j] = (typename WOf<T>::type)acc;
  }
}

// ---- fan-out reduce --------------------------------------------------------
// inv (optional): g holds the slot rows in GROUPED order (slot t*F+j is row
// inv[t*F+j]); null = slot order.  Same summation order either way.
template <typename T, bool VEC, int FK>
__global__ void __launch_bounds__(kRowThreads) fanout_reduce_kernel(const T *__restrict__ g,
                                                                     int64_t Trows, int F_,
                                                                     int64_t d,
                                                                     T *__restrict__ dx,
                                                                     const int32_t *__restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (t >= Trows) return;
  using A = typename AccOf<T>::type;
  const int F = FK > 0 ? FK : F_;   // FK > 0: compile-time fan-out, all k loads in flight
  const T *src = g + t * F * d;
  T *dst = dx + t * d;
  int64_t roff[FK > 0 ? FK : 1];
  if (FK > 0) {
#pragma unroll
    for (int j = 0; j < (FK > 0 ? FK : 1); ++j) roff[j] = (inv ? (int64_t)inv[t * F + j] - t * F : j) * d;
  }
  if (VEC) {
    constexpr int N = Vec<T>::N;
    for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
      A acc[N];
#pragma unroll
      for (int q = 0; q < N; ++q) acc[q] = 0;
#pragma unroll
      for (int j = 0; j < (FK > 0 ? FK : F); ++j) {
        const int64_t ro = FK > 0 ? roff[j] : (inv ? (int64_t)inv[t * F + j] - t * F : j) * d;
        Vec<T> v = ldv(src + ro + c);
#pragma unroll
        for (int q = 0; q < N; ++q) acc[q] += Conv<T>::to_acc(v.v[q]);
      }
      Vec<T> o;
#pragma unroll
      for (int q = 0; q < N; ++q) o.v[q] = Conv<T>::from_acc(acc[q]);
      stv(dst + c, o);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      A acc = 0;
      for (int j = 0; j < F; ++j) acc += Conv<T>::to_acc(src[(inv ? (int64_t)inv[t * F + j] - t * F : j) * d + c]);
      dst[c] = Conv<T>::from_acc(acc);
    }
  }
}

// ---- activation ------------------------------------------------------------
template <typename T>
__global__ void activation_kernel(const T *__restrict__ x, int64_t numel, int act, int deriv,
                                  T *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
       i += (int64_t)gridDim.x * blockDim.x) {
    const auto z = Conv<T>::to_acc(x[i]);   // fp32 storage: 64-bit evaluation, one rounding
    out[i] = Conv<T>::from_acc(deriv ? act_grad(act, z) : act_fwd(act, z));
  }
}

// ---- dispatch --------------------------------------------------------------
static inline unsigned row_blocks(int64_t rows) { return (unsigned)((rows + kRowWarps - 1) / kRowWarps); }

int group(const void *x, int64_t d, const int32_t *order, int64_t n, int fan_out, const void *w, int dtype,
          void *out, cudaStream_t st) {
  if (n == 0 || d == 0) return SMOE_OK;
  SMOE_DTYPE_DISPATCH(dtype, {
    using W = typename WOf<T>::type;
    if (vec_ok(x, d, sizeof(T)) && vec_ok(out, d, sizeof(T)))
      group_kernel<T, true><<<row_blocks(n), kRowThreads, 0, st>>>((const T *)x, d, order, n, fan_out,
                                                                   (const W *)w, (T *)out);
    else
      group_kernel<T, false><<<row_blocks(n), kRowThreads, 0, st>>>((const T *)x, d, order, n, fan_out,
                                                                    (const W *)w, (T *)out);
  });
  return check_launch("group");
}

int group_inv(const void *x, int64_t t_rows, int64_t d, const int32_t *inv, int fan_out, const void *w, int dtype,
              void *out, cudaStream_t st) {
  if (t_rows == 0 || d == 0) return SMOE_OK;
  SMOE_DTYPE_DISPATCH(dtype, {
    using W = typename WOf<T>::type;
    if (vec_ok(x, d, sizeof(T)) && vec_ok(out, d, sizeof(T)))
      SMOE_FANOUT_DISPATCH(fan_out, (group_inv_kernel<T, true, FKC><<<row_blocks(t_rows), kRowThreads, 0, st>>>(
                                        (const T *)x, d, inv, t_rows, fan_out, (const W *)w, (T *)out)));
    else
      group_inv_kernel<T, false, 0><<<row_blocks(t_rows), kRowThreads, 0, st>>>((const T *)x, d, inv, t_rows, fan_out,
                                                                                 (const W *)w, (T *)out);
  });
  return check_launch("group_inv");
}

int combine(const void *y_hat, const void *p, int64_t S, int J, int64_t d, int dtype, void *y, cudaStream_t st,
            const int32_t *inv) {
  if (S == 0 || d == 0) return SMOE_OK;
  SMOE_DTYPE_DISPATCH(dtype, {
    using W = typename WOf<T>::type;
    if (vec_ok(y_hat, d, sizeof(T)) && vec_ok(y, d, sizeof(T)))
      SMOE_FANOUT_DISPATCH(J, (combine_kernel<T, true, FKC><<<row_blocks(S), kRowThreads, 0, st>>>(
                                  (const T *)y_hat, (const W *)p, S, J, d, (T *)y, inv)));
    else
      combine_kernel<T, false, 0><<<row_blocks(S), kRowThreads, 0, st>>>((const T *)y_hat, (const W *)p, S, J, d,
                                                                         (T *)y, inv);
  });
  return check_launch("combine");
}

int combine_grad_p(const void *dy, const void *y_hat, int64_t S, int J, int64_t d, int dtype, void *dp,
                   cudaStream_t st, const int32_t *inv) {
  if (S == 0) return SMOE_OK;
  SMOE_DTYPE_DISPATCH(dtype, {
    using W = typename WOf<T>::type;
    if (vec_ok(dy, d, sizeof(T)) && vec_ok(y_hat, d, sizeof(T)))
      combine_grad_p_kernel<T, true><<<row_blocks(S), kRowThreads, 0, st>>>((const T *)dy, (const T *)y_hat, S, J, d,
                                                                            (W *)dp, inv);
    else
      combine_grad_p_kernel<T, false><<<row_blocks(S), kRowThreads, 0, st>>>((const T *)dy, (const T *)y_hat, S, J, d,
                                                                             (W *)dp, inv);
  });
  return check_launch("combine_grad_p");
}

// dp[order[i]] = sum_j part[i * parts + j]: one thread per grouped row, the
// partials summed in a fixed order (deterministic).
__global__ void dp_from_partials_kernel(const float *__restrict__ part, int64_t n, int parts,
                                        const int32_t *__restrict__ order, float *__restrict__ dp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float *r = part + i * parts;
  float s = 0.0f;
  for (int j = 0; j < parts; ++j) s += r[j];
  dp[order[i]] = s;
}

int dp_from_partials(const float *part, int64_t n, int parts, const int32_t *order, float *dp, cudaStream_t st) {
  if (n == 0) return SMOE_OK;
  dp_from_partials_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, n, parts, order, dp);
  return check_launch("dp_from_partials");
}

int fanout_reduce(const void *g, int64_t Trows, int F, int64_t d, int dtype, void *dx, cudaStream_t st,
                  const int32_t *inv) {
  if (Trows == 0 || d == 0) return SMOE_OK;
  SMOE_DTYPE_DISPATCH(dtype, {
    if (vec_ok(g, d, sizeof(T)) && vec_ok(dx, d, sizeof(T)))
      SMOE_FANOUT_DISPATCH(F, (fanout_reduce_kernel<T, true, FKC><<<row_blocks(Trows), kRowThreads, 0, st>>>(
                                  (const T *)g, Trows, F, d, (T *)dx, inv)));
    else
      fanout_reduce_kernel<T, false, 0><<<row_blocks(Trows), kRowThreads, 0, st>>>((const T *)g, Trows, F, d, (T *)dx,
                                                                                   inv);
  });
  return check_launch("fanout_reduce");
}

int activation(const void *x, int64_t numel, int act, int deriv, int dtype, void *out, cudaStream_t st) {
  if (numel == 0) return SMOE_OK;
  int64_t blocks64 = (numel + 255) / 256;
  unsigned blocks = (unsigned)(blocks64 < 148 * 32 ? blocks64 : 148 * 32);
  SMOE_DTYPE_DISPATCH(dtype, (activation_kernel<T><<<blocks, 256, 0, st>>>((const T *)x, numel, act, deriv, (T *)out)));
  return check_launch("activation");
}

}  // namespace smoe
