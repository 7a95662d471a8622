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
#ifndef SMOE_GROUP_INV_UNROLL
#define SMOE_GROUP_INV_UNROLL 1
#endif
constexpr int kGroupInvUnroll = SMOE_GROUP_INV_UNROLL;   // source chunks in flight per lane (A/B)
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
#pragma unroll kGroupInvUnroll
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
// Slot rows <-> the attention core's head layout.  One warp moves kHeadRows
// grouped rows per pass: every lane issues its 16-byte loads for all of them
// before the first store (a row is only h * d_head * 2 B = 1 KB at C3, so one
// row per warp left the copy latency-bound at ~4.4 TB/s).  C3 (268 MB moved,
// scripts/heads_move_bench.py): 2 rows 65 us, 4 rows 53.7, 8 rows 50.4, 16 rows
// 53; the 16-byte-element torch permute of the same bytes takes 42 us.
//   TO_HEADS = false: out[i] (grouped row) <- heads[b][hh*k + j][pos][:]
//   TO_HEADS = true : heads[b][hh*k + j][pos][:] <- grouped[i]
#ifndef SMOE_HEAD_ROWS
#define SMOE_HEAD_ROWS 8
#endif
constexpr int kHeadRows = SMOE_HEAD_ROWS;
template <typename T, bool TO_HEADS>
__global__ void __launch_bounds__(kRowThreads) heads_grouped_kernel(const T *__restrict__ src, int64_t seq_len,
                                                                    int k, int h, int dh,
                                                                    const int32_t *__restrict__ order, int64_t n,
                                                                    T *__restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5)) * kHeadRows;
  constexpr int N = 16 / sizeof(T);           // elements per 16-byte chunk
  const int cph = dh / N;                     // chunks per head
  const int cpr = h * cph;                    // chunks per row
  // lane r < kHeadRows resolves row i0 + r once: its head-layout base (head 0)
  int64_t hb = -1;
  if (lane < kHeadRows && i0 + lane < n) {
    const int64_t s = order[i0 + lane];
    const int64_t t = s / k;
    const int j = (int)(s - t * k);
    const int64_t b = t / seq_len, pos = t - b * seq_len;
    hb = ((b * h * k + j) * seq_len + pos) * (int64_t)dh;
  }
  const int64_t head_stride = (int64_t)k * seq_len * dh;   // head hh -> hh + 1 of one slot
  const int total = kHeadRows * cpr;
  for (int c0 = 0; c0 < total; c0 += 32 * 8) {
    uint4 v[8];
    int64_t doff[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      const int r = c < total ? c / cpr : 0;
      const int64_t base = __shfl_sync(0xffffffffu, hb, r);
      doff[u] = -1;
      if (c >= total || base < 0) continue;
      const int cc = c - r * cpr;
      const int hh = cc / cph, q = cc - hh * cph;
      const int64_t hoff = base + hh * head_stride + q * N;
      const int64_t goff = (i0 + r) * (int64_t)h * dh + (int64_t)cc * N;
      v[u] = __ldg(reinterpret_cast<const uint4 *>(src + (TO_HEADS ? goff : hoff)));
      doff[u] = TO_HEADS ? hoff : goff;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (doff[u] >= 0) *reinterpret_cast<uint4 *>(dst + doff[u]) = v[u];
  }
}

// out[i] = x[i] * w[order[i]] over grouped rows (the routing weight of each
// grouped row's slot), rounded once.
template <typename T>
__global__ void __launch_bounds__(kRowThreads) scale_grouped_rows_kernel(const T *__restrict__ x, int64_t d,
                                                                         const int32_t *__restrict__ order,
                                                                         int64_t n,
                                                                         const typename WOf<T>::type *__restrict__ w,
                                                                         T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  using A = typename AccOf<T>::type;
  const A wi = (A)w[order[i]];
  const T *src = x + i * d;
  T *dst = out + i * d;
  constexpr int N = Vec<T>::N;
  for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
    Vec<T> v = ldv(src + c), o;
#pragma unroll
    for (int q = 0; q < N; ++q) o.v[q] = Conv<T>::from_acc(Conv<T>::to_acc(v.v[q]) * wi);
    stv(dst + c, o);
  }
}

static inline unsigned row_blocks(int64_t rows);

int grouped_to_heads(const void *grouped, int64_t seq_len, int k, int h, int dh, const int32_t *order, int64_t n,
                     int dtype, void *heads, cudaStream_t st) {
  if (dtype == SMOE_F64) return fail(SMOE_ENOTSUP, "grouped_to_heads: bf16 / fp32 only");
  const int esz = dtype == SMOE_BF16 ? 2 : 4;
  if ((dh * esz) % 16 || (reinterpret_cast<uintptr_t>(heads) | reinterpret_cast<uintptr_t>(grouped)) % 16)
    return fail(SMOE_ENOTSUP, "grouped_to_heads: d_head * element size must be a multiple of 16 bytes (aligned)");
  if (n == 0) return SMOE_OK;
  if (dtype == SMOE_BF16)
    heads_grouped_kernel<__nv_bfloat16, true><<<row_blocks((n + kHeadRows - 1) / kHeadRows), kRowThreads, 0, st>>>(
        (const __nv_bfloat16 *)grouped, seq_len, k, h, dh, order, n, (__nv_bfloat16 *)heads);
  else
    heads_grouped_kernel<float, true><<<row_blocks((n + kHeadRows - 1) / kHeadRows), kRowThreads, 0, st>>>(
        (const float *)grouped, seq_len, k, h, dh, order, n, (float *)heads);
  return check_launch("grouped_to_heads");
}

int scale_grouped_rows(const void *x, int64_t d, const int32_t *order, int64_t n, const void *w, int dtype, void *out,
                       cudaStream_t st) {
  if (n == 0 || d == 0) return SMOE_OK;
  if (!vec_ok(x, d, dtype == SMOE_BF16 ? 2 : dtype == SMOE_F32 ? 4 : 8) ||
      !vec_ok(out, d, dtype == SMOE_BF16 ? 2 : dtype == SMOE_F32 ? 4 : 8))
    return fail(SMOE_ENOTSUP, "scale_grouped_rows: rows must be 16-byte aligned");
  SMOE_DTYPE_DISPATCH(dtype, {
    using W = typename WOf<T>::type;
    scale_grouped_rows_kernel<T><<<row_blocks(n), kRowThreads, 0, st>>>((const T *)x, d, order, n, (const W *)w,
                                                                        (T *)out);
  });
  return check_launch("scale_grouped_rows");
}

int heads_to_grouped(const void *heads, int64_t batch, int64_t seq_len, int k, int h, int dh, const int32_t *order,
                     int64_t n, int dtype, void *out, cudaStream_t st) {
  (void)batch;
  if (dtype == SMOE_F64) return fail(SMOE_ENOTSUP, "heads_to_grouped: bf16 / fp32 only");
  const int esz = dtype == SMOE_BF16 ? 2 : 4;
  if ((dh * esz) % 16 || (reinterpret_cast<uintptr_t>(heads) | reinterpret_cast<uintptr_t>(out)) % 16)
    return fail(SMOE_ENOTSUP, "heads_to_grouped: d_head * element size must be a multiple of 16 bytes (aligned)");
  if (dtype == SMOE_BF16)
    heads_grouped_kernel<__nv_bfloat16, false><<<row_blocks((n + kHeadRows - 1) / kHeadRows), kRowThreads, 0, st>>>(
        (const __nv_bfloat16 *)heads, seq_len, k, h, dh, order, n, (__nv_bfloat16 *)out);
  else
    heads_grouped_kernel<float, false><<<row_blocks((n + kHeadRows - 1) / kHeadRows), kRowThreads, 0, st>>>(
        (const float *)heads, seq_len, k, h, dh, order, n, (float *)out);
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
