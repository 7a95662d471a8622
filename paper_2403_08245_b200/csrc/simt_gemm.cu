// K10: SIMT (FFMA) grouped GEMMs — the fp32 check mode of SURVEY.md §2.3.
//
// fp32 inputs need real fp32 products (TF32 misses the 1e-4 bar),
// so the check mode runs on the CUDA cores.  The same kernels also accept bf16
// storage (fp32 accumulate) and serve as the engine=SIMT cross-check of the
// tcgen05 path.  Index semantics are those of kernels.py:143-220 (scatter2scatter),
// :242-286 (scatter_combine) and :329-361 (group_xty).
//
// Tile: 64x64 outputs per 256-thread CTA, K staged 16 deep in shared memory,
// 4x4 outputs per thread, one rounding on store.  fp32 storage accumulates in
// 64-bit (the reference's contract, core_tensor.py:1-7: "every dot-product
// style reduction accumulates in 64-bit and rounds once"), bf16 in fp32.  Row tiles
// never straddle a bin (kernels.py:127-135), so every output row is written by
// exactly one CTA and there are no atomics (except the inference combine).
#include <type_traits>

#include "common.cuh"

namespace smoe {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16, S_THREADS = 256;

// Locate the (expert, row-tile) pair of linear m-tile `mt`; returns false past the end.
__device__ __forceinline__ bool find_mtile(const int32_t *s_off, int E, int64_t mt, int &e,
                                           int64_t &row0, int64_t &row1) {
  int64_t cum = 0;
  for (int x = 0; x < E; ++x) {
    int64_t cnt = s_off[x + 1] - s_off[x];
    int64_t tiles = (cnt + SB_M - 1) / SB_M;
    if (mt < cum + tiles) {
      e = x;
      row0 = s_off[x] + (mt - cum) * SB_M;
      row1 = s_off[x + 1];
      return true;
    }
    cum += tiles;
  }
  return false;
}

template <typename T>
__global__ void __launch_bounds__(S_THREADS) simt_s2s_kernel(
    const T *__restrict__ x, const T *__restrict__ w, int E, int64_t w_rows, int64_t w_cols,
    const int32_t *__restrict__ order, const int32_t *__restrict__ offsets, int fan_out,
    int grouped_in, int grouped_out, int trans_w, int epi, int act, T *__restrict__ out,
    T *__restrict__ out2, const T *__restrict__ aux, int64_t max_mtiles,
    // inference combine (scatter_combine): non-null -> atomically accumulate
    const typename WOf<T>::type *__restrict__ p_flat, int combine_cols,
    typename WOf<T>::type *__restrict__ y_accum) {
  using A = typename AccOf<T>::type;
  extern __shared__ int32_t s_off[];
  __shared__ A As[SB_K][SB_M + 4];
  __shared__ A Bs[SB_K][SB_N + 4];
  __shared__ int64_t s_src[SB_M];
  __shared__ int64_t s_dst[SB_M];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_off[i] = offsets[i];
  __syncthreads();

  const int64_t d_in = trans_w ? w_cols : w_rows;
  const int64_t d_out = trans_w ? w_rows : w_cols;
  const int64_t n0 = (int64_t)blockIdx.x * SB_N;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;

  for (int64_t mt = blockIdx.y; mt < max_mtiles; mt += gridDim.y) {
    int e;
    int64_t row0, row1;
    if (!find_mtile(s_off, E, mt, e, row0, row1)) return;
    const T *we = w + (int64_t)e * w_rows * w_cols;
    __syncthreads();
    if (tid < SB_M) {
      int64_t i = row0 + tid;
      int64_t src = -1, dst = -1;
      if (i < row1) {
        int64_t slot = order[i];
        src = grouped_in ? i : slot / fan_out;
        dst = grouped_out ? i : slot;
      }
      s_src[tid] = src;
      s_dst[tid] = dst;
    }
    __syncthreads();

    A acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0;

    for (int64_t k0 = 0; k0 < d_in; k0 += SB_K) {
      // A tile: 64 rows x 16 k (4 elements per thread)
      {
        int r = tid / 4, kq = (tid % 4) * 4;
        int64_t src = s_src[r];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int64_t kk = k0 + kq + q;
          As[kq + q][r] = (src >= 0 && kk < d_in) ? Conv<T>::to_acc(x[src * d_in + kk]) : A(0);
        }
      }
      // B tile: 16 k x 64 n; B[k][n] = trans ? W[e][n][k] : W[e][k][n]
      {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int idx = tid + q * S_THREADS;  // 0..1023
          int kr, nc;
          if (trans_w) { nc = idx / SB_K; kr = idx % SB_K; }   // contiguous along k
          else { kr = idx / SB_N; nc = idx % SB_N; }            // contiguous along n
          int64_t kk = k0 + kr, nn = n0 + nc;
          A v = 0;
          if (kk < d_in && nn < d_out) v = Conv<T>::to_acc(trans_w ? we[nn * w_cols + kk] : we[kk * w_cols + nn]);
          Bs[kr][nc] = v;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < SB_K; ++kk) {
        A a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { a[q] = As[kk][ty + 16 * q]; b[q] = Bs[kk][tx + 16 * q]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = ty + 16 * i;
      int64_t dst = s_dst[r];
      if (dst < 0) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int64_t nn = n0 + tx + 16 * j;
        if (nn >= d_out) continue;
        const A v = acc[i][j];
        if (y_accum) {
          const A pv = (A)p_flat[dst];
          atomicAdd(&y_accum[(dst / combine_cols) * d_out + nn], (typename WOf<T>::type)(pv * v));
          continue;
        }
        int64_t off = dst * d_out + nn;
        if (epi == SMOE_EPI_ACT) {
          // pre-activation rounded to storage, activation of the rounded value
          // rounded once more (moe_layers.py:169-175)
          T pre = Conv<T>::from_acc(v);
          out[off] = pre;
          out2[off] = Conv<T>::from_acc(act_fwd(act, Conv<T>::to_acc(pre)));
        } else if (epi == SMOE_EPI_ACT_ONLY) {
          out[off] = Conv<T>::from_acc(act_fwd(act, Conv<T>::to_acc(Conv<T>::from_acc(v))));
        } else if (epi == SMOE_EPI_ACT_GRAD) {
          if constexpr (std::is_same<T, float>::value) {
            // check mode: dH = round(round(acc) * round(act'(h_pre))), the
            // storage-precision product of moe_layers.py:203-206
            const T g = Conv<T>::from_acc(v);
            const T d = Conv<T>::from_acc(act_grad(act, Conv<T>::to_acc(aux[off])));
            out[off] = g * d;
          } else {
            out[off] = Conv<T>::from_acc(v * act_grad(act, Conv<T>::to_acc(aux[off])));  // as the tcgen05 epilogue
          }
        } else {
          out[off] = Conv<T>::from_acc(v);
        }
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(S_THREADS) simt_xty_kernel(const T *__restrict__ xg,
                                                             const T *__restrict__ yg,
                                                             const int32_t *__restrict__ offsets,
                                                             int64_t d_in, int64_t d_out,
                                                             T *__restrict__ dw,
                                                             const int32_t *__restrict__ order = nullptr,
                                                             int fa = 1, int ga = 1, int fb = 1, int gb = 1) {
  using A = typename AccOf<T>::type;
  __shared__ A As[SB_K][SB_M + 4];
  __shared__ A Bs[SB_K][SB_N + 4];
  const int e = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * SB_M, n0 = (int64_t)blockIdx.x * SB_N;
  const int64_t r0 = offsets[e], r1 = offsets[e + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  A acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0;

  for (int64_t k0 = r0; k0 < r1; k0 += SB_K) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + q * S_THREADS;
      int kr = idx / SB_M, c = idx % SB_M;
      int64_t r = k0 + kr;
      int64_t mm = m0 + c, nn = n0 + c;
      // scattered operands: grouped position r reads row order[r] / fan_out
      const int64_t ra = (r < r1 && !ga) ? order[r] / fa : r;
      const int64_t rb = (r < r1 && !gb) ? order[r] / fb : r;
      As[kr][c] = (r < r1 && mm < d_in) ? Conv<T>::to_acc(xg[ra * d_in + mm]) : A(0);
      Bs[kr][c] = (r < r1 && nn < d_out) ? Conv<T>::to_acc(yg[rb * d_out + nn]) : A(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      A a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[kk][ty + 16 * q]; b[q] = Bs[kk][tx + 16 * q]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  T *dwe = dw + (int64_t)e * d_in * d_out;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t mm = m0 + ty + 16 * i;
    if (mm >= d_in) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t nn = n0 + tx + 16 * j;
      if (nn < d_out) dwe[mm * d_out + nn] = Conv<T>::from_acc(acc[i][j]);
    }
  }
}

template <typename T> __global__ void round_copy_kernel(const float *__restrict__ src, int64_t numel, T *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = Num<T>::from_f(src[i]);
}

static inline void s2s_grid(int64_t n, int E, int64_t d_out, dim3 &grid, int64_t &max_mt) {
  max_mt = (n + SB_M - 1) / SB_M + E;
  int64_t gy = max_mt < 65535 ? max_mt : 65535;
  grid = dim3((unsigned)((d_out + SB_N - 1) / SB_N), (unsigned)(gy > 0 ? gy : 1), 1);
}

int simt_scatter2scatter(const void *x, const void *w, int E, int64_t w_rows, int64_t w_cols,
                         const int32_t *order, const int32_t *offsets, int64_t n, int fan_out,
                         int gin, int gout, int trans, int dtype, int epi, int act, void *out,
                         void *out2, const void *aux, cudaStream_t st) {
  int64_t d_out = trans ? w_rows : w_cols;
  if (n == 0 || d_out == 0) return SMOE_OK;
  dim3 grid;
  int64_t max_mt;
  s2s_grid(n, E, d_out, grid, max_mt);
  size_t smem = (E + 1) * sizeof(int32_t);
  SMOE_DTYPE_DISPATCH(dtype, (simt_s2s_kernel<T><<<grid, S_THREADS, smem, st>>>(
                                 (const T *)x, (const T *)w, E, w_rows, w_cols, order, offsets, fan_out, gin, gout,
                                 trans, epi, act, (T *)out, (T *)out2, (const T *)aux, max_mt, nullptr, 1, nullptr)));
  return check_launch("simt_scatter2scatter");
}

int simt_group_xty(const void *xg, const void *yg, const int32_t *offsets, int E, int64_t d_in,
                   int64_t d_out, int dtype, void *dw, cudaStream_t st) {
  if (d_in == 0 || d_out == 0) return SMOE_OK;
  dim3 grid((unsigned)((d_out + SB_N - 1) / SB_N), (unsigned)((d_in + SB_M - 1) / SB_M), (unsigned)E);
  SMOE_DTYPE_DISPATCH(dtype, (simt_xty_kernel<T><<<grid, S_THREADS, 0, st>>>((const T *)xg, (const T *)yg, offsets,
                                                                             d_in, d_out, (T *)dw)));
  return check_launch("simt_group_xty");
}

int simt_group_xty_scattered(const void *x, int fa, int ga, const void *y, int fb, int gb, const int32_t *order,
                             const int32_t *offsets, int E, int64_t d_in, int64_t d_out, int dtype, void *dw,
                             cudaStream_t st) {
  if (d_in == 0 || d_out == 0) return SMOE_OK;
  dim3 grid((unsigned)((d_out + SB_N - 1) / SB_N), (unsigned)((d_in + SB_M - 1) / SB_M), (unsigned)E);
  SMOE_DTYPE_DISPATCH(dtype, (simt_xty_kernel<T><<<grid, S_THREADS, 0, st>>>((const T *)x, (const T *)y, offsets,
                                                                             d_in, d_out, (T *)dw, order, fa, ga, fb,
                                                                             gb)));
  return check_launch("simt_group_xty_scattered");
}

// y = round(y_accum) (bf16), or a no-op when y aliases the fp32 accumulator.
int round_copy(const float *y_accum, int64_t numel, int dtype, void *y, cudaStream_t st) {
  if (numel <= 0 || (const void *)y == (const void *)y_accum) return SMOE_OK;
  int64_t b = (numel + 255) / 256;
  unsigned blocks = (unsigned)(b < 148 * 16 ? b : 148 * 16);
  if (dtype == SMOE_BF16)
    round_copy_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(y_accum, numel, (__nv_bfloat16 *)y);
  else
    round_copy_kernel<float><<<blocks, 256, 0, st>>>(y_accum, numel, (float *)y);
  return check_launch("round_copy");
}

// Inference combine on the SIMT engine: p-scaled slot products accumulated into
// y_accum (fp32; float64 and aliasing y when dtype == SMOE_F64), then rounded
// into y.
int simt_scatter_combine(const void *x, const void *w, int E, int64_t d_in, int64_t d_out,
                         const int32_t *order, const int32_t *offsets, int64_t n, int fan_out,
                         const void *p_flat, int combine_cols, int gin, int dtype,
                         void *y_accum, void *y, cudaStream_t st) {
  int64_t out_rows = n / combine_cols;
  const size_t acc_esz = dtype == SMOE_F64 ? 8 : 4;
  if (out_rows * d_out > 0) cudaMemsetAsync(y_accum, 0, acc_esz * out_rows * d_out, st);
  if (n > 0 && d_out > 0) {
    dim3 grid;
    int64_t max_mt;
    s2s_grid(n, E, d_out, grid, max_mt);
    size_t smem = (E + 1) * sizeof(int32_t);
    SMOE_DTYPE_DISPATCH(dtype, {
      using W = typename WOf<T>::type;
      simt_s2s_kernel<T><<<grid, S_THREADS, smem, st>>>((const T *)x, (const T *)w, E, d_in, d_out, order, offsets,
                                                        fan_out, gin, 0, 0, SMOE_EPI_NONE, 0, nullptr, nullptr,
                                                        nullptr, max_mt, (const W *)p_flat, combine_cols,
                                                        (W *)y_accum);
    });
  }
  int64_t numel = out_rows * d_out;
  const bool copy = numel > 0 && (void *)y != y_accum && dtype != SMOE_F64;
  if (copy) {
    int64_t b = (numel + 255) / 256;
    unsigned blocks = (unsigned)(b < 148 * 16 ? b : 148 * 16);
    if (dtype == SMOE_BF16)
      round_copy_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((const float *)y_accum, numel, (__nv_bfloat16 *)y);
    else
      round_copy_kernel<float><<<blocks, 256, 0, st>>>((const float *)y_accum, numel, (float *)y);
  }
  return check_launch("simt_scatter_combine", (n > 0 && d_out > 0) + copy);
}

}  // namespace smoe
