// K2/K3/K6/K7: tcgen05 + TMEM + TMA grouped GEMMs for sm_100a (bf16 in, fp32 accumulate).
//
// One warp-specialized persistent kernel template covers every GEMM of the
// ParallelLinear path:
//
//   scatter2scatter (kernels.py:143-220), "grouped-M" schedule:
//     tiles = sum_e ceil(count_e / 128) x ceil(d_out / 256); K = d_in
//     A rows: grouped (TMA 2D tile) or gathered straight from the scattered
//             input by 4 cp.async warps (row = order[i] / fan_out), written in
//             the 128-B swizzle pattern — no padded or grouped copy of X is
//             ever made (TMA tile::gather4 measured 3x slower: 32 issues/stage);
//     B     : W[e] as a 3D tensor map, MN-major (forward) or K-major (W^T for
//             the input gradients, never materialised transposed);
//     epilogue: TMEM -> registers -> (pre, act(pre)) | act | acc*act'(aux) ->
//             bf16 rows stored at i (grouped) or order[i] (scattered).
//   group_xty (kernels.py:329-361), "grouped-K" schedule:
//     tiles = E x ceil(d_in / 128) x ceil(d_out / 256); K = the expert's bin,
//     A = Xg^T and B = Yg both MN-major; bin-tail rows are zeroed in shared
//     memory before the last MMA; empty bins write zeros (no MMA).
//
// This single-CTA engine (128 x 256 tiles) is kept as the SMOE_TC_CTAS=1
// alternative and A/B reference; the default bf16 engine is the CTA-pair
// kernel of tc2_gemm.cu.
// Roles (one CTA per SM, grid = #SMs, static round-robin tiles):
//   warps 0..7   epilogue (warp w reads TMEM lanes 32*(w%4) .. +31, column half w/4)
//   warps 8..11  cp.async gather of A rows (gather mode only)
//   next warp    TMA producer;  last warp  TMEM allocator + tcgen05.mma issuer
// Pipelines: 4-stage smem ring (full/empty mbarriers, 48 KB per stage) and a
// 2-stage TMEM accumulator ring (2 x 256 fp32 columns = all 512 columns), so the
// epilogue of tile t overlaps the MMAs of tile t+1.
#include <cuda.h>

#include <cstdlib>

#include "tc_common.cuh"

namespace smoe {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 32;  // m-blocks per raster band (L2 reuse of B panels)

// ---- the kernel --------------------------------------------------------------------
constexpr int EPI_WARPS = 8;                 // 2 warps per TMEM lane quarter, 128 columns each
constexpr int GATHER_WARPS = 4;              // cp.async gather of A rows (A_GATHER only)
constexpr int EPI_COLS = BN / (EPI_WARPS / 4);
__host__ __device__ constexpr int kernel_threads(int am) { return 64 + 32 * EPI_WARPS + (am == A_GATHER ? 32 * GATHER_WARPS : 0); }


template <int AM, int BMODE, bool GK>
__global__ void __launch_bounds__(kernel_threads(AM), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, Params p) {
  constexpr int THREADS = kernel_threads(AM);
  // Warp roles.  The warp scheduler favours higher warp ids, so the latency-
  // critical producer and MMA warps take the highest ids and never queue behind
  // epilogue math: epilogue 0..7 | gather 8..11 (A_GATHER) | producer | MMA.
  constexpr int WP = EPI_WARPS + (AM == A_GATHER ? GATHER_WARPS : 0);
  constexpr int WM = WP + 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *tiles_smem = smem;
  uint64_t *bars = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *full_bar = bars;                     // [STAGES]
  uint64_t *empty_bar = bars + STAGES;           // [STAGES]
  uint64_t *tfull_bar = bars + 2 * STAGES;       // [2]
  uint64_t *tempty_bar = bars + 2 * STAGES + 2;  // [2]
  uint32_t *s_tmem = (uint32_t *)(bars + 2 * STAGES + 4);
  int64_t *s_start = (int64_t *)(bars + 2 * STAGES + 6);  // [E+1]
  int32_t *s_off = (int32_t *)(s_start + p.E + 1);         // [E+1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nN = (p.N + BN - 1) / BN;
  const int64_t mM = (p.M + BM - 1) / BM;

  // ---- one-time setup ----
  for (int i = threadIdx.x; i <= p.E; i += THREADS) s_off[i] = p.offsets[i];
  if (warp == WP && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), AM == A_GATHER ? 1 + 32 * GATHER_WARPS : 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull_bar[s]), 1);
      mbar_init(smem_u32(&tempty_bar[s]), EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == WM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int e = 0; e < p.E; ++e) {
      s_start[e] = acc;
      if (!GK) {
        int64_t cnt = s_off[e + 1] - s_off[e];
        acc += ((cnt + BM - 1) / BM) * nN;
      } else {
        acc += mM * nN;
      }
    }
    s_start[p.E] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  const int64_t total = s_start[p.E];

  if (warp == WP) {
    // ===================== TMA producer (B, and A unless gathered) =====================
    // The whole warp runs the schedule (converged: uniform operands); one
    // elected lane issues.
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile tl = decode_tile<GK, BM, BN>(t, p, s_start, s_off, nN, mM);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          const uint32_t fb = smem_u32(&full_bar[stage]);
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t sa = smem_u32(tiles_smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
          const int kk = kb * BK;
          if (elect_one_sync()) {
            mbar_expect_tx(fb, AM == A_GATHER ? B_BYTES : STAGE_BYTES);
            if (BMODE == B_W_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_3d(&tma_b, fb, sb + j * 8192, (int)tl.n0 + 64 * j, kk, tl.e);
            } else if (BMODE == B_W_K) {
              tma_load_3d(&tma_b, fb, sb, kk, (int)tl.n0, tl.e);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_2d(&tma_b, fb, sb + j * 8192, (int)tl.n0 + 64 * j, (int)(tl.k0 + kk));
            }
            if (AM == A_ROWS) {
              tma_load_2d(&tma_a, fb, sa, kk, (int)tl.m0);
            } else if (AM == A_MN) {
              tma_load_2d(&tma_a, fb, sa, (int)tl.m0, (int)(tl.k0 + kk));
              tma_load_2d(&tma_a, fb, sa + 8192, (int)tl.m0 + 64, (int)(tl.k0 + kk));
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == WM) {
    // ===================== MMA issuer =====================
    constexpr uint32_t a_mn = (AM == A_MN) ? 1u : 0u;
    constexpr uint32_t b_mn = (BMODE == B_W_K) ? 0u : 1u;
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) |
                               ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const Tile tl = decode_tile<GK, BM, BN>(t, p, s_start, s_off, nN, mM);
      if (tl.nkb == 0) continue;
      mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
      for (int kb = 0; kb < tl.nkb; ++kb) {
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        tc_fence_after();
        uint8_t *sa_ptr = tiles_smem + stage * STAGE_BYTES;
        if (GK && kb == tl.nkb - 1) {
          const int valid = (int)(tl.k_len - (int64_t)kb * BK);
          if (valid < BK) {
            // zero K rows >= valid in all 6 boxes (2 of A, 4 of B); 128 B per row
            const int rows = BK - valid;
            const int chunks = rows * 6 * 8;
            for (int c = lane; c < chunks; c += 32) {
              const int box = c / (rows * 8);
              const int rem = c - box * rows * 8;
              const int r = valid + rem / 8;
              const int q = rem % 8;
              *reinterpret_cast<uint4 *>(sa_ptr + box * 8192 + r * 128 + q * 16) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncwarp();
          }
        }
        if (AM == A_GATHER) fence_proxy_async_smem();
        const uint32_t sa = smem_u32(sa_ptr);
        const uint32_t sb = sa + A_BYTES;
        if (elect_one_sync()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad, bd;
            if (AM == A_MN) ad = sdesc(sa + k * 2048, 8192, 1024);
            else ad = sdesc(sa + k * 32, 16, 1024);
            if (BMODE == B_W_K) bd = sdesc(sb + k * 32, 16, 1024);
            else bd = sdesc(sb + k * 2048, 8192, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(smem_u32(&empty_bar[stage]));
          if (kb == tl.nkb - 1) umma_commit(smem_u32(&tfull_bar[acc]));
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp < EPI_WARPS) {
    // ===================== epilogue =====================
    const int ew = warp;
    const int q = warp & 3;               // TMEM lane quarter this warp may access
    const int c_begin = (ew / 4) * EPI_COLS;
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const Tile tl = decode_tile<GK, BM, BN>(t, p, s_start, s_off, nN, mM);
      const int64_t row = tl.m0 + r;
      const bool valid = row < tl.m_end;
      __nv_bfloat16 *orow = nullptr, *orow2 = nullptr;
      const __nv_bfloat16 *arow = nullptr;
      if (valid) {
        int64_t dst;
        if (GK) dst = (int64_t)tl.e * p.M + row;
        else dst = p.grouped_out ? row : (int64_t)p.order[row];
        orow = p.out + dst * p.N;
        if (p.out2) orow2 = p.out2 + dst * p.N;
        if (p.aux) arow = p.aux + dst * p.N;
      }
      const bool has_acc = tl.nkb > 0;
      // prefetch the first aux chunk (act-grad epilogue) before waiting on the MMA
      uint4 av[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      const bool use_aux = (p.epi == SMOE_EPI_ACT_GRAD) && valid;
      if (use_aux) {
        const int64_t c0 = tl.n0 + c_begin;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (c0 + 8 * j < p.N) av[j] = __ldg(reinterpret_cast<const uint4 *>(arow + c0 + 8 * j));
      }
      if (has_acc) {
        mbar_wait(smem_u32(&tfull_bar[acc]), acc_phase);
        tc_fence_after();
      }
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c_begin);
#pragma unroll 1
      for (int c = 0; c < EPI_COLS; c += 16) {
        uint32_t v[16];
        if (has_acc) {
          tmem_ld16(tbase + c, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0u;
        }
        const int64_t col0 = tl.n0 + c_begin + c;
        uint4 avn[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
        if (use_aux && c + 16 < EPI_COLS) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (col0 + 16 + 8 * j < p.N) avn[j] = __ldg(reinterpret_cast<const uint4 *>(arow + col0 + 16 + 8 * j));
        }
        if (has_acc) tmem_ld_wait();
        if (valid && col0 < p.N) epilogue_chunk(p, v, av, orow, orow2, col0);
        av[0] = avn[0];
        av[1] = avn[1];
      }
      if (has_acc) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[acc]));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (AM == A_GATHER) {
    // ===================== cp.async gather of A rows =====================
    // Each k-block moves 128 rows x 128 B.  Thread g copies 16-B chunk (g % 8)
    // of rows j*16 + g/8 (j = 0..7), so one warp instruction covers 4 whole
    // 128-B row slices (4 L1 wavefronts, not 32).  Chunks are written with the
    // SWIZZLE_128B pattern the UMMA descriptor expects: chunk c of tile row r
    // lands at chunk c ^ (r % 8).  Arrival is signalled when the copies land.
    const int g = threadIdx.x - 32 * EPI_WARPS;
    const int chunk = g & 7;
    const int rsub = g >> 3;  // 0..15
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const Tile tl = decode_tile<GK, BM, BN>(t, p, s_start, s_off, nN, mM);
      const __nv_bfloat16 *src[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t row = min(tl.m0 + j * 16 + rsub, tl.m_end - 1);
        src[j] = p.x + (int64_t)(p.order[row] / p.fan_out) * p.K + chunk * 8;
      }
      for (int kb = 0; kb < tl.nkb; ++kb) {
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        const uint32_t sa = smem_u32(tiles_smem + stage * STAGE_BYTES);
        const int64_t col = (int64_t)kb * BK;
        const bool ok = col + chunk * 8 < p.K;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = j * 16 + rsub;
          cp_async16(sa + r * 128 + ((chunk ^ (r & 7)) << 4), ok ? (const void *)(src[j] + col) : (const void *)src[j],
                     ok ? 16u : 0u);
        }
        cp_async_arrive_noinc(smem_u32(&full_bar[stage]));
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  }

  __syncthreads();
  if (warp == WM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ---- host side ----------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)ptr;
  }
  return fn;
}

// dims/strides innermost first; strides (bytes) for dims 1.. ; box in elements.
bool encode_map(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims, const uint64_t *strides,
                   const uint32_t *box) {
  EncodeTiledFn fn = get_encode();
  if (!fn) return false;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void *>(ptr),
                  (const cuuint64_t *)dims, (const cuuint64_t *)strides, (const cuuint32_t *)box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int group_m_setting() {
  static int gm = -1;
  if (gm < 0) {
    const char *env = getenv("SMOE_GROUP_M");
    gm = env ? atoi(env) : GROUP_M;
    if (gm < 1) gm = GROUP_M;
  }
  return gm;
}

static size_t smem_bytes(int E) { return 1024 + STAGES * STAGE_BYTES + 8 * (2 * STAGES + 6) + 12 * (E + 1) + 64; }

template <int AM, int BMODE, bool GK>
static int launch(const CUtensorMap &ta, const CUtensorMap &tb, const Params &p, int64_t max_tiles, cudaStream_t st) {
  auto kern = tc_gemm_kernel<AM, BMODE, GK>;
  size_t smem = smem_bytes(p.E);
  static size_t configured = 0;
  if (configured < smem) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("tc_gemm: smem attribute");
    configured = smem;
  }
  int grid = num_sms();
  if (max_tiles < grid) grid = (int)(max_tiles > 0 ? max_tiles : 1);
  kern<<<grid, kernel_threads(AM), smem, st>>>(ta, tb, p);
  return check_launch("tc_gemm");
}

}  // namespace tc

bool tc_available() {
  static int avail = -1;
  if (avail < 0) {
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    avail = (major == 10 && minor == 0 && tc::get_encode() != nullptr) ? 1 : 0;
  }
  return avail == 1;
}

static inline bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }

namespace tc2 {
int scatter2scatter(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *,
                    int64_t, int, int, int, int, int, int, void *, void *, const void *, cudaStream_t);
int group_xty(const void *, const void *, const int32_t *, int, int64_t, int64_t, int64_t, void *, cudaStream_t,
              const unsigned long long *arrive = nullptr);
int scatter_combine(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *,
                    int64_t, int, int, const float *, int, float *, cudaStream_t);
int group_xty_scattered(const void *, int64_t, int, int, const void *, int64_t, int, int, const int32_t *,
                        const int32_t *, int, int64_t, int64_t, int64_t, void *, cudaStream_t);
int scatter2scatter_peer(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                         const int32_t *, int64_t, int, const uint64_t *, const int32_t *, const int32_t *,
                         cudaStream_t);
int scatter2scatter_scaled(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                           const int32_t *, int64_t, int, int, int, int, int, int, const float *, void *, void *,
                           const void *, float *, int, cudaStream_t);
int scatter2scatter_scaled_gated(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                                 const int32_t *, int64_t, int, int, int, const float *, void *, void *, const void *,
                                 float *, int, const unsigned long long *, cudaStream_t);
int scatter2scatter_heads(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *,
                          int64_t, int, int, int, int, int, const float *, const void *, float *, int, int64_t, int, int,
                          void *, cudaStream_t);
}  // namespace tc2
bool tc2_supports_experts(int E);  // the CTA-pair kernel's smem holds a per-expert tile table

// 2 = CTA-pair kernels (tc2_gemm.cu, default), 1 = single-CTA kernels (this file).
static int tc_ctas() {
  static int v = -1;
  if (v < 0) {
    const char *env = getenv("SMOE_TC_CTAS");
    v = (env && atoi(env) == 1) ? 1 : 2;
  }
  return v;
}

bool tc_supports_s2s(int64_t d_in, int64_t d_out, const void *x, const void *w, const void *out) {
  return d_in % 8 == 0 && d_out % 8 == 0 && d_in > 0 && d_out > 0 && al16(x) && al16(w) && al16(out) &&
         d_in < (1ll << 31) && d_out < (1ll << 31);
}

int tc_scatter2scatter(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                       const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int gout,
                       int trans, int epi, int act, void *out, void *out2, const void *aux, cudaStream_t st) {
  using namespace tc;
  const int64_t d_in = trans ? w_cols : w_rows;
  const int64_t d_out = trans ? w_rows : w_cols;
  if (!tc_supports_s2s(d_in, d_out, x, w, out))
    return fail(SMOE_ENOTSUP, "tcgen05 scatter2scatter needs d_in, d_out multiples of 8 and 16-byte aligned buffers");
  if (E > 1024) return fail(SMOE_ENOTSUP, "tcgen05 path supports up to 1024 experts");
  if (tc_ctas() == 2 && tc2_supports_experts(E))
    return tc2::scatter2scatter(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, gout, trans, epi,
                                act, out, out2, aux, st);
  CUtensorMap ta, tb;
  // A: x [x_rows, d_in] row-major
  {
    uint64_t dims[2] = {(uint64_t)d_in, (uint64_t)x_rows};
    uint64_t strides[1] = {(uint64_t)d_in * 2};
    uint32_t box[2] = {64, gin ? (uint32_t)BM : 1u};
    if (!encode_map(&ta, x, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(A) failed");
  }
  // B: W [E][w_rows][w_cols]
  {
    uint64_t dims[3] = {(uint64_t)w_cols, (uint64_t)w_rows, (uint64_t)E};
    uint64_t strides[2] = {(uint64_t)w_cols * 2, (uint64_t)w_cols * w_rows * 2};
    uint32_t box[3];
    if (!trans) { box[0] = 64; box[1] = 64; box[2] = 1; }      // [K][N]: MN-major 64x64 boxes
    else { box[0] = 64; box[1] = (uint32_t)BN; box[2] = 1; }   // [N][K]: K-major 64 x 256 box
    if (!encode_map(&tb, w, 3, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(B) failed");
  }
  Params p{};
  p.E = E;
  p.M = n;
  p.N = d_out;
  p.K = d_in;
  p.order = order;
  p.offsets = offsets;
  p.fan_out = fan_out;
  p.grouped_out = gout;
  p.epi = epi;
  p.act = act;
  p.out = (__nv_bfloat16 *)out;
  p.out2 = (epi == SMOE_EPI_ACT) ? (__nv_bfloat16 *)out2 : nullptr;
  p.aux = (epi == SMOE_EPI_ACT_GRAD) ? (const __nv_bfloat16 *)aux : nullptr;
  p.x = (const __nv_bfloat16 *)x;
  p.group_m = group_m_setting();
  const int64_t max_tiles = ((n + BM - 1) / BM + E) * ((d_out + BN - 1) / BN);
  if (gin) {
    if (!trans) return launch<A_ROWS, B_W_MN, false>(ta, tb, p, max_tiles, st);
    return launch<A_ROWS, B_W_K, false>(ta, tb, p, max_tiles, st);
  }
  if (!trans) return launch<A_GATHER, B_W_MN, false>(ta, tb, p, max_tiles, st);
  return launch<A_GATHER, B_W_K, false>(ta, tb, p, max_tiles, st);
}

// The combine epilogue exists in the CTA-pair kernels only.
bool tc_supports_combine(int E, int64_t d_in, int64_t d_out, const void *x, const void *w, const void *yacc) {
  return tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && tc_supports_s2s(d_in, d_out, x, w, yacc);
}

int tc_scatter_combine(const void *x, int64_t x_rows, const void *w, int E, int64_t d_in, int64_t d_out,
                       const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin,
                       const float *p_flat, int combine_cols, float *yacc, cudaStream_t st) {
  if (!tc_supports_combine(E, d_in, d_out, x, w, yacc))
    return fail(SMOE_ENOTSUP, "tcgen05 scatter_combine needs the CTA-pair engine, d_in, d_out multiples of 8 and "
                              "16-byte aligned buffers");
  return tc2::scatter_combine(x, x_rows, w, E, d_in, d_out, order, offsets, n, fan_out, gin, p_flat, combine_cols,
                              yacc, st);
}

// gathered rows are addressed by 31-bit offsets in 16-byte chunks
static bool xty_offsets_fit(int64_t rows, int64_t cols) { return rows * (cols / 8) < (1ll << 31); }

int tc_scatter2scatter_peer(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                            const int32_t *order, const int32_t *offsets, int64_t n, int trans,
                            const uint64_t *peer_out, const int32_t *row_src, const int32_t *row_slot,
                            cudaStream_t st) {
  const int64_t d_in = trans ? w_cols : w_rows, d_out = trans ? w_rows : w_cols;
  if (!(tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && tc_supports_s2s(d_in, d_out, x, w, x)))
    return fail(SMOE_ENOTSUP, "peer-store GEMM needs the CTA-pair engine, d_in, d_out multiples of 8");
  return tc2::scatter2scatter_peer(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, trans, peer_out, row_src,
                                   row_slot, st);
}

int tc_scatter2scatter_scaled(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                              const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int gout,
                              int trans, int epi, int act, const float *row_scale, void *out, void *out2,
                              const void *aux, float *dp_part, int dp_parts, cudaStream_t st) {
  const int64_t d_in = trans ? w_cols : w_rows, d_out = trans ? w_rows : w_cols;
  if (!(tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && tc_supports_s2s(d_in, d_out, x, w, out)))
    return fail(SMOE_ENOTSUP, "scaled epilogues need the CTA-pair engine, d_in, d_out multiples of 8");
  return tc2::scatter2scatter_scaled(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, gout, trans, epi,
                                     act, row_scale, out, out2, aux, dp_part, dp_parts, st);
}

int tc_scatter2scatter_heads(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                             const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int trans,
                             int epi, int act, const float *row_scale, const void *aux, float *dp_part, int dp_parts,
                             int64_t seq_len, int k_slots, int d_head, void *heads, cudaStream_t st) {
  const int64_t d_in = trans ? w_cols : w_rows, d_out = trans ? w_rows : w_cols;
  if (!(tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && tc_supports_s2s(d_in, d_out, x, w, heads)))
    return fail(SMOE_ENOTSUP, "head-layout output needs the CTA-pair engine, d_in, d_out multiples of 8");
  if (d_head % 64 || d_out % d_head)
    return fail(SMOE_ENOTSUP, "head-layout output needs d_head a multiple of 64 dividing d_out");
  return tc2::scatter2scatter_heads(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, trans, epi, act,
                                    row_scale, aux, dp_part, dp_parts, seq_len, k_slots, d_head, heads, st);
}

// group_xty with scattered (gathered) operands: CTA-pair kernels only.
bool tc_supports_xty_scattered(int E, int64_t x_rows, int64_t d_in, int64_t y_rows, int64_t d_out, const void *x,
                               const void *y, const void *dw) {
  return tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && d_in % 8 == 0 && d_out % 8 == 0 && al16(x) &&
         al16(y) && al16(dw) && xty_offsets_fit(x_rows, d_in) && xty_offsets_fit(y_rows, d_out);
}

int tc_group_xty_scattered(const void *x, int64_t x_rows, int fa, int ga, const void *y, int64_t y_rows, int fb,
                           int gb, const int32_t *order, const int32_t *offsets, int E, int64_t n, int64_t d_in,
                           int64_t d_out, void *dw, cudaStream_t st) {
  if (!tc_supports_xty_scattered(E, x_rows, d_in, y_rows, d_out, x, y, dw))
    return fail(SMOE_ENOTSUP, "tcgen05 group_xty over scattered operands needs the CTA-pair engine, d_in, d_out "
                              "multiples of 8 and 16-byte aligned buffers");
  return tc2::group_xty_scattered(x, x_rows, fa, ga, y, y_rows, fb, gb, order, offsets, E, n, d_in, d_out, dw, st);
}

// Expert parallelism: GEMMs on rows stored by peers, each tile gated on its
// expert's arrival counter (CTA-pair engine only).
int tc_ep_scaled_gated(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                       const int32_t *order, const int32_t *offsets, int64_t n, int trans, int epi, int act,
                       const float *row_scale, void *out, void *out2, const void *aux, float *dp_part, int dp_parts,
                       const unsigned long long *arrive, cudaStream_t st) {
  const int64_t d_in = trans ? w_cols : w_rows, d_out = trans ? w_rows : w_cols;
  if (!(tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && tc_supports_s2s(d_in, d_out, x, w, out)))
    return fail(SMOE_ENOTSUP, "gated expert GEMM needs the CTA-pair engine, d_in, d_out multiples of 8");
  return tc2::scatter2scatter_scaled_gated(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, trans, epi, act,
                                           row_scale, out, out2, aux, dp_part, dp_parts, arrive, st);
}

int tc_ep_group_xty_gated(const void *xg, const void *yg, const int32_t *offsets, int E, int64_t n, int64_t d_in,
                          int64_t d_out, void *dw, const unsigned long long *arrive, cudaStream_t st) {
  if (!(tc_ctas() == 2 && E <= 1024 && tc2_supports_experts(E) && d_in % 8 == 0 && d_out % 8 == 0 && al16(xg) &&
        al16(yg) && al16(dw)))
    return fail(SMOE_ENOTSUP, "gated group_xty needs the CTA-pair engine, d_in, d_out multiples of 8");
  return tc2::group_xty(xg, yg, offsets, E, n, d_in, d_out, dw, st, arrive);
}

int tc_group_xty(const void *xg, const void *yg, const int32_t *offsets, int E, int64_t n, int64_t d_in,
                 int64_t d_out, void *dw, cudaStream_t st) {
  using namespace tc;
  if (!(d_in % 8 == 0 && d_out % 8 == 0 && al16(xg) && al16(yg) && al16(dw)))
    return fail(SMOE_ENOTSUP, "tcgen05 group_xty needs d_in, d_out multiples of 8 and 16-byte aligned buffers");
  if (E > 1024) return fail(SMOE_ENOTSUP, "tcgen05 path supports up to 1024 experts");
  if (tc_ctas() == 2 && tc2_supports_experts(E)) return tc2::group_xty(xg, yg, offsets, E, n, d_in, d_out, dw, st);
  CUtensorMap ta, tb;
  uint64_t rows = (uint64_t)(n > 0 ? n : 1);
  {
    uint64_t dims[2] = {(uint64_t)d_in, rows};
    uint64_t strides[1] = {(uint64_t)d_in * 2};
    uint32_t box[2] = {64, 64};
    if (!encode_map(&ta, xg, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(Xg) failed");
  }
  {
    uint64_t dims[2] = {(uint64_t)d_out, rows};
    uint64_t strides[1] = {(uint64_t)d_out * 2};
    uint32_t box[2] = {64, 64};
    if (!encode_map(&tb, yg, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(Yg) failed");
  }
  Params p{};
  p.E = E;
  p.M = d_in;
  p.N = d_out;
  p.K = 0;
  p.order = nullptr;
  p.offsets = offsets;
  p.fan_out = 1;
  p.grouped_out = 1;
  p.epi = SMOE_EPI_NONE;
  p.act = 0;
  p.out = (__nv_bfloat16 *)dw;
  p.group_m = group_m_setting();
  const int64_t max_tiles = (int64_t)E * ((d_in + BM - 1) / BM) * ((d_out + BN - 1) / BN);
  return launch<A_MN, B_ROWS_MN, true>(ta, tb, p, max_tiles, st);
}

}  // namespace smoe
