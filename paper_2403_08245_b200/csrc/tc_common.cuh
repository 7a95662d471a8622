// Shared PTX wrappers, parameters and tile schedule of the tcgen05 GEMM engines
// (tc_gemm.cu: 1-CTA tiles; tc2_gemm.cu: 2-CTA cta_group::2 tiles).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace smoe {
namespace tc {

// A_MN_G / B_ROWS_MN_G: grouped-K operands gathered row by row from a scattered
// tensor (slot i of the bin reads row order[i] / fan_out) by the cp.async warps.
enum AMode { A_ROWS = 0, A_GATHER = 1, A_MN = 2, A_MN_G = 3 };
enum BMode { B_W_MN = 0, B_W_K = 1, B_ROWS_MN = 2, B_ROWS_MN_G = 3 };
// Internal epilogue (smoe_scatter_combine, not a public SMOE_EPI_* value): each
// accumulator row is scaled by its slot's combine weight and added into the
// fp32 token row yacc[order[i] / combine_cols] (vector reductions in L2).
constexpr int EPI_COMBINE = 16;

struct Params {
  int E;
  int64_t M;  // grouped-M: slots n;  grouped-K: d_in
  int64_t N;  // d_out
  int64_t K;  // grouped-M: d_in;     grouped-K: unused (bins)
  const int32_t *order;
  const int32_t *offsets;
  int fan_out;
  int grouped_out;
  int epi;
  int act;
  __nv_bfloat16 *out;
  __nv_bfloat16 *out2;
  const __nv_bfloat16 *aux;
  const __nv_bfloat16 *x;  // A_GATHER: the scattered input rows [x_rows, K]
  int group_m;             // m-blocks per raster band
  int timing;              // debug: print issue-loop wait counters (SMOE_TC_TIMING)
  uint32_t *tile_ctr;      // CTA-pair kernels: zeroed global counter tiles are claimed from (in order)
  const float *pw;         // EPI_COMBINE: combine weight per scattered slot
  float *yacc;             // EPI_COMBINE: fp32 [n / combine_cols, N] accumulator
  int combine_cols;        // EPI_COMBINE: slots per output row
  const __nv_bfloat16 *y;  // B_ROWS_MN_G: the scattered B rows [y_rows, N]
  int fan_out_b;           // B_ROWS_MN_G: slots per B row
  // Peer-store epilogue (expert-parallel return): output row i goes to row
  // row_slot[i] of the buffer at peer_out[row_src[i]] (another rank's memory).
  const uint64_t *peer_out;
  const int32_t *row_src;
  const int32_t *row_slot;
  float *dp_part;          // EPI_ACT_GRAD_SCALED: [M, dp_parts] partial dot products
  int dp_parts;
  int wide_defer;          // tc2 wide tiles: stages per first / last MMA group
  uint64_t pol_a, pol_b;   // tc2 TMA loads: L2 eviction-priority policy per operand
  // Expert-parallel arrival gate (grouped inputs written by peers): before
  // loading a tile of local expert e the producer waits until arrive[e] (a
  // peer-incremented row counter) reaches the expert's bin length.
  const unsigned long long *arrive;
  // K-lockstep of the cluster pairs (see tc2_gemm.cu, "wave lockstep"): each
  // leader publishes the ring chunks it has issued in prog[cluster] and issues
  // chunk v only while v <= min over clusters + sync_slack.  0 = off.
  uint32_t *prog;
  int sync_chunk;   // k-blocks per chunk
  int sync_slack;   // chunks
  int nclusters;
  // Serpentine K order (tc2, SMOE_TC_SERP): tiles of odd waves (tile index
  // within its expert / 74) stream their k-blocks last-to-first, so a wave
  // starts on the K range the previous wave read last.  0 = off.
  int serp;
  // Head-layout output (staged epilogue, grouped-M, hd_dh > 0): out is the
  // attention core's [batch][h * hd_k][hd_seq][hd_dh] tensor and output row i
  // (slot s = order[i]: token s / hd_k, choice s % hd_k) is scattered into
  // its h heads; an act-grad operand (aux) is then read by grouped row.
  int64_t hd_seq;
  int hd_k;
  int hd_dh;
};

__device__ __forceinline__ uint32_t ld_relaxed_gpu_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Wait (one elected lane of the producer warp) until peers delivered every row
// of expert e, then order those generic-proxy stores before this thread's
// async-proxy (TMA) reads of them.
__device__ __forceinline__ void arrival_gate(const unsigned long long *arrive, int e, int64_t need) {
  while ((int64_t)ld_acquire_sys_u64(arrive + e) < need) __nanosleep(128);
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ bool epi_scaled(int epi) {
  return epi == SMOE_EPI_ACT_SCALED || epi == SMOE_EPI_ACT_GRAD_SCALED;
}
__device__ __forceinline__ bool epi_act_grad(int epi) {
  return epi == SMOE_EPI_ACT_GRAD || epi == SMOE_EPI_ACT_GRAD_SCALED;
}

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// mbarrier waits use try_wait (a potentially blocking wait: the warp is parked
// until the phase completes, a barrier event in the CTA wakes it, or the
// suspend-time hint expires) rather than a test_wait busy loop.  Measured
// (round 2, scripts/_bin variants): the explicit hint changes nothing against
// try_wait's default limit — C1 256x256 GEMM 417.7 vs 418.6 M executed warp
// instructions, dW 261.7 vs 260.5 M, step within noise — and the wait loops
// are ~12 % of the 256x256 kernel's instructions (ncu source counters: TMA
// producer ~25 %, MMA issue loop ~29 %, epilogue ~34 %).  SMOE_WAIT_HINT=0
// builds the hint-free form (A/B).
#ifndef SMOE_WAIT_HINT
#define SMOE_WAIT_HINT 0x989680
#endif
#if SMOE_WAIT_HINT
#define SMOE_TRY_WAIT(scope) "mbarrier.try_wait.parity" scope ".shared::cta.b64 P1, [%0], %1, %2;\n"
#else
#define SMOE_TRY_WAIT(scope) "mbarrier.try_wait.parity" scope ".shared::cta.b64 P1, [%0], %1;\n"
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      SMOE_TRY_WAIT("")
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity), "n"(SMOE_WAIT_HINT)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap *map, uint32_t bar, uint32_t dst, int col, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(dst),
      "l"((uint64_t)map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}

// SMOE_GATHER_L2_HINT (build-time A/B): L2 prefetch size of the gather copies
#ifndef SMOE_GATHER_L2_HINT
#define SMOE_GATHER_L2_HINT 256
#endif
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
#if SMOE_GATHER_L2_HINT == 256
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
#elif SMOE_GATHER_L2_HINT == 128
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// One lane of the (converged) warp; lets uniform values stay in uniform registers
// around single-thread tcgen05 issue (no per-lane waterfall of R2UR moves).
__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---- cluster helpers (2-CTA pairs) ---------------------------------------------
// wait with cluster-scope acquire (data written by the peer CTA before its
// release-arrive on this barrier is visible afterwards)
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      SMOE_TRY_WAIT(".acquire.cluster")
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity), "n"(SMOE_WAIT_HINT)
      : "memory");
}
// release-arrive (cluster scope) on the barrier at this offset in CTA `cta`
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t local_bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(local_bar),
      "r"(cta)
      : "memory");
}
// relaxed arrive (cluster scope) on the barrier at this offset in CTA `cta`: no
// ordering of this thread's earlier memory operations (a release arrive costs
// MEMBAR.GPU + ERRBAR, i.e. waits for every outstanding global store)
__device__ __forceinline__ void mbar_arrive_relaxed_cluster(uint32_t local_bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(local_bar),
      "r"(cta)
      : "memory");
}
// 32-bit store into the same shared offset of CTA `cta`
__device__ __forceinline__ void st_cluster_u32(uint32_t local_addr, uint32_t cta, uint32_t v) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "st.shared::cluster.u32 [ra], %2;\n\t}" ::"r"(local_addr),
      "r"(cta), "r"(v)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t local_bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(local_bar),
      "r"(cta)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      SMOE_TRY_WAIT("")
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity), "n"(SMOE_WAIT_HINT)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// commit prior cta_group::2 MMAs to the barrier at this offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_cg2_mc(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(mask)
               : "memory");
}

// ---- tile schedule --------------------------------------------------------------
struct Tile {
  int e;
  int64_t m0;     // first row of the tile (grouped-M: grouped position; grouped-K: d_in row)
  int64_t m_end;  // rows >= m_end are masked
  int64_t n0;
  int64_t k0;     // grouped-K: first bin row
  int64_t k_len;  // reduction length
  int nkb;        // number of BK blocks
  bool rev;       // k-blocks streamed last-to-first (Params::serp)
};

// Position (k-block index) of the tile's kb-th streamed k-block.
__device__ __forceinline__ int kpos(const Tile &tl, int kb) { return tl.rev ? tl.nkb - 1 - kb : kb; }

// Tile t -> (expert, m-block, n-block) with band rasterisation: group_m m-blocks
// share each B panel while it is hot in L2.  s_start[e] = first tile of expert e.
template <bool GK, int TM, int TN>
__device__ __forceinline__ Tile decode_tile(int64_t t, const Params &p, const int64_t *s_start, const int32_t *s_off,
                                            int64_t nN, int64_t mM) {
  Tile tl;
  int64_t e, local, mt;
  if (!GK) {
    int lo = 0, hi = p.E;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (s_start[mid] <= t) lo = mid; else hi = mid;
    }
    e = lo;
    local = t - s_start[e];
    mt = (s_off[e + 1] - s_off[e] + TM - 1) / TM;
  } else {
    e = t / (mM * nN);
    local = t - e * (mM * nN);
    mt = mM;
  }
  const int64_t band = local / (p.group_m * nN);
  const int64_t rem = local - band * (p.group_m * nN);
  const int64_t rows = min((int64_t)p.group_m, mt - band * p.group_m);
  const int64_t mb = band * p.group_m + rem % rows;
  const int64_t nb = rem / rows;
  tl.e = (int)e;
  tl.n0 = nb * TN;
  if (!GK) {
    tl.m0 = s_off[e] + mb * TM;
    tl.m_end = s_off[e + 1];
    tl.k0 = 0;
    tl.k_len = p.K;
  } else {
    tl.m0 = mb * TM;
    tl.m_end = p.M;
    tl.k0 = s_off[e];
    tl.k_len = s_off[e + 1] - s_off[e];
  }
  tl.nkb = (int)((tl.k_len + 63) / 64);
  // waves of 74 tiles (one per CTA pair) counted from the expert's first tile:
  // a function of the tile's place in its expert only, so the expert-parallel
  // kernels (a rank's experts, renumbered) reverse exactly the same tiles
  // (serp 2, A/B: by global tile id / grid pairs instead)
  tl.rev = p.serp == 1 ? ((local / 74) & 1) : p.serp == 2 ? ((t / p.nclusters) & 1) : false;
  return tl;
}

// Zero K rows [r0, r1) of `boxes` consecutive 64-row x 128-B boxes (MN-major
// tiles); 128-B rows are swizzle-invariant as a whole.  Called by one warp.
__device__ __forceinline__ void zero_k_rows(uint8_t *base, int boxes, int r0, int r1, int lane) {
  const int rows = r1 - r0;
  const int chunks = rows * boxes * 8;
  for (int c = lane; c < chunks; c += 32) {
    const int box = c / (rows * 8);
    const int rem = c - box * rows * 8;
    const int r = r0 + rem / 8;
    const int q = rem % 8;
    *reinterpret_cast<uint4 *>(base + box * 8192 + r * 128 + q * 16) = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  __syncwarp();
}
__device__ __forceinline__ void zero_k_tail(uint8_t *base, int boxes, int valid, int lane) {
  zero_k_rows(base, boxes, valid, 64, lane);
}

// SMOE_STORE_EVICT_FIRST (build-time A/B): epilogue output stores carry an
// L2 evict-first policy, so the GEMM's streaming outputs do not push its
// re-read operand panels out of L2.
#ifndef SMOE_STORE_EVICT_FIRST
#define SMOE_STORE_EVICT_FIRST 0
#endif
__device__ __forceinline__ void st_out128(void *p, uint4 v) {
#if SMOE_STORE_EVICT_FIRST
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(0x12F0000000000000ull)
               : "memory");
#else
  *reinterpret_cast<uint4 *>(p) = v;
#endif
}

// Epilogue for one 16-column chunk of one accumulator row (fp32 in v[]);
// scale / dpacc serve the *_SCALED epilogues (see epilogue_pack32).
__device__ __forceinline__ void epilogue_chunk(const Params &p, const uint32_t (&v)[16], const uint4 (&av)[2],
                                               __nv_bfloat16 *orow, __nv_bfloat16 *orow2, int64_t col0,
                                               float scale = 1.0f, float *dpacc = nullptr) {
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
  uint32_t o1[8], o2[8];
  if (p.epi == SMOE_EPI_ACT_GRAD_SCALED) {
    const __nv_bfloat162 *ah = reinterpret_cast<const __nv_bfloat162 *>(av);
    float dsum = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float h0, g0, h1, g1;
      act_both_fast(p.act, __bfloat162float(ah[i].x), h0, g0);
      act_both_fast(p.act, __bfloat162float(ah[i].y), h1, g1);
      dsum = fmaf(f[2 * i], __bfloat162float(__float2bfloat16_rn(h0)), dsum);
      dsum = fmaf(f[2 * i + 1], __bfloat162float(__float2bfloat16_rn(h1)), dsum);
      o1[i] = pack_bf16(scale * f[2 * i] * g0, scale * f[2 * i + 1] * g1);
    }
    *dpacc += dsum;
  } else if (p.epi == SMOE_EPI_ACT || p.epi == SMOE_EPI_ACT_ONLY || p.epi == SMOE_EPI_ACT_SCALED) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 pre = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      o1[i] = *reinterpret_cast<uint32_t *>(&pre);
      float a0 = scale * act_fwd_fast(p.act, __bfloat162float(pre.x));
      float a1 = scale * act_fwd_fast(p.act, __bfloat162float(pre.y));
      o2[i] = pack_bf16(a0, a1);
    }
    if (p.epi == SMOE_EPI_ACT_ONLY) {
#pragma unroll
      for (int i = 0; i < 8; ++i) o1[i] = o2[i];
    }
  } else if (p.epi == SMOE_EPI_ACT_GRAD) {
    const __nv_bfloat162 *ah = reinterpret_cast<const __nv_bfloat162 *>(av);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float g0 = act_grad_fast(p.act, __bfloat162float(ah[i].x));
      float g1 = act_grad_fast(p.act, __bfloat162float(ah[i].y));
      o1[i] = pack_bf16(f[2 * i] * g0, f[2 * i + 1] * g1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) o1[i] = pack_bf16(f[2 * i], f[2 * i + 1]);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (col0 + 8 * j >= p.N) break;
    st_out128(orow + col0 + 8 * j, make_uint4(o1[4 * j], o1[4 * j + 1], o1[4 * j + 2], o1[4 * j + 3]));
    if (p.epi == SMOE_EPI_ACT || p.epi == SMOE_EPI_ACT_SCALED)
      st_out128(orow2 + col0 + 8 * j, make_uint4(o2[4 * j], o2[4 * j + 1], o2[4 * j + 2], o2[4 * j + 3]));
  }
}

// ---- host helpers ----------------------------------------------------------------
bool encode_map(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims, const uint64_t *strides,
                const uint32_t *box);
int group_m_setting();

}  // namespace tc
}  // namespace smoe

namespace smoe {
namespace tc {
// ---- CTA-pair TMA: data lands in this CTA, bytes are counted on the LEADER's
// barrier (same shared offset with the peer bit cleared), as the cta_group::2
// TMA form requires.
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_load_2d_cg2(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar & kPeerBitMask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1,
                                                int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar & kPeerBitMask)
      : "memory");
}
// The same loads with an L2 eviction-priority hint (createpolicy encodings, as
// CUTLASS's TMA::CacheHintSm90): the operand a raster band re-reads across
// tile waves is kept (EVICT_LAST), the one consumed within a wave goes first.
constexpr uint64_t kL2EvictNormal = 0x1000000000000000ull;
constexpr uint64_t kL2EvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kL2EvictLast = 0x14F0000000000000ull;
__device__ __forceinline__ void tma_load_2d_cg2_h(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1,
                                                  uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar & kPeerBitMask), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2_h(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1,
                                                  int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar & kPeerBitMask), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_h(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_h(const CUtensorMap *map, uint32_t bar, uint32_t dst, int c0, int c1,
                                              int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
// Zero K rows [valid, 64) of `boxes` MN-major 64-row boxes in the PEER CTA's
// shared memory (DSMEM stores), then make them visible to the async proxy.
__device__ __forceinline__ void zero_k_tail_peer(uint32_t local_base, uint32_t peer, int boxes, int valid, int lane) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_base), "r"(peer));
  const int rows = 64 - valid;
  const int chunks = rows * boxes * 8;
  for (int c = lane; c < chunks; c += 32) {
    const int box = c / (rows * 8);
    const int rem = c - box * rows * 8;
    const int r = valid + rem / 8;
    const int q = rem % 8;
    const uint32_t a = remote + box * 8192 + r * 128 + q * 16;
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(0u) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
  __syncwarp();
}
// 16-byte DSMEM bulk copy from this CTA to CTA 0 of the cluster; its
// complete_tx is counted on CTA 0's barrier at offset `bar` (async proxy).
__device__ __forceinline__ void bulk_signal_cta0(uint32_t dst_local, uint32_t src_local, uint32_t bar_local) {
  uint32_t dst, bar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(dst) : "r"(dst_local));
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(bar) : "r"(bar_local));
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(dst),
               "r"(src_local), "r"(bar)
               : "memory");
}

// ---- staged epilogue helpers (CTA-pair kernel) -----------------------------------
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// Fire-and-forget fp32 vector reduction into global memory (performed in L2).
__device__ __forceinline__ void red_add_v4(float *addr, uint4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(__uint_as_float(v.x)),
               "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}

// TMA tile store smem -> global (bulk-group completion), SWIZZLE_128B maps.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int c0, int c1) {
#if SMOE_STORE_EVICT_FIRST
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"((uint64_t)map),
               "r"(src), "r"(c0), "r"(c1), "l"(0x12F0000000000000ull)
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)map),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem source of every committed store has been read (buffer reusable)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed store is complete
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 32 fp32 accumulators of one row -> 16 packed bf16x2 words in io.
//   act_pass = false: round(acc) (EPI_NONE / EPI_ACT's pre-activation) or, for
//                     EPI_ACT_ONLY, act(round(acc)); for EPI_ACT_GRAD io holds the
//                     32 bf16 of h_pre on entry and acc * act'(h_pre) on return;
//   act_pass = true : act(round(acc)) (EPI_ACT's second output).
//   EPI_ACT_SCALED's act pass multiplies by the row scale before rounding;
//   EPI_ACT_GRAD_SCALED returns scale * acc * act'(h_pre) and adds
//   sum(acc * round(act(h_pre))) to dpacc.
__device__ __forceinline__ void epilogue_pack32(const Params &p, const uint32_t (&v)[32], uint32_t (&io)[16],
                                                bool act_pass, float scale = 1.0f, float *dpacc = nullptr) {
  const bool apply_act = act_pass || p.epi == SMOE_EPI_ACT_ONLY;
  if (p.epi == SMOE_EPI_ACT_GRAD_SCALED) {
    float dsum = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&io[i]);
      float f0, g0, f1, g1;
      act_both_fast(p.act, __bfloat162float(a.x), f0, g0);
      act_both_fast(p.act, __bfloat162float(a.y), f1, g1);
      const float v0 = __uint_as_float(v[2 * i]), v1 = __uint_as_float(v[2 * i + 1]);
      dsum = fmaf(v0, __bfloat162float(__float2bfloat16_rn(f0)), dsum);
      dsum = fmaf(v1, __bfloat162float(__float2bfloat16_rn(f1)), dsum);
      io[i] = pack_bf16(scale * v0 * g0, scale * v1 * g1);
    }
    *dpacc += dsum;
  } else if (p.epi == SMOE_EPI_ACT_GRAD) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&io[i]);
      io[i] = pack_bf16(__uint_as_float(v[2 * i]) * act_grad_fast(p.act, __bfloat162float(a.x)),
                        __uint_as_float(v[2 * i + 1]) * act_grad_fast(p.act, __bfloat162float(a.y)));
    }
  } else if (apply_act) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const __nv_bfloat162 pre = __floats2bfloat162_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
      io[i] = pack_bf16(scale * act_fwd_fast(p.act, __bfloat162float(pre.x)),
                        scale * act_fwd_fast(p.act, __bfloat162float(pre.y)));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) io[i] = pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
  }
}

// Coalesced copy of a warp's staging tile (32 rows x 128 B, 16-byte chunks
// XOR-swizzled by row) to global: lane (cr, cc) writes chunk cc of rows
// cr + 4 i to row cdst[i] (< 0: masked) of `base` — 4 full 128-byte row
// segments per store instruction instead of 32 scattered 16-byte pieces.
// With base == nullptr, cdst[i] is the row's absolute byte address (peer rows).
__device__ __forceinline__ void store_staged_rows(uint32_t stg, __nv_bfloat16 *base, const long long (&cdst)[8],
                                                  int64_t col0, bool col_ok, int64_t ld, int cr, int cc) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rl = cr + 4 * i;
    const uint4 val = lds128(stg + rl * 128 + ((cc ^ (rl & 7)) << 4));
    if (cdst[i] >= 0 && col_ok) {
      __nv_bfloat16 *rowp = base ? base + cdst[i] * ld : reinterpret_cast<__nv_bfloat16 *>(cdst[i]);
      st_out128(rowp + col0 + cc * 8, val);
    }
  }
  __syncwarp();
}
}  // namespace tc
}  // namespace smoe
