// 2-CTA (cta_group::2) tcgen05 grouped GEMM: the default bf16 engine.
//
// Same GEMM family as tc_gemm.cu (scatter2scatter grouped-M, group_xty
// grouped-K; see that file's header), but each tile is 256 x 256 and is
// computed by a CTA pair on the two SMs of a TPC:
//   * CTA rank r loads A rows [m0 + 128 r, +128) and B columns [n0 + 128 r, +128)
//     into its own shared memory (32 KB per stage, 6 stages);
//   * the leader (rank 0) issues tcgen05.mma.cta_group::2 (M=256, N=256, K=16),
//     which reads both CTAs' operands and accumulates rows 128 r.. into each
//     CTA's own TMEM (2 x 256 columns, double-buffered);
//   * each CTA's epilogue drains its own TMEM rows.
// Halving the B bytes each SM stages and reads per MMA is what lets the tensor
// pipe run at full rate (SURVEY.md §7 "2-CTA 256-row tiles").
// WIDE variant (template flag): 512 x 256 pair tiles — each CTA stages 256 A
// rows as two 128-row halves next to its 128 B columns, and the leader issues
// two M=256 MMAs per K16 step (rows m0.. into TMEM columns [0,256), rows
// m0+256.. into [256,512)), cutting operand bytes per FLOP to 3/4; see
// wide_stages() for why, and the grouped issue order in the MMA warp.
//
// Synchronisation (mbarriers; "L" = leader only):
//   lfull[s]  per CTA: its own TMA bytes (+128 cp.async gather arrivals) landed.
//             TMA-only modes count BOTH CTAs' bytes on the leader's lfull
//             (cta_group::2 TMA).  Gather mode: the peer's relay warp waits on
//             its own lfull and forwards a 16-byte DSMEM bulk copy whose
//             complete_tx lands on the leader's lfull.
//             Weight-gradient K tails are zeroed by the leader in both CTAs.
//   empty[s]  per CTA: the leader's MMAs consumed stage s (multicast commit)
//   tfull[a]  per CTA: accumulator a complete (multicast commit); WIDE: a = half
//   tempty[a] L: both CTAs' epilogues drained accumulator a (16 arrivals); WIDE: a = half
#include <atomic>

#include "tc_common.cuh"

namespace smoe {
namespace tc2 {

using namespace smoe::tc;

constexpr int TM = 256, TN = 256, BK = 64;
constexpr int RING = 4;  // tile-id ring entries (dynamic schedule)
// Epilogue styles (template STAGED):
//   direct : each thread stores its own accumulator row (7-stage ring);
//   staged : rows go through a per-warp 4 KB smem tile (6-stage ring) and leave
//            as one TMA tile store (grouped outputs, full 32-row slabs) or as
//            coalesced 128-byte row segments (scattered outputs, bin tails).
// Gather-mode kernels always stage (their cp.async operand traffic shares the
// LSU with the stores); which TMA-fed kernels stage is chosen per launch.
__host__ __device__ constexpr int ring_stages(bool staged) { return staged ? 6 : 7; }
constexpr int HM = TM / 2, HN = TN / 2;  // per-CTA halves
constexpr int A_BYTES = HM * BK * 2;     // 16 KB
constexpr int B_BYTES = HN * BK * 2;     // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
// Wide tiles (TMA-fed kernels with long K): a pair tile is 512 x 256 — each CTA
// stages 256 A rows (two 128-row halves, one per M=256 MMA) and 128 B columns,
// so every B stage feeds two MMAs.  Operand bytes per FLOP drop to 3/4 of the
// 256 x 256 tile; under the B200 power cap the operand fill is ~17 % of a
// GEMM's energy (scripts/energy.py with SMOE_TC_TIMING=5: 1.36 -> 1.64
// TFLOP/J without fills).  The 512 accumulator columns leave no second buffer:
// the epilogue drains the first half while the next tile's first MMAs run.
// 48 KB stages: 4 fit beside the staging tiles.
__host__ __device__ constexpr int wide_stages(bool staged, bool wide) { return wide ? 4 : ring_stages(staged); }
__host__ __device__ constexpr int sig_slots(int stages) { return stages < 5 ? 5 : stages; }
constexpr int TMEM_COLS = 512;
constexpr int EPI_WARPS = 8;
constexpr int GATHER_WARPS = 4;
constexpr int G_RSTEP = GATHER_WARPS * 4;   // rows covered by one pass of all gather threads
// Gather mode: A rows fetched by TMA tile::gather4 from the producer lanes
// instead of cp.async.  Measured at C1 layer 1 (base clock, tensor-pipe active):
// 0 rows 72 %, 32 rows 57 % — each gather4 costs far more TMA issue time than
// the 512 B it moves, so the cp.async warps carry all rows.  Round 2 (ncu, no
// clock lock): 0 rows 5.58 ms / 89.7 % tensor-pipe, 64 rows 9.87 ms / 35.7 %
// (MMA issuer waiting on operands 78 % of the time).  SMOE_TG_ROWS (a multiple
// of 16 below 128) rebuilds the split for A/B.
#ifndef SMOE_TG_ROWS
#define SMOE_TG_ROWS 0
#endif
constexpr int TG_ROWS = SMOE_TG_ROWS;
constexpr int G_RPT = (128 - TG_ROWS) / G_RSTEP;  // rows per cp.async gather thread per k-block
constexpr int EPI_COLS = TN / (EPI_WARPS / 4);
constexpr int STG_BYTES = 32 * 128;        // per-epilogue-warp staging tile: 32 rows x 64 bf16
__host__ __device__ constexpr bool has_gather(int am, int bm) {
  return am == A_GATHER || am == A_MN_G || bm == B_ROWS_MN_G;
}
// Copy warps of the grouped-K gather (rows change every k-block).  8 warps
// measured slower than 4 (C1 dW1 7.3 vs 7.0 ms in-step; profiles/r1_gather_ab.txt).
constexpr int KG_WARPS = 4;
__host__ __device__ constexpr int gather_warps(int am, int bm) {
  return am == A_GATHER ? GATHER_WARPS : (has_gather(am, bm) ? KG_WARPS : 0);
}
__host__ __device__ constexpr int kernel_threads(int am, int bm) {
  return 64 + 32 * EPI_WARPS + 32 * gather_warps(am, bm);
}

// The epilogue warps wait for an accumulator through one of them: warp 0 polls
// the tile-full mbarrier, the others block on a named barrier (no issue slots
// while blocked).  A suspended mbarrier try_wait is woken by every barrier
// event of the CTA (a ring stage or an empty slot every few hundred cycles),
// so eight polling warps re-issued their wait loop ~300 M times per C1 GEMM
// launch (ncu smsp__inst_executed, 256 x 256 tiles: 420 M of which ~100 M are
// work) regardless of the suspend hint.
__device__ __forceinline__ void epi_wait_full(uint32_t bar, uint32_t parity, int epi_warp) {
  if (epi_warp == 0) mbar_wait_cluster(bar, parity);
  asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
}

template <int AM, int BMODE, bool GK, bool STAGED, bool WIDE>
__global__ void __launch_bounds__(kernel_threads(AM, BMODE), 1) __cluster_dims__(2, 1, 1)
    tc2_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                    const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_c2, Params p) {
  constexpr int THREADS = kernel_threads(AM, BMODE);
  constexpr int STAGES = wide_stages(STAGED, WIDE);
  // WIDE: 512-row pair tiles (two M=256 MMAs share each B stage; see wide_stages)
  constexpr int TMT = WIDE ? 2 * TM : TM;           // rows per tile
  constexpr int ABYTES = WIDE ? 2 * A_BYTES : A_BYTES;
  constexpr int SBYTES = ABYTES + B_BYTES;          // bytes per ring stage per CTA
  constexpr int BOXES = SBYTES / 8192;              // 64-row x 128-B boxes per stage
  // Warp roles.  The warp scheduler favours higher warp ids, so the latency-
  // critical producer and MMA warps take the highest ids and never queue behind
  // epilogue math: epilogue 0..7 | gather 8..11 (A_GATHER) | producer | MMA.
  constexpr bool GATHER = has_gather(AM, BMODE);
  // grouped-K with gathered operand(s): the cp.async warps fill them, TMA the rest
  constexpr bool KGATHER = GK && GATHER;
  constexpr bool GA = (AM == A_MN_G), GB = (BMODE == B_ROWS_MN_G);
  static_assert(!WIDE || (!GATHER && STAGED), "wide tiles: TMA-fed operands, staged epilogue");
  constexpr int GW = gather_warps(AM, BMODE);
  constexpr int WP = EPI_WARPS + GW;
  constexpr int WM = WP + 1;
  // cp.async data cannot signal the leader's barrier: gather mode relays it
  constexpr bool RELAY = GATHER;
  // Warps that read every tile id from the ring: both CTAs' epilogue (and
  // gather) warps, the leader's MMA warp, the peer's producer, and the peer's
  // relay / bin-tail fixer warp.
  constexpr int RING_READERS = 2 * (EPI_WARPS + GW) + 2 + ((RELAY || GK) ? 1 : 0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *tiles_smem = smem;
  uint8_t *staging = smem + STAGES * SBYTES;  // [EPI_WARPS][STG_BYTES]
  uint64_t *bars = (uint64_t *)(staging + (STAGED ? EPI_WARPS * STG_BYTES : 0));
  uint64_t *lfull_bar = bars;                    // [STAGES]
  // relay payload (16 B) + landing slot (16 B), 16-byte aligned inside bars[STAGES, 2*STAGES)
  constexpr int SIG = sig_slots(STAGES);        // 8-byte slots holding the relay signal
  uint8_t *signal = (uint8_t *)((((uintptr_t)(bars + STAGES)) + 15) & ~(uintptr_t)15);
  static_assert(SIG * 8 >= 32 + 8, "relay slots need room");
  uint64_t *empty_bar = bars + STAGES + SIG;     // [STAGES]
  uint64_t *tfull_bar = empty_bar + STAGES;      // [2]
  uint64_t *tempty_bar = tfull_bar + 2;          // [2]
  uint64_t *ring_full = tempty_bar + 2;          // [RING] tile id written (both CTAs)
  uint64_t *ring_empty = ring_full + RING;       // [RING] L: every consumer warp has read it
  uint32_t *s_tmem = (uint32_t *)(ring_empty + RING);
  int32_t *s_tile = (int32_t *)(ring_empty + RING + 1);      // [RING] claimed tile ids (-1 = done)
  int64_t *s_start = (int64_t *)(ring_empty + RING + 1 + RING / 2);  // [E+1]
  int32_t *s_off = (int32_t *)(s_start + p.E + 1);         // [E+1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t nN = (p.N + TN - 1) / TN;
  const int64_t mM = (p.M + TMT - 1) / TMT;
  const int64_t cluster_id = blockIdx.x >> 1;

  for (int i = threadIdx.x; i <= p.E; i += THREADS) s_off[i] = p.offsets[i];
  if (warp == WP && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&lfull_bar[s]), GATHER ? 1 + 32 * GW : 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull_bar[s]), 1);
      mbar_init(smem_u32(&tempty_bar[s]), 2 * EPI_WARPS);
    }
    for (int s = 0; s < RING; ++s) {
      mbar_init(smem_u32(&ring_full[s]), 1);
      mbar_init(smem_u32(&ring_empty[s]), RING_READERS);
    }
    fence_barrier_init();
  }
  if (warp == WM) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int e = 0; e < p.E; ++e) {
      s_start[e] = acc;
      if (!GK) acc += ((s_off[e + 1] - s_off[e] + TMT - 1) / TMT) * nN;
      else acc += mM * nN;
    }
    s_start[p.E] = acc;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  const int64_t total = s_start[p.E];

  // ---- dynamic tile schedule -------------------------------------------------
  // The leader's producer claims tile ids in increasing order from a global
  // counter and broadcasts each to both CTAs through a RING-entry shared-memory
  // ring; every role reads the same sequence.  Pairs that run at the same time
  // therefore hold neighbouring tiles (band raster stays intact), where a static
  // round-robin schedule lets pairs drift apart by whole waves and turns the
  // band's L2 reuse into DRAM re-reads.
  auto next_tile = [&](int it) -> int64_t {  // ring reader (whole warp)
    const int slot = it & (RING - 1);
    // the peer's copy of the id arrives by a remote store: cluster-scope acquire
    // (an L1 invalidation); the leader's own readers only need the CTA scope
    if (leader) mbar_wait(smem_u32(&ring_full[slot]), (uint32_t)(it / RING) & 1u);
    else mbar_wait_acq_cluster(smem_u32(&ring_full[slot]), (uint32_t)(it / RING) & 1u);
    const int32_t t = *(volatile int32_t *)&s_tile[slot];
    __syncwarp();
    // The arrive only tells the leader the slot may be rewritten.  It is relaxed
    // (a cluster-scope release would first drain this warp's global stores —
    // the epilogue's previous tile); the branch on t orders it after the load.
    if (elect_one_sync() && t != INT32_MIN) {
      if (leader) mbar_arrive(smem_u32(&ring_empty[slot]));
      else mbar_arrive_relaxed_cluster(smem_u32(&ring_empty[slot]), 0);
    }
    return t;
  };
  auto claim_tile = [&](int it) -> int64_t {  // leader producer (whole warp)
    const int slot = it & (RING - 1);
    mbar_wait(smem_u32(&ring_empty[slot]), ((uint32_t)(it / RING) & 1u) ^ 1u);
    if (elect_one_sync()) {
      const uint32_t c = atomicAdd(p.tile_ctr, 1u);
      const int32_t t = (int64_t)c < total ? (int32_t)c : -1;
      s_tile[slot] = t;
      st_cluster_u32(smem_u32(&s_tile[slot]), 1, (uint32_t)t);
      mbar_arrive(smem_u32(&ring_full[slot]));
      mbar_arrive_release_cluster(smem_u32(&ring_full[slot]), 1);
    }
    __syncwarp();
    return *(volatile int32_t *)&s_tile[slot];
  };

  if (warp == WP) {
    // ===================== TMA producer (own halves of A and B) =====================
    // Gather mode: lanes 0..TG_ROWS/4-1 also fetch the first TG_ROWS A rows with
    // TMA tile::gather4 (4 rows per instruction), offloading the cp.async warps.
    int stage = 0;
    uint32_t phase = 0;
    // the leader claims one tile ahead, so the atomic's latency hides behind a tile's loads
    int64_t t_next = leader ? claim_tile(0) : 0;
    // wave lockstep (leader only): chunks issued so far, and the last seen
    // minimum over all clusters (refreshed only when it no longer admits us)
    const bool lockstep = leader && p.sync_chunk > 0;
    uint32_t v_mine = 0, v_min = 0;
    auto lockstep_gate = [&]() {
      ++v_mine;
      if (lane == 0) st_relaxed_gpu_u32(p.prog + cluster_id, v_mine);
      while (v_mine > v_min + (uint32_t)p.sync_slack) {
        uint32_t m = 0xffffffffu;
        for (int c = lane; c < p.nclusters; c += 32) m = min(m, ld_relaxed_gpu_u32(p.prog + c));
        v_min = __reduce_min_sync(0xffffffffu, m);
        if (v_mine > v_min + (uint32_t)p.sync_slack) __nanosleep(256);
      }
    };
    for (int it = 0;; ++it) {
      int64_t t;
      if (leader) {
        t = t_next;
        if (t >= 0) t_next = claim_tile(it + 1);
      } else {
        t = next_tile(it);
      }
      if (t < 0) {
        // out of tiles: never gate the others again
        if (lockstep && lane == 0) st_relaxed_gpu_u32(p.prog + cluster_id, 0xffffffffu);
        break;
      }
      if (p.timing == 7 && leader && lane == 0 && it < 16) {  // debug: tile start times (wave drift)
        uint64_t gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        printf("tiletrace %d %lld %llu\n", (int)cluster_id, (long long)t, (unsigned long long)gt);
      }
      const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
      const int m_half = (int)(tl.m0 + HM * rank);  // A rows / B columns of this CTA
      const int n_half = (int)(tl.n0 + HN * rank);
      // WIDE: rows m0+256.. (the second MMA's A operand) exist in this tile
      const bool bot = WIDE && tl.m0 + TM < tl.m_end;
      const int a_bytes = bot ? 2 * A_BYTES : A_BYTES;
      int gr[4] = {0, 0, 0, 0};
      const bool g4_lane = (AM == A_GATHER) && lane < TG_ROWS / 4;
      if (g4_lane) {
#pragma unroll
        for (int j = 0; j < 4; ++j) gr[j] = __ldg(p.order + min((int64_t)m_half + 4 * lane + j, tl.m_end - 1)) / p.fan_out;
      }
      // expert parallelism: the tile's input rows were stored by peers — wait
      // until every row of this expert has arrived (grouped inputs only)
      if (p.arrive && tl.nkb > 0) {
        if (elect_one_sync()) arrival_gate(p.arrive, tl.e, (int64_t)s_off[tl.e + 1] - s_off[tl.e]);
        __syncwarp();
      }
      for (int kb = 0; kb < tl.nkb; ++kb) {
        const uint32_t fb = smem_u32(&lfull_bar[stage]);
        const uint32_t sa = smem_u32(tiles_smem + stage * SBYTES);
        const int kk = kpos(tl, kb) * BK;
        // all lanes wait (keeps the warp converged, so coordinates and
        // addresses stay in uniform registers); one elected lane issues
        if (lockstep && kb % p.sync_chunk == 0) lockstep_gate();
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        if (elect_one_sync()) {
          const uint32_t sb = sa + ABYTES;
          if (KGATHER) {
            // this CTA's TMA bytes (non-gathered operand) are counted locally;
            // the leader also expects the peer's 16-byte relay signal
            mbar_expect_tx(fb, (GA ? 0 : A_BYTES) + (GB ? 0 : B_BYTES) + (leader ? 16 : 0));
            if (!GB) {
              tma_load_2d_h(&tma_b, fb, sb, n_half, (int)(tl.k0 + kk), p.pol_b);
              tma_load_2d_h(&tma_b, fb, sb + 8192, n_half + 64, (int)(tl.k0 + kk), p.pol_b);
            }
            if (!GA) {
              tma_load_2d_h(&tma_a, fb, sa, m_half, (int)(tl.k0 + kk), p.pol_a);
              tma_load_2d_h(&tma_a, fb, sa + 8192, m_half + 64, (int)(tl.k0 + kk), p.pol_a);
            }
          } else if (RELAY) {
            // gather mode: this CTA's bytes are counted locally; the leader also
            // expects the peer's 16-byte relay signal on the same barrier
            mbar_expect_tx(fb, B_BYTES + TG_ROWS * 128 + (leader ? 16 : 0));
            if (BMODE == B_W_MN) {
              tma_load_3d_h(&tma_b, fb, sb, n_half, kk, tl.e, p.pol_b);
              tma_load_3d_h(&tma_b, fb, sb + 8192, n_half + 64, kk, tl.e, p.pol_b);
            } else {
              tma_load_3d_h(&tma_b, fb, sb, kk, n_half, tl.e, p.pol_b);
            }
          } else if (GK && AM == A_MN && tl.k_len - kk < BK) {
            // bin-tail stage of a grouped-K tile: each CTA counts its own bytes
            // locally, zeroes its rows past the bin, and the peer then signals
            // the leader (see the tail fixer below)
            mbar_expect_tx(fb, B_BYTES + a_bytes + (leader ? 16 : 0));
            tma_load_2d_h(&tma_b, fb, sb, n_half, (int)(tl.k0 + kk), p.pol_b);
            tma_load_2d_h(&tma_b, fb, sb + 8192, n_half + 64, (int)(tl.k0 + kk), p.pol_b);
            tma_load_2d_h(&tma_a, fb, sa, m_half, (int)(tl.k0 + kk), p.pol_a);
            tma_load_2d_h(&tma_a, fb, sa + 8192, m_half + 64, (int)(tl.k0 + kk), p.pol_a);
            if (bot) {
              tma_load_2d_h(&tma_a, fb, sa + A_BYTES, m_half + TM, (int)(tl.k0 + kk), p.pol_a);
              tma_load_2d_h(&tma_a, fb, sa + A_BYTES + 8192, m_half + TM + 64, (int)(tl.k0 + kk), p.pol_a);
            }
          } else if (p.timing == 5 && it > 0) {
            // energy probe (SMOE_TC_TIMING=5, debug): after the first tile no
            // operand is fetched; the MMAs run on stale shared memory
            if (leader) mbar_arrive(fb);
          } else {
            // both CTAs' bytes are counted on the leader's barrier
            if (leader) mbar_expect_tx(fb, 2 * (B_BYTES + a_bytes));
            if (BMODE == B_W_MN) {
              tma_load_3d_cg2_h(&tma_b, fb, sb, n_half, kk, tl.e, p.pol_b);
              tma_load_3d_cg2_h(&tma_b, fb, sb + 8192, n_half + 64, kk, tl.e, p.pol_b);
            } else if (BMODE == B_W_K) {
              tma_load_3d_cg2_h(&tma_b, fb, sb, kk, n_half, tl.e, p.pol_b);
            } else {
              tma_load_2d_cg2_h(&tma_b, fb, sb, n_half, (int)(tl.k0 + kk), p.pol_b);
              tma_load_2d_cg2_h(&tma_b, fb, sb + 8192, n_half + 64, (int)(tl.k0 + kk), p.pol_b);
            }
            if (AM == A_ROWS) {
              tma_load_2d_cg2_h(&tma_a, fb, sa, (int)(tl.k0 + kk), m_half, p.pol_a);
              if (bot) tma_load_2d_cg2_h(&tma_a, fb, sa + A_BYTES, (int)(tl.k0 + kk), m_half + TM, p.pol_a);
            } else if (AM == A_MN) {
              tma_load_2d_cg2_h(&tma_a, fb, sa, m_half, (int)(tl.k0 + kk), p.pol_a);
              tma_load_2d_cg2_h(&tma_a, fb, sa + 8192, m_half + 64, (int)(tl.k0 + kk), p.pol_a);
              if (bot) {
                tma_load_2d_cg2_h(&tma_a, fb, sa + A_BYTES, m_half + TM, (int)(tl.k0 + kk), p.pol_a);
                tma_load_2d_cg2_h(&tma_a, fb, sa + A_BYTES + 8192, m_half + TM + 64, (int)(tl.k0 + kk), p.pol_a);
              }
            }
          }
        }
        __syncwarp();
        if (g4_lane) tma_gather4(&tma_a, fb, sa + lane * 512, kk, gr[0], gr[1], gr[2], gr[3]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    // Producer tail: wait until every stage's last fill was consumed, so no
    // multicast commit can still be in flight to this CTA when it exits.
    if (lane == 0) {
      for (int i = 0; i < STAGES; ++i) {
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == WM) {
    if (leader) {
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t a_mn = (AM == A_MN || GA) ? 1u : 0u;
      constexpr uint32_t b_mn = (BMODE == B_W_K) ? 0u : 1u;
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) |
                                 ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // p.timing: per-cluster cycle counters of the issue loop (SMOE_TC_TIMING=1, debug)
      long long c_start = clock64(), c_tempty = 0, c_lfull = 0;
      // WIDE issue order.  A tile's stages are issued in groups: MMA#1 (rows
      // m0.., accumulator columns [0, 256)) for every stage of the group, then
      // MMA#2 (rows m0+256.., columns [256, 512)) for the same stages, each
      // stage released after its MMA#2.  The first group (up to `defer`
      // stages) lets MMA#1 run while the epilogue still drains the previous
      // tile's second half; the last group completes the first half `defer`
      // stages early (tfull[0] before tfull[1]), so its drain overlaps the
      // tile's final MMA#2s.  Middle groups are single stages.
      auto wide_group = [&](const Tile &tl, bool bot, int kb0, int kb1, bool first, bool last, int &stage,
                            uint32_t &phase, long long &c_lfull, long long &c_tempty) {
        const int st0 = stage;
        int nk_last = BK / 16;
        for (int kb = kb0; kb < kb1; ++kb) {
          long long c1 = p.timing ? clock64() : 0;
          mbar_wait(smem_u32(&lfull_bar[stage]), phase);
          if (p.timing) c_lfull += clock64() - c1;
          uint8_t *sa_ptr = tiles_smem + stage * SBYTES;
          int nk = BK / 16;
          if (GK && kpos(tl, kb) == tl.nkb - 1) {
            const int valid = (int)(tl.k_len - (int64_t)kpos(tl, kb) * BK);
            if (valid < BK) {
              nk = (valid + 15) / 16;
              if (valid < 16 * nk) zero_k_rows(sa_ptr, BOXES, valid, 16 * nk, lane);
            }
            nk_last = nk;
          }
          tc_fence_after();
          const uint32_t sa = smem_u32(sa_ptr), sb = sa + ABYTES;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              if (GK && k >= nk) break;
              const uint64_t ad = AM == A_MN ? sdesc(sa + k * 2048, 8192, 1024) : sdesc(sa + k * 32, 16, 1024);
              const uint64_t bd = BMODE == B_W_K ? sdesc(sb + k * 32, 16, 1024) : sdesc(sb + k * 2048, 8192, 1024);
              umma_bf16_cg2(tmem_base, ad, bd, idesc, (kb | k) != 0);
            }
            if (!bot) umma_commit_cg2_mc(smem_u32(&empty_bar[stage]), 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (last && elect_one_sync()) {
          umma_commit_cg2_mc(smem_u32(&tfull_bar[0]), 0x3);
          if (!bot) umma_commit_cg2_mc(smem_u32(&tfull_bar[1]), 0x3);
        }
        __syncwarp();
        if (!bot) return;
        if (first) {
          long long c2 = p.timing ? clock64() : 0;
          mbar_wait_cluster(smem_u32(&tempty_bar[1]), acc_phase ^ 1);
          if (p.timing) c_tempty += clock64() - c2;
          tc_fence_after();
        }
        int sg = st0;
        for (int kb = kb0; kb < kb1; ++kb) {
          const int nk = (GK && kpos(tl, kb) == tl.nkb - 1) ? nk_last : BK / 16;
          const uint32_t sa = smem_u32(tiles_smem + sg * SBYTES), sb = sa + ABYTES;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              if (GK && k >= nk) break;
              const uint64_t ad = AM == A_MN ? sdesc(sa + A_BYTES + k * 2048, 8192, 1024)
                                             : sdesc(sa + A_BYTES + k * 32, 16, 1024);
              const uint64_t bd = BMODE == B_W_K ? sdesc(sb + k * 32, 16, 1024) : sdesc(sb + k * 2048, 8192, 1024);
              umma_bf16_cg2(tmem_base + TN, ad, bd, idesc, (kb | k) != 0);
            }
            umma_commit_cg2_mc(smem_u32(&empty_bar[sg]), 0x3);
          }
          __syncwarp();
          if (++sg == STAGES) sg = 0;
        }
        if (last && elect_one_sync()) umma_commit_cg2_mc(smem_u32(&tfull_bar[1]), 0x3);
        __syncwarp();
      };
      const int defer = p.wide_defer < 1 ? 1 : (p.wide_defer > STAGES ? STAGES : p.wide_defer);
      for (int it = 0; WIDE; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        if (tl.nkb == 0) continue;
        const bool bot = tl.m0 + TM < tl.m_end;
        long long c0 = p.timing ? clock64() : 0;
        mbar_wait_cluster(smem_u32(&tempty_bar[0]), acc_phase ^ 1);
        if (p.timing) c_tempty += clock64() - c0;
        tc_fence_after();
        const int n = tl.nkb;
        const int h1 = n < defer ? n : defer;            // first group [0, h1)
        const int t0 = n - defer > h1 ? n - defer : h1;  // last group [t0, n) (empty if t0 == n)
        wide_group(tl, bot, 0, h1, true, h1 == n, stage, phase, c_lfull, c_tempty);
        for (int kb = h1; kb < t0; ++kb) wide_group(tl, bot, kb, kb + 1, false, false, stage, phase, c_lfull, c_tempty);
        if (t0 < n) wide_group(tl, bot, t0, n, false, true, stage, phase, c_lfull, c_tempty);
        acc_phase ^= 1;
      }
      for (int it = 0; !WIDE; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        if (tl.nkb == 0) continue;
        long long c0 = p.timing ? clock64() : 0;
        mbar_wait_cluster(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
        if (p.timing) c_tempty += clock64() - c0;
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * TN);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          long long c1 = p.timing ? clock64() : 0;
          mbar_wait(smem_u32(&lfull_bar[stage]), phase);
          if (p.timing) c_lfull += clock64() - c1;
          uint8_t *sa_ptr = tiles_smem + stage * SBYTES;
          int nk = BK / 16;  // K16 steps issued for this stage
          if (GK && kpos(tl, kb) == tl.nkb - 1) {
            // bin tail: rows past the expert's bin belong to the next expert.
            // K16 steps wholly past the bin are skipped; the rest of the last
            // partial step is zeroed by each CTA in its own tiles.
            const int valid = (int)(tl.k_len - (int64_t)kpos(tl, kb) * BK);
            if (valid < BK) {
              nk = (valid + 15) / 16;
              // TMA-fed operands only (a gathered operand's copies zero-fill past the bin)
              if (!(GA && GB) && valid < 16 * nk)
                zero_k_rows(sa_ptr + ((KGATHER && GA) ? A_BYTES : 0), KGATHER ? 2 : 4, valid, 16 * nk, lane);
            }
          }
          if (RELAY) fence_proxy_async_smem();
          tc_fence_after();
          const uint32_t sa = smem_u32(sa_ptr);
          const uint32_t sb = sa + ABYTES;
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              if (GK && k >= nk) break;
              uint64_t ad, bd;
              if (AM == A_MN || GA) ad = sdesc(sa + k * 2048, 8192, 1024);
              else ad = sdesc(sa + k * 32, 16, 1024);
              if (BMODE == B_W_K) bd = sdesc(sb + k * 32, 16, 1024);
              else bd = sdesc(sb + k * 2048, 8192, 1024);
              umma_bf16_cg2(tmem_d, ad, bd, idesc, (kb | k) != 0);
            }
            umma_commit_cg2_mc(smem_u32(&empty_bar[stage]), 0x3);
            if (kb == tl.nkb - 1) umma_commit_cg2_mc(smem_u32(&tfull_bar[acc]), 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.timing == 1 && lane == 0 && cluster_id < 4)
        printf("tc2 timing cluster %d: total %lld cyc, wait tempty %lld (%.1f%%), wait lfull %lld (%.1f%%)\n",
               (int)cluster_id, clock64() - c_start, c_tempty, 100.0 * c_tempty / (clock64() - c_start), c_lfull,
               100.0 * c_lfull / (clock64() - c_start));
    } else if (GK && !RELAY) {
      // ===================== tail fixer (peer CTA, grouped-K) =====================
      // For each tile's bin-tail stage: wait for this CTA's own bytes, zero the
      // A rows past the bin, then signal the leader's lfull (16-byte DSMEM bulk
      // copy).  Non-tail stages never touch this CTA's lfull, so each stage's
      // parity is tracked separately.
      int stage = 0;
      uint32_t parity_bits = 0;
      for (int it = 0;; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          const int valid = (int)(tl.k_len - (int64_t)kpos(tl, kb) * BK);
          if (valid < BK) {
            mbar_wait(smem_u32(&lfull_bar[stage]), (parity_bits >> stage) & 1u);
            parity_bits ^= 1u << stage;
            const int upto = 16 * ((valid + 15) / 16);  // the leader skips K16 steps past the bin
            if (valid < upto) zero_k_rows(tiles_smem + stage * SBYTES, BOXES, valid, upto, lane);
            else fence_proxy_async_smem();
            if (elect_one_sync()) bulk_signal_cta0(smem_u32(signal + 16), smem_u32(signal), smem_u32(&lfull_bar[stage]));
            __syncwarp();
          }
          if (++stage == STAGES) stage = 0;
        }
      }
    } else if (RELAY) {
      // ===================== relay (peer CTA, gather mode): own stage landed -> leader =====================
      int stage = 0;
      uint32_t phase = 0;
      long long r_start = clock64(), r_wait = 0;  // p.timing == 2: relay busy/wait cycles
      for (int it = 0;; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          long long w0 = p.timing ? clock64() : 0;
          mbar_wait(smem_u32(&lfull_bar[stage]), phase);
          if (p.timing) r_wait += clock64() - w0;
          if (KGATHER && !(GA && GB)) {
            // grouped-K bin tail: the TMA operand's rows past the bin belong to
            // the next expert; zero them up to the K16 step the leader issues
            const int valid = (int)(tl.k_len - (int64_t)kb * BK);
            const int upto = 16 * ((valid + 15) / 16);
            // only the TMA-fed operand's two boxes: the gathered one's rows past
            // the bin were zero-filled by its copies (src-size 0)
            if (valid < BK && valid < upto)
              zero_k_rows(tiles_smem + stage * SBYTES + (GA ? A_BYTES : 0), 2, valid, upto, lane);
          }
          fence_proxy_async_smem();
          __syncwarp();
          // Signal the leader through the async proxy: a 16-byte DSMEM bulk copy
          // whose complete_tx lands on the leader's lfull[stage].  Unlike a
          // remote mbarrier.arrive it does not stall this thread.
          if (elect_one_sync()) bulk_signal_cta0(smem_u32(signal + 16), smem_u32(signal), smem_u32(&lfull_bar[stage]));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (p.timing == 2 && lane == 0 && cluster_id < 4)
        printf("tc2 relay cluster %d: total %lld cyc, waiting on own stage %lld (%.1f%%)\n", (int)cluster_id,
               clock64() - r_start, r_wait, 100.0 * r_wait / (clock64() - r_start));
    }
  } else if (warp < EPI_WARPS) {
    if constexpr (STAGED) {
      // ===================== epilogue (own 128 rows) =====================
      // TMEM -> registers -> activation math -> a per-warp 4 KB staging tile ->
      // coalesced global stores (8 lanes per 128-byte row segment, 4 rows per
      // instruction).  Row-per-thread stores touch 32 lines per instruction and
      // cost up to 16 % of the tensor pipe on C1 layer 1 (base-clock ncu); the
      // act-grad operand (h_pre) is read through the same staging tile.
      const int q = warp & 3;
      const int c_begin = (warp / 4) * EPI_COLS;
      const int r = q * 32 + lane;
      const uint32_t stg = smem_u32(staging + warp * STG_BYTES);
      const int cr = lane >> 3, cc = lane & 7;  // copy role: rows cr + 4 i, 16-byte chunk cc
      // grouped outputs are contiguous row ranges: whole 32-row slabs leave by TMA
      const bool tma_out = GK || p.grouped_out;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = 0;; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        const bool has_acc = tl.nkb > 0;
        // WIDE tiles drain their two 256-row halves in turn (accumulator columns
        // [256 h, 256 h + 256)), releasing each as soon as it is read
#pragma unroll 1
        for (int h = 0; h < (WIDE ? 2 : 1); ++h) {
        const int abuf = WIDE ? h : acc;
        const int64_t mb = tl.m0 + (int64_t)TM * h;
        const int64_t row = mb + HM * rank + r;
        const int64_t slab0 = mb + HM * rank + q * 32;
        // a slab straddling the bin end must not touch the next expert's rows
        const bool slab_tma = tma_out && slab0 + 32 <= tl.m_end;
        const int slab_row = (int)(GK ? (int64_t)tl.e * p.M + slab0 : slab0);
        long long dst = -1;
        const bool heads = !GK && p.hd_dh > 0;
        if (row < tl.m_end) {
          if (!GK && p.peer_out) {  // absolute address of the row in its owner's buffer
            dst = (long long)(p.peer_out[p.row_src[row]] + (uint64_t)p.row_slot[row] * (uint64_t)p.N * 2u);
          } else if (heads) {       // element offset of the slot's head 0 in the head layout
            const int64_t s = p.order[row];
            const int64_t t = s / p.hd_k;
            const int64_t b = t / p.hd_seq;
            dst = (((b * (p.N / p.hd_dh)) * p.hd_k + (s - t * p.hd_k)) * p.hd_seq + (t - b * p.hd_seq)) * p.hd_dh;
          } else {
            dst = GK ? (int64_t)tl.e * p.M + row : (p.grouped_out ? row : (int64_t)p.order[row]);
          }
        }
        long long cdst[8];
  #pragma unroll
        for (int i = 0; i < 8; ++i) cdst[i] = __shfl_sync(0xffffffffu, dst, cr + 4 * i);
        const bool combine = p.epi == EPI_COMBINE;
        // *_SCALED epilogues: this thread's row scale and combine-weight-gradient partial
        float rscale = 1.0f, dpacc = 0.0f;
        // gated (expert-parallel) tiles: the row scales were stored by peers; they
        // are read only after this thread's own acquire of the arrival counter below
        if (epi_scaled(p.epi) && dst >= 0 && !p.arrive) rscale = __ldcg(p.pw + p.order[row]);
        float cscale = 0.f;  // combine: this thread's row weight; cdst becomes the token row
        if (combine) {
          if (dst >= 0) cscale = __ldcg(p.pw + dst);
  #pragma unroll
          for (int i = 0; i < 8; ++i) cdst[i] = cdst[i] >= 0 ? cdst[i] / p.combine_cols : -1;
        }
        if (has_acc && (WIDE || h == 0)) {  // WIDE: each half has its own tfull
          epi_wait_full(smem_u32(&tfull_bar[abuf]), acc_phase, warp);
          tc_fence_after();
        }
        if (p.arrive && epi_scaled(p.epi) && dst >= 0) {
          (void)ld_acquire_sys_u64(p.arrive + tl.e);   // the tile ran, so the count is complete
          rscale = __ldcg(p.pw + p.order[row]);
        }
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(abuf * TN + c_begin);
        // WIDE: the second half may lie past the bin / matrix.  SMOE_TC_TIMING=6
        // (debug probe): no epilogue work at all, accumulators released unread.
        const bool live = mb < tl.m_end && p.timing != 6;
  #pragma unroll 1
        for (int cg = 0; live && cg < EPI_COLS; cg += 64) {
          const int64_t col0 = tl.n0 + c_begin + cg;
          const bool col_ok = col0 + cc * 8 < p.N;
          if (col0 >= p.N) break;
          // the staging tile is reused: the previous TMA store must have read it
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
          if (combine) {
            // p-scaled fp32 rows -> staging tile (32 rows x 32 columns x 4 B per
            // half) -> coalesced 16-byte vector reductions into the token rows
  #pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t v[32];
              if (has_acc) {
                tmem_ld16(tbase + cg + 32 * hf, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(tbase + cg + 32 * hf + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld_wait();
              } else {
  #pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0u;
              }
  #pragma unroll
              for (int c = 0; c < 8; ++c)
                sts128(stg + lane * 128 + ((c ^ (lane & 7)) << 4),
                       make_uint4(__float_as_uint(__uint_as_float(v[4 * c]) * cscale),
                                  __float_as_uint(__uint_as_float(v[4 * c + 1]) * cscale),
                                  __float_as_uint(__uint_as_float(v[4 * c + 2]) * cscale),
                                  __float_as_uint(__uint_as_float(v[4 * c + 3]) * cscale)));
              __syncwarp();
              const int64_t ccol = col0 + 32 * hf + cc * 4;
  #pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rl = cr + 4 * i;
                const uint4 val = lds128(stg + rl * 128 + ((cc ^ (rl & 7)) << 4));
                if (cdst[i] >= 0 && ccol < p.N) red_add_v4(p.yacc + cdst[i] * p.N + ccol, val);
              }
              __syncwarp();
            }
            continue;
          }
          if (epi_act_grad(p.epi)) {
            // coalesced read of the 32 rows' h_pre segments into the staging tile
  #pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rl = cr + 4 * i;
              uint4 val = make_uint4(0, 0, 0, 0);
              // head-layout output: the act-grad operand is read by grouped row
              const long long arow = heads ? (long long)(slab0 + rl) : cdst[i];
              if (cdst[i] >= 0 && col_ok) val = __ldg(reinterpret_cast<const uint4 *>(p.aux + arow * p.N + col0 + cc * 8));
              sts128(stg + rl * 128 + ((cc ^ (rl & 7)) << 4), val);
            }
            __syncwarp();
          }
          // one pass per output (EPI_ACT writes h_pre, then act(h_pre) from a TMEM re-read);
          // each pass builds this lane's 128-byte row segment in two 32-column halves
          const int passes = (p.epi == SMOE_EPI_ACT || p.epi == SMOE_EPI_ACT_SCALED) ? 2 : 1;
          for (int pass = 0; pass < passes; ++pass) {
  #pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t v[32];
              if (has_acc) {
                tmem_ld16(tbase + cg + 32 * hf, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(tbase + cg + 32 * hf + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
              } else {
  #pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0u;
              }
              uint32_t io[16];
              if (epi_act_grad(p.epi)) {
  #pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const uint4 val = lds128(stg + lane * 128 + (((4 * hf + c) ^ (lane & 7)) << 4));
                  io[4 * c] = val.x; io[4 * c + 1] = val.y; io[4 * c + 2] = val.z; io[4 * c + 3] = val.w;
                }
              }
              if (has_acc) tmem_ld_wait();
              epilogue_pack32(p, v, io, pass == 1, rscale, &dpacc);
  #pragma unroll
              for (int c = 0; c < 4; ++c)
                sts128(stg + lane * 128 + (((4 * hf + c) ^ (lane & 7)) << 4),
                       make_uint4(io[4 * c], io[4 * c + 1], io[4 * c + 2], io[4 * c + 3]));
            }
            if (slab_tma) {
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(pass == 0 ? &tma_c : &tma_c2, stg, (int)col0, slab_row);
                bulk_commit();
                if (pass + 1 < passes) bulk_wait_read0();
              }
              __syncwarp();
            } else {
              __syncwarp();
              if (heads) {
                // the 64-column chunk lies in one head: shift the base so that
                // row offset + col0 + 8 cc lands at head (col0 / dh), column col0 % dh
                const int64_t hstride = (int64_t)p.hd_k * p.hd_seq * p.hd_dh;
                __nv_bfloat16 *hb = p.out + ((col0 / p.hd_dh) * hstride + (col0 % p.hd_dh) - col0);
                store_staged_rows(stg, hb, cdst, col0, col_ok, 1, cr, cc);
              } else {
                store_staged_rows(stg, (!GK && p.peer_out) ? nullptr : (pass == 0 ? p.out : p.out2), cdst, col0, col_ok,
                                  p.N, cr, cc);
              }
            }
          }
        }
        if (p.dp_part && dst >= 0) p.dp_part[row * p.dp_parts + (tl.n0 / TN) * 2 + warp / 4] = dpacc;
        if (has_acc) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(smem_u32(&tempty_bar[abuf]));
            else mbar_arrive_cluster(smem_u32(&tempty_bar[abuf]), 0);
          }
        }
        }  // halves
        if (has_acc) {
          if (WIDE) acc_phase ^= 1;
          else if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
      if (lane == 0) bulk_wait0();
    } else {
      // ---- direct epilogue: each thread stores its own row ----
      const int ew = warp;
      const int q = warp & 3;
      const int c_begin = (ew / 4) * EPI_COLS;
      const int r = q * 32 + lane;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = 0;; ++it) {
        const int64_t t = next_tile(it);
        if (t < 0) break;
        const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
        const int64_t row = tl.m0 + HM * rank + r;
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
        uint4 av[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
        const bool use_aux = epi_act_grad(p.epi) && valid;
        float rscale = 1.0f, dpacc = 0.0f;
        if (epi_scaled(p.epi) && valid && !p.arrive) rscale = __ldcg(p.pw + p.order[row]);
        if (use_aux) {
          const int64_t c0 = tl.n0 + c_begin;
  #pragma unroll
          for (int j = 0; j < 2; ++j)
            if (c0 + 8 * j < p.N) av[j] = __ldg(reinterpret_cast<const uint4 *>(arow + c0 + 8 * j));
        }
        if (has_acc) {
          epi_wait_full(smem_u32(&tfull_bar[acc]), acc_phase, ew);
          tc_fence_after();
        }
        if (p.arrive && epi_scaled(p.epi) && valid) {
          (void)ld_acquire_sys_u64(p.arrive + tl.e);
          rscale = __ldcg(p.pw + p.order[row]);
        }
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * TN + c_begin);
  #pragma unroll 1
        for (int c = 0; c < (p.timing == 6 ? 0 : EPI_COLS); c += 16) {
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
          if (valid && col0 < p.N) epilogue_chunk(p, v, av, orow, orow2, col0, rscale, &dpacc);
          av[0] = avn[0];
          av[1] = avn[1];
        }
        if (p.dp_part && valid) p.dp_part[row * p.dp_parts + (tl.n0 / TN) * 2 + ew / 4] = dpacc;
        if (has_acc) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(smem_u32(&tempty_bar[acc]));
            else mbar_arrive_cluster(smem_u32(&tempty_bar[acc]), 0);
          }
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else if (KGATHER) {
    // ===================== cp.async gather of grouped-K operand rows =====================
    // Per k-block each gathered operand is 64 K rows (bin slots) x this CTA's
    // 128 M (or N) columns = two 64-row x 128-B boxes, 128-B swizzled.  Thread
    // (rsub, chunk) copies 16-byte chunk `chunk` of rows rsub + RSTR q; rows
    // past the bin and columns past the matrix are zero-filled (src-size 0).
    constexpr int RPT = GW > 0 ? 32 / GW : 1;  // rows per thread per k-block
    constexpr int RSTR = 2 * GW;       // row stride between a thread's rows
    const int g = threadIdx.x - 32 * EPI_WARPS;
    const int chunk = g & 15;
    const int rsub = g >> 4;
    const int box = chunk >> 3, cq = chunk & 7;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      const int64_t t = next_tile(it);
      if (t < 0) break;
      const Tile tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
      const int64_t acol = tl.m0 + HM * rank + chunk * 8;
      const int64_t bcol = tl.n0 + HN * rank + chunk * 8;
      const bool a_ok = acol < p.M, b_ok = bcol < p.N;
      // Source rows run IDX_PF k-blocks ahead.  Per k-block each warp needs the
      // 2 RPT bin rows 2w + b + RSTR q (b = lane >> 4).  Lane b + 2q turns
      // row q's slot into the A source row's offset in 16-byte chunks
      // ((slot / fan_out) * M / 8; bit 31 set = past the bin), lane
      // 16 + b + 2q the B offset, and the warp shares them by shuffles: the
      // copy loop does one shuffle, one address and one cp.async per row.
      const int wl = g >> 5;
      const int64_t prow = 2 * wl + (lane & 1) + RSTR * ((lane >> 1) & (RPT - 1));
      const uint32_t fdiv = (uint32_t)(lane < 16 ? p.fan_out : p.fan_out_b);
      const uint32_t rchunks = (uint32_t)((lane < 16 ? p.M : p.N) >> 3);
      // raw slot ids are loaded IDX_PF k-blocks ahead and converted only when used
      const int32_t *optr = p.order + tl.k0 + prow;
      const int64_t rows_left = tl.k_len - prow;  // row kb*BK + prow exists iff kb*BK < rows_left
      auto ld_slot = [&](int kb) -> int32_t {
        return (int64_t)kb * BK < rows_left ? __ldg(optr + (int64_t)kb * BK) : -1;
      };
      constexpr int IDX_PF = 4;
      int32_t pf[IDX_PF];
#pragma unroll
      for (int j = 0; j < IDX_PF; ++j) pf[j] = ld_slot(j);
      const uint4 *xa = reinterpret_cast<const uint4 *>(p.x + (a_ok ? acol : 0));
      const uint4 *yb = reinterpret_cast<const uint4 *>(p.y + (b_ok ? bcol : 0));
      const uint32_t asz = a_ok ? 16u : 0u, bsz = b_ok ? 16u : 0u;
      uint32_t doff[RPT];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = rsub + RSTR * q;
        doff[q] = box * 8192 + r * 128 + ((cq ^ (r & 7)) << 4);
      }
      // unrolled by IDX_PF so each prefetch register is consumed in place (a
      // register rotation would wait on the loads still in flight)
      for (int kb0 = 0; kb0 < tl.nkb; kb0 += IDX_PF) {
#pragma unroll
        for (int j = 0; j < IDX_PF; ++j) {
          const int kb = kb0 + j;
          if (kb >= tl.nkb) break;
          const uint32_t mine = pf[j] >= 0 ? ((uint32_t)pf[j] / fdiv) * rchunks : 0x80000000u;
          pf[j] = ld_slot(kb + IDX_PF);
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t sa = smem_u32(tiles_smem + stage * SBYTES);
          const uint32_t sb = sa + ABYTES;
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            if (GA) {
              const uint32_t o = __shfl_sync(0xffffffffu, mine, (lane >> 4) + 2 * q);
              cp_async16(sa + doff[q], xa + (o & 0x7fffffffu), asz & ~(uint32_t)((int32_t)o >> 31));
            }
            if (GB) {
              const uint32_t o = __shfl_sync(0xffffffffu, mine, 16 + (lane >> 4) + 2 * q);
              cp_async16(sb + doff[q], yb + (o & 0x7fffffffu), bsz & ~(uint32_t)((int32_t)o >> 31));
            }
          }
          cp_async_arrive_noinc(smem_u32(&lfull_bar[stage]));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (AM == A_GATHER) {
    // ===================== cp.async gather of this CTA's 128 A rows =====================
    const int g = threadIdx.x - 32 * EPI_WARPS;
    const int chunk = g & 7;
    const int rsub = g >> 3;
    // Row indices of the NEXT tile are fetched while this tile streams (after
    // its first stage is issued), so no index-load bubble sits at tile boundaries.
    auto load_rows = [&](const Tile &tn, int32_t (&dst)[G_RPT]) {
      const int64_t mh = tn.m0 + HM * rank;
#pragma unroll
      for (int j = 0; j < G_RPT; ++j) dst[j] = __ldg(p.order + min(mh + TG_ROWS + j * G_RSTEP + rsub, tn.m_end - 1));
    };
    int stage = 0;
    uint32_t phase = 0;
    int64_t t = next_tile(0);
    Tile tl{};
    int32_t cur[G_RPT] = {}, nxt[G_RPT] = {};
    if (t >= 0) {
      tl = decode_tile<GK, TMT, TN>(t, p, s_start, s_off, nN, mM);
      load_rows(tl, cur);
    }
    for (int it = 0; t >= 0; ++it) {
      int64_t t_n = -1;
      Tile tl_n{};
      auto prefetch_next = [&]() {
        t_n = next_tile(it + 1);
        if (t_n >= 0) {
          tl_n = decode_tile<GK, TMT, TN>(t_n, p, s_start, s_off, nN, mM);
          load_rows(tl_n, nxt);
        }
      };
      const __nv_bfloat16 *src[G_RPT];
#pragma unroll
      for (int j = 0; j < G_RPT; ++j) src[j] = p.x + (int64_t)(cur[j] / p.fan_out) * p.K + chunk * 8;
      for (int kb = 0; kb < tl.nkb; ++kb) {
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        const uint32_t sa = smem_u32(tiles_smem + stage * SBYTES);
        const int64_t col = (int64_t)kb * BK;
        const bool ok = col + chunk * 8 < p.K;
#pragma unroll
        for (int j = 0; j < G_RPT; ++j) {
          const int rr = TG_ROWS + j * G_RSTEP + rsub;
          cp_async16(sa + rr * 128 + ((chunk ^ (rr & 7)) << 4), ok ? (const void *)(src[j] + col) : (const void *)src[j],
                     ok ? 16u : 0u);
        }
        cp_async_arrive_noinc(smem_u32(&lfull_bar[stage]));
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (kb == 0) prefetch_next();
      }
      if (tl.nkb == 0) prefetch_next();
      t = t_n;
      tl = tl_n;
#pragma unroll
      for (int j = 0; j < G_RPT; ++j) cur[j] = nxt[j];
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == WM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// m-blocks per raster band for the grouped-K (weight-gradient) schedule: a
// near-square block of the 74 concurrent cluster tiles (8 x ~9) maximises
// panel sharing while each tile streams its long K (= bin) panels.
static int group_m_k_setting() {
  static int gm = -1;
  if (gm < 0) {
    const char *env = getenv("SMOE_GROUP_M_K");
    gm = env ? atoi(env) : 8;
    if (gm < 1) gm = 8;
  }
  return gm;
}

static size_t smem_bytes(int E, bool staged, bool wide = false) {
  const int stages = wide_stages(staged, wide);
  return 1024 + stages * (wide ? STAGE_BYTES + A_BYTES : STAGE_BYTES) + (staged ? EPI_WARPS * STG_BYTES : 0) + 8 * (2 * stages + sig_slots(stages) + 4 + 2 * RING + 2 + RING / 2) +
         12 * (E + 1) + 64;
}

}  // namespace tc2

bool tc2_supports_experts(int E) {
  return tc2::smem_bytes(E, true) <= 232448 && tc2::smem_bytes(E, false) <= 232448 &&
         tc2::smem_bytes(E, true, true) <= 232448;
}

namespace tc2 {

// SMs the persistent GEMMs leave free (smoe_set_sm_reserve): a GEMM occupies
// one CTA per SM with ~230 KB of shared memory, so a kernel that must run
// concurrently with it on another stream (NCCL's all-to-all in ep.py) needs
// SMs of its own.
static std::atomic<int> g_sm_reserve{0};
static int sm_reserve() { return g_sm_reserve.load(std::memory_order_relaxed); }

}  // namespace tc2
}  // namespace smoe

extern "C" int smoe_set_sm_reserve(int32_t sms) {
  if (sms < 0 || sms > smoe::num_sms() - 2) return smoe::fail(SMOE_EINVAL, "sm_reserve out of range");
  smoe::tc2::g_sm_reserve.store(sms & ~1, std::memory_order_relaxed);   // whole CTA pairs
  return SMOE_OK;
}

namespace smoe {
namespace tc2 {

// Tile counters of the dynamic schedule: one zeroed (stream-ordered memset) per
// launch; a 64-entry pool so launches in flight on different streams never
// share one.
// Each entry: [0] the tile counter, [1, 1 + 128) the clusters' lockstep
// progress; both zeroed by one memset per launch.
constexpr int kSyncSlots = 128;
__device__ uint32_t g_tile_ctr[64][1 + kSyncSlots];

static uint32_t *tile_counter(cudaStream_t st, bool with_prog) {
  static uint32_t *base = nullptr;
  static std::atomic<unsigned> seq{0};
  if (!base && cudaGetSymbolAddress((void **)&base, g_tile_ctr) != cudaSuccess) return nullptr;
  uint32_t *c = base + (seq.fetch_add(1) % 64) * (1 + kSyncSlots);
  if (cudaMemsetAsync(c, 0, sizeof(uint32_t) * (with_prog ? 1 + kSyncSlots : 1), st) != cudaSuccess) return nullptr;
  return c;
}

// Wave lockstep of the long-K GEMMs.  With the in-order dynamic schedule the
// pairs running at once hold neighbouring tiles whose operand panels (up to
// 512 rows x K) they share — but only while they stream K in step: measured at
// C1 layer 2, the start times within a 74-tile wave spread to a whole tile
// duration (p10-p90 ~200 us of 222) after four waves, tile times vary
// 185-277 us, and each tile re-reads its panels from DRAM (9.5 GB against
// 3.4 GB algorithmic; profiles/r2_lockstep.txt).  Each leader therefore issues
// its ring chunk v (sync_chunk k-blocks) only while v <= min over clusters of
// the chunks issued + sync_slack, so concurrent tiles stay within slack chunks
// of each other and a panel slice is fetched from DRAM about once per wave.
// The slowest cluster never waits, so the gate cannot deadlock while all
// clusters are resident (the grid is sized to the resident pairs); clusters
// out of tiles publish UINT_MAX.  Off for the expert-parallel gated kernels.
// Measured: layer 2 DRAM 9.9 -> 6.4 GB per launch, but the gated kernels lose
// what their fastest pairs idle at the gate and the power-capped step is
// unchanged, so it is off by default (an A/B knob).
// SMOE_TC_SYNC = k-blocks per chunk (0 = off), SMOE_TC_SYNC_SLACK = chunks.
static void set_lockstep(Params &q, int clusters, bool eligible) {
  static int chunk = -1, slack = -1;
  if (chunk < 0) {
    const char *env = getenv("SMOE_TC_SYNC");
    chunk = env ? atoi(env) : 0;
    env = getenv("SMOE_TC_SYNC_SLACK");
    slack = env ? atoi(env) : 8;
  }
  q.sync_chunk = (eligible && chunk > 0 && !q.arrive && clusters <= kSyncSlots) ? chunk : 0;
  q.sync_slack = slack;
  q.nclusters = clusters;
}

// Serpentine K order (SMOE_TC_SERP: 0 off, 1 wide TMA-fed kernels, 2 every
// TMA-fed kernel, 3 every TMA-fed kernel by global tile id / grid pairs, 4 the
// TMA-fed grouped-K (weight-gradient) kernels): a
// tile streams its k-blocks in reverse when its index within its expert, / 74
// (the CTA pairs), is odd, so each wave of concurrent tiles starts on the K
// range the previous wave read last (still in L2).  A tile's accumulation
// order then depends on its tile shape and place within its expert (never on
// the grid or the other experts).  Measured (profiles/r2_lockstep.txt): the dW
// GEMM -1.2 % (C1 5.86 -> 5.80 ms, C2 3.15 -> 3.10), step +0.3 %; applied to the
// grouped-M kernels too (modes 1-3) it gains little more and would make the
// expert-parallel layer 1 (a TMA-fed kernel) differ in rounding from the
// single-GPU gather kernel — so the default is 4, the weight-gradient kernels.
static void set_serp(Params &q, bool tma_fed, bool wide, bool gk) {
  static int mode = -1;
  if (mode < 0) {
    const char *env = getenv("SMOE_TC_SERP");
    mode = env ? atoi(env) : 4;
  }
  const bool on = tma_fed && (mode == 2 || mode == 3 || (mode == 1 && wide) || (mode == 4 && gk));
  q.serp = on ? (mode == 3 ? 2 : 1) : 0;
}

// L2 eviction priority of the TMA operand loads (SMOE_L2_HINT: off (default) |
// keep | keepfirst).  A raster band is group_m row-blocks x all column blocks,
// visited row-block-fastest.  When a band holds more tiles than the 74
// concurrent CTA pairs, a tile wave sweeps the band's columns and every wave
// re-reads the band's A panels: A is kept (EVICT_LAST).  When the band is
// smaller than a wave, each wave spans whole bands and it is the B panels
// (weights / the grouped-K right operand) that the next bands re-read: B is kept.
// Measured at C1 under the power cap (profiles/r2_l2_hint_ab.log): "keep" leaves
// DRAM bytes and J per launch unchanged (l2 9.26 -> 9.25 GB), "keepfirst" adds
// 4-6 GB of DRAM reads and costs 4 % — so the default issues no hint.
static void set_l2_policy(Params &q, int clusters, int tn) {
  static int mode = -1;
  if (mode < 0) {
    const char *env = getenv("SMOE_L2_HINT");
    mode = (!env || !strcmp(env, "off")) ? 0 : !strcmp(env, "keepfirst") ? 2 : 1;
  }
  q.pol_a = q.pol_b = kL2EvictNormal;
  if (mode == 0) return;
  const int64_t n_blocks = (q.N + tn - 1) / tn;
  const bool a_persists = (int64_t)q.group_m * n_blocks > clusters;
  const uint64_t other = mode == 2 ? kL2EvictFirst : kL2EvictNormal;
  q.pol_a = a_persists ? kL2EvictLast : other;
  q.pol_b = a_persists ? other : kL2EvictLast;
}

template <int AM, int BMODE, bool GK, bool STAGED, bool WIDE = false>
static int launch(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &tc, const CUtensorMap &tc2,
                  const Params &p, int64_t max_tiles, cudaStream_t st) {
  auto kern = tc2_gemm_kernel<AM, BMODE, GK, STAGED, WIDE>;
  size_t smem = smem_bytes(p.E, STAGED, WIDE);
  static size_t configured = 0;
  if (configured < smem) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("tc2_gemm: smem attribute");
    configured = smem;
  }
  int clusters = (num_sms() - sm_reserve()) / 2;
  if (clusters < 1) clusters = 1;
  if (max_tiles < clusters) clusters = (int)(max_tiles > 0 ? max_tiles : 1);
  Params q = p;
  set_l2_policy(q, clusters, TN);
  // the wide (long-K, TMA-fed) kernels only: gating the gather kernels' ring
  // starves their cp.async warps (C1 layer 1: 5.6 -> 6.7 ms under ncu)
  set_lockstep(q, clusters, WIDE && !has_gather(AM, BMODE));
  set_serp(q, !has_gather(AM, BMODE), WIDE, GK);
  q.tile_ctr = tile_counter(st, q.sync_chunk > 0);
  if (!q.tile_ctr) return check_launch("tc2_gemm: tile counter");
  q.prog = q.tile_ctr + 1;
  kern<<<2 * clusters, kernel_threads(AM, BMODE), smem, st>>>(ta, tb, tc, tc2, q);
  return check_launch("tc2_gemm");
}

// Which kernels stage their epilogue (see ring_stages): the gather-mode kernels.
// For the TMA-fed kernels the 7th ring stage is worth more than TMA stores
// (base-clock ncu, C1: rows 88.2 -> 86.8 %, dh 81.0 -> 79.7 %, xty 70.1 -> 69.3 %
// tensor-pipe active when staged; gather 75.0 -> 77.0 %, l1 68.4 -> 70.6 %).
// SMOE_TC_EPI=all stages every grouped-output kernel too (A/B experiments).
// Short-K GEMMs (K <= SMOE_TC_STAGE_K, default 1024: the MoMHA projections'
// d_proj = 512 side) are epilogue-bound, so they stage too: a tile's mainloop
// is only K/64 ring stages long and the 7th stage buys nothing.
// Scattered-output kernels stage too (SMOE_TC_STAGE_SCATTERED=0 turns it off):
// row-per-thread stores to scattered slots cost the C2 K = 1792 layer-2 / dX
// GEMMs 6 % of tensor-pipe activity (86 % vs 92 % with the epilogue removed,
// SMOE_TC_TIMING=6); staged, coalesced row segments take them to 88 % and
// 2.75 -> 2.66 ms (scripts/c2_epi_variants.sh).
static bool staged_for(bool gather, bool grouped_out, int64_t K) {
  static int all = -1, scattered = -1;
  static int64_t small_k = -1;
  if (all < 0) {
    const char *env = getenv("SMOE_TC_EPI");
    all = (env && !strcmp(env, "all")) ? 1 : 0;
    const char *k = getenv("SMOE_TC_STAGE_K");
    small_k = k ? atoll(k) : 1024;
    const char *sc = getenv("SMOE_TC_STAGE_SCATTERED");
    scattered = sc ? atoi(sc) : 1;
  }
  return gather || (all && grouped_out) || K <= small_k || (scattered && !grouped_out);
}

// Wide 512-row tiles (see wide_stages) for the TMA-fed kernels whose K is long
// enough to hide the exposed part of the epilogue: the next tile's MMAs wait
// for the first half's drain, its second MMA for the second half's.  C1
// (SMOE_TC_TIMING=1, MMA-issuer wait on the epilogue): K = 14336 4.3 %, the
// grouped-K dW GEMMs (bins of 8192) 5.0 %, K = 4096 10.8 %, and 42 % for the
// act-grad epilogue (it reads h_pre) at K = 4096 — so wide tiles go to plain
// epilogues with K >= 8192 and to the dW GEMMs with bins >= 4096 rows (C2: +0.8 %;
// scripts/wide_ab*.sh, scripts/wide_c2.sh, profiles/r1_wide_tiles.txt).
// SMOE_TC_WIDE=0 disables them, =1 forces them whenever the kernel allows.
static int wide_mode() {
  static int mode = -2;
  if (mode == -2) {
    const char *env = getenv("SMOE_TC_WIDE");
    mode = env ? atoi(env) : -1;
  }
  return mode;
}
// Stages per first / last MMA group of a wide tile (SMOE_TC_WIDE_DEFER, 1..4).
static int wide_defer() {
  static int d = -1;
  if (d < 0) {
    const char *env = getenv("SMOE_TC_WIDE_DEFER");
    d = env ? atoi(env) : 4;
  }
  return d;
}
static bool wide_for(int64_t K, int epi, bool grouped_k = false) {
  if (wide_mode() >= 0) return wide_mode() == 1;
  // K thresholds: SMOE_TC_WIDE_MIN_K (grouped-M kernels), SMOE_TC_WIDE_MIN_BIN
  // (grouped-K kernels, mean bin length)
  static int64_t min_k = -1, min_bin = -1;
  if (min_k < 0) {
    const char *env = getenv("SMOE_TC_WIDE_MIN_K");
    min_k = env ? atoll(env) : 8192;
    env = getenv("SMOE_TC_WIDE_MIN_BIN");
    min_bin = env ? atoll(env) : 4096;
  }
  return K >= (grouped_k ? min_bin : min_k) && epi != SMOE_EPI_ACT_GRAD && epi != SMOE_EPI_ACT_GRAD_SCALED;
}

// Row-blocks (256 rows) per raster band of the grouped-M schedule.  With the
// in-order dynamic schedule the pairs running at once cover ~one band, whose A
// panels (256 rows x K) should stay L2-resident while the band's W panels
// stream: about 32 MB of A panels -> 16 blocks at K = 4096, 4 at K = 14336
// (C1 layer 2: DRAM reads 23 -> 12 GB and +2.5 % FLOP/J under the power cap
// vs a fixed 16).  SMOE_GROUP_M (in 128-row units, as for the 1-CTA engine)
// overrides.
static int band_rows(int64_t K) {
  if (getenv("SMOE_GROUP_M")) return (group_m_setting() + 1) / 2;
  const int64_t panel = 256 * K * 2;
  int64_t h = (32ll << 20) / (panel > 0 ? panel : 1);
  return (int)(h < 2 ? 2 : (h > 16 ? 16 : h));
}

// Output tile map for TMA stores: [rows, cols] bf16, 32-row x 64-column boxes.
static bool encode_out_map(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols) {
  uint64_t dims[2] = {(uint64_t)cols, (uint64_t)(rows > 0 ? rows : 1)};
  uint64_t strides[1] = {(uint64_t)cols * 2};
  uint32_t box[2] = {64, 32};
  return encode_map(m, ptr, 2, dims, strides, box);
}

static int s2s_impl(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                    const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int gout, int trans,
                    int epi, int act, void *out, void *out2, const void *aux, const float *pw, float *yacc,
                    int combine_cols, cudaStream_t st, const uint64_t *peer_out = nullptr,
                    const int32_t *row_src = nullptr, const int32_t *row_slot = nullptr,
                    float *dp_part = nullptr, int dp_parts = 0, const unsigned long long *arrive = nullptr,
                    int64_t hd_seq = 0, int hd_k = 0, int hd_dh = 0) {
  const int64_t d_in = trans ? w_cols : w_rows;
  const int64_t d_out = trans ? w_rows : w_cols;
  CUtensorMap ta, tb;
  {
    uint64_t dims[2] = {(uint64_t)d_in, (uint64_t)x_rows};
    uint64_t strides[1] = {(uint64_t)d_in * 2};
    uint32_t box[2] = {64, gin ? (uint32_t)HM : 1u};  // gather mode: tile::gather4 rows
    if (!encode_map(&ta, x, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(A) failed");
  }
  {
    uint64_t dims[3] = {(uint64_t)w_cols, (uint64_t)w_rows, (uint64_t)E};
    uint64_t strides[2] = {(uint64_t)w_cols * 2, (uint64_t)w_cols * w_rows * 2};
    uint32_t box[3] = {64, trans ? (uint32_t)HN : 64u, 1};
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
  p.out2 = (epi == SMOE_EPI_ACT || epi == SMOE_EPI_ACT_SCALED) ? (__nv_bfloat16 *)out2 : nullptr;
  p.aux = (epi == SMOE_EPI_ACT_GRAD || epi == SMOE_EPI_ACT_GRAD_SCALED) ? (const __nv_bfloat16 *)aux : nullptr;
  p.dp_part = dp_part;
  p.dp_parts = dp_parts;
  p.x = (const __nv_bfloat16 *)x;
  p.pw = pw;
  p.yacc = yacc;
  p.peer_out = peer_out;
  p.row_src = row_src;
  p.row_slot = row_slot;
  p.combine_cols = combine_cols;
  p.group_m = band_rows(d_in);
  p.timing = getenv("SMOE_TC_TIMING") ? atoi(getenv("SMOE_TC_TIMING")) : 0;
  p.arrive = arrive;
  p.hd_seq = hd_seq;
  p.hd_k = hd_k;
  p.hd_dh = hd_dh;
  const int64_t max_tiles = ((n + TM - 1) / TM + E) * ((d_out + TN - 1) / TN);
  CUtensorMap tc = ta, tc2 = ta;  // unused unless the output is grouped
  if (gout) {
    if (!encode_out_map(&tc, out, n, d_out)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(out) failed");
    if (p.out2 && !encode_out_map(&tc2, out2, n, d_out)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(out2) failed");
  }
  if (gin) {
    if (!peer_out && !hd_dh && wide_for(d_in, epi)) {
      const int64_t wide_tiles = ((n + 2 * TM - 1) / (2 * TM) + E) * ((d_out + TN - 1) / TN);
      p.group_m = (p.group_m + 1) / 2;  // bands in 512-row blocks
      p.wide_defer = wide_defer();
      if (!trans) return launch<A_ROWS, B_W_MN, false, true, true>(ta, tb, tc, tc2, p, wide_tiles, st);
      return launch<A_ROWS, B_W_K, false, true, true>(ta, tb, tc, tc2, p, wide_tiles, st);
    }
    if (epi == EPI_COMBINE || peer_out || hd_dh || staged_for(false, gout, d_in)) {
      if (!trans) return launch<A_ROWS, B_W_MN, false, true>(ta, tb, tc, tc2, p, max_tiles, st);
      return launch<A_ROWS, B_W_K, false, true>(ta, tb, tc, tc2, p, max_tiles, st);
    }
    if (!trans) return launch<A_ROWS, B_W_MN, false, false>(ta, tb, tc, tc2, p, max_tiles, st);
    return launch<A_ROWS, B_W_K, false, false>(ta, tb, tc, tc2, p, max_tiles, st);
  }
  if (!trans) return launch<A_GATHER, B_W_MN, false, true>(ta, tb, tc, tc2, p, max_tiles, st);
  return launch<A_GATHER, B_W_K, false, true>(ta, tb, tc, tc2, p, max_tiles, st);
}

int scatter2scatter(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                    const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int gout, int trans,
                    int epi, int act, void *out, void *out2, const void *aux, cudaStream_t st) {
  return s2s_impl(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, gout, trans, epi, act, out, out2,
                  aux, nullptr, nullptr, 1, st);
}

// Routing-weight-scaled epilogues (SMOE_EPI_ACT_SCALED / SMOE_EPI_ACT_GRAD_SCALED).
int scatter2scatter_scaled(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                           const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int gout,
                           int trans, int epi, int act, const float *row_scale, void *out, void *out2,
                           const void *aux, float *dp_part, int dp_parts, cudaStream_t st) {
  return s2s_impl(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, gout, trans, epi, act, out, out2,
                  aux, row_scale, nullptr, 1, st, nullptr, nullptr, nullptr, dp_part, dp_parts);
}

// Output rows scattered straight into the attention core's head layout
// (MoMHA): plain or routing-weight-scaled act-grad epilogue (aux by grouped row).
int scatter2scatter_heads(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                          const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, int trans,
                          int epi, int act, const float *row_scale, const void *aux, float *dp_part, int dp_parts,
                          int64_t seq_len, int k_slots, int d_head, void *heads, cudaStream_t st) {
  return s2s_impl(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, fan_out, gin, 0, trans, epi, act, heads, nullptr,
                  aux, row_scale, nullptr, 1, st, nullptr, nullptr, nullptr, dp_part, dp_parts, nullptr, seq_len, k_slots,
                  d_head);
}

// The scaled epilogues on rows delivered by peers (expert parallelism): grouped
// in / grouped out, each tile gated on its expert's arrival counter.
int scatter2scatter_scaled_gated(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                                 const int32_t *order, const int32_t *offsets, int64_t n, int trans, int epi, int act,
                                 const float *row_scale, void *out, void *out2, const void *aux, float *dp_part,
                                 int dp_parts, const unsigned long long *arrive, cudaStream_t st) {
  return s2s_impl(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, 1, 1, 1, trans, epi, act, out, out2, aux,
                  row_scale, nullptr, 1, st, nullptr, nullptr, nullptr, dp_part, dp_parts, arrive);
}

// Grouped-input GEMM whose epilogue stores output row i straight into row
// row_slot[i] of rank row_src[i]'s buffer (peer memory): the expert-parallel
// return fused into the expert GEMM (ep_peer.py).
int scatter2scatter_peer(const void *x, int64_t x_rows, const void *w, int E, int64_t w_rows, int64_t w_cols,
                         const int32_t *order, const int32_t *offsets, int64_t n, int trans, const uint64_t *peer_out,
                         const int32_t *row_src, const int32_t *row_slot, cudaStream_t st) {
  return s2s_impl(x, x_rows, w, E, w_rows, w_cols, order, offsets, n, 1, 1, 0, trans, SMOE_EPI_NONE, 0, nullptr,
                  nullptr, nullptr, nullptr, nullptr, 1, st, peer_out, row_src, row_slot);
}

// scatter_combine (kernels.py:242-286): scattered-output GEMM whose epilogue
// adds p_flat[slot] * row into yacc[slot / combine_cols] (fp32, zeroed here).
int scatter_combine(const void *x, int64_t x_rows, const void *w, int E, int64_t d_in, int64_t d_out,
                    const int32_t *order, const int32_t *offsets, int64_t n, int fan_out, int gin, const float *p_flat,
                    int combine_cols, float *yacc, cudaStream_t st) {
  if (cudaMemsetAsync(yacc, 0, sizeof(float) * (n / combine_cols) * d_out, st) != cudaSuccess)
    return check_launch("scatter_combine: zero accumulator");
  return s2s_impl(x, x_rows, w, E, d_in, d_out, order, offsets, n, fan_out, gin, 0, 0, EPI_COMBINE, 0, yacc,
                  nullptr, nullptr, p_flat, yacc, combine_cols, st);
}

int group_xty(const void *xg, const void *yg, const int32_t *offsets, int E, int64_t n, int64_t d_in, int64_t d_out,
              void *dw, cudaStream_t st, const unsigned long long *arrive) {
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
  p.offsets = offsets;
  p.fan_out = 1;
  p.grouped_out = 1;
  p.epi = SMOE_EPI_NONE;
  p.out = (__nv_bfloat16 *)dw;
  p.group_m = group_m_k_setting();
  p.timing = getenv("SMOE_TC_TIMING") ? atoi(getenv("SMOE_TC_TIMING")) : 0;
  p.arrive = arrive;
  const int64_t max_tiles = (int64_t)E * ((d_in + TM - 1) / TM) * ((d_out + TN - 1) / TN);
  CUtensorMap tc;
  if (!encode_out_map(&tc, dw, (int64_t)E * d_in, d_out)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(dW) failed");
  if (wide_for(E > 0 ? n / E : 0, SMOE_EPI_NONE, true)) {  // K = the bins, 8192 rows on average at C1
    const int64_t mw = (d_in + 2 * TM - 1) / (2 * TM);
    const int64_t wide_tiles = (int64_t)E * mw * ((d_out + TN - 1) / TN);
    // band in 512-row blocks: 4 (the whole d_model = 4096 side at C1), 2 when the
    // M side is long (d_expert = 14336: 28 blocks; 0.7 % less energy per launch,
    // scripts/xty_wide_band.sh); SMOE_GROUP_M_K overrides
    p.group_m = getenv("SMOE_GROUP_M_K") ? (p.group_m + 1) / 2 : (mw >= 16 ? 2 : 4);
    p.wide_defer = wide_defer();
    return launch<A_MN, B_ROWS_MN, true, true, true>(ta, tb, tc, tc, p, wide_tiles, st);
  }
  if (staged_for(false, true, INT64_MAX)) return launch<A_MN, B_ROWS_MN, true, true>(ta, tb, tc, tc, p, max_tiles, st);
  return launch<A_MN, B_ROWS_MN, true, false>(ta, tb, tc, tc, p, max_tiles, st);
}

// group_xty over scattered operands (parallel_linear.py:224-234 without the
// grouped copies): operand rows are gathered by slot (order[i] / fan_out) when
// the operand is scattered, read by TMA when it is already grouped.
int group_xty_scattered(const void *x, int64_t x_rows, int fa, int ga, const void *y, int64_t y_rows, int fb, int gb,
                        const int32_t *order, const int32_t *offsets, int E, int64_t n, int64_t d_in, int64_t d_out,
                        void *dw, cudaStream_t st) {
  CUtensorMap ta, tb;
  {
    uint64_t dims[2] = {(uint64_t)d_in, (uint64_t)(x_rows > 0 ? x_rows : 1)};
    uint64_t strides[1] = {(uint64_t)d_in * 2};
    uint32_t box[2] = {64, 64};
    if (!encode_map(&ta, x, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(X) failed");
  }
  {
    uint64_t dims[2] = {(uint64_t)d_out, (uint64_t)(y_rows > 0 ? y_rows : 1)};
    uint64_t strides[1] = {(uint64_t)d_out * 2};
    uint32_t box[2] = {64, 64};
    if (!encode_map(&tb, y, 2, dims, strides, box)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(Y) failed");
  }
  Params p{};
  p.E = E;
  p.M = d_in;
  p.N = d_out;
  p.K = 0;
  p.order = order;
  p.offsets = offsets;
  p.fan_out = fa;
  p.fan_out_b = fb;
  p.x = (const __nv_bfloat16 *)x;
  p.y = (const __nv_bfloat16 *)y;
  p.grouped_out = 1;
  p.epi = SMOE_EPI_NONE;
  p.out = (__nv_bfloat16 *)dw;
  p.group_m = group_m_k_setting();
  p.timing = getenv("SMOE_TC_TIMING") ? atoi(getenv("SMOE_TC_TIMING")) : 0;
  const int64_t max_tiles = (int64_t)E * ((d_in + TM - 1) / TM) * ((d_out + TN - 1) / TN);
  CUtensorMap tc;
  if (!encode_out_map(&tc, dw, (int64_t)E * d_in, d_out)) return fail(SMOE_ECUDA, "cuTensorMapEncodeTiled(dW) failed");
  if (ga && gb) return launch<A_MN, B_ROWS_MN, true, false>(ta, tb, tc, tc, p, max_tiles, st);
  if (gb) return launch<A_MN_G, B_ROWS_MN, true, false>(ta, tb, tc, tc, p, max_tiles, st);
  if (ga) return launch<A_MN, B_ROWS_MN_G, true, false>(ta, tb, tc, tc, p, max_tiles, st);
  return launch<A_MN_G, B_ROWS_MN_G, true, false>(ta, tb, tc, tc, p, max_tiles, st);
}

}  // namespace tc2
}  // namespace smoe
