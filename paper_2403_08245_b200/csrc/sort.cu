// K1: stable counting sort of the flattened routing ids.
//
// Replaces router.compute_grouped_order (router.py:154-164):
//   o = argsort(flat, kind="stable"); counts = bincount(flat); offsets = [0, cumsum]
// Every key is an expert id in [0, E), so a single counting-sort digit suffices.
// Default path (E <= 256 and each CTA's chunk of 1/2-byte keys fits in shared
// memory, n <~ 28 M): sort_onepass, ONE cooperative launch — read the int64 ids
// once, histogram, grid barrier, rank and write from shared memory (see the
// kernel's comment).  HBM traffic = the algorithmic 20 B per slot.
// Two-pass path (larger n, E > 256, or SMOE_SORT_ONEPASS=0):
//   1. sort_hist:    per 2048-slot tile, a shared-memory histogram -> hist[e][tile],
//                    and each slot's key compacted to 1 byte (E < 255) or 2 bytes;
//   2. sort_scan:    one block per expert scans its row of hist (tile-minor) to
//                    tile bases inside the expert's bin, and writes the bin size;
//                    (expert-major, tile-minor) is exactly the stable output order.
//   3. sort_scatter: every block rebuilds the bin starts from the E bin sizes,
//                    ranks its tile's slots stably (per-warp histograms over
//                    contiguous 512-slot chunks, equal-key lane masks from one
//                    ballot per key bit inside each 32-slot round), reorders the
//                    tile in shared memory and writes each expert's run
//                    contiguously (coalesced), plus the inverse permutation in
//                    slot order.  ~22 B of traffic per slot (the compact keys
//                    are written and read back through L2).
// Output order is the stable order (slots ascend inside each bin), bit-exact
// against numpy's stable argsort on both paths.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace smoe {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortMaxExperts = 1024;
// Slots per thread: 8 (2048-slot tiles) for large n; 4 (1024-slot tiles) below
// 2^20 slots so the bench-size sorts (n = 65,536 .. 262,144) still fill the GPU.
// The scatter kernel is latency-bound: tiles are sized for >= 4 resident blocks.
__host__ __device__ constexpr int sort_per_thread(int64_t n) { return n >= (1 << 20) ? 8 : 4; }

// Lanes of this warp holding the same key (key < 0 = invalid, matches only other
// invalid lanes), from one ballot per key bit (NB >= bits of E-1).  Cheaper than
// match.any, whose latency dominated the tile ranking.
template <int NB>
__device__ __forceinline__ unsigned warp_peers(int32_t key) {
  const bool valid = key >= 0;
  const unsigned vb = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? vb : ~vb;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const bool bit = (key >> b) & 1;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bb : ~bb;
  }
  return peers;
}

// compact per-slot key written by the histogram pass (all ones = invalid id)
template <typename KT>
__device__ __forceinline__ KT compact_key(int64_t id, int E) {
  return (id >= 0 && id < E) ? (KT)id : (KT)~(KT)0;
}

template <int kSortPerThread, typename KT>
__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const int64_t *__restrict__ ids,
                                                                 int64_t n, int E, int num_tiles,
                                                                 int32_t *__restrict__ hist, KT *__restrict__ keys_out) {
  constexpr int kSortTile = kSortThreads * kSortPerThread;
  extern __shared__ int32_t s_hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  int64_t keys[kSortPerThread];
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const int64_t i = base + (int64_t)r * kSortThreads + threadIdx.x;
    keys[r] = i < n ? ids[i] : -1;
  }
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const int64_t i = base + (int64_t)r * kSortThreads + threadIdx.x;
    if (i < n) keys_out[i] = compact_key<KT>(keys[r], E);
    if (keys[r] >= 0 && keys[r] < E) atomicAdd(&s_hist[keys[r]], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[(int64_t)e * num_tiles + blockIdx.x] = s_hist[e];
}

// Exclusive scan of v[0..count) in place by one block (count <= per_thread *
// blockDim.x); returns the total.  s_warp: 32 ints of shared scratch.
template <int PER>
__device__ int32_t block_exclusive_scan(int32_t *v, int count, int32_t *s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int first = threadIdx.x * PER;
  int32_t loc[PER];
  int32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    loc[j] = (first + j < count) ? v[first + j] : 0;
    sum += loc[j];
  }
  int32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int32_t run = (warp > 0 ? s_warp[warp - 1] : 0) + x - sum;
  const int32_t total = s_warp[nw - 1];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (first + j < count) v[first + j] = run;
    run += loc[j];
  }
  __syncthreads();
  return total;
}

// Block e: exclusive scan of hist[e][0..num_tiles) (in place) and bin size -> totals[e].
__global__ void __launch_bounds__(1024) sort_scan_kernel(int32_t *__restrict__ hist, int num_tiles,
                                                         int32_t *__restrict__ totals) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  int32_t *row = hist + (int64_t)blockIdx.x * num_tiles;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < num_tiles; c0 += 4 * 1024) {
    const int cnt = min(4 * 1024, num_tiles - c0);
    // bias the chunk by the running carry after the scan
    const int32_t t = block_exclusive_scan<4>(row + c0, cnt, s_warp);
    const int32_t carry = s_carry;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) row[c0 + i] += carry;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + t;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = s_carry;
}

// Shared layout of sort_scatter (dynamic): cnt[W][E] | lstart[E] | gbase[E] |
// slot[4096] | key[4096] | warp scratch[32]
template <int kSortPerThread, int NB, typename KT>
__global__ void __launch_bounds__(kSortThreads, 4) sort_scatter_kernel(
    const KT *__restrict__ ids, int64_t n, int E, int num_tiles, const int32_t *__restrict__ hist,
    const int32_t *__restrict__ totals, int32_t *__restrict__ sorted_scattered, int32_t *__restrict__ sorted_expert,
    int32_t *__restrict__ inverse, int32_t *__restrict__ offsets) {
  constexpr int kSortTile = kSortThreads * kSortPerThread;
  extern __shared__ int32_t sm[];
  int32_t *s_cnt = sm;                         // [kSortWarps][E]
  int32_t *s_lstart = s_cnt + kSortWarps * E;  // tile-local start of each expert's run
  int32_t *s_gbase = s_lstart + E;             // global position of that run
  int32_t *s_slot = s_gbase + E;               // [kSortTile] slots in sorted tile order
  int32_t *s_key = s_slot + kSortTile;         // [kSortTile] their expert ids
  int32_t *s_warp = s_key + kSortTile;         // [32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * E; i += blockDim.x) s_cnt[i] = 0;
  // bin starts = exclusive scan of the bin sizes
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_gbase[e] = totals[e];
  __syncthreads();
  block_exclusive_scan<kSortMaxExperts / kSortThreads>(s_gbase, E, s_warp);
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) offsets[e] = s_gbase[e];
    if (threadIdx.x == 0) offsets[E] = (int32_t)n;
  }

  const int64_t tile0 = (int64_t)blockIdx.x * kSortTile;
  const int64_t chunk0 = tile0 + (int64_t)warp * (32 * kSortPerThread);
  int32_t keys[kSortPerThread];
  unsigned pmask[kSortPerThread];  // equal-key lanes of each round
  // Pass 1: per-warp histogram of this warp's contiguous chunk.
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    int64_t i = chunk0 + r * 32 + lane;
    int32_t key = -1;
    if (i < n) {
      const KT kc = ids[i];
      key = kc == (KT)~(KT)0 ? -1 : (int32_t)kc;
    }
    keys[r] = key;
    const unsigned peers = warp_peers<NB>(key);
    pmask[r] = peers;
    if (key >= 0 && lane == __ffs(peers) - 1) s_cnt[warp * E + key] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Per expert: cross-warp exclusive offsets (tile-local, within the expert's
  // run) and the run length; then the runs' tile-local starts.
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    for (int w = 0; w < kSortWarps; ++w) {
      int32_t c = s_cnt[w * E + e];
      s_cnt[w * E + e] = run;
      run += c;
    }
    s_lstart[e] = run;
    s_gbase[e] += hist[(int64_t)e * num_tiles + blockIdx.x];
  }
  __syncthreads();
  block_exclusive_scan<kSortMaxExperts / kSortThreads>(s_lstart, E, s_warp);
  // Pass 2: stable rank -> tile-local sorted position; inverse in slot order.
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const int32_t key = keys[r];
    const unsigned peers = pmask[r];
    const int leader = __ffs(peers) - 1;
    if (key >= 0) {
      const int32_t within = s_cnt[warp * E + key] + __popc(peers & lt_mask);
      const int32_t lpos = s_lstart[key] + within;
      const int32_t slot = (int32_t)(chunk0 + r * 32 + lane);
      s_slot[lpos] = slot;
      s_key[lpos] = key;
      if (inverse) inverse[slot] = s_gbase[key] + within;
    }
    __syncwarp();
    if (key >= 0 && lane == leader) s_cnt[warp * E + key] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Write-out in sorted tile order: each expert's run lands contiguously.
  const int valid = (int)min((int64_t)kSortTile, n - tile0);
  for (int i = threadIdx.x; i < valid; i += blockDim.x) {
    const int32_t key = s_key[i];
    const int32_t pos = s_gbase[key] + (i - s_lstart[key]);
    sorted_scattered[pos] = s_slot[i];
    if (sorted_expert) sorted_expert[pos] = key;
  }
}

static size_t scatter_smem(int E, int tile) { return sizeof(int32_t) * ((size_t)kSortWarps * E + 2 * E + 2 * tile + 32); }

// ---------------------------------------------------------------------------
// One-pass variant (the default while every CTA's chunk of keys fits in its
// shared memory): ONE cooperative launch of at most one CTA per SM.
//   A. each CTA reads its contiguous chunk of int64 ids once (16-byte loads),
//      keeps them as 1/2-byte keys in shared memory and publishes the chunk's
//      histogram hist[cta][e];
//   B. grid barrier; every CTA derives the bin offsets and its chunk's base in
//      each bin from the E x grid histogram (L2-resident, a few KB);
//   C. the chunk is ranked and written tile by tile from shared memory with the
//      same stable warp ranking as sort_scatter, carrying per-expert run
//      lengths across tiles.
// HBM traffic is the algorithmic 20 B per slot (8 B id in, three 4 B outputs):
// the ids are never re-read and no key array goes through L2.
constexpr int kOneThreads = 256;
constexpr int kOneMinBlocks = 4;                    // co-resident CTAs per SM (latency overlap in C)
constexpr int kOneWarps = kOneThreads / 32;
// slots per thread per tile: 16 (4096-slot tiles, fewer barriers per slot) for
// large n, 8 below 2^21 slots so the bench-size sorts spread over more CTAs
__host__ __device__ constexpr int onepass_per(int64_t n) { return n >= (1 << 21) ? 16 : 8; }
constexpr int kOneMaxExperts = 256;
constexpr size_t kOneSmemLimit = 227 * 1024;

static size_t onepass_fixed_smem(int E, int kOneTile) {
  // cnt[W][E] | gbase[E] | lstart[E] | slot[tile] | warp scratch[32] | key[tile] (int16) | keys[chunk]
  return sizeof(int32_t) * ((size_t)kOneWarps * E + 2 * E + kOneTile + 32) + sizeof(int16_t) * kOneTile + 64;
}

template <int NB, typename KT, bool MATCH, int kOnePer>
__global__ void __launch_bounds__(kOneThreads, kOneMinBlocks) sort_onepass_kernel(
    const int64_t *__restrict__ ids, int64_t n, int E, int64_t chunk, int32_t *__restrict__ hist,
    int32_t *__restrict__ sorted_scattered, int32_t *__restrict__ sorted_expert, int32_t *__restrict__ inverse,
    int32_t *__restrict__ offsets) {
  constexpr int kOneTile = kOneThreads * kOnePer;
  extern __shared__ __align__(16) uint8_t sm1[];
  int32_t *s_cnt = reinterpret_cast<int32_t *>(sm1);  // [W][E]
  int32_t *s_gbase = s_cnt + kOneWarps * E;            // next position of this CTA in bin e
  int32_t *s_lstart = s_gbase + E;                     // bin position of a tile-local position, per expert
  int32_t *s_slot = s_lstart + E;                      // [tile]
  int32_t *s_warp = s_slot + kOneTile;                 // [32]
  int16_t *s_key = reinterpret_cast<int16_t *>(s_warp + 32);  // [tile]
  KT *s_keys = reinterpret_cast<KT *>(reinterpret_cast<uint8_t *>(s_key + kOneTile) +
                                      ((16 - (kOneTile * sizeof(int16_t)) % 16) % 16));  // [chunk]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * chunk;
  const int64_t c1 = min(n, c0 + chunk);
  const int64_t len = c1 > c0 ? c1 - c0 : 0;

  // ---- A: ids -> compact keys in shared memory + this chunk's histogram ----
  for (int i = threadIdx.x; i < kOneWarps * E; i += kOneThreads) s_cnt[i] = 0;
  __syncthreads();
  {
    int32_t *wh = s_cnt + warp * E;
    // chunk starts are multiples of the tile (even): pairs of ids per 16-byte load
    const int64_t pairs = len >> 1;
    const int4 *src = reinterpret_cast<const int4 *>(ids + c0);
    constexpr int U = 8;
    for (int64_t b0 = 0; b0 < pairs; b0 += (int64_t)U * kOneThreads) {
      const int64_t j0 = b0 + threadIdx.x;
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + (int64_t)u * kOneThreads;
        v[u] = j < pairs ? __ldcs(src + j) : make_int4(-1, -1, -1, -1);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + (int64_t)u * kOneThreads;
        if (j < pairs) {
          // id in [0, E) <=> high word 0 and low word < E (unsigned)
          const int32_t ka = (v[u].y == 0 && (uint32_t)v[u].x < (uint32_t)E) ? v[u].x : -1;
          const int32_t kb = (v[u].w == 0 && (uint32_t)v[u].z < (uint32_t)E) ? v[u].z : -1;
          constexpr uint32_t inv = (KT)~(KT)0;
          const uint32_t pa = ka < 0 ? inv : (uint32_t)ka, pb = kb < 0 ? inv : (uint32_t)kb;
          if (sizeof(KT) == 1) reinterpret_cast<uint16_t *>(s_keys)[j] = (uint16_t)(pa | (pb << 8));
          else reinterpret_cast<uint32_t *>(s_keys)[j] = pa | (pb << 16);
          // shared-memory atomics into this warp's histogram (lanes with equal
          // keys are serialised by the hardware: far fewer issue slots than a
          // ballot-per-bit match for this count-only pass)
          if (ka >= 0) atomicAdd(&wh[ka], 1);
          if (kb >= 0) atomicAdd(&wh[kb], 1);
        }
      }
    }
    if ((len & 1) && threadIdx.x == 0) {  // odd tail (only the last chunk)
      const int64_t a = ids[c1 - 1];
      const int32_t ka = (a >= 0 && a < E) ? (int32_t)a : -1;
      s_keys[len - 1] = ka < 0 ? (KT)~(KT)0 : (KT)ka;
      if (ka >= 0) wh[ka] += 1;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kOneThreads) {
    int32_t s = 0;
    for (int w = 0; w < kOneWarps; ++w) s += s_cnt[w * E + e];
    __stcg(hist + (int64_t)blockIdx.x * E + e, s);
  }
  cg::this_grid().sync();

  // ---- B: bin sizes and this CTA's base inside each bin ----
  // CTA e scans column e of hist over the CTAs (in place, exclusive) and
  // writes the bin size after the matrix; a second barrier publishes them, so
  // every CTA then reads only 2 E values (no grid x E reads per CTA).
  const int G = (int)gridDim.x;  // <= 4 * kOneThreads (checked at launch)
  for (int e = blockIdx.x; e < E; e += G) {
    for (int c = threadIdx.x; c < G; c += kOneThreads) s_slot[c] = __ldcg(hist + (int64_t)c * E + e);
    __syncthreads();
    const int32_t tot = block_exclusive_scan<4>(s_slot, G, s_warp);
    for (int c = threadIdx.x; c < G; c += kOneThreads) __stcg(hist + (int64_t)c * E + e, s_slot[c]);
    if (threadIdx.x == 0) __stcg(hist + (int64_t)G * E + e, tot);
    __syncthreads();
  }
  cg::this_grid().sync();
  for (int e = threadIdx.x; e < E; e += kOneThreads) {
    s_gbase[e] = __ldcg(hist + (int64_t)G * E + e);
    s_lstart[e] = __ldcg(hist + (int64_t)blockIdx.x * E + e);
  }
  __syncthreads();
  block_exclusive_scan<1>(s_gbase, E, s_warp);  // bin starts (E <= kOneThreads)
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < E; e += kOneThreads) offsets[e] = s_gbase[e];
    if (threadIdx.x == 0) offsets[E] = (int32_t)n;
  }
  for (int e = threadIdx.x; e < E; e += kOneThreads) {
    s_gbase[e] += s_lstart[e];
  }
  __syncthreads();

  // ---- C: stable ranking and write-out, one tile at a time ----
  // Per tile: (1) each warp ranks its contiguous 32*kOnePer slots (equal-key
  // lane masks, running per-warp counts); (2) warp 0 turns the W x E counts
  // into tile-local run starts per (warp, expert) and advances the CTA's
  // per-expert global base; (3) slots are placed in tile-sorted order in
  // shared memory (inverse written in slot order); (4) the tile leaves as
  // contiguous per-expert runs.  Three CTA barriers per tile.
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < kOneWarps * E; i += kOneThreads) s_cnt[i] = 0;
  __syncthreads();
  constexpr int EPL_MAX = kOneMaxExperts / 32;
  const int epl = (E + 31) / 32;  // experts per lane of warp 0 (contiguous)
  for (int64_t t0 = 0; t0 < len; t0 += kOneTile) {
    const int64_t w0 = t0 + (int64_t)warp * (32 * kOnePer);  // this warp's contiguous slots
    // key (8 bits, E <= 256) | rank among this warp's earlier slots of the key << 8; -1 = no id
    int32_t kl[kOnePer];
#pragma unroll
    for (int r = 0; r < kOnePer; ++r) {
      const int64_t i = w0 + r * 32 + lane;
      int32_t key = -1;
      if (i < len) {
        const KT kc = s_keys[i];
        key = kc == (KT)~(KT)0 ? -1 : (int32_t)kc;
      }
      const unsigned peers = MATCH ? __match_any_sync(0xffffffffu, key) : warp_peers<NB>(key);
      // the key group's first lane advances the warp's running count with a
      // shared-memory atomic and shares the old value: no load -> store chain
      // between rounds, so the 16 rounds' atomics pipeline (one warp's shared
      // accesses to an address are performed in issue order)
      const int leader = __ffs(peers) - 1;
      int32_t old = 0;
      if (key >= 0 && lane == leader) old = atomicAdd(&s_cnt[warp * E + key], __popc(peers));
      old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
      kl[r] = key >= 0 ? key | ((old + __popc(peers & lt_mask)) << 8) : -1;
    }
    __syncthreads();
    if (warp == 0) {
      int32_t tot[EPL_MAX];
      int32_t mine = 0;
#pragma unroll
      for (int j = 0; j < EPL_MAX; ++j) {
        const int e = lane * epl + j;
        int32_t t = 0;
        if (j < epl && e < E)
          for (int w = 0; w < kOneWarps; ++w) t += s_cnt[w * E + e];
        tot[j] = t;
        mine += t;
      }
      int32_t incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int32_t run = incl - mine;  // tile-local start of this lane's first expert
#pragma unroll
      for (int j = 0; j < EPL_MAX; ++j) {
        const int e = lane * epl + j;
        if (j < epl && e < E) {
          const int32_t lstart = run;
          for (int w = 0; w < kOneWarps; ++w) {
            const int32_t c = s_cnt[w * E + e];
            s_cnt[w * E + e] = run;  // tile-local start of (warp w, expert e)
            run += c;
          }
          s_lstart[e] = s_gbase[e] - lstart;  // global position = this + tile-local position
          s_gbase[e] += tot[j];
        }
      }
      if (lane == 31) s_warp[0] = incl;  // slots with valid ids in this tile
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kOnePer; ++r) {
      const int32_t v = kl[r];
      if (v >= 0) {
        const int32_t key = v & 0xff;
        const int32_t lpos = s_cnt[warp * E + key] + (v >> 8);
        const int32_t slot = (int32_t)(c0 + w0 + r * 32 + lane);
        s_slot[lpos] = slot;
        s_key[lpos] = (int16_t)key;
        if (inverse) __stcs(inverse + slot, s_lstart[key] + lpos);
      }
    }
    __syncthreads();
    const int32_t tcount = s_warp[0];
#pragma unroll 4
    for (int i = threadIdx.x; i < tcount; i += kOneThreads) {
      const int32_t key = s_key[i];
      const int32_t pos = s_lstart[key] + i;
      __stcs(sorted_scattered + pos, s_slot[i]);
      if (sorted_expert) __stcs(sorted_expert + pos, key);
    }
    for (int i = threadIdx.x; i < kOneWarps * E; i += kOneThreads) s_cnt[i] = 0;
    __syncthreads();
  }
}

// Per-device cache of the co-resident CTA limit of one one-pass instantiation.
struct OnePassCfg {
  int max_blocks = -1;
  size_t smem_set = 0;
};

template <int NB, typename KT, bool MATCH, int kOnePer>
static int launch_onepass(const int64_t *ids, int64_t n, int E, int32_t *hist, size_t hist_ints,
                          int32_t *sorted_scattered, int32_t *sorted_expert, int32_t *offsets, int32_t *inverse,
                          cudaStream_t stream, bool *used) {
  *used = false;
  auto kern = sort_onepass_kernel<NB, KT, MATCH, kOnePer>;
  constexpr int kOneTile = kOneThreads * kOnePer;
  const int sms = num_sms();
  // smallest grid whose chunks fit; chunks are whole tiles
  const size_t fixed = onepass_fixed_smem(E, kOneTile);
  if (fixed + 1024 > kOneSmemLimit) return 0;
  const int64_t tiles = (n + kOneTile - 1) / kOneTile;
  // the most CTAs per SM (up to kOneMinBlocks) whose chunks fit their share of
  // shared memory; chunks are whole tiles
  int64_t chunk = 0;
  int grid = 0;
  size_t smem = 0;
  for (int occ = kOneMinBlocks; occ >= 1 && !grid; --occ) {
    const int64_t per_cta = (tiles + (int64_t)occ * sms - 1) / ((int64_t)occ * sms);
    const size_t need = fixed + (size_t)per_cta * kOneTile * sizeof(KT) + 64;
    if ((need + 1024) * occ <= 228 * 1024) {
      chunk = per_cta * kOneTile;
      grid = (int)((tiles + per_cta - 1) / per_cta);
      smem = need;
    }
  }
  if (!grid || grid > 4 * kOneThreads || (size_t)grid * E + E > hist_ints) return 0;
  static OnePassCfg cfg[64];
  int dev = 0;
  cudaGetDevice(&dev);
  OnePassCfg &c = cfg[dev & 63];
  if (smem > c.smem_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOneSmemLimit) != cudaSuccess)
      return check_launch("route_sort: one-pass smem attribute", 0);
    c.smem_set = kOneSmemLimit;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kOneThreads, smem) != cudaSuccess)
    return check_launch("route_sort: occupancy", 0);
  if (per_sm < 1 || grid > per_sm * sms) return 0;  // cannot be co-resident: two-pass path
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kOneThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  const cudaError_t e =
      cudaLaunchKernelEx(&lc, kern, ids, n, E, chunk, hist, sorted_scattered, sorted_expert, inverse, offsets);
  if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
    (void)cudaGetLastError();   // no co-resident grid here (e.g. a partitioned device): two-pass path
    return 0;
  }
  *used = true;
  return check_launch("route_sort(one-pass)", 1);
}

static bool onepass_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *env = getenv("SMOE_SORT_ONEPASS");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}

static size_t key_bytes(int E) { return E < 255 ? 1 : 2; }

size_t route_sort_workspace(int64_t n, int E) {
  const int tile = kSortThreads * sort_per_thread(n);
  int64_t tiles = (n + tile - 1) / tile;
  if (tiles < 1) tiles = 1;
  const size_t hist = (size_t)(tiles * E + E) * sizeof(int32_t);
  return ((hist + 255) & ~(size_t)255) + (size_t)n * key_bytes(E);
}

int route_sort(const int64_t *ids, int64_t n, int E, int32_t *sorted_scattered,
               int32_t *sorted_expert, int32_t *offsets, int32_t *inverse, void *ws,
               size_t ws_bytes, cudaStream_t stream) {
  if (E < 1 || E > kSortMaxExperts)
    return fail(SMOE_EINVAL, "route_sort: num_experts must be in [1, 1024], got " + std::to_string(E));
  if (n < 0 || n >= (int64_t)INT32_MAX)
    return fail(SMOE_EINVAL, "route_sort: n must be in [0, 2^31-1), got " + std::to_string(n));
  if (ws_bytes < route_sort_workspace(n, E))
    return fail(SMOE_EINVAL, "route_sort: workspace too small");
  int32_t *hist = static_cast<int32_t *>(ws);
  if (n > 0 && E <= kOneMaxExperts && onepass_enabled() && ((uintptr_t)ids & 15) == 0) {
    const int per0 = sort_per_thread(n);
    const int64_t tiles0 = (n + kSortThreads * per0 - 1) / (kSortThreads * per0);
    const size_t hist_ints = (size_t)(tiles0 * E + E);
    const int nbc1 = E <= 8 ? 0 : E <= 16 ? 1 : E <= 64 ? 2 : 3;
    bool used = false;
    int rc;
    // equal-key lane masks: match.any for E <= 8 (cheaper than 4 ballots there),
    // one ballot per key bit above (SMOE_SORT_MATCH=0/1 forces either)
    static const int match_env = [] {
      const char *env = getenv("SMOE_SORT_MATCH");
      return env ? atoi(env) : -1;
    }();
    const bool match = match_env < 0 ? E <= 8 : match_env != 0;
    const bool big = onepass_per(n) == 16;
#define SMOE_ONEPASS_P(NBV, KTV, M, P) \
  launch_onepass<NBV, KTV, M, P>(ids, n, E, hist, hist_ints, sorted_scattered, sorted_expert, offsets, inverse, stream, &used)
#define SMOE_ONEPASS(NBV, KTV)                                                                      \
  (big ? (match ? SMOE_ONEPASS_P(NBV, KTV, true, 16) : SMOE_ONEPASS_P(NBV, KTV, false, 16))        \
       : (match ? SMOE_ONEPASS_P(NBV, KTV, true, 8) : SMOE_ONEPASS_P(NBV, KTV, false, 8)))
    if (E < 255) {
      rc = nbc1 == 0 ? SMOE_ONEPASS(3, uint8_t) : nbc1 == 1 ? SMOE_ONEPASS(4, uint8_t)
         : nbc1 == 2 ? SMOE_ONEPASS(6, uint8_t) : SMOE_ONEPASS(8, uint8_t);
    } else {
      rc = SMOE_ONEPASS(8, uint16_t);
    }
#undef SMOE_ONEPASS
#undef SMOE_ONEPASS_P
    if (used || rc != 0) return rc;
  }
  const int per = sort_per_thread(n);
  const int tile = kSortThreads * per;
  int tiles = (int)((n + tile - 1) / tile);
  int32_t *totals = hist + (int64_t)tiles * E;
  if (tiles == 0) {
    // Empty routing: offsets are all zero.
    cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), stream);
    return check_launch("route_sort(empty)", 0);
  }
  const size_t smem = scatter_smem(E, tile);
  const size_t hist_bytes = (((size_t)tiles * E + E) * sizeof(int32_t) + 255) & ~(size_t)255;
  void *keys = static_cast<uint8_t *>(ws) + hist_bytes;
  // key bits for the ballot ranking: E <= 8, 16, 64, 256, 1024
  const int nbc = E <= 8 ? 0 : E <= 16 ? 1 : E <= 64 ? 2 : E <= 256 ? 3 : 4;
  if (key_bytes(E) == 1) {
    using KT = uint8_t;
    auto hist_k = per == 8 ? sort_hist_kernel<8, KT> : sort_hist_kernel<4, KT>;
    using ScatterFn = void (*)(const KT *, int64_t, int, int, const int32_t *, const int32_t *, int32_t *, int32_t *,
                               int32_t *, int32_t *);
    static const ScatterFn table[2][4] = {
        {sort_scatter_kernel<4, 3, KT>, sort_scatter_kernel<4, 4, KT>, sort_scatter_kernel<4, 6, KT>,
         sort_scatter_kernel<4, 8, KT>},
        {sort_scatter_kernel<8, 3, KT>, sort_scatter_kernel<8, 4, KT>, sort_scatter_kernel<8, 6, KT>,
         sort_scatter_kernel<8, 8, KT>}};
    const ScatterFn scat_k = table[per == 8][nbc];
    static size_t configured[2][4] = {};
    size_t &cfg = configured[per == 8][nbc];
    if (smem > cfg) {
      if ((smem > 48 * 1024 &&
           cudaFuncSetAttribute(scat_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) ||
          cudaFuncSetAttribute(scat_k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
        return check_launch("route_sort: smem attribute", 0);
      cfg = smem;
    }
    hist_k<<<tiles, kSortThreads, E * sizeof(int32_t), stream>>>(ids, n, E, tiles, hist, (KT *)keys);
    sort_scan_kernel<<<E, 1024, 0, stream>>>(hist, tiles, totals);
    scat_k<<<tiles, kSortThreads, smem, stream>>>((const KT *)keys, n, E, tiles, hist, totals, sorted_scattered,
                                                  sorted_expert, inverse, offsets);
  } else {
    using KT = uint16_t;
    auto hist_k = per == 8 ? sort_hist_kernel<8, KT> : sort_hist_kernel<4, KT>;
    using ScatterFn = void (*)(const KT *, int64_t, int, int, const int32_t *, const int32_t *, int32_t *, int32_t *,
                               int32_t *, int32_t *);
    static const ScatterFn table[2][2] = {{sort_scatter_kernel<4, 8, KT>, sort_scatter_kernel<4, 10, KT>},
                                          {sort_scatter_kernel<8, 8, KT>, sort_scatter_kernel<8, 10, KT>}};
    const ScatterFn scat_k = table[per == 8][nbc == 4];
    static size_t configured[2][2] = {};
    size_t &cfg = configured[per == 8][nbc == 4];
    if (smem > cfg) {
      if ((smem > 48 * 1024 &&
           cudaFuncSetAttribute(scat_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) ||
          cudaFuncSetAttribute(scat_k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
        return check_launch("route_sort: smem attribute", 0);
      cfg = smem;
    }
    hist_k<<<tiles, kSortThreads, E * sizeof(int32_t), stream>>>(ids, n, E, tiles, hist, (KT *)keys);
    sort_scan_kernel<<<E, 1024, 0, stream>>>(hist, tiles, totals);
    scat_k<<<tiles, kSortThreads, smem, stream>>>((const KT *)keys, n, E, tiles, hist, totals, sorted_scattered,
                                                  sorted_expert, inverse, offsets);
  }
  return check_launch("route_sort", 3);
}

}  // namespace smoe
