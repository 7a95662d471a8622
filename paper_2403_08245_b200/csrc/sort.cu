// K1: stable counting sort of the flattened routing ids.
//
// Replaces router.compute_grouped_order (router.py:154-164):
//   o = argsort(flat, kind="stable"); counts = bincount(flat); offsets = [0, cumsum]
// Every key is an expert id in [0, E), so a single counting-sort digit suffices:
//   1. sort_hist:    per 4096-slot tile, a shared-memory histogram -> hist[e][tile]
//   2. sort_scan:    one block per expert scans its row of hist (tile-minor) to
//                    tile bases inside the expert's bin, and writes the bin size;
//                    (expert-major, tile-minor) is exactly the stable output order.
//   3. sort_scatter: every block rebuilds the bin starts from the E bin sizes,
//                    ranks its tile's slots stably (per-warp histograms over
//                    contiguous 512-slot chunks, equal-key lane masks from one
//                    ballot per key bit inside each 32-slot round), reorders the tile in shared memory and writes
//                    each expert's run contiguously (coalesced), plus the inverse
//                    permutation in slot order.
// Output order is the stable order (slots ascend inside each bin), bit-exact
// against numpy's stable argsort.
// HBM traffic: the int64 ids are read once (8 B per slot); the histogram pass
// also writes each slot's key in 1 byte (E < 256) or 2 bytes, which the scatter
// pass reads back — 16 MB at n = 16 M, L2-resident between the two passes —
// and three int32 outputs (12 B): ~20 B of DRAM traffic per slot.
#include "common.cuh"

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
