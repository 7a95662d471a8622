// K1: stable counting sort of the flattened routing ids.
//
// Replaces router.compute_grouped_order (router.py:154-164):
//   o = argsort(flat, kind="stable"); counts = bincount(flat); offsets = [0, cumsum]
// Every key is an expert id in [0, E), so a single counting-sort digit suffices:
//   1. sort_hist:    per 4096-slot tile, a shared-memory histogram -> hist[e][tile]
//   2. sort_scan:    exclusive scan of hist in (expert-major, tile-minor) order;
//                    that order is exactly the stable order of the output, so
//                    base[e][tile] is where tile's first e-slot lands.
//   3. sort_scatter: each warp owns a contiguous 512-slot chunk of the tile; the
//                    in-warp rank among equal ids comes from __match_any_sync,
//                    the cross-warp offset from a per-tile warp histogram.
// Output order is the stable order (slots ascend inside each bin), bit-exact
// against numpy's stable argsort.
#include "common.cuh"

namespace smoe {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortPerThread = 16;
constexpr int kSortTile = kSortThreads * kSortPerThread;  // 4096 slots
constexpr int kSortMaxExperts = 1024;

__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const int64_t *__restrict__ ids,
                                                                 int64_t n, int E, int num_tiles,
                                                                 int32_t *__restrict__ hist) {
  extern __shared__ int32_t s_hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortPerThread; ++r) {
    int64_t i = base + (int64_t)r * kSortThreads + threadIdx.x;
    if (i < n) {
      int64_t key = ids[i];
      if (key >= 0 && key < E) atomicAdd(&s_hist[key], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[(int64_t)e * num_tiles + blockIdx.x] = s_hist[e];
}

// Single-block exclusive scan over E*num_tiles counts (expert-major).
__global__ void __launch_bounds__(1024) sort_scan_kernel(int32_t *__restrict__ hist, int64_t total,
                                                         int E, int num_tiles, int64_t n,
                                                         int32_t *__restrict__ offsets) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t chunk = 0; chunk < total; chunk += blockDim.x) {
    int64_t i = chunk + threadIdx.x;
    int32_t v = i < total ? hist[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    int32_t carry = s_carry;
    int32_t excl = carry + (warp > 0 ? s_warp[warp - 1] : 0) + x - v;
    if (i < total) {
      hist[i] = excl;
      if (i % num_tiles == 0) offsets[i / num_tiles] = excl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[E] = (int32_t)n;
}

__global__ void __launch_bounds__(kSortThreads) sort_scatter_kernel(
    const int64_t *__restrict__ ids, int64_t n, int E, int num_tiles,
    const int32_t *__restrict__ base, int32_t *__restrict__ sorted_scattered,
    int32_t *__restrict__ sorted_expert, int32_t *__restrict__ inverse) {
  extern __shared__ int32_t s_cnt[];  // [kSortWarps][E]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();

  const int64_t chunk0 = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * (32 * kSortPerThread);
  int32_t keys[kSortPerThread];
  // Pass 1: per-warp histogram of this warp's contiguous chunk.
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    int64_t i = chunk0 + r * 32 + lane;
    int32_t key = -1;
    if (i < n) {
      int64_t k64 = ids[i];
      key = (k64 >= 0 && k64 < E) ? (int32_t)k64 : -1;
    }
    keys[r] = key;
    unsigned peers = __match_any_sync(0xffffffffu, key);
    int leader = __ffs(peers) - 1;
    if (key >= 0 && lane == leader) s_cnt[warp * E + key] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Exclusive scan across warps per expert, seeded with the tile's global base.
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = base[(int64_t)e * num_tiles + blockIdx.x];
    for (int w = 0; w < kSortWarps; ++w) {
      int32_t c = s_cnt[w * E + e];
      s_cnt[w * E + e] = run;
      run += c;
    }
  }
  __syncthreads();
  // Pass 2: stable rank inside each 32-slot round, then bump the running base.
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    int32_t key = keys[r];
    unsigned peers = __match_any_sync(0xffffffffu, key);
    int leader = __ffs(peers) - 1;
    if (key >= 0) {
      int32_t pos = s_cnt[warp * E + key] + __popc(peers & lt_mask);
      int32_t slot = (int32_t)(chunk0 + r * 32 + lane);
      sorted_scattered[pos] = slot;
      if (sorted_expert) sorted_expert[pos] = key;
      if (inverse) inverse[slot] = pos;
    }
    __syncwarp();
    if (key >= 0 && lane == leader) s_cnt[warp * E + key] += __popc(peers);
    __syncwarp();
  }
}

size_t route_sort_workspace(int64_t n, int E) {
  int64_t tiles = (n + kSortTile - 1) / kSortTile;
  if (tiles < 1) tiles = 1;
  return (size_t)(tiles * E) * sizeof(int32_t);
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
  int tiles = (int)((n + kSortTile - 1) / kSortTile);
  if (tiles == 0) {
    // Empty routing: offsets are all zero.
    cudaMemsetAsync(offsets, 0, sizeof(int32_t) * (E + 1), stream);
    return check_launch("route_sort(empty)", 0);
  }
  sort_hist_kernel<<<tiles, kSortThreads, E * sizeof(int32_t), stream>>>(ids, n, E, tiles, hist);
  sort_scan_kernel<<<1, 1024, 0, stream>>>(hist, (int64_t)tiles * E, E, tiles, n, offsets);
  sort_scatter_kernel<<<tiles, kSortThreads, kSortWarps * E * sizeof(int32_t), stream>>>(
      ids, n, E, tiles, hist, sorted_scattered, sorted_expert, inverse);
  return check_launch("route_sort", 3);
}

}  // namespace smoe
