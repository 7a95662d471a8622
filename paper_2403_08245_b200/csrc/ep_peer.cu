// Expert-parallel dispatch / return over peer memory (NVLink / NVSwitch P2P).
//
// SURVEY.md §8(e) and §8(f)-2.  Instead of packing rows into a send buffer and
// calling an all-to-all, each rank stores its routed rows straight into the
// owning rank's receive buffer — already at their final position in the
// receiver's local grouped order (expert-major, then source rank, then source
// order), so the receiver runs its grouped GEMMs on the rows as they landed
// (TMA-fed, no group() copy) — and the expert outputs travel back the same way
// into the source's slot-ordered buffer.  Peer buffers are CUDA IPC mappings
// (smoe_ipc_*), so the same kernels run across GPUs (P2P over NVLink) and
// across processes sharing one GPU (the single-GPU test rig).
//
// Completion: a signal kernel (system-scope fence, then one atomic increment
// per peer on that peer's flag word for this source) and a wait kernel (spin
// on the local flags until every source reached the expected epoch, with a
// timeout that reports SMOE_ECUDA through an error word instead of hanging).
#include <cuda.h>

#include <cstring>

#include "common.cuh"

namespace smoe {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Dispatch: grouped row i of this rank -> (owner q, row j of q's receive
// buffer); dstart[e] = first receive row of (this source, global expert e) at
// the owner, i.e. its final position in the owner's local grouped order.
// Each CTA moves up to kRowsPerCta rows of ONE global expert; blockIdx.y walks
// the experts in (local expert, owner) order, so every owner receives its
// first local expert from every source first and its grouped GEMM can start on
// it while the later experts are still in flight.  After its rows (and their
// slot / source / routing-weight words) are stored, the CTA fences at system
// scope and adds its row count to the owner's arrival counter of that local
// expert (the GEMM producer's gate).  Rows that would land at or past
// `capacity` are not written: the overflow bit of *err is set instead.
constexpr int kRowsPerCta = 64;

template <typename T>
__global__ void __launch_bounds__(kThreads) dispatch_kernel(const T *__restrict__ x, int64_t d,
                                                            const int32_t *__restrict__ order,
                                                            const int32_t *__restrict__ bin_offsets, int E,
                                                            int fan_out, const float *__restrict__ weights,
                                                            const int64_t *__restrict__ dstart, int e_per_rank,
                                                            int world, const uint64_t *__restrict__ peer_rows,
                                                            const uint64_t *__restrict__ peer_slot,
                                                            const uint64_t *__restrict__ peer_src, int me,
                                                            const float *__restrict__ slot_p,
                                                            const uint64_t *__restrict__ peer_p, int64_t capacity,
                                                            const uint64_t *__restrict__ peer_arrive,
                                                            int32_t *__restrict__ err) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // CTA b -> chunk of an expert, experts ordered (local expert, owner): walk the
  // chunk counts ceil(count_e / kRowsPerCta) in that order
  __shared__ int s_e;
  __shared__ int64_t s_r0;
  if (threadIdx.x == 0) {
    int64_t b = blockIdx.x;
    s_e = -1;
    for (int jy = 0; jy < E; ++jy) {
      const int e = (jy % world) * e_per_rank + jy / world;
      const int64_t nch = (bin_offsets[e + 1] - bin_offsets[e] + kRowsPerCta - 1) / kRowsPerCta;
      if (b < nch) {
        s_e = e;
        s_r0 = bin_offsets[e] + b * kRowsPerCta;
        break;
      }
      b -= nch;
    }
  }
  __syncthreads();
  if (s_e < 0) return;
  const int e = s_e, q = e / e_per_rank, le = e - q * e_per_rank;
  const int64_t b0 = bin_offsets[e], b1 = bin_offsets[e + 1];
  const int64_t r0 = s_r0;
  const int64_t r1 = min(r0 + (int64_t)kRowsPerCta, b1);
  const int64_t base = dstart[e] - b0;
  T *rows = reinterpret_cast<T *>(peer_rows[q]);
  constexpr int N = 16 / sizeof(T);
  bool over = false;
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const int64_t j = base + i;
    if (j >= capacity) {
      over = true;
      continue;
    }
    const int32_t slot = order[i];
    const T *src = x + (int64_t)(slot / fan_out) * d;
    T *dst = rows + j * d;
    const float w = weights ? weights[slot] : 1.0f;
    for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N) {
      uint4 raw = __ldg(reinterpret_cast<const uint4 *>(src + c));
      if (weights) {
        T *v = reinterpret_cast<T *>(&raw);
#pragma unroll
        for (int u = 0; u < N; ++u) v[u] = Num<T>::from_f(Num<T>::to_f(v[u]) * w);
      }
      *reinterpret_cast<uint4 *>(dst + c) = raw;
    }
    if (lane == 0 && peer_slot) {
      reinterpret_cast<int32_t *>(peer_slot[q])[j] = slot;
      reinterpret_cast<int32_t *>(peer_src[q])[j] = me;
    }
    if (lane == 0 && peer_p) reinterpret_cast<float *>(peer_p[q])[j] = slot_p[slot];
  }
  if (over && lane == 0) atomicOr(err, 2);
  if (peer_arrive) {
    // every thread's row stores reach system scope before the CTA's count: a
    // fence orders only the calling thread's own writes, so each writer fences
    // (measured: with one fence in thread 0 the owner's first step could read
    // rows still in flight)
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
      atomicAdd_system(reinterpret_cast<unsigned long long *>(peer_arrive[q]) + le, (unsigned long long)(r1 - r0));
  }
}

// dp of received row j (sum of its partials, fixed order) -> the source's
// slot-ordered dp buffer
__global__ void dp_return_kernel(const float *__restrict__ part, int64_t n, int parts,
                                 const int32_t *__restrict__ recv_slot, const int32_t *__restrict__ recv_src,
                                 const uint64_t *__restrict__ peer_dp, const int32_t *__restrict__ n_valid) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (n_valid && j >= *n_valid)) return;
  const float *r = part + j * parts;
  float s = 0.0f;
  for (int u = 0; u < parts; ++u) s += r[u];
  reinterpret_cast<float *>(peer_dp[recv_src[j]])[recv_slot[j]] = s;
}

// local row j -> the source rank's slot-ordered buffer, row recv_slot[j]
template <typename T>
__global__ void __launch_bounds__(kThreads) return_kernel(const T *__restrict__ y, int64_t d, int64_t n,
                                                          const int32_t *__restrict__ recv_slot,
                                                          const int32_t *__restrict__ recv_src,
                                                          const uint64_t *__restrict__ peer_out,
                                                          const int32_t *__restrict__ n_valid) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (j >= n || (n_valid && j >= *n_valid)) return;
  const T *src = y + j * d;
  T *dst = reinterpret_cast<T *>(peer_out[recv_src[j]]) + (int64_t)recv_slot[j] * d;
  constexpr int N = 16 / sizeof(T);
  for (int64_t c = (int64_t)lane * N; c < d; c += 32 * N)
    *reinterpret_cast<uint4 *>(dst + c) = __ldg(reinterpret_cast<const uint4 *>(src + c));
}

// copy `bytes` (multiple of 4) to every peer at the same byte offset
__global__ void put_kernel(const uint32_t *__restrict__ src, int64_t words, const uint64_t *__restrict__ peer_dst,
                           int64_t offset_bytes) {
  uint32_t *dst = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(peer_dst[blockIdx.x]) + offset_bytes);
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
}

// Completion flags, one 64-bit word per (slot, source) on every rank, plus this
// rank's own per-slot signal count (`mine`, local memory).  Both sides keep
// their epochs on the device, so the signal / wait pair is stream-ordered and
// replays inside a CUDA graph: the wait completes when every source has
// signalled `slot` as many times as this rank has.
__global__ void signal_kernel(const uint64_t *__restrict__ peer_flags, int world, int me, int slot,
                              unsigned long long *__restrict__ mine) {
  const int q = threadIdx.x;
  if (q == 0) mine[slot] += 1ull;   // read only by this rank's later wait (same stream)
  if (q >= world) return;
  __threadfence_system();
  unsigned long long *f = reinterpret_cast<unsigned long long *>(peer_flags[q]) + (int64_t)slot * world + me;
  atomicAdd_system(f, 1ull);
}

__global__ void wait_kernel(const uint64_t *flags, int world, int slot, const unsigned long long *__restrict__ mine,
                            int64_t timeout_ns, int32_t *err) {
  const int s = threadIdx.x;
  if (s >= world) return;
  const unsigned long long target = mine[slot];
  const volatile unsigned long long *f =
      reinterpret_cast<const volatile unsigned long long *>(flags) + (int64_t)slot * world + s;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*f < target) {
    __nanosleep(256);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if ((int64_t)(t - t0) > timeout_ns) {
      atomicOr(err, 1);
      return;
    }
  }
  __threadfence_system();
}

// Capacity check of this rank's receive side: rows routed to it this step
// (the last local bin offset) against the receive buffer's rows.
__global__ void capacity_kernel(const int32_t *__restrict__ off_loc, int e_local, int64_t capacity,
                                int32_t *__restrict__ err) {
  if (threadIdx.x == 0 && (int64_t)off_loc[e_local] > capacity) atomicOr(err, 2);
}

inline unsigned row_blocks(int64_t rows) { return (unsigned)((rows + kWarps - 1) / kWarps); }
inline bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace

bool tc_available();
int tc_ep_scaled_gated(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *, const int32_t *,
                       int64_t, int, int, int, const float *, void *, void *, const void *, float *, int,
                       const unsigned long long *, cudaStream_t);
int tc_ep_group_xty_gated(const void *, const void *, const int32_t *, int, int64_t, int64_t, int64_t, void *,
                          const unsigned long long *, cudaStream_t);
int tc_scatter2scatter_peer(const void *, int64_t, const void *, int, int64_t, int64_t, const int32_t *,
                            const int32_t *, int64_t, int, const uint64_t *, const int32_t *, const int32_t *,
                            cudaStream_t);
}  // namespace smoe

using namespace smoe;

extern "C" {

size_t smoe_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int smoe_ipc_get_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return fail(SMOE_EINVAL, "ipc_get_handle: null pointer");
  // the handle names the whole allocation (a caching allocator hands out
  // sub-ranges): report where dev_ptr sits inside it
  using AddressRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
  static AddressRangeFn range_fn = nullptr;
  if (!range_fn) {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(SMOE_ECUDA, "cuMemGetAddressRange entry point unavailable");
    range_fn = (AddressRangeFn)fp;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return fail(SMOE_ECUDA, "cuMemGetAddressRange failed");
  *offset_out = (int64_t)((CUdeviceptr)dev_ptr - base);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr));
  if (e != cudaSuccess) return fail(SMOE_ECUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  return SMOE_OK;
}

int smoe_ipc_open(const void *handle, void **dev_ptr_out) {
  if (!handle || !dev_ptr_out) return fail(SMOE_EINVAL, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SMOE_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return SMOE_OK;
}

int smoe_ipc_close(void *dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return fail(SMOE_ECUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
  return SMOE_OK;
}

int smoe_ep_dispatch_rows(const void *x, int64_t x_rows, int64_t d, const int32_t *order,
                          const int32_t *bin_offsets, int32_t num_experts, int32_t fan_out, const float *weights,
                          int64_t n, const int64_t *dstart, int32_t experts_per_rank, int32_t world,
                          const uint64_t *peer_rows, const uint64_t *peer_slot, const uint64_t *peer_src, int32_t me,
                          const float *slot_p, const uint64_t *peer_p, int64_t capacity, const uint64_t *peer_arrive,
                          int32_t *err, int32_t dtype, void *stream) {
  if (fan_out < 1 || experts_per_rank < 1 || world < 1 || num_experts != experts_per_rank * world)
    return fail(SMOE_EINVAL, "ep_dispatch: fan_out >= 1 and num_experts == experts_per_rank * world");
  if ((slot_p == nullptr) != (peer_p == nullptr)) return fail(SMOE_EINVAL, "ep_dispatch: slot_p and peer_p go together");
  if (x_rows * fan_out != n) return fail(SMOE_ESHAPE, "ep_dispatch: x rows * fan_out must equal the slot count");
  if (n == 0 || d == 0) return SMOE_OK;
  if (!x || !order || !bin_offsets || !dstart || !peer_rows || !err)
    return fail(SMOE_EINVAL, "ep_dispatch: null pointer");
  if ((peer_slot == nullptr) != (peer_src == nullptr))
    return fail(SMOE_EINVAL, "ep_dispatch: peer_slot and peer_src go together");
  const size_t esz = dtype == SMOE_BF16 ? 2 : 4;
  if (!al16(x) || (d * (int64_t)esz) % 16) return fail(SMOE_ENOTSUP, "ep_dispatch: rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // one CTA per non-empty (expert, 64-row chunk): at most n / 64 + E of them
  const unsigned blocks = (unsigned)((n + kRowsPerCta - 1) / kRowsPerCta + num_experts);
  if (dtype == SMOE_BF16)
    dispatch_kernel<__nv_bfloat16><<<blocks, kThreads, 0, st>>>(
        (const __nv_bfloat16 *)x, d, order, bin_offsets, num_experts, fan_out, weights, dstart, experts_per_rank,
        world, peer_rows, peer_slot, peer_src, me, slot_p, peer_p, capacity, peer_arrive, err);
  else if (dtype == SMOE_F32)
    dispatch_kernel<float><<<blocks, kThreads, 0, st>>>((const float *)x, d, order, bin_offsets, num_experts, fan_out,
                                                        weights, dstart, experts_per_rank, world, peer_rows,
                                                        peer_slot, peer_src, me, slot_p, peer_p, capacity,
                                                        peer_arrive, err);
  else
    return fail(SMOE_EINVAL, "ep_dispatch: unsupported dtype");
  return check_launch("ep_dispatch_rows");
}

int smoe_ep_check_capacity(const int32_t *local_offsets, int32_t experts_per_rank, int64_t capacity, int32_t *err,
                           void *stream) {
  if (!local_offsets || !err || experts_per_rank < 1) return fail(SMOE_EINVAL, "ep_check_capacity: bad arguments");
  capacity_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(local_offsets, experts_per_rank, capacity,
                                                                         err);
  return check_launch("ep_check_capacity");
}

int smoe_ep_return_rows(const void *y, int64_t n, int64_t d, const int32_t *recv_slot, const int32_t *recv_src,
                        const uint64_t *peer_out, const int32_t *n_valid, int32_t dtype, void *stream) {
  if (n == 0 || d == 0) return SMOE_OK;
  if (!y || !recv_slot || !recv_src || !peer_out) return fail(SMOE_EINVAL, "ep_return: null pointer");
  const size_t esz = dtype == SMOE_BF16 ? 2 : 4;
  if (!al16(y) || (d * (int64_t)esz) % 16) return fail(SMOE_ENOTSUP, "ep_return: rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == SMOE_BF16)
    return_kernel<__nv_bfloat16><<<row_blocks(n), kThreads, 0, st>>>((const __nv_bfloat16 *)y, d, n, recv_slot,
                                                                       recv_src, peer_out, n_valid);
  else if (dtype == SMOE_F32)
    return_kernel<float><<<row_blocks(n), kThreads, 0, st>>>((const float *)y, d, n, recv_slot, recv_src, peer_out,
                                                             n_valid);
  else
    return fail(SMOE_EINVAL, "ep_return: unsupported dtype");
  return check_launch("ep_return_rows");
}

int smoe_ep_gemm_return(const void *x, int64_t n, const void *w, int32_t num_experts, int64_t w_rows, int64_t w_cols,
                        const int32_t *expert_offsets, int32_t transpose_w, const int32_t *recv_slot,
                        const int32_t *recv_src, const uint64_t *peer_out, void *stream) {
  if (n == 0) return SMOE_OK;
  if (!x || !w || !expert_offsets || !recv_slot || !recv_src || !peer_out)
    return fail(SMOE_EINVAL, "ep_gemm_return: null pointer");
  if (!tc_available()) return fail(SMOE_ENOTSUP, "ep_gemm_return: needs the tcgen05 engine");
  // grouped input: the order array is only read for scattered layouts; the
  // bin offsets drive the tile schedule
  return tc_scatter2scatter_peer(x, n, w, num_experts, w_rows, w_cols, recv_slot, expert_offsets, n, transpose_w,
                                 peer_out, recv_src, recv_slot, reinterpret_cast<cudaStream_t>(stream));
}

int smoe_ep_expert_gemm_gated(const void *x, int64_t n, const void *w, int32_t num_experts, int64_t w_rows,
                              int64_t w_cols, const int32_t *order, const int32_t *local_offsets, int32_t transpose_w,
                              int32_t epilogue,
                              int32_t activation, const float *row_scale, void *out, void *out2, const void *aux,
                              float *dp_part, int32_t dp_parts, const uint64_t *arrive, void *stream) {
  if (n == 0) return SMOE_OK;
  if (epilogue != SMOE_EPI_ACT_SCALED && epilogue != SMOE_EPI_ACT_GRAD_SCALED)
    return fail(SMOE_EINVAL, "ep_expert_gemm_gated takes SMOE_EPI_ACT_SCALED or SMOE_EPI_ACT_GRAD_SCALED");
  if (!x || !w || !order || !local_offsets || !row_scale || !out || !arrive)
    return fail(SMOE_EINVAL, "ep_expert_gemm_gated: null pointer");
  if (epilogue == SMOE_EPI_ACT_SCALED && !out2) return fail(SMOE_EINVAL, "ep_expert_gemm_gated: EPI_ACT_SCALED needs out2");
  if (epilogue == SMOE_EPI_ACT_GRAD_SCALED && !aux) return fail(SMOE_EINVAL, "ep_expert_gemm_gated: act-grad needs aux");
  if (!tc_available()) return fail(SMOE_ENOTSUP, "ep_expert_gemm_gated: needs the tcgen05 engine");
  return tc_ep_scaled_gated(x, n, w, num_experts, w_rows, w_cols, order, local_offsets, n, transpose_w,
                            epilogue, activation, row_scale, out, out2, aux, dp_part, dp_parts,
                            (const unsigned long long *)arrive, reinterpret_cast<cudaStream_t>(stream));
}

int smoe_ep_group_xty_gated(const void *xg, const void *yg, const int32_t *local_offsets, int32_t num_experts,
                            int64_t n, int64_t d_in, int64_t d_out, void *dw, const uint64_t *arrive_y, void *stream) {
  if (!xg || !yg || !local_offsets || !dw || !arrive_y) return fail(SMOE_EINVAL, "ep_group_xty_gated: null pointer");
  if (n == 0) return fail(SMOE_EINVAL, "ep_group_xty_gated: zero-capacity receive buffer");
  if (!tc_available()) return fail(SMOE_ENOTSUP, "ep_group_xty_gated: needs the tcgen05 engine");
  return tc_ep_group_xty_gated(xg, yg, local_offsets, num_experts, n, d_in, d_out, dw,
                               (const unsigned long long *)arrive_y, reinterpret_cast<cudaStream_t>(stream));
}

int smoe_ep_dp_return(const float *dp_part, int64_t n, int32_t parts, const int32_t *recv_slot,
                      const int32_t *recv_src, const uint64_t *peer_dp, const int32_t *n_valid, void *stream) {
  if (n == 0) return SMOE_OK;
  if (!dp_part || !recv_slot || !recv_src || !peer_dp || parts < 1) return fail(SMOE_EINVAL, "ep_dp_return: bad arguments");
  dp_return_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      dp_part, n, parts, recv_slot, recv_src, peer_dp, n_valid);
  return check_launch("ep_dp_return");
}

int smoe_ep_put(const void *src, int64_t bytes, const uint64_t *peer_dst, int64_t offset_bytes, int32_t world,
                void *stream) {
  if (bytes % 4 || offset_bytes % 4) return fail(SMOE_EINVAL, "ep_put: sizes must be multiples of 4 bytes");
  if (bytes == 0) return SMOE_OK;
  put_kernel<<<world, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>((const uint32_t *)src, bytes / 4, peer_dst,
                                                                         offset_bytes);
  return check_launch("ep_put");
}

int smoe_ep_signal(const uint64_t *peer_flags, int32_t world, int32_t me, int32_t slot, uint64_t *my_epochs,
                   void *stream) {
  if (world < 1 || world > 1024 || me < 0 || me >= world) return fail(SMOE_EINVAL, "ep_signal: bad rank");
  if (!my_epochs) return fail(SMOE_EINVAL, "ep_signal: null epoch array");
  signal_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(peer_flags, world, me, slot,
                                                                         (unsigned long long *)my_epochs);
  return check_launch("ep_signal");
}

int smoe_ep_wait(const uint64_t *flags, int32_t world, int32_t slot, const uint64_t *my_epochs, int64_t timeout_ns,
                 int32_t *err, void *stream) {
  if (world < 1 || world > 1024 || !err || !my_epochs) return fail(SMOE_EINVAL, "ep_wait: bad arguments");
  wait_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, world, slot,
                                                                       (const unsigned long long *)my_epochs,
                                                                       timeout_ns, err);
  return check_launch("ep_wait");
}

}  // extern "C"
