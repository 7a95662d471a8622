// Microbenchmark: CTA-pair tcgen05.mma.cta_group::2 (M=256 N=256 K=16) issue rate by
// operand major-ness while another warp streams bulk copies (global -> a separate
// shared region, ~the TMA fill traffic of the GEMM) into each CTA.  Random
// operand data.  One cluster of 2 CTAs per TPC.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int A_MN, int B_MN, int WRITER>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) bench(int iters, unsigned long long *out, const uint4 *gsrc, volatile int *stop_flag) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) {
    uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
    uint32_t v = 0x3c003c00u ^ (h & 0x03ff03ffu);  // bf16 values in [1, 2) with random mantissas... as pairs
    ((uint4 *)smem)[i] = make_uint4(v, v ^ 0x00010001u, v ^ 0x00050005u, v ^ 0x00110011u);
  }
  __shared__ uint64_t wbar[4];
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    s_stop = 0;
    for (int j = 0; j < 4; ++j) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar[j])));
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)A_MN << 15) | ((uint32_t)B_MN << 16) |
                         ((256u >> 3) << 17) | ((256u >> 4) << 24);
  if (WRITER && threadIdx.x == 32) {
    // stream into smem[32K, 64K) from an L2-resident buffer: 4 x 8 KB copies in flight
    const uint32_t dst = smem_u32(smem + 32768);
    uint32_t phase = 0;
    long long rounds = 0;
    for (int j = 0; j < 4; ++j) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wbar[j])), "r"(8192) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(dst + j * 8192),
                   "l"(gsrc + (size_t)blockIdx.x * 16384 + j * 512), "r"(smem_u32(&wbar[j])) : "memory");
    }
    while (!*(volatile int *)&s_stop && rounds < 100000000) {
      const int j = rounds & 3;
      asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D2;\nbra W2;\nD2:\n}\n" ::"r"(smem_u32(&wbar[j])), "r"(phase));
      if (j == 3) phase ^= 1;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wbar[j])), "r"(8192) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];" ::"r"(dst + j * 8192),
                   "l"(gsrc + (size_t)blockIdx.x * 16384 + ((rounds + 4) & 31) * 512), "r"(smem_u32(&wbar[j])) : "memory");
      ++rounds;
    }
    for (int j = 0; j < 4; ++j) {  // drain
      const int jj = (rounds + j) & 3;
      const uint32_t ph = ((rounds + j) >> 2) & 1;
      asm volatile("{\n.reg .pred P1;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D3;\nbra W3;\nD3:\n}\n" ::"r"(smem_u32(&wbar[jj])), "r"(ph));
    }
    if (rank == 0) out[128 + blockIdx.x / 2] = rounds / 4;
  }
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = A_MN ? sdesc(sa + k * 2048, 8192, 1024) : sdesc(sa + k * 32, 16, 1024);
        uint64_t bd = B_MN ? sdesc(sb + k * 2048, 8192, 1024) : sdesc(sb + k * 32, 16, 1024);
        uint32_t acc = (it | k) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)),
                 "h"((uint16_t)1));
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(&bar)));
    unsigned long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  }
  if (threadIdx.x == 0 && rank == 0) {
    s_stop = 1;
    // tell the peer's writer to stop too
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(remote) : "r"(smem_u32(&s_stop)));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(1) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int A, int B, int W>
void run(const char *name, int sms) {
  unsigned long long *d, h[256];
  cudaMalloc(&d, sizeof(h));
  uint4 *g;
  cudaMalloc(&g, (size_t)sms * 262144 + 65536);
  cudaMemset(g, 0x3c, (size_t)sms * 262144 + 65536);
  auto k = bench<A, B, W>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 66 * 1024>>>(iters, d, g, nullptr);
  k<<<sms, 128, 66 * 1024>>>(iters, d, g, nullptr);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms / 2; ++i) avg += h[i];
  avg /= (sms / 2);
  double wr = 0;
  for (int i = 0; i < sms / 2; ++i) wr += h[128 + i];
  wr /= (sms / 2);
  printf("cg2 %-22s writer=%d cycles/MMA = %.1f  (ideal 128)  writer B/clk per SM = %.1f  err=%s\n", name, W,
         avg / (iters * 4.0), W ? wr * 32768.0 / avg : 0.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(g);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 0, 0>("A K-major, B K-major", sms);
  run<0, 1, 0>("A K-major, B MN-major", sms);
  run<1, 0, 0>("A MN-major, B K-major", sms);
  run<1, 1, 0>("A MN-major, B MN-major", sms);
  run<0, 0, 1>("A K-major, B K-major", sms);
  run<0, 1, 1>("A K-major, B MN-major", sms);
  run<1, 0, 1>("A MN-major, B K-major", sms);
  run<1, 1, 1>("A MN-major, B MN-major", sms);
  return 0;
}
