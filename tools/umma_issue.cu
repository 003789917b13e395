// Diagnostic: issue cost of a burst of kind::tf32 TS MMAs (M = 128, N = 64)
// from one thread, as a function of the CTA size and of alternating between
// two accumulators 256 columns apart (conv1 wgrad's M-tile layout).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/umma_issue tools/umma_issue.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void burst(long long *out, int n, int alt, int kspread) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < 64 * 200; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.5f;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    const uint32_t b_s = su32(sm);
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
      const int ks = kspread ? (i >> alt) % 24 : (i & 3);
      const int m = alt ? (i & 1) : 0;
      const uint64_t db = sdesc(b_s + ks * 2 * 64 * 16, 64 * 16, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem + m * 256),
          "r"(tmem + m * 256 + 64 + ks * 8), "l"(db), "r"(i > 1 ? 1 : 0), "r"(idesc));
    }
    long long c1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar)));
    long long c2 = clock64();
    out[blockIdx.x * 2] = c1 - c0;
    out[blockIdx.x * 2 + 1] = c2 - c0;
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long *d;
  cudaMalloc(&d, sizeof(long long) * 2 * 256);
  const int smem = 64 * 200 * 4;
  cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int threads : {128, 1024})
    for (int alt : {0, 1})
      for (int ksp : {0, 1})
        for (int n : {8, 25, 50}) {
          for (int rep = 0; rep < 2; ++rep) burst<<<64, threads, smem>>>(d, n, alt, ksp);
          cudaDeviceSynchronize();
          long long h[128];
          cudaMemcpy(h, d, sizeof(long long) * 128, cudaMemcpyDeviceToHost);
          double is = 0, dn = 0;
          for (int i = 0; i < 64; ++i) { is += h[2 * i]; dn += h[2 * i + 1]; }
          printf("threads %4d alt %d kspread %d n %2d: issue %6.0f cyc (%5.1f/MMA), done %6.0f cyc\n", threads,
                 alt, ksp, n, is / 64, is / 64 / n, dn / 64);
        }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
