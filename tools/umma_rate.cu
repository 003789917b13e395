// Diagnostic: tcgen05.mma.kind::tf32 throughput per SM, A from shared memory
// (SS) vs A from tensor memory (TS), M = 128, N in {32, 64, 128, 256}.
// One CTA per SM on all SMs, each issuing `iters` MMAs into one accumulator;
// reports cycles per MMA and the implied dense TF32 TFLOP/s of the GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/umma_rate tools/umma_rate.cu
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

template <int N, bool TS>
__global__ void rate(long long *cycles, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < (128 * 32 + N * 32); i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.5f;
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    const uint32_t a_s = su32(sm), b_s = a_s + 128 * 32 * 4;
    const uint32_t a_t = tmem + 256;        // A in TMEM columns 256..287 (contents irrelevant)
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      const uint64_t db = sdesc(b_s + ks * 2 * N * 16, N * 16, 128);
      if (TS) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem),
            "r"(a_t + ks * 8), "l"(db), "r"(i), "r"(idesc));
      } else {
        const uint64_t da = sdesc(a_s + ks * 2 * 128 * 16, 128 * 16, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(i));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar)));
    cycles[blockIdx.x] = clock64() - c0;
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS>
void run(long long *d, int sms, int iters = 4096) {
  const int smem = (128 * 32 + N * 32) * 4;
  cudaFuncSetAttribute(rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate<N, TS><<<sms, 128, smem>>>(d, iters);
  rate<N, TS><<<sms, 128, smem>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cpm = mx / iters;
  const double flop = 2.0 * 128 * N * 8;
  if (iters < 4096) {      // latency mode: issue of `iters` MMAs -> their commit observed
    printf("%s N=%3d : %5d MMAs issued -> completion seen after %7.0f cycles (%.2f us)\n",
           TS ? "TS" : "SS", N, iters, mx, mx / 1965.0);
    return;
  }
  printf("%s N=%3d : %6.1f cycles/MMA  -> %7.1f TFLOP/s tf32 at 1.965 GHz x %d SMs\n", TS ? "TS" : "SS", N,
         cpm, flop / cpm * 1.965e9 * sms / 1e12, sms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *d;
  cudaMalloc(&d, sizeof(long long) * 1024);
  run<32, false>(d, sms);
  run<64, false>(d, sms);
  run<128, false>(d, sms);
  run<256, false>(d, sms);
  run<32, true>(d, sms);
  run<64, true>(d, sms);
  run<128, true>(d, sms);
  run<256, true>(d, sms);
  // latency: one CTA, a short burst of MMAs, issue -> commit arrival
  for (int n : {1, 2, 4, 8, 16, 32, 64}) run<64, true>(d, 1, n);
  for (int n : {1, 8, 16}) run<128, false>(d, 1, n);
  return 0;
}
