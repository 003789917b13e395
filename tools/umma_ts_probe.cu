// Diagnostic: layout of the TMEM A operand of tcgen05.mma.kind::tf32 (TS form)
// and the N-concatenated B operand [B_hi ; B_lo] (2*BN rows, K-major).
// A[m][k] = m * 8 + k + 1 written with tcgen05.st.32x32b (lane m, column k);
// B[n][k] = (n % 8 == k) for n < 16 (two stacked 8-row identities), N = 16,
// so D[m][n] = A[m][n % 8] for n < 16 if lane = row and column = k.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/umma_ts_probe tools/umma_ts_probe.cu
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

constexpr int N = 16;

__global__ void probe(float *out) {
  __shared__ __align__(1024) float B[N * 8];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B K-major no-swizzle, R = N rows: chunk (row, k/4) at (k/4)*(N*16) + (row/8)*128 + (row%8)*16
  for (int i = t; i < N * 8; i += blockDim.x) {
    const int row = i / 8, k = i % 8;
    B[((k >> 2) * (N * 16) + (row >> 3) * 128 + (row & 7) * 16) / 4 + (k & 3)] = (row % 8 == k) ? 1.f : 0.f;
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  // A: columns 32..39 of lane (32 * warp + lane)
  {
    uint32_t r[8];
    const int m = 32 * warp + lane;
    for (int k = 0; k < 8; ++k) r[k] = __float_as_uint((float)(m * 8 + k + 1));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + ((uint32_t)(32 * warp) << 16) + 32),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    const uint64_t db = sdesc(su32(B), N * 16, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}" ::"r"(tmem),
        "r"(tmem + 32), "l"(db), "r"(0), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int m = 32 * warp + lane;
    for (int j = 0; j < 16; ++j) out[m * 16 + j] = __uint_as_float(r[j]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  float *d, h[128 * 16];
  cudaMalloc(&d, sizeof(h));
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      const float want = (float)(m * 8 + (n % 8) + 1);
      if (h[m * 16 + n] != want) {
        if (bad < 10) printf("m %d n %d got %.0f want %.0f\n", m, n, h[m * 16 + n], want);
        ++bad;
      }
    }
  printf("TS probe: %d mismatches of %d\n", bad, 128 * 16);
  for (int m = 0; m < 3; ++m) {
    for (int n = 0; n < 16; ++n) printf(" %5.0f", h[m * 16 + n]);
    printf("\n");
  }
  return 0;
}
