// Diagnostic: which shared-memory word does tcgen05.mma.kind::tf32 read for
// B(n, k) under a given descriptor?  A[m][k] = (m == k) for m < 8 (K-major,
// the known-good layout), B smem word w holds float(w), so D[k][n] = index of
// the word read for B(n, k).
// nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/umma_probe tools/umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

constexpr int N = 32;

__global__ void probe(float *out, uint32_t lbo, uint32_t sbo, int b_mn) {
  __shared__ __align__(1024) float A[128 * 8];
  __shared__ __align__(1024) float B[2048];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  // A K-major no-swizzle: chunk (row, k/4) at (k/4)*(128*16) + (row/8)*128 + (row%8)*16
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int row = i / 8, k = i % 8;
    const int off = ((k >> 2) * (128 * 16) + (row >> 3) * 128 + (row & 7) * 16) / 4 + (k & 3);
    A[off] = (row < 8 && row == k) ? 1.f : 0.f;
  }
  for (int i = t; i < 2048; i += blockDim.x) B[i] = (float)(i + 1);   // 0 = read outside B
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)b_mn << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = sdesc(su32(A), 128 * 16, 128);
    const uint64_t db = b_mn ? sdesc(su32(B), lbo, sbo) : sdesc(su32(B), N * 16, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t < 32) {   // warp 0: lanes 0..31 = rows 0..31; read 32 columns
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) out[t * 32 + j] = __uint_as_float(r[j]);
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  float *d, h[32 * 32];
  cudaMalloc(&d, sizeof(h));
  const uint32_t vals[] = {16, 32, 64, 128, 256, 512, 1024};
  // K-major reference first
  probe<<<1, 128>>>(d, 0, 0, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("K-major: k0 n0..7:");
  for (int n = 0; n < 8; ++n) printf(" %.0f", h[n]);
  printf("\n");
  for (uint32_t lbo : vals)
    for (uint32_t sbo : vals) {
      probe<<<1, 128>>>(d, lbo, sbo, 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("lbo %4u sbo %4u |", lbo, sbo);
      for (int k = 0; k < 8; k += 1) {
        for (int n = 0; n < 9; ++n) printf(" %.0f", h[k * 32 + n]);
        printf(" |");
      }
      printf(" n16..19@k0: %.0f %.0f %.0f %.0f\n", h[16], h[17], h[18], h[19]);
    }
  return 0;
}
