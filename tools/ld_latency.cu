// Diagnostic: global-load latency and burst time on the B200 for data that
// is L2-resident (a 4 MB buffer touched just before).
//  1. pointer chase (one thread): ns per dependent load, __ldg vs plain;
//  2. burst: 148 CTAs x 512 threads each load 4 x 16 B (LDG.128) at
//     scattered 64 B rows and use them -- time from kernel entry to the
//     last use (globaltimer), like the first k-block of a GEMM tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/bin/ld_latency tools/ld_latency.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool NC>
__global__ void chase(const unsigned *p, int n, unsigned long long *out) {
  unsigned i = 0;
  const unsigned long long t0 = gt();
  for (int k = 0; k < n; ++k) i = NC ? __ldg(p + i) : p[i];
  const unsigned long long t1 = gt();
  out[0] = t1 - t0;
  out[1] = i;
}

template <bool NC>
__global__ void burst(const float4 *src, int rows, unsigned long long *out, float *sink) {
  const unsigned long long t0 = gt();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (g * 7919) % rows;         // scattered 64-byte rows
  const float4 *q = src + (size_t)row * 4;
  float4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = NC ? __ldg(q + j) : q[j];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += v[j].x + v[j].y + v[j].z + v[j].w;
  __syncthreads();
  const unsigned long long t1 = gt();
  if (s == 12345.f) sink[g] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const int n = 1 << 20;                      // 4 MB of u32
  unsigned *h = new unsigned[n];
  // random cyclic permutation with 64-byte stride between hops
  const int lines = n / 16;
  int *perm = new int[lines];
  for (int i = 0; i < lines; ++i) perm[i] = i;
  unsigned s = 12345;
  for (int i = lines - 1; i > 0; --i) {
    s = s * 1103515245u + 12345u;
    const int j = s % (i + 1);
    const int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  for (int i = 0; i < lines; ++i) h[perm[i] * 16] = perm[(i + 1) % lines] * 16;
  unsigned *d;
  unsigned long long *o, ho[256];
  float *sink;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  const int hops = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    chase<true><<<1, 1>>>(d, hops, o);
    cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
    printf("chase __ldg : %.1f ns per dependent load\n", (double)ho[0] / hops);
    chase<false><<<1, 1>>>(d, hops, o);
    cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
    printf("chase plain : %.1f ns per dependent load\n", (double)ho[0] / hops);
  }
  for (int rep = 0; rep < 3; ++rep) {
    burst<true><<<148, 512>>>((const float4 *)d, n / 16, o, sink);
    cudaMemcpy(ho, o, 148 * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sum = 0;
    for (int i = 0; i < 148; ++i) { mx = ho[i] > mx ? ho[i] : mx; sum += ho[i]; }
    printf("burst __ldg : mean %.2f us max %.2f us (entry -> all 64 B used, per CTA)\n", sum / 148e3, mx / 1e3);
    burst<false><<<148, 512>>>((const float4 *)d, n / 16, o, sink);
    cudaMemcpy(ho, o, 148 * 8, cudaMemcpyDeviceToHost);
    mx = 0; sum = 0;
    for (int i = 0; i < 148; ++i) { mx = ho[i] > mx ? ho[i] : mx; sum += ho[i]; }
    printf("burst plain : mean %.2f us max %.2f us\n", sum / 148e3, mx / 1e3);
  }
  return 0;
}
