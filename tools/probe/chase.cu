// L2 / DRAM load latency: one thread chases a pointer chain (ld.global.cg) through a buffer
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chase(const unsigned* __restrict__ next, int steps, unsigned long long* out, unsigned* sink) {
  unsigned i = 0;
  unsigned long long a, b;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b) : "r"(i));
  out[0] = b - a;
  sink[0] = i;
}
__global__ void fill(unsigned* next, unsigned n, unsigned stride) {
  for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    next[j] = (j + stride) % n;
}
__global__ void stream(const uint4* x, size_t n, unsigned* sink) {   // evicts L2
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    uint4 v = __ldcs(x + j);
    acc.x ^= v.x;
  }
  if (acc.x == 12345) sink[1] = acc.x;
}
int main() {
  const unsigned n = 1 << 22;   // 16 MB buffer
  unsigned *next, *sink;
  unsigned long long* out;
  uint4* big;
  size_t bigN = (size_t)1 << 28;  // 4 GB
  cudaMalloc(&next, n * 4); cudaMalloc(&sink, 16); cudaMalloc(&out, 8); cudaMalloc(&big, bigN * 16);
  cudaMemset(big, 0, bigN * 16);
  fill<<<1024, 256>>>(next, n, 4099);   // stride of 16 KB + 12 B: a new line every step
  unsigned long long h;
  for (int rep = 0; rep < 2; ++rep) {
    chase<<<1, 1>>>(next, 2000, out, sink);   // first pass: DRAM (cold) then warm
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("chase pass %d: %.1f ns per load\n", rep, h / 2000.0);
  }
  stream<<<148 * 8, 256>>>(big, bigN, sink);
  chase<<<1, 1>>>(next, 2000, out, sink);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("chase after a 4 GB stream: %.1f ns per load\n", h / 2000.0);
  chase<<<1, 1>>>(next, 2000, out, sink);
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("chase again: %.1f ns per load\n", h / 2000.0);
  return 0;
}
