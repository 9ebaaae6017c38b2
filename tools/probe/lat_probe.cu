// microbenchmark: latency of dependent fp64 ops and warp shuffles on one thread / one warp
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  unsigned long long a, b;
  // dependent DADD chain
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  for (int i = 0; i < n; ++i) x = x + 1.000001;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b) : "d"(x));
  if (threadIdx.x == 0) t[0] = b - a;
  // dependent sqrt chain
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a) : "d"(x));
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b) : "d"(x));
  if (threadIdx.x == 0) t[1] = b - a;
  // dependent division chain
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a) : "d"(x));
  for (int i = 0; i < n; ++i) x = 3.0 / x + 1.0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b) : "d"(x));
  if (threadIdx.x == 0) t[2] = b - a;
  // dependent shuffle+add chain
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a) : "d"(x));
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 << (i % 5));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b) : "d"(x));
  if (threadIdx.x == 0) t[3] = b - a;
  // bar.sync chain (8 warps)
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a) : "d"(x));
  for (int i = 0; i < n; ++i) __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
  if (threadIdx.x == 0) t[4] = b - a;
  // globaltimer back-to-back
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
  if (threadIdx.x == 0) t[5] = b - a;
  out[threadIdx.x] = x;
}
int main() {
  double* o; unsigned long long* t;
  cudaMalloc(&o, 256 * 8); cudaMalloc(&t, 64);
  unsigned long long h[6];
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 256>>>(o, t, 2.0, 1000);
    cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
    printf("per op ns: dadd %.2f sqrt %.2f div %.2f shfl+dadd %.2f bar %.2f | timer b2b %llu ns\n", h[0] / 1000.0,
           h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0, h[5]);
  }
  return 0;
}
