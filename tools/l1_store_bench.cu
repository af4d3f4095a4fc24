// Latency of a dependent global load chain through L1 (1 warp), with and without a
// store to the same line before each load: does a global store invalidate the L1 line?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* a, int iters, int mode, long long* out) {
  int idx = threadIdx.x;
  for (int i = 0; i < 4096; i += 32) a[i + threadIdx.x] = (i + threadIdx.x + 32) & 4095;  // a[x] -> next chunk
  __syncwarp();
  int v = a[idx];  // warm
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 1 && threadIdx.x == 0) a[(v & ~31) + 31] = a[(v & ~31) + 31];  // store into the line we read next
    if (mode == 2 && threadIdx.x == 0) a[((v + 2048) & 4095)] = 7;             // store elsewhere
    __syncwarp();
    v = a[v];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[mode] = (t1 - t0) / iters;
  if (v == -1) out[3] = v;
}
int main() {
  int* a; long long* o; long long h[4];
  cudaMalloc(&a, 4096 * 4); cudaMalloc(&o, 32);
  for (int m = 0; m < 3; ++m) k<<<1, 32>>>(a, 10000, m, o);
  cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  printf("dependent ld.global chain (L1-resident 16 KB): %lld cycles/iter; with a store to the next line: %lld; "
         "with a store elsewhere: %lld\n", h[0], h[1], h[2]);
  return 0;
}
