// Dependent-load latency on one warp (lane 0 chases, others idle): global L1-resident,
// global after a store to the line, global L2-resident (working set > L1), shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* a, int n, int iters, int mode, long long* out) {
  __shared__ int s[4096];
  for (int i = threadIdx.x; i < n; i += 32) a[i] = (int)(((long long)i * 7919 + 4099) % n);
  for (int i = threadIdx.x; i < 4096; i += 32) s[i] = (i * 97 + 31) & 4095;
  __syncwarp();
  int v = 0;
  for (int i = 0; i < 2 * n / 32 + 64; ++i) v = (mode == 3) ? s[v] : a[v];  // warm
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 1 && threadIdx.x == 0) a[v] = a[v];
    v = (mode == 3) ? s[v] : a[v];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  if (v == -1) out[1] = v;
}
int main() {
  int* a; long long* o; long long h[2];
  cudaMalloc(&a, 64 << 20); cudaMalloc(&o, 16);
  const char* names[] = {"global L1-resident (16 KB)", "global L1 + store to same word", "global 64 KB", "shared"};
  int ns[] = {4096, 4096, 16384, 4096};
  for (int m = 0; m < 4; ++m) {
    k<<<1, 32>>>(a, ns[m], 20000, m, o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("%-36s %lld cycles/load\n", names[m], h[0]);
  }
  int big[] = {1 << 16, 1 << 18, 1 << 20, 1 << 22};
  for (int b : big) {
    k<<<1, 32>>>(a, b, 20000, 2, o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("global working set %8d KB            %lld cycles/load\n", b * 4 / 1024, h[0]);
  }
  return 0;
}
