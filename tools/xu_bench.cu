// Throughput microbenchmark for the instructions the engine kernels use most that
// are not plain ALU: POPC, FLO (__clz), BREV, I2F.F64 (int -> double), F2I, ballot/REDUX,
// SHFL. grid = 148 * ctas, block = 32 * warps; 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(unsigned* out, int iters, unsigned seed) {
  unsigned a[8];
  double d[8];
  for (int j = 0; j < 8; ++j) { a[j] = seed * (threadIdx.x + 7 * j + 1); d[j] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] += __popc(a[j] ^ i);
      if (OP == 1) a[j] += __clz(a[j] ^ i);
      if (OP == 2) a[j] += __brev(a[j] ^ i);
      if (OP == 3) d[j] += (double)(int)(a[j] ^ i), a[j] += 1;
      if (OP == 4) a[j] += __ballot_sync(0xffffffffu, (a[j] ^ i) & 1);
      if (OP == 5) a[j] += __reduce_add_sync(0xffffffffu, a[j] ^ i);
      if (OP == 6) a[j] += __shfl_xor_sync(0xffffffffu, a[j] ^ i, 1);
      if (OP == 7) a[j] = a[j] * 3 + i;
      if (OP == 8) a[j] += __ffs(a[j] ^ i);
      if (OP == 9) d[j] = __dadd_rn(d[j], 1.5);
    }
  }
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s += a[j] + (unsigned)d[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  unsigned* out;
  cudaMalloc(&out, 148 * 32 * 1024 * 4);
  const char* names[] = {"POPC", "FLO(clz)", "BREV", "I2F.F64", "VOTE(ballot)", "REDUX.add", "SHFL", "IMAD", "ffs", "DADD"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int warps_list[] = {1, 4, 8, 16};
  for (int op = 0; op < 10; ++op) {
    for (int wi = 0; wi < 4; ++wi) {
      int w = warps_list[wi];
      const int iters = 4096;
      auto launch = [&]() {
        switch (op) {
          case 0: k<0><<<148, 32 * w>>>(out, iters, 3); break;
          case 1: k<1><<<148, 32 * w>>>(out, iters, 3); break;
          case 2: k<2><<<148, 32 * w>>>(out, iters, 3); break;
          case 3: k<3><<<148, 32 * w>>>(out, iters, 3); break;
          case 4: k<4><<<148, 32 * w>>>(out, iters, 3); break;
          case 5: k<5><<<148, 32 * w>>>(out, iters, 3); break;
          case 6: k<6><<<148, 32 * w>>>(out, iters, 3); break;
          case 7: k<7><<<148, 32 * w>>>(out, iters, 3); break;
          case 8: k<8><<<148, 32 * w>>>(out, iters, 3); break;
          case 9: k<9><<<148, 32 * w>>>(out, iters, 3); break;
        }
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double per_sm_cycles = ms * 1e-3 * 1.965e9;
      double warp_ops_per_sm = (double)w * iters * 8;
      printf("%-13s warps/SM %2d: %6.2f SM-cycles per warp-instruction\n", names[op], w, per_sm_cycles / warp_ops_per_sm);
    }
  }
  return 0;
}
