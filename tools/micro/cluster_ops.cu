// Latency of the primitives the pipelined cluster kernel's routing warp uses, on one warp of
// rank 0 of a 2-CTA cluster (clock64 around N repetitions): MEMBAR.ALL.CTA (the
// sync_restrict release) alone / after a remote (DSMEM) store / after a global load in
// flight; a remote relaxed store; a remote relaxed load round trip; a dependent 64-bit
// warp minimum (two CREDUX); match_any; a shuffle chain.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_ops tools/micro/cluster_ops.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ void rel() { asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory"); }
__global__ void __cluster_dims__(2, 1, 1) k(const double* g, long long* out, int iters) {
  __shared__ unsigned long long buf[64];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x & 63] = 0;
  cl.sync();
  unsigned long long* remote = cl.map_shared_rank(buf, 1);
  if (cl.block_rank() == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long t0, r[8];
    unsigned long long acc = 0;
    // 0: release alone
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { buf[lane] = i; rel(); }
    r[0] = (clock64() - t0) / iters;
    // 1: release after a remote store
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile("st.relaxed.cluster.u64 [%0], %1;" ::"l"(remote + lane), "l"((unsigned long long)i) : "memory");
      rel();
    }
    r[1] = (clock64() - t0) / iters;
    // 2: release after a global load in flight (value used after the fence)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      double v = g[(i * 4099 + lane * 131) & ((1 << 22) - 1)];
      rel();
      acc += (unsigned long long)v;
    }
    r[2] = (clock64() - t0) / iters;
    // 3: remote store issue only
    t0 = clock64();
    for (int i = 0; i < iters; ++i)
      asm volatile("st.relaxed.cluster.u64 [%0], %1;" ::"l"(remote + lane), "l"((unsigned long long)i) : "memory");
    r[3] = (clock64() - t0) / iters;
    // 4: remote load round trip (dependent chain)
    unsigned long long x = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      unsigned long long v;
      asm volatile("ld.relaxed.cluster.u64 %0, [%1];" : "=l"(v) : "l"(remote + ((lane + x) & 31)) : "memory");
      x += v & 1;
    }
    r[4] = (clock64() - t0) / iters;
    // 5: dependent 64-bit warp minimum (two CREDUX + compare/select)
    unsigned long long key = (unsigned long long)lane * 0x9E3779B97F4A7C15ULL;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)(key >> 32));
      const unsigned lo = __reduce_min_sync(0xffffffffu, (unsigned)(key >> 32) == hi ? (unsigned)key : 0xffffffffu);
      key += ((unsigned long long)hi << 32 | lo) & 1;
    }
    r[5] = (clock64() - t0) / iters;
    // 6: match_any chain
    unsigned m = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) m = __match_any_sync(0xffffffffu, m & 7) + lane;
    r[6] = (clock64() - t0) / iters;
    // 7: shuffle chain
    int s = lane;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __shfl_sync(0xffffffffu, s, (s + 1) & 31);
    r[7] = (clock64() - t0) / iters;
    if (lane == 0) for (int j = 0; j < 8; ++j) out[j] = r[j];
    if (acc == 12345 && m == 1 && s == 7 && key == 3 && x == 9) out[9] = 1;
  }
  cl.sync();
}
int main() {
  double* g; long long* o; long long h[10];
  cudaMalloc(&g, 8 << 22); cudaMemset(g, 0, 8 << 22); cudaMalloc(&o, 80);
  k<<<2, 64>>>(g, o, 2000);
  k<<<2, 64>>>(g, o, 2000);
  cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
  const char* names[] = {"release (MEMBAR.ALL.CTA) after a local STS", "release after a remote (DSMEM) store",
                         "release with a global load in flight", "remote relaxed store, issue",
                         "remote relaxed load round trip", "64-bit warp min (2x CREDUX) chain",
                         "match_any chain", "shfl chain"};
  for (int j = 0; j < 8; ++j) printf("%-46s %6lld cycles\n", names[j], h[j]);
  return 0;
}
