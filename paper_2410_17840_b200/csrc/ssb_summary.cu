// ssb_summary.cu — exact Summary (metrics.py:80-99) of many record groups on the device.
//
// Nearest-rank percentiles (metrics.py:46-54: sorted(values)[ceil(p/100*n)-1])
// are computed exactly with a most-significant-digit radix select on the
// order-preserving 64-bit image of each binary64 value: 8 passes of 8-bit
// digits, each pass a shared-memory histogram per (group, rank slot) over the
// elements whose key matches the slot's current prefix, then one thread per
// slot picks the digit holding rank k. No sort, O(8 N) element reads.
//
// Per record (all binary64, same operation order as the reference):
//   arrival   = arrival_trace / qps_factor              (workload.py:193)
//   ttft      = first_token - arrival                   (metrics.py:34-35)
//   norm_ttft = ttft / prompt_len                       (:37-39)
//   gen_time  = finish - arrival                        (:41-43)
//   tpot      = (finish - first_token) / (output - 1), output > 1   [north-star extra]
//   queue     = first_dispatch - arrival                            [north-star extra]
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/ssb.h"

namespace {

constexpr int NSLOT = 13;  // ttft 50/95/99, norm 50/95, gen 50/95, tpot 50/95/99, queue 50/95/99
constexpr int CHUNK = 4096;
constexpr int THREADS = 256;
__constant__ int SLOT_STAT[NSLOT] = {0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 4, 4, 4};

struct GroupWork {
  unsigned long long prefix[NSLOT];
  long long k[NSLOT];  // remaining rank (1-based) within the prefix bucket
  unsigned hist[NSLOT][256];
  long long n_tpot;
  long long n_pre;
  unsigned long long max_fin_key;  // dkey(max finish)
  unsigned long long min_arr_key;  // dkey(min arrival)
};

__device__ __forceinline__ unsigned long long dkey(double x) {
  long long b = __double_as_longlong(x);
  return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ void element_keys(const ssb_summary_group& G, ssb_trace tr, ssb_records rec, long long i,
                                             unsigned long long key[5], bool& has_tpot) {
  const long long t = G.trace_offset + i, r = G.record_offset + i;
  double arr = tr.arrival[t];
  if (G.qps_factor != 1.0) arr = __ddiv_rn(arr, G.qps_factor);
  const double ft = rec.first_token[r], fin = rec.finish[r];
  const int prompt = tr.prompt[t], out = tr.output[t];
  const double ttft = __dsub_rn(ft, arr);
  key[0] = dkey(ttft);
  key[1] = dkey(__ddiv_rn(ttft, (double)prompt));
  key[2] = dkey(__dsub_rn(fin, arr));
  has_tpot = out > 1;
  key[3] = has_tpot ? dkey(__ddiv_rn(__dsub_rn(fin, ft), (double)(out - 1))) : 0ULL;
  key[4] = dkey(__dsub_rn(rec.first_dispatch[r], arr));
}

// one statistic's key (element_keys' operations for that statistic only); ~0 (sorts last) for a
// record without a TPOT (output 1)
__device__ __forceinline__ unsigned long long stat_key(const ssb_summary_group& G, ssb_trace tr, ssb_records rec,
                                                       long long i, int st) {
  const long long t = G.trace_offset + i, r = G.record_offset + i;
  if (st == 3) {
    const int out = tr.output[t];
    if (out <= 1) return ~0ULL;
    return dkey(__ddiv_rn(__dsub_rn(rec.finish[r], rec.first_token[r]), (double)(out - 1)));
  }
  double arr = tr.arrival[t];
  if (G.qps_factor != 1.0) arr = __ddiv_rn(arr, G.qps_factor);
  if (st == 2) return dkey(__dsub_rn(rec.finish[r], arr));
  if (st == 4) return dkey(__dsub_rn(rec.first_dispatch[r], arr));
  const double ttft = __dsub_rn(rec.first_token[r], arr);
  return st == 0 ? dkey(ttft) : dkey(__ddiv_rn(ttft, (double)tr.prompt[t]));
}

// chunk c -> (group, element range) through the prefix array cstart[]
__device__ __forceinline__ int find_group(const long long* cstart, int n_groups, long long c) {
  int lo = 0, hi = n_groups - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cstart[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_init(const ssb_summary_group* __restrict__ groups, int n_groups, GroupWork* __restrict__ work) {
  for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
    GroupWork& W = work[g];
    for (int i = threadIdx.x; i < NSLOT * 256; i += blockDim.x) (&W.hist[0][0])[i] = 0u;
    if (threadIdx.x < NSLOT) {
      W.prefix[threadIdx.x] = 0ULL;
      W.k[threadIdx.x] = threadIdx.x < 7 ? groups[g].rank[threadIdx.x < 3 ? threadIdx.x : (threadIdx.x < 5 ? threadIdx.x - 3 : threadIdx.x - 5)] : 0;
    }
    if (threadIdx.x == 0) {
      W.n_tpot = 0; W.n_pre = 0; W.max_fin_key = 0ULL; W.min_arr_key = ~0ULL;
    }
  }
}

__global__ void __launch_bounds__(THREADS) k_hist(ssb_trace tr, ssb_records rec,
                                                  const ssb_summary_group* __restrict__ groups, int n_groups,
                                                  const long long* __restrict__ cstart, long long n_chunks,
                                                  GroupWork* __restrict__ work, int pass) {
  __shared__ unsigned hist[NSLOT][256];
  __shared__ unsigned long long s_prefix[NSLOT];
  __shared__ int s_active[NSLOT];
  const int shift = 56 - 8 * pass;
  for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int g = find_group(cstart, n_groups, c);
    const ssb_summary_group G = groups[g];
    GroupWork& W = work[g];
    for (int i = threadIdx.x; i < NSLOT * 256; i += blockDim.x) (&hist[0][0])[i] = 0u;
    if (threadIdx.x < NSLOT) {
      s_prefix[threadIdx.x] = W.prefix[threadIdx.x];
      s_active[threadIdx.x] = W.k[threadIdx.x] > 0;
    }
    __syncthreads();
    const long long e0 = (c - cstart[g]) * CHUNK;
    const long long e1 = (e0 + CHUNK < G.n) ? e0 + CHUNK : G.n;
    long long n_tpot = 0, n_pre = 0;
    unsigned long long mfin = 0ULL, marr = ~0ULL;
    const unsigned long long hmask = pass == 0 ? 0ULL : (~0ULL << (shift + 8));
    for (long long i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
      unsigned long long key[5];
      bool has_tpot;
      element_keys(G, tr, rec, i, key, has_tpot);
      if (pass == 0) {
        n_tpot += has_tpot;
        n_pre += rec.preempt_count[G.record_offset + i] > 0;
        unsigned long long fk = dkey(rec.finish[G.record_offset + i]);
        double a = tr.arrival[G.trace_offset + i];
        if (G.qps_factor != 1.0) a = __ddiv_rn(a, G.qps_factor);
        unsigned long long ak = dkey(a);
        mfin = fk > mfin ? fk : mfin;
        marr = ak < marr ? ak : marr;
      }
#pragma unroll
      for (int s = 0; s < NSLOT; ++s) {
        const int st = SLOT_STAT[s];
        if (st == 3 && !has_tpot) continue;
        if (pass > 0 && !s_active[s]) continue;
        if ((key[st] & hmask) != s_prefix[s]) continue;
        atomicAdd(&hist[s][(unsigned)(key[st] >> shift) & 255u], 1u);
      }
    }
    if (pass == 0) {
      // block reductions of the scalar statistics
      for (int o = 16; o; o >>= 1) {
        n_tpot += __shfl_xor_sync(0xffffffffu, n_tpot, o);
        n_pre += __shfl_xor_sync(0xffffffffu, n_pre, o);
        unsigned long long a = __shfl_xor_sync(0xffffffffu, mfin, o), b = __shfl_xor_sync(0xffffffffu, marr, o);
        mfin = a > mfin ? a : mfin;
        marr = b < marr ? b : marr;
      }
      if ((threadIdx.x & 31) == 0) {
        atomicAdd((unsigned long long*)&W.n_tpot, (unsigned long long)n_tpot);
        atomicAdd((unsigned long long*)&W.n_pre, (unsigned long long)n_pre);
        atomicMax(&W.max_fin_key, mfin);
        atomicMin(&W.min_arr_key, marr);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NSLOT * 256; i += blockDim.x) {
      unsigned v = (&hist[0][0])[i];
      if (v) atomicAdd(&(&W.hist[0][0])[i], v);
    }
    __syncthreads();
  }
}

__global__ void k_select(const ssb_summary_group* __restrict__ groups, int n_groups, GroupWork* __restrict__ work,
                         int pass) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_groups * NSLOT) return;
  const int g = (int)(t / NSLOT), s = (int)(t % NSLOT);
  GroupWork& W = work[g];
  if (pass == 0 && s >= 7) {  // TPOT / queue ranks from the sample sizes (integer nearest rank)
    const long long n = s < 10 ? W.n_tpot : groups[g].n;
    const int p = (s == 7 || s == 10) ? 50 : ((s == 8 || s == 11) ? 95 : 99);
    W.k[s] = (s < 10 && groups[g].rank[s - 4] > 0) ? groups[g].rank[s - 4] : (n > 0 ? (p * n + 99) / 100 : 0);
  }
  const int shift = 56 - 8 * pass;
  long long k = W.k[s];
  if (k > 0) {
    long long cum = 0;
    int d = 0;
    for (; d < 256; ++d) {
      long long h = W.hist[s][d];
      if (cum + h >= k) break;
      cum += h;
    }
    if (d > 255) d = 255;  // cannot happen for a valid rank
    W.prefix[s] |= (unsigned long long)d << shift;
    W.k[s] = k - cum;
  }
  for (int d = 0; d < 256; ++d) W.hist[s][d] = 0u;
}

__global__ void k_finish(const ssb_summary_group* __restrict__ groups, int n_groups, const GroupWork* __restrict__ work,
                         ssb_summary* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const GroupWork& W = work[g];
  const long long n = groups[g].n;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  ssb_summary S;
  S.n_requests = n;
  double v[NSLOT];
  for (int s = 0; s < NSLOT; ++s) v[s] = W.k[s] > 0 ? dkey_inv(W.prefix[s]) : nan;
  S.ttft_p50 = v[0]; S.ttft_p95 = v[1]; S.ttft_p99 = v[2];
  S.norm_ttft_p50 = v[3]; S.norm_ttft_p95 = v[4];
  S.gen_time_p50 = v[5]; S.gen_time_p95 = v[6];
  S.tpot_p50 = v[7]; S.tpot_p95 = v[8]; S.tpot_p99 = v[9];
  S.queue_p50 = v[10]; S.queue_p95 = v[11]; S.queue_p99 = v[12];
  S.n_tpot = W.n_tpot;
  S.n_preempted = W.n_pre;
  S.preemption_rate = n > 0 ? __ddiv_rn((double)W.n_pre, (double)n) : nan;  // metrics.py:97
  S.max_finish = dkey_inv(W.max_fin_key);
  S.min_arrival = dkey_inv(W.min_arr_key);
  const double span = __dsub_rn(S.max_finish, S.min_arrival);  // metrics.py:86
  S.throughput_rps = span > 0 ? __ddiv_rn((double)n, span) : __longlong_as_double(0x7ff0000000000000LL);
  out[g] = S;
}

// Pooled histogram over ALL groups (one record set spread over many instances and,
// across ranks, over many GPUs): the per-pass digit histogram of every rank slot whose
// key matches that slot's current prefix, summed over the groups. The host all-gathers
// these 13 x 256 counts across ranks and picks the digits (pooled.py), so an exact
// nearest-rank percentile of the union of every rank's records costs 8 small
// collectives and no record movement.
__global__ void __launch_bounds__(THREADS) k_pool_hist(ssb_trace tr, ssb_records rec,
                                                       const ssb_summary_group* __restrict__ groups, int n_groups,
                                                       const long long* __restrict__ cstart, long long n_chunks,
                                                       const unsigned long long* __restrict__ prefix,
                                                       const int* __restrict__ active, int pass,
                                                       unsigned* __restrict__ out_hist,
                                                       unsigned long long* __restrict__ out_counts) {
  __shared__ unsigned hist[NSLOT][256];
  __shared__ unsigned long long s_prefix[NSLOT];
  __shared__ int s_active[NSLOT];
  const int shift = 56 - 8 * pass;
  const unsigned long long hmask = pass == 0 ? 0ULL : (~0ULL << (shift + 8));
  for (int i = threadIdx.x; i < NSLOT * 256; i += blockDim.x) (&hist[0][0])[i] = 0u;
  if (threadIdx.x < NSLOT) {
    s_prefix[threadIdx.x] = prefix[threadIdx.x] & hmask;
    s_active[threadIdx.x] = active[threadIdx.x];
  }
  __syncthreads();
  unsigned long long n_all = 0, n_tpot = 0, n_pre = 0;
  for (long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int g = find_group(cstart, n_groups, c);
    const ssb_summary_group G = groups[g];
    const long long e0 = (c - cstart[g]) * CHUNK;
    const long long e1 = (e0 + CHUNK < G.n) ? e0 + CHUNK : G.n;
    for (long long i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
      unsigned long long key[5];
      bool has_tpot;
      element_keys(G, tr, rec, i, key, has_tpot);
      if (pass == 0) {
        n_all += 1;
        n_tpot += has_tpot;
        n_pre += rec.preempt_count[G.record_offset + i] > 0;
      }
#pragma unroll
      for (int s = 0; s < NSLOT; ++s) {
        const int st = SLOT_STAT[s];
        if (!s_active[s] || (st == 3 && !has_tpot)) continue;
        if ((key[st] & hmask) != s_prefix[s]) continue;
        atomicAdd(&hist[s][(unsigned)(key[st] >> shift) & 255u], 1u);
      }
    }
  }
  if (pass == 0) {
    for (int o = 16; o; o >>= 1) {
      n_all += __shfl_xor_sync(0xffffffffu, n_all, o);
      n_tpot += __shfl_xor_sync(0xffffffffu, n_tpot, o);
      n_pre += __shfl_xor_sync(0xffffffffu, n_pre, o);
    }
    if ((threadIdx.x & 31) == 0 && n_all) {
      atomicAdd(&out_counts[0], n_all);
      atomicAdd(&out_counts[1], n_tpot);
      atomicAdd(&out_counts[2], n_pre);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NSLOT * 256; i += blockDim.x) {
    const unsigned v = (&hist[0][0])[i];
    if (v) atomicAdd(&out_hist[i], v);
  }
}

// Small groups (every group <= SMALL_MAX records, e.g. the C4 sweep's ~1.8k per instance): one
// CTA per group sorts each statistic's order-preserving keys in shared memory (bitonic) and
// reads the nearest ranks directly — one launch instead of 8 histogram + 8 select passes.
// Same keys, same ranks, so the same values as the radix path.
constexpr int SMALL_MAX = 4096;
constexpr int SMALL_THREADS = 512;
__global__ void __launch_bounds__(SMALL_THREADS) k_small_summary(ssb_trace tr, ssb_records rec,
                                                                 const ssb_summary_group* __restrict__ groups,
                                                                 int n_groups, ssb_summary* __restrict__ out) {
  __shared__ unsigned long long keys[SMALL_MAX];
  __shared__ unsigned long long red[SMALL_THREADS / 32][2];
  __shared__ long long cnt[SMALL_THREADS / 32][2];
  __shared__ double vals[NSLOT];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const ssb_summary_group G = groups[g];
    const int n = (int)G.n;
    int P = 1;
    while (P < n) P <<= 1;
    long long n_tpot = 0, n_pre = 0;
    unsigned long long mfin = 0ULL, marr = ~0ULL;
    for (int i = tid; i < n; i += SMALL_THREADS) {
      const long long t = G.trace_offset + i, r = G.record_offset + i;
      n_tpot += tr.output[t] > 1;
      n_pre += rec.preempt_count[r] > 0;
      const unsigned long long fk = dkey(rec.finish[r]);
      double a = tr.arrival[t];
      if (G.qps_factor != 1.0) a = __ddiv_rn(a, G.qps_factor);
      const unsigned long long ak = dkey(a);
      mfin = fk > mfin ? fk : mfin;
      marr = ak < marr ? ak : marr;
    }
    for (int o = 16; o; o >>= 1) {
      n_tpot += __shfl_xor_sync(0xffffffffu, n_tpot, o);
      n_pre += __shfl_xor_sync(0xffffffffu, n_pre, o);
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, mfin, o), b = __shfl_xor_sync(0xffffffffu, marr, o);
      mfin = a > mfin ? a : mfin;
      marr = b < marr ? b : marr;
    }
    if (lane == 0) { red[wid][0] = mfin; red[wid][1] = marr; cnt[wid][0] = n_tpot; cnt[wid][1] = n_pre; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < SMALL_THREADS / 32; ++w) {
        mfin = red[w][0] > mfin ? red[w][0] : mfin;
        marr = red[w][1] < marr ? red[w][1] : marr;
        n_tpot += cnt[w][0];
        n_pre += cnt[w][1];
      }
      cnt[0][0] = n_tpot; cnt[0][1] = n_pre; red[0][0] = mfin; red[0][1] = marr;
    }
    __syncthreads();
    n_tpot = cnt[0][0];
#pragma unroll 1
    for (int st = 0; st < 5; ++st) {
      for (int i = tid; i < P; i += SMALL_THREADS) keys[i] = i < n ? stat_key(G, tr, rec, i, st) : ~0ULL;  // padding sorts last
      __syncthreads();
      for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int i = tid; i < P / 2; i += SMALL_THREADS) {
            const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
            const bool up = (lo & size) == 0;
            const unsigned long long a = keys[lo], b = keys[hi];
            if ((a > b) == up) { keys[lo] = b; keys[hi] = a; }
          }
          __syncthreads();
        }
      if (tid < NSLOT && SLOT_STAT[tid] == st) {  // nearest rank, as k_init / k_select pick it
        long long k;
        if (tid < 7) k = G.rank[tid < 3 ? tid : (tid < 5 ? tid - 3 : tid - 5)];
        else {
          const long long m = tid < 10 ? n_tpot : G.n;
          const int p = (tid == 7 || tid == 10) ? 50 : ((tid == 8 || tid == 11) ? 95 : 99);
          k = (tid < 10 && G.rank[tid - 4] > 0) ? G.rank[tid - 4] : (m > 0 ? (p * m + 99) / 100 : 0);
        }
        vals[tid] = k > 0 ? dkey_inv(keys[k - 1]) : __longlong_as_double(0x7ff8000000000000LL);
      }
      __syncthreads();
    }
    if (tid == 0) {
      ssb_summary S;
      S.n_requests = G.n;
      S.ttft_p50 = vals[0]; S.ttft_p95 = vals[1]; S.ttft_p99 = vals[2];
      S.norm_ttft_p50 = vals[3]; S.norm_ttft_p95 = vals[4];
      S.gen_time_p50 = vals[5]; S.gen_time_p95 = vals[6];
      S.tpot_p50 = vals[7]; S.tpot_p95 = vals[8]; S.tpot_p99 = vals[9];
      S.queue_p50 = vals[10]; S.queue_p95 = vals[11]; S.queue_p99 = vals[12];
      S.n_tpot = n_tpot;
      S.n_preempted = cnt[0][1];
      S.preemption_rate = G.n > 0 ? __ddiv_rn((double)cnt[0][1], (double)G.n) : __longlong_as_double(0x7ff8000000000000LL);
      S.max_finish = dkey_inv(red[0][0]);
      S.min_arrival = dkey_inv(red[0][1]);
      const double span = __dsub_rn(S.max_finish, S.min_arrival);  // metrics.py:86
      S.throughput_rps = span > 0 ? __ddiv_rn((double)G.n, span) : __longlong_as_double(0x7ff0000000000000LL);
      out[g] = S;
    }
    __syncthreads();
  }
}

long long chunks_of(long long n) { return n > 0 ? (n + CHUNK - 1) / CHUNK : 0; }

}  // namespace

extern "C" size_t ssb_summary_work_bytes(const ssb_summary_group* h_groups, int32_t n_groups) {
  return sizeof(GroupWork) * (size_t)(n_groups > 0 ? n_groups : 1) + sizeof(long long) * (size_t)(n_groups + 1) + 256;
}

extern "C" int32_t ssb_summarize(ssb_trace trace, ssb_records records, const ssb_summary_group* h_groups,
                                 const ssb_summary_group* d_groups, int32_t n_groups, ssb_summary* d_summary,
                                 void* d_work, size_t work_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n_groups <= 0) return SSB_OK;
  if (!h_groups || !d_groups || !d_summary || !d_work) return SSB_E_ARG;
  if (work_bytes < ssb_summary_work_bytes(h_groups, n_groups)) return SSB_E_ARG;
  std::vector<long long> cstart(n_groups + 1, 0);
  bool all_small = getenv("SSB_SUMMARY_RADIX") == nullptr;  // experiments: force the radix path
  for (int g = 0; g < n_groups; ++g) {
    if (h_groups[g].n < 1) return SSB_E_ARG;  // metrics.py:81-82 "no records to summarize"
    cstart[g + 1] = cstart[g] + chunks_of(h_groups[g].n);
    all_small &= h_groups[g].n <= SMALL_MAX;
  }
  if (all_small) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_small_summary<<<(unsigned)std::min<long long>(n_groups, 6L * sms), SMALL_THREADS, 0, stream>>>(
        trace, records, d_groups, n_groups, d_summary);
    return cudaGetLastError() == cudaSuccess ? SSB_OK : SSB_E_CUDA;
  }
  const long long n_chunks = cstart[n_groups];
  GroupWork* work = (GroupWork*)d_work;
  long long* d_cstart = (long long*)((char*)d_work + sizeof(GroupWork) * (size_t)n_groups);
  if (cudaMemcpyAsync(d_cstart, cstart.data(), sizeof(long long) * cstart.size(), cudaMemcpyHostToDevice, stream) !=
      cudaSuccess)
    return SSB_E_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_init<<<(unsigned)std::min<long long>(n_groups, 4L * sms), 256, 0, stream>>>(d_groups, n_groups, work);
  const unsigned hist_grid = (unsigned)std::min<long long>(n_chunks, 8L * sms);
  const unsigned sel_grid = (unsigned)(((long long)n_groups * NSLOT + 255) / 256);
  for (int pass = 0; pass < 8; ++pass) {
    k_hist<<<hist_grid, THREADS, 0, stream>>>(trace, records, d_groups, n_groups, d_cstart, n_chunks, work, pass);
    k_select<<<sel_grid, 256, 0, stream>>>(d_groups, n_groups, work, pass);
  }
  k_finish<<<(n_groups + 127) / 128, 128, 0, stream>>>(d_groups, n_groups, work, d_summary);
  return cudaGetLastError() == cudaSuccess ? SSB_OK : SSB_E_CUDA;
}

extern "C" int32_t ssb_pool_hist(ssb_trace trace, ssb_records records, const ssb_summary_group* h_groups,
                                 const ssb_summary_group* d_groups, int32_t n_groups, const uint64_t* d_prefix,
                                 const int32_t* d_active, int32_t pass, uint32_t* d_hist, uint64_t* d_counts,
                                 void* d_work, size_t work_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n_groups <= 0) return SSB_OK;
  if (!h_groups || !d_groups || !d_prefix || !d_active || !d_hist || !d_counts || !d_work) return SSB_E_ARG;
  if (pass < 0 || pass > 7 || work_bytes < sizeof(long long) * (size_t)(n_groups + 1)) return SSB_E_ARG;
  std::vector<long long> cstart(n_groups + 1, 0);
  for (int g = 0; g < n_groups; ++g) {
    if (h_groups[g].n < 0) return SSB_E_ARG;
    cstart[g + 1] = cstart[g] + chunks_of(h_groups[g].n);
  }
  const long long n_chunks = cstart[n_groups];
  long long* d_cstart = (long long*)d_work;
  if (cudaMemcpyAsync(d_cstart, cstart.data(), sizeof(long long) * cstart.size(), cudaMemcpyHostToDevice, stream) !=
      cudaSuccess)
    return SSB_E_CUDA;
  if (cudaMemsetAsync(d_hist, 0, sizeof(uint32_t) * NSLOT * 256, stream) != cudaSuccess) return SSB_E_CUDA;
  if (pass == 0 && cudaMemsetAsync(d_counts, 0, sizeof(uint64_t) * 3, stream) != cudaSuccess) return SSB_E_CUDA;
  if (n_chunks == 0) return SSB_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<long long>(n_chunks, 4L * sms);
  k_pool_hist<<<grid, THREADS, 0, stream>>>(trace, records, d_groups, n_groups, d_cstart, n_chunks,
                                           (const unsigned long long*)d_prefix, d_active, pass, d_hist,
                                           (unsigned long long*)d_counts);
  return cudaGetLastError() == cudaSuccess ? SSB_OK : SSB_E_CUDA;
}
