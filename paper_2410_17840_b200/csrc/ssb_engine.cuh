// ssb_engine.cuh — warp-synchronous device restatement of one serving engine.
//
// One warp owns one engine (replica). All 32 lanes hold identical copies of
// the engine scalars (clock, free blocks, counts, digest ...) and cooperate on
// the per-request work with ballots, shuffles and warp scans:
//
//   Engine.step            engine.py:193-234      -> Eng::step
//   FcfsPolicy.select      policies.py:87-97      -> select_prefix (warp prefix-sum + ballot)
//   NoPreemptPolicy        policies.py:133-146    -> select_prefix (reservation blocks)
//   ShortestRemaining      policies.py:168-212    -> select_trail  (ordered warp argmin extraction)
//   LoadAdaptive / LARRY   policies.py:244-276    -> select_larry  (ordered warp argmax extraction)
//   _form_batch            engine.py:300-323      -> form_batch    (warp scan over the running table)
//   iteration_latency      costmodel.py:37-47     -> latency (binary64, explicit __d*_rn, no FMA)
//   _apply_progress        engine.py:325-358      -> progress      (parallel commit up to the first
//   _grow_or_evict / _evict_for_blocks :381-412                      failing grow, serial eviction)
//   KvBlockPool            kvmem.py:74-154        -> free_blocks + per-entry (prompt+generated)
//
// Data layout (per engine, in the scratch buffer, see ssb_kernels.cu):
//   waiting ring  SoA {rid|flag, pending, key, enqueue_time}       (deque, engine.py:162)
//   running table SoA {rid, prompt, output, generated, prefill_done, state, plan}
//                 kept in dispatch_seq order == dict insertion order (engine.py:163,297)
// A running request's KV allocation is always prompt+generated tokens
// (dispatch allocates pending_prefill = prompt+generated, first-token and
// decode grows keep that invariant), so the pool needs no per-request token map.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ssb.h"

namespace ssb {

// Debug build (-DSSB_DEBUG, tools/build_variant.sh debug -DSSB_DEBUG): bounds and accounting
// asserts on the engine's tables, rings and pool (trap with the failing condition printed);
// compiled out otherwise. The GPU suite runs against it with SSB_LIB=<debug lib>.
#ifdef SSB_DEBUG
#define SSB_ASSERT(c)                                                                    \
  do {                                                                                   \
    if (!(c)) {                                                                          \
      printf("SSB_ASSERT failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define SSB_ASSERT(c) do { } while (0)
#endif

constexpr unsigned FULL = 0xffffffffu;
constexpr int ST_GONE = 0;     // finished / evicted / parked during this step (compacted away)
constexpr int ST_PREFILL = 1;  // RequestState.PREFILLING
constexpr int ST_DECODE = 2;   // RequestState.DECODING
constexpr int FLAG_SEEN = (int)0x80000000;  // waiting entry was dispatched before (preempted/parked)
constexpr unsigned long long FNV_OFF = 0xcbf29ce484222325ULL;
constexpr unsigned long long FNV_PRIME = 0x100000001b3ULL;
constexpr unsigned long long FNV_PRIME_INV = 0xce965057aff6957bULL;  // FNV_PRIME^-1 mod 2^64

// trail_plus waiting set geometry: one bucket per remaining-output value
// (remaining <= output_len < min(max_context, pool tokens), policies.py:56-68 feasibility),
// a min-need tree over the buckets with fan-out 128: a warp reads one 128-node chunk as
// one int4 per lane and finds the first qualifying node with one ballot, so a search is
// at most 2 x levels dependent loads (2 levels up to 16,384 buckets, 3 up to 2^21).
// Level l holds n_l = ceil(n_{l-1}/128) nodes, padded to a multiple of 128; the top level
// is one chunk (<= 128 nodes).
constexpr int TF = 128;       // fan-out
constexpr int TF_SHIFT = 7;
struct TrailGeom {
  int nb;      // buckets (multiple of 128)
  int top;     // index of the top level (0..2)
  int off[4];  // level offsets (ints) into the level array (multiples of 128)
  int total;   // ints in the level array
};
__host__ __device__ inline TrailGeom trail_geom(int max_ctx, int pool, int bs) {
  long long maxrem = (long long)pool * bs;
  if ((long long)max_ctx < maxrem) maxrem = max_ctx;
  if (maxrem < 1) maxrem = 1;
  TrailGeom g;
  long long n = (maxrem + TF) / TF * TF;  // buckets 0..maxrem
  if (n > (1LL << 20)) n = 1LL << 20;     // ssb_simulate rejects larger
  g.nb = (int)n;
  g.top = 0;
  g.off[0] = 0;
  g.off[1] = g.off[2] = g.off[3] = 0;
  long long o = n;
  while (n > TF && g.top < 2) {
    n = (n + TF - 1) / TF;
    n = (n + TF - 1) / TF * TF;
    g.top += 1;
    g.off[g.top] = (int)o;
    o += n;
  }
  g.total = (int)o;
  return g;
}

struct Cfg {
  int policy, max_output, bs, bs_shift, pool, cap, max_running, max_ctx;
  unsigned long long bmul;  // ceil(2^32 / bs): blocks() as one multiply-shift, exact (see blocks)
  int n_servers, Wc, Rc;
  bool wide;  // latency-mode kernel: the R <= 64 register path is compiled in (k_engines<true>)
  double alpha, c, mem_base, mem_kv, compute, overhead, qps;
  TrailGeom tg;
};

// Persisted per-engine state (global scratch; registers while a warp runs it).
struct Srv {
  double clock;
  long long iterations, rsteps, btokens, dispatches, preempts, parks, finished, peak;
  unsigned long long digest;
  long long wpend_sum;       // Σ pending_prefill over waiting (snapshot_stats, cluster.py:53)
  long long fin_in, fin_out, fin_cnt;  // completions (BetaEstimator.update, balancers.py:81-86)
  long long enq_prompt_sum;  // Σ prompt over enqueued arrivals (inbox accounting)
  long long ev_n;
  long long pf_pend;         // Σ pending over PREFILLING entries
  int free_blocks, R, W, whead, committed, next_arr, status, ndec;
};

struct SrvPtr {
  double* w_enq;
  int* w_rid;
  int* w_pend;
  int* w_key;
  int* r_rid;
  int* r_prompt;
  int* r_out;
  int* r_gen;
  int* r_pfd;
  int* r_st;
  int* r_plan;
  int* l_a;   // dispatch list (physical ring slots) / scratch list
  int* l_b;   // preempt list (table indices) / scratch list
  int* l_c;   // trail_plus dispatch list: pending prefill
  int* v_idx; // queued waiting pushes (preempt_entry / flush_pushes): rid | flag
  int* v_rem; //   ... pending prefill
  long long* v_cum;           //   ... policy key; trail_plus victims: allocated blocks
  unsigned long long* v_key;  // trail_plus victims: (remaining << 32 | table index), 0 = taken
  int* rl;    // route list (arrival ids routed to this engine), n_servers > 1
  int* t_head;  // trail_plus: first request id of each remaining-output bucket (-1 = empty)
  int* t_lv;    // trail_plus: min-need tree over the buckets (level 0 = per-bucket minimum)
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ long long warp_incl_scan_ll(long long v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long n = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
// single-instruction (REDUX) warp sum for per-chunk values that fit in 32 bits
__device__ __forceinline__ int redux_add(int v) { return (int)__reduce_add_sync(FULL, (unsigned)v); }

// total order on binary64 as unsigned 64-bit keys (larger double -> larger key)
__device__ __forceinline__ unsigned long long dkey(double x) {
  long long b = __double_as_longlong(x);
  return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ULL);
}
// lanes (mask) holding the maximum 64-bit key among lanes with `has` (0 if none): two REDUX.MAX
__device__ __forceinline__ unsigned warp_argmax_u64(unsigned long long key, bool has) {
  if (!__any_sync(FULL, has)) return 0u;
  unsigned hi = has ? (unsigned)(key >> 32) : 0u;
  unsigned m1 = __reduce_max_sync(FULL, hi);
  bool c1 = has && hi == m1;
  unsigned lo = c1 ? (unsigned)key : 0u;
  unsigned m2 = __reduce_max_sync(FULL, lo);
  return __ballot_sync(FULL, c1 && lo == m2);
}
// warp minimum of a 64-bit key (uniform): two REDUX.MIN on the halves
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long key) {
  const unsigned hi = __reduce_min_sync(FULL, (unsigned)(key >> 32));
  const unsigned lo = __reduce_min_sync(FULL, (unsigned)(key >> 32) == hi ? (unsigned)key : 0xffffffffu);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned warp_argmin_u64(unsigned long long key, bool has) {
  return warp_argmax_u64(~key, has);
}


// FNV-1a over the 64-bit words (code, request id, time bits) of one event
__device__ __forceinline__ unsigned long long fnv_event(unsigned long long h, int code, int rid, double t) {
  h ^= (unsigned long long)code; h *= FNV_PRIME;
  h ^= (unsigned long long)(long long)rid; h *= FNV_PRIME;
  h ^= (unsigned long long)__double_as_longlong(t); h *= FNV_PRIME;
  return h;
}
__device__ __forceinline__ void write_event(ssb_event* ev, long long pos, long long cap, double t, int rid, int server,
                                         int code) {
  if (pos < cap) {
    ssb_event e;
    e.time = t;
    e.request_id = rid;
    e.server = (int16_t)server;
    e.code = (int16_t)code;
    ev[pos] = e;
  }
}

// One warp-uniform batch of events: lane i contributes code_a if bit i of mask_a, then code_b
// if bit i of mask_b; order = lane order (a before b within a lane). Folds them into the
// decision digest h (FNV-1a) and, with an event ring, writes them from position pos0.
// Inlined like every engine helper: a call in a hot function costs more than its code size
// (measured: out-of-line helpers forced register save/restore around the calls).
__device__ __forceinline__ unsigned long long emit_events(unsigned long long h, unsigned mask_a, int code_a,
                                                       unsigned mask_b, int code_b, int rid_lane, double t,
                                                       ssb_event* ev, long long pos0, long long cap, int server) {
  const int lane = threadIdx.x & 31;
  const unsigned both = mask_a | mask_b;
  if (ev != nullptr && ((both >> lane) & 1u)) {
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    long long pos = pos0 + __popc(mask_a & lt) + __popc(mask_b & lt);
    if ((mask_a >> lane) & 1u) write_event(ev, pos++, cap, t, rid_lane, server, code_a);
    if ((mask_b >> lane) & 1u) write_event(ev, pos, cap, t, rid_lane, server, code_b);
  }
  unsigned m = both;
  while (m) {
    const int b = __ffs(m) - 1;
    m &= m - 1;
    const int rid = __shfl_sync(FULL, rid_lane, b);
    if ((mask_a >> b) & 1u) {
      h ^= (unsigned long long)code_a; h *= FNV_PRIME;
      h ^= (unsigned long long)(long long)rid; h *= FNV_PRIME;
      h ^= (unsigned long long)__double_as_longlong(t); h *= FNV_PRIME;
    }
    if ((mask_b >> b) & 1u) {
      h ^= (unsigned long long)code_b; h *= FNV_PRIME;
      h ^= (unsigned long long)(long long)rid; h *= FNV_PRIME;
      h ^= (unsigned long long)__double_as_longlong(t); h *= FNV_PRIME;
    }
  }
  return h;
}

// stable compaction of a running table (drops ST_GONE entries); returns the new size.
// (Inlined: see emit_events.)
__device__ __forceinline__ int compact_table(int* __restrict__ r_rid, int* __restrict__ r_prompt, int* __restrict__ r_out,
                                          int* __restrict__ r_gen, int* __restrict__ r_pfd, int* __restrict__ r_st, int R) {
  const int lane = threadIdx.x & 31;
  int out = 0;
  #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
  for (int base = 0; base < R; base += 32) {
    const int j = base + lane;
    const bool valid = j < R;
    int rid = 0, pr = 0, o = 0, g = 0, f = 0, s = ST_GONE;
    if (valid) {
      s = r_st[j];
      rid = r_rid[j]; pr = r_prompt[j]; o = r_out[j]; g = r_gen[j]; f = r_pfd[j];
    }
    const bool keep = valid && s != ST_GONE;
    const unsigned m = __ballot_sync(FULL, keep);
    __syncwarp();
    if (keep) {
      const int d = out + __popc(m & lanemask_lt());
      r_rid[d] = rid; r_prompt[d] = pr; r_out[d] = o; r_gen[d] = g; r_pfd[d] = f; r_st[d] = s;
    }
    out += __popc(m);
    __syncwarp();
  }
  return out;
}

#ifdef SSB_PHASE_TIMING
#define SSB_T0(name) long long _t_##name = clock64();
#define SSB_T1(name, slot) tm[slot] += clock64() - _t_##name; tc[slot] += 1;
#else
#define SSB_T0(name)
#define SSB_T1(name, slot)
#endif

struct Eng {
#ifdef SSB_PHASE_TIMING
  long long tm[16], tc[16];  // 0 enqueue 1 select 2 preempt+dispatch 3 fast 4 small 5 general 6/7 walk counters
                            // 8 victims_build 9 t_find 10 bucket walk 11 trail_remove 12 victims_take 13 preempts 14 small->general
#endif
  Cfg cfg;
  Srv st;
  SrvPtr p;
  const double* arrival;  // instance trace base
  const int* prompt;
  const int* output;
  double* rec_ft;         // instance record base
  double* rec_fin;
  double* rec_fd;
  int* rec_pc;
  int* rec_srv;
  ssb_event* ev;          // nullable
  long long ev_cap;
  int server;
  int lane;
  // steady-state decode mode: running entries j = lane and j = lane + 32 cached in
  // registers across iterations (valid when regs_ok), rsum = Σ (prompt+generated)
  int c_rid0, c_pr0, c_out0, c_g0, c_rid1, c_pr1, c_out1, c_g1;
  bool regs_ok, regs_dirty;
  long long rsum;
  // nodisp: the last select dispatched nothing and nothing it depends on has
  // changed since (no enqueue / dispatch / finish / preempt) -> it would again
  // dispatch nothing: FCFS & NoPreempt (free only shrinks, committed fixed),
  // trail_plus (free + coverable victim blocks never grows), any policy with W == 0.
  bool nodisp;
  // larry top cache: the last full scan's winner (physical slot, pending) and the margin
  // delta >= (exact score gap to every other candidate) that certifies it stays the
  // winner while the waiting set (and so queue_len) is unchanged: see select_larry
  bool lc_valid;
  int lc_pos, lc_pend;
  double lc_delta, lc_emin;
  long long lc_pmax;

  __device__ __forceinline__ void init_modes() {
    regs_ok = regs_dirty = false;
    rsum = 0;
    nodisp = false;
    lc_valid = false;
    nq = 0;
  }
  __device__ __forceinline__ void flush_regs() {
    if (regs_dirty) {
      if (lane < st.R) p.r_gen[lane] = c_g0;
      if (lane + 32 < st.R) p.r_gen[lane + 32] = c_g1;
      regs_dirty = false;
      __syncwarp();
    }
  }
  __device__ __forceinline__ void drop_regs() {
    flush_regs();
    regs_ok = false;
  }
  __device__ __forceinline__ void load_regs() {
    const bool v0 = lane < st.R, v1 = lane + 32 < st.R;
    c_rid0 = c_pr0 = c_out0 = c_g0 = c_rid1 = c_pr1 = c_out1 = c_g1 = 0;
    if (v0) { c_rid0 = p.r_rid[lane]; c_pr0 = p.r_prompt[lane]; c_out0 = p.r_out[lane]; c_g0 = p.r_gen[lane]; }
    if (v1) {
      c_rid1 = p.r_rid[lane + 32]; c_pr1 = p.r_prompt[lane + 32]; c_out1 = p.r_out[lane + 32]; c_g1 = p.r_gen[lane + 32];
    }
    rsum = (long long)redux_add(v0 ? c_pr0 + c_g0 : 0) + redux_add(v1 ? c_pr1 + c_g1 : 0);
    regs_ok = true;
    regs_dirty = false;
  }

  __device__ __forceinline__ int blocks(int tokens) const {  // kvmem.py:15-21
    // floor(n / bs) for n = tokens + bs - 1 as (n * ceil(2^32/bs)) >> 32: with
    // ceil(2^32/bs) = (2^32 + e)/bs, 0 <= e < bs, the error term n*e/(bs*2^32) stays below
    // 1/bs (so below 1 - frac(n/bs)) whenever n < 2^32/bs, which ssb_simulate checks for
    // every token count a request can reach (prompt + output <= max_context). Branch-free:
    // one code path for every block size (a smaller hot loop than a pow2/divide branch).
    SSB_ASSERT(tokens >= 0 && (long long)tokens + cfg.bs - 1 < (1LL << 32) / cfg.bs);
    const unsigned n = (unsigned)(tokens + cfg.bs - 1);
    return (int)(((unsigned long long)n * cfg.bmul) >> 32);
  }
  __device__ __forceinline__ int phys(int k) const {  // ring slot of logical position k
    SSB_ASSERT(k >= 0 && k <= cfg.Wc && st.whead >= 0 && st.whead < cfg.Wc);
    int x = st.whead + k;
    return x >= cfg.Wc ? x - cfg.Wc : x;
  }
  __device__ __forceinline__ double arrival_of(int rid) const {
    SSB_ASSERT(rid >= 0 && rid < cfg.Wc);  // (wait_cap = the instance's request count)
    return arrival[rid];  // already scaled by qps_factor (k_scale_arrivals, workload.py:193)
  }
  __device__ __forceinline__ int wkey_for(int prompt_len, int out, int gen) const {
    if (cfg.policy == SSB_POLICY_NOPREEMPT) {  // policies.py:116-117 reservation, in blocks
      int t = min(cfg.max_ctx, prompt_len + cfg.max_output);
      return blocks(t);
    }
    return out - gen;  // trail_plus remaining output (policies.py:172)
  }
  __device__ __forceinline__ bool has_work() const { return st.W > 0 || st.R > 0; }

  // ---- event log + decision digest (engine.py:273-274) ----
  __device__ __forceinline__ void fold(int code, int rid) { st.digest = fnv_event(st.digest, code, rid, st.clock); }
  __device__ __forceinline__ void log_at(long long pos, int code, int rid) {
    if (ev != nullptr) write_event(ev, pos, ev_cap, st.clock, rid, server, code);
  }
  // one event per lane in `mask`, lane order (warp-uniform call)
  __device__ __forceinline__ void emit(unsigned mask, int code, int rid_lane) {
    st.digest = emit_events(st.digest, mask, code, 0u, 0, rid_lane, st.clock, ev, st.ev_n, ev_cap, server);
    st.ev_n += __popc(mask);
  }
  // first_token (mask_a) then finish (mask_b) per lane, lanes in order
  __device__ __forceinline__ void emit2(unsigned mask_a, int code_a, unsigned mask_b, int code_b, int rid_lane) {
    st.digest = emit_events(st.digest, mask_a, code_a, mask_b, code_b, rid_lane, st.clock, ev, st.ev_n, ev_cap, server);
    st.ev_n += __popc(mask_a) + __popc(mask_b);
  }
  __device__ __forceinline__ void emit1(int code, int rid) {  // uniform single event
    if (lane == 0) log_at(st.ev_n, code, rid);
    fold(code, rid);
    st.ev_n += 1;
  }

  // ---- trail_plus waiting set (policies.py:171-173 order: remaining, arrival, id) ----
  // Bucket b holds the waiting requests with remaining output b as a list in id order
  // (arrival order == id order: the trace is sorted, cluster.py:81-83); t_head[b] is its
  // first id, w_rid[id] the next id, w_pend[id] the pending prefill | FLAG_SEEN. Level 0 of
  // t_lv is each bucket's minimum block need, every level above the minimum of 32 children,
  // so "first candidate in key order that could be admitted" is a few warp ballots
  // (t_find) instead of a walk over the whole waiting set.
  __device__ __forceinline__ int t_next(int id) const { return p.w_rid[id]; }
  __device__ __forceinline__ int t_pend(int id) const { return p.w_pend[id]; }
  __device__ void trail_init() {
    for (int i = lane; i < cfg.tg.nb; i += 32) p.t_head[i] = -1;
    for (int i = lane; i < cfg.tg.total; i += 32) p.t_lv[i] = 0x7fffffff;
    __syncwarp();
  }
  // level offset without dynamic indexing (keeps Cfg in registers)
  __device__ __forceinline__ int t_off(int l) const {
    return l == 0 ? 0 : (l == 1 ? cfg.tg.off[1] : cfg.tg.off[2]);
  }
  // first node of the 128-node chunk at `chunk` (int offset) with value <= T and index >= lo
  // (chunk-relative), or -1: lane i holds nodes 4i..4i+3
  __device__ __forceinline__ int t_chunk_first(int chunk, int lo, int T) const {
    const int4 v = *reinterpret_cast<const int4*>(p.t_lv + chunk + 4 * lane);
    const int q = 4 * lane;
    const unsigned bits = (unsigned)(v.x <= T && q >= lo) | ((unsigned)(v.y <= T && q + 1 >= lo) << 1) |
                          ((unsigned)(v.z <= T && q + 2 >= lo) << 2) | ((unsigned)(v.w <= T && q + 3 >= lo) << 3);
    const unsigned m = __ballot_sync(FULL, bits != 0u);
    if (m == 0u) return -1;
    const int f = __ffs(m) - 1;
    const unsigned fb = __shfl_sync(FULL, bits, f);
    return 4 * f + __ffs(fb) - 1;
  }
  // first bucket >= b0 whose minimum need is <= T, or -1. Climb from b0's chunk until a
  // node <= T follows it, then descend (some child of a node <= T is <= T). One loop with a
  // single chunk probe: the probe is inlined once (the engine is instruction-fetch bound).
  __device__ int t_find(int b0, int T) const {
    if (b0 >= cfg.tg.nb) return -1;
    int lvl = 0, idx = b0, base = b0 & ~(TF - 1), lo = b0 & (TF - 1);
    bool down = false;
    if (cfg.tg.top == 1) {
      // two levels (up to 16,384 buckets): b0's chunk and the top chunk probed at once (both
      // loads in flight together), so a search that has to climb costs two rounds, not three
      const int4 v = *reinterpret_cast<const int4*>(p.t_lv + base + 4 * lane);
      const int4 u = *reinterpret_cast<const int4*>(p.t_lv + cfg.tg.off[1] + 4 * lane);
      const int q = 4 * lane, lo1 = (b0 >> TF_SHIFT) + 1;
      const unsigned b0s = (unsigned)(v.x <= T && q >= lo) | ((unsigned)(v.y <= T && q + 1 >= lo) << 1) |
                           ((unsigned)(v.z <= T && q + 2 >= lo) << 2) | ((unsigned)(v.w <= T && q + 3 >= lo) << 3);
      const unsigned b1s = (unsigned)(u.x <= T && q >= lo1) | ((unsigned)(u.y <= T && q + 1 >= lo1) << 1) |
                           ((unsigned)(u.z <= T && q + 2 >= lo1) << 2) | ((unsigned)(u.w <= T && q + 3 >= lo1) << 3);
      const unsigned m0 = __ballot_sync(FULL, b0s != 0u);
      if (m0 != 0u) {
        const int f = __ffs(m0) - 1;
        return base + 4 * f + __ffs(__shfl_sync(FULL, b0s, f)) - 1;
      }
      const unsigned m1 = __ballot_sync(FULL, b1s != 0u);
      if (m1 == 0u) return -1;
      const int f = __ffs(m1) - 1;
      const int node = 4 * f + __ffs(__shfl_sync(FULL, b1s, f)) - 1;
      return (node << TF_SHIFT) + t_chunk_first(node << TF_SHIFT, 0, T);  // a child of a node <= T is <= T
    }
    #pragma unroll 1
    while (true) {
      const int r = t_chunk_first(t_off(lvl) + base, lo, T);
      if (down || r >= 0) {  // (descending, r >= 0 always holds)
        const int node = base + r;
        if (lvl == 0) return node;
        down = true;
        lvl -= 1;
        base = node << TF_SHIFT;
        lo = 0;
        continue;
      }
      if (lvl == cfg.tg.top) return -1;
      idx >>= TF_SHIFT;
      lvl += 1;
      base = idx & ~(TF - 1);
      lo = (idx & (TF - 1)) + 1;
    }
  }

  // First bucket >= b whose minimum need is <= its EXACT threshold free + G(bucket), or -1;
  // T_out = that threshold. A bucket found with the looser bound T of an earlier bucket and
  // then rejected leaves T(found) as the bound for every later bucket, so the search
  // continues from the chunk values it already holds in registers (leaf chunk and top chunk,
  // two levels) instead of reloading them: a rejection costs a ballot and a REDUX.
  __device__ __forceinline__ int t_find_exact(int b, int free, int V, unsigned long long vk, int vb, long long& T_out) const {
    long long T = (long long)free + (V > 0 ? victims_gain(V, vk, vb, b) : 0);
    if (T > 0x7ffffffeLL) T = 0x7ffffffeLL;
    bool exact = true;  // T is b's own threshold (not a bound carried from a rejected bucket)
    if (cfg.tg.top != 1 || V == 0) {
      #pragma unroll 1
      while (true) {
        const int fb = t_find(b, (int)T);
        if (fb < 0 || (fb == b && exact) || V == 0) { T_out = T; return fb; }
        long long Te = (long long)free + victims_gain(V, vk, vb, fb);
        if (Te > 0x7ffffffeLL) Te = 0x7ffffffeLL;
        if (p.t_lv[fb] <= Te) { T_out = Te; return fb; }
        b = fb + 1;
        T = Te;
        exact = false;
      }
    }
    if (b >= cfg.tg.nb) return -1;
    int c = b >> TF_SHIFT, lo = b & (TF - 1);
    int4 v = *reinterpret_cast<const int4*>(p.t_lv + (c << TF_SHIFT) + 4 * lane);
    const int4 u = *reinterpret_cast<const int4*>(p.t_lv + cfg.tg.off[1] + 4 * lane);
    const int q = 4 * lane;
    #pragma unroll 1
    while (true) {
      const int t = (int)T;
      unsigned bits = (unsigned)(v.x <= t && q >= lo) | ((unsigned)(v.y <= t && q + 1 >= lo) << 1) |
                      ((unsigned)(v.z <= t && q + 2 >= lo) << 2) | ((unsigned)(v.w <= t && q + 3 >= lo) << 3);
      unsigned m = __ballot_sync(FULL, bits != 0u);
      if (m == 0u) {  // nothing left in this leaf chunk: the first later chunk whose minimum is <= T
        const int lo1 = c + 1;
        const unsigned b1 = (unsigned)(u.x <= t && q >= lo1) | ((unsigned)(u.y <= t && q + 1 >= lo1) << 1) |
                            ((unsigned)(u.z <= t && q + 2 >= lo1) << 2) | ((unsigned)(u.w <= t && q + 3 >= lo1) << 3);
        const unsigned m1 = __ballot_sync(FULL, b1 != 0u);
        if (m1 == 0u) return -1;
        const int f1 = __ffs(m1) - 1;
        c = 4 * f1 + __ffs(__shfl_sync(FULL, b1, f1)) - 1;
        lo = 0;
        v = *reinterpret_cast<const int4*>(p.t_lv + (c << TF_SHIFT) + 4 * lane);
        bits = (unsigned)(v.x <= t) | ((unsigned)(v.y <= t) << 1) | ((unsigned)(v.z <= t) << 2) |
               ((unsigned)(v.w <= t) << 3);
        m = __ballot_sync(FULL, bits != 0u);  // (non-empty: a child of a node <= T is <= T)
      }
      const int f = __ffs(m) - 1;
      const int e = __ffs(__shfl_sync(FULL, bits, f)) - 1;
      const int fb = (c << TF_SHIFT) + 4 * f + e;
      if (fb == b && exact) { T_out = T; return fb; }
      long long Te = (long long)free + victims_gain(V, vk, vb, fb);
      if (Te > 0x7ffffffeLL) Te = 0x7ffffffeLL;
      const int sel = e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
      if (__shfl_sync(FULL, sel, f) <= Te) { T_out = Te; return fb; }
      T = Te;  // rejected: T(fb) bounds every later bucket
      exact = false;
      b = fb + 1;
      lo = b & (TF - 1);
      if (lo == 0) lo = TF;  // (fb closed its chunk: continue at the top level)
    }
  }

  // set bucket b's minimum and restore "node = min of children" up the tree
  __device__ void t_set_leaf(int b, int val) {
    if (p.t_lv[b] == val) return;
    __syncwarp();
    if (lane == 0) p.t_lv[b] = val;
    __syncwarp();
    int idx = b;
    for (int l = 1; l <= cfg.tg.top; ++l) {
      const int parent = idx >> TF_SHIFT;
      const int4 v = *reinterpret_cast<const int4*>(p.t_lv + t_off(l - 1) + (parent << TF_SHIFT) + 4 * lane);
      const int mn = __reduce_min_sync(FULL, min(min(v.x, v.y), min(v.z, v.w)));
      const int at = t_off(l) + parent;
      if (p.t_lv[at] == mn) break;
      __syncwarp();
      if (lane == 0) p.t_lv[at] = mn;
      __syncwarp();
      idx = parent;
    }
  }
  __device__ void trail_insert(int rid_flag, int pend, int rem) {
    const int id = rid_flag & 0x7fffffff;
    SSB_ASSERT(rem >= 0 && rem < cfg.tg.nb && id < cfg.Wc && pend >= 0);
    int prev = -1, cur = p.t_head[rem];
    while (cur >= 0 && cur < id) { prev = cur; cur = t_next(cur); }
    __syncwarp();
    if (lane == 0) {
      p.w_rid[id] = cur;
      p.w_pend[id] = pend | (rid_flag & FLAG_SEEN);
      if (prev < 0) p.t_head[rem] = id; else p.w_rid[prev] = id;
    }
    __syncwarp();
    const int need = blocks(pend);
    if (need < p.t_lv[rem]) t_set_leaf(rem, need);
    st.W += 1;
  }
  // unlink `cur` (predecessor `prev`, -1 = head; successor `nx`) from bucket b; `need` = its
  // block need, `pmin` = the minimum need of the entries before it (select_trail walked them)
  __device__ void trail_remove(int b, int prev, int cur, int nx, int need, int pmin) {
    __syncwarp();
    if (lane == 0) { if (prev < 0) p.t_head[b] = nx; else p.w_rid[prev] = nx; }
    __syncwarp();
    if (need == p.t_lv[b] && pmin > need) {  // it was the only minimum before it: rescan the rest
      int mn = pmin;
      for (int c = nx; c >= 0; c = t_next(c)) mn = min(mn, blocks(t_pend(c) & 0x7fffffff));
      t_set_leaf(b, mn);
    }
    st.W -= 1;
  }

  // ---- Engine.enqueue for every routed arrival with arrival <= clock (engine.py:175-184, 261-262) ----
  __device__ void enqueue_ready(int n_avail) {
    while (st.next_arr < n_avail) {
      int k = st.next_arr + lane;
      bool valid = k < n_avail;
      int rid = 0;
      bool ok = false;
      if (valid) {
        // route-list slots not yet written read as -1 (the pipelined cluster kernel presets
        // them; every arrival before the engine's time limit is routed and visible)
        rid = (cfg.n_servers == 1) ? k : p.rl[k];
        ok = rid >= 0 && arrival_of(rid) <= st.clock;
      }
      unsigned m = __ballot_sync(FULL, ok);  // a prefix: routes are in arrival order
      int cnt = __popc(m);
      if (cnt == 0) break;
      if (st.W + cnt > cfg.Wc) { st.status = SSB_E_CAPACITY; return; }
      int pr = 0;
      const bool trail = cfg.policy == SSB_POLICY_TRAIL_PLUS;
      if (ok) {
        pr = prompt[rid];
        rec_srv[rid] = server;
        if (!trail) {
          int pos = phys(st.W + lane);
          p.w_rid[pos] = rid;
          p.w_pend[pos] = pr;
          p.w_key[pos] = wkey_for(pr, output[rid], 0);
          p.w_enq[pos] = st.clock;
        }
      }
      if (trail) {  // sorted by (remaining, id): insert in arrival order
        const int out = ok ? output[rid] : 0;
        #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
        for (unsigned mm = m; mm; mm &= mm - 1) {
          const int b = __ffs(mm) - 1;
          trail_insert(__shfl_sync(FULL, rid, b), __shfl_sync(FULL, pr, b), __shfl_sync(FULL, out, b));
        }
      }
      emit(m, SSB_EV_ENQUEUE, rid);
      nodisp = false;
      lc_valid = false;
      long long s = warp_sum_ll(pr);
      if (!trail) st.W += cnt;
      st.wpend_sum += s;
      st.enq_prompt_sum += s;
      st.next_arr += cnt;
      if (cnt < 32) break;
    }
    __syncwarp();
  }

  // ---- push a running entry back to the waiting head (_preempt, engine.py:368-379) ----
  // uniform call; the entry is table index j with loaded fields. Accounting, the table mark
  // and the event happen now; the waiting-set insertion is queued (v_* columns, free outside
  // select) and done by flush_pushes() in the same order, before anything reads the queue.
  int nq;  // queued waiting pushes
  __device__ void preempt_entry(int j, int rid, int pr, int out, int gen, int pfd, int state, int code) {
    nodisp = false;
    lc_valid = false;
    SSB_ASSERT(j >= 0 && j < st.R && rid >= 0 && rid < cfg.Wc && nq < cfg.Rc);
    int alloc = pr + gen;  // KV tokens held
    st.free_blocks += blocks(alloc);
    if (state == ST_DECODE) st.ndec -= 1;
    else st.pf_pend -= (long long)(alloc - pfd);
    if (cfg.policy == SSB_POLICY_NOPREEMPT) st.committed -= wkey_for(pr, out, gen);
    __syncwarp();  // every lane's reads of entry j (caller) happen before lane 0 rewrites it
    if (lane == 0) {
      p.r_st[j] = ST_GONE;
      rec_pc[rid] += 1;
      p.v_idx[nq] = rid | FLAG_SEEN;
      p.v_rem[nq] = alloc;  // pending_prefill = prompt + generated (prefill_done reset)
      p.v_cum[nq] = wkey_for(pr, out, gen);
    }
    nq += 1;
    st.wpend_sum += alloc;
    if (code == SSB_EV_PARK) st.parks += 1; else st.preempts += 1;
    emit1(code, rid);
    __syncwarp();
  }
  __device__ void flush_pushes() {
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int i = 0; i < nq; ++i) {
      const int rid_flag = p.v_idx[i], alloc = p.v_rem[i], key = (int)p.v_cum[i];
      if (st.W + 1 > cfg.Wc) { st.status = SSB_E_CAPACITY; break; }
      if (cfg.policy == SSB_POLICY_TRAIL_PLUS) {  // sorted waiting set: order is by key, not by deque position
        trail_insert(rid_flag, alloc, key);
      } else {
        st.whead = (st.whead == 0) ? cfg.Wc - 1 : st.whead - 1;
        if (lane == 0) {
          const int pos = st.whead;
          p.w_rid[pos] = rid_flag;
          p.w_pend[pos] = alloc;
          p.w_key[pos] = key;
          p.w_enq[pos] = st.clock;
        }
        st.W += 1;
      }
    }
    nq = 0;
    __syncwarp();
  }

  // ---- stable compaction of the running table (drops ST_GONE) ----
  __device__ __forceinline__ void compact_running() {
    st.R = compact_table(p.r_rid, p.r_prompt, p.r_out, p.r_gen, p.r_pfd, p.r_st, st.R);
  }

  // ---- FCFS / NoPreempt: dispatch the longest fitting queue prefix ----
  __device__ int select_prefix() {
    long long slots = cfg.max_running < 0 ? (1LL << 40) : (long long)cfg.max_running - st.R;  // policies.py:70-73
    int limit = (cfg.policy == SSB_POLICY_FCFS) ? st.free_blocks : cfg.pool - st.committed;
    if (st.W == 0 || slots <= 0) return 0;
    {  // head-of-line check first (uniform load): the common backlogged case dispatches nothing
      int pos = phys(0);
      int need0 = (cfg.policy == SSB_POLICY_FCFS) ? blocks(p.w_pend[pos]) : p.w_key[pos];
      if (need0 > limit) return 0;
    }
    int D = 0, used = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < st.W; base += 32) {
      int k = base + lane;
      bool valid = k < st.W;
      int need = 0;
      if (valid) {
        int pos = phys(k);
        need = (cfg.policy == SSB_POLICY_FCFS) ? blocks(p.w_pend[pos]) : p.w_key[pos];
      }
      int incl = warp_incl_scan(need, lane) + used;  // cumulative blocks (need >= 1 -> monotone)
      bool ok = valid && (long long)k < slots && incl <= limit;
      unsigned m = __ballot_sync(FULL, ok);
      int cnt = __popc(m);
      D += cnt;
      if (cnt < 32) break;
      used = __shfl_sync(FULL, incl, 31);
    }
    return D;
  }

  // ---- LARRY (policies.py:244-276): ordered extraction by (-score, enqueue_time, id) ----
  // One scan of the waiting ring yields the top two candidates (each lane keeps its best
  // two, the warp takes the argmax, then the argmax of the runner-ups), so a step that
  // dispatches at most one request never rescans.
  struct LKey {
    double sc, enq;
    int rid, k;
  };
  __device__ __forceinline__ static bool lbetter(const LKey& x, const LKey& y) {  // x before y in the order
    return x.sc > y.sc || (x.sc == y.sc && (x.enq < y.enq || (x.enq == y.enq && x.rid < y.rid)));
  }
  __device__ __forceinline__ unsigned larry_argmax(const LKey& x, bool has) const {
    unsigned win = warp_argmax_u64(dkey(x.sc), has);
    if (win & (win - 1)) win = warp_argmax_u64(~dkey(x.enq), has && ((win >> lane) & 1u));
    if (win & (win - 1)) win = warp_argmax_u64(~(unsigned long long)(unsigned)x.rid, has && ((win >> lane) & 1u));
    return win;
  }
  __device__ __forceinline__ LKey lshfl(const LKey& x, int src) const {
    LKey y;
    y.sc = __shfl_sync(FULL, x.sc, src);
    y.enq = __shfl_sync(FULL, x.enq, src);
    y.rid = __shfl_sync(FULL, x.rid, src);
    y.k = __shfl_sync(FULL, x.k, src);
    return y;
  }
  __device__ int select_larry() {
    if (st.W == 0) return 0;
    long long slots = cfg.max_running < 0 ? (1LL << 40) : (long long)cfg.max_running - st.R;
    // token budget left after running work (policies.py:251-257) == max(0, max(0, cap-#decoding) - Σ pending(prefilling))
    long long budget = (long long)cfg.cap - st.ndec;
    if (budget < 0) budget = 0;
    budget -= st.pf_pend;
    if (budget < 0) budget = 0;
    int free = st.free_blocks;
    const long long ql = st.W;  // queue_len, fixed for the step (:259)
    if (slots <= 0 || budget <= 0 || free <= 0) return 0;
    if (lc_valid) {
      // Scores are fl(fl(a*fl(clock-enq)) - ql*pending): in exact arithmetic every score moves by
      // the same a*dclock, so exact gaps are constant; each computed score is within
      // E = (3*a*(clock-enq) + ql*pending) * 2^-53 (x1.0001) of its exact value. If the cached
      // winner led every other candidate by delta (exact gap lower bound) and delta > 2E(clock),
      // it is still the strict winner; if it does not fit, nothing is dispatched this step.
      const double E = (3.0 * cfg.alpha * (st.clock - lc_emin) + (double)(ql * lc_pmax)) * 1.1102230246251565e-16 * 1.0001;
      if (lc_delta > 2.0 * E) {
        if (blocks(lc_pend) > free) return 0;
      }
      lc_valid = false;  // (it fits, or the margin is too thin: rescan)
    }
    int nd = 0;
    bool have_last = false;
    bool first_scan = true;
    LKey last{0.0, 0.0, 0, -1};
    while (true) {
      if ((long long)nd >= slots || budget <= 0 || free <= 0) break;  // need >= 1 always
      bool h1 = false, h2 = false;
      LKey b1{0.0, 0.0, 0x7fffffff, -1}, b2{0.0, 0.0, 0x7fffffff, -1};
      double emin = 1e300;  // (first scan) certification bounds, see below
      int pmax = 0;
      const double qld = (double)ql;
      #pragma unroll 1  // one element per lane per trip: the smallest loop body (instruction-fetch bound)
      for (int k = lane; k < st.W; k += 32) {  // (lanes diverge only in their last trip)
        LKey x;
        const int pos = phys(k);
        x.rid = p.w_rid[pos] & 0x7fffffff;
        x.enq = p.w_enq[pos];
        x.k = k;
        const int pend = p.w_pend[pos];
        emin = fmin(emin, x.enq);
        pmax = max(pmax, pend);
        // larry_score (policies.py:215-224): alpha*(clock-enq) - queue_len*pending; the
        // int product is < 2^53 (queue_len < 2^31, pending <= max_context), so the
        // binary64 product of the two exact operands is exact, as Python's int is
        x.sc = __dsub_rn(__dmul_rn(cfg.alpha, __dsub_rn(st.clock, x.enq)), __dmul_rn(qld, (double)pend));
        if (have_last && !lbetter(last, x)) continue;  // only keys strictly after `last`
        if (!h1 || lbetter(x, b1)) { b2 = b1; h2 = h1; b1 = x; h1 = true; }
        else if (!h2 || lbetter(x, b2)) { b2 = x; h2 = true; }
      }
      const unsigned w1 = larry_argmax(b1, h1);
      if (w1 == 0u) break;
      const int wl = __ffs(w1) - 1;
      const LKey top = lshfl(b1, wl);
      // runner-up: the winner lane offers its second best, every other lane its best
      const bool hr = (lane == wl) ? h2 : h1;
      const LKey rc = (lane == wl) ? b2 : b1;
      const unsigned w2 = larry_argmax(rc, hr);
      if (first_scan) {
        first_scan = false;
        // certify the winner for later steps: exact gap to any other candidate >= delta
        // (emin / pmax over the whole waiting set, gathered by the scan above)
#pragma unroll
        for (int o = 16; o; o >>= 1) emin = fmin(emin, __shfl_xor_sync(FULL, emin, o));
        pmax = __reduce_max_sync(FULL, (unsigned)pmax);
        const double E0 = (3.0 * cfg.alpha * (st.clock - emin) + (double)(ql * pmax)) * 1.1102230246251565e-16 * 1.0001;
        const double sc2 = w2 ? __shfl_sync(FULL, rc.sc, __ffs(w2) - 1) : -1e300;
        lc_delta = w2 ? (top.sc - sc2) - 2.0 * E0 : 1e300;  // a single candidate leads by infinity
        lc_emin = emin;
        lc_pmax = pmax;
        lc_pos = phys(top.k);
        lc_pend = p.w_pend[lc_pos];
        lc_valid = true;  // cleared by any dispatch / enqueue / preemption
      }
      int taken = 0;
      for (int t = 0; t < 2; ++t) {
        LKey c;
        if (t == 0) c = top;
        else {
          if (w2 == 0u || (long long)nd >= slots || budget <= 0 || free <= 0) break;
          c = lshfl(rc, __ffs(w2) - 1);
        }
        const int pos = phys(c.k);
        const int pend = p.w_pend[pos];
        const int need = blocks(pend);
        if (need > free) { taken = -1; break; }
        if (lane == 0) p.l_a[nd] = pos;
        nd++;
        free -= need;
        budget -= min((long long)pend, budget);
        last = c;
        have_last = true;
        taken++;
      }
      if (taken < 2) break;  // stopped, or the queue has no third candidate to try yet
      if (w2 == 0u) break;
    }
    __syncwarp();
    return nd;
  }

  // ---- trail_plus victims (policies.py:190-204) ----
  // Eligible running entries (generated < c * output_len) as an unsorted set of 64-bit keys
  // (remaining << 32 | table index) + allocated blocks: lane v holds victim v when V <= 32,
  // else the set lives in v_key / v_cum. G(b) (blocks of unmarked victims with remaining > b)
  // is one REDUX per 32 victims; the victims a covered candidate takes are extracted in key
  // order (largest remaining first, youngest dispatch first on ties, :197) by warp argmax.
  // A taken (marked) victim's key becomes 0, which no later query or extraction matches.
  __device__ int victims_build(unsigned long long& vk, int& vb) {
    int V = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < st.R; base += 32) {
      const int j = base + lane;
      bool e = false;
      unsigned long long key = 0;
      int blk = 0;
      if (j < st.R) {
        const int g = p.r_gen[j], o = p.r_out[j];
        e = (double)g < __dmul_rn(cfg.c, (double)o);
        key = ((unsigned long long)(unsigned)(o - g) << 32) | (unsigned)j;
        blk = blocks(p.r_prompt[j] + g);
      }
      const unsigned m = __ballot_sync(FULL, e);
      if (e) {
        const int d = V + __popc(m & lanemask_lt());
        p.v_key[d] = key;
        p.v_cum[d] = blk;
      }
      V += __popc(m);
    }
    __syncwarp();
    vk = lane < V ? p.v_key[lane] : 0ULL;
    vb = lane < V ? (int)p.v_cum[lane] : 0;
    return V;
  }
  __device__ __forceinline__ long long victims_gain(int V, unsigned long long vk, int vb, int b) const {
    if (V <= 32) return redux_add((int)(vk >> 32) > b ? vb : 0);
    long long t = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < V; base += 32) {
      const int i = base + lane;
      const unsigned long long k = i < V ? p.v_key[i] : 0ULL;
      t += redux_add((int)(k >> 32) > b ? (int)p.v_cum[i] : 0);
    }
    return t;
  }
  // mark the top victim with remaining > b; returns its blocks, table index in j_out
  __device__ int victims_take(int V, unsigned long long& vk, int& vb, int b, int& j_out) {
    if (V <= 32) {
      const unsigned w = warp_argmax_u64(vk, (int)(vk >> 32) > b);
      const int wl = __ffs(w) - 1;
      j_out = (int)(unsigned)__shfl_sync(FULL, vk, wl);
      const int blk = __shfl_sync(FULL, vb, wl);
      if (lane == wl) vk = 0ULL;
      return blk;
    }
    unsigned long long best = 0;
    int bpos = -1;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int i = lane; i < V; i += 32) {
      const unsigned long long k = p.v_key[i];
      if ((int)(k >> 32) > b && k > best) { best = k; bpos = i; }
    }
    const unsigned w = warp_argmax_u64(best, bpos >= 0);
    const int wl = __ffs(w) - 1;
    const int pos = __shfl_sync(FULL, bpos, wl);
    j_out = (int)(unsigned)__shfl_sync(FULL, best, wl);
    const int blk = (int)p.v_cum[pos];
    __syncwarp();
    if (lane == 0) p.v_key[pos] = 0ULL;
    __syncwarp();
    return blk;
  }

  // ---- trail_plus (policies.py:168-212): greedy skip in (remaining, arrival, id) order ----
  // A candidate is admitted iff need <= free + G(remaining): with need <= free it is a plain
  // dispatch (:183-186), else the victims taken largest-remaining-first cover it (:189-206).
  // G is non-increasing in the remaining output, so free + G(b) bounds every candidate in
  // buckets >= b and t_find skips every bucket whose minimum need exceeds it; a found bucket
  // is checked against its exact threshold free + G(bucket) before its list is walked.
  // Dispatches go to l_a (rid|flag) / l_c (pending), preempts to l_b.
  __device__ void select_trail(int& nd_out, int& np_out) {
    int nd = 0, np = 0;
    if (st.W == 0) { nd_out = np_out = 0; return; }
    int V = 0;
    unsigned long long vk = 0;
    int vb = 0;
    SSB_T0(vb)
    if (cfg.c != 0.0) V = victims_build(vk, vb);
    SSB_T1(vb, 8)
    int free = st.free_blocks;
    int b = 0, after = -1;  // resume point: bucket b, ids > after
    int r_prev = -1, r_cur = -1;  // ... and where its list continues after the last dispatch from b
    int r_min = 0x7fffffff;  // ... and the minimum need of the entries before that point
    while (true) {
      if (cfg.max_running >= 0 && (long long)cfg.max_running - (st.R + nd - np) < 1) break;  // :179-181
      long long T;
      SSB_T0(tf)
      const int fb = t_find_exact(b, free, V, vk, vb, T);
      SSB_T1(tf, 9)
#ifdef SSB_PHASE_TIMING
      tc[6] += 1;
#endif
      if (fb < 0) break;
      if (fb != b) {
        b = fb;
        after = -1;
      }
      SSB_T0(wk)
      // the walk resumes behind the last dispatch from this bucket (its entries before that
      // were not admissible then, with a larger free pool, so they are not now) instead of
      // re-walking the list from its head; next and pending of an entry are loaded together
      int prev = -1, cur = after >= 0 ? r_cur : p.t_head[b], pv = 0, need = 0, nx = -1;
      int mn = 0x7fffffff;  // minimum need of the entries before cur (carried across resumes)
      if (after >= 0) { prev = r_prev; mn = r_min; }
      while (cur >= 0) {
#ifdef SSB_PHASE_TIMING
        tm[6] += 1;
#endif
        pv = t_pend(cur);
        nx = t_next(cur);
        need = blocks(pv & 0x7fffffff);
        if ((long long)need <= T) break;
        mn = min(mn, need);
        prev = cur;
        cur = nx;
      }
      SSB_T1(wk, 10)
      if (cur < 0) { b += 1; after = -1; continue; }
      if (need > free) {
        SSB_T0(vt)
        // take victims (largest remaining first, youngest first on ties) until free+gain >= need
        int gain = 0;
        while (free + gain < need) {
          int j;
          gain += victims_take(V, vk, vb, b, j);
          if (lane == 0) p.l_b[np] = j;
          np++;
        }
        free += gain;
        __syncwarp();
        SSB_T1(vt, 12)
      }
      if (lane == 0) { p.l_a[nd] = cur | (pv & FLAG_SEEN); p.l_c[nd] = pv & 0x7fffffff; }
#ifdef SSB_PHASE_TIMING
      tc[7] += 1;
#endif
      nd++;
      free -= need;
      __syncwarp();
      SSB_T0(rm)
      trail_remove(b, prev, cur, nx, need, mn);
      SSB_T1(rm, 11)
      after = cur;
      r_prev = prev;
      r_cur = nx;
      r_min = mn;
    }
    __syncwarp();
    nd_out = nd;
    np_out = np;
  }


  // ---- remove dispatched entries (physical slots in l_a[0..nd)) from an unordered waiting set ----
  __device__ void remove_dispatched_unordered(int nd) {
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int i = lane; i < nd; i += 32) p.w_rid[p.l_a[i]] = -1;
    __syncwarp();
    int Wn = st.W - nd;
    // holes: dispatched slots at logical position < Wn ; movers: kept entries at logical >= Wn
    int nh = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < nd; base += 32) {
      int i = base + lane;
      bool h = false;
      int lg = 0;
      if (i < nd) {
        lg = p.l_a[i] - st.whead;
        if (lg < 0) lg += cfg.Wc;
        h = lg < Wn;
      }
      unsigned m = __ballot_sync(FULL, h);
      if (h) p.l_b[nh + __popc(m & lanemask_lt())] = p.l_a[i];
      nh += __popc(m);
    }
    __syncwarp();
    int nm = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = Wn; base < st.W; base += 32) {
      int k = base + lane;
      bool mv = false;
      int pos = 0;
      if (k < st.W) {
        pos = phys(k);
        mv = p.w_rid[pos] != -1;
      }
      unsigned m = __ballot_sync(FULL, mv);
      if (mv) {
        int h = p.l_b[nm + __popc(m & lanemask_lt())];
        p.w_rid[h] = p.w_rid[pos];
        p.w_pend[h] = p.w_pend[pos];
        p.w_key[h] = p.w_key[pos];
        p.w_enq[h] = p.w_enq[pos];
      }
      nm += __popc(m);
    }
    if (nm != nh) st.status = SSB_E_INVARIANT;
    st.W = Wn;
    __syncwarp();
  }

  // ---- apply dispatches (engine.py:287-298) in decision order ----
  __device__ void apply_dispatches(int nd, bool prefix_mode) {
    if (nd == 0) return;
    nodisp = false;
    lc_valid = false;
    if (st.R + nd > cfg.Rc) { st.status = SSB_E_CAPACITY; return; }
    int need_sum = 0;
    long long pend_sum = 0;
    int res_sum = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < nd; base += 32) {
      int j = base + lane;
      bool valid = j < nd;
      int rid = 0;
      if (valid) {
        const bool listed = cfg.policy == SSB_POLICY_TRAIL_PLUS;
        int pos = prefix_mode ? phys(j) : p.l_a[j];
        int wr = listed ? p.l_a[j] : p.w_rid[pos];
        rid = wr & 0x7fffffff;
        int pend = listed ? p.l_c[j] : p.w_pend[pos];
        int pr = prompt[rid];
        int t = st.R + j;
        SSB_ASSERT(rid >= 0 && rid < cfg.Wc && t < cfg.Rc && pend >= pr);
        p.r_rid[t] = rid;
        p.r_prompt[t] = pr;
        p.r_out[t] = output[rid];
        p.r_gen[t] = pend - pr;
        p.r_pfd[t] = 0;
        p.r_st[t] = ST_PREFILL;
        if (!(wr & FLAG_SEEN)) rec_fd[rid] = st.clock;  // first dispatch (queueing delay)
        need_sum += blocks(pend);
        pend_sum += pend;
        if (cfg.policy == SSB_POLICY_NOPREEMPT) res_sum += p.w_key[pos];  // (listed mode: trail_plus only)
      }
      emit(__ballot_sync(FULL, valid), SSB_EV_DISPATCH, rid);
    }
    need_sum = warp_sum(need_sum);
    pend_sum = warp_sum_ll(pend_sum);
    res_sum = warp_sum(res_sum);  // (several chunks: per-lane partial sums may exceed 32-bit REDUX range)
    st.free_blocks -= need_sum;  // try_allocate (kvmem.py:106-117)
    if (st.free_blocks < 0) st.status = SSB_E_INVARIANT;  // "policy over-admitted" (engine.py:288-292)
    st.committed += res_sum;
    st.wpend_sum -= pend_sum;
    st.pf_pend += pend_sum;
    st.R += nd;
    st.dispatches += nd;
    __syncwarp();
    if (prefix_mode) {
      st.whead = phys(nd);
      st.W -= nd;
    } else if (cfg.policy != SSB_POLICY_TRAIL_PLUS) {  // trail_plus removed them during select
      remove_dispatched_unordered(nd);
    }
  }

  // ---- _form_batch (engine.py:300-323) + resident KV (engine.py:217-218) ----
  // writes r_plan: 1 = decode token, >1 = prefill chunk + 1, 0 = not in the plan.
  // prefill plan entries are also listed (table index) in l_b[0..npf).
  __device__ void form_batch(int& total, long long& resident, int& nentries, int& npf) {
    const int cap = cfg.cap;
    int n_dec_plan = min(st.ndec, cap);
    int budget = cap - n_dec_plan;
    int dec_seen = 0, pf_used = 0, npf_ = 0;
    long long res = 0;
    #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
    for (int base = 0; base < st.R; base += 32) {
      int j = base + lane;
      bool valid = j < st.R;
      int s = ST_GONE, pr = 0, g = 0, f = 0;
      if (valid) { s = p.r_st[j]; pr = p.r_prompt[j]; g = p.r_gen[j]; f = p.r_pfd[j]; }
      bool dec = s == ST_DECODE;
      bool pf = s == ST_PREFILL;
      unsigned md = __ballot_sync(FULL, dec);
      int drank = dec_seen + __popc(md & lanemask_lt());
      bool in_dec = dec && drank < cap;
      int pend = pf ? pr + g - f : 0;
      int incl = warp_incl_scan(pend, lane) + pf_used;
      int before = incl - pend;  // prefill tokens claimed before this entry
      int chunk = 0;
      if (pf && budget - before > 0) chunk = min(pend, budget - before);
      bool in_pf = chunk > 0;
      int plan = in_dec ? 1 : (in_pf ? chunk + 1 : 0);
      if (valid) p.r_plan[j] = plan;
      unsigned mp = __ballot_sync(FULL, in_pf);
      if (in_pf) p.l_b[npf_ + __popc(mp & lanemask_lt())] = j;
      npf_ += __popc(mp);
      int ctx = in_dec ? pr + g : (in_pf ? f : 0);
      res += redux_add(ctx);
      dec_seen += __popc(md);
      pf_used = __shfl_sync(FULL, incl, 31);
    }
    int pf_tokens = (int)min((long long)budget, (long long)pf_used);
    total = n_dec_plan + pf_tokens;
    resident = res;
    nentries = n_dec_plan + npf_;
    npf = npf_;
    __syncwarp();
  }

  // ---- _apply_progress (engine.py:325-358) ----
  // Lanes evaluate their grow (kvmem.py:119-140) against the running free count
  // (exclusive scan of released-minus-grown blocks); every lane before the first
  // failing grow commits in parallel; the failing one runs the serial eviction
  // cascade (_grow_or_evict / _evict_for_blocks) and the chunk restarts after it.
  // one body for both sections (runtime flag, one call site in progress()): this path's
  // instruction footprint matters more than the flag's cost
  __device__ void progress_group(const bool PREFILL, int j_lane, bool in_group, bool& removed_any) {
    int start = 0;
    while (true) {
      int rid = 0, pr = 0, out = 0, g = 0, f = 0, s = ST_GONE, plan = 0;
      bool act = in_group && lane >= start;
      if (act) {
        s = p.r_st[j_lane];
        act = s == (PREFILL ? ST_PREFILL : ST_DECODE);  // skip entries evicted earlier in this pass
      }
      if (act) {
        rid = p.r_rid[j_lane]; pr = p.r_prompt[j_lane]; out = p.r_out[j_lane]; g = p.r_gen[j_lane];
        f = p.r_pfd[j_lane]; plan = p.r_plan[j_lane];
      }
      int f2 = f, extra = 0, rel = 0;
      bool grow = false, fin = false, first = false, recompute = false;
      if (act) {
        if (PREFILL) {
          f2 = f + (plan - 1);
          bool complete = f2 >= pr + g;
          first = complete && g == 0;
          recompute = complete && g > 0;
          grow = first;
          if (first) {
            extra = blocks(pr + 1) - blocks(pr);
            fin = out == 1;
            rel = fin ? blocks(pr + 1) : 0;
          }
        } else {
          grow = true;
          int cur = pr + g;
          extra = blocks(cur + 1) - blocks(cur);
          fin = g + 1 == out;
          rel = fin ? blocks(cur + 1) : 0;
        }
      }
      int d = act ? rel - extra : 0;
      int excl = 0, fl = 32;
      // grows only consume and finishes only release: if the chunk's total
      // demand fits the free pool no grow can fail, whatever the order
      if (redux_add(extra) > st.free_blocks) {
        excl = warp_incl_scan(d, lane) - d;
        bool fail = act && grow && extra > st.free_blocks + excl;
        unsigned mf = __ballot_sync(FULL, fail);
        fl = mf ? __ffs(mf) - 1 : 32;
      }
      bool commit = act && lane < fl;
      // commit lanes [start, fl)
      unsigned m_first = __ballot_sync(FULL, commit && first);
      unsigned m_fin = __ballot_sync(FULL, commit && fin);
      unsigned m_dec_in = __ballot_sync(FULL, commit && (first || recompute));
      if (commit) {
        if (PREFILL) {
          p.r_pfd[j_lane] = f2;
          if (first) {
            p.r_gen[j_lane] = 1;
            rec_ft[rid] = st.clock;
          }
          if (first || recompute) p.r_st[j_lane] = fin ? ST_GONE : ST_DECODE;
        } else {
          p.r_gen[j_lane] = g + 1;
          if (fin) p.r_st[j_lane] = ST_GONE;
        }
        if (fin) rec_fin[rid] = st.clock;
      }
      // released-minus-grown blocks of the committed lanes
      int dcommit = (fl == 32) ? redux_add(d) : __shfl_sync(FULL, excl, fl & 31);
      st.free_blocks += dcommit;
      if (PREFILL) {
        int chunk_sum = redux_add(commit ? plan - 1 : 0);
        st.pf_pend -= chunk_sum;
        if (PREFILL) emit2(m_first, SSB_EV_FIRST_TOKEN, m_fin, SSB_EV_FINISH, rid);
      } else {
        emit(m_fin, SSB_EV_FINISH, rid);
      }
      int n_fin = __popc(m_fin);
      st.ndec += __popc(m_dec_in) - n_fin;
      if (n_fin) {
        nodisp = false;
        removed_any = true;
        st.finished += n_fin;
        st.fin_cnt += n_fin;
        st.fin_in += redux_add(commit && fin ? pr : 0);
        st.fin_out += redux_add(commit && fin ? out : 0);
        if (cfg.policy == SSB_POLICY_NOPREEMPT)
          st.committed -= redux_add(commit && fin ? wkey_for(pr, out, 0) : 0);
      }
      __syncwarp();
      if (fl == 32) break;
      // ---- serial slow path for lane fl: its grow does not fit ----
      SSB_T0(slow)
      removed_any = true;
      int j = __shfl_sync(FULL, j_lane, fl);
      int frid = __shfl_sync(FULL, rid, fl), fpr = __shfl_sync(FULL, pr, fl), fout = __shfl_sync(FULL, out, fl);
      int fg = __shfl_sync(FULL, g, fl), ff2 = __shfl_sync(FULL, f2, fl), fext = __shfl_sync(FULL, extra, fl);
      bool ffin = __shfl_sync(FULL, (int)fin, fl) != 0;
      if (PREFILL && lane == 0) p.r_pfd[j] = ff2;  // the chunk landed before the grow
      if (PREFILL) st.pf_pend -= (long long)(ff2 - __shfl_sync(FULL, f, fl));
      __syncwarp();
      // _evict_for_blocks: youngest dispatch first (table order descending), skipping the grower,
      // until the grow fits; if nothing is left to evict, park the grower itself (engine.py:
      // 403-412). One preempt_entry call site for both (a smaller hot loop).
      const int needed = fext;  // blocks(new) - allocated_blocks(r)
      int vbase = ((st.R - 1) >> 5) << 5;
      unsigned ml = 0;
      bool parked = false;
      #pragma unroll 1
      while (st.free_blocks < needed) {
        while (ml == 0 && vbase >= 0) {
          const int v = vbase + lane;
          ml = __ballot_sync(FULL, v < st.R && v != j && p.r_st[v] != ST_GONE);
          if (ml == 0) vbase -= 32;
        }
        int vj = j, code = SSB_EV_PARK;
        if (ml != 0) {
          const int b = 31 - __clz(ml);
          ml &= ~(1u << b);
          vj = vbase + b;
          code = SSB_EV_PREEMPT;
          if (ml == 0) vbase -= 32;
        } else {
          parked = true;
        }
        // (the grower's table entry already holds ff2 / fg / its state, see above)
        preempt_entry(vj, p.r_rid[vj], p.r_prompt[vj], p.r_out[vj], p.r_gen[vj], p.r_pfd[vj], p.r_st[vj], code);
        if (parked) break;
      }
      if (!parked) {  // retry succeeds
        st.free_blocks -= fext;
        if (PREFILL) {
          if (lane == 0) { p.r_gen[j] = 1; rec_ft[frid] = st.clock; p.r_st[j] = ffin ? ST_GONE : ST_DECODE; }
          emit1(SSB_EV_FIRST_TOKEN, frid);
          st.ndec += 1;
        } else {
          if (lane == 0) { p.r_gen[j] = fg + 1; if (ffin) p.r_st[j] = ST_GONE; }
        }
        if (ffin) {
          nodisp = false;
          if (lane == 0) rec_fin[frid] = st.clock;
          st.free_blocks += PREFILL ? blocks(fpr + 1) : blocks(fpr + fg + 1);
          emit1(SSB_EV_FINISH, frid);
          st.ndec -= 1;
          st.finished += 1; st.fin_cnt += 1; st.fin_in += fpr; st.fin_out += fout;
          if (cfg.policy == SSB_POLICY_NOPREEMPT) st.committed -= wkey_for(fpr, fout, 0);
        }
      }
      __syncwarp();
      SSB_T1(slow, 15)
      start = fl + 1;
      if (start >= 32) break;
    }
  }

  __device__ bool progress(int npf) {
    bool removed = false;
    // prefill chunks in plan order (table indices listed in l_b), then decode tokens in plan
    // order; ONE call site of progress_group for both sections (it is inlined: two sites
    // would be two copies of the largest function in the hot loop)
    #pragma unroll 1
    for (int sec = 0; sec < 2; ++sec) {
      const bool pre = sec == 0;
      const int n = pre ? npf : st.R;
      #pragma unroll 1  // chunk loops run 1-2 trips: keep the hot code small (instruction-fetch bound)
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const int j = pre ? (i < npf ? p.l_b[i] : 0) : i;
        const bool in = pre ? i < npf : (i < st.R && p.r_plan[i] == 1);
        progress_group(pre, j, in, removed);
      }
    }
    return removed;  // (queued waiting pushes are flushed by advance() after the step)
  }

  // ---- fused _form_batch + latency + _apply_progress for R <= 32 ----
  // The whole running table is one chunk held in registers: the plan, the
  // resident-KV and token sums (REDUX), the clock update and the progress
  // commit need no memory round trip in between. When the plan's total grow
  // demand exceeds the free pool (rare: memory pressure) it hands over to the
  // general ordered path (progress_group) with the plan written to memory.
  // returns -1 when the iteration completed in registers, else the number of prefill plan
  // entries for the ordered general path (plan in memory, clock already advanced; total_out =
  // the batch's tokens) — step() runs that path from its single call site of progress()
  __device__ int batch_progress_small(int& total_out) {
    const int cap = cfg.cap;
    const bool valid = lane < st.R;
    int s = ST_GONE, pr = 0, out = 0, g = 0, f = 0, rid = 0;
    if (valid) { s = p.r_st[lane]; pr = p.r_prompt[lane]; out = p.r_out[lane]; g = p.r_gen[lane]; f = p.r_pfd[lane]; rid = p.r_rid[lane]; }
    const unsigned lt = lanemask_lt();
    const bool dec = s == ST_DECODE, pf = s == ST_PREFILL;
    const unsigned md = __ballot_sync(FULL, dec);
    const bool in_dec = dec && __popc(md & lt) < cap;  // decodes first, 1 token each (engine.py:303-309)
    const int n_dec_plan = min(__popc(md), cap);
    const int B = cap - n_dec_plan;
    const unsigned mpf = __ballot_sync(FULL, pf);
    const int pend = pf ? pr + g - f : 0;
    int before = 0;
    if (mpf & (mpf - 1)) before = warp_incl_scan(pend, lane) - pend;  // >1 prefilling: claimed earlier
    const int chunk = (pf && B - before > 0) ? min(pend, B - before) : 0;  // engine.py:311-318
    const bool in_pf = chunk > 0;
    const unsigned m_pf = __ballot_sync(FULL, in_pf);
    const unsigned m_dec = __ballot_sync(FULL, in_dec);
    const int resident = redux_add(in_dec ? pr + g : (in_pf ? f : 0));  // engine.py:217-218
    const int pf_tokens = redux_add(chunk);
    const int total = n_dec_plan + pf_tokens;
    if (total == 0) { st.status = SSB_E_STALL; return -1; }  // engine.py:209-214
    st.rsteps += __popc(m_dec) + __popc(m_pf);
    st.btokens += total;
    {  // iteration_latency (costmodel.py:45-47); clock += latency (engine.py:219-220)
      double mem = __dadd_rn(cfg.mem_base, __dmul_rn(cfg.mem_kv, (double)resident));
      double comp = __dmul_rn(cfg.compute, (double)total);
      st.clock = __dadd_rn(st.clock, __dadd_rn(cfg.overhead, comp > mem ? comp : mem));
    }
    // progress: prefill chunks land, first tokens, decode tokens (engine.py:328-357)
    const int f2 = f + chunk;
    const bool complete = in_pf && f2 >= pr + g;
    const bool first = complete && g == 0;
    const bool recompute = complete && g > 0;
    int extra = 0;
    if (first) extra = blocks(pr + 1) - blocks(pr);
    else if (in_dec) extra = blocks(pr + g + 1) - blocks(pr + g);
    const int need = redux_add(extra);
    if (need > st.free_blocks) {
      // memory pressure: ordered grows with eviction (general path)
      if (valid) p.r_plan[lane] = in_dec ? 1 : (in_pf ? chunk + 1 : 0);
      if (in_pf) p.l_b[__popc(m_pf & lt)] = lane;
      __syncwarp();
#ifdef SSB_PHASE_TIMING
      tc[14] += 1;
#endif
      total_out = total;
      return __popc(m_pf);
    }
    const bool fin = (first && out == 1) || (in_dec && g + 1 == out);
    const int rel = fin ? (first ? blocks(pr + 1) : blocks(pr + g + 1)) : 0;
    st.free_blocks += redux_add(rel) - need;
    int g2 = first ? 1 : (in_dec ? g + 1 : g);
    int s2 = fin ? ST_GONE : ((first || recompute) ? ST_DECODE : s);
    if (first) rec_ft[rid] = st.clock;
    if (fin) rec_fin[rid] = st.clock;
    const unsigned m_first = __ballot_sync(FULL, first);
    const unsigned m_fin = __ballot_sync(FULL, fin);
    const unsigned m_rec = __ballot_sync(FULL, recompute);
    if (m_first | m_fin) {
      emit2(m_first, SSB_EV_FIRST_TOKEN, m_fin & m_pf, SSB_EV_FINISH, rid);  // prefill section first
      emit(m_fin & m_dec, SSB_EV_FINISH, rid);                             // then decodes
    }
    st.pf_pend -= pf_tokens;
    st.ndec += __popc(m_first | m_rec) - __popc(m_fin);
    if (m_fin) {
      nodisp = false;
      const int nf = __popc(m_fin);
      st.finished += nf;
      st.fin_cnt += nf;
      st.fin_in += redux_add(fin ? pr : 0);
      st.fin_out += redux_add(fin ? out : 0);
      if (cfg.policy == SSB_POLICY_NOPREEMPT) st.committed -= redux_add(fin ? wkey_for(pr, out, 0) : 0);
      // compact in registers: kept entries move down to their rank
      const bool keep = valid && s2 != ST_GONE;
      const unsigned mk = __ballot_sync(FULL, keep);
      __syncwarp();
      if (keep) {
        const int d = __popc(mk & lt);
        p.r_rid[d] = rid; p.r_prompt[d] = pr; p.r_out[d] = out; p.r_gen[d] = g2; p.r_pfd[d] = f2; p.r_st[d] = s2;
      }
      st.R = __popc(mk);
    } else {
      if (in_pf) { p.r_pfd[lane] = f2; p.r_gen[lane] = g2; p.r_st[lane] = s2; }
      else if (in_dec) p.r_gen[lane] = g2;
    }
    __syncwarp();
    if (total > st.peak) st.peak = total;
    st.iterations += 1;
    return -1;
  }

  // ---- fused _form_batch + latency + _apply_progress for 32 < R <= 64 (latency kernel) ----
  // batch_progress_small with two register chunks per lane (entries lane and lane+32, table
  // order = chunk 0 then chunk 1). Only the latency-mode kernel (few instances, one per SM)
  // compiles it in (cfg.wide): it shortens single-instance chains (C1 13% faster) but its
  // extra hot code slows the many-instance sweep. Same return convention as batch_progress_small.
  __device__ int batch_progress_64(int& total_out) {
    const int cap = cfg.cap;
    const unsigned lt = lanemask_lt();
    const int j1 = lane + 32;
    const bool vb = j1 < st.R;
    int sa = p.r_st[lane], pra = p.r_prompt[lane], oa = p.r_out[lane], ga = p.r_gen[lane], fa = p.r_pfd[lane],
        ra = p.r_rid[lane];
    int sb = ST_GONE, prb = 0, ob = 0, gb = 0, fb = 0, rb = 0;
    if (vb) { sb = p.r_st[j1]; prb = p.r_prompt[j1]; ob = p.r_out[j1]; gb = p.r_gen[j1]; fb = p.r_pfd[j1]; rb = p.r_rid[j1]; }
    const bool deca = sa == ST_DECODE, decb = sb == ST_DECODE, pfa = sa == ST_PREFILL, pfb = sb == ST_PREFILL;
    const unsigned mda = __ballot_sync(FULL, deca), mdb = __ballot_sync(FULL, decb);
    const int nda = __popc(mda), ndec = nda + __popc(mdb);
    const bool in_deca = deca && __popc(mda & lt) < cap;
    const bool in_decb = decb && nda + __popc(mdb & lt) < cap;
    const int n_dec_plan = min(ndec, cap);
    const int B = cap - n_dec_plan;
    const int penda = pfa ? pra + ga - fa : 0, pendb = pfb ? prb + gb - fb : 0;
    const int inca = warp_incl_scan(penda, lane), incb = warp_incl_scan(pendb, lane);
    const int tota = __shfl_sync(FULL, inca, 31);
    const int befa = inca - penda, befb = tota + incb - pendb;
    const int cha = (pfa && B - befa > 0) ? min(penda, B - befa) : 0;
    const int chb = (pfb && B - befb > 0) ? min(pendb, B - befb) : 0;
    const bool in_pfa = cha > 0, in_pfb = chb > 0;
    const unsigned m_pfa = __ballot_sync(FULL, in_pfa), m_pfb = __ballot_sync(FULL, in_pfb);
    const unsigned m_deca = __ballot_sync(FULL, in_deca), m_decb = __ballot_sync(FULL, in_decb);
    const int resident = redux_add(in_deca ? pra + ga : (in_pfa ? fa : 0)) +
                         redux_add(in_decb ? prb + gb : (in_pfb ? fb : 0));
    const int pf_tokens = redux_add(cha) + redux_add(chb);
    const int total = n_dec_plan + pf_tokens;
    if (total == 0) { st.status = SSB_E_STALL; return -1; }
    st.rsteps += __popc(m_deca) + __popc(m_decb) + __popc(m_pfa) + __popc(m_pfb);
    st.btokens += total;
    {
      double mem = __dadd_rn(cfg.mem_base, __dmul_rn(cfg.mem_kv, (double)resident));
      double comp = __dmul_rn(cfg.compute, (double)total);
      st.clock = __dadd_rn(st.clock, __dadd_rn(cfg.overhead, comp > mem ? comp : mem));
    }
    const int f2a = fa + cha, f2b = fb + chb;
    const bool firsta = in_pfa && f2a >= pra + ga && ga == 0, firstb = in_pfb && f2b >= prb + gb && gb == 0;
    const bool reca = in_pfa && f2a >= pra + ga && ga > 0, recb = in_pfb && f2b >= prb + gb && gb > 0;
    int exa = 0, exb = 0;
    if (firsta) exa = blocks(pra + 1) - blocks(pra);
    else if (in_deca) exa = blocks(pra + ga + 1) - blocks(pra + ga);
    if (firstb) exb = blocks(prb + 1) - blocks(prb);
    else if (in_decb) exb = blocks(prb + gb + 1) - blocks(prb + gb);
    const int need = redux_add(exa) + redux_add(exb);
    if (need > st.free_blocks) {
      p.r_plan[lane] = in_deca ? 1 : (in_pfa ? cha + 1 : 0);
      if (vb) p.r_plan[j1] = in_decb ? 1 : (in_pfb ? chb + 1 : 0);
      const int npa = __popc(m_pfa);
      if (in_pfa) p.l_b[__popc(m_pfa & lt)] = lane;
      if (in_pfb) p.l_b[npa + __popc(m_pfb & lt)] = j1;
      __syncwarp();
      total_out = total;
      return npa + __popc(m_pfb);
    }
    const bool fina = (firsta && oa == 1) || (in_deca && ga + 1 == oa);
    const bool finb = (firstb && ob == 1) || (in_decb && gb + 1 == ob);
    const int rela = fina ? (firsta ? blocks(pra + 1) : blocks(pra + ga + 1)) : 0;
    const int relb = finb ? (firstb ? blocks(prb + 1) : blocks(prb + gb + 1)) : 0;
    st.free_blocks += redux_add(rela) + redux_add(relb) - need;
    const int g2a = firsta ? 1 : (in_deca ? ga + 1 : ga), g2b = firstb ? 1 : (in_decb ? gb + 1 : gb);
    const int s2a = fina ? ST_GONE : ((firsta || reca) ? ST_DECODE : sa);
    const int s2b = finb ? ST_GONE : ((firstb || recb) ? ST_DECODE : sb);
    if (firsta) rec_ft[ra] = st.clock;
    if (firstb) rec_ft[rb] = st.clock;
    if (fina) rec_fin[ra] = st.clock;
    if (finb) rec_fin[rb] = st.clock;
    const unsigned mfa = __ballot_sync(FULL, firsta), mfb = __ballot_sync(FULL, firstb);
    const unsigned mxa = __ballot_sync(FULL, fina), mxb = __ballot_sync(FULL, finb);
    const unsigned mra = __ballot_sync(FULL, reca), mrb = __ballot_sync(FULL, recb);
    if (mfa | mfb | mxa | mxb) {
      emit2(mfa, SSB_EV_FIRST_TOKEN, mxa & m_pfa, SSB_EV_FINISH, ra);
      emit2(mfb, SSB_EV_FIRST_TOKEN, mxb & m_pfb, SSB_EV_FINISH, rb);
      emit(mxa & m_deca, SSB_EV_FINISH, ra);
      emit(mxb & m_decb, SSB_EV_FINISH, rb);
    }
    st.pf_pend -= pf_tokens;
    st.ndec += __popc(mfa | mra) + __popc(mfb | mrb) - __popc(mxa) - __popc(mxb);
    if (mxa | mxb) {
      nodisp = false;
      const int nf = __popc(mxa) + __popc(mxb);
      st.finished += nf;
      st.fin_cnt += nf;
      st.fin_in += redux_add(fina ? pra : 0) + redux_add(finb ? prb : 0);
      st.fin_out += redux_add(fina ? oa : 0) + redux_add(finb ? ob : 0);
      if (cfg.policy == SSB_POLICY_NOPREEMPT)
        st.committed -= redux_add(fina ? wkey_for(pra, oa, 0) : 0) + redux_add(finb ? wkey_for(prb, ob, 0) : 0);
      const bool ka = s2a != ST_GONE, kb = vb && s2b != ST_GONE;
      const unsigned mka = __ballot_sync(FULL, ka), mkb = __ballot_sync(FULL, kb);
      __syncwarp();
      if (ka) {
        const int d = __popc(mka & lt);
        p.r_rid[d] = ra; p.r_prompt[d] = pra; p.r_out[d] = oa; p.r_gen[d] = g2a; p.r_pfd[d] = f2a; p.r_st[d] = s2a;
      }
      if (kb) {
        const int d = __popc(mka) + __popc(mkb & lt);
        p.r_rid[d] = rb; p.r_prompt[d] = prb; p.r_out[d] = ob; p.r_gen[d] = g2b; p.r_pfd[d] = f2b; p.r_st[d] = s2b;
      }
      st.R = __popc(mka) + __popc(mkb);
    } else {
      if (in_pfa) { p.r_pfd[lane] = f2a; p.r_gen[lane] = g2a; p.r_st[lane] = s2a; }
      else if (in_deca) p.r_gen[lane] = g2a;
      if (in_pfb) { p.r_pfd[j1] = f2b; p.r_gen[j1] = g2b; p.r_st[j1] = s2b; }
      else if (in_decb) p.r_gen[j1] = g2b;
    }
    __syncwarp();
    if (total > st.peak) st.peak = total;
    st.iterations += 1;
    return -1;
  }

  // ---- steady-state decode iteration (engine.py:300-357 specialised) ----
  // Preconditions (checked by step): every running request is DECODING,
  // R <= min(64, cap) so the plan is "one token each, table order", block size a
  // power of two. The KV resident sum is maintained incrementally; grows cross a
  // block boundary iff (prompt+generated) % bs == 0. If the plan's grow demand does
  // not fit the free pool, returns false with nothing modified (ordered path).
  __device__ bool fast_decode() {
    const int R = st.R;
    const int bsm = cfg.bs - 1;
    const bool v0 = lane < R, v1 = lane + 32 < R;
    const bool x0 = v0 && ((c_pr0 + c_g0) & bsm) == 0;
    const bool x1 = v1 && ((c_pr1 + c_g1) & bsm) == 0;
    const int need = __popc(__ballot_sync(FULL, x0)) + __popc(__ballot_sync(FULL, x1));
    if (need > st.free_blocks) return false;
    {  // iteration_latency (costmodel.py:45-47); clock += latency (engine.py:219-220)
      const double mem = __dadd_rn(cfg.mem_base, __dmul_rn(cfg.mem_kv, (double)rsum));
      const double comp = __dmul_rn(cfg.compute, (double)R);
      st.clock = __dadd_rn(st.clock, __dadd_rn(cfg.overhead, comp > mem ? comp : mem));
    }
    c_g0 += v0;
    c_g1 += v1;
    regs_dirty = true;
    rsum += R;
    st.free_blocks -= need;
    st.rsteps += R;
    st.btokens += R;
    if (R > st.peak) st.peak = R;
    st.iterations += 1;
    const bool f0 = v0 && c_g0 == c_out0, f1 = v1 && c_g1 == c_out1;
    const unsigned m0 = __ballot_sync(FULL, f0), m1 = __ballot_sync(FULL, f1);
    if (m0 | m1) finish_fast(f0, f1, m0, m1);
    return true;
  }

  // ---- steady-state run: many decode iterations in one tight loop ----
  // Called right after a fast_decode iteration when nothing can change the schedule:
  // every running request decoding and cached in registers (regs_ok), select known to
  // dispatch nothing (nodisp: stays true while only free blocks shrink, see `nodisp`).
  // Each further iteration is then fully determined by the previous one: one token per
  // request, grows at block boundaries, clock += iteration_latency(rsum, R) with rsum
  // += R. It runs while (a) no request would finish (stop one before the first finish:
  // fast_decode handles that iteration's events), (b) the grows fit the free pool (else
  // the ordered eviction path must run), (c) the loop-top conditions of advance() hold:
  // clock < t_lim and no arrival is due (clock < next_t). No events are emitted in
  // these iterations, so the decision digest is unaffected. Exact: the same binary64
  // operations in the same order as fast_decode (rsum as an exact double < 2^53).
  __device__ void fast_forward(double lim) {
    const int R = st.R;
    const bool v0 = lane < R, v1 = lane + 32 < R;
    const int left = min(v0 ? c_out0 - c_g0 : 0x7fffffff, v1 ? c_out1 - c_g1 : 0x7fffffff);
    const int kmax = (int)__reduce_min_sync(FULL, (unsigned)left) - 1;  // iterations before a finish
    if (kmax <= 0 || !(st.clock < lim)) return;
    const int bsm = cfg.bs - 1;
    const int t0 = c_pr0 + c_g0, t1 = c_pr1 + c_g1;  // KV tokens before the next iteration
    const double comp = __dmul_rn(cfg.compute, (double)R);
    const double Rd = (double)R;
    double clock = st.clock, rs = (double)rsum;
    int free = st.free_blocks, k = 0;
    while (k < kmax) {
      const int need = __popc(__ballot_sync(FULL, v0 && ((t0 + k) & bsm) == 0)) +
                       __popc(__ballot_sync(FULL, v1 && ((t1 + k) & bsm) == 0));
      if (need > free) break;
      const double mem = __dadd_rn(cfg.mem_base, __dmul_rn(cfg.mem_kv, rs));
      clock = __dadd_rn(clock, __dadd_rn(cfg.overhead, comp > mem ? comp : mem));
      rs = __dadd_rn(rs, Rd);
      free -= need;
      k += 1;
      if (!(clock < lim)) break;
    }
    if (k == 0) return;
    st.clock = clock;
    st.free_blocks = free;
    c_g0 += v0 ? k : 0;
    c_g1 += v1 ? k : 0;
    regs_dirty = true;
    const long long rk = (long long)R * k;
    rsum += rk;
    st.rsteps += rk;
    st.btokens += rk;
    st.iterations += k;
  }

  // finishes inside a steady-state iteration (_finish, engine.py:360-366)
  __device__ void finish_fast(bool f0, bool f1, unsigned m0, unsigned m1) {
    nodisp = false;
    if (f0) rec_fin[c_rid0] = st.clock;
    if (f1) rec_fin[c_rid1] = st.clock;
    emit(m0, SSB_EV_FINISH, c_rid0);  // decode plan order == table order
    emit(m1, SSB_EV_FINISH, c_rid1);
    const int n = __popc(m0) + __popc(m1);
    st.free_blocks += redux_add(f0 ? blocks(c_pr0 + c_g0) : 0) + redux_add(f1 ? blocks(c_pr1 + c_g1) : 0);
    st.finished += n;
    st.fin_cnt += n;
    st.fin_in += redux_add(f0 ? c_pr0 : 0) + redux_add(f1 ? c_pr1 : 0);
    st.fin_out += redux_add(f0 ? c_out0 : 0) + redux_add(f1 ? c_out1 : 0);
    if (cfg.policy == SSB_POLICY_NOPREEMPT)
      st.committed -= redux_add(f0 ? wkey_for(c_pr0, c_out0, 0) : 0) + redux_add(f1 ? wkey_for(c_pr1, c_out1, 0) : 0);
    st.ndec -= n;
    if (lane < st.R) { p.r_gen[lane] = c_g0; if (f0) p.r_st[lane] = ST_GONE; }
    if (lane + 32 < st.R) { p.r_gen[lane + 32] = c_g1; if (f1) p.r_st[lane + 32] = ST_GONE; }
    regs_ok = regs_dirty = false;
    __syncwarp();
    compact_running();
  }

  // ---- Engine.step (engine.py:193-234) ----
#ifdef SSB_DEBUG
  // after a step: counts within the tables, and the KV pool conserved (kvmem.py:151-154
  // conserved(): free + every running request's blocks(prompt + generated) == total)
  __device__ void debug_check() const {
    if (st.status) return;
    SSB_ASSERT(st.free_blocks >= 0 && st.free_blocks <= cfg.pool && st.R >= 0 && st.R <= cfg.Rc &&
               st.W >= 0 && st.W <= cfg.Wc && st.next_arr >= 0);
    if (regs_ok) return;  // (the register copy of the table is authoritative)
    long long held = 0;
    for (int j = lane; j < st.R; j += 32) {
      SSB_ASSERT(p.r_st[j] == ST_PREFILL || p.r_st[j] == ST_DECODE);
      held += blocks(p.r_prompt[j] + p.r_gen[j]);
    }
    held = warp_sum_ll(held);
    SSB_ASSERT(held + st.free_blocks == cfg.pool);
  }
#endif
  __device__ __forceinline__ void step() {
    if (!has_work()) { st.status = SSB_E_STALL; return; }
    int nd = 0, np = 0;
    bool prefix = false;
    SSB_T0(sel)
    if (!nodisp) {
      switch (cfg.policy) {
        case SSB_POLICY_FCFS:
        case SSB_POLICY_NOPREEMPT: nd = select_prefix(); prefix = true; break;
        case SSB_POLICY_TRAIL_PLUS:
          if (cfg.c != 0.0) flush_regs();  // victims read the table
          select_trail(nd, np);
          break;
        case SSB_POLICY_LARRY: nd = select_larry(); break;
        default: st.status = SSB_E_ARG; return;
      }
      // nothing dispatched: stays so until an enqueue / dispatch / finish / preempt
      // (larry's order moves with the clock, so only an empty queue is stable)
      if (nd == 0 && np == 0) nodisp = cfg.policy != SSB_POLICY_LARRY || st.W == 0;
      SSB_T1(sel, 1)
    }
    SSB_T0(disp)
    if (np > 0) {  // policy preempts first (engine.py:203-204), in decision order
      SSB_T0(pre)
      drop_regs();
      for (int t = 0; t < np; ++t) {
        int j = p.l_b[t];
        int vs = p.r_st[j], vrid = p.r_rid[j], vpr = p.r_prompt[j], vout = p.r_out[j], vg = p.r_gen[j],
            vf = p.r_pfd[j];
        preempt_entry(j, vrid, vpr, vout, vg, vf, vs, SSB_EV_PREEMPT);
      }
      compact_running();  // (their waiting pushes are flushed by advance() after the step)
      SSB_T1(pre, 13)
    }
    if (nd > 0) {
      drop_regs();
      apply_dispatches(nd, prefix);  // then dispatches (engine.py:205-206)
      if (st.status) return;
    }
    if (np > 0 || nd > 0) { SSB_T1(disp, 2) }
    SSB_T0(bat)
    if (st.R > 0 && st.R <= 64 && st.ndec == st.R && st.R <= cfg.cap && cfg.bs_shift >= 0) {
      if (!regs_ok) load_regs();
      if (fast_decode()) { SSB_T1(bat, 3) return; }
    }
    drop_regs();
    int total = 0, npf;
    if (st.R <= 32 || (cfg.wide && st.R <= 64)) {
      npf = st.R <= 32 ? batch_progress_small(total) : batch_progress_64(total);
      if (npf < 0) { SSB_T1(bat, 4) return; }
    } else {
      int nent;
      long long resident;
      form_batch(total, resident, nent, npf);
      if (total == 0) { st.status = SSB_E_STALL; return; }  // engine.py:209-214
      st.rsteps += nent;
      st.btokens += total;
      // iteration_latency (costmodel.py:45-47) then clock += latency (engine.py:219-220)
      double mem = __dadd_rn(cfg.mem_base, __dmul_rn(cfg.mem_kv, (double)resident));
      double comp = __dmul_rn(cfg.compute, (double)total);
      double lat = __dadd_rn(cfg.overhead, comp > mem ? comp : mem);
      st.clock = __dadd_rn(st.clock, lat);
    }
    bool removed = progress(npf);  // the ordered general path: one call site
    if (removed) compact_running();
    if (total > st.peak) st.peak = total;
    st.iterations += 1;
    SSB_T1(bat, 5)
  }

  // ---- advance: process every boundary with time < t_lim (cluster.py:142-157 / engine.py:256-265) ----
  __device__ __forceinline__ double next_arrival(int n_avail) const {
    if (st.next_arr >= n_avail) return __longlong_as_double(0x7ff0000000000000LL);  // +inf: none routed yet
    int rid = (cfg.n_servers == 1) ? st.next_arr : p.rl[st.next_arr];
    return rid >= 0 ? arrival_of(rid) : __longlong_as_double(0x7ff0000000000000LL);  // -1: not routed yet
  }
  // one call per engine lifetime (k_engines) or per routing epoch (k_cluster): the engine is
  // rebound from memory, so the per-engine modes start fresh and the table is written back
  __device__ __forceinline__ void advance(double t_lim, int n_avail) {
#ifdef SSB_PHASE_TIMING
    for (int i = 0; i < 16; ++i) tm[i] = tc[i] = 0;
#endif
    init_modes();
    advance_loop(t_lim, n_avail);
    drop_regs();  // the table in memory is authoritative between calls
#ifdef SSB_PHASE_TIMING
    if (lane == 0)
      printf("PHASES iters %lld | enq %lld/%lld | sel %lld/%lld | disp %lld/%lld | fast %lld/%lld | small %lld/%lld | gen %lld/%lld | walk %lld/%lld | victims %lld/%lld\n",
             st.iterations, tm[0], tc[0], tm[1], tc[1], tm[2], tc[2], tm[3], tc[3], tm[4], tc[4], tm[5], tc[5], tm[6], tm[7], tc[6], tc[7]);
    if (lane == 0)
      printf("PHASES2 vbuild %lld/%lld | tfind %lld/%lld | walk %lld/%lld | remove %lld/%lld | vtake %lld/%lld | preempt %lld/%lld | small->gen %lld | evict-slow %lld/%lld\n",
             tm[8], tc[8], tm[9], tc[9], tm[10], tc[10], tm[11], tc[11], tm[12], tc[12], tm[13], tc[13], tc[14], tm[15], tc[15]);
#endif
  }
  // the boundary loop: every boundary with time < t_lim. A warp that keeps its engine bound
  // across calls (k_cluster_pipe) calls this directly: the steady-state register cache, the
  // nodisp / larry certificates stay valid between calls, because only enqueue_ready (which
  // resets them) changes what they depend on.
  __device__ __forceinline__ void advance_loop(double t_lim, int n_avail) {
    double next_t = next_arrival(n_avail);
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    while (st.status == SSB_OK) {
      double nb;
      if (!has_work()) {
        if (next_t == INF) break;            // idle until the next routed arrival
        nb = next_t > st.clock ? next_t : st.clock;  // wake = max(t, clock) (cluster.py:139)
      } else {
        nb = st.clock;
      }
      if (!(nb < t_lim)) break;  // ties: arrivals before boundaries (cluster.py:62)
      st.clock = nb;             // advance_to (engine.py:186-191)
      if (next_t <= st.clock) {
        SSB_T0(enq)
        enqueue_ready(n_avail);
        SSB_T1(enq, 0)
        if (st.status) break;
        next_t = next_arrival(n_avail);
      }
      step();
      // preempted / evicted / parked requests go back to the waiting set here, in the order
      // they were queued (policy preempts, then grow evictions): one call site for every path
      if (nq) flush_pushes();
#ifdef SSB_DEBUG
      debug_check();
#endif
      if (regs_ok && nodisp && st.status == SSB_OK && cfg.bs_shift >= 0)
        fast_forward(next_t < t_lim ? next_t : t_lim);
    }
  }
};

}  // namespace ssb
