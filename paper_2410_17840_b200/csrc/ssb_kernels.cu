// ssb_kernels.cu — sm_100a simulation kernels + the C ABI of include/ssb.h.
//
//   k_engines : persistent, one warp per single-server instance (run_cluster
//               with n_servers == 1 == Engine.run, engine.py:236-265). Warps
//               pull instances from an atomic queue, longest first.
//   k_cluster : one CTA per multi-server instance (run_cluster, cluster.py:65-174).
//               Warp 0 routes arrivals (balancers.py:132-216, incl. numpy PCG64
//               Generator.integers); every warp advances its replicas between
//               routing barriers. Barriers are only needed where a route reads
//               engine state: at poll instants (p2c, sal) and for sal routes
//               whose argmin depends on beta. See DESIGN.md §cluster.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "ssb_engine.cuh"

using namespace ssb;
namespace cg = cooperative_groups;

namespace {

#ifndef SSB_ENGINE_WARPS_PER_CTA
#define SSB_ENGINE_WARPS_PER_CTA 4
#endif
constexpr int ENGINE_WARPS_PER_CTA = SSB_ENGINE_WARPS_PER_CTA;

__host__ __device__ inline long long align_up(long long x, long long a) { return (x + a - 1) / a * a; }

struct Layout {
  long long srv, w_enq, w_rid, w_pend, w_key, r_rid, r_prompt, r_out, r_gen, r_pfd, r_st, r_plan, l_a, l_b, v_idx,
      v_rem, v_cum, v_key, l_c, rl, t_head, t_lv, total;
};

__host__ __device__ inline Layout make_layout(long long Wc, long long Rc, long long N, int n_servers,
                                              const ssb_engine_params& e) {
  Layout L;
  long long o = 0;
  L.srv = o;      o = align_up(o + (long long)sizeof(Srv), 64);
  L.w_enq = o;    o = align_up(o + 8 * Wc, 64);
  L.w_rid = o;    o = align_up(o + 4 * Wc, 64);
  L.w_pend = o;   o = align_up(o + 4 * Wc, 64);
  L.w_key = o;    o = align_up(o + 4 * Wc, 64);
  L.r_rid = o;    o = align_up(o + 4 * Rc, 64);
  L.r_prompt = o; o = align_up(o + 4 * Rc, 64);
  L.r_out = o;    o = align_up(o + 4 * Rc, 64);
  L.r_gen = o;    o = align_up(o + 4 * Rc, 64);
  L.r_pfd = o;    o = align_up(o + 4 * Rc, 64);
  L.r_st = o;     o = align_up(o + 4 * Rc, 64);
  L.r_plan = o;   o = align_up(o + 4 * Rc, 64);
  L.l_a = o;      o = align_up(o + 4 * Rc, 64);
  L.l_b = o;      o = align_up(o + 4 * Rc, 64);
  L.v_idx = o;    o = align_up(o + 4 * Rc, 64);
  L.v_rem = o;    o = align_up(o + 4 * Rc, 64);
  L.v_cum = o;    o = align_up(o + 8 * Rc, 64);
  L.v_key = o;    o = align_up(o + 8 * Rc, 64);
  L.l_c = o;      o = align_up(o + 4 * Rc, 64);
  L.rl = o;       o = align_up(o + (n_servers > 1 ? 4 * N : 0), 64);
  const bool trail = e.policy == SSB_POLICY_TRAIL_PLUS;
  const TrailGeom tg = trail_geom(e.max_context, e.pool_blocks, e.block_size);
  L.t_head = o;   o = align_up(o + (trail ? 4LL * tg.nb : 0), 64);
  L.t_lv = o;     o = align_up(o + (trail ? 4LL * tg.total : 0), 64);
  L.total = align_up(o, 256);
  return L;
}

// Server s's parameter set: its own when the instance carries prebuilt engines that differ
// (ssb_instance.d_servers, cluster.py:66-79), else the instance's one set.
__device__ inline const ssb_engine_params& server_params(const ssb_instance& I, int s) {
  return I.d_servers != nullptr ? I.d_servers[s] : I.engine;
}
// The instance's layout with the per-server stride ssb_prepare chose. Every field before the
// trail tree sits at the same offset for every parameter set (only t_head / t_lv depend on
// it), so this layout addresses any server's Srv / route list; server_layout gives server s's
// own tree offsets under the same stride.
__host__ __device__ inline Layout inst_layout(const ssb_instance& I) {
  Layout L = make_layout(I.wait_cap, I.run_cap, I.n_requests, I.n_servers, I.engine);
  if (I.server_stride > 0) L.total = I.server_stride;
  return L;
}
__device__ inline Layout server_layout(const ssb_instance& I, int s) {
  Layout L = make_layout(I.wait_cap, I.run_cap, I.n_requests, I.n_servers, server_params(I, s));
  if (I.server_stride > 0) L.total = I.server_stride;
  return L;
}

// Arrival times of an instance as the engines read them: the trace itself when qps_factor is
// 1, else the instance's scaled copy (arrival / qps_factor, workload.py:193 scale_qps) that
// k_scale_arrivals writes into its scratch after the servers' regions — so no binary64
// division (a subroutine call on sm_100a) sits in the engine's hot loop.
__host__ __device__ inline long long scaled_arrivals_offset(const ssb_instance& I, const Layout& L) {
  return I.scratch_offset + L.total * (long long)(I.n_servers > 0 ? I.n_servers : 1);
}
__device__ inline const double* instance_arrivals(const ssb_instance& I, const Layout& L, ssb_trace tr,
                                                  unsigned char* scratch) {
  return I.qps_factor == 1.0 ? tr.arrival + I.trace_offset
                             : (const double*)(scratch + scaled_arrivals_offset(I, L));
}

__device__ inline SrvPtr make_ptrs(unsigned char* base, const Layout& L) {
  SrvPtr p;
  p.w_enq = (double*)(base + L.w_enq);
  p.w_rid = (int*)(base + L.w_rid);
  p.w_pend = (int*)(base + L.w_pend);
  p.w_key = (int*)(base + L.w_key);
  p.r_rid = (int*)(base + L.r_rid);
  p.r_prompt = (int*)(base + L.r_prompt);
  p.r_out = (int*)(base + L.r_out);
  p.r_gen = (int*)(base + L.r_gen);
  p.r_pfd = (int*)(base + L.r_pfd);
  p.r_st = (int*)(base + L.r_st);
  p.r_plan = (int*)(base + L.r_plan);
  p.l_a = (int*)(base + L.l_a);
  p.l_b = (int*)(base + L.l_b);
  p.v_idx = (int*)(base + L.v_idx);
  p.v_rem = (int*)(base + L.v_rem);
  p.v_cum = (long long*)(base + L.v_cum);
  p.v_key = (unsigned long long*)(base + L.v_key);
  p.l_c = (int*)(base + L.l_c);
  p.rl = (int*)(base + L.rl);
  p.t_head = (int*)(base + L.t_head);
  p.t_lv = (int*)(base + L.t_lv);
  return p;
}

__device__ inline Cfg make_cfg(const ssb_instance& I, const ssb_engine_params& e) {
  Cfg c;
  c.policy = e.policy;
  c.max_output = e.max_output;
  c.bs = e.block_size;
  c.bs_shift = (e.block_size & (e.block_size - 1)) == 0 ? __ffs(e.block_size) - 1 : -1;
  c.bmul = (0x100000000ULL + (unsigned long long)e.block_size - 1ULL) / (unsigned long long)e.block_size;
  c.pool = e.pool_blocks;
  c.cap = e.max_tokens_per_batch;
  c.max_running = e.max_running;
  c.max_ctx = e.max_context;
  c.n_servers = I.n_servers;
  c.Wc = I.wait_cap;
  c.Rc = I.run_cap;
  c.alpha = e.alpha;
  c.c = e.c;
  c.mem_base = e.mem_base_s;
  c.mem_kv = e.mem_per_kv_token_s;
  c.compute = e.compute_per_token_s;
  c.overhead = e.overhead_s;
  c.qps = I.qps_factor;
  c.wide = false;
  c.tg = trail_geom(e.max_context, e.pool_blocks, e.block_size);
  return c;
}
__device__ inline Cfg make_cfg(const ssb_instance& I) { return make_cfg(I, I.engine); }

__device__ inline void init_srv(Srv& s, const Cfg& c) {
  s.clock = 0.0;
  s.iterations = s.rsteps = s.btokens = s.dispatches = s.preempts = s.parks = s.finished = s.peak = 0;
  s.digest = FNV_OFF;
  s.wpend_sum = s.fin_in = s.fin_out = s.fin_cnt = s.enq_prompt_sum = s.ev_n = s.pf_pend = 0;
  s.free_blocks = c.pool;
  s.R = s.W = s.whead = s.committed = s.next_arr = s.status = s.ndec = 0;
}

// shared running table columns: r_rid r_prompt r_out r_gen r_pfd r_st r_plan l_a l_b
// v_idx v_rem v_cum(2) v_key(2) l_c
constexpr int SM_COLS = 16;
constexpr int RS = SSB_SMEM_RUN_CAP;

// sm_tab: this engine's shared-memory running table (SM_COLS x RS ints) or
// nullptr for the global layout (SSB_FLAG_GLOBAL_TABLES).
__device__ inline void bind_engine(Eng& E, const ssb_instance& I, const Cfg& cfg, unsigned char* scratch, int server,
                                   const Layout& L, ssb_trace tr, ssb_records rec, ssb_event* ev, long long ev_cap,
                                   int* sm_tab = nullptr) {
  E.cfg = cfg;
  E.p = make_ptrs(scratch + I.scratch_offset + (long long)server * L.total, L);
  if (sm_tab != nullptr && !(I.flags & SSB_FLAG_GLOBAL_TABLES)) {
    E.p.r_rid = sm_tab;
    E.p.r_prompt = sm_tab + RS;
    E.p.r_out = sm_tab + 2 * RS;
    E.p.r_gen = sm_tab + 3 * RS;
    E.p.r_pfd = sm_tab + 4 * RS;
    E.p.r_st = sm_tab + 5 * RS;
    E.p.r_plan = sm_tab + 6 * RS;
    E.p.l_a = sm_tab + 7 * RS;
    E.p.l_b = sm_tab + 8 * RS;
    E.p.v_idx = sm_tab + 9 * RS;
    E.p.v_rem = sm_tab + 10 * RS;
    E.p.v_cum = (long long*)(sm_tab + 11 * RS);
    E.p.v_key = (unsigned long long*)(sm_tab + 13 * RS);
    E.p.l_c = sm_tab + 15 * RS;
    if (E.cfg.Rc > RS) E.cfg.Rc = RS;  // overflow -> SSB_E_CAPACITY -> host re-runs with global tables
  }
  E.arrival = instance_arrivals(I, L, tr, scratch);
  E.prompt = tr.prompt + I.trace_offset;
  E.output = tr.output + I.trace_offset;
  E.rec_ft = rec.first_token + I.record_offset;
  E.rec_fin = rec.finish + I.record_offset;
  E.rec_fd = rec.first_dispatch + I.record_offset;
  E.rec_pc = rec.preempt_count + I.record_offset;
  E.rec_srv = rec.server + I.record_offset;
  // event ring: instance slice split evenly between the instance's servers;
  // unused entries keep code -1 (filled by fill_events)
  const long long slice = ev_cap / (I.n_servers > 0 ? I.n_servers : 1);
  E.ev = ev ? ev + (long long)server * slice : nullptr;
  E.ev_cap = slice;
  E.server = server;
  E.lane = lane_id();
}

__device__ inline void fill_events(const Eng& E, int lane_base, int stride) {
  if (!E.ev) return;
  for (long long i = lane_base; i < E.ev_cap; i += stride) {
    ssb_event e;
    e.time = 0.0;
    e.request_id = -1;
    e.server = (int16_t)E.server;
    e.code = -1;
    E.ev[i] = e;
  }
}

__device__ inline void clear_records(const Eng& E, long long N, int lane_base, int stride) {
  for (long long i = lane_base; i < N; i += stride) {
    E.rec_ft[i] = __longlong_as_double(0x7ff8000000000000LL);
    E.rec_fin[i] = __longlong_as_double(0x7ff8000000000000LL);
    E.rec_fd[i] = __longlong_as_double(0x7ff8000000000000LL);
    E.rec_pc[i] = 0;
    E.rec_srv[i] = -1;
  }
}

// ------------------------------------------------------------------------
// scale_qps (workload.py:187-194) fused into the launch: arrival / qps_factor once per
// request of every instance with a factor != 1 (IEEE division == Python's float division),
// one CTA per instance, coalesced
// ------------------------------------------------------------------------
__global__ void k_scale_arrivals(const ssb_instance* __restrict__ inst, int n_inst, ssb_trace tr,
                                 unsigned char* __restrict__ scratch) {
  for (int i = blockIdx.x; i < n_inst; i += gridDim.x) {
    const ssb_instance I = inst[i];
    if (I.qps_factor == 1.0) continue;
    const Layout L = inst_layout(I);
    double* out = (double*)(scratch + scaled_arrivals_offset(I, L));
    const double* in = tr.arrival + I.trace_offset;
    for (long long k = threadIdx.x; k < I.n_requests; k += blockDim.x) out[k] = __ddiv_rn(in[k], I.qps_factor);
  }
}

#ifdef SSB_TIMELINE
// debug build only (tools/probe_timeline.py): per single-server instance the %globaltimer
// ns at start and end and the SM it ran on, read back with ssb_debug_timeline
constexpr int TIMELINE_MAX = 1 << 16;
__device__ unsigned long long g_timeline[3 * TIMELINE_MAX];
#endif
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned sm_id();

// ------------------------------------------------------------------------
// single-server instances: one warp each, persistent
// ------------------------------------------------------------------------
// POL: the instance's policy as a compile-time constant, so the kernel holds one engine copy per
// policy and an SM (which serves one policy at a time, see k_engines) executes only its copy:
// a smaller hot code footprint and no policy branches in the loop.
template <int POL, bool WIDE>
__device__ __forceinline__ void run_instance(const ssb_instance* __restrict__ inst, int idx, ssb_trace tr,
                                             ssb_records rec, ssb_stats* __restrict__ stats,
                                             unsigned char* __restrict__ scratch, ssb_event* events, long long ev_cap,
                                             int64_t* ev_count, int* sm_tab) {
  const int lane = lane_id();
  const long long t0 = clock64();
#ifdef SSB_TIMELINE
  const unsigned long long g0 = globaltimer_ns();
#endif
  const ssb_instance I = inst[idx];
  Cfg cfg = make_cfg(I);
  cfg.policy = POL;  // compile-time policy: this copy of the engine holds only POL's code
  cfg.wide = WIDE;   // latency-mode kernel only (see k_engines)
  const Layout L = inst_layout(I);
  Eng E;
  bind_engine(E, I, cfg, scratch, 0, L, tr, rec, events ? events + (long long)idx * ev_cap : nullptr, ev_cap, sm_tab);
  clear_records(E, I.n_requests, lane, 32);
  fill_events(E, lane, 32);
  init_srv(E.st, cfg);
  if (cfg.policy == SSB_POLICY_TRAIL_PLUS) E.trail_init();
  __syncwarp();
  E.advance(__longlong_as_double(0x7ff0000000000000LL), (int)I.n_requests);  // t_lim = +inf
  if (E.st.status == SSB_OK && (E.st.finished != I.n_requests || E.has_work())) E.st.status = SSB_E_INVARIANT;
  if (lane == 0) {
    ssb_stats s;
    s.iterations = E.st.iterations;
    s.request_steps = E.st.rsteps;
    s.batch_tokens = E.st.btokens;
    s.dispatches = E.st.dispatches;
    s.preempts = E.st.preempts;
    s.parks = E.st.parks;
    s.finished = E.st.finished;
    s.peak_batch_tokens = E.st.peak;
    unsigned long long h = FNV_OFF;
    h ^= E.st.digest; h *= FNV_PRIME;
    s.digest = h;
    s.status = E.st.status;
    s._pad = 0;
    s.device_cycles = clock64() - t0;
    stats[idx] = s;
    if (ev_count) ev_count[idx] = E.st.ev_n;
#ifdef SSB_TIMELINE
    g_timeline[3 * idx] = g0;
    g_timeline[3 * idx + 1] = globaltimer_ns();
    g_timeline[3 * idx + 2] = sm_id();
#endif
  }
  __syncwarp();
}

__device__ __forceinline__ unsigned sm_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Persistent single-server kernel. The host assigns each SM a policy (SMs split in
// proportion to each policy's estimated work); a warp serves the queue of its SM's policy,
// longest estimated cost first, and steals from the other queues once its own is empty.
// Keeping one policy per SM keeps the policy-specific code of each SM's warps the same.
// Queues: 2 per policy (queue 2p + c: class c of policy p — small / large KV pools, see
// ssb_simulate) and
// queue Q_HEAVY for the longest trail_plus instances when SSB_HEAVY_SMS reserves SMs for them.
constexpr int NQ = 9;
constexpr int Q_HEAVY = 8;
__device__ __forceinline__ bool known_sm(unsigned smid, int n_sm_policy) { return smid < (unsigned)n_sm_policy; }
struct EngineQueues {
  int n[NQ];    // instances per queue
  int off[NQ];  // offset of each queue's order list in order[]
  int nsm[NQ];  // SMs whose home is the queue (the head of the queue is dealt among them)
};
// The head of each queue (its DEAL_ROUNDS x SMs longest instances) is dealt among the queue's
// SMs like cards, snake order: claim c of the SM with rank r takes item c*S + (c odd ? S-1-r : r).
// Without it the longest instances went to whichever warps reached the atomic first — often one
// SM's eight (measured: the 8 longest trail_plus instances on one SM, 144 ms vs 123 ms).
#ifndef SSB_DEAL_ROUNDS
#define SSB_DEAL_ROUNDS 1
#endif
constexpr int DEAL_ROUNDS = SSB_DEAL_ROUNDS;
#ifndef SSB_ENGINE_MIN_CTAS
#define SSB_ENGINE_MIN_CTAS 1
#endif
// WIDE: latency mode for batches with at most one instance per SM (each runs alone, so a
// larger hot loop costs nothing and the R <= 64 register path shortens its serial chain); the
// many-instance kernel (WIDE = false) keeps the smaller code.
template <bool WIDE>
__global__ void __launch_bounds__(32 * ENGINE_WARPS_PER_CTA, SSB_ENGINE_MIN_CTAS)
k_engines(const ssb_instance* __restrict__ inst, const int* __restrict__ order, EngineQueues qs,
          int* __restrict__ queue, const unsigned char* __restrict__ sm_policy, int n_sm_policy,
          int* __restrict__ sm_slot, int* __restrict__ sm_done, int* __restrict__ sm_claim,
          const int* __restrict__ sm_rank, ssb_trace tr, ssb_records rec,
          ssb_stats* __restrict__ stats, unsigned char* __restrict__ scratch, ssb_event* events, long long ev_cap,
          int64_t* ev_count) {
  extern __shared__ int sm_engines[];
  __shared__ int s_slot;
  int* sm_tab = sm_engines + (threadIdx.x >> 5) * (SM_COLS * RS);  // this warp's running table
  const int lane = lane_id();
  const unsigned smid = sm_id();
  const int first = known_sm(smid, n_sm_policy) ? sm_policy[smid] : 0;
  if (threadIdx.x == 0) s_slot = known_sm(smid, n_sm_policy) ? atomicAdd(sm_slot + smid, 1) : 0;
  __syncthreads();
  if (first == Q_HEAVY && s_slot > 0) return;  // SMs of the longest instances run one CTA (see ssb_simulate)
  // queue order: own queue, the other class of the same policy, the other policies, the heavy
  // queue last (a heavy SM continues with trail_plus)
  const int home = first == Q_HEAVY ? 2 * SSB_POLICY_TRAIL_PLUS : first;
  int k = first == Q_HEAVY ? -1 : 0;
  bool switched = false;
  bool dealt = first != Q_HEAVY && known_sm(smid, n_sm_policy) && sm_rank[smid] >= 0;
  while (k < NQ) {
    // k = -1: the heavy queue; 0: home; 1: home's other class; 2..7: the other policies; 8: heavy
    int pol;
    if (k < 0) pol = Q_HEAVY;
    else if (k == 0) pol = home;
    else if (k == 1) pol = home ^ 1;
    else if (k < 8) pol = ((home & ~1) + k) & 7;
    else pol = Q_HEAVY;
    if (k == 8 && first == Q_HEAVY) break;
    if (k == 2 && !switched && first != Q_HEAVY && known_sm(smid, n_sm_policy)) {
      switched = true;
      // The SM switches policy as a whole: a warp whose own policy is drained waits until every
      // warp resident on this SM is, then all steal in the same order and so run the same
      // policy's code (a warp running another policy's engine beside the home policy's warps
      // would share the SM's instruction cache between two hot loops — measured slower).
      if (lane == 0) {
        atomicAdd(sm_done + smid, 1);
        const int resident = *((volatile int*)(sm_slot + smid)) * (int)(blockDim.x >> 5);
#ifndef SSB_SWITCH_SLACK
#define SSB_SWITCH_SLACK 0
#endif
        while (*((volatile int*)(sm_done + smid)) < resident - SSB_SWITCH_SLACK) __nanosleep(2000);
      }
      __syncwarp();
    }
    int q = 0;
    if (k == 0 && dealt) {  // this SM's dealt share of the home queue's head first
      if (lane == 0) q = atomicAdd(sm_claim + smid, 1);
      const int c = __shfl_sync(FULL, q, 0);
      const int S = qs.nsm[pol], r = sm_rank[smid];
      q = c * S + ((c & 1) ? S - 1 - r : r);
      if (c >= DEAL_ROUNDS || q >= qs.n[pol]) {  // dealt share done (later claims only go further)
        dealt = false;
        continue;
      }
    } else {
      if (lane == 0) q = atomicAdd(queue + pol, 1);
      q = __shfl_sync(FULL, q, 0);
      if (q >= qs.n[pol]) {  // this queue is drained: steal from the next one
        k += 1;
        continue;
      }
    }
    const int idx = order[qs.off[pol] + q];
    switch (inst[idx].engine.policy) {  // the instance's own policy (a queue may mix them: SSB_ONE_QUEUE)
      case SSB_POLICY_FCFS: run_instance<SSB_POLICY_FCFS, WIDE>(inst, idx, tr, rec, stats, scratch, events, ev_cap, ev_count, sm_tab); break;
      case SSB_POLICY_NOPREEMPT: run_instance<SSB_POLICY_NOPREEMPT, WIDE>(inst, idx, tr, rec, stats, scratch, events, ev_cap, ev_count, sm_tab); break;
      case SSB_POLICY_TRAIL_PLUS: run_instance<SSB_POLICY_TRAIL_PLUS, WIDE>(inst, idx, tr, rec, stats, scratch, events, ev_cap, ev_count, sm_tab); break;
      default: run_instance<SSB_POLICY_LARRY, WIDE>(inst, idx, tr, rec, stats, scratch, events, ev_cap, ev_count, sm_tab); break;
    }
  }
}

// ------------------------------------------------------------------------
// numpy PCG64 (XSL-RR 128/64) + Generator.integers (32-bit Lemire, buffered
// next_uint32: low half first) — bit-exact with np.random.default_rng(seed)
// ------------------------------------------------------------------------
struct Pcg {
  unsigned long long shi, slo, ihi, ilo;
  unsigned buf;
  int has;
  __device__ unsigned long long next64() {
    const unsigned long long MHI = 0x2360ED051FC65DA4ULL, MLO = 0x4385DF649FCCF645ULL;
    unsigned long long lo = slo * MLO;
    unsigned long long hi = __umul64hi(slo, MLO) + slo * MHI + shi * MLO;
    unsigned long long nlo = lo + ilo;
    hi += ihi + (nlo < lo ? 1ULL : 0ULL);
    slo = nlo;
    shi = hi;
    unsigned rot = (unsigned)(shi >> 58);
    unsigned long long x = shi ^ slo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ unsigned next32() {
    if (has) { has = 0; return buf; }
    unsigned long long v = next64();
    has = 1;
    buf = (unsigned)(v >> 32);
    return (unsigned)v;
  }
  __device__ int integers(int high) {  // [0, high)
    unsigned rng = (unsigned)(high - 1);
    if (rng == 0) return 0;
    unsigned excl = rng + 1u;
    unsigned long long m = (unsigned long long)next32() * excl;
    unsigned left = (unsigned)m;
    if (left < excl) {
      unsigned thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = (unsigned long long)next32() * excl;
        left = (unsigned)m;
      }
    }
    return (int)(m >> 32);
  }
};

// ------------------------------------------------------------------------
// multi-server instances: one thread-block cluster each (1..8 CTAs x 8 warps)
// ------------------------------------------------------------------------
// The routing state (S, the BalancerView columns, per-server routed counts, next-boundary
// bounds) lives in the shared memory of the cluster's rank-0 CTA; the other CTAs read and
// write it through distributed shared memory. Warp w of CTA r advances servers
// r*8+w, r*8+w + 8*G, ... so a 64-replica instance (C5) gets one warp per replica on
// 8 SMs instead of 8 replicas per warp on one; cluster barriers separate the phases.
struct ClusterShared {
  double t_lim;
  double last_poll;
  double beta;
  int k;
  int done;
  int synced;
  int err;
  int epochs, polls;  // routing phases / view refreshes (cost diagnostics)
  long long fin_cnt, fin_in, fin_out;  // completions of every engine (BetaEstimator sums)
};

constexpr int CLUSTER_MAX_WARPS = 8;
constexpr int CLUSTER_MAX_CTAS = 8;       // portable cluster size
constexpr int CLUSTER_SMEM_SERVERS = 12;  // shared running tables per CTA (12 x 16 KiB)

template <int B> struct BalTag { static constexpr int value = B; };

// The cluster body with the instance's policy as a compile-time constant (one engine copy per
// policy, like k_engines); k_cluster dispatches on the instance's policy.
template <int POL>
__device__ __forceinline__ void cluster_body(const ssb_instance* __restrict__ inst, const int* __restrict__ order,
                                             ssb_trace tr, ssb_records rec, ssb_stats* __restrict__ stats,
                                             unsigned char* __restrict__ scratch, ssb_event* events, long long ev_cap,
                                             int64_t* ev_count, int smem_tabs, long long* smem_ll,
                                             ClusterShared& S_own) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int idx = order[blockIdx.x / G];
  const ssb_instance I = inst[idx];
  const int n = I.n_servers;
  const long long N = I.n_requests;
  // rank 0 owns the routing state; everyone addresses it through one generic pointer
  long long* R0 = rank == 0 ? smem_ll : cl.map_shared_rank(smem_ll, 0);
  ClusterShared& S = *(rank == 0 ? &S_own : cl.map_shared_rank(&S_own, 0));
  long long* v_q = R0;               // BalancerView.stats[s].queued_tokens
  long long* v_f = R0 + n;           // .free_mem_tokens
  long long* v_if = R0 + 2 * n;      // .in_flight
  long long* rps = R0 + 3 * n;       // Σ prompt routed to s
  int* cnt = (int*)(R0 + 4 * n);     // arrivals routed to s
  // lower bound of each engine's next boundary time: an advance phase skips every engine
  // whose bound is >= its time limit (it would process nothing)
  double* s_nb = (double*)(R0 + 5 * ((n + 1) & ~1));
  // this CTA's shared running tables (its own servers), when they fit
  int* sm_tabs = (int*)(smem_ll + 6 * ((n + 1) & ~1));
  const bool tabs_in_smem = smem_tabs != 0;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5, lane = lane_id();
  const int gw = rank * nwarps + warp, GW = G * nwarps;  // cluster-wide warp index / count
  // cluster barrier (also orders the DSMEM and global accesses around it); a one-CTA
  // cluster (<= 8 replicas) uses the cheaper CTA barrier
  auto csync = [&]() { if (G == 1) __syncthreads(); else cl.sync(); };
  auto tab_of = [&](int s) { return tabs_in_smem ? sm_tabs + ((s / GW) * nwarps + warp) * SM_COLS * RS : nullptr; };
  if (I.d_servers != nullptr) {  // heterogeneous engines here: one policy (a warp runs several servers)
    bool mixed = false;
    for (int q = 1; q < n; ++q) mixed |= I.d_servers[q].policy != I.d_servers[0].policy;
    if (mixed) {
      if (rank == 0 && threadIdx.x == 0) {
        ssb_stats out = {};
        out.status = SSB_E_ARG;
        stats[idx] = out;
      }
      return;  // (every CTA of the cluster returns before its first cluster barrier)
    }
  }
  Cfg cfg = make_cfg(I);
  cfg.policy = POL;
  const Layout L = inst_layout(I);
  ssb_event* evb = events ? events + (long long)idx * ev_cap : nullptr;
  // server s's engine: its own parameters and tree offsets when the prebuilt engines differ
  auto bind_server = [&](Eng& E, int s) {
    bind_engine(E, I, cfg, scratch, s, L, tr, rec, evb, ev_cap, tab_of(s));
    if (I.d_servers != nullptr) {  // (rare: only the parameter-dependent parts are rebound)
      const Cfg cs = make_cfg(I, server_params(I, s));
      const Layout Ls = server_layout(I, s);
      const int rc = E.cfg.Rc;  // (bind_engine may have clipped it to the shared table)
      E.cfg = cs;
      E.cfg.policy = POL;
      E.cfg.Rc = rc;
      unsigned char* base = scratch + I.scratch_offset + (long long)s * L.total;
      E.p.t_head = (int*)(base + Ls.t_head);
      E.p.t_lv = (int*)(base + Ls.t_lv);
    }
  };

  // init engines + view (cluster.py:122: refresh at 0.0 from ground truth = empty engines)
  for (int s = gw; s < n; s += GW) {
    Eng E;
    bind_server(E, s);
    init_srv(E.st, E.cfg);
    if (cfg.policy == SSB_POLICY_TRAIL_PLUS) E.trail_init();
    fill_events(E, lane, 32);
    if (lane == 0) *(Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv) = E.st;
  }
  if (rank == 0) {
    for (int s = threadIdx.x; s < n; s += blockDim.x) {
      v_q[s] = 0;
      v_f[s] = (long long)server_params(I, s).pool_blocks * server_params(I, s).block_size;
      v_if[s] = 0;
      rps[s] = 0;
      cnt[s] = 0;
      s_nb[s] = __longlong_as_double(0x7ff0000000000000LL);  // idle, nothing routed
    }
    if (threadIdx.x == 0) {
      S.k = 0; S.done = 0; S.synced = 1; S.err = 0; S.epochs = 0; S.polls = 0;
      S.last_poll = 0.0;
      S.beta = I.beta_prior;
      S.fin_cnt = S.fin_in = S.fin_out = 0;
    }
  }
  {
    Eng E;
    bind_engine(E, I, cfg, scratch, 0, L, tr, rec, evb, ev_cap);
    clear_records(E, N, rank * blockDim.x + threadIdx.x, G * blockDim.x);
  }
  csync();

  const bool est_beta = I.balancer == SSB_BAL_SAL && isnan(I.beta_fixed);
  // SAL's cap is the settings' max_tokens_per_batch (cluster.py:101), not the engines' own
  const int route_cap = I.route_cap;
  const bool cap_pow2 = route_cap > 0 && (route_cap & (route_cap - 1)) == 0;
  const double inv_cap = cap_pow2 ? __ddiv_rn(1.0, (double)route_cap) : 0.0;
  Pcg rng;
  rng.shi = I.pcg_state_hi; rng.slo = I.pcg_state_lo; rng.ihi = I.pcg_inc_hi; rng.ilo = I.pcg_inc_lo;
  rng.has = 0; rng.buf = 0;
  long long rr = 0;
  const double* arr = instance_arrivals(I, L, tr, scratch);  // already divided by qps_factor
  const int* prm = tr.prompt + I.trace_offset;
  int* rec_srv = rec.server + I.record_offset;
  const double poll = I.poll_interval_s;
#ifdef SSB_EPOCH_PROBE
  long long pr_route = 0, pr_sync = 0, pr_adv_own = 0;
#endif

  while (true) {
#ifdef SSB_EPOCH_PROBE
    const long long pt0 = clock64();
#endif
    // ---------------- routing phase (warp 0 of rank 0) ----------------
    if (rank == 0 && warp == 0) {
      // rank 0's own shared memory under the same names: plain shared loads/stores instead of
      // the generic (DSMEM-capable) accesses the other ranks need
      long long* const v_q = smem_ll;
      long long* const v_f = smem_ll + n;
      long long* const v_if = smem_ll + 2 * n;
      long long* const rps = smem_ll + 3 * n;
      int* const cnt = (int*)(smem_ll + 4 * n);
      double* const s_nb = (double*)(smem_ll + 5 * ((n + 1) & ~1));
      ClusterShared& S = S_own;
      // sync point: fold the completions of the advance phase that just ended into beta
      // (on_finish, cluster.py:153-154; balancers.py:96-100) — here rather than behind a barrier
      // of its own; the first pass folds nothing (beta stays the prior)
      if (lane == 0) {
        if (est_beta)
          S.beta = S.fin_cnt == 0 ? I.beta_prior : __ddiv_rn((double)(S.fin_in + S.fin_out), (double)S.fin_out);
        S.synced = 1;
        S.epochs += 1;
        if (S.k >= N || S.err) S.done = 1;
      }
      __syncwarp();
      int k = S.k;
      int synced = S.synced;
      double last_poll = S.last_poll;
      const double beta = isnan(I.beta_fixed) ? S.beta : I.beta_fixed;
      if (I.balancer == SSB_BAL_RR || I.balancer == SSB_BAL_RANDOM) {
        // round robin and random read no engine state (balancers.py:139-153): every arrival
        // is routed in one phase, 32 at a time — lane i takes arrival k0+i: server (rr+i) mod n,
        // or the i-th of 32 consecutive Generator.integers(n) draws (drawn in order by every
        // lane, kept by lane i); lanes that share a server append to its list in arrival
        // order (match_any + rank in group)
        for (int k0 = k; k0 < N; k0 += 32) {
          const int kk = k0 + lane;
          const bool valid = kk < N;
          const double t = valid ? arr[kk] : 0.0;
          const int pr = valid ? prm[kk] : 0;
          int s = (int)((rr + lane) % n);
          if (I.balancer == SSB_BAL_RANDOM) {
            const int m = N - k0 < 32 ? (int)(N - k0) : 32;
            for (int j = 0; j < m; ++j) {
              const int d = rng.integers(n);
              if (j == lane) s = d;
            }
          }
          const unsigned grp = __match_any_sync(FULL, valid ? s : -1);
          const int before = __popc(grp & lanemask_lt());
          const bool leader = before == 0;
          const int base = valid ? cnt[s] : 0;
          __syncwarp();
          if (valid) {
            int* rl = (int*)(scratch + I.scratch_offset + (long long)s * L.total + L.rl);
            rl[base + before] = kk;
            rec_srv[kk] = s;
            atomicAdd((unsigned long long*)&rps[s], (unsigned long long)(long long)pr);
            if (leader) {
              cnt[s] = base + __popc(grp);
              if (t < s_nb[s]) s_nb[s] = t;  // the group's earliest arrival
            }
          }
          __syncwarp();
          rr += N - k0 < 32 ? N - k0 : 32;
        }
        k = (int)N;
      }
      // p2c / sal: one arrival at a time (each route may read the view);
      // the arrivals' times and prompts are fetched 32 at a time (lane i holds c0 + i)
      int c0 = -64;
      double c_t = 0.0;
      int c_pr = 0;
      // one copy of the per-arrival loop per balancer (no balancer branches inside it); random
      // and round robin never get here (routed above)
      auto route_loop = [&](auto bal_tag) {
      constexpr int BAL = decltype(bal_tag)::value;
      // engines are synced to the phase's first arrival; they stay synced for the arrivals that
      // share its time (no simulated time passes), not beyond
      double t_prev = k < N ? arr[k] : 0.0;
      while (k < N) {
        if (k >= c0 + 32) {
          c0 = k;
          const int kk = k + lane;
          c_t = kk < N ? arr[kk] : __longlong_as_double(0x7ff0000000000000LL);
          c_pr = kk < N ? prm[kk] : 0;
        }
        const double t = __shfl_sync(FULL, c_t, k - c0);
        const int pr = __shfl_sync(FULL, c_pr, k - c0);
        synced = t == t_prev ? synced : 0;  // equal times need no sync
        t_prev = t;
        if (__dsub_rn(t, last_poll) >= poll) {  // BalancerView.due (balancers.py:42-43)
          if (!synced) break;
          // ground truth incl. routed-but-unseen inbox (cluster.py:110-120, 50-59)
          #pragma unroll 1  // n <= 64 in practice: 1-2 trips, no unrolled remainder chain
          for (int s = lane; s < n; s += 32) {
            const Srv* sv = (const Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv);
            v_q[s] = sv->wpend_sum + (rps[s] - sv->enq_prompt_sum);
            v_f[s] = (long long)sv->free_blocks * server_params(I, s).block_size;
            v_if[s] = (long long)sv->W + sv->R + (cnt[s] - sv->next_arr);
          }
          __syncwarp();
          last_poll = t;
          if (lane == 0) S.polls += 1;
        }
        int s = 0;
        if constexpr (BAL == SSB_BAL_P2C) {  // :167-176
          if (n > 1) {
            int i = rng.integers(n);
            int j = rng.integers(n - 1);
            if (j >= i) j += 1;
            s = v_if[j] < v_if[i] ? j : i;
          }
        } else {  // SAL (:204-212)
          // fast path (cap a power of two, beta > 0, prompt > 0, every queued+prompt < 2^51): Q
          // orders exactly as the integer queued+prompt, an unconstrained server's load is Q and
          // a constrained one's is >= Q for every beta, so when the (Q, server) minimum is
          // unconstrained it is the load argmin whatever beta is (no barrier needed either):
          // one 64-bit warp minimum over (queued+prompt) << 13 | server << 1 | constrained (n <= 4096)
          bool fast = false;
          if (cap_pow2 && beta > 0.0 && pr > 0) {
            unsigned long long kx = ~0ULL;
            bool big = false;
            #pragma unroll 1  // n <= 64 in practice: 1-2 trips, no unrolled remainder chain
            for (int q = lane; q < n; q += 32) {
              const unsigned long long X = (unsigned long long)(v_q[q] + pr);
              big |= X >= (1ULL << 51);
              // low bit: constrained (free < prompt); (X, q) is unique, so it never decides
              const unsigned long long key = (X << 13) | ((unsigned)q << 1) | (unsigned)(v_f[q] < pr);
              kx = key < kx ? key : kx;
            }
            if (!__any_sync(FULL, big)) {
              const unsigned long long m = warp_min_u64(kx);
              if (!(m & 1ULL)) { s = (int)((m >> 1) & 0xfffULL); fast = true; }
              else if (est_beta && !synced) break;  // a constrained server leads: beta decides
            }
          }
          if (!fast) {
          // per server (lane q, q+32, ...): the queue term Q = (queued+prompt)/cap (exact
          // integers < 2^53; a power-of-two cap divides exactly as a product with 2^-k),
          // the load max(beta*(prompt-free), Q) (sal_load, balancers.py:103-112) and whether
          // the server is memory-constrained (free < prompt); each lane keeps its best
          // (value, server) per quantity, then REDUX picks the warp minimum and the lowest
          // server index among the lanes holding it (min(range(n), key=...) tie rule, :210)
          unsigned long long kl = ~0ULL, ku = ~0ULL, kc = ~0ULL;
          int sl = 0x7fffffff, su = 0x7fffffff, sc = 0x7fffffff;
          #pragma unroll 1  // n <= 64 in practice: 1-2 trips, no unrolled remainder chain
          for (int q = lane; q < n; q += 32) {
            const double que = cap_pow2 ? __dmul_rn((double)(v_q[q] + pr), inv_cap)
                                        : __ddiv_rn((double)(v_q[q] + pr), (double)route_cap);
            const double mem = __dmul_rn(beta, (double)((long long)pr - v_f[q]));
            const double load = que > mem ? que : mem;
            const unsigned long long k1 = dkey(load), kq = dkey(que);
            if (k1 < kl) { kl = k1; sl = q; }  // q ascending: ties keep the lower server
            if (v_f[q] < pr) { if (kq < kc) { kc = kq; sc = q; } }
            else if (kq < ku) { ku = kq; su = q; }
          }
          if (est_beta && !synced) {
            // beta moves with completions the routing warp has not seen; a server with
            // free >= prompt has load == Q (beta*(prompt-free) <= 0 < Q), a constrained one
            // load >= Q for every beta: if the best unconstrained (Q, server) beats every
            // constrained one, the argmin is the same for every beta and no barrier is needed
            const unsigned long long mc = warp_min_u64(kc);
            if (mc != ~0ULL) {
              const unsigned long long mu = warp_min_u64(ku);
              const int iu = mu == ~0ULL ? 0x7fffffff : (int)__reduce_min_sync(FULL, ku == mu ? (unsigned)su : 0x7fffffffu);
              const int ic = (int)__reduce_min_sync(FULL, kc == mc ? (unsigned)sc : 0x7fffffffu);
              const bool indep = mu != ~0ULL && (mu < mc || (mu == mc && iu < ic));
              if (!indep) break;
            }
          }
          const unsigned long long ml = warp_min_u64(kl);
          s = (int)__reduce_min_sync(FULL, kl == ml ? (unsigned)sl : 0x7fffffffu);
          }
        }
        // bookkeeping: every lane reads (one address: broadcast), lane 0 stores — predicated
        // stores instead of a divergent lane-0 block on the routing chain
        {
          const bool w0 = lane == 0;
          const int cs = cnt[s];
          const long long rq = rps[s];
          const double nb0 = s_nb[s];
          int* rl = (int*)(scratch + I.scratch_offset + (long long)s * L.total + L.rl);
          if constexpr (BAL == SSB_BAL_SAL) {  // note_routed (balancers.py:59-64)
            const long long vq = v_q[s], vf = v_f[s] - pr, vi = v_if[s];
            if (w0) v_q[s] = vq + pr;
            if (w0) v_f[s] = vf > 0 ? vf : 0;
            if (w0) v_if[s] = vi + 1;
          }
          if (w0) rl[cs] = k;
          if (w0) cnt[s] = cs + 1;
          if (w0) rps[s] = rq + pr;
          if (w0) rec_srv[k] = s;
          if (w0 && t < nb0) s_nb[s] = t;  // its boundary is max(t, clock) >= t
        }
        __syncwarp();
        k++;
      }
      };
      if (I.balancer == SSB_BAL_SAL) route_loop(BalTag<SSB_BAL_SAL>{});
      else if (I.balancer == SSB_BAL_P2C) route_loop(BalTag<SSB_BAL_P2C>{});
      const double t_next = k >= N ? __longlong_as_double(0x7ff0000000000000LL)
                          : (k >= c0 && k < c0 + 32) ? __shfl_sync(FULL, c_t, k - c0) : arr[k];
      if (lane == 0) {
        S.k = k;
        S.synced = synced;
        S.last_poll = last_poll;
        S.t_lim = t_next;
      }
    }
#ifdef SSB_EPOCH_PROBE
    const long long pt1 = clock64();
#endif
    csync();
#ifdef SSB_EPOCH_PROBE
    const long long pt2 = clock64();
#endif
    if (S.done) break;
    // ---------------- advance phase: every replica to its boundaries < t_lim ----------------
    const double t_lim = S.t_lim;
    long long dc = 0, di = 0, dout = 0;  // this warp's completions (beta sums)
    for (int s = gw; s < n; s += GW) {
      if (!(s_nb[s] < t_lim)) continue;  // no boundary before t_lim: advance would do nothing
      Eng E;
      bind_server(E, s);
      Srv* sp = (Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv);
      E.st = *sp;
      const long long c0 = E.st.fin_cnt, i0 = E.st.fin_in, o0 = E.st.fin_out;
      E.advance(t_lim, cnt[s]);
      dc += E.st.fin_cnt - c0; di += E.st.fin_in - i0; dout += E.st.fin_out - o0;
      const double na = E.next_arrival(cnt[s]);
      const double nb = E.has_work() ? E.st.clock : (na > E.st.clock ? na : E.st.clock);
      __syncwarp();
      if (lane == 0) {
        *sp = E.st;
        s_nb[s] = nb;
        if (E.st.status) atomicExch(&S.err, E.st.status);
      }
    }
    if (lane == 0 && dc) {
      atomicAdd((unsigned long long*)&S.fin_cnt, (unsigned long long)dc);
      atomicAdd((unsigned long long*)&S.fin_in, (unsigned long long)di);
      atomicAdd((unsigned long long*)&S.fin_out, (unsigned long long)dout);
    }
#ifdef SSB_EPOCH_PROBE
    const long long pt3 = clock64();
#endif
    csync();
#ifdef SSB_EPOCH_PROBE
    if (rank == 0 && threadIdx.x == 0) {
      pr_route += pt1 - pt0; pr_sync += (pt2 - pt1) + (clock64() - pt3); pr_adv_own += pt3 - pt2;
    }
#endif
  }
  csync();  // every CTA has read S.done: rank 0's shared memory may go away after this

  // ---------------- per-instance stats ----------------
  if (rank == 0 && threadIdx.x == 0) {
    ssb_stats out;
    memset(&out, 0, sizeof(out));
    unsigned long long h = FNV_OFF;
    int status = S.err;
    long long evn = 0;
    for (int s = 0; s < n; ++s) {
      const Srv* sv = (const Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv);
      out.iterations += sv->iterations;
      out.request_steps += sv->rsteps;
      out.batch_tokens += sv->btokens;
      out.dispatches += sv->dispatches;
      out.preempts += sv->preempts;
      out.parks += sv->parks;
      out.finished += sv->finished;
      if (sv->peak > out.peak_batch_tokens) out.peak_batch_tokens = sv->peak;
      h ^= sv->digest; h *= FNV_PRIME;
      if (!status && (sv->W != 0 || sv->R != 0)) status = SSB_E_INVARIANT;
      evn += sv->ev_n;
    }
    if (!status && out.finished != N) status = SSB_E_INVARIANT;  // cluster.py:159-161
    out.digest = h;
    out.status = status;
#ifdef SSB_EPOCH_PROBE
    out._pad = S.epochs;
    out.device_cycles = S.polls;
    printf("EPOCHS inst %d servers %d epochs %d: route %lld cyc, warp0 advance %lld cyc, barrier wait (incl. slowest warp) %lld cyc\n",
           idx, n, S.epochs, pr_route, pr_adv_own, pr_sync);
#endif
    stats[idx] = out;
    if (ev_count) ev_count[idx] = evn;
  }
}

__global__ void __launch_bounds__(32 * CLUSTER_MAX_WARPS, 1) k_cluster(const ssb_instance* __restrict__ inst, const int* __restrict__ order, ssb_trace tr,
                          ssb_records rec, ssb_stats* __restrict__ stats, unsigned char* __restrict__ scratch,
                          ssb_event* events, long long ev_cap, int64_t* ev_count, int smem_tabs) {
  extern __shared__ long long smem_ll[];
  __shared__ ClusterShared S_own;
  const int G = (int)cg::this_cluster().num_blocks();
  switch (inst[order[blockIdx.x / G]].engine.policy) {
    case SSB_POLICY_FCFS: cluster_body<SSB_POLICY_FCFS>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_tabs, smem_ll, S_own); break;
    case SSB_POLICY_NOPREEMPT: cluster_body<SSB_POLICY_NOPREEMPT>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_tabs, smem_ll, S_own); break;
    case SSB_POLICY_TRAIL_PLUS: cluster_body<SSB_POLICY_TRAIL_PLUS>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_tabs, smem_ll, S_own); break;
    default: cluster_body<SSB_POLICY_LARRY>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_tabs, smem_ll, S_own); break;
  }
}

// ------------------------------------------------------------------------
// multi-server instances, pipelined (k_cluster_pipe): one thread-block cluster per
// instance with a dedicated routing warp (warp 0 of rank 0) and one engine warp per
// replica (server s = cluster warp s + 1), n <= PIPE_MAX_SERVERS
// ------------------------------------------------------------------------
// The classic k_cluster alternates a routing phase and an advance phase with two cluster
// barriers per epoch, so an epoch costs route + advance + barriers. Here they overlap: an
// engine never needs more than "every arrival before my next boundary is routed"
// (cluster.py:128-157: arrivals precede boundaries at equal times), so the router publishes
// a watermark wt = the time of the first unrouted arrival and every engine advances through
// its boundaries < wt while the router routes on. Only a route that reads engine state (a
// p2c/sal poll refresh, a sal route whose argmin depends on beta) needs the engines at
// exactly its time t: the router publishes wt = t with the sync bit, waits until every
// engine has reached t and published its ground-truth snapshot (snapshot_stats,
// cluster.py:50-59, 110-120), and reads the snapshots.
//
// All router <-> engine traffic is in shared memory, each datum written by its owner into
// its own CTA's shared memory and read by the other side over DSMEM, so the release is
// fence.release.sync_restrict::shared::cta.cluster (MEMBAR.ALL.CTA in SASS) and the acquire
// fence.acquire.sync_restrict::shared::cluster.cluster (no instruction): no global-scope
// fence and no L1 invalidation (a fence.acq_rel.cluster is MEMBAR.ALL.GPU + CCTL.IVALL,
// which flushed the engines' L1 at every wake in a first version).
//   router -> engine: per server a ring of routed arrival ids and its published count in
//     rank 0, the watermark word pushed into each CTA, a wake hint (the count) pushed next
//     to it; the engine copies new ids into its own global route list and reports how far
//     it has taken (flow control: the router waits before overwriting an untaken slot).
//   engine -> router: at a sync the snapshot in the engine's CTA, then its done word pushed
//     into rank 0.
constexpr int PIPE_WARPS = 8;
constexpr int PIPE_MAX_CTAS = 16;  // non-portable cluster size (cudaFuncAttributeNonPortableClusterSizeAllowed)
constexpr int PIPE_MAX_SERVERS = PIPE_WARPS * (PIPE_MAX_CTAS - 1);
constexpr int PIPE_RING = 128;     // routed ids in flight per server (>= 32: one route-log flush)
constexpr unsigned long long SYNC_BIT = 0x8000000000000000ULL;  // watermark times are >= 0 (sign bit free)

// cluster warp of server s: rank 0 is the routing warp's alone (its SM's issue slots and
// shared-memory port serve the serial routing chain), the servers take every warp of ranks 1..
// epc engine warps per CTA (4 for small clusters: fewer co-resident engines per SM; 8 for large)
__host__ __device__ constexpr int pipe_rank(int s, int epc) { return 1 + s / epc; }
__host__ __device__ constexpr int pipe_warp(int s, int epc) { return s % epc; }
__device__ __forceinline__ int pipe_server(int rank, int warp, int epc) {
  return rank >= 1 && warp < epc ? (rank - 1) * epc + warp : -1;
}

__device__ __forceinline__ void release_smem() {
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
__device__ __forceinline__ void acquire_smem() {
  asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}
__device__ __forceinline__ void st_rc_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.cluster.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rc_s32(int* p, int v) {
  asm volatile("st.relaxed.cluster.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_rc_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.cluster.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rc_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.cluster.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_rc_s64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.cluster.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// an engine's ground truth at a sync (snapshot_stats + BetaEstimator sums), in its own CTA
struct PipeSnap {
  long long wpend, enq, fc, fi, fo;
  int free_b, wr, next, _pad;
  unsigned long long done;  // the last sync word the engine reached (read by the router over DSMEM)
};
#ifdef SSB_PIPE_TIMELINE
// sync timeline of the first instance (tools/probe_sync.py): per sync, the router's publish and
// all-done %globaltimer ns, then per server (wake ns, done ns, iterations run in that wake)
constexpr int SYNC_TL_MAX = 4096, SYNC_TL_W = 2 + 3 * 128;
__device__ unsigned long long g_sync_tl[SYNC_TL_MAX * SYNC_TL_W];
#endif
// per-CTA control block (static shared); rank 0's abort / err / counters are the instance's
struct PipeCtl {
  unsigned long long wt;  // watermark word (router -> this CTA): time bits | SYNC_BIT
  int hint[PIPE_WARPS];   // published route counts of this CTA's engines (wake hints)
  int abort, err;
  int syncs, polls;       // diagnostics
  PipeSnap snap[PIPE_WARPS];
#ifdef SSB_PIPE_PROBE
  unsigned long long p_wait, p_route, p_flush, p_busy_sum, p_busy_max, p_wakes, p_iters_max, p_take, p_arr, p_pub, p_sync, p_chunk;
#endif
};

// rank 0's dynamic shared memory, per server (n_al = n rounded up to even)
struct PipeArrays {
  long long* rps;    // Σ prompt routed (router)
  int *cnt, *taken;  // routed (router) / taken by the engine (engine -> router, flow control)
  int* ring;         // [n][PIPE_RING] routed arrival ids
  __device__ PipeArrays(long long* b, int n_al) {
    rps = b;
    int* ib = (int*)(b + n_al);
    cnt = ib; taken = ib + n_al;
    ring = ib + 2 * n_al;
  }
};
__host__ __device__ constexpr long long pipe_array_bytes(int n) {
  return 8LL * ((n + 1) & ~1) + 4LL * 2 * ((n + 1) & ~1) + 4LL * PIPE_RING * n;
}

// the routing warp. Plain locals and force-inlined helpers that take them by reference
// (a struct or lambdas holding the view put it in local memory: measured, the fast path then
// paid local loads per arrival)
struct PipeLog {  // route log: lane i holds the server / prompt of arrival klog + i
  int slog, plog, nlog, klog;
};
// publish: append the logged routes to their rings, ONE release (MEMBAR.ALL.CTA: it waits for
// the warp's outstanding stores, so a publish costs one), then the wake hints (the new counts)
// and the watermark word. The log holds at most 32 routes (publish_every <= 32), and it is
// only flushed here, so every ring slot the flow control waits on was hinted before.
template <int BAL>
__device__ __forceinline__ void pipe_publish(PipeLog& g, PipeArrays& A, PipeCtl& C, int lane,
                                             unsigned long long* wt_lane, unsigned long long word, int epc) {
#ifdef SSB_PIPE_PROBE
  const long long pf0 = clock64();
#endif
  cg::cluster_group cl = cg::this_cluster();
  const bool valid = lane < g.nlog;
  const int s = valid ? g.slog : -1;
  const unsigned grp = __match_any_sync(FULL, s);
  const int leader = __ffs(grp) - 1;
  const int before = __popc(grp & lanemask_lt());
  const int gsz = __popc(grp);
  int base = 0;
  if (g.nlog) {
    base = valid ? A.cnt[s] : 0;
    // flow control: the engine has taken everything published (base) up to the ring size
    while (__any_sync(FULL, valid && base + gsz - *(volatile int*)&A.taken[s] > PIPE_RING)) __nanosleep(64);
    if (valid) {
      A.ring[s * PIPE_RING + ((base + before) & (PIPE_RING - 1))] = g.klog + lane;
      if (BAL == SSB_BAL_SAL || BAL == SSB_BAL_P2C) atomicAdd((unsigned long long*)&A.rps[s], (unsigned long long)(long long)g.plog);
      if (lane == leader) A.cnt[s] = base + gsz;
    }
    __syncwarp();
  }
  release_smem();  // ring slots (and abort) before their counts and the watermark
  if (valid && lane == leader)
    st_rc_s32(&cl.map_shared_rank(&C, pipe_rank(s, epc))->hint[pipe_warp(s, epc)], base + gsz);
  if (wt_lane) st_rc_u64(wt_lane, word);
  __syncwarp();
  g.klog += g.nlog;
  g.nlog = 0;
#ifdef SSB_PIPE_PROBE
  if (lane == 0) C.p_flush += clock64() - pf0;
#endif
}

template <int BAL, int VPL>
__device__ __forceinline__ void pipe_router(const ssb_instance& I, const Cfg& cfg, const double* __restrict__ arr,
                                            const int* __restrict__ prm, PipeArrays A, PipeCtl& C, int G,
                                            int publish_every, int epc) {
  cg::cluster_group cl = cg::this_cluster();
  const int lane = lane_id();
  const int n = I.n_servers;
  const long long N = I.n_requests;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const bool est_beta = BAL == SSB_BAL_SAL && isnan(I.beta_fixed);
  const double beta_prior = I.beta_prior;
  const int route_cap = I.route_cap;
  const bool cap_pow2 = route_cap > 0 && (route_cap & (route_cap - 1)) == 0;
  const double inv_cap = cap_pow2 ? __ddiv_rn(1.0, (double)route_cap) : 0.0;
  const double poll = I.poll_interval_s;
  const int bs = cfg.bs;
  Pcg rng;
  rng.shi = I.pcg_state_hi; rng.slo = I.pcg_state_lo; rng.ihi = I.pcg_inc_hi; rng.ilo = I.pcg_inc_lo;
  rng.has = 0; rng.buf = 0;
  unsigned long long* const wt_lane = lane < G ? &cl.map_shared_rank(&C, lane)->wt : nullptr;
  // the polled BalancerView (balancers.py:29-64) in registers: queued tokens also as the SAL
  // key key0 = queued << 13 | server << 1 (the argmin order of queued+prompt with the lowest
  // server among ties; ~0 for lanes past n), free memory, in-flight; where each snapshot lives
  unsigned long long key0[VPL];
  long long vq[VPL], vf[VPL];
  int vif[VPL], bsj[VPL];  // bsj: each server's own block size (prebuilt engines may differ)
  const PipeSnap* snp[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int q = lane + 32 * j;
    key0[j] = q < n ? (unsigned long long)q << 1 : ~0ULL;
    bsj[j] = q < n ? server_params(I, q).block_size : bs;
    vq[j] = 0; vf[j] = q < n ? (long long)server_params(I, q).pool_blocks * bsj[j] : 0; vif[j] = 0;
    snp[j] = q < n ? &cl.map_shared_rank(&C, pipe_rank(q, epc))->snap[pipe_warp(q, epc)] : nullptr;
  }
  bool anybig = false;  // some queued >= 2^50: the integer key would not be exact (warp-uniform)
  double beta = isnan(I.beta_fixed) ? beta_prior : I.beta_fixed;
  PipeLog g;
  g.slog = g.plog = g.nlog = g.klog = 0;
  int k = 0, k_pub = 0;
  double last_poll = 0.0;  // the refresh at 0.0 (cluster.py:122) sees the empty engines: the init above
  int synced = 1;
  int rr_next = 0;
  // arrival times / prompts 32 at a time, the next 32 in flight (lane i holds c0 + i)
  int c0 = 0;
  double c_t = lane < N ? arr[lane] : 0.0, n_t = 0.0;
  int c_pr = lane < N ? prm[lane] : 0, n_pr = 0;
  if (32 + lane < N) { n_t = arr[32 + lane]; n_pr = prm[32 + lane]; }
  // per chunk, as bit masks over its 32 arrivals: the arrival's time equals the previous one's
  // (no simulated time passes: a sync stays valid), and the arrival is due for a poll refresh
  // (BalancerView.due, balancers.py:42-43, against the current last_poll)
  unsigned eq_mask = 0, due_mask = 0;
  auto chunk_masks = [&](double t_last) {
    const double up = __shfl_up_sync(FULL, c_t, 1);
    eq_mask = __ballot_sync(FULL, (lane == 0 ? t_last : up) == c_t);
    if (BAL == SSB_BAL_SAL || BAL == SSB_BAL_P2C) due_mask = __ballot_sync(FULL, __dsub_rn(c_t, last_poll) >= poll);
  };
  chunk_masks(__shfl_sync(FULL, c_t, 0));  // arrival 0: the engines are synced at the start
  bool aborted = false, need_sync = false;
  double t_sync = 0.0;
#ifdef SSB_PIPE_PROBE
  const long long pr0 = clock64();
#endif
  while (true) {
    if (need_sync) {
      // the one sync site (a route that reads engine state, or the final drain): every engine
      // to time t_sync (wt = t_sync with the sync bit), then their snapshots are readable
      need_sync = false;
#ifdef SSB_PIPE_PROBE
      const long long ps0 = clock64();
#endif
      const unsigned long long word = (unsigned long long)__double_as_longlong(t_sync) | SYNC_BIT;
#ifdef SSB_PIPE_TIMELINE
      const unsigned long long tl0 = globaltimer_ns();
#endif
      pipe_publish<BAL>(g, A, C, lane, wt_lane, word, epc);
      k_pub = k;
#ifdef SSB_PIPE_PROBE
      const long long pw0 = clock64();
#endif
      bool ok;
      do {  // each engine's done word in its own CTA, polled over DSMEM (one round trip per pass)
        ok = true;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (snp[j]) ok &= ld_rc_u64(&snp[j]->done) == word;
      } while (!__all_sync(FULL, ok));
      acquire_smem();
#ifdef SSB_PIPE_PROBE
      if (lane == 0) C.p_wait += clock64() - pw0;
#endif
#ifdef SSB_PIPE_TIMELINE
      if (lane == 0 && blockIdx.x == 0 && C.syncs < SYNC_TL_MAX) {
        g_sync_tl[(long long)C.syncs * SYNC_TL_W] = tl0;
        g_sync_tl[(long long)C.syncs * SYNC_TL_W + 1] = globaltimer_ns();
      }
#endif
      if (lane == 0) C.syncs += 1;
      if (*(volatile int*)&C.err) { aborted = true; break; }
      if (est_beta) {  // on_finish sums of every engine (balancers.py:81-100) folded at the sync
        long long fc = 0, fi = 0, fo = 0;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (snp[j]) { fc += ld_rc_s64(&snp[j]->fc); fi += ld_rc_s64(&snp[j]->fi); fo += ld_rc_s64(&snp[j]->fo); }
        fc = warp_sum_ll(fc); fi = warp_sum_ll(fi); fo = warp_sum_ll(fo);
        beta = fc == 0 ? beta_prior : __ddiv_rn((double)(fi + fo), (double)fo);
      }
      synced = 1;
#ifdef SSB_PIPE_PROBE
      if (lane == 0) C.p_sync += clock64() - ps0;
#endif
      if (k >= N) break;
    }
    if (k >= N) { t_sync = INF; need_sync = true; continue; }  // drain: every engine to the end
#ifdef SSB_PIPE_PROBE
    const long long pc0 = clock64();
#endif
    if (k >= c0 + 32) {
      const double t_last = __shfl_sync(FULL, c_t, 31);
      c0 += 32;
      c_t = n_t; c_pr = n_pr;
      const long long kk = (long long)c0 + 32 + lane;
      if (kk < N) { n_t = arr[kk]; n_pr = prm[kk]; }
      chunk_masks(t_last);
    }
#ifdef SSB_PIPE_PROBE
    const long long pa0 = clock64();
    if (lane == 0) C.p_chunk += pa0 - pc0;
#endif
    const int ik = k - c0;
    const int pr = __shfl_sync(FULL, c_pr, ik);
    synced = (eq_mask >> ik) & 1u ? synced : 0;  // equal times need no sync (no simulated time passes)
    int s = 0;
    if constexpr (BAL == SSB_BAL_SAL || BAL == SSB_BAL_P2C) {
      if ((due_mask >> ik) & 1u) {  // BalancerView.due (balancers.py:42-43)
        const double t = __shfl_sync(FULL, c_t, ik);
        if (!synced) { need_sync = true; t_sync = t; eq_mask |= 1u << ik; continue; }
        // ground truth incl. routed-but-unseen inbox (cluster.py:110-120, 50-59)
        bool big = false;
#pragma unroll
        for (int j = 0; j < VPL; ++j)
          if (snp[j]) {
            const int q = lane + 32 * j;
            const long long wp = ld_rc_s64(&snp[j]->wpend), en = ld_rc_s64(&snp[j]->enq);
            const int fb = ld_rc_s32(&snp[j]->free_b), wr = ld_rc_s32(&snp[j]->wr), nx = ld_rc_s32(&snp[j]->next);
            vq[j] = wp + (A.rps[q] - en);
            key0[j] = ((unsigned long long)vq[j] << 13) | ((unsigned)q << 1);
            big |= vq[j] >= (1LL << 50);
            vf[j] = (long long)fb * bsj[j];  // snapshot_stats: free_blocks * block_size (cluster.py:54)
            vif[j] = wr + (A.cnt[q] - nx);
          }
        anybig = __any_sync(FULL, big);
        last_poll = t;
        due_mask = __ballot_sync(FULL, __dsub_rn(c_t, last_poll) >= poll);
        if (lane == 0) C.polls += 1;
      }
    }
    if constexpr (BAL == SSB_BAL_RR) {  // balancers.py:132-142
      s = rr_next;
      rr_next = rr_next + 1 == n ? 0 : rr_next + 1;
    } else if constexpr (BAL == SSB_BAL_RANDOM) {  // :145-153
      s = rng.integers(n);
    } else if constexpr (BAL == SSB_BAL_P2C) {  // :156-176, the polled in_flight only
      if (n > 1) {
        const int i = rng.integers(n);
        int j2 = rng.integers(n - 1);
        if (j2 >= i) j2 += 1;
        int a = vif[0], b = vif[0];
        const unsigned mi = 1u << (i >> 5), mj = 1u << (j2 >> 5);
#pragma unroll
        for (int j = 1; j < VPL; ++j) { a = (mi >> j) & 1u ? vif[j] : a; b = (mj >> j) & 1u ? vif[j] : b; }
        a = __shfl_sync(FULL, a, i & 31);
        b = __shfl_sync(FULL, b, j2 & 31);
        s = b < a ? j2 : i;
      }
    } else {  // SAL (:179-216)
      // fast path (see k_cluster): a 64-bit warp minimum over queued << 13 | server << 1 |
      // constrained ((queued + prompt, server) orders as (queued, server): the prompt is
      // common); an unconstrained winner is the load argmin for every beta
      bool fast = false;
      if (cap_pow2 && beta > 0.0 && pr > 0 && !anybig) {
        unsigned long long kx = key0[0] | (unsigned long long)(vf[0] < pr);
#pragma unroll
        for (int j = 1; j < VPL; ++j) {
          const unsigned long long key = key0[j] | (unsigned long long)(vf[j] < pr);
          kx = key < kx ? key : kx;
        }
        const unsigned long long m = warp_min_u64(kx);
        if (!(m & 1ULL)) {
          s = (int)((m >> 1) & 0xfffULL);
          fast = true;
          anybig = (long long)(m >> 13) + pr >= (1LL << 50);  // the winner's queued after note_routed
        } else if (est_beta && !synced) {  // a constrained server leads: beta decides
          need_sync = true; t_sync = __shfl_sync(FULL, c_t, ik); eq_mask |= 1u << ik;
          continue;  // then route arrival k again
        }
      }
      if (!fast) {
        unsigned long long kl = ~0ULL, ku = ~0ULL, kc = ~0ULL;
        int sl = 0x7fffffff, su = 0x7fffffff, sc = 0x7fffffff;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int q = lane + 32 * j;
          if (q < n) {
            const double que = cap_pow2 ? __dmul_rn((double)(vq[j] + pr), inv_cap)
                                        : __ddiv_rn((double)(vq[j] + pr), (double)route_cap);
            const double mem = __dmul_rn(beta, (double)((long long)pr - vf[j]));
            const double load = que > mem ? que : mem;  // sal_load (balancers.py:103-112)
            const unsigned long long k1 = dkey(load), kq = dkey(que);
            if (k1 < kl) { kl = k1; sl = q; }  // q ascending: ties keep the lower server
            if (vf[j] < pr) { if (kq < kc) { kc = kq; sc = q; } }
            else if (kq < ku) { ku = kq; su = q; }
          }
        }
        if (est_beta && !synced) {  // beta-independent argmin? (see k_cluster)
          const unsigned long long mc = warp_min_u64(kc);
          if (mc != ~0ULL) {
            const unsigned long long mu = warp_min_u64(ku);
            const int iu = mu == ~0ULL ? 0x7fffffff : (int)__reduce_min_sync(FULL, ku == mu ? (unsigned)su : 0x7fffffffu);
            const int ic = (int)__reduce_min_sync(FULL, kc == mc ? (unsigned)sc : 0x7fffffffu);
            const bool indep = mu != ~0ULL && (mu < mc || (mu == mc && iu < ic));
            if (!indep) { need_sync = true; t_sync = __shfl_sync(FULL, c_t, ik); eq_mask |= 1u << ik; continue; }
          }
        }
        const unsigned long long ml = warp_min_u64(kl);
        s = (int)__reduce_min_sync(FULL, kl == ml ? (unsigned)sl : 0x7fffffffu);
        const unsigned own = lane == (s & 31) ? 1u << (s >> 5) : 0u;
        bool b = false;
#pragma unroll
        for (int j = 0; j < VPL; ++j) b |= ((own >> j) & 1u) && vq[j] + pr >= (1LL << 50);
        anybig = __any_sync(FULL, b) || anybig;
      }
      // note_routed (balancers.py:59-64) on the owner lane: per-element selects on a bit mask,
      // so that no dynamically indexed access puts the view in local memory
      const unsigned own = lane == (s & 31) ? 1u << (s >> 5) : 0u;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const bool o = (own >> j) & 1u;
        key0[j] = o ? key0[j] + ((unsigned long long)pr << 13) : key0[j];  // exact while queued < 2^50 (else anybig)
        vq[j] = o ? vq[j] + pr : vq[j];
        const long long f = vf[j] - pr;
        vf[j] = o ? (f > 0 ? f : 0) : vf[j];
        vif[j] = o ? vif[j] + 1 : vif[j];
      }
    }
#ifdef SSB_PIPE_PROBE
    if (lane == 0) C.p_arr += clock64() - pa0;
#endif
    if (publish_every == 1 && k + 1 < N) {
      // streamlined publish of one route (no log, no match_any): the ring slot, one release,
      // the wake hint and the watermark = the next arrival's time
      cg::cluster_group cl = cg::this_cluster();
      SSB_ASSERT(s >= 0 && s < n);
      const int base = A.cnt[s];
      while (base + 1 - *(volatile int*)&A.taken[s] > PIPE_RING) __nanosleep(64);  // flow control
      if (lane == 0) {
        A.ring[s * PIPE_RING + (base & (PIPE_RING - 1))] = k;
        if (BAL == SSB_BAL_SAL || BAL == SSB_BAL_P2C) A.rps[s] += pr;
        A.cnt[s] = base + 1;
      }
      __syncwarp();
      release_smem();
      if (lane == 0) st_rc_s32(&cl.map_shared_rank(&C, pipe_rank(s, epc))->hint[pipe_warp(s, epc)], base + 1);
      k += 1;
      const double tn = k < c0 + 32 ? __shfl_sync(FULL, c_t, k - c0) : __shfl_sync(FULL, n_t, k - c0 - 32);
      if (wt_lane) st_rc_u64(wt_lane, (unsigned long long)__double_as_longlong(tn));
      __syncwarp();
      g.klog = k;
      k_pub = k;
      continue;
    }
    SSB_ASSERT(s >= 0 && s < n);  // cluster.py:134-135 (the reference raises for an invalid server)
    if (lane == g.nlog) { g.slog = s; g.plog = pr; }
    g.nlog += 1;
    k += 1;
    if (k - k_pub >= publish_every && k < N) {
      const double tn = k < c0 + 32 ? __shfl_sync(FULL, c_t, k - c0) : __shfl_sync(FULL, n_t, k - c0 - 32);
#ifdef SSB_PIPE_PROBE
      const long long pp0 = clock64();
#endif
      pipe_publish<BAL>(g, A, C, lane, wt_lane, (unsigned long long)__double_as_longlong(tn), epc);
      k_pub = k;
#ifdef SSB_PIPE_PROBE
      if (lane == 0) C.p_pub += clock64() - pp0;
#endif
    }
  }
#ifdef SSB_PIPE_PROBE
  if (lane == 0) C.p_route = clock64() - pr0;
#endif
  if (aborted) {
    if (lane == 0) C.abort = 1;
    pipe_publish<BAL>(g, A, C, lane, wt_lane, (unsigned long long)__double_as_longlong(INF) | SYNC_BIT, epc);  // wake everyone
  }
}

#ifndef SSB_PIPE_NAP_MAX
#define SSB_PIPE_NAP_MAX 256  // ns: the engines' watermark-poll back-off cap
#endif
template <int POL>
__device__ __forceinline__ void pipe_body(const ssb_instance* __restrict__ inst, const int* __restrict__ order,
                                          ssb_trace tr, ssb_records rec, ssb_stats* __restrict__ stats,
                                          unsigned char* __restrict__ scratch, ssb_event* events, long long ev_cap,
                                          int64_t* ev_count, long long* smem_ll, PipeCtl& C, int publish_every, int epc) {
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int idx = order[blockIdx.x / G];
  const ssb_instance I = inst[idx];
  const int n = I.n_servers;
  const long long N = I.n_requests;
  const int n_al = (n + 1) & ~1;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int gw = rank * PIPE_WARPS + warp;
  const int s = pipe_server(rank, warp, epc);  // this warp's server (-1: the router or a spare warp)
  PipeCtl& C0 = rank == 0 ? C : *cl.map_shared_rank(&C, 0);
  PipeArrays A(rank == 0 ? smem_ll : cl.map_shared_rank(smem_ll, 0), n_al);
  int* const tab = (int*)((unsigned char*)smem_ll + align_up(pipe_array_bytes(n), 16)) + warp * SM_COLS * RS;
  const int s_own = s >= 0 && s < n ? s : 0;  // the router / spare warps take server 0's set
  Cfg cfg = make_cfg(I, server_params(I, s_own));  // each replica with its own engine parameters
  cfg.policy = POL;
  const Layout L = inst_layout(I);
  const Layout Ls = server_layout(I, s_own);  // its own trail tree offsets
  ssb_event* evb = events ? events + (long long)idx * ev_cap : nullptr;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);

  // ---- init: control blocks, rank 0's counters, records, engines ----
  if (threadIdx.x == 0) {
    C.wt = 0ULL;  // +0.0, no sync: nothing routed
    C.abort = C.err = C.syncs = C.polls = 0;
#ifdef SSB_PIPE_PROBE
    C.p_wait = C.p_route = C.p_flush = C.p_busy_sum = C.p_busy_max = C.p_wakes = C.p_iters_max = C.p_take = 0;
    C.p_arr = C.p_pub = C.p_sync = C.p_chunk = 0;
#endif
  }
  if (threadIdx.x < PIPE_WARPS) C.hint[threadIdx.x] = 0;
  if (rank == 0)
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      A.rps[q] = 0;
      A.cnt[q] = A.taken[q] = 0;
    }
  {
    Eng E;
    bind_engine(E, I, cfg, scratch, 0, L, tr, rec, evb, ev_cap);
    clear_records(E, N, rank * blockDim.x + threadIdx.x, G * blockDim.x);
  }
  Eng E;
  const bool engine = s >= 0 && s < n;
  if (engine) {
    bind_engine(E, I, cfg, scratch, s, Ls, tr, rec, evb, ev_cap, tab);
    init_srv(E.st, cfg);
    if (POL == SSB_POLICY_TRAIL_PLUS) E.trail_init();
    fill_events(E, lane, 32);
    if (lane == 0) {  // the snapshot of the empty engine: a refresh before the first sync reads it
      PipeSnap& sn = C.snap[warp];
      sn.wpend = sn.enq = sn.fc = sn.fi = sn.fo = 0;
      sn.free_b = cfg.pool;
      sn.wr = sn.next = sn._pad = 0;
      sn.done = 0ULL;
    }
  }
  cl.sync();

  if (gw == 0) {
    const double* arr = instance_arrivals(I, L, tr, scratch);  // already divided by qps_factor
    const int* prm = tr.prompt + I.trace_offset;
    const bool v2 = n <= 64;
    switch (I.balancer) {
      case SSB_BAL_RR: pipe_router<SSB_BAL_RR, 1>(I, cfg, arr, prm, A, C, G, 32, epc); break;
      case SSB_BAL_RANDOM: pipe_router<SSB_BAL_RANDOM, 1>(I, cfg, arr, prm, A, C, G, 32, epc); break;
      case SSB_BAL_P2C:
        if (v2) pipe_router<SSB_BAL_P2C, 2>(I, cfg, arr, prm, A, C, G, publish_every, epc);
        else pipe_router<SSB_BAL_P2C, 4>(I, cfg, arr, prm, A, C, G, publish_every, epc);
        break;
      default:
        if (v2) pipe_router<SSB_BAL_SAL, 2>(I, cfg, arr, prm, A, C, G, publish_every, epc);
        else pipe_router<SSB_BAL_SAL, 4>(I, cfg, arr, prm, A, C, G, publish_every, epc);
        break;
    }
  } else if (engine) {
    // ---- engine: take the new routes, advance to every watermark that lets it progress ----
    E.init_modes();
    unsigned long long seen = 0ULL;
    int seen_hint = 0, taken = 0;
    double nb_lb = INF;  // lower bound of its next boundary: idle with nothing routed
    bool reported = false;
#ifdef SSB_PIPE_PROBE
    long long p_bs = 0, p_wk = 0, p_tk = 0;
#endif
#ifdef SSB_PIPE_TIMELINE
    long long p_sy = 0;
#endif
    volatile PipeCtl& V = C;
    const int* ring = A.ring + s * PIPE_RING;
    while (true) {
      unsigned long long w;
      int h, nap = 32;
      while (true) {
        w = V.wt;
        acquire_smem();  // the watermark word (or the hint) is the flag of a release pattern
        h = V.hint[warp];  // the published route count: ring slots below it are readable
        if (w != seen || h != seen_hint) {
          const double wt = __longlong_as_double((long long)(w & ~SYNC_BIT));
          if ((w & SYNC_BIT) || nb_lb < wt || h != seen_hint) break;
          seen = w;  // nothing to do before this watermark
        } else {
          __nanosleep(nap);  // back off: polling warps share the issue slots with working ones
          nap = nap < SSB_PIPE_NAP_MAX ? 2 * nap : SSB_PIPE_NAP_MAX;
        }
      }
      seen = w;
#ifdef SSB_PIPE_PROBE
      const long long pe0 = clock64();
      p_wk += 1;
#endif
#ifdef SSB_PIPE_TIMELINE
      const unsigned long long tw0 = globaltimer_ns();
      const long long it0 = E.st.iterations;
#endif
      // take the published routes into the engine's own route list (global, rl)
      const int cp = h;
      if (cp > taken) {
        int dep = 0;
        for (int b = taken; b < cp; b += 32) {
          const int i = b + lane;
          if (i < cp) {
            const int v = ld_rc_s32(&ring[i & (PIPE_RING - 1)]);
            SSB_ASSERT(i < N && v >= 0 && v < N);  // a published route: an arrival id of this instance
            E.p.rl[i] = v;
            dep |= v;
          }
        }
        taken = cp;
        // the reported count depends on the loaded ids: the slots are read before the router reuses them
        dep = __reduce_or_sync(FULL, dep);
        if (lane == 0) st_rc_s32(&A.taken[s], dep == -1 ? 0 : cp);
        __syncwarp();
      }
      seen_hint = cp;
      const bool sync = (w & SYNC_BIT) != 0;
      const double wt = __longlong_as_double((long long)(w & ~SYNC_BIT));
#ifndef SSB_ABORT_EVERY_SYNC
      // the router aborts by publishing +inf with the sync bit after setting C.abort: only
      // that word needs the (DSMEM) abort load, not every poll sync
      if (sync && !(wt < INF) && ld_rc_s32(&C0.abort)) {
#else
      if (sync && ld_rc_s32(&C0.abort)) {
#endif
        if (lane == 0) *(volatile unsigned long long*)&C.snap[warp].done = w;
        break;
      }
#ifdef SSB_PIPE_PROBE
      p_tk += clock64() - pe0;
#endif
#ifndef SSB_PIPE_NOENGINE
      // still in the steady state the last wake ended in (the watermark stopped it, nothing was
      // enqueued since): continue the decode-only iterations in the tight loop right away,
      // instead of a full step() per wake (exactly what advance_loop's first boundary would do)
      if (E.regs_ok && E.nodisp && E.st.status == SSB_OK && E.cfg.bs_shift >= 0 && E.has_work()) {
        const double na = E.next_arrival(taken);
        E.fast_forward(na < wt ? na : wt);
      }
      E.advance_loop(wt, taken);
#endif
#ifdef SSB_PIPE_PROBE
      p_bs += clock64() - pe0;
#endif
      if (E.st.status && !reported) {
        reported = true;
        if (lane == 0) st_rc_s32(&C0.err, E.st.status);
      }
      if (E.has_work()) {
        nb_lb = E.st.clock;
      } else {
        const double na = E.next_arrival(taken);
        nb_lb = na > E.st.clock ? na : E.st.clock;
      }
      if (sync) {
        if (lane == 0) {  // the ground-truth snapshot at wt (snapshot_stats, cluster.py:50-59)
          PipeSnap& sn = C.snap[warp];
          sn.wpend = E.st.wpend_sum;
          sn.enq = E.st.enq_prompt_sum;
          sn.fc = E.st.fin_cnt;
          sn.fi = E.st.fin_in;
          sn.fo = E.st.fin_out;
          sn.free_b = E.st.free_blocks;
          sn.wr = E.st.W + E.st.R;
          sn.next = E.st.next_arr;
        }
        __syncwarp();
        release_smem();
#ifdef SSB_PIPE_TIMELINE
        if (lane == 0 && blockIdx.x < G && p_sy < SYNC_TL_MAX && s < 128) {
          unsigned long long* r = g_sync_tl + (long long)p_sy * SYNC_TL_W + 2 + 3 * s;
          r[0] = tw0; r[1] = globaltimer_ns(); r[2] = (unsigned long long)(E.st.iterations - it0);
        }
        p_sy += 1;
#endif
        if (lane == 0) *(volatile unsigned long long*)&C.snap[warp].done = w;
        if (!(wt < INF)) break;
      }
    }
    E.drop_regs();
    if (lane == 0) *(Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv) = E.st;
#ifdef SSB_PIPE_PROBE
    if (lane == 0) {
      atomicAdd(&C0.p_busy_sum, (unsigned long long)p_bs);
      atomicMax(&C0.p_busy_max, (unsigned long long)p_bs);
      atomicAdd(&C0.p_wakes, (unsigned long long)p_wk);
      atomicAdd(&C0.p_take, (unsigned long long)p_tk);
      atomicMax(&C0.p_iters_max, (unsigned long long)E.st.iterations);
    }
#endif
  }
  cl.sync();  // every engine's state is in memory; rank 0's shared memory outlives its readers

  // ---------------- per-instance stats ----------------
  if (rank == 0 && threadIdx.x == 0) {
    ssb_stats out;
    memset(&out, 0, sizeof(out));
    unsigned long long h = FNV_OFF;
    int status = C.err;
    long long evn = 0;
    for (int q = 0; q < n; ++q) {
      const Srv* sv = (const Srv*)(scratch + I.scratch_offset + (long long)q * L.total + L.srv);
      out.iterations += sv->iterations;
      out.request_steps += sv->rsteps;
      out.batch_tokens += sv->btokens;
      out.dispatches += sv->dispatches;
      out.preempts += sv->preempts;
      out.parks += sv->parks;
      out.finished += sv->finished;
      if (sv->peak > out.peak_batch_tokens) out.peak_batch_tokens = sv->peak;
      h ^= sv->digest; h *= FNV_PRIME;
      if (!status && sv->status) status = sv->status;
      if (!status && (sv->W != 0 || sv->R != 0)) status = SSB_E_INVARIANT;
      evn += sv->ev_n;
    }
    if (!status && out.finished != N) status = SSB_E_INVARIANT;  // cluster.py:159-161
    out.digest = h;
    out.status = status;
#ifdef SSB_PIPE_PROBE
    out._pad = C.syncs;            // diagnostics: engine syncs (routing epochs)
    out.device_cycles = C.polls;   //              view refreshes
    printf("PIPE inst %d n %d N %lld syncs %d polls %d | router total %llu wait %llu flush %llu | engines busy sum %llu max %llu "
           "wakes %llu take %llu iters_max %llu | per-arrival %llu publish %llu sync %llu chunk %llu\n", idx, n, N, C.syncs, C.polls, C.p_route, C.p_wait, C.p_flush,
           C.p_busy_sum, C.p_busy_max, C.p_wakes, C.p_take, C.p_iters_max, C.p_arr, C.p_pub, C.p_sync, C.p_chunk);
#endif
    stats[idx] = out;
    if (ev_count) ev_count[idx] = evn;
  }
}

__global__ void __launch_bounds__(32 * PIPE_WARPS, 1)
k_cluster_pipe(const ssb_instance* __restrict__ inst, const int* __restrict__ order, ssb_trace tr, ssb_records rec,
               ssb_stats* __restrict__ stats, unsigned char* __restrict__ scratch, ssb_event* events, long long ev_cap,
               int64_t* ev_count, int publish_every, int epc) {
  extern __shared__ long long smem_ll[];
  __shared__ PipeCtl C;
  const int G = (int)cg::this_cluster().num_blocks();
  const ssb_instance* const Ip = inst + order[blockIdx.x / G];
  int pol = Ip->engine.policy;
  if (Ip->d_servers != nullptr) {  // prebuilt engines that differ: each engine warp runs its own server's
    // policy (a warp-uniform choice; every instantiation passes the same two cluster barriers and
    // talks to the router through the same shared-memory protocol); the router takes server 0's
    const int s = pipe_server((int)cg::this_cluster().block_rank(), threadIdx.x >> 5, epc);
    if (s >= 0 && s < Ip->n_servers) pol = Ip->d_servers[s].policy;
  }
  switch (pol) {
    case SSB_POLICY_FCFS: pipe_body<SSB_POLICY_FCFS>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_ll, C, publish_every, epc); break;
    case SSB_POLICY_NOPREEMPT: pipe_body<SSB_POLICY_NOPREEMPT>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_ll, C, publish_every, epc); break;
    case SSB_POLICY_TRAIL_PLUS: pipe_body<SSB_POLICY_TRAIL_PLUS>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_ll, C, publish_every, epc); break;
    default: pipe_body<SSB_POLICY_LARRY>(inst, order, tr, rec, stats, scratch, events, ev_cap, ev_count, smem_ll, C, publish_every, epc); break;
  }
}

// per-engine counters: a cluster's servers from the per-server state k_cluster leaves in
// the scratch buffer after every advance; a single-server instance from its ssb_stats
// (k_engines keeps no per-engine copy: one more store of the engine state at the end of
// run_instance measured 130 vs 119 ms on the C4 sweep), its clock = its latest finish
__global__ void k_engine_stats(const ssb_instance* __restrict__ inst, int n_inst,
                               const unsigned char* __restrict__ scratch, const ssb_stats* __restrict__ stats,
                               const double* __restrict__ finish, const int64_t* __restrict__ ev_count,
                               const int64_t* __restrict__ row0, ssb_engine_stats* __restrict__ out) {
  __shared__ double red[32];
  for (int i = blockIdx.x; i < n_inst; i += gridDim.x) {
    const ssb_instance I = inst[i];
    if (I.n_servers == 1) {
      double m = 0.0;  // Engine.clock starts at 0.0 (engine.py:164)
      for (long long r = threadIdx.x; r < I.n_requests; r += blockDim.x) m = fmax(m, finish[I.record_offset + r]);
      #pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        const ssb_stats st = stats[i];
        ssb_engine_stats e;
        e.iterations = st.iterations;
        e.request_steps = st.request_steps;
        e.batch_tokens = st.batch_tokens;
        e.dispatches = st.dispatches;
        e.preempts = st.preempts;
        e.parks = st.parks;
        e.finished = st.finished;
        e.peak_batch_tokens = st.peak_batch_tokens;
        // instance digest = (FNV_OFF ^ d) * FNV_PRIME over its one engine: invert the multiply
        e.digest = (st.digest * FNV_PRIME_INV) ^ FNV_OFF;
        e.event_count = ev_count ? ev_count[i] : 0;
        e.clock = m;
        e.status = st.status;
        e._pad = 0;
        out[row0[i]] = e;
      }
      __syncthreads();
      continue;
    }
    const Layout L = inst_layout(I);
    for (int s = threadIdx.x; s < I.n_servers; s += blockDim.x) {
      const Srv* sv = (const Srv*)(scratch + I.scratch_offset + (long long)s * L.total + L.srv);
      ssb_engine_stats e;
      e.iterations = sv->iterations;
      e.request_steps = sv->rsteps;
      e.batch_tokens = sv->btokens;
      e.dispatches = sv->dispatches;
      e.preempts = sv->preempts;
      e.parks = sv->parks;
      e.finished = sv->finished;
      e.peak_batch_tokens = sv->peak;
      e.digest = sv->digest;
      e.event_count = sv->ev_n;
      e.clock = sv->clock;
      e.status = sv->status;
      e._pad = 0;
      out[row0[i] + s] = e;
    }
  }
}

}  // namespace

// ==========================================================================
// C ABI
// ==========================================================================
// scheduling header of ssb_simulate: queue counters, per-SM policy table and CTA slot
// counters (sized for up to MAX_SMS SMs), instance order lists
constexpr int MAX_SMS = 1024;
static long long header_bytes(int n_inst) { return align_up(4LL * (16 + (MAX_SMS + 3) / 4 + 4 + 4 * MAX_SMS) + 8LL * n_inst, 256); }

extern "C" int32_t ssb_abi_version(void) { return SSB_ABI_VERSION; }

extern "C" const char* ssb_error_string(int32_t code) {
  switch (code) {
    case SSB_OK: return "ok";
    case SSB_E_INFEASIBLE: return "infeasible request";
    case SSB_E_STALL: return "engine stalled (no schedulable tokens)";
    case SSB_E_CAPACITY: return "device table capacity exceeded";
    case SSB_E_INVARIANT: return "invariant violation";
    case SSB_E_CUDA: return "CUDA error";
    case SSB_E_ARG: return "bad argument";
    default: return "unknown";
  }
}

extern "C" int32_t ssb_struct_sizes(int64_t* out) {
  out[0] = sizeof(ssb_engine_params);
  out[1] = sizeof(ssb_instance);
  out[2] = sizeof(ssb_stats);
  out[3] = sizeof(ssb_event);
  out[4] = sizeof(ssb_summary);
  out[5] = sizeof(ssb_summary_group);
  out[6] = sizeof(ssb_engine_stats);
  return 7;
}

extern "C" int32_t ssb_engine_stats_gather(const ssb_instance* h_inst, const ssb_instance* d_inst, int32_t n_inst,
                                           const void* d_scratch, const ssb_stats* d_stats, ssb_records records,
                                           const int64_t* d_event_count, const int64_t* d_engine_offset,
                                           ssb_engine_stats* d_out, void* stream_) {
  if (n_inst <= 0) return SSB_OK;
  if (!h_inst || !d_inst || !d_scratch || !d_stats || !records.finish || !d_engine_offset || !d_out) return SSB_E_ARG;
  for (int i = 0; i < n_inst; ++i)
    if (h_inst[i].n_servers < 1) return SSB_E_ARG;
  k_engine_stats<<<(unsigned)std::min(n_inst, 4096), 256, 0, (cudaStream_t)stream_>>>(
      d_inst, n_inst, (const unsigned char*)d_scratch, d_stats, records.finish, d_event_count, d_engine_offset, d_out);
  return cudaGetLastError() == cudaSuccess ? SSB_OK : SSB_E_CUDA;
}

extern "C" size_t ssb_prepare(ssb_instance* h, int32_t n_inst) {
  long long off = header_bytes(n_inst);
  for (int i = 0; i < n_inst; ++i) {
    ssb_instance& I = h[i];
    long long N = I.n_requests;
    long long Wc = std::max(1LL, N);
    // heterogeneous prebuilt engines: tables sized for the largest server, one stride for all
    const int n_sets = I.h_servers != nullptr ? std::max(1, I.n_servers) : 1;
    long long Rc = 1;
    for (int s = 0; s < n_sets; ++s) {
      const ssb_engine_params& e = I.h_servers != nullptr ? I.h_servers[s] : I.engine;
      long long r = std::min<long long>(e.pool_blocks, N);
      if (e.max_running > 0) r = std::min<long long>(r, e.max_running);
      Rc = std::max(Rc, r);
    }
    I.wait_cap = (int32_t)Wc;
    I.run_cap = (int32_t)Rc;
    I.scratch_offset = off;
    long long stride = 0;
    for (int s = 0; s < n_sets; ++s)
      stride = std::max(stride, make_layout(Wc, Rc, N, I.n_servers, I.h_servers != nullptr ? I.h_servers[s] : I.engine).total);
    I.server_stride = stride;
    off += stride * (long long)std::max(1, I.n_servers);
    if (I.qps_factor != 1.0) off += align_up(8 * N, 256);  // scaled arrival times
  }
  return (size_t)off;
}

extern "C" int32_t ssb_simulate(const ssb_instance* h_inst, const ssb_instance* d_inst, int32_t n_inst,
                                ssb_trace trace, ssb_records records, ssb_stats* d_stats, void* d_scratch,
                                size_t scratch_bytes, ssb_event* d_events, int64_t event_cap,
                                int64_t* d_event_count, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n_inst <= 0) return SSB_OK;
  if (!h_inst || !d_inst || !d_stats || !d_scratch) return SSB_E_ARG;
  long long hb = header_bytes(n_inst);
  long long need = hb;
  int max_servers = 1;
  std::vector<int> singles, multis;
  for (int i = 0; i < n_inst; ++i) {
    const ssb_instance& I = h_inst[i];
    if (I.n_servers < 1 || I.n_requests < 0 || I.n_requests > 0x7fffffffLL || I.wait_cap < 1 || I.run_cap < 1)
      return SSB_E_ARG;
    if (I.h_servers != nullptr) {  // heterogeneous engines: one policy and block size, pipelined kernel
      if (I.d_servers == nullptr || I.n_servers < 2) return SSB_E_ARG;
      if (I.n_servers > PIPE_MAX_SERVERS)  // the epoch kernel: one policy for all servers
        for (int s = 1; s < I.n_servers; ++s)
          if (I.h_servers[s].policy != I.h_servers[0].policy) return SSB_E_ARG;
      if (I.server_stride < inst_layout(I).total) return SSB_E_ARG;  // not prepared
    }
    const int n_sets = I.h_servers != nullptr ? I.n_servers : 1;
    for (int s = 0; s < n_sets; ++s) {
      const ssb_engine_params& e = I.h_servers != nullptr ? I.h_servers[s] : I.engine;
      if (e.block_size < 1 || ((long long)e.max_context + e.block_size) * e.block_size >= (1LL << 32))
        return SSB_E_ARG;  // blocks(): multiply-shift division exact for token counts < 2^32 / block_size
      if (e.policy == SSB_POLICY_LARRY && e.max_context >= (1 << 22))
        return SSB_E_ARG;  // larry_score: queue_len * pending < 2^31 * 2^22 is exact in binary64
      if (e.policy == SSB_POLICY_TRAIL_PLUS &&
          std::min<long long>(e.max_context, (long long)e.pool_blocks * e.block_size) >= (1LL << 20))
        return SSB_E_ARG;  // remaining-output buckets: 3 tree levels (2^20 buckets) at most
    }
    Layout L = inst_layout(I);
    need = std::max(need, scaled_arrivals_offset(I, L) + (I.qps_factor != 1.0 ? 8 * I.n_requests : 0));
    if (I.n_servers == 1) singles.push_back(i); else { multis.push_back(i); max_servers = std::max(max_servers, I.n_servers); }
  }
  if ((long long)scratch_bytes < need) return SSB_E_ARG;
  if (max_servers > 4096) return SSB_E_ARG;
  // Singles: one persistent kernel, SMs partitioned by policy (see k_engines).
  // Multis: one CTA per instance.
  std::vector<int> sg[8];
  const bool one_queue = getenv("SSB_ONE_QUEUE") != nullptr;  // experiments: no per-policy SM partition
  // Each policy's instances form two classes by KV pool size: pools of more than 2^16 tokens
  // run much larger batches (the R > 32 table paths) than small ones, so giving the two their
  // own SMs keeps each SM's executed code smaller (C4: 146 -> 142 ms, SSB_SPLIT_POOL=<blocks>
  // overrides the threshold; 0 = no split).
  long long split_tokens = 1LL << 16;
  if (const char* e = getenv("SSB_SPLIT_POOL")) split_tokens = (long long)atoi(e) * 16;
  for (int i : singles) {
    const long long pool_tokens = (long long)h_inst[i].engine.pool_blocks * h_inst[i].engine.block_size;
    const int cls = split_tokens > 0 && pool_tokens > split_tokens ? 1 : 0;
    sg[one_queue ? 0 : 2 * (h_inst[i].engine.policy & 3) + cls].push_back(i);
  }
  double gwork[8] = {0, 0, 0, 0, 0, 0, 0, 0}, total_work = 0;
  for (int p = 0; p < 8; ++p) {
    std::stable_sort(sg[p].begin(), sg[p].end(),
                     [&](int a, int b) { return h_inst[a].est_cost > h_inst[b].est_cost; });
    for (int i : sg[p]) gwork[p] += (double)std::max(1, h_inst[i].est_cost);
    total_work += gwork[p];
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int sms_tab = std::min(sms, MAX_SMS);
  // header (ints): [queue counters x4, pad x12][sm policy table (bytes)][per-SM CTA slot
  // counters][singles by policy][multis]
  const int smtab_ints = (MAX_SMS + 3) / 4 + 4;
  // + per-SM CTA slot counters, drained-warp counters, deal claim counters, rank within its home queue
  const int hdr0 = 16 + smtab_ints + 4 * MAX_SMS;
  std::vector<int> hdr(hdr0 + n_inst, 0);
  // The longest trail_plus instances (the critical path of a sweep) get SMs of their own
  // with one CTA (4 warps): trail_plus is instruction-fetch bound, so 4 warps keep the
  // SM's throughput while each instance runs faster than among 8 (profiles/).
  // Off by default: it paid (227 -> 220 ms on C4) while trail_plus was instruction-fetch bound
  // at 8 warps/SM; after the code-size work 8 warps win (166 vs 171-175 ms, tools/probe_heavy.py).
  int heavy_sms = 0;
  if (const char* e = getenv("SSB_HEAVY_SMS")) heavy_sms = std::max(0, atoi(e));  // experiments
  heavy_sms = std::min<int>(heavy_sms, (int)sg[2 * SSB_POLICY_TRAIL_PLUS].size() / ENGINE_WARPS_PER_CTA);
  heavy_sms = std::min(heavy_sms, sms_tab / 2);
  const int n_heavy = heavy_sms * ENGINE_WARPS_PER_CTA;
  std::vector<int> heavy(sg[2 * SSB_POLICY_TRAIL_PLUS].begin(), sg[2 * SSB_POLICY_TRAIL_PLUS].begin() + n_heavy);
  sg[2 * SSB_POLICY_TRAIL_PLUS].erase(sg[2 * SSB_POLICY_TRAIL_PLUS].begin(), sg[2 * SSB_POLICY_TRAIL_PLUS].begin() + n_heavy);
  total_work = 0;
  for (int p = 0; p < 8; ++p) {
    gwork[p] = 0;
    for (int i : sg[p]) gwork[p] += (double)std::max(1, h_inst[i].est_cost);
    total_work += gwork[p];
  }
  const int sms_rest = sms_tab - heavy_sms;
  unsigned char* smpol = (unsigned char*)(hdr.data() + 16);
  for (int k = 0; k < heavy_sms; ++k) smpol[sms_rest + k] = (unsigned char)Q_HEAVY;
  {  // SMs per policy in proportion to estimated work (largest remainder), >= 1 if it has work
    int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, given = 0;
    double rem[8];
    for (int p = 0; p < 8; ++p) {
      const double want = total_work > 0 ? sms_rest * gwork[p] / total_work : 0.0;
      cnt[p] = sg[p].empty() ? 0 : std::max(1, (int)want);
      rem[p] = want - cnt[p];
      given += cnt[p];
    }
    while (given > sms_rest) {
      int pm = 0;
      for (int p = 1; p < 8; ++p) if (cnt[p] > cnt[pm]) pm = p;
      cnt[pm]--; given--;
    }
    while (given < sms_rest) {
      int pm = -1;
      for (int p = 0; p < 8; ++p) if (!sg[p].empty() && (pm < 0 || rem[p] > rem[pm])) pm = p;
      if (pm < 0) break;
      cnt[pm]++; rem[pm] -= 1.0; given++;
    }
    int s0 = 0;
    for (int p = 0; p < 8; ++p) for (int k = 0; k < cnt[p] && s0 < sms_rest; ++k) smpol[s0++] = (unsigned char)p;
    for (; s0 < sms_rest; ++s0) smpol[s0] = 0;
  }
  EngineQueues qs;
  int o = hdr0;
  for (int p = 0; p < 8; ++p) { qs.off[p] = o - hdr0; qs.n[p] = (int)sg[p].size(); for (int i : sg[p]) hdr[o++] = i; }
  qs.off[Q_HEAVY] = o - hdr0;
  qs.n[Q_HEAVY] = (int)heavy.size();
  {  // deal: each SM's rank among its home queue's SMs; the queue's FIFO starts after the dealt head
    int* sm_rank = hdr.data() + 16 + smtab_ints + 3 * MAX_SMS;
    for (int p = 0; p < NQ; ++p) qs.nsm[p] = 0;
    for (int m = 0; m < MAX_SMS; ++m) sm_rank[m] = -1;
    for (int m = 0; m < sms_tab; ++m)
      if (smpol[m] < 8) sm_rank[m] = qs.nsm[smpol[m]]++;
    for (int p = 0; p < 8; ++p) hdr[p] = std::min(DEAL_ROUNDS * qs.nsm[p], qs.n[p]);
  }
  for (int i : heavy) hdr[o++] = i;
  const int off_multi = o;
  for (int i : multis) hdr[o++] = i;
  unsigned char* scratch = (unsigned char*)d_scratch;
  if (cudaMemcpyAsync(scratch, hdr.data(), sizeof(int) * hdr.size(), cudaMemcpyHostToDevice, stream) != cudaSuccess)
    return SSB_E_CUDA;
  const int* d_hdr = (const int*)scratch;
  bool any_scaled = false;
  for (int i = 0; i < n_inst; ++i) any_scaled |= h_inst[i].qps_factor != 1.0;
  if (any_scaled) {
    k_scale_arrivals<<<(unsigned)std::min(n_inst, 8 * sms), 256, 0, stream>>>(d_inst, n_inst, trace, scratch);
    if (cudaGetLastError() != cudaSuccess) return SSB_E_CUDA;
  }
  bool multis_done = multis.empty();
  if (!multis_done && max_servers <= PIPE_MAX_SERVERS && getenv("SSB_CLUSTER_CLASSIC") == nullptr) {
    // pipelined: one cluster of G CTAs x 8 warps per instance, a routing warp + one warp per
    // replica (G = 9 for 64 replicas: a non-portable cluster size)
    // engine warps per CTA: 4 when the cluster still fits 16 CTAs (small clusters, C2: two engine
    // SMs instead of one), else 8 (C5's 64 replicas: 9 CTAs)
    int epc = 1 + (max_servers + 3) / 4 <= PIPE_MAX_CTAS ? 4 : PIPE_WARPS;
    if (const char* e = getenv("SSB_PIPE_EPC")) epc = std::min(PIPE_WARPS, std::max(1, atoi(e)));  // experiments
    if (1 + (max_servers + epc - 1) / epc > PIPE_MAX_CTAS) epc = PIPE_WARPS;
    const int G = 1 + (max_servers + epc - 1) / epc;
    // watermark publish period (<= 32: the route log is one lane per route): every route for
    // small clusters (C2, 8 replicas: the engines see each arrival at once; 209 -> 200 ms on
    // C2/sal), every 8 routes for large ones (C5, 64 replicas: 64 engines waking per publish
    // cost more than they gain, 99 vs 104 ms)
    int publish_every = max_servers <= 16 ? 1 : 8;
    if (const char* e = getenv("SSB_PIPE_PUBLISH")) publish_every = std::min(32, std::max(1, atoi(e)));  // experiments
    const size_t smc = align_up(pipe_array_bytes(max_servers), 16) + sizeof(int) * SM_COLS * RS * PIPE_WARPS;
    cudaFuncSetAttribute(k_cluster_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    if (G > 8) cudaFuncSetAttribute(k_cluster_pipe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(multis.size() * G));
    lc.blockDim = dim3(32 * PIPE_WARPS);
    lc.dynamicSmemBytes = smc;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (getenv("SSB_DEBUG_CLUSTERS")) {  // diagnostics: how many of these clusters fit the GPU at once
      int nc = -1;
      cudaOccupancyMaxActiveClusters(&nc, k_cluster_pipe, &lc);
      fprintf(stderr, "k_cluster_pipe: %zu clusters of %d CTAs x %d threads, %zu B shared each; max active clusters %d\n",
              multis.size(), G, 32 * PIPE_WARPS, smc, nc);
    }
    if (cudaLaunchKernelEx(&lc, k_cluster_pipe, (const ssb_instance*)d_inst, (const int*)(d_hdr + off_multi), trace,
                           records, d_stats, scratch, d_events, (long long)event_cap, (int64_t*)d_event_count,
                           publish_every, epc) == cudaSuccess)
      multis_done = true;
    else
      cudaGetLastError();  // e.g. the cluster size does not fit: the classic kernel below
  }
  if (!multis_done) {
    // one cluster of G CTAs x nw warps per instance: enough warps for one replica each (<= 64)
    const int nw = std::min(CLUSTER_MAX_WARPS, max_servers);
    const int G = std::min(CLUSTER_MAX_CTAS, (max_servers + nw - 1) / nw);
    const int per_warp = (max_servers + G * nw - 1) / (G * nw);  // replicas per warp
    const int tabs = per_warp * nw <= CLUSTER_SMEM_SERVERS ? 1 : 0;
    size_t smc = sizeof(long long) * 6 * ((max_servers + 1) & ~1);
    if (tabs) smc += sizeof(int) * SM_COLS * RS * per_warp * nw;
    if (smc > 48 * 1024) cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(multis.size() * G));
    lc.blockDim = dim3(32 * nw);
    lc.dynamicSmemBytes = smc;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, k_cluster, (const ssb_instance*)d_inst, (const int*)(d_hdr + off_multi), trace, records,
                           d_stats, scratch, d_events, (long long)event_cap, (int64_t*)d_event_count, tabs) != cudaSuccess)
      return SSB_E_CUDA;
    if (cudaGetLastError() != cudaSuccess) return SSB_E_CUDA;
  }
  if (!singles.empty()) {
    // latency mode when every instance can have an SM to itself (see k_engines<WIDE>)
    const bool wide = (int)singles.size() <= sms && getenv("SSB_NO_LATENCY_MODE") == nullptr;
    auto kern = wide ? k_engines<true> : k_engines<false>;
    int occ = 1;
    const size_t sm = sizeof(int) * SM_COLS * RS * ENGINE_WARPS_PER_CTA;
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * ENGINE_WARPS_PER_CTA, sm);
    if (const char* cap = getenv("SSB_CTAS_PER_SM")) occ = std::min(occ, std::max(1, atoi(cap)));  // experiments
    const int grid = sms * std::max(1, occ);
    kern<<<grid, 32 * ENGINE_WARPS_PER_CTA, sm, stream>>>(
        d_inst, d_hdr + hdr0, qs, (int*)scratch, (const unsigned char*)(d_hdr + 16), sms_tab,
        (int*)scratch + 16 + smtab_ints, (int*)scratch + 16 + smtab_ints + MAX_SMS,
        (int*)scratch + 16 + smtab_ints + 2 * MAX_SMS, d_hdr + 16 + smtab_ints + 3 * MAX_SMS, trace, records, d_stats, scratch,
        d_events, event_cap, d_event_count);
    if (cudaGetLastError() != cudaSuccess) return SSB_E_CUDA;
  }
  return SSB_OK;
}

#ifdef SSB_PIPE_TIMELINE
extern "C" int32_t ssb_debug_sync_timeline(unsigned long long* out, int32_t n_syncs) {
  if (n_syncs > SYNC_TL_MAX) n_syncs = SYNC_TL_MAX;
  return cudaMemcpyFromSymbol(out, g_sync_tl, sizeof(unsigned long long) * SYNC_TL_W * (size_t)n_syncs) == cudaSuccess
             ? n_syncs : -1;
}
#endif
#ifdef SSB_TIMELINE
extern "C" int32_t ssb_debug_timeline(unsigned long long* out, int32_t n) {
  if (n > TIMELINE_MAX) n = TIMELINE_MAX;
  return cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * 3 * (size_t)n) == cudaSuccess ? n : -1;
}
#endif
