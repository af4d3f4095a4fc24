/*
 * ssb.h — C ABI of the B200 batched serving-scheduler simulator (libssb.so).
 *
 * This is the drop-in boundary for the reference's simulation path
 * (servesim, /root/reference/pkg/src/servesim). One call simulates a batch of
 * independent *instances*; an instance is exactly one reference
 * `run_cluster(settings, trace)` call (cluster.py:65-174), and with
 * n_servers == 1 it is also exactly one `Engine(...).run(trace)` call
 * (engine.py:236-265, equivalence pinned by tests/test_cluster.py:39-60).
 *
 * Plugin surface mirrored:
 *   - scheduler registry  POLICY_NAMES   policies.py:279 / make_policy   policies.py:282
 *   - balancer registry   BALANCER_NAMES balancers.py:219 / make_balancer balancers.py:222
 *   - EngineSettings / BalancerSettings / ClusterSettings fields   config.py:26-56
 * Custom Python SchedulerPolicy/LoadBalancer subclasses have no ABI: the host
 * shim rejects them (there is no CPU fallback).
 *
 * Conventions: every pointer handed to ssb_simulate/ssb_summarize is a DEVICE
 * pointer owned by the caller; the library never allocates device memory on
 * its own. Calls are asynchronous on the given stream. All times are
 * IEEE-754 binary64 seconds; all token counts are exact integers.
 */
#ifndef SSB_H_
#define SSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_ABI_VERSION 3

/* scheduler registry keys, policies.py:279 ("fcfs","nopreempt","trail_plus","larry") */
enum { SSB_POLICY_FCFS = 0, SSB_POLICY_NOPREEMPT = 1, SSB_POLICY_TRAIL_PLUS = 2, SSB_POLICY_LARRY = 3 };
/* balancer registry keys, balancers.py:219 ("rr","random","p2c","sal") */
enum { SSB_BAL_RR = 0, SSB_BAL_RANDOM = 1, SSB_BAL_P2C = 2, SSB_BAL_SAL = 3 };

/* status codes (per instance and per call) */
enum {
  SSB_OK = 0,
  SSB_E_INFEASIBLE = 1,  /* policies.py:56-68,119-131 InfeasibleRequestError (host pre-checks) */
  SSB_E_STALL = 2,       /* engine.py:209-214 StallError                                      */
  SSB_E_CAPACITY = 3,    /* a device table (waiting ring / running table / route list) is full */
  SSB_E_INVARIANT = 4,   /* over-admission or unfinished requests (engine.py:288-292, cluster.py:159-161) */
  SSB_E_CUDA = 5,        /* CUDA launch/runtime error                                         */
  SSB_E_ARG = 6          /* bad arguments                                                      */
};

/* event codes of the optional event log / decision digest (engine.py:165,273-274) */
enum { SSB_EV_ENQUEUE = 0, SSB_EV_DISPATCH = 1, SSB_EV_PREEMPT = 2, SSB_EV_PARK = 3,
       SSB_EV_FIRST_TOKEN = 4, SSB_EV_FINISH = 5 };

/* Engine parameters = EngineSettings (config.py:26-39) after build_engine()
 * resolved the pool size, cost parameters and context window (cluster.py:28-47). */
typedef struct {
  int32_t policy;               /* SSB_POLICY_*                                   */
  int32_t max_output;           /* nopreempt max_output   (policies.py:111)       */
  double alpha;                 /* larry alpha            (policies.py:239)       */
  double c;                     /* trail_plus c           (policies.py:163)       */
  int32_t block_size;           /* KvBlockPool.block_size (kvmem.py:82)           */
  int32_t pool_blocks;          /* KvBlockPool.total_blocks                       */
  int32_t max_tokens_per_batch; /* EngineLimits           (policies.py:22-36)     */
  int32_t max_running;          /* -1 = None (unlimited)                          */
  int32_t max_context;          /* ModelProfile.max_context (kvmem.py:35-48)      */
  int32_t _pad0;
  double mem_base_s;            /* CostParams (costmodel.py:22-27)                */
  double mem_per_kv_token_s;
  double compute_per_token_s;
  double overhead_s;
} ssb_engine_params;

/* One simulation instance = one run_cluster(settings, trace) call. */
typedef struct {
  ssb_engine_params engine;
  int32_t n_servers;            /* ClusterSettings.n_servers (config.py:52)       */
  int32_t balancer;             /* SSB_BAL_*                                      */
  double poll_interval_s;       /* BalancerSettings (config.py:42-47)             */
  double beta_prior;
  double beta_fixed;            /* NaN = None (estimate beta)                     */
  /* numpy PCG64 state of default_rng(ClusterSettings.seed) (cluster.py:94),
   * taken on the host from np.random.PCG64(seed).state                          */
  uint64_t pcg_state_hi, pcg_state_lo, pcg_inc_hi, pcg_inc_lo;
  double qps_factor;            /* scale_qps divisor (workload.py:187-194); 1.0 = none */
  int64_t trace_offset;         /* first request of this instance in the trace SoA  */
  int64_t record_offset;        /* first request of this instance in the records SoA */
  int64_t n_requests;
  /* filled by ssb_prepare(): device capacities and scratch offset               */
  int64_t scratch_offset;       /* bytes into the scratch buffer                    */
  int32_t wait_cap;             /* waiting-ring capacity per server                 */
  int32_t run_cap;              /* running-table capacity per server                */
  int32_t est_cost;             /* scheduling hint (larger = start earlier)         */
  int32_t flags;                /* SSB_FLAG_*                                       */
  /* SAL's token cap: settings.engine.max_tokens_per_batch as run_cluster hands it to
   * make_balancer (cluster.py:96-104), independent of the engines' own batching cap
   * (engine.max_tokens_per_batch above), which prebuilt engines may set differently */
  int32_t route_cap;
  int32_t _pad1;
  /* Heterogeneous prebuilt engines (run_cluster(settings, trace, engines=[...]) with engines
   * that differ, cluster.py:66-79): n_servers parameter sets, server s batching, allocating
   * and costing with its own; NULL = every server uses `engine`. h_servers is the host array
   * (read by ssb_prepare / ssb_simulate's planning), d_servers a device copy of it (read by
   * the kernels), policy included (each engine warp of the pipelined kernel runs its own
   * server's policy); beyond 120 servers (the epoch kernel, several servers per warp) the sets
   * must share the policy, else ssb_simulate returns SSB_E_ARG. */
  const ssb_engine_params* h_servers;
  const ssb_engine_params* d_servers;
  int64_t server_stride;        /* filled by ssb_prepare(): scratch bytes per server   */
} ssb_instance;

/* Running tables live in shared memory with SSB_SMEM_RUN_CAP entries per
 * engine unless SSB_FLAG_GLOBAL_TABLES is set (then global, sized run_cap).
 * An instance that outgrows the shared table ends with SSB_E_CAPACITY and is
 * simply re-run with the flag (the host shim does this automatically). */
#ifndef SSB_SMEM_RUN_CAP
#define SSB_SMEM_RUN_CAP 256
#endif
#define SSB_FLAG_GLOBAL_TABLES 1

/* Trace SoA, TraceEntry (workload.py:42-56); arrivals sorted per instance. */
typedef struct {
  const double* arrival;
  const int32_t* prompt;
  const int32_t* output;
} ssb_trace;

/* Per-request results, MetricsRecord (metrics.py:20-31) + first_dispatch
 * (time of the first `dispatch` event: queueing delay, not in the reference). */
typedef struct {
  double* first_token;
  double* finish;
  double* first_dispatch;
  int32_t* preempt_count;
  int32_t* server;
} ssb_records;

/* Per-instance counters (sums over the instance's engines). */
typedef struct {
  int64_t iterations;      /* Σ Engine.iterations (engine.py:226)                        */
  int64_t request_steps;   /* Σ len(decode_ids)+len(prefill_chunks) per step (engine.py:300-323) */
  int64_t batch_tokens;    /* Σ BatchPlan.total_tokens                                    */
  int64_t dispatches;
  int64_t preempts;        /* policy preempts + grow evictions ("preempt" events)         */
  int64_t parks;
  int64_t finished;
  int64_t peak_batch_tokens; /* max Engine.peak_batch_tokens over engines                 */
  uint64_t digest;         /* FNV-1a fold of per-engine event digests  */
  int32_t status;          /* SSB_OK or SSB_E_*                                           */
  int32_t _pad;
  int64_t device_cycles;   /* SM clock cycles the instance took (scheduling feedback: feed
                              back as ssb_instance.est_cost to order the next launch)     */
} ssb_stats;

/* Per-engine counters (one row per server of an instance, server order): the
 * reference keeps iterations / peak_batch_tokens on each Engine object
 * (engine.py:165-166,225-226) and its criterion-8 audit reads them per engine
 * (tests/test_acceptance.py:371-382). Filled by ssb_engine_stats_gather after a
 * simulation from the per-server state left in the scratch buffer. */
typedef struct {
  int64_t iterations;
  int64_t request_steps;
  int64_t batch_tokens;
  int64_t dispatches;
  int64_t preempts;
  int64_t parks;
  int64_t finished;
  int64_t peak_batch_tokens;
  uint64_t digest;         /* FNV-1a of this engine's event log (before the instance fold) */
  int64_t event_count;     /* events this engine produced (> its ring slice = truncated log) */
  double clock;            /* Engine.clock at the end of the run                            */
  int32_t status;
  int32_t _pad;
} ssb_engine_stats;

/* Optional event log (engine.py:267-274) */
typedef struct {
  double time;
  int32_t request_id;
  int16_t server;
  int16_t code;            /* SSB_EV_*   */
} ssb_event;

/* Summary (metrics.py:57-99) + north-star extras (TPOT, queueing delay). */
typedef struct {
  int64_t n_requests;
  double ttft_p50, ttft_p95, ttft_p99;
  double norm_ttft_p50, norm_ttft_p95;
  double gen_time_p50, gen_time_p95;
  double preemption_rate;
  double throughput_rps;
  /* extras: TPOT = (finish-first)/(output-1) over output>1 requests, queue = first_dispatch-arrival */
  int64_t n_tpot;
  double tpot_p50, tpot_p95, tpot_p99;
  double queue_p50, queue_p95, queue_p99;
  int64_t n_preempted;
  double max_finish, min_arrival;
} ssb_summary;

/* Library/ABI identification. ssb_struct_sizes writes sizeof() of
 * ssb_engine_params, ssb_instance, ssb_stats, ssb_event, ssb_summary,
 * ssb_summary_group, ssb_engine_stats (in that order) to out[0..6]; returns 7. */
int32_t ssb_abi_version(void);
const char* ssb_error_string(int32_t code);
int32_t ssb_struct_sizes(int64_t* out);

/* Host-side planning: fills scratch_offset / wait_cap / run_cap of every
 * instance (host array) and returns the scratch bytes ssb_simulate needs. */
size_t ssb_prepare(ssb_instance* h_inst, int32_t n_inst);

/* Simulate n_inst instances. h_inst: the prepared host descriptors (launch
 * planning: instances with n_servers == 1 run one per warp in a persistent
 * kernel, longest est_cost first; a multi-server instance runs on one
 * thread-block cluster: a routing warp + one engine warp per replica up to 120
 * replicas (k_cluster_pipe), the epoch kernel k_cluster beyond).
 * d_inst: device copy of the same array. d_scratch: ssb_prepare() bytes.
 * d_events (nullable): per-instance event ring of event_cap entries each,
 * instance i writes [i*event_cap, (i+1)*event_cap); d_event_count (nullable
 * iff d_events is) receives each instance's total event count.
 * Returns SSB_OK once the work is enqueued; per-instance status is in d_stats. */
int32_t ssb_simulate(const ssb_instance* h_inst, const ssb_instance* d_inst, int32_t n_inst,
                     ssb_trace trace, ssb_records records, ssb_stats* d_stats,
                     void* d_scratch, size_t scratch_bytes,
                     ssb_event* d_events, int64_t event_cap, int64_t* d_event_count,
                     void* stream /* cudaStream_t */);

/* After ssb_simulate (same stream, same scratch, stats, records and event counts):
 * per-engine counters of every instance. Row (i, s) = instance i's server s is
 * written to d_out[d_engine_offset[i] + s] (d_engine_offset: device array of n_inst
 * row offsets, typically the exclusive prefix sum of n_servers). A cluster's
 * servers keep their state in the scratch buffer; a single-server instance's row
 * is its ssb_stats (digest unfolded), its clock the time of its last step (= its
 * latest finish: the last step finishes the last request, engine.py:256-265) and
 * its event count d_event_count[i] (NULL when no events were recorded: 0).
 * Replaces reading engine.iterations / engine.peak_batch_tokens / engine.clock off
 * the engines passed to run_cluster(..., engines=...) (cluster.py:66-79). */
int32_t ssb_engine_stats_gather(const ssb_instance* h_inst, const ssb_instance* d_inst, int32_t n_inst,
                                const void* d_scratch, const ssb_stats* d_stats, ssb_records records,
                                const int64_t* d_event_count, const int64_t* d_engine_offset,
                                ssb_engine_stats* d_out, void* stream);

/* One summary group = one summarize(records) call (metrics.py:80-99) over
 * records [record_offset, record_offset+n) whose trace entries are
 * [trace_offset, trace_offset+n), arrivals divided by qps_factor.
 * rank[0..2]: nearest ranks ceil(p/100*n) for p = 50,95,99 (metrics.py:53),
 * computed on the host in Python float arithmetic exactly as the reference;
 * rank[3..5]: the same for the TPOT sample size n_tpot (0 if unknown yet:
 * ssb_summarize then derives it with the integer identity (p*n+99)/100,
 * which equals the float form for n <= 1e7). */
typedef struct {
  int64_t record_offset;
  int64_t trace_offset;
  int64_t n;
  double qps_factor;
  int64_t rank[6];
} ssb_summary_group;

size_t ssb_summary_work_bytes(const ssb_summary_group* h_groups, int32_t n_groups);
/* h_groups: host copy (launch planning); d_groups: device copy. */
int32_t ssb_summarize(ssb_trace trace, ssb_records records,
                      const ssb_summary_group* h_groups, const ssb_summary_group* d_groups,
                      int32_t n_groups, ssb_summary* d_summary,
                      void* d_work, size_t work_bytes, void* stream);

/* Pooled percentiles (one metric set over the union of many groups, and across
 * GPUs): pass `pass` (0..7) of an MSD radix select with 8-bit digits on the
 * order-preserving 64-bit image of each metric value. For each of the 13 rank
 * slots (TTFT p50/95/99, nTTFT p50/95, TGT p50/95, TPOT p50/95/99, queueing
 * delay p50/95/99; same per-record metrics as ssb_summarize) with
 * d_active[s] != 0, counts the records of ALL groups whose key matches
 * d_prefix[s] in the bits above the pass's digit into d_hist[s*256 + digit]
 * (zeroed by the call). Pass 0 also writes d_counts = {n, n_tpot,
 * n_preempted}. d_work: >= 8*(n_groups+1) bytes. The host sums the
 * histograms over ranks (one all-gather per pass) and extends the prefixes
 * (paper_2410_17840_b200/pooled.py). Replaces summarize() (metrics.py:80-99)
 * over concatenated record lists, without moving records between GPUs. */
int32_t ssb_pool_hist(ssb_trace trace, ssb_records records,
                      const ssb_summary_group* h_groups, const ssb_summary_group* d_groups,
                      int32_t n_groups, const uint64_t* d_prefix, const int32_t* d_active,
                      int32_t pass, uint32_t* d_hist, uint64_t* d_counts,
                      void* d_work, size_t work_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSB_H_ */
