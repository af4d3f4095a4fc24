"""B200-native batched serving-scheduler simulator.

Drop-in for the simulation path of the reference package ``servesim``
(arXiv 2410.17840): the same registries (policies fcfs / nopreempt /
trail_plus / larry; balancers rr / random / p2c / sal), settings and entry
points (run_cluster, Engine.run, summarize, capacity_sweep), executed by
hand-written sm_100a kernels behind the C ABI in include/ssb.h.
"""

from .balancers import (BALANCER_NAMES, BetaEstimator, LoadBalancer, PowerOfTwoBalancer, RandomBalancer,
                        RoundRobinBalancer, ServerAwareBalancer, ServerStats, make_balancer, sal_load)
from .cluster import Engine, JobResult, StallError, build_engine, run_cluster, simulate_jobs
from .metrics import (MetricsRecord, RecordsSoA, Summary, SummaryExtras, capacity_sweep, percentile, summarize,
                      summarize_many, write_records_csv, write_summary_csv, write_summary_json)
from .policies import (POLICY_NAMES, EngineLimits, FcfsPolicy, InfeasibleRequestError, LoadAdaptivePolicy,
                       NoPreemptPolicy, SchedulerPolicy, ShortestRemainingPolicy, larry_score, make_policy)
from .settings import (DEFAULT_BLOCK_SIZE, PROFILES, BalancerSettings, ClusterSettings, CostParams, EngineSettings,
                       KvBlockPool, ModelProfile, blocks_needed, default_params, pool_blocks_for)
from .workload import LengthDist, SynthSpec, Trace, TraceEntry, scale_qps, synthesize

__version__ = "0.1.0"
