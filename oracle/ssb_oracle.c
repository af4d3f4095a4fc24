/*
 * ssb_oracle.c — CPU ORACLE for the servesim simulation path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is a literal, serial restatement of the
 * reference algorithm in /root/reference/pkg/src/servesim (engine.py,
 * policies.py, kvmem.py, costmodel.py, balancers.py, cluster.py). It is used
 * by tests/ (as the parity checker), by __graft_entry__.smoke() and by
 * bench.py's cpu_baseline / --impl reference leg. The product path
 * (paper_2410_17840_b200) never links, loads or calls it.
 *
 * Parity of this oracle is PINNED against the reference itself: the golden
 * fixtures in tests/golden/ were produced by importing the Python reference
 * (tests/golden/make_golden.py) and tests/test_oracle_golden.py checks this
 * file against them (records, event-log digests, iteration / request-step /
 * batch-token counts).
 *
 * Data structures deliberately mirror the reference's (a deque for the
 * waiting queue, an insertion-ordered running list, a per-request token map
 * for the pool, a binary heap for run_cluster's event loop, full re-sorts in
 * the trail_plus / larry policies), so that each function reads against the
 * file:line it restates. Floating point: compile with -ffp-contract=off so
 * every expression rounds exactly like CPython's binary64 arithmetic.
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/ssb.h"

#define ST_WAITING 0
#define ST_PREFILLING 1
#define ST_DECODING 2
#define ST_FINISHED 3

#define FNV_OFF 0xcbf29ce484222325ULL
#define FNV_PRIME 0x100000001b3ULL

/* engine.py:55-116 Request */
typedef struct Req {
  int64_t id;
  double arrival;
  int32_t prompt, output;
  int32_t state;
  int32_t prefill_done, generated;
  double enqueue_time, first_token, finish, first_dispatch;
  int32_t preempt_count;
  int64_t dispatch_seq; /* -1 = None */
  int64_t kv_tokens;    /* KvBlockPool._tokens[id] (kvmem.py:90) */
  int32_t has_alloc;
  int32_t server;
} Req;

static inline int64_t prefill_target(const Req* r) { return (int64_t)r->prompt + r->generated; } /* engine.py:85-87 */
static inline int64_t pending_prefill(const Req* r) { return prefill_target(r) - r->prefill_done; } /* :90-91 */
static inline int64_t context_len(const Req* r) { /* engine.py:110-116 */
  if (r->state == ST_DECODING) return (int64_t)r->prompt + r->generated;
  if (r->state == ST_PREFILLING) return r->prefill_done;
  return 0;
}

/* kvmem.py:15-21 blocks_needed = -(-tokens // block_size) */
static inline int64_t blocks_needed(int64_t tokens, int64_t bs) { return (tokens + bs - 1) / bs; }

/* ---- collections.deque[Request] ------------------------------------------ */
typedef struct {
  Req** buf;
  int64_t cap, head, len;
} Deque;

static int dq_init(Deque* d, int64_t cap) {
  d->cap = cap < 4 ? 4 : cap;
  d->buf = (Req**)malloc(sizeof(Req*) * d->cap);
  d->head = d->len = 0;
  return d->buf != NULL;
}
static inline Req* dq_get(const Deque* d, int64_t i) { return d->buf[(d->head + i) % d->cap]; }
static void dq_grow(Deque* d) {
  if (d->len < d->cap) return;
  int64_t nc = d->cap * 2;
  Req** nb = (Req**)malloc(sizeof(Req*) * nc);
  for (int64_t i = 0; i < d->len; i++) nb[i] = dq_get(d, i);
  free(d->buf);
  d->buf = nb; d->cap = nc; d->head = 0;
}
static void dq_push_back(Deque* d, Req* r) { dq_grow(d); d->buf[(d->head + d->len) % d->cap] = r; d->len++; }
static void dq_push_front(Deque* d, Req* r) { dq_grow(d); d->head = (d->head + d->cap - 1) % d->cap; d->buf[d->head] = r; d->len++; }
static Req* dq_pop_front(Deque* d) { Req* r = d->buf[d->head]; d->head = (d->head + 1) % d->cap; d->len--; return r; }
static void dq_remove(Deque* d, Req* r) { /* deque.remove: first occurrence, O(len) */
  int64_t i = 0;
  while (i < d->len && dq_get(d, i) != r) i++;
  for (; i + 1 < d->len; i++) d->buf[(d->head + i) % d->cap] = d->buf[(d->head + i + 1) % d->cap];
  d->len--;
}

/* ---- trail_plus waiting set, fast mode (C3-size backlogs only; see select_trail_fast) ----
 * The literal select_trail re-sorts the whole waiting list and visits every candidate on every
 * step, and dispatch removes from the deque by a linear search: O(W log W + W*R) per step, which
 * does not finish C3's 1M-request backlog. Fast mode keeps the waiting set as one list per
 * remaining-output value (ascending id == (arrival, id) order: the trace is sorted) plus a
 * segment tree of each list's minimum block need, and visits only admissible candidates.
 * It makes the same decisions in the same order (tests/test_oracle_golden.py checks it against
 * the literal path); it is enabled only for single-engine trail_plus runs by
 * ssb_oracle_set_trail_fast(1) (tools/make_c3_golden.py). */
typedef struct {
  int64_t nb, size;    /* buckets (remaining 0..nb-1), tree leaves (power of two) */
  int32_t *head, *tail, *next, *prev;
  int32_t* tree;       /* [2*size]: leaf size+b = min need in bucket b (INT32_MAX empty) */
} TrailFast;
static int g_trail_fast = 0;
void ssb_oracle_set_trail_fast(int32_t on) { g_trail_fast = on != 0; }

/* ---- engine ------------------------------------------------------------- */
typedef struct {
  ssb_engine_params p;
  int64_t free_blocks;        /* KvBlockPool.free_blocks */
  double clock;
  Deque waiting;              /* engine.py:162 */
  Req** running;              /* engine.py:163 dict (insertion order) */
  int64_t nrun, runcap;
  int64_t iterations, peak, next_seq;
  /* instrumentation: request-steps / batch tokens (wrap of _form_batch), events */
  int64_t rsteps, btokens, dispatches, preempts, parks, finished;
  uint64_t digest;
  int server;
  ssb_event* ev;
  int64_t ev_cap;
  int64_t* ev_n;
  int status;
  /* per-step scratch */
  Req** tmp;
  Req** tmp2;
  Req** dispatch;
  Req** preempt;
  int64_t ndisp, npre;
  Req** plan_dec;
  Req** plan_pf;
  int64_t* plan_chunk;
  int64_t nplan_dec, nplan_pf;
  Req** finished_now;
  int64_t nfinished_now;
  TrailFast* tf;      /* fast-mode trail_plus waiting set (NULL: the literal deque) */
  Req* reqs;          /* request array (fast mode indexes it by id) */
} Eng;

static void eng_log(Eng* e, int code, const Req* r) { /* engine.py:273-274 */
  uint64_t w[3] = {(uint64_t)code, (uint64_t)r->id, 0};
  memcpy(&w[2], &e->clock, 8);
  for (int k = 0; k < 3; k++) { e->digest ^= w[k]; e->digest *= FNV_PRIME; }
  if (e->ev) {
    int64_t n = *e->ev_n;
    if (n < e->ev_cap) {
      e->ev[n].time = e->clock;
      e->ev[n].request_id = (int32_t)r->id;
      e->ev[n].server = (int16_t)e->server;
      e->ev[n].code = (int16_t)code;
    }
    *e->ev_n = n + 1;
  }
}

/* per-step scratch is shared by all engines of an instance (one steps at a time) */
typedef struct {
  Req** tmp; Req** tmp2; Req** dispatch; Req** preempt; Req** plan_dec; Req** plan_pf;
  int64_t* plan_chunk; Req** finished_now;
} Shared;
static int shared_init(Shared* sh, int64_t nreq) {
  int64_t cap = nreq + 4;
  sh->tmp = (Req**)malloc(sizeof(Req*) * cap);
  sh->tmp2 = (Req**)malloc(sizeof(Req*) * cap);
  sh->dispatch = (Req**)malloc(sizeof(Req*) * cap);
  sh->preempt = (Req**)malloc(sizeof(Req*) * cap);
  sh->plan_dec = (Req**)malloc(sizeof(Req*) * cap);
  sh->plan_pf = (Req**)malloc(sizeof(Req*) * cap);
  sh->plan_chunk = (int64_t*)malloc(sizeof(int64_t) * cap);
  sh->finished_now = (Req**)malloc(sizeof(Req*) * cap);
  return sh->tmp && sh->tmp2 && sh->dispatch && sh->preempt && sh->plan_dec && sh->plan_pf &&
         sh->plan_chunk && sh->finished_now;
}
static void shared_free(Shared* sh) {
  free(sh->tmp); free(sh->tmp2); free(sh->dispatch); free(sh->preempt);
  free(sh->plan_dec); free(sh->plan_pf); free(sh->plan_chunk); free(sh->finished_now);
}
static int eng_init(Eng* e, const ssb_engine_params* p, const Shared* sh, int server) {
  memset(e, 0, sizeof(*e));
  e->p = *p;
  e->free_blocks = p->pool_blocks;
  e->clock = 0.0;
  e->digest = FNV_OFF;
  e->server = server;
  if (!dq_init(&e->waiting, 64)) return 0;
  e->runcap = 64;
  e->running = (Req**)malloc(sizeof(Req*) * e->runcap);
  e->tmp = sh->tmp; e->tmp2 = sh->tmp2; e->dispatch = sh->dispatch; e->preempt = sh->preempt;
  e->plan_dec = sh->plan_dec; e->plan_pf = sh->plan_pf; e->plan_chunk = sh->plan_chunk;
  e->finished_now = sh->finished_now;
  return e->running != NULL;
}
static void eng_free(Eng* e) { free(e->waiting.buf); free(e->running); }
static inline int eng_has_work(const Eng* e) { return e->waiting.len > 0 || e->nrun > 0; } /* engine.py:171-173 */

/* ---- KvBlockPool (kvmem.py:74-154) ---- */
static int pool_try_allocate(Eng* e, Req* r, int64_t tokens) { /* :106-117 */
  int64_t need = blocks_needed(tokens, e->p.block_size);
  if (need > e->free_blocks) return 0;
  r->kv_tokens = tokens; r->has_alloc = 1;
  e->free_blocks -= need;
  return 1;
}
static int pool_try_grow(Eng* e, Req* r, int64_t new_total) { /* :119-140 */
  int64_t extra = blocks_needed(new_total, e->p.block_size) - blocks_needed(r->kv_tokens, e->p.block_size);
  if (extra > e->free_blocks) return 0;
  r->kv_tokens = new_total;
  e->free_blocks -= extra;
  return 1;
}
static int64_t pool_allocated_blocks(const Eng* e, const Req* r) { return blocks_needed(r->kv_tokens, e->p.block_size); }
static void pool_free(Eng* e, Req* r) { /* :142-149 */
  e->free_blocks += blocks_needed(r->kv_tokens, e->p.block_size);
  r->has_alloc = 0; r->kv_tokens = 0;
}

static void running_remove(Eng* e, Req* r) { /* del self.running[id] */
  int64_t i = 0;
  while (i < e->nrun && e->running[i] != r) i++;
  for (; i + 1 < e->nrun; i++) e->running[i] = e->running[i + 1];
  e->nrun--;
}

static void tf_fix_up(TrailFast* t, int64_t i) { /* restore node = min(children) above leaf i */
  for (i >>= 1; i >= 1; i >>= 1) {
    int32_t m = t->tree[2 * i] < t->tree[2 * i + 1] ? t->tree[2 * i] : t->tree[2 * i + 1];
    if (t->tree[i] == m) break;
    t->tree[i] = m;
  }
}
static void tf_insert(Eng* e, Req* r) { /* into bucket output-generated, ascending id */
  TrailFast* t = e->tf;
  int64_t b = (int64_t)r->output - r->generated;
  int32_t id = (int32_t)r->id;
  int32_t after = t->tail[b];
  if (after >= 0 && after > id) { /* a re-queued request: find its place from the head */
    after = -1;
    for (int32_t c = t->head[b]; c >= 0 && c < id; c = t->next[c]) after = c;
  }
  int32_t before = after >= 0 ? t->next[after] : t->head[b];
  t->prev[id] = after; t->next[id] = before;
  if (after >= 0) t->next[after] = id; else t->head[b] = id;
  if (before >= 0) t->prev[before] = id; else t->tail[b] = id;
  int64_t need = blocks_needed(pending_prefill(r), e->p.block_size);
  int64_t leaf = t->size + b;
  if (need < t->tree[leaf]) { t->tree[leaf] = (int32_t)need; tf_fix_up(t, leaf); }
  e->waiting.len++;
}
static void tf_remove(Eng* e, Req* r) {
  TrailFast* t = e->tf;
  int64_t b = (int64_t)r->output - r->generated;
  int32_t id = (int32_t)r->id, p = t->prev[id], n = t->next[id];
  if (p >= 0) t->next[p] = n; else t->head[b] = n;
  if (n >= 0) t->prev[n] = p; else t->tail[b] = p;
  int32_t m = INT32_MAX;
  for (int32_t c = t->head[b]; c >= 0; c = t->next[c]) {
    int64_t need = blocks_needed(pending_prefill(&e->reqs[c]), e->p.block_size);
    if (need < m) m = (int32_t)need;
  }
  int64_t leaf = t->size + b;
  if (t->tree[leaf] != m) { t->tree[leaf] = m; tf_fix_up(t, leaf); }
  e->waiting.len--;
}
/* first bucket >= b whose minimum need is <= T, or -1 */
static int64_t tf_first(const TrailFast* t, int64_t b, int64_t T) {
  if (b >= t->nb) return -1;
  int64_t i = t->size + b;
  if (t->tree[i] <= T) return b;
  while (i > 1) {
    if (!(i & 1) && t->tree[i + 1] <= T) { i = i + 1; break; }
    i >>= 1;
  }
  if (i == 1) return -1;
  while (i < t->size) { i = 2 * i; if (t->tree[i] > T) i++; }
  return i - t->size < t->nb ? i - t->size : -1;
}

/* ---- engine internals (engine.py:287-412) ---- */
static void eng_enqueue(Eng* e, Req* r) { /* :175-184 */
  r->enqueue_time = e->clock;
  if (e->tf) tf_insert(e, r); else dq_push_back(&e->waiting, r);
  eng_log(e, SSB_EV_ENQUEUE, r);
}
static void eng_preempt(Eng* e, Req* r, int code) { /* :368-379 */
  pool_free(e, r);
  r->state = ST_WAITING;
  r->prefill_done = 0;
  r->preempt_count += 1;
  r->enqueue_time = e->clock;
  r->dispatch_seq = -1;
  running_remove(e, r);
  if (e->tf) tf_insert(e, r); else dq_push_front(&e->waiting, r);
  if (code == SSB_EV_PARK) e->parks++; else e->preempts++;
  eng_log(e, code, r);
}
static void eng_dispatch(Eng* e, Req* r) { /* :287-298 */
  if (!pool_try_allocate(e, r, pending_prefill(r))) { e->status = SSB_E_INVARIANT; return; }
  if (e->tf) tf_remove(e, r); else dq_remove(&e->waiting, r);
  r->state = ST_PREFILLING;
  r->dispatch_seq = e->next_seq++;
  if (r->preempt_count == 0 && isnan(r->first_dispatch)) r->first_dispatch = e->clock;
  if (e->nrun == e->runcap) {
    e->runcap *= 2;
    e->running = (Req**)realloc(e->running, sizeof(Req*) * e->runcap);
  }
  e->running[e->nrun++] = r;
  e->dispatches++;
  eng_log(e, SSB_EV_DISPATCH, r);
}
static void eng_finish(Eng* e, Req* r) { /* :360-366 */
  pool_free(e, r);
  r->state = ST_FINISHED;
  r->finish = e->clock;
  running_remove(e, r);
  e->finished_now[e->nfinished_now++] = r;
  e->finished++;
  eng_log(e, SSB_EV_FINISH, r);
}
static int cmp_seq_desc(const void* a, const void* b) {
  int64_t x = (*(Req* const*)a)->dispatch_seq, y = (*(Req* const*)b)->dispatch_seq;
  return (x < y) - (x > y);
}
static void eng_evict_for_blocks(Eng* e, int64_t needed, const Req* exclude) { /* :381-388 */
  int64_t n = e->nrun;
  memcpy(e->tmp2, e->running, sizeof(Req*) * n);
  qsort(e->tmp2, n, sizeof(Req*), cmp_seq_desc);
  for (int64_t i = 0; i < n; i++) {
    if (e->free_blocks >= needed) break;
    if (e->tmp2[i] == exclude) continue;
    eng_preempt(e, e->tmp2[i], SSB_EV_PREEMPT);
  }
}
static int eng_grow_or_evict(Eng* e, Req* r, int64_t new_total) { /* :390-412 */
  if (pool_try_grow(e, r, new_total)) return 1;
  int64_t needed = blocks_needed(new_total, e->p.block_size) - pool_allocated_blocks(e, r);
  eng_evict_for_blocks(e, needed, r);
  if (pool_try_grow(e, r, new_total)) return 1;
  eng_preempt(e, r, SSB_EV_PARK); /* logger.warning(...) then park */
  return 0;
}

/* ---- policies (policies.py) ---- */
static int64_t open_slots(const Eng* e, int64_t running_count) { /* :70-73 */
  if (e->p.max_running < 0) return INT64_MAX;
  return (int64_t)e->p.max_running - running_count;
}

static void select_fcfs(Eng* e) { /* policies.py:87-97 */
  int64_t free = e->free_blocks;
  int64_t slots = open_slots(e, e->nrun);
  for (int64_t i = 0; i < e->waiting.len; i++) {
    Req* r = dq_get(&e->waiting, i);
    int64_t need = blocks_needed(pending_prefill(r), e->p.block_size);
    if (e->ndisp >= slots || need > free) break;
    e->dispatch[e->ndisp++] = r;
    free -= need;
  }
}

static int64_t reservation_tokens(const Eng* e, const Req* r) { /* policies.py:116-117 */
  int64_t a = e->p.max_context, b = (int64_t)r->prompt + e->p.max_output;
  return a < b ? a : b;
}
static void select_nopreempt(Eng* e) { /* policies.py:133-146 */
  int64_t bs = e->p.block_size, committed = 0;
  for (int64_t i = 0; i < e->nrun; i++) committed += blocks_needed(reservation_tokens(e, e->running[i]), bs);
  int64_t slots = open_slots(e, e->nrun);
  for (int64_t i = 0; i < e->waiting.len; i++) {
    Req* r = dq_get(&e->waiting, i);
    int64_t need = blocks_needed(reservation_tokens(e, r), bs);
    if (e->ndisp >= slots || committed + need > e->p.pool_blocks) break;
    e->dispatch[e->ndisp++] = r;
    committed += need;
  }
}

static int cmp_trail(const void* a, const void* b) { /* key (output-generated, arrival, id), :171-173 */
  const Req* x = *(Req* const*)a; const Req* y = *(Req* const*)b;
  int64_t rx = (int64_t)x->output - x->generated, ry = (int64_t)y->output - y->generated;
  if (rx != ry) return rx < ry ? -1 : 1;
  if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}
static int cmp_victim(const void* a, const void* b) { /* key (-(remaining), -dispatch_seq), :197 */
  const Req* x = *(Req* const*)a; const Req* y = *(Req* const*)b;
  int64_t rx = (int64_t)x->output - x->generated, ry = (int64_t)y->output - y->generated;
  if (rx != ry) return rx > ry ? -1 : 1;
  return (x->dispatch_seq < y->dispatch_seq) - (x->dispatch_seq > y->dispatch_seq);
}
static void select_trail(Eng* e, uint8_t* marked /* indexed by running position */) { /* :168-212 */
  int64_t bs = e->p.block_size, free = e->free_blocks;
  int64_t W = e->waiting.len;
  for (int64_t i = 0; i < W; i++) e->tmp[i] = dq_get(&e->waiting, i);
  qsort(e->tmp, W, sizeof(Req*), cmp_trail);
  int64_t running_count = e->nrun;
  memset(marked, 0, (size_t)e->nrun);
  for (int64_t k = 0; k < W; k++) {
    Req* r = e->tmp[k];
    int64_t slots = open_slots(e, running_count + e->ndisp - e->npre);
    if (slots < 1) continue;
    int64_t need = blocks_needed(pending_prefill(r), bs);
    if (need <= free) { e->dispatch[e->ndisp++] = r; free -= need; continue; }
    if (e->p.c == 0.0) continue;
    int64_t remaining = (int64_t)r->output - r->generated;
    int64_t nv = 0;
    for (int64_t i = 0; i < e->nrun; i++) {
      Req* q = e->running[i];
      if (!marked[i] && (double)q->generated < e->p.c * (double)q->output &&
          ((int64_t)q->output - q->generated) > remaining)
        e->tmp2[nv++] = q;
    }
    qsort(e->tmp2, nv, sizeof(Req*), cmp_victim);
    int64_t gain = 0, nchosen = 0;
    for (int64_t i = 0; i < nv; i++) {
      if (free + gain >= need) break;
      gain += pool_allocated_blocks(e, e->tmp2[i]);
      nchosen++;
    }
    if (free + gain < need) continue;
    for (int64_t i = 0; i < nchosen; i++) {
      Req* q = e->tmp2[i];
      e->preempt[e->npre++] = q;
      for (int64_t j = 0; j < e->nrun; j++) if (e->running[j] == q) marked[j] = 1;
    }
    free += gain;
    e->dispatch[e->ndisp++] = r;
    free -= need;
  }
}

/* select_trail with the same decisions: candidates in (remaining, arrival, id) order, but only
 * the admissible ones are visited. A candidate with remaining b is admissible iff
 * need <= free + G(b), G(b) = blocks of the unmarked eligible running requests with remaining
 * > b (exactly when the literal victim loop reaches free + gain >= need, :183-206); G is
 * non-increasing in b, so free + G(b) bounds every candidate in buckets >= b and tf_first skips
 * buckets whose minimum need exceeds it. Skipped candidates are never revisited (literal: each
 * is visited once), and nothing changes between dispatches. slots < 1 skips every later
 * candidate (nothing changes while skipping), so it ends the loop. */
static void select_trail_fast(Eng* e, uint8_t* marked) {
  TrailFast* t = e->tf;
  int64_t bs = e->p.block_size, free = e->free_blocks;
  int64_t running_count = e->nrun;
  memset(marked, 0, (size_t)e->nrun);
  int64_t nv = 0; /* eligible victims (:190-196), in (-remaining, -dispatch_seq) order (:197) */
  if (e->p.c != 0.0)
    for (int64_t i = 0; i < e->nrun; i++) {
      Req* q = e->running[i];
      if ((double)q->generated < e->p.c * (double)q->output) e->tmp2[nv++] = q;
    }
  qsort(e->tmp2, nv, sizeof(Req*), cmp_victim);
  uint8_t* taken = marked; /* indexed by position in tmp2 here */
  int64_t b = 0;
  int32_t after = -1;
  for (;;) {
    if (open_slots(e, running_count + e->ndisp - e->npre) < 1) break; /* :179-181 */
    int64_t g = 0;
    for (int64_t i = 0; i < nv; i++)
      if (!taken[i] && (int64_t)e->tmp2[i]->output - e->tmp2[i]->generated > b) g += pool_allocated_blocks(e, e->tmp2[i]);
    int64_t T = free + g;
    int64_t fb = tf_first(t, b, T);
    if (fb < 0) break;
    if (fb != b) { b = fb; after = -1; continue; } /* re-derive G at the found bucket */
    int32_t c = after >= 0 ? t->next[after] : t->head[b];
    int64_t need = 0;
    for (; c >= 0; c = t->next[c]) {
      need = blocks_needed(pending_prefill(&e->reqs[c]), bs);
      if (need <= T) break;
    }
    if (c < 0) { b += 1; after = -1; continue; }
    Req* r = &e->reqs[c];
    if (need > free) { /* victims largest remaining first, youngest first, until it fits */
      int64_t gain = 0;
      for (int64_t i = 0; i < nv && free + gain < need; i++) {
        Req* q = e->tmp2[i];
        if (taken[i] || (int64_t)q->output - q->generated <= b) continue;
        taken[i] = 1;
        gain += pool_allocated_blocks(e, q);
        e->preempt[e->npre++] = q;
      }
      free += gain;
    }
    e->dispatch[e->ndisp++] = r;
    free -= need;
    after = c;
  }
}

typedef struct { Req* r; double neg_score; } LarryKey;
static int cmp_larry(const void* a, const void* b) { /* key (-score, enqueue_time, id), :260-267 */
  const LarryKey* x = (const LarryKey*)a; const LarryKey* y = (const LarryKey*)b;
  if (x->neg_score != y->neg_score) return x->neg_score < y->neg_score ? -1 : 1;
  if (x->r->enqueue_time != y->r->enqueue_time) return x->r->enqueue_time < y->r->enqueue_time ? -1 : 1;
  return (x->r->id > y->r->id) - (x->r->id < y->r->id);
}
/* policies.py:215-224 larry_score; Python: alpha*wait - queue_len*pending (int product -> float) */
static inline double larry_score(const Req* r, double clock, int64_t queue_len, double alpha) {
  double wait = clock - r->enqueue_time;
  return alpha * wait - (double)(queue_len * pending_prefill(r));
}
static void select_larry(Eng* e, LarryKey* keys) { /* :244-276 */
  int64_t bs = e->p.block_size, free = e->free_blocks;
  int64_t slots = open_slots(e, e->nrun);
  int64_t budget = e->p.max_tokens_per_batch;
  for (int64_t i = 0; i < e->nrun; i++) if (e->running[i]->state == ST_DECODING) budget -= 1;
  if (budget < 0) budget = 0;
  /* prefilling requests sorted by dispatch_seq == running (insertion) order */
  for (int64_t i = 0; i < e->nrun; i++) {
    Req* q = e->running[i];
    if (q->state != ST_PREFILLING) continue;
    if (budget == 0) break;
    int64_t pp = pending_prefill(q);
    budget -= pp < budget ? pp : budget;
  }
  int64_t W = e->waiting.len, queue_len = W;
  for (int64_t i = 0; i < W; i++) {
    Req* r = dq_get(&e->waiting, i);
    keys[i].r = r;
    keys[i].neg_score = -larry_score(r, e->clock, queue_len, e->p.alpha);
  }
  qsort(keys, W, sizeof(LarryKey), cmp_larry);
  for (int64_t i = 0; i < W; i++) {
    Req* r = keys[i].r;
    int64_t need = blocks_needed(pending_prefill(r), bs);
    if (e->ndisp >= slots || need > free || budget <= 0) break;
    e->dispatch[e->ndisp++] = r;
    free -= need;
    int64_t pp = pending_prefill(r);
    budget -= pp < budget ? pp : budget;
  }
}

/* ---- Engine.step (engine.py:193-234) ---- */
typedef struct { uint8_t* marked; LarryKey* keys; } StepScratch;

static void eng_step(Eng* e, StepScratch* sc) {
  if (!eng_has_work(e)) { e->status = SSB_E_STALL; return; }
  e->ndisp = e->npre = 0;
  e->nfinished_now = 0;
  switch (e->p.policy) {
    case SSB_POLICY_FCFS: select_fcfs(e); break;
    case SSB_POLICY_NOPREEMPT: select_nopreempt(e); break;
    case SSB_POLICY_TRAIL_PLUS: if (e->tf) select_trail_fast(e, sc->marked); else select_trail(e, sc->marked); break;
    case SSB_POLICY_LARRY: select_larry(e, sc->keys); break;
    default: e->status = SSB_E_ARG; return;
  }
  for (int64_t i = 0; i < e->npre; i++) eng_preempt(e, e->preempt[i], SSB_EV_PREEMPT); /* :203-204 */
  for (int64_t i = 0; i < e->ndisp; i++) { eng_dispatch(e, e->dispatch[i]); if (e->status) return; } /* :205-206 */

  /* _form_batch (engine.py:300-323); running is in dispatch_seq order */
  int64_t cap = e->p.max_tokens_per_batch, budget = cap;
  e->nplan_dec = e->nplan_pf = 0;
  for (int64_t i = 0; i < e->nrun; i++) {
    Req* q = e->running[i];
    if (q->state != ST_DECODING) continue;
    if (budget == 0) break;
    e->plan_dec[e->nplan_dec++] = q;
    budget -= 1;
  }
  for (int64_t i = 0; i < e->nrun; i++) {
    Req* q = e->running[i];
    if (q->state != ST_PREFILLING) continue;
    if (budget == 0) break;
    int64_t pp = pending_prefill(q), chunk = pp < budget ? pp : budget;
    e->plan_pf[e->nplan_pf] = q;
    e->plan_chunk[e->nplan_pf++] = chunk;
    budget -= chunk;
  }
  int64_t total = cap - budget;
  if (total == 0) { e->status = SSB_E_STALL; return; } /* :209-214 */
  e->rsteps += e->nplan_dec + e->nplan_pf;
  e->btokens += total;

  /* engine.py:217-220 */
  int64_t resident = 0;
  for (int64_t i = 0; i < e->nplan_dec; i++) resident += context_len(e->plan_dec[i]);
  for (int64_t i = 0; i < e->nplan_pf; i++) resident += context_len(e->plan_pf[i]);
  /* costmodel.py:45-47 iteration_latency */
  double mem = e->p.mem_base_s + e->p.mem_per_kv_token_s * (double)resident;
  double compute = e->p.compute_per_token_s * (double)total;
  double latency = e->p.overhead_s + (compute > mem ? compute : mem);
  e->clock += latency;

  /* _apply_progress (engine.py:325-358) */
  for (int64_t i = 0; i < e->nplan_pf; i++) {
    Req* r = e->plan_pf[i];
    if (r->state != ST_PREFILLING) continue; /* evicted earlier in this pass */
    r->prefill_done += (int32_t)e->plan_chunk[i];
    if (r->prefill_done < prefill_target(r)) continue;
    if (r->generated == 0) {
      if (!eng_grow_or_evict(e, r, (int64_t)r->prompt + 1)) continue;
      r->generated = 1;
      r->first_token = e->clock;
      r->state = ST_DECODING;
      eng_log(e, SSB_EV_FIRST_TOKEN, r);
      if (r->generated == r->output) eng_finish(e, r);
    } else {
      r->state = ST_DECODING; /* recompute: no token */
    }
  }
  for (int64_t i = 0; i < e->nplan_dec; i++) {
    Req* r = e->plan_dec[i];
    if (r->state != ST_DECODING) continue;
    if (!eng_grow_or_evict(e, r, (int64_t)r->prompt + r->generated + 1)) continue;
    r->generated += 1;
    if (r->generated == r->output) eng_finish(e, r);
  }
  if (total > e->peak) e->peak = total;
  e->iterations++;
}

/* ---- PCG64 + Generator.integers (numpy) ---- */
typedef struct {
  unsigned __int128 state, inc;
  int has32;
  uint32_t buf32;
} Pcg64;
static uint64_t pcg64_next64(Pcg64* g) { /* pcg_setseq_128_xsl_rr_64: step, then output */
  const unsigned __int128 MULT = (((unsigned __int128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
  g->state = g->state * MULT + g->inc;
  uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
  unsigned rot = (unsigned)(g->state >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}
static uint32_t pcg64_next32(Pcg64* g) { /* buffered: low half first */
  if (g->has32) { g->has32 = 0; return g->buf32; }
  uint64_t v = pcg64_next64(g);
  g->has32 = 1;
  g->buf32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}
static int64_t rng_integers(Pcg64* g, int64_t high) { /* Generator.integers(high), 32-bit Lemire */
  uint64_t rng = (uint64_t)(high - 1);
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return pcg64_next32(g);
  uint32_t rng_excl = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)pcg64_next32(g) * rng_excl;
  uint32_t left = (uint32_t)m;
  if (left < rng_excl) {
    uint32_t thr = (uint32_t)(UINT32_MAX - (uint32_t)rng) % rng_excl;
    while (left < thr) {
      m = (uint64_t)pcg64_next32(g) * rng_excl;
      left = (uint32_t)m;
    }
  }
  return (int64_t)(m >> 32);
}

/* ---- run_cluster heap (cluster.py:124-157) ---- */
typedef struct { double t; int32_t kind; int64_t key, payload; } HEv;
static int hev_less(const HEv* a, const HEv* b) {
  if (a->t != b->t) return a->t < b->t;
  if (a->kind != b->kind) return a->kind < b->kind;
  if (a->key != b->key) return a->key < b->key;
  return a->payload < b->payload;
}
typedef struct { HEv* a; int64_t n, cap; } Heap;
static void heap_push(Heap* h, HEv v) {
  int64_t i = h->n++;
  h->a[i] = v;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!hev_less(&h->a[i], &h->a[p])) break;
    HEv t = h->a[i]; h->a[i] = h->a[p]; h->a[p] = t; i = p;
  }
}
static HEv heap_pop(Heap* h) {
  HEv top = h->a[0];
  h->a[0] = h->a[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && hev_less(&h->a[l], &h->a[m])) m = l;
    if (r < h->n && hev_less(&h->a[r], &h->a[m])) m = r;
    if (m == i) break;
    HEv t = h->a[i]; h->a[i] = h->a[m]; h->a[m] = t; i = m;
  }
  return top;
}

/* feasibility: SchedulerPolicy.check_feasible (policies.py:56-68) + NoPreempt (:119-131) */
static int check_feasible(const ssb_engine_params* p, const Req* r) {
  int64_t peak = (int64_t)r->prompt + r->output;
  if (peak > p->max_context) return 0;
  if (blocks_needed(peak, p->block_size) > p->pool_blocks) return 0;
  if (p->policy == SSB_POLICY_NOPREEMPT) {
    if (r->output > p->max_output) return 0;
    int64_t res = p->max_context < (int64_t)r->prompt + p->max_output ? p->max_context : (int64_t)r->prompt + p->max_output;
    if (blocks_needed(res, p->block_size) > p->pool_blocks) return 0;
  }
  return 1;
}

typedef struct { int64_t queued, free_mem, in_flight; } SStats; /* balancers.py:20-26 */

/* mode 0: run_cluster (cluster.py:65-174); mode 1: Engine.run (engine.py:236-265, n_servers==1) */
int ssb_oracle_run(const ssb_instance* inst, ssb_trace trace, ssb_records rec, ssb_stats* st,
                   ssb_event* ev, int64_t ev_cap, int64_t* ev_count, int32_t mode) {
  memset(st, 0, sizeof(*st));
  int64_t N = inst->n_requests, n = inst->n_servers;
  const ssb_engine_params* p = &inst->engine;
  if (n < 1 || N < 0 || (mode == 1 && n != 1)) { st->status = SSB_E_ARG; return SSB_E_ARG; }
  int64_t ev_local = 0;
  if (!ev_count) ev_count = &ev_local;
  *ev_count = 0;

  Req* reqs = (Req*)calloc((size_t)(N > 0 ? N : 1), sizeof(Req));
  Eng* engs = (Eng*)calloc((size_t)n, sizeof(Eng));
  StepScratch sc;
  Shared sh;
  sc.marked = (uint8_t*)malloc((size_t)N + 4);
  sc.keys = (LarryKey*)malloc(sizeof(LarryKey) * ((size_t)N + 4));
  int status = SSB_OK;
  int sh_ok = shared_init(&sh, N);
  if (!reqs || !engs || !sc.marked || !sc.keys || !sh_ok) { status = SSB_E_ARG; goto out_nofree_engs; }
  for (int64_t i = 0; i < N; i++) {
    Req* r = &reqs[i];
    r->id = i;
    r->arrival = trace.arrival[inst->trace_offset + i] / inst->qps_factor; /* workload.py:193 */
    r->prompt = trace.prompt[inst->trace_offset + i];
    r->output = trace.output[inst->trace_offset + i];
    r->state = ST_WAITING;
    r->first_token = r->finish = r->first_dispatch = NAN;
    r->dispatch_seq = -1;
    r->server = -1;
  }
  for (int64_t i = 0; i + 1 < N; i++)
    if (reqs[i + 1].arrival < reqs[i].arrival) { status = SSB_E_ARG; goto out_nofree_engs; } /* cluster.py:81-83 */
  /* prebuilt engines that differ (cluster.py:66-79): server s with its own parameters */
#define SERVER_PARAMS(s) (inst->h_servers ? &inst->h_servers[(s)] : p)
  for (int64_t s = 0; s < (inst->h_servers ? n : 1); s++) /* every engine checks every request */
    for (int64_t i = 0; i < N; i++)
      if (!check_feasible(SERVER_PARAMS(s), &reqs[i])) { status = SSB_E_INFEASIBLE; goto out_nofree_engs; } /* cluster.py:90-92 */
  for (int64_t s = 0; s < n; s++) {
    if (!eng_init(&engs[s], SERVER_PARAMS(s), &sh, (int)s)) { status = SSB_E_ARG; goto out; }
    engs[s].ev = ev; engs[s].ev_cap = ev_cap; engs[s].ev_n = ev_count;
    engs[s].reqs = reqs;
  }
  TrailFast tfs;
  memset(&tfs, 0, sizeof(tfs));
  if (g_trail_fast && mode == 1 && p->policy == SSB_POLICY_TRAIL_PLUS) {
    int64_t maxo = 1;
    for (int64_t i = 0; i < N; i++) if (reqs[i].output > maxo) maxo = reqs[i].output;
    tfs.nb = maxo + 1;
    tfs.size = 1;
    while (tfs.size < tfs.nb) tfs.size *= 2;
    tfs.head = (int32_t*)malloc(sizeof(int32_t) * tfs.nb);
    tfs.tail = (int32_t*)malloc(sizeof(int32_t) * tfs.nb);
    tfs.next = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
    tfs.prev = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
    tfs.tree = (int32_t*)malloc(sizeof(int32_t) * 2 * tfs.size);
    if (!tfs.head || !tfs.tail || !tfs.next || !tfs.prev || !tfs.tree) { status = SSB_E_ARG; goto out; }
    for (int64_t i = 0; i < tfs.nb; i++) tfs.head[i] = tfs.tail[i] = -1;
    for (int64_t i = 0; i < 2 * tfs.size; i++) tfs.tree[i] = INT32_MAX;
    engs[0].tf = &tfs;
  }

  if (mode == 1) {
    /* Engine.run (engine.py:256-265) */
    Eng* e = &engs[0];
    int64_t pending = 0, done = 0;
    while (done < N) {
      if (!eng_has_work(e)) { double t = reqs[pending].arrival; if (t > e->clock) e->clock = t; }
      while (pending < N && reqs[pending].arrival <= e->clock) { reqs[pending].server = 0; eng_enqueue(e, &reqs[pending++]); }
      eng_step(e, &sc);
      if (e->status) { status = e->status; goto out; }
      done += e->nfinished_now;
    }
  } else {
    /* run_cluster */
    Pcg64 rng;
    rng.state = (((unsigned __int128)inst->pcg_state_hi) << 64) | inst->pcg_state_lo;
    rng.inc = (((unsigned __int128)inst->pcg_inc_hi) << 64) | inst->pcg_inc_lo;
    rng.has32 = 0; rng.buf32 = 0;
    SStats* view = (SStats*)calloc((size_t)n, sizeof(SStats));
    Deque* inbox = (Deque*)calloc((size_t)n, sizeof(Deque));
    uint8_t* scheduled = (uint8_t*)calloc((size_t)n, 1);
    Heap heap; heap.cap = N + n + 4; heap.n = 0; heap.a = (HEv*)malloc(sizeof(HEv) * heap.cap);
    for (int64_t s = 0; s < n; s++) dq_init(&inbox[s], 64);
    double last_poll = -INFINITY;
    int64_t rr_i = 0, beta_count = 0, beta_in = 0, beta_out = 0;
    const int estimate_beta = isnan(inst->beta_fixed);

    /* ground_truth (cluster.py:110-120) + snapshot_stats (:50-59) + refresh (balancers.py:45-50) */
#define REFRESH(tnow)                                                              \
  do {                                                                             \
    for (int64_t s_ = 0; s_ < n; s_++) {                                           \
      Eng* e_ = &engs[s_];                                                         \
      int64_t q_ = 0;                                                              \
      for (int64_t k_ = 0; k_ < e_->waiting.len; k_++) q_ += pending_prefill(dq_get(&e_->waiting, k_)); \
      int64_t inf_ = e_->waiting.len + e_->nrun;                                   \
      for (int64_t k_ = 0; k_ < inbox[s_].len; k_++) { q_ += pending_prefill(dq_get(&inbox[s_], k_)); inf_++; } \
      view[s_].queued = q_;                                                        \
      view[s_].free_mem = e_->free_blocks * e_->p.block_size;                      \
      view[s_].in_flight = inf_;                                                   \
    }                                                                              \
    last_poll = (tnow);                                                            \
  } while (0)

    REFRESH(0.0); /* cluster.py:122 */
    for (int64_t i = 0; i < N; i++) heap_push(&heap, (HEv){reqs[i].arrival, 0, i, i});
    while (heap.n > 0) {
      HEv top = heap_pop(&heap);
      if (top.kind == 0) {
        Req* req = &reqs[top.payload];
        double t = top.t;
        if (t - last_poll >= inst->poll_interval_s) REFRESH(t); /* BalancerView.poll, balancers.py:42-57 */
        int64_t s = 0;
        switch (inst->balancer) {
          case SSB_BAL_RR: s = rr_i % n; rr_i++; break; /* :139-142 */
          case SSB_BAL_RANDOM: s = rng_integers(&rng, n); break; /* :152-153 */
          case SSB_BAL_P2C: { /* :167-176 */
            if (n == 1) { s = 0; break; }
            int64_t i = rng_integers(&rng, n), j = rng_integers(&rng, n - 1);
            if (j >= i) j += 1;
            s = (view[j].in_flight < view[i].in_flight) ? j : i;
            break;
          }
          case SSB_BAL_SAL: { /* :204-212 */
            double beta = estimate_beta ? (beta_count == 0 ? inst->beta_prior
                                                            : (double)(beta_in + beta_out) / (double)beta_out)
                                        : inst->beta_fixed;
            double best = 0.0;
            int64_t bi = 0;
            for (int64_t k = 0; k < n; k++) {
              /* sal_load, balancers.py:103-112 */
              double memory_term = beta * (double)((int64_t)req->prompt - view[k].free_mem);
              double queue_term = (double)(view[k].queued + req->prompt) / (double)inst->route_cap; /* settings cap, cluster.py:101 */
              double load = queue_term > memory_term ? queue_term : memory_term;
              if (k == 0 || load < best) { best = load; bi = k; }
            }
            s = bi;
            /* note_routed, balancers.py:59-64 */
            view[s].queued += req->prompt;
            view[s].free_mem = view[s].free_mem - req->prompt > 0 ? view[s].free_mem - req->prompt : 0;
            view[s].in_flight += 1;
            break;
          }
          default: status = SSB_E_ARG; break;
        }
        if (status) break;
        req->server = (int32_t)s;
        dq_push_back(&inbox[s], req);
        if (!scheduled[s]) {
          double wake = t > engs[s].clock ? t : engs[s].clock;
          heap_push(&heap, (HEv){wake, 1, s, 0});
          scheduled[s] = 1;
        }
      } else {
        int64_t s = top.key;
        Eng* e = &engs[s];
        scheduled[s] = 0;
        if (top.t > e->clock) e->clock = top.t; /* advance_to (engine.py:186-191) */
        while (inbox[s].len > 0) eng_enqueue(e, dq_pop_front(&inbox[s]));
        if (!eng_has_work(e)) continue;
        eng_step(e, &sc);
        if (e->status) { status = e->status; break; }
        for (int64_t k = 0; k < e->nfinished_now; k++) { /* on_finish, cluster.py:153-154 */
          if (inst->balancer == SSB_BAL_SAL && estimate_beta) {
            beta_count++;
            beta_in += e->finished_now[k]->prompt;
            beta_out += e->finished_now[k]->output;
          }
        }
        if (eng_has_work(e)) { heap_push(&heap, (HEv){e->clock, 1, s, 0}); scheduled[s] = 1; }
      }
    }
#undef REFRESH
    for (int64_t s = 0; s < n; s++) free(inbox[s].buf);
    free(inbox); free(view); free(scheduled); free(heap.a);
    if (status) goto out;
    for (int64_t i = 0; i < N; i++)
      if (reqs[i].state != ST_FINISHED) { status = SSB_E_INVARIANT; goto out; } /* cluster.py:159-161 */
  }

  /* records (cluster.py:162-174) and counters */
  for (int64_t i = 0; i < N; i++) {
    int64_t o = inst->record_offset + i;
    rec.first_token[o] = reqs[i].first_token;
    rec.finish[o] = reqs[i].finish;
    rec.first_dispatch[o] = reqs[i].first_dispatch;
    rec.preempt_count[o] = reqs[i].preempt_count;
    rec.server[o] = reqs[i].server;
  }
  st->digest = FNV_OFF;
  for (int64_t s = 0; s < n; s++) {
    Eng* e = &engs[s];
    st->iterations += e->iterations;
    st->request_steps += e->rsteps;
    st->batch_tokens += e->btokens;
    st->dispatches += e->dispatches;
    st->preempts += e->preempts;
    st->parks += e->parks;
    st->finished += e->finished;
    if (e->peak > st->peak_batch_tokens) st->peak_batch_tokens = e->peak;
    st->digest ^= e->digest;
    st->digest *= FNV_PRIME;
  }
out:
  free(tfs.head); free(tfs.tail); free(tfs.next); free(tfs.prev); free(tfs.tree);
  for (int64_t s = 0; s < n; s++) eng_free(&engs[s]);
out_nofree_engs:
  shared_free(&sh);
  free(engs); free(reqs); free(sc.marked); free(sc.keys);
  st->status = status;
  return status;
}

/* ---- multi-threaded batch driver (the CPU baseline times this) ---- */
typedef struct {
  const ssb_instance* inst;
  int32_t n_inst;
  ssb_trace trace;
  ssb_records rec;
  ssb_stats* st;
  int32_t mode;
  atomic_int next;
} Batch;
static void* batch_worker(void* arg) {
  Batch* b = (Batch*)arg;
  for (;;) {
    int i = atomic_fetch_add(&b->next, 1);
    if (i >= b->n_inst) break;
    int32_t mode = (b->mode == 1 && b->inst[i].n_servers == 1) ? 1 : 0;
    ssb_oracle_run(&b->inst[i], b->trace, b->rec, &b->st[i], NULL, 0, NULL, mode);
  }
  return NULL;
}
int ssb_oracle_run_many(const ssb_instance* inst, int32_t n_inst, ssb_trace trace, ssb_records rec,
                        ssb_stats* st, int32_t n_threads, int32_t mode) {
  Batch b;
  b.inst = inst; b.n_inst = n_inst; b.trace = trace; b.rec = rec; b.st = st; b.mode = mode;
  atomic_init(&b.next, 0);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, batch_worker, &b);
  for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
  free(th);
  int32_t worst = 0;
  for (int32_t i = 0; i < n_inst; i++) if (st[i].status) worst = st[i].status;
  return worst;
}

/* PCG64 / Generator.integers test hook: draw k values of integers(high) */
void ssb_oracle_rng_integers(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                             const int64_t* highs, int64_t k, int64_t* out) {
  Pcg64 g;
  g.state = (((unsigned __int128)state_hi) << 64) | state_lo;
  g.inc = (((unsigned __int128)inc_hi) << 64) | inc_lo;
  g.has32 = 0; g.buf32 = 0;
  for (int64_t i = 0; i < k; i++) out[i] = rng_integers(&g, highs[i]);
}

int32_t ssb_oracle_struct_sizes(int64_t* out) {
  out[0] = sizeof(ssb_engine_params); out[1] = sizeof(ssb_instance); out[2] = sizeof(ssb_stats);
  out[3] = sizeof(ssb_event); out[4] = sizeof(ssb_summary); out[5] = sizeof(ssb_summary_group);
  out[6] = sizeof(ssb_engine_stats);
  return 7;
}
