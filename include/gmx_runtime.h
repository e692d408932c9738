/*
 * gmx_runtime.h — native driver loop: scheduler decisions -> coalesced launches.
 *
 * Restates the reference's event loop (gpumux/engine.py:320-367) natively so a
 * serving step costs no Python: all events at one timestamp are drained
 * (COMPLETE before ARRIVAL before WAKEUP, ascending id), then the scheduler
 * steps once; the members of every dispatch returned by that step are executed
 * by ONE gmx_exec_launch; each dispatch's completion event is queued at d.end
 * and the wakeup (if any) as a WAKEUP event.
 *
 * Mode GMX_RT_LOCKSTEP: virtual time, completions at the decision model's
 * d.end (the reference's clock) — decisions are bit-identical to the
 * reference engine for the same arrivals, while the launches really run on
 * the GPU, back to back on the caller's stream.
 *
 * Straggler eviction (engine.py:345-351) is not run by this loop: in lockstep
 * mode observed == predicted, so no stream can exceed the threshold.
 */
#ifndef GMX_RUNTIME_H
#define GMX_RUNTIME_H

#include <stdint.h>

#include "gmx_core.h"
#include "gmx_exec.h"

#ifdef __cplusplus
extern "C" {
#endif

#define GMX_RT_LOCKSTEP 0
/* Wall-clock mode: `now` is the host clock in ns since the runtime's
 * origin; arrivals fire when their time has passed; a launch's dispatches complete when the
 * CUDA event recorded after the launch has completed (observed time); wakeups fire on the
 * clock. Every step is logged (time, events applied, decisions) for replay parity. */
#define GMX_RT_REALTIME 1

typedef struct gmx_runtime gmx_runtime;

typedef struct gmx_runtime_stats {
    int64_t now;                 /* virtual time after the run */
    int64_t steps;               /* scheduler steps taken */
    int64_t launches;            /* coalesced kernel launches issued */
    int64_t dispatches;          /* superkernels dispatched */
    int64_t kernels;             /* member kernels executed */
    int64_t withheld;            /* clusters withheld */
    int64_t completed_requests;
    int64_t useful_flops;        /* padding excluded (engine.py:425) */
    int64_t slo_misses;          /* completions after the request deadline */
    int64_t evicted_requests;    /* requests evicted: straggler streams (engine.py:345-351) + arrivals on them */
    int64_t cancelled_dispatches;
} gmx_runtime_stats;

/* Borrows `sched` and `ex` (caller keeps them alive). ex == NULL (lockstep only): a
 * decisions-only engine — same event loop, nothing launched (host-cost and parity runs). */
int gmx_runtime_create(gmx_sched* sched, gmx_exec* ex, int32_t mode, gmx_runtime** out);
void gmx_runtime_destroy(gmx_runtime* rt);
/* Queue one request's ARRIVAL (engine.py:316-318) and bind each kernel id to
 * the executor slot holding its operands. CSR deps as in gmx_sched_add_request. */
int gmx_runtime_submit(gmx_runtime* rt, int64_t request_id, int32_t stream, int64_t arrival,
                       int64_t deadline, const gmx_kernel_desc* kernels, int32_t n,
                       const int64_t* dep_ids, const int32_t* dep_offsets, const int32_t* slots);
/* Run the event loop until the heap is empty or the next event is later than
 * `until`; launches go to `cuda_stream`. Accumulates into the runtime's stats. */
int gmx_runtime_run(gmx_runtime* rt, int64_t until, void* cuda_stream, gmx_runtime_stats* out);
/* Completion records since the last call: request id and virtual completion time. */
int gmx_runtime_drain_completions(gmx_runtime* rt, int64_t* request_ids, int64_t* times,
                                  int32_t capacity, int32_t* n_out);
const char* gmx_runtime_last_error(void);
/* Realtime mode: set the clock origin (ns since the process steady-clock epoch); the first
 * run() sets it if unset. gmx_runtime_clock_ns returns the current runtime time. */
int gmx_runtime_set_origin(gmx_runtime* rt, int64_t steady_ns);
/* Realtime mode: launch round-robin over `n` runtime-owned CUDA streams so independent small
 * steps co-run on idle SMs (dependencies are already enforced by the scheduler: a kernel is
 * dispatched only after its predecessors' launches completed). n = 1 uses the run() stream. */
int gmx_runtime_set_streams(gmx_runtime* rt, int32_t n);
/* Cumulative host nanoseconds spent in the decision core (add_request, step, complete) and in
 * the executor's launch/enqueue path, for host-cost accounting of the serving loop. */
int gmx_runtime_host_profile(const gmx_runtime* rt, int64_t* ns4);
int gmx_runtime_set_profiling(gmx_runtime* rt, int32_t on);   /* off by default */
/* Wall-clock mode: feed the straggler windows with OBSERVED dispatch durations (completion seen
 * minus launch time) instead of the modeled ones — meaningful once the decision profile / a
 * measured TuningTable predicts real step times. Off by default. */
int gmx_runtime_set_measured_stragglers(gmx_runtime* rt, int32_t on);
int64_t gmx_runtime_clock_ns(const gmx_runtime* rt);
/* Replay log (realtime mode). Records, in order:
 *   kind 0: complete(dispatch_id=a) at time t; off = the observed duration fed to the straggler
 *           windows (set_measured_stragglers), -1 when the modeled duration was used
 *   kind 1: add_request(request_id=a) at t
 *   kind 2: step(t) -> dispatch a with kernels [off, off+n) of kernel_ids
 *   kind 3: step(t) withheld group [off, off+n)       kind 4: step(t) wakeup a (-1: none)
 *   kind 5: step(t) (marks the step boundary; precedes its kind 2/3/4 records)
 *   kind 6: straggler eviction of stream a at t (before the step at t)
 * Copies up to `capacity` records; *n_out = total available. */
typedef struct gmx_replay_rec {
    int32_t kind;
    int32_t n;
    int64_t t;
    int64_t a;
    int64_t off;
} gmx_replay_rec;
int gmx_runtime_replay_log(const gmx_runtime* rt, gmx_replay_rec* recs, int64_t capacity, int64_t* n_out,
                           int64_t* kernel_ids, int64_t kid_capacity, int64_t* n_kids);

#ifdef __cplusplus
}
#endif
#endif /* GMX_RUNTIME_H */
