/*
 * gmx_exec.h — C ABI of the coalesced sm_100a executor (libgmx_exec.so).
 *
 * The reference never executes a kernel: a dispatch's "execution" is the
 * number roofline_duration() returns (gpumux/device.py:140-150), turned into
 * a COMPLETE event at d.end (gpumux/engine.py:359-364). This library is the
 * real thing: ONE persistent launch per scheduler step whose work list spans
 * every member of every superkernel dispatched in that step.
 *
 *   gmx_exec_register  <- a kernel's operands (KernelSpec has none in the
 *                         reference: kernels.py:95-124 is shape-only)
 *   gmx_exec_launch    <- the execution of a step's dispatches
 *                         (engine.py:359-364, scheduler.py:294-316)
 *
 * Members run at their TRUE dims: coalescing padding is a billing concept of
 * the decision model (coalesce.py:7-8), not materialised on the device.
 *
 * Operand conventions (row-major, leading dims in ELEMENTS):
 *   gemm (m,n,k):  C[m x n] = act(A[m x k] . B[k x n] + bias[m])
 *                  A given as A[m][lda] (K contiguous), B given TRANSPOSED as
 *                  Bt[n][ldb] (K contiguous: the NHWC im2col layout), C[m][ldc].
 *                  bf16 in (tcgen05 kind::f16) or fp32 in (kind::tf32: fp32-labelled
 *                  GEMMs), fp32 accumulate in TMEM, bf16 or fp32 out. lda, ldb rows
 *                  multiples of 16 bytes; pointers 16-byte aligned (TMA).
 *   gemv (m,n):    y[m] = act(W[m x n] . x[n] + bias[m]); W[m][lda]; fp32 or bf16 (W
 *                  streamed as 2D TMA tensor boxes when W rows and x are 16-byte aligned).
 *   elementwise n: y[i] = act(x[i] + bias?) ; x, y contiguous; fp32 or bf16.
 * All device pointers are caller-owned (torch tensors); the executor owns its
 * descriptor table, plans, and split-K workspace. Launches are asynchronous on
 * the caller's stream; one executor handle must not be launched from two
 * streams concurrently (shared split-K workspace). Not thread-safe.
 */
#ifndef GMX_EXEC_H
#define GMX_EXEC_H

#include <stdint.h>

#include "gmx_core.h"

#ifdef __cplusplus
extern "C" {
#endif

#define GMX_ST_BF16 0      /* storage dtypes */
#define GMX_ST_F32 1

#define GMX_ACT_NONE 0     /* fused epilogue activation */
#define GMX_ACT_RELU 1
#define GMX_ACT_GELU 2     /* erf form: 0.5 x (1 + erf(x / sqrt 2)) */

typedef struct gmx_exec gmx_exec;

typedef struct gmx_problem_desc {
    int32_t op;            /* GMX_OP_GEMM / GMX_OP_GEMV / GMX_OP_ELEMENTWISE */
    int32_t in_dtype;      /* GMX_ST_*: gemm BF16 (bf16 tensor cores) or F32 (tf32 tensor cores) */
    int32_t out_dtype;     /* GMX_ST_* */
    int32_t activation;    /* GMX_ACT_* */
    int64_t m, n, k;       /* gemm (m,n,k); gemv (m,n,-); elementwise (n,-,-) in m */
    const void* a;         /* gemm A / gemv W / elementwise x */
    int64_t lda;
    const void* b;         /* gemm Bt / gemv x / unused */
    int64_t ldb;
    void* c;               /* output */
    int64_t ldc;
    const float* bias;     /* optional, length m (gemm/gemv); NULL for none */
    int32_t tile_n;        /* gemm: UMMA N of the output tiles, 64 or 128; 0 = automatic (a
                            * measured TuningTable's tile_n, see autotune.py) */
    int32_t _reserved;
} gmx_problem_desc;

typedef struct gmx_plan_stats {
    int32_t grid;               /* CTAs launched (<= SM count, persistent) */
    int32_t n_items;            /* work items in the list */
    int32_t n_gemm_tiles;       /* 128 x BN output tiles (before split-K) */
    int32_t n_split_items;      /* items that are split-K partials */
    int32_t n_gemv_items;
    int32_t n_eltwise_items;
    int32_t cached;             /* 1 if the plan came from the plan cache */
    int32_t _pad;
    int64_t operand_bytes;      /* algorithmic bytes: each operand + result once */
    int64_t tile_load_bytes;    /* bytes the tile loads request (re-reads included) */
    int64_t flops;              /* useful flops of the launch */
    double max_cta_cost;        /* planner's makespan estimate (ns of one SM) */
    double mean_cta_cost;
} gmx_plan_stats;

/* message of the last failed executor call on this thread */
const char* gmx_exec_last_error(void);
int gmx_exec_create(int32_t device, gmx_exec** out);
void gmx_exec_destroy(gmx_exec* ex);
/* number of SMs / persistent CTAs of the device */
int gmx_exec_num_sms(const gmx_exec* ex, int32_t* out);
/* Register one member's operands; returns a slot (encodes its TMA descriptors). */
int gmx_exec_register(gmx_exec* ex, const gmx_problem_desc* desc, int32_t* out_slot);
int gmx_exec_unregister(gmx_exec* ex, int32_t slot);
/* One coalesced persistent launch over `n` registered slots (order irrelevant).
 * Plans (tile list, LPT assignment across SMs, split-K choice) are cached per
 * slot set. `stream` is a cudaStream_t (NULL = legacy default stream). */
int gmx_exec_launch(gmx_exec* ex, const int32_t* slots, int32_t n, void* stream);
/* Same with flags. Launches use programmatic dependent launch (PDL): a step's prologue
 * (barrier init, TMEM alloc, descriptor prefetch) overlaps the previous step's tail.
 * GMX_LAUNCH_INDEPENDENT: no member reads anything the previous launch on this stream
 * writes, so the step also skips griddepcontrol.wait and its CTAs start on SMs as the
 * previous step's CTAs retire (the executor still waits when split-K state could alias). */
#define GMX_LAUNCH_INDEPENDENT 1
/* GMX_LAUNCH_FENCE: members read outputs of earlier steps whose completion the caller already
 * OBSERVED (wall-clock serving), so no ordering wait is needed, only the generic -> async proxy
 * fence before the step's TMA loads (resident mode). */
#define GMX_LAUNCH_FENCE 2
/* Hazards are tracked by the executor over the slots: a per-step launch that writes a slot
 * read or written, or reads a slot written, by any launch since the last fully ordered one is
 * itself launched fully ordered (no PDL: it starts after ALL earlier work on the stream); a
 * resident step waits for the last steps that wrote (RAW/WAW) or read (WAR) its slots. Slots
 * may therefore be reused by later requests on one stream; across the streams of a
 * multi-stream caller, reuse needs the earlier user's completion (the wall-clock runtime only
 * launches a member after observing its producers). */
int gmx_exec_launch_ex(gmx_exec* ex, const int32_t* slots, int32_t n, void* stream, int32_t flags);
/* As launch_ex, plus the slots whose OUTPUTS this step's members read (their producers): in
 * resident mode the step then waits only for the steps that last wrote those slots (and for
 * earlier users of its plan/slots), so independent chains overlap; any dependency makes a
 * per-step launch dependent. *step_seq (may be NULL) = the step's queue position in resident
 * mode, else -1. */
int gmx_exec_launch_deps(gmx_exec* ex, const int32_t* slots, int32_t n, const int32_t* dep_slots, int32_t ndep,
                         void* stream, int32_t flags, int64_t* step_seq);
/* Stats of the plan used by the last launch. */
int gmx_exec_last_plan(const gmx_exec* ex, gmx_plan_stats* out);

/* Resident (persistent) mode. begin launches ONE cooperative kernel on `stream` that stays on
 * the GPU; every gmx_exec_launch_ex until end() appends its step to a queue (pinned host ring,
 * relayed to a device ring) instead of launching, so consecutive steps stream through the same
 * smem/TMEM pipelines with no launch gap. Steps run in queue order with bounded skew; a step
 * without GMX_LAUNCH_INDEPENDENT (or reusing a slot/plan of the last 2 steps) waits for all
 * earlier steps. end() queues a stop; the kernel exits after the last step, so later work on
 * `stream` is ordered after every queued step. completed() = longest finished prefix of steps. */
int gmx_exec_resident_begin(gmx_exec* ex, void* stream);
/* hold != 0: the kernel relays no step until gmx_exec_resident_release (or end), so a batch
 * queued meanwhile runs back to back; resident_device_ns then gives the device time from the
 * release to the last step's completion (%globaltimer), i.e. the kernel alone. */
int gmx_exec_resident_begin_ex(gmx_exec* ex, void* stream, int32_t hold);
int gmx_exec_resident_release(gmx_exec* ex);
int gmx_exec_resident_device_ns(gmx_exec* ex, int64_t* ns);
int gmx_exec_resident_end(gmx_exec* ex);
/* After a residency ended (and its stream was synchronized): the dispatcher SM's average clock
 * in MHz from the kernel's start to the stop step (%clock64 / %globaltimer on the device), and
 * that span in ns. Clocks under load without host-side sampling. */
int gmx_exec_resident_sm_clock(gmx_exec* ex, double* mhz, int64_t* span_ns);
int gmx_exec_resident_completed(gmx_exec* ex, int64_t* steps_done);
int gmx_exec_resident_active(const gmx_exec* ex);
/* 1 once resident step `seq` (from gmx_exec_launch_deps) completed on the device, else 0. */
int gmx_exec_resident_step_done(gmx_exec* ex, int64_t seq);
/* A caller-owned stream is about to be destroyed: wait for its work and stop using it for
 * the stream-ordered release of plan memory. */
int gmx_exec_stream_retired(gmx_exec* ex, void* stream);
/* Drop cached plans (e.g. after unregistering many slots). */
int gmx_exec_clear_plans(gmx_exec* ex);
/* Knobs: "max_split" (1 disables split-K), "cache_plans" (0/1), "pdl" (0/1), "trace" (0/1: the kernel
 * stamps %globaltimer per work item: producer start, last UMMA issued, epilogue start, end,
 * then epilogue sub-phases: staging start, staged, barrier, store issued). */
int gmx_exec_set_option(gmx_exec* ex, const char* name, int64_t value);
/* Copy the last traced launch: stamps[8*n_items], items[8*n_items] (raw 32-byte work items),
 * cta_off[grid+1]. Call with capacity 0 to query sizes. With capacity >= n_items + grid, stamps
 * also receives grid rows of per-CTA kernel stamps (entry, prologue done, role loops done, exit;
 * 4 used of 8) after the item rows. Synchronizes the device. */
int gmx_exec_read_trace(const gmx_exec* ex, uint64_t* stamps, int32_t* items, int32_t* cta_off,
                        int32_t capacity, int32_t* n_items, int32_t* grid);

#ifdef __cplusplus
}
#endif
#endif /* GMX_EXEC_H */
