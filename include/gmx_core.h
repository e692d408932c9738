/*
 * gmx_core.h — C ABI of the coalescing decision core (libgmx_core.so).
 *
 * Plain C: pointers, sizes, int status codes; no C++ types or exceptions
 * cross this boundary. The library owns only opaque handles; all arrays are
 * caller-owned unless a function returns a *view* (pointers into
 * handle-owned storage, valid until the next call on the same handle).
 * Handles are single-owner and NOT thread-safe, like the reference's
 * scheduler (gpumux/scheduler.py:19-20).
 *
 * The reference (`gpumux` 0.1.0, pure Python) has no FFI; each entry point
 * below replaces one function of its decision path and cites it as
 * `path:line` under /root/reference/pkg/src/gpumux/. Results are bit-exact
 * against the reference: integer ns, IEEE-754 double arithmetic evaluated in
 * the reference's order, Python int/int true division reproduced with
 * correct rounding, Python int-vs-float comparisons reproduced exactly.
 */
#ifndef GMX_CORE_H
#define GMX_CORE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define GMX_OK 0
#define GMX_EINVAL -1     /* bad argument: maps to Python ValueError        */
#define GMX_ENOTFOUND -2  /* unknown dispatch / kernel id: maps to KeyError */
#define GMX_EOVERFLOW -3  /* arithmetic beyond the supported 127-bit range  */
#define GMX_ESTATE -4     /* call not valid in the handle's current state   */
#define GMX_ECUDA -5      /* CUDA runtime / driver failure (executor only)  */
#define GMX_ENOMEM -6

/* ---- enumerations (codes follow the reference strings' sort order, so
 *      integer comparison == the reference's string comparison) ---------- */
#define GMX_OP_ELEMENTWISE 0 /* kernels.py:21 OP_KINDS */
#define GMX_OP_GEMM 1
#define GMX_OP_GEMV 2
#define GMX_DT_FP16 0        /* kernels.py:22; bf16 storage is billed as "fp16" */
#define GMX_DT_FP32 1
#define GMX_PATH_DENSE 0     /* device.py:56-61 */
#define GMX_PATH_SCALAR 1
#define GMX_POLICY_FIFO 0    /* scheduler.py:35 POLICY_VARIANTS */
#define GMX_POLICY_EDF 1
#define GMX_POLICY_OOO 2
#define GMX_POLICY_TIME_MUX 3
#define GMX_POLICY_SPACE_MUX 4
#define GMX_CONTEXT_JIT (-2) /* context id "jit" of coalesced dispatches (scheduler.py:450) */

/* ---- plain records ----------------------------------------------------- */
typedef struct gmx_profile {            /* device.py:33-61 DeviceProfile */
    int64_t sm_count;
    int64_t blocks_per_sm;
    double peak_flops_dense;
    double peak_flops_scalar;
    double mem_bandwidth;
    int64_t context_switch_cost;
} gmx_profile;

typedef struct gmx_policy_params {      /* scheduler.py:39-58 PolicyParams */
    double pad_budget;
    double max_delay_fraction;
    double straggler_threshold;
    int64_t eviction_window;
    int64_t eviction_min_samples;
    double jitter_width;
    int64_t stagger_horizon;
    double duration_noise;
} gmx_policy_params;

typedef struct gmx_tuning_config {      /* tuning.py:32-45 TuningConfig */
    int64_t tile_m;
    int64_t tile_n;
    double sm_footprint;
    double efficiency_factor;
} gmx_tuning_config;

typedef struct gmx_kernel_desc {        /* kernels.py:95-124 KernelSpec */
    int64_t kernel_id;
    int32_t stream;                     /* interned stream id (gmx_sched_intern_stream) */
    int32_t op;                         /* GMX_OP_* */
    int32_t dtype;                      /* GMX_DT_* */
    int32_t ndims;                      /* 3 gemm, 2 gemv, 1 elementwise */
    int64_t dims[3];
    int64_t arrival;
    int64_t deadline;
} gmx_kernel_desc;

typedef struct gmx_cost {               /* device.py:64-70 CostEstimate */
    int64_t flops;
    int64_t bytes;
    int64_t block_count;
    double efficiency;
    int64_t duration;                   /* ns */
} gmx_cost;

/* ---- errors ----------------------------------------------------------- */
const char* gmx_last_error(void);       /* thread-local message of the last failure */
int gmx_core_version(void);

/* ---- L2/L1 cost model -------------------------------------------------- */
/* kernels.py:34-54 validate_dims + flop_count */
int gmx_flop_count(int32_t op, const int64_t* dims, int32_t ndims, int64_t* out);
/* kernels.py:57-69 bytes_moved */
int gmx_bytes_moved(int32_t op, const int64_t* dims, int32_t ndims, int32_t dtype, int64_t* out);
/* kernels.py:202-213 block_count */
int gmx_block_count(int32_t op, const int64_t* dims, int32_t ndims, int64_t tile_m,
                    int64_t tile_n, int64_t* out);
/* device.py:130-137 occupancy_efficiency */
int gmx_occupancy_efficiency(const gmx_profile* p, int64_t block_count, double factor,
                             double* out);
/* device.py:140-150 roofline_duration */
int gmx_roofline_duration(const gmx_profile* p, int64_t flops, int64_t nbytes,
                          double efficiency, int32_t path, int64_t* out);
/* kernels.py:216-222 kernel_cost */
int gmx_kernel_cost(const gmx_profile* p, const gmx_kernel_desc* k,
                    const gmx_tuning_config* cfg, gmx_cost* out);

/* ---- L3 tuning table (lookup side only; tuning.py:147-191) ------------- */
typedef struct gmx_tuning_table gmx_tuning_table;
int gmx_tuning_table_create(gmx_tuning_table** out);
void gmx_tuning_table_destroy(gmx_tuning_table* t);
/* tuning.py:155-156 TuningTable.put */
int gmx_tuning_table_put(gmx_tuning_table* t, int32_t op, int32_t dtype, const int64_t* dims,
                         int32_t ndims, int64_t tenancy, const gmx_tuning_config* cfg);
/* tuning.py:152-160 lookup_or_default: *found = 0 and the 64x64 default on a miss */
int gmx_tuning_table_lookup(const gmx_tuning_table* t, int32_t op, int32_t dtype,
                            const int64_t* dims, int32_t ndims, int64_t tenancy,
                            gmx_tuning_config* out, int32_t* found);

/* ---- L4 coalescer ------------------------------------------------------ */
/* coalesce.py:56-66 _padding_waste / pad_cost */
int gmx_padding_waste(int32_t op, const int64_t* member_flops, int32_t n,
                      const int64_t* padded_dims, int32_t ndims, double* out);
/* coalesce.py:69-106 cluster_shapes.
 * Outputs (caller-allocated, capacity n each; offsets n+1; padded 3*n):
 *   out_members[]  indices into `pending`, cluster by cluster, admission order
 *   out_offsets[c] start of cluster c in out_members (out_offsets[nc] == n)
 *   out_padded[3c..3c+ndims) padded dims; out_waste[c] pad_cost */
int gmx_cluster_shapes(const gmx_kernel_desc* pending, int32_t n, double pad_budget,
                       int32_t* out_members, int32_t* out_offsets, int64_t* out_padded,
                       double* out_waste, int32_t* out_num_clusters);
/* coalesce.py:109-131 form_superkernel (cost part; `table` may be NULL) */
int gmx_form_superkernel(const gmx_profile* p, const gmx_tuning_table* table, int32_t op,
                         int32_t dtype, const int64_t* padded_dims, int32_t ndims,
                         int64_t batch, int64_t co_tenancy, gmx_cost* out);

/* ---- L5 scheduler state machine --------------------------------------- */
typedef struct gmx_sched gmx_sched;

typedef struct gmx_dispatch_rec {       /* scheduler.py:81-96 Dispatch */
    int64_t dispatch_id;
    int64_t start;
    int64_t end;
    int64_t useful_flops;
    int64_t padded_flops;
    int64_t predicted_duration;
    int64_t duration;
    int32_t sm_allocation;
    int32_t context;                    /* stream id, or GMX_CONTEXT_JIT */
    int32_t ctx_switch;
    int32_t infeasible;
    int32_t is_super;                   /* super_id = "sk-" + "-".join(kernel ids) */
    int32_t kernel_offset;              /* into the view's kernel_ids */
    int32_t n_kernels;
    int32_t _pad;
} gmx_dispatch_rec;

typedef struct gmx_step_view {          /* scheduler.py:320 step() return */
    int32_t n_dispatches;
    const gmx_dispatch_rec* dispatches;
    const int64_t* dispatch_kernel_ids;
    int32_t n_withheld;
    const int32_t* withheld_offsets;    /* n_withheld + 1 */
    const int64_t* withheld_kernel_ids;
    int32_t has_wakeup;
    int64_t wakeup;
} gmx_step_view;

typedef struct gmx_complete_view {      /* scheduler.py:210-235 complete() */
    gmx_dispatch_rec dispatch;
    const int64_t* kernel_ids;
    int32_t n_finished;
    const int64_t* finished_request_ids;
    int32_t n_unlocked;                 /* kernels moved blocked -> ready, in order */
    const int64_t* unlocked_kernel_ids;
} gmx_complete_view;

typedef struct gmx_evict_view {         /* scheduler.py:256-278 evict_straggler() */
    int32_t n_cancelled;
    const int64_t* cancelled_dispatch_ids;
    int32_t n_evicted;
    const int64_t* evicted_request_ids; /* sorted */
    int32_t n_dropped;                  /* kernels removed from ready/blocked */
    const int64_t* dropped_kernel_ids;
} gmx_evict_view;

/* scheduler.py:137-163. `table` is copied (may be NULL); footprint model
 * constants come from the tuning model (presets.json tuning_model);
 * jitter_state is the SplitMix64 state (rng.py:19-35). */
int gmx_sched_create(const gmx_profile* p, int32_t policy, const gmx_policy_params* params,
                     const gmx_tuning_table* table, double footprint_base,
                     double footprint_slope, uint64_t jitter_state, gmx_sched** out);
void gmx_sched_destroy(gmx_sched* s);
/* Stream ids are strings in the reference; the core interns them. Ordering
 * of stream names is byte order (== Python str order for UTF-8). */
int gmx_sched_intern_stream(gmx_sched* s, const char* name, int32_t* out_id);
/* scheduler.py:167-187 add_request. kernels[i].deps are given as a CSR:
 * dep_ids[dep_offsets[i] .. dep_offsets[i+1]). out_predicted[i] = solo
 * prediction; *accepted = 0 when the stream was evicted. */
int gmx_sched_add_request(gmx_sched* s, int64_t request_id, int32_t stream, int64_t arrival,
                          const gmx_kernel_desc* kernels, int32_t n, const int64_t* dep_ids,
                          const int32_t* dep_offsets, int64_t* out_predicted,
                          int32_t* accepted);
/* scheduler.py:320-454 step */
int gmx_sched_step(gmx_sched* s, int64_t now, gmx_step_view* out);
/* scheduler.py:210-235 complete; GMX_ENOTFOUND for an unknown dispatch id */
int gmx_sched_complete(gmx_sched* s, int64_t dispatch_id, int64_t now, gmx_complete_view* out);
/* Serving loops: drop finished requests from the scheduler's tables once they outnumber the
 * live ones (decisions are unchanged; finished kernels can no longer be queried by id and kernel
 * ids must not be reused). Off by default: the reference keeps everything (scheduler.py:150-163). */
int gmx_sched_set_retire(gmx_sched* s, int32_t on);
/* Kernels currently ready (dependencies met, not dispatched). A step with none dispatches and
 * withholds nothing under every policy, so a serving loop may skip it. */
int32_t gmx_sched_ready_count(const gmx_sched* s);
/* complete() with the observed duration in the straggler window (ratio = measured / predicted)
 * instead of the dispatch's modeled one; measured_ns < 0 is plain complete(). */
int gmx_sched_complete_measured(gmx_sched* s, int64_t dispatch_id, int64_t now, int64_t measured_ns,
                                gmx_complete_view* out);
/* scheduler.py:237-254 find_stragglers(): stream codes in stream-id order; *n = how many (only the
 * first `cap` are written). The engine evicts each with gmx_sched_evict_stream. */
int gmx_sched_find_stragglers(gmx_sched* s, int32_t* streams, int32_t cap, int32_t* n);
/* scheduler.py:256-278 evict_straggler */
int gmx_sched_evict_stream(gmx_sched* s, int32_t stream, int64_t now, gmx_evict_view* out);
/* scheduler.py:195-206 */
int gmx_sched_predicted_remaining(const gmx_sched* s, int64_t kernel_id, int64_t* out);
int gmx_sched_kernel_slack(const gmx_sched* s, int64_t kernel_id, int64_t now, int64_t* out);
int gmx_sched_free_sms(const gmx_sched* s, int64_t* out);
int gmx_sched_set_free_sms(gmx_sched* s, int64_t value);
int gmx_sched_num_ready(const gmx_sched* s, int64_t* out);
int gmx_sched_jitter_state(const gmx_sched* s, uint64_t* out);
int gmx_sched_set_jitter_state(gmx_sched* s, uint64_t state);

#ifdef __cplusplus
}
#endif
#endif /* GMX_CORE_H */
