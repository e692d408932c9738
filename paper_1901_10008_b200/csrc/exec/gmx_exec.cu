// gmx_exec.cu — coalesced persistent executor for sm_100a (B200) behind include/gmx_exec.h.
//
// One launch per scheduler step. The launch's work list spans every member of every
// superkernel the OoO scheduler dispatched in that step (gpumux/scheduler.py:414-454 decides
// WHAT runs together; this file is HOW it runs on the device):
//
//   GEMM items   128 x BN output tiles (BN in {32..128}), K streamed in 64-element blocks:
//                TMA (SWIZZLE_128B) -> 6-stage smem ring -> tcgen05.mma (M=128, fp32 accumulate
//                in TMEM, double-buffered accumulators) -> tcgen05.ld epilogue with fused bias +
//                activation -> bf16/fp32 stores. Long-K tiles are split along K; partials are
//                added into an fp32 L2 workspace (red.global.add, arrival order: NOT bitwise
//                deterministic run to run; option max_split=1 is) and the last-arriving split
//                finalizes. The side needing fewer tile loads goes on UMMA-M ("role swap").
//   GEMV items   row blocks of y = W x, streamed with 16-byte non-allocating loads.
//   Eltwise      vectorised y = act(x) ranges.
//
// Warp roles (6 warps per step launch, 8 resident; 1 CTA per SM, grid <= #SMs):
//   warp 0  TMA producer (warp-wide, one elected lane issues)
//   warp 1  TMEM owner + UMMA issuer (warp-wide, one elected lane issues)
//   warps 2-5  epilogue: TMEM -> registers -> global, and the CUDA-core GEMV / eltwise items.
// Each role walks the same per-CTA item list; only the roles an item needs act on it.
//
// Host side: operand registration encodes the TMA descriptors once (tensor maps live in a
// device-resident problem table); a per-slot-set plan (tile list, split-K choice, LPT
// assignment of items to CTAs) is built once and cached, so a recurring step costs one
// kernel launch.

#include "../../../include/gmx_exec.h"
#include "sm100_ptx.cuh"
#include "../core/flatmap.hpp"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstddef>
#include <cstdlib>
#include <map>
#include <memory>
#include <numeric>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

namespace gmx {

// ------------------------------------------------------------------ device-side types

enum : int32_t { kItemGemm = 0, kItemGemv = 1, kItemEltwise = 2 };
// WorkItem.type flag: a GEMM item over fp32 operands, run as tcgen05.mma kind::tf32 (32-element
// K blocks: the same 128-byte swizzle rows as 64 bf16, so ring stages and UMMA descriptors are shared)
constexpr uint8_t kItemTf32 = 0x40;
__host__ __device__ __forceinline__ int item_kind(uint8_t t) { return t & 0x3f; }

constexpr int kThreads = 256;             // 6 role warps + queue dispatcher / accountant + list scheduler (resident)
constexpr int kThreadsPerStep = 192;      // per-step launches: the 6 role warps only (warps 6-7 are resident-only)
constexpr int kInlineMaxMembers = 32;   // members of an inline (device-enumerated) step
constexpr size_t kSeenSlots = 4096;     // slot-set sighting counters (inline promotion)
constexpr int kInlineMaxItems = 48;     // work items one CTA may hold in an inline step
constexpr int kInlineGemvRows = 64;     // inline GEMV item: rows
constexpr int kInlineEltwise = 32768;   // inline elementwise item: elements

// Two build shapes of the same kernel (selected per executor, option "ctas_per_sm"):
//   1 CTA/SM : 6-stage ring, 32 KB output staging (one resident CTA streams alone)
//   2 CTAs/SM: 3-stage ring each, 16 KB staging; two CTAs (of one launch, or of consecutive
//              launches) share an SM, so one's epilogue / pipeline fill overlaps the other's loads
template <int kCtasPerSm>
struct SmemCfg {
    static constexpr int stages = kCtasPerSm == 1 ? 6 : 3;          // 32 KB stages (A 16 KB + B <= 16 KB)
    static constexpr int stage_out = kCtasPerSm == 1 ? 32 * 1024 : 16 * 1024;
    static constexpr int align_pad = kCtasPerSm == 1 ? 1024 : 0;   // 2/SM: base must already be aligned
    static constexpr int acc_bufs = kCtasPerSm == 1 ? 4 : 2;        // TMEM accumulators (128 cols each)
    static constexpr int tmem_cols = acc_bufs * 128;                // 512 per SM either way
    static constexpr int stage_bufs = kCtasPerSm == 1 ? 2 : 1;      // output staging ping-pong
    static constexpr int unit_q = kCtasPerSm == 1 ? 8 : 1;          // resident work units (1-CTA shape only)
};
constexpr int kTileRows = 128;             // UMMA M
constexpr int kBlockK = 64;                // 64 bf16 = 128 B = one swizzle atom row (32 fp32 for tf32 items)
__host__ __device__ __forceinline__ int kblock_elems(bool tf32) { return tf32 ? kBlockK / 2 : kBlockK; }
// UMMA N <= 128. (N = 256 would load the rows operand once per 256 columns — 19% fewer C2 tile
// bytes — but its 48 KB stages leave room for only 4 in the ring, and the lost bytes in flight
// cost more than the saved loads: 7.9 vs 7.1 us per C2 step, measured.)
constexpr int kMaxBN = 128;
constexpr int kStageA = kTileRows * kBlockK * 2;   // 16 KB
constexpr int kStageB = kMaxBN * kBlockK * 2;      // 16 KB
constexpr int kStageBytes = kStageA + kStageB;
// GEMV W streamed through the TMA ring as 2D TENSOR tiles (a 1D bulk copy moves ~30 GB/s per
// SM, a tensor box ~3x that): a stage is two {256-element x R-row} boxes side by side (R = 16
// fp32 / 32 bf16 rows, 16 KB per box), i.e. R rows x 512 columns; an item is a whole number of
// R-row blocks, each block one stage per 512 columns. Problems whose W / x cannot be described
// by a tensor map (16-byte alignment) stream rows with 16-byte loads instead (gemv_rows).
constexpr int kGvBoxCols = 256;
constexpr int kGvStageCols = 2 * kGvBoxCols;
__host__ __device__ constexpr int gv_box_rows(bool f32) { return f32 ? 16 : 32; }
__host__ __device__ __forceinline__ int gv_stages(int rows, int cols, bool f32) {
    const int R = gv_box_rows(f32);
    return ((rows + R - 1) / R) * ((cols + kGvStageCols - 1) / kGvStageCols);
}

template <int kCtasPerSm>
constexpr int smem_bytes() {
    using C = SmemCfg<kCtasPerSm>;
    return C::stages * kStageBytes + C::stage_out + C::align_pad + C::unit_q * 192 /*unit ring*/ + 512 /*barriers*/;
}
static_assert(2 * (smem_bytes<2>() + 1024) <= 233472, "two CTAs must fit one SM's shared memory");
constexpr int kMaxGrid = 512;              // upper bound of a launch's grid (2 x SMs), trace rows
constexpr int kWsBlock = 4096;             // split-K workspace allocation unit (floats)

struct alignas(64) DevProblem {
    CUtensorMap tm_rows;     // operand on the UMMA-M side (128-row boxes)
    CUtensorMap tm_cols;     // operand on the UMMA-N side (BN-row boxes)
    CUtensorMap tm_out;      // output C[m][n]: 128-byte-wide boxes, SWIZZLE_128B (if tma_out)
    void* out;
    const void* in0;         // gemv W / eltwise x
    const void* in1;         // gemv x
    const float* bias;
    int64_t ld_out;
    int64_t ld_in0;
    int32_t kind;            // kItem*
    int32_t swap;            // gemm: rows side is n (Bt), cols side is m (A)
    int32_t rows;            // gemm: extent on the M side; gemv: m; eltwise: count
    int32_t cols;            // gemm: extent on the N side; gemv: n
    int32_t K;
    int32_t bn;
    int32_t act;
    int32_t in_dt;
    int32_t out_dt;
    int32_t kblocks;
    int32_t tma_out;         // 1: epilogue stages the tile in smem and TMA-stores it
    int32_t _pad[5];
};
static_assert(sizeof(DevProblem) % 64 == 0, "DevProblem must keep 64-byte tensor map alignment");

struct WorkItem {
    int32_t problem;
    uint8_t type;
    uint8_t nsplit;
    uint8_t split;
    uint8_t bn;              // gemm: the problem's UMMA N (64 / 128)
    int32_t row0;            // gemm: M-side origin; gemv: first row; eltwise: first element
    int32_t col0;            // gemm: N-side origin; gemv: end row;  eltwise: end element
    int32_t kb0, kb1;        // gemm: k-block range of this (split) item
    int32_t tile_slot;       // split-K: arrival counter index
    int32_t ws_blk;          // split-K: workspace offset in kWsBlock units
};
static_assert(sizeof(WorkItem) == 32, "WorkItem layout");

// ---- resident mode: one persistent launch consumes a queue of steps ----------------------
// The host appends StepDescs to a ring in pinned, device-mapped host memory and publishes a
// count; one dispatcher lane (block 0) copies each new descriptor into a device-memory ring and
// publishes it there, so the 2 x #SM role leaders poll L2, not PCIe. Steps run back to back
// through the same smem/TMEM pipelines: the producer streams step k+1's tiles while the
// epilogue drains step k. Each CTA counts its finish of a step into a monotonic per-slot
// counter; a step may start only when step k - kWindow has completed everywhere (bounded
// skew, so split-K state and outputs of a plan reused kWindow+ steps later are free), and a
// step flagged `wait_all` (dependent members, or slots/plans reused inside the window) waits
// for every earlier step.
constexpr int kQueue = 1024;  // ring slots (host and device)
constexpr int kMaxWindow = 512;   // max steps a CTA may run ahead of the slowest (option, <= this; < kQueue)

struct StepDesc {
    const DevProblem* probs;
    const WorkItem* items;
    const int32_t* cta_off;   // cta_off[grid + 1] (items of CTA c: [cta_off[c], cta_off[c + 1]))
    float* ws;
    int32_t* counters;
    int32_t grid;             // CTAs holding items in this step (<= gridDim.x)
    int32_t wait_all;         // a member depends on earlier outputs of unknown steps: all first
    int32_t stop;             // bit 0: stop entry; bit 1: the plan is still being uploaded — wait for
                              // DevQueue::plan_ready[slot] == seq + 1 (copy-engine stream write)
    int32_t nwait;            // entries of wait_steps in use
    int64_t wait_steps[4];    // earlier steps that must be complete first: producers of this
                              // step's inputs, users of its plan (split-K state) or slots (outputs)
    int32_t inline_n;         // > 0: inline step (no plan): items enumerated from these slots
    int32_t inline_slots[kInlineMaxMembers];
    int32_t _pad[9];
};
static_assert(sizeof(StepDesc) == 256, "StepDesc layout");
static_assert(offsetof(StepDesc, inline_n) < 96 && offsetof(StepDesc, inline_slots) == 92,
              "the dispatcher relays a 96-byte head that includes inline_n");

struct DevQueue {
    StepDesc ring[kQueue];
    int64_t published;        // steps available in `ring` (dispatcher -> role leaders)
    uint64_t t_first;         // %globaltimer when step 0 was relayed (after a held start's release)
    uint64_t t_last;          // %globaltimer of the latest step completion
    uint64_t t_relay;         // %globaltimer of the dispatcher's latest relay
    uint64_t t_stop;          // %globaltimer when the dispatcher relayed the stop entry
    uint64_t c_first;         // dispatcher SM's %clock64 at t_first / t_stop: the SM clock over
    uint64_t c_stop;          // the residency, measured on the device (no host-side sampling)
    int64_t _pad[1];
    uint32_t done[kQueue];    // monotonic count of item lists finished, per slot
    uint32_t grab[kQueue];    // monotonic list-grab counter, per slot (2 x grid per step)
    uint32_t plan_ready[kQueue];   // seq + 1 once a plan uploaded during the residency has landed
};

struct KernelArgs {
    const DevProblem* probs;
    const WorkItem* items;
    const int32_t* cta_off;
    const int32_t* cta_flags;
    float* ws;
    int32_t* counters;
    uint64_t* trace;         // optional: 8 globaltimer stamps per item (debug/profiling)
    int32_t dbg;             // experiment flags (reserved)
    int32_t independent;     // 1: no data dependency on the previous launch (skip griddepcontrol.wait)
    int32_t early_trigger;   // 1: let the next launch start as soon as all our CTAs are resident
    int32_t resident;        // 1: persistent: steps come from the queue below, not the fields above
    DevQueue* dq;
    const StepDesc* hring;   // host-mapped ring + published count (resident mode)
    const int64_t* hpub;
    int64_t* hdone;          // host-mapped: step seq + 1 written when a slot's step completed
    int32_t window;          // resident: max steps a CTA may run ahead of the slowest
    int32_t grab_ahead;      // resident: units the list scheduler may keep ahead of the producer
                             // before it grabs another list of the same step
    uint64_t* rtrace;        // resident diagnostics: 4 stamps per (step, CTA), or null
    int32_t rtrace_steps;
    // inline step (no host plan): the members' work items are enumerated on the device, item
    // g of the concatenated tile space going to CTA g % gridDim.x (no split-K, no LPT)
    int32_t inline_n;
    int32_t inline_slots[kInlineMaxMembers];
};

// The items/tables one step works on, as seen by one CTA.
// Profiling build (-DGMX_INSTR, tools/instr_resident.py): per-CTA cycles each role spends
// waiting on its inputs, dumped at the stop into the last two rtrace rows.
enum InstrCounter { kIPUnit, kIPEmpty, kIMUnit, kIMTempty, kIMFull, kIEUnit, kIETfull, kISUempty, kISPub, kISOrder,
                    kISLists, kIPStages, kIEStaged, kIESplit, kIEComplete, kIEAcct, kIABar, kIAWait, kIARed, kIXNext, kIXLd, kIXStage, kIXBar2, kIXIssue, kICount };
[[maybe_unused]] constexpr int kInstrRows = (kICount + 7) / 8;
#ifdef GMX_INSTR
#define GMX_INSTR_INC(i) (++ic[i])
#else
#define GMX_INSTR_INC(i) ((void)0)
#endif
template <typename W>
__device__ __forceinline__ void timed(long long* ic, int i, bool on, W&& w) {
#ifdef GMX_INSTR
    const long long t0 = clock64();
    w();
    if (on) ic[i] += clock64() - t0;
#else
    w();
#endif
}
__device__ __forceinline__ void instr_dump(const KernelArgs& a, const long long* ic, int f0, int f1) {
#ifdef GMX_INSTR
    if (a.rtrace && a.rtrace_steps >= kInstrRows) {
        uint64_t* o = a.rtrace + (int64_t)(a.rtrace_steps - kInstrRows) * gridDim.x * 8;
        for (int f = f0; f < f1; ++f) o[(f / 8) * gridDim.x * 8 + blockIdx.x * 8 + f % 8] = (uint64_t)ic[f];
    }
#endif
}

struct StepView {
    const DevProblem* probs;
    const WorkItem* items;
    float* ws;
    int32_t* counters;
    int beg, end;
    bool stop;
    // inline step: list `idx` holds the members' virtual items g with g % G == idx
    int inl_n;
    const int32_t* inl_slots;
    int idx;
    uint32_t G;
    int ibase;   // items[i - ibase] is item i (a resident unit's items live in shared memory)
};

// Walks one list's work items: a planned list's array, or an inline step's virtual items
// (each member's 128 x BN tiles / 64-row GEMV blocks / 32K-element chunks, concatenated).
// Apply f(item, index) to every work item of a list; the planned-array and inline paths are
// separate instantiations of f, so a planned list pays nothing for the inline enumeration.
struct ItemCursor;
__device__ __forceinline__ ItemCursor item_begin(const StepView& v);
__device__ __forceinline__ bool next_item(const StepView& v, ItemCursor& c, WorkItem& it);
template <typename F, typename D>
__device__ __forceinline__ void for_each_item(const StepView& v, F&& f, D&& done_reading);

struct ItemCursor {
    int i;        // planned: next index
    int m, u;     // inline: member, unit within member
    uint32_t g;   // inline: global virtual item index
};
__device__ __forceinline__ ItemCursor item_begin(const StepView& v) { return ItemCursor{v.beg, 0, 0, 0u}; }
__device__ __forceinline__ bool next_item(const StepView& v, ItemCursor& c, WorkItem& it) {
    if (v.inl_n == 0) {
        if (c.i >= v.end) return false;
        it = v.items[c.i++];
        return true;
    }
    while (c.m < v.inl_n) {
        const int32_t slot = v.inl_slots[c.m];
        const DevProblem* P = v.probs + slot;
        const int kind = P->kind, rows = P->rows;
        int units, per_row = 1;
        if (kind == kItemGemm) {
            per_row = (P->cols + P->bn - 1) / P->bn;
            units = ((rows + kTileRows - 1) / kTileRows) * per_row;
        } else if (kind == kItemGemv) {
            units = (rows + kInlineGemvRows - 1) / kInlineGemvRows;
        } else {
            units = (rows + kInlineEltwise - 1) / kInlineEltwise;
        }
        while (c.u < units) {
            const uint32_t gg = c.g++;
            const int u = c.u++;
            if (gg % v.G != (uint32_t)v.idx) continue;
            it.problem = slot;
            it.type = (uint8_t)kind | (kind == kItemGemm && P->in_dt == GMX_ST_F32 ? kItemTf32 : 0);
            it.nsplit = 1;
            it.split = 0;
            it.bn = (uint8_t)P->bn;
            it.kb0 = 0;
            it.tile_slot = -1;
            it.ws_blk = 0;
            if (kind == kItemGemm) {
                it.row0 = (u / per_row) * kTileRows;
                it.col0 = (u % per_row) * P->bn;
                it.kb1 = P->kblocks;
            } else if (kind == kItemGemv) {
                it.row0 = u * kInlineGemvRows;
                it.col0 = min(rows, it.row0 + kInlineGemvRows);
                // ring stages (0: unstaged); P->bn = 1 when W has its tensor map
                it.kb1 = P->bn ? gv_stages(it.col0 - it.row0, P->cols, P->in_dt == GMX_ST_F32) : 0;
            } else {
                it.row0 = u * kInlineEltwise;
                it.col0 = min(rows, it.row0 + kInlineEltwise);
                it.kb1 = 0;
            }
            return true;
        }
        ++c.m;
        c.u = 0;
    }
    return false;
}

// `done_reading()` runs once the last item was read, before it is processed: a resident
// consumer releases its shared-memory unit there, so the list scheduler can refill the slot
// while the consumer still works on the list's last item.
template <typename F, typename D>
__device__ __forceinline__ void for_each_item(const StepView& v, F&& f, D&& done_reading) {
    if (v.inl_n == 0) {
        if (v.beg >= v.end) done_reading();
        for (int i = v.beg; i < v.end; ++i) {
            const WorkItem it = v.items[i - v.ibase];
            if (i + 1 == v.end) done_reading();
            f(it, i);
        }
    } else {
        ItemCursor c = item_begin(v);
        WorkItem it;
        while (next_item(v, c, it)) f(it, -1);
        done_reading();
    }
}

__device__ __forceinline__ int64_t ld_acquire_gpu_s64(const int64_t* p) {
    int64_t v;
    asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int64_t ld_acquire_sys_s64(const int64_t* p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Spin (with backoff) until the step in `slot` of round `round` (= seq / kQueue) was finished
// by all `nctas` CTAs. A watchdog turns a protocol bug into a launch error instead of a hang.
__device__ __forceinline__ void wait_step_done(const DevQueue* q, int64_t seq, uint32_t nctas) {
    if (seq < 0) return;
    const uint32_t need = nctas * (uint32_t)(seq / kQueue + 1);
    const uint32_t* c = &q->done[seq % kQueue];
    if ((int32_t)(ld_acquire_gpu_u32(c) - need) >= 0) return;
    const uint64_t t0 = global_timer_ns();
    while ((int32_t)(ld_acquire_gpu_u32(c) - need) < 0) {
        __nanosleep(64);
        if (global_timer_ns() - t0 > 8000000000ull) __trap();
    }
}

// GELU (erf form) out of line: erff inlined at every activation site made up over a quarter of
// the kernel's SASS, spreading the hot code (instruction-cache misses were the top stall)
__device__ __noinline__ float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

__device__ __forceinline__ float apply_act(float x, int32_t act) {
    if (act == GMX_ACT_RELU) return fmaxf(x, 0.0f);
    if (act == GMX_ACT_GELU) return gelu_erf(x);
    return x;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void store_one(void* out, int64_t idx, int32_t dt, float v) {
    if (dt == GMX_ST_BF16)
        reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
    else
        reinterpret_cast<float*>(out)[idx] = v;
}

// Epilogue parameters copied out of the (global) problem descriptor once per item so the
// compiler keeps them in registers: stores to the output may alias global memory, so reading
// DevProblem fields inside the store loops would re-load them after every store.
struct EpiParams {
    void* out;
    const float* bias;
    const CUtensorMap* tm_out;
    int64_t ld_out;
    int32_t swap, rows, cols, bn, act, out_dt, tma_out;
};

__device__ __forceinline__ EpiParams load_epi(const DevProblem* P) {
    EpiParams e;
    e.tm_out = &P->tm_out;
    e.tma_out = P->tma_out;
    e.out = P->out;
    e.bias = P->bias;
    e.ld_out = P->ld_out;
    e.swap = P->swap;
    e.rows = P->rows;
    e.cols = P->cols;
    e.bn = P->bn;
    e.act = P->act;
    e.out_dt = P->out_dt;
    return e;
}


// bias + activation over one 32-column accumulator chunk, with every branch hoisted out of
// the (fully unrolled) element loops: the epilogue runs one warp per SMSP, so per-element
// control flow would be paid at full latency.
//   non-swap: the chunk is one output row m (bias[m] scalar)
//   swap:     the chunk is 32 output rows m0..m0+31 (bias per element)
__device__ __forceinline__ void transform_chunk(float (&v)[32], const EpiParams& E, int m, bool swap) {
    if (E.bias) {
        if (!swap) {
            const float b = m < E.rows ? __ldg(E.bias + m) : 0.0f;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += b;
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (m + j < E.cols) ? __ldg(E.bias + m + j) : 0.0f;
        }
    }
    if (E.act == GMX_ACT_RELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
    } else if (E.act == GMX_ACT_GELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
    }
}

// Write 32 accumulator columns of the thread's tile row to the output.
__device__ __forceinline__ void store_tile_chunk(const EpiParams& E, int row0, int col0, int trow, int c,
                                                 float (&v)[32]) {
    const int gr = row0 + trow;                     // M-side index
    if (gr >= E.rows) return;
    const int gc0 = col0 + c * 32;                  // N-side index of v[0]
    const int nvalid = min(32, E.cols - gc0);
    if (nvalid <= 0) return;
    transform_chunk(v, E, E.swap ? gc0 : gr, E.swap);
    if (!E.swap) {
        // gr = m (output row), columns = n: contiguous in memory
        const int64_t base = (int64_t)gr * E.ld_out + gc0;
        if (E.out_dt == GMX_ST_BF16) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(E.out) + base;
            if (nvalid == 32 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
                uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    o4[q] = make_uint4(pack_bf16x2(v[8 * q + 0], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                                       pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
                return;
            }
        } else {
            float* o = reinterpret_cast<float*>(E.out) + base;
            if (nvalid == 32 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
                float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
                for (int q = 0; q < 8; ++q) o4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                return;
            }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) store_one(E.out, base + j, E.out_dt, v[j]);
    } else {
        // gr = n (output column), columns = m (output rows): lanes write consecutive n
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < nvalid) store_one(E.out, (int64_t)(gc0 + j) * E.ld_out + gr, E.out_dt, v[j]);
    }
}

// ---- staged output: chunk values -> output staging (TMA box layout) -> TMA store ---------
//   non-swap: tile rows = m (128), chunk = 32 n-columns; box {128 B of n, 128 m-rows}
//   swap:     tile rows = n (128), chunk = 32 m-rows;    box {128 B of n, 32 m-rows}
// Staging slots hold 128 x 32 output elements (8 KB bf16 / 16 KB fp32), SWIZZLE_128B.
__device__ __forceinline__ int out_chunks_per_pass(const EpiParams& E, int stage_out) {
    return stage_out / (128 * 32 * (E.out_dt == GMX_ST_BF16 ? 2 : 4));
}

__device__ __forceinline__ void stage_out_chunk(const EpiParams& E, const float (&v)[32], int slot, int trow,
                                                uint32_t stg_u32) {
    const int esz = E.out_dt == GMX_ST_BF16 ? 2 : 4;
    if (!E.swap) {
        const uint32_t row_base = (uint32_t)trow * 128u;
        const uint32_t sw = (uint32_t)(trow & 7);
        if (esz == 2) {
            const uint32_t sub = stg_u32 + (uint32_t)(slot >> 1) * 16384u + row_base;
            const uint32_t h = (uint32_t)(slot & 1) * 4u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                st_shared_v4(sub + (((h + q) ^ sw) << 4), pack_bf16x2(v[8 * q], v[8 * q + 1]),
                             pack_bf16x2(v[8 * q + 2], v[8 * q + 3]), pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                             pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        } else {
            const uint32_t sub = stg_u32 + (uint32_t)slot * 16384u + row_base;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                st_shared_v4(sub + (((uint32_t)q ^ sw) << 4), __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                             __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
        }
    } else {
        // swapped tile: the staging holds 128/inner output boxes of [per_pass x 32 m rows][inner n]
        // (box-major, SWIZZLE_128B rows), so one TMA store per box covers the whole pass
        const int inner = 128 / esz;
        const uint32_t box_bytes = (uint32_t)(16384 / (128 * 32 * esz)) * 4096u;   // per_pass x 32 rows x 128 B
        const uint32_t sb = (uint32_t)(trow / inner);
        const uint32_t byte = (uint32_t)(trow % inner) * (uint32_t)esz;
        const uint32_t base = stg_u32 + sb * box_bytes + (uint32_t)slot * 4096u + (byte & 15u);
        const uint32_t unit = byte >> 4;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t addr = base + (uint32_t)j * 128u + ((unit ^ (uint32_t)(j & 7)) << 4);
            if (esz == 2)
                st_shared_u16(addr, __bfloat16_as_ushort(__float2bfloat16_rn(v[j])));
            else
                st_shared_f32(addr, v[j]);
        }
    }
}

// Output staging ring: `nbuf` buffers of `half` bytes used round-robin, one TMA-store bulk
// group per pass, so a pass only waits for the store issued nbuf passes ago to have read its
// buffer. Every epilogue thread walks the ring identically (uniform control flow).
struct Staging {
    uint8_t* base;
    int half;
    int nbuf;
    uint32_t pass;
    // wait (one thread) until the next buffer is free; the caller then syncs the epilogue warps
    __device__ __forceinline__ uint8_t* next(int etid) {
        if (etid == 0) {
            if (nbuf == 2)
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
                bulk_wait_read0();
        }
        return base + (nbuf == 2 ? (int)(pass & 1u) * half : 0);
    }
    __device__ __forceinline__ void done() { ++pass; }
};

// One thread: TMA-store the staged chunks c0..cend-1 of the tile at (row0, col0).
__device__ __forceinline__ void issue_out_stores(const EpiParams& E, int row0, int col0, int c0, int cend,
                                                 uint8_t* stg) {
    const int esz = E.out_dt == GMX_ST_BF16 ? 2 : 4;
    const int inner = 128 / esz;
    for (int c = c0; c < cend; ++c) {
        const int slot = c - c0;
        if (!E.swap) {
            if (esz == 2) {
                if ((slot & 1) == 0) tma_store_2d(E.tm_out, stg + (slot >> 1) * 16384, col0 + c * 32, row0);
            } else {
                tma_store_2d(E.tm_out, stg + slot * 16384, col0 + c * 32, row0);
            }
        } else if (c == c0) {
            const int box_bytes = (16384 / (128 * 32 * esz)) * 4096;
            for (int sb = 0; sb < 128 / inner; ++sb)
                tma_store_2d(E.tm_out, stg + sb * box_bytes, row0 + sb * inner, col0 + c0 * 32);
        }
    }
    bulk_commit();
}

// Epilogue of an unsplit tile: TMEM chunks -> bias/activation -> staging -> TMA store. The
// accumulator is released to the MMA warp right after its last tcgen05.ld.
__device__ __forceinline__ uint32_t epilogue_staged(const EpiParams& E, int row0, int col0, Staging& S, int trow,
                                                int etid, uint32_t taddr, uint64_t* tempty_bar,
                                                uint64_t* tr = nullptr, long long* ic = nullptr) {
    const int nchunks = E.bn / 32;
    const int per_pass = out_chunks_per_pass(E, S.half);
    const int lane = lane_id();
    uint32_t groups = 0;
    for (int c0 = 0; c0 < nchunks; c0 += per_pass) {
        const int cend = min(nchunks, c0 + per_pass);
        uint8_t* stg;
        timed(ic, kIXNext, true, [&] {
            stg = S.next(etid);   // staging free: the store that last used it has read it
            named_bar_sync(3, 128);
        });
        const uint32_t stg_u32 = smem_u32(stg);
        if (tr && etid == 0 && c0 == 0) tr[4] = global_timer_ns();
        for (int c = c0; c < cend; ++c) {
            float v[32];
            timed(ic, kIXLd, true, [&] { tmem_ld32(taddr + (uint32_t)(c * 32), v); });
            if (c == nchunks - 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty_bar);
            }
            timed(ic, kIXStage, true, [&] {
                transform_chunk(v, E, E.swap ? col0 + c * 32 : row0 + trow, E.swap);
                stage_out_chunk(E, v, c - c0, trow, stg_u32);
            });
        }

        if (tr && etid == 0 && c0 == 0) tr[5] = global_timer_ns();
        timed(ic, kIXBar2, true, [&] {
            fence_async_smem();
            named_bar_sync(3, 128);
        });
        if (tr && etid == 0 && c0 == 0) tr[6] = global_timer_ns();
        if (etid == 0) {
            timed(ic, kIXIssue, true, [&] { issue_out_stores(E, row0, col0, c0, cend, stg); });
            if (tr && c0 == 0) tr[7] = global_timer_ns();
        }
        S.done();
        ++groups;
    }
    return groups;
}

// ---- split-K: partials reduced in L2, completion deferred, last arrival finalizes -----------
// Every split of a tile adds into the same fp32 accumulator tile in an L2-resident workspace,
// blocked [chunk (32 cols)][quad (4 cols)][row (128)][4] so that (a) one warp-wide 16-byte
// reduction covers 512 contiguous bytes and (b) a chunk is one contiguous 16 KB block.
//   1. reduce: TMEM -> registers -> `red.global.add.v4.f32` (no smem, no TMA-engine time, so
//      the producer's loads are not delayed); the TMEM accumulator is released right away.
//   2. complete (deferred until the epilogue warps finished the CTA's NEXT item, so the L2
//      round trip overlaps useful work): every thread fences its reductions, then one acq_rel
//      ticket on the tile counter. The split drawing the last ticket sees all the sums and
//   3. finalizes: bulk-loads the summed chunks into smem, bias/activation, staged TMA store,
//      and re-zeroes the workspace + counter for the next launch of the plan.
// No split ever waits for another CTA, so no placement of items across CTAs (or concurrent
// launches on other streams) can deadlock. fp32 add order is arrival order (within tolerance;
// `max_split=1` is bitwise-stable).

// cp.async.bulk.wait_group takes an immediate: wait until at most n groups are pending.
__device__ __forceinline__ void bulk_wait_upto(uint32_t n) {
    switch (n) {
        case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group 7;" ::: "memory"); break;
    }
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ void split_reduce(const EpiParams& E, float* acc_tile, int trow, uint32_t taddr,
                                             uint64_t* tempty_bar) {
    const int nchunks = E.bn / 32;
    const int lane = lane_id();
    for (int c = 0; c < nchunks; ++c) {
        float v[32];
        tmem_ld32(taddr + (uint32_t)(c * 32), v);
        if (c == nchunks - 1) {   // accumulator free for the next tile's MMAs
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar);
        }
        float* base = acc_tile + ((int64_t)c * 8 * kTileRows + trow) * 4;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            red_add_v4(base + q * kTileRows * 4, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
}

// Last split: summed chunks L2 -> registers (16-byte loads, 512 contiguous bytes per warp
// instruction, two chunks in flight) -> epilogue; re-zero the workspace for the next launch.
__device__ __forceinline__ void ld_sum_chunk(float* acc_tile, int c, int trow, float (&v)[32]) {
    float4* base = reinterpret_cast<float4*>(acc_tile) + (int64_t)c * 8 * kTileRows + trow;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 x = __ldcg(base + q * kTileRows);
        v[4 * q] = x.x;
        v[4 * q + 1] = x.y;
        v[4 * q + 2] = x.z;
        v[4 * q + 3] = x.w;
    }
}
__device__ __forceinline__ void zero_sum_chunk(float* acc_tile, int c, int trow) {
    float4* base = reinterpret_cast<float4*>(acc_tile) + (int64_t)c * 8 * kTileRows + trow;
#pragma unroll
    for (int q = 0; q < 8; ++q) st_global_cg_v4(base + q * kTileRows, make_uint4(0u, 0u, 0u, 0u));
}

__device__ __forceinline__ uint32_t split_finalize(const EpiParams& E, int row0, int col0, float* acc_tile,
                                                  Staging& S, int trow, int etid) {
    const int nchunks = E.bn / 32;
    const int per_pass = out_chunks_per_pass(E, S.half);
    uint32_t groups = 0;
    for (int c0 = 0; c0 < nchunks; c0 += per_pass) {
        const int cend = min(nchunks, c0 + per_pass);
        uint8_t* stg = S.next(etid);   // output staging free
        const uint32_t stg_u32 = smem_u32(stg);
        named_bar_sync(3, 128);
        for (int c = c0; c < cend; c += 2) {
            const bool two = c + 1 < cend;
            float v0[32], v1[32];
            ld_sum_chunk(acc_tile, c, trow, v0);
            if (two) ld_sum_chunk(acc_tile, c + 1, trow, v1);
            zero_sum_chunk(acc_tile, c, trow);
            if (two) zero_sum_chunk(acc_tile, c + 1, trow);
            transform_chunk(v0, E, E.swap ? col0 + c * 32 : row0 + trow, E.swap);
            stage_out_chunk(E, v0, c - c0, trow, stg_u32);
            if (two) {
                transform_chunk(v1, E, E.swap ? col0 + (c + 1) * 32 : row0 + trow, E.swap);
                stage_out_chunk(E, v1, c + 1 - c0, trow, stg_u32);
            }
        }
        fence_async_smem();
        named_bar_sync(3, 128);
        if (etid == 0) issue_out_stores(E, row0, col0, c0, cend, stg);
        S.done();
        ++groups;
    }
    return groups;
}

template <typename T>
__device__ __forceinline__ float load_f(const T* p);
template <>
__device__ __forceinline__ float load_f<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float load_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

__device__ __forceinline__ float dot_v4(uint4 w, uint4 x, float) {
    return __uint_as_float(w.x) * __uint_as_float(x.x) + __uint_as_float(w.y) * __uint_as_float(x.y) +
           __uint_as_float(w.z) * __uint_as_float(x.z) + __uint_as_float(w.w) * __uint_as_float(x.w);
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
__device__ __forceinline__ float dot_v4(uint4 w, uint4 x, __nv_bfloat16) {
    return bf_lo(w.x) * bf_lo(x.x) + bf_hi(w.x) * bf_hi(x.x) + bf_lo(w.y) * bf_lo(x.y) + bf_hi(w.y) * bf_hi(x.y) +
           bf_lo(w.z) * bf_lo(x.z) + bf_hi(w.z) * bf_hi(x.z) + bf_lo(w.w) * bf_lo(x.w) + bf_hi(w.w) * bf_hi(x.w);
}

// y[r] for r in [r0, r1): each epilogue warp owns every 4th row and works on kRowsPerWarp of
// its rows at once, so every lane keeps kRowsPerWarp x 4 sixteen-byte non-allocating loads of W
// in flight (8 KB per warp, 32 KB per SM): a batch-1 GEMV is a pure HBM stream and only enough
// bytes in flight reach the bandwidth. x is re-read through L1.
template <typename T>
__device__ void gemv_rows(const DevProblem* Pg, int r0, int r1, int ew) {
    constexpr int kRowsPerWarp = 4;
    const T* __restrict__ W = reinterpret_cast<const T*>(Pg->in0);
    const T* __restrict__ x = reinterpret_cast<const T*>(Pg->in1);
    const int n = Pg->cols;
    const int64_t ld = Pg->ld_in0;
    void* out = Pg->out;
    const float* bias = Pg->bias;
    const int32_t act = Pg->act, out_dt = Pg->out_dt;
    constexpr int kVec = 16 / sizeof(T);
    const int lane = lane_id();
    const bool vec_ok = (n % kVec == 0) && (ld % kVec == 0) &&
                        ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    for (int rb = r0 + ew; rb < r1; rb += 4 * kRowsPerWarp) {
        float acc[kRowsPerWarp];
        const T* w[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            acc[q] = 0.0f;
            const int r = min(rb + 4 * q, r1 - 1);   // rows past the end recompute the last one
            w[q] = W + (int64_t)r * ld;
        }
        if (vec_ok) {
            const int nv = n / kVec;
            int j = lane;
            for (; j + 96 < nv; j += 128) {
                uint4 wv[kRowsPerWarp][4];
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q)
#pragma unroll
                    for (int u = 0; u < 4; ++u) wv[q][u] = ld_stream_v4(w[q] + (int64_t)(j + 32 * u) * kVec);
                uint4 xx[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) xx[u] = __ldg(xv + j + 32 * u);
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q)
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[q] += dot_v4(wv[q][u], xx[u], T());
            }
            for (; j < nv; j += 32) {
                const uint4 xx = __ldg(xv + j);
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q)
                    acc[q] += dot_v4(ld_stream_v4(w[q] + (int64_t)j * kVec), xx, T());
            }
        } else {
            for (int jj = lane; jj < n; jj += 32) {
                const float xs = load_f<T>(x + jj);
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q) acc[q] += load_f<T>(w[q] + jj) * xs;
            }
        }
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < kRowsPerWarp; ++q) {
                const int r = rb + 4 * q;
                if (r < r1) {
                    const float b = bias ? __ldg(bias + r) : 0.0f;
                    store_one(out, r, out_dt, apply_act(acc[q] + b, act));
                }
            }
        }
    }
}

// Staged GEMV item (4 epilogue warps): W arrives in ring stages of two tensor boxes (R rows x
// 512 columns); warp ew accumulates rows ew*R/4 .. of each R-row block against x (L1-resident),
// the 4 warps release each stage together, and a block's rows are reduced across the lanes and
// stored once its last column stage is done.
// The ring position comes in by value and the new one is returned packed (stage | phase << 16).
// (Measured: these CUDA-core item functions out of line — __noinline__ — cost C2 5 % through
// the call ABI's spills; inlined they cost it ~1 %.)
template <typename T>
__device__ __forceinline__ uint32_t gemv_staged(const DevProblem* Pg, const WorkItem it, int ew, int etid, uint8_t* smem,
                                             uint64_t* full, uint64_t* empty, int rstage, uint32_t rphase, int kStages) {
    constexpr bool kF32 = sizeof(T) == 4;
    constexpr int R = gv_box_rows(kF32), RW = R / 4;             // block rows, rows per warp
    constexpr int kVec = 16 / sizeof(T);                         // elements per 16-byte vector
    constexpr uint32_t kRowBytes = kGvBoxCols * sizeof(T);       // one box row
    constexpr uint32_t kBoxBytes = kRowBytes * R;                // 16 KB
    constexpr int kPerLane = kGvBoxCols / (32 * kVec);           // vectors per lane per box row
    const int n = Pg->cols;
    const int nck = (n + kGvStageCols - 1) / kGvStageCols;
    const int nb = (it.col0 - it.row0 + R - 1) / R;
    const uint4* xv = reinterpret_cast<const uint4*>(Pg->in1);
    void* out = Pg->out;
    const float* bias = Pg->bias;
    const int32_t act = Pg->act, out_dt = Pg->out_dt;
    const int lane = lane_id();
    for (int rb = 0; rb < nb; ++rb) {
        float acc[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) acc[r] = 0.0f;
        for (int cc = 0; cc < nck; ++cc) {
            mbar_wait(&full[rstage], rphase);
            const uint32_t base = smem_u32(smem + rstage * kStageBytes);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int c0 = cc * kGvStageCols + b * kGvBoxCols;
                uint4 xx[kPerLane];
#pragma unroll
                for (int q = 0; q < kPerLane; ++q) {
                    const int col = c0 + (lane + 32 * q) * kVec;   // n % kVec == 0 (registration)
                    xx[q] = col < n ? __ldg(xv + col / kVec) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int r = 0; r < RW; ++r) {
                    const uint32_t ra = base + (uint32_t)b * kBoxBytes + (uint32_t)(ew * RW + r) * kRowBytes;
#pragma unroll
                    for (int q = 0; q < kPerLane; ++q)
                        acc[r] += dot_v4(ld_shared_v4(ra + 16u * (uint32_t)(lane + 32 * q)), xx[q], T());
                }
            }
            named_bar_sync(4, 128);   // every warp is done reading the stage
            if (etid == 0) mbar_arrive(&empty[rstage]);
            if (++rstage == kStages) { rstage = 0; rphase ^= 1; }
        }
#pragma unroll
        for (int r = 0; r < RW; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                const int row = it.row0 + rb * R + ew * RW + r;
                if (row < it.col0) {
                    const float bv = bias ? __ldg(bias + row) : 0.0f;
                    store_one(out, row, out_dt, apply_act(acc[r] + bv, act));
                }
            }
        }
    }
    return (uint32_t)rstage | (rphase << 16);
}

template <typename T>
__device__ void eltwise_range(const DevProblem* Pg, int e0, int e1, int tid, int nthreads) {
    const T* __restrict__ x = reinterpret_cast<const T*>(Pg->in0);
    T* __restrict__ y = reinterpret_cast<T*>(Pg->out);
    const int32_t act = Pg->act;
    constexpr int kVec = 16 / sizeof(T);
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0 &&
                        (e0 % kVec) == 0;
    int i = e0;
    if (vec_ok) {
        const int nvec = (e1 - e0) / kVec;
        for (int v = tid; v < nvec; v += nthreads) {
            const int64_t idx = (int64_t)e0 + (int64_t)v * kVec;
            uint4 u = ld_stream_v4(x + idx);
            if constexpr (sizeof(T) == 4) {
                u.x = __float_as_uint(apply_act(__uint_as_float(u.x), act));
                u.y = __float_as_uint(apply_act(__uint_as_float(u.y), act));
                u.z = __float_as_uint(apply_act(__uint_as_float(u.z), act));
                u.w = __float_as_uint(apply_act(__uint_as_float(u.w), act));
            } else {
                u.x = pack_bf16x2(apply_act(bf_lo(u.x), act), apply_act(bf_hi(u.x), act));
                u.y = pack_bf16x2(apply_act(bf_lo(u.y), act), apply_act(bf_hi(u.y), act));
                u.z = pack_bf16x2(apply_act(bf_lo(u.z), act), apply_act(bf_hi(u.z), act));
                u.w = pack_bf16x2(apply_act(bf_lo(u.w), act), apply_act(bf_hi(u.w), act));
            }
            *reinterpret_cast<uint4*>(y + idx) = u;
        }
        i = e0 + nvec * kVec;
    }
    for (int j = i + tid; j < e1; j += nthreads) {
        const float v = apply_act(load_f<T>(x + j), act);
        store_one(y, j, sizeof(T) == 4 ? GMX_ST_F32 : GMX_ST_BF16, v);
    }
}

// Items of list `idx` of step k (non-resident: the launch's own plan, k == 0).
__device__ __forceinline__ StepView list_view(const KernelArgs& a, int64_t k, int idx) {
    StepView v{};
    if (!a.resident) {
        v.probs = a.probs; v.items = a.items; v.ws = a.ws; v.counters = a.counters;
        if (a.inline_n > 0) {   // inline launch: the slots are kernel parameters
            v.inl_n = a.inline_n;
            v.inl_slots = a.inline_slots;
            v.idx = idx;
            v.G = gridDim.x;
            return v;
        }
        v.beg = a.cta_off[idx];
        v.end = a.cta_off[idx + 1];
        return v;
    }
    const StepDesc* d = &a.dq->ring[k % kQueue];
    const int inl = __ldcg(&d->inline_n);
    if (inl > 0) {   // inline resident step: slots in the device ring entry
        v.probs = (const DevProblem*)__ldcg((const long long*)&d->probs);
        v.inl_n = inl;
        v.inl_slots = d->inline_slots;
        v.idx = idx;
        v.G = (uint32_t)__ldcg(&d->grid);   // the step's lists (items spread over them)
        return v;
    }
    v.probs = (const DevProblem*)__ldcg((const long long*)&d->probs);
    v.items = (const WorkItem*)__ldcg((const long long*)&d->items);
    v.ws = (float*)__ldcg((const long long*)&d->ws);
    v.counters = (int32_t*)__ldcg((const long long*)&d->counters);
    const int32_t* off = (const int32_t*)__ldcg((const long long*)&d->cta_off);
    if (idx < __ldcg(&d->grid)) {
        v.beg = __ldcg(off + idx);
        v.end = __ldcg(off + idx + 1);
    }
    return v;
}

// Count one finished item list of step k: a fire-and-forget release reduction (the caller's
// earlier writes are ordered before it); the dispatcher warp notices completed steps and tells
// the host, so no list waits for a round trip to L2 here.
// A finished list of step k counts into the step (release: covers the list's writes). The count
// that completes the step (G lists per round of the slot) reports it to the host right here: a
// system-scope release store of seq + 1 into the host-mapped flag (cumulative over the other
// lists' releases this acq_rel atomic observed). Reporting at the completing count instead of
// from a polling lane took ~4.5 us off every step's completion latency as the host sees it.
__device__ __forceinline__ void count_list_done(const KernelArgs& a, int64_t k, uint32_t n = 1) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(&a.dq->done[k % kQueue]), "r"(n) : "memory");
    if (old + n != gridDim.x * (uint32_t)(k / kQueue + 1)) return;
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(&a.hdone[k % kQueue]), "l"(k + 1) : "memory");
    const uint64_t t = global_timer_ns();
    atomicMax(reinterpret_cast<unsigned long long*>(&a.dq->t_last), (unsigned long long)t);
    if (a.rtrace && k < a.rtrace_steps)   // diagnostics: when step k was reported to the host
        a.rtrace[(int64_t)a.rtrace_steps * gridDim.x * 8 + a.rtrace_steps + k] = t;
}

// Resident producer: wait until step k is published; returns true for the stop step.
__device__ __forceinline__ bool step_published(const KernelArgs& a, int64_t k) {
    const uint64_t t0 = global_timer_ns();
    while (ld_acquire_gpu_s64(&a.dq->published) <= k) {
        __nanosleep(128);
        if (global_timer_ns() - t0 > 60000000000ull) __trap();   // host never published
    }
    return (__ldcg(&a.dq->ring[k % kQueue].stop) & 1) != 0;
}

// Resident list scheduler: wait until step k is relayed (the descriptor is then read whole).
__device__ __forceinline__ void step_relayed(const KernelArgs& a, int64_t k) {
    const uint64_t t0 = global_timer_ns();
    while (ld_acquire_gpu_s64(&a.dq->published) <= k) {
        __nanosleep(64);
        if (global_timer_ns() - t0 > 60000000000ull) __trap();   // host never published
    }
}

// Ordering of step k from its descriptor head already in registers (one round trip for every
// field instead of one per field).
__device__ __forceinline__ void step_order_head(const KernelArgs& a, int64_t k, const StepDesc& d) {
    if (d.wait_all) {
        for (int64_t j = k - 1; j >= 0 && j >= k - a.window; --j) wait_step_done(a.dq, j, gridDim.x);
        fence_proxy_async_global();   // later TMA loads read what those steps wrote
    } else {
        wait_step_done(a.dq, k - a.window, gridDim.x);
        for (int q = 0; q < d.nwait; ++q) wait_step_done(a.dq, d.wait_steps[q], gridDim.x);
        if (d.nwait != 0) fence_proxy_async_global();   // later TMA loads may read what they wrote
    }
}

// Resident producer: bounded skew + explicit ordering before taking lists of step k.
__device__ __forceinline__ void step_order(const KernelArgs& a, int64_t k) {
    const StepDesc* d = &a.dq->ring[k % kQueue];
    if (__ldcg(&d->wait_all)) {
        for (int64_t j = k - 1; j >= 0 && j >= k - a.window; --j) wait_step_done(a.dq, j, gridDim.x);
        fence_proxy_async_global();   // later TMA loads read what those steps wrote
    } else {
        // bounded skew, plus the listed steps: producers of this step's inputs and the latest
        // earlier users of its plan or slots (those waited for any earlier sharer, transitively)
        wait_step_done(a.dq, k - a.window, gridDim.x);
        const int nw = __ldcg(&d->nwait);   // -1: nothing to wait for, fence only
        for (int q = 0; q < nw; ++q)
            wait_step_done(a.dq, (int64_t)__ldcg((const long long*)&d->wait_steps[q]), gridDim.x);
        if (nw != 0) fence_proxy_async_global();   // later TMA loads may read what they wrote
    }
}

// Work units flow producer -> (MMA, epilogue) through a small smem ring: the producer takes
// item lists of step k from a per-step counter (any CTA may take any list: the device balances
// the lists dynamically, like the block scheduler does for separate launches), then issues
// their loads; the MMA issuer and the epilogue consume the same units in order.
// Resident mode: a list-scheduler warp takes the lists, resolves them (the step's plan
// pointers, the list's item range and items) and hands them to the producer, MMA issuer and
// epilogue as units in shared memory — the three roles then never wait on a global load for
// their work, only on their pipelines (measured: the producer used to spend ~40 % of a C2
// step in dependent L2 round trips: publication / ordering polls, list offsets, items).
constexpr int kUnitItems = 4;          // items per unit; longer lists span several units
constexpr int32_t kUnitEndStep = -1;   // this CTA took no more lists of step k
constexpr int32_t kUnitStop = -2;
struct alignas(16) Unit {
    int64_t k;
    int32_t idx;            // list index, or kUnitEndStep / kUnitStop
    int32_t n;              // items in it[] (resident); -1: not resolved, use list_view
    int32_t beg;            // index of it[0] within the list's items (trace / split bookkeeping)
    int32_t last;           // 1: the list's last unit (the epilogue counts the list done)
    const DevProblem* probs;
    float* ws;
    int32_t* counters;
    int64_t _pad;
    WorkItem it[kUnitItems];
};
static_assert(sizeof(Unit) == 192, "Unit layout");

// Dispatcher (resident mode; block 0, warp 6): host ring -> device ring.
__device__ void dispatch_steps(const KernelArgs& a) {
    // held start: relay nothing until the host sets the go flag (hpub[1]), so a batch queued
    // beforehand runs back to back and t_first..t_last times the device alone
    const uint64_t th = global_timer_ns();
    while (ld_acquire_sys_s64(a.hpub + 1) == 0) {
        __nanosleep(512);
        if (global_timer_ns() - th > 60000000000ull) __trap();
    }
    a.dq->t_first = global_timer_ns();
    a.dq->c_first = clock64();
    // relay in batches: one poll of the host count, then up to kBatch entries whose PCIe loads
    // are all in flight together (a PCIe round trip costs ~1-2 us; one per step would cap the
    // step rate)
    constexpr int kBatch = 4;
    int64_t k = 0;
    // completions are reported to the host by the count that completes each step (count_list_done)
    for (;;) {
        int64_t avail;
        const uint64_t t0 = global_timer_ns();
        uint32_t nap = 64;   // back off while idle: each poll is a PCIe round trip
        while ((avail = ld_acquire_sys_s64(a.hpub)) <= k) {
            __nanosleep(nap);
            nap = nap < 256 ? 2 * nap : nap;   // a new step waits at most ~0.25 us + one PCIe read
            if (global_timer_ns() - t0 > 60000000000ull) __trap();   // host never published
        }
        const int n = (int)(avail - k < kBatch ? avail - k : kBatch);
        // the fixed head of each entry (6 x 16 B: pointers, grid, flags, waits, inline_n and the
        // first inline slot) for the whole batch in flight together; the rest of an inline
        // step's slot list only when it has more than one member
        constexpr int kHead = 6;
        uint4 w[kBatch][kHead];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            if (b < n) {
                const uint4* src = reinterpret_cast<const uint4*>(&a.hring[(k + b) % kQueue]);
#pragma unroll
                for (int q = 0; q < kHead; ++q)   // system-scope loads of host-written entries (after the acquire)
                    asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(w[b][q].x), "=r"(w[b][q].y), "=r"(w[b][q].z), "=r"(w[b][q].w)
                                 : "l"(src + q));
            }
        }
        bool stop = false;
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            if (b < n && !stop) {
                const int slot = (int)((k + b) % kQueue);
                uint4* dst = reinterpret_cast<uint4*>(&a.dq->ring[slot]);
#pragma unroll
                for (int q = 0; q < kHead; ++q) __stcg(dst + q, w[b][q]);
                const StepDesc* head = reinterpret_cast<const StepDesc*>(w[b]);
                const int inl = head->inline_n;
                if (inl > 1) {
                    const uint4* src = reinterpret_cast<const uint4*>(&a.hring[slot]);
                    const int nq = (int)((offsetof(StepDesc, inline_slots) + 4 * inl + 15) / 16);
                    for (int q = kHead; q < nq; ++q) {
                        uint4 x;
                        asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                                     : "l"(src + q));
                        __stcg(dst + q, x);
                    }
                }
                stop = (head->stop & 1) != 0;
            }
        }
        k += n;
        asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(&a.dq->published), "l"(k) : "memory");
        a.dq->t_relay = global_timer_ns();
        if (a.rtrace)   // diagnostics: when steps k-n..k-1 were relayed (published + one PCIe read)
            for (int64_t j = k - n; j < k && j < a.rtrace_steps; ++j)
                a.rtrace[(int64_t)a.rtrace_steps * gridDim.x * 8 + j] = a.dq->t_relay;
        if (stop) break;
    }
    a.dq->t_stop = global_timer_ns();
    a.dq->c_stop = clock64();
}

// Register cap per shape (the 2-CTA shape keeps two CTAs' registers within one SM's 64K).
template <int kCtasPerSm>
__global__ void __maxnreg__(kCtasPerSm == 2 ? 144 : 255) coalesced_step_kernel(const __grid_constant__ KernelArgs args) {
    using Cfg = SmemCfg<kCtasPerSm>;
    constexpr int kStages = Cfg::stages;
    constexpr int kStageOut = Cfg::stage_out;
    extern __shared__ __align__(16) uint8_t smem_raw[];   // 1024-aligned in practice (no static smem); checked below
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (Cfg::align_pad == 0 && smem != smem_raw) __trap();   // SWIZZLE_128B tiles need 1024-byte alignment
    uint8_t* stg = smem + kStages * kStageBytes;                       // epilogue staging (1024-aligned)
    constexpr int kUnitQ = Cfg::unit_q;
    Unit* uq = reinterpret_cast<Unit*>(stg + kStageOut);               // resident work-unit ring
    uint64_t* full = reinterpret_cast<uint64_t*>(uq + kUnitQ);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    constexpr int kAcc = Cfg::acc_bufs;
    uint64_t* tempty = tfull + kAcc;
    uint64_t* ufull = tempty + kAcc;
    uint64_t* uempty = ufull + kUnitQ;
    // list-accounting ring (resident, blocks != 0): epilogue -> accountant lane (warp 6)
    constexpr int kAcctQ = 8;
    uint64_t* afull = uempty + kUnitQ;
    uint64_t* aempty = afull + kAcctQ;
    int64_t* aq = reinterpret_cast<int64_t*>(aempty + kAcctQ);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aq + kAcctQ);
    int32_t* split_flag = reinterpret_cast<int32_t*>(tmem_slot + 1);
    uint32_t* prod_units = reinterpret_cast<uint32_t*>(split_flag + 1);   // units the producer took (shared atomics)

    const int warp = threadIdx.x >> 5;
    const int lane = lane_id();
    // trace mode (per-step launches): per-CTA stamps after the item rows: entry, prologue done,
    // role loops done, exit
    uint64_t* ktr = (args.trace && !args.resident)
                        ? args.trace + 8 * ((int64_t)args.cta_off[gridDim.x] + blockIdx.x) : nullptr;
    if (ktr && threadIdx.x == 0) ktr[0] = global_timer_ns();
#ifdef GMX_INSTR
    long long ic[kICount] = {};
#else
    long long* ic = nullptr;   // counters compiled out
#endif

    // CTA owns GEMM tiles (host-computed; resident / inline steps: any list may bring some)
    const bool has_gemm = args.resident || args.inline_n > 0 || (args.cta_flags[blockIdx.x] & 1) != 0;
    // CTA streams GEMV rows (planner flag 2): its producer lane prefetches them into L2 up front
    const bool has_gemv = args.resident || args.inline_n > 0 || (args.cta_flags[blockIdx.x] & 2) != 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < kAcc; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);   // one arrival per epilogue warp
        }
        for (int u = 0; u < kUnitQ; ++u) {
            mbar_init(&ufull[u], 1);
            mbar_init(&uempty[u], 6);   // producer + MMA issuer + 4 epilogue warps
        }
        for (int q = 0; q < kAcctQ; ++q) {
            mbar_init(&afull[q], 1);
            mbar_init(&aempty[q], 1);
        }
        mbar_fence_init();
        *prod_units = 0u;
    }
    if (warp == 1 && has_gemm) tmem_alloc(tmem_slot, Cfg::tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = has_gemm ? *tmem_slot : 0u;
    if (ktr && threadIdx.x == 0) ktr[1] = global_timer_ns();
    // Programmatic dependent launch: everything above overlapped the previous step's tail; a
    // dependent step waits here until that grid has completed and flushed its memory.
    if (!args.independent) asm volatile("griddepcontrol.wait;" ::: "memory");
    // Early trigger: the next step's grid may launch as soon as every CTA of this one is
    // resident; its CTAs then take SMs as ours retire, so a step's tail overlaps the next
    // step's start (a dependent next step still waits for our completion and flush).
    if (args.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // Units: non-resident = this CTA's own list of the launch's plan, then stop; resident =
    // the unit ring filled by the list scheduler. A consumer reads the unit in place and
    // releases it when done with its items.
    int uslot = 0;
    uint32_t uphase = 0;
    Unit own{};   // non-resident: synthetic units
    auto next_unit = [&](bool first) -> const Unit* {
        if (!args.resident) {
            own.k = 0;
            own.idx = first ? (int32_t)blockIdx.x : kUnitStop;
            own.n = -1;
            return &own;
        }
        mbar_wait(&ufull[uslot], uphase);
        return &uq[uslot];
    };
    auto release_unit = [&]() {   // one thread per consumer role: done with the current unit
        if (args.resident) mbar_arrive(&uempty[uslot]);
    };
    auto advance_unit = [&]() {
        if (args.resident && ++uslot == kUnitQ) { uslot = 0; uphase ^= 1; }
    };
    auto view = [&](int64_t k, int idx) -> StepView { return list_view(args, k, idx); };
    auto unit_view = [&](const Unit* u) -> StepView {
        if (u->n < 0) return list_view(args, u->k, u->idx);
        StepView v{};
        v.probs = u->probs;
        v.ws = u->ws;
        v.counters = u->counters;
        v.items = u->it;
        v.beg = u->beg;
        v.end = u->beg + u->n;
        v.ibase = u->beg;
        return v;
    };

    // The gpu-scope release that counts a finished list into its step (~0.9 us under load: it
    // waits for the CTA's writes to be acknowledged) is taken off the epilogue's critical path:
    // the epilogue hands the list to an accountant lane through a small mbarrier ring (block 0,
    // whose warp 6 is the queue dispatcher, counts in the epilogue itself).
    const bool accountant = args.resident && blockIdx.x != 0;
    if (warp == 6) {
        // ---------------- queue dispatcher (resident mode, block 0) / accountant ----------------
        if (lane == 0 && args.resident && blockIdx.x == 0) dispatch_steps(args);
        if (lane == 0 && accountant) {
            for (int q = 0, ph = 0;; ) {
                mbar_wait(&afull[q], (uint32_t)ph);
                const int64_t kq = aq[q];
                if (kq < 0) break;
                // (lists << 48) | step: a CTA's lists of one step are counted together
                count_list_done(args, kq & ((int64_t(1) << 48) - 1), (uint32_t)(kq >> 48));   // release: covers the
                                                                                               // epilogue's writes (afull)
                mbar_arrive(&aempty[q]);
                if (++q == kAcctQ) { q = 0; ph ^= 1; }
            }
        }
    } else if (warp == 7) {
        // ---------------- list scheduler (resident mode) ----------------
        if (lane == 0 && args.resident) {
            auto unit_slot = [&]() -> Unit* {
                timed(ic, kISUempty, true, [&] { mbar_wait(&uempty[uslot], uphase ^ 1); });
                return &uq[uslot];
            };
            uint32_t pub_units = 0;
            auto publish = [&]() {
                mbar_arrive(&ufull[uslot]);   // release: the unit is visible to the consumers
                advance_unit();
                ++pub_units;
            };
            auto push_ctl = [&](int64_t k, int32_t code) {
                Unit* u = unit_slot();
                u->k = k;
                u->idx = code;
                u->n = 0;
                publish();
            };
            const uint32_t G = gridDim.x;
            auto grab_base = [&](int64_t k) { return 2u * G * (uint32_t)(k / kQueue); };   // 2 x G grabs per step
            uint32_t pre = 0;
            bool have_pre = false;
            for (int64_t k = 0;; ++k) {
                timed(ic, kISPub, k > 0, [&] { step_relayed(args, k); });
                // the descriptor head (6 x 16 B) in one round trip: flags, waits, plan pointers
                StepDesc d;
                {
                    const uint4* hp = reinterpret_cast<const uint4*>(&args.dq->ring[k % kQueue]);
                    uint4* hd = reinterpret_cast<uint4*>(&d);
#pragma unroll
                    for (int q = 0; q < 6; ++q) hd[q] = __ldcg(hp + q);
                }
                if (d.stop & 1) {
                    push_ctl(k, kUnitStop);
                    instr_dump(args, ic, kISUempty, kISLists + 1);
                    break;
                }
                timed(ic, kISOrder, true, [&] { step_order_head(args, k, d); });
                if (d.stop & 2) {   // plan still uploading: wait for its flag
                    const uint32_t want = (uint32_t)(k + 1);
                    const uint64_t t0 = global_timer_ns();
                    while (ld_acquire_sys_u32(&args.dq->plan_ready[k % kQueue]) != want) {
                        __nanosleep(64);
                        if (global_timer_ns() - t0 > 8000000000ull) __trap();
                    }
                }
                if (args.rtrace && k < args.rtrace_steps)
                    args.rtrace[(k * G + blockIdx.x) * 8] = global_timer_ns();
                const uint32_t base = grab_base(k);
                uint32_t* grab = &args.dq->grab[k % kQueue];
                uint32_t idx = have_pre ? pre : atomicAdd(grab, 1u) - base;
                have_pre = false;
                // the step's plan pointers (from the head read above)
                const uint32_t L = (uint32_t)d.grid;   // lists past L are empty
                const int inl = d.inline_n;
                const DevProblem* probs = d.probs;
                const WorkItem* items = d.items;
                float* ws = d.ws;
                int32_t* counters = d.counters;
                const int32_t* off = d.cta_off;
                auto begin_unit = [&](int32_t list, int32_t beg) -> Unit* {
                    Unit* u = unit_slot();
                    u->k = k;
                    u->idx = list;
                    u->beg = beg;
                    u->probs = probs;
                    u->ws = ws;
                    u->counters = counters;
                    return u;
                };
                for (;;) {
                    if (idx >= G) { push_ctl(k, kUnitEndStep); break; }
                    if (idx >= L) {
                        count_list_done(args, k);
                        idx = atomicAdd(grab, 1u) - base;
                        continue;
                    }
                    GMX_INSTR_INC(kISLists);
                    if (inl == 0) {
                        const int32_t beg = __ldcg(off + idx), end = __ldcg(off + idx + 1);
                        int32_t c = beg;
                        do {
                            const int n = min(kUnitItems, end - c);
                            WorkItem w[kUnitItems];
#pragma unroll
                            for (int j = 0; j < kUnitItems; ++j)   // all loads in flight together
                                if (j < n) {
                                    const uint4* q = reinterpret_cast<const uint4*>(items + c + j);
                                    reinterpret_cast<uint4*>(&w[j])[0] = __ldcg(q);
                                    reinterpret_cast<uint4*>(&w[j])[1] = __ldcg(q + 1);
                                }
                            Unit* u = begin_unit((int32_t)idx, c - beg);
#pragma unroll
                            for (int j = 0; j < kUnitItems; ++j)
                                if (j < n) u->it[j] = w[j];
                            u->n = n;
                            c += n;
                            u->last = c >= end ? 1 : 0;
                            publish();
                        } while (c < end);
                    } else {
                        // inline step: enumerate the list's virtual items into units
                        const StepView v = list_view(args, k, (int)idx);
                        ItemCursor cur = item_begin(v);
                        WorkItem w;
                        bool have = next_item(v, cur, w);
                        int32_t cnt = 0;
                        do {
                            Unit* u = begin_unit((int32_t)idx, cnt);
                            int n = 0;
                            while (have && n < kUnitItems) {
                                u->it[n++] = w;
                                have = next_item(v, cur, w);
                            }
                            u->n = n;
                            cnt += n;
                            u->last = have ? 0 : 1;
                            publish();
                        } while (have);
                    }
                    // Another list of this step only once the producer has (nearly) caught up:
                    // grabbing eagerly let the first CTAs to arrive take two lists each while
                    // others got none (a lone step ran ~2x its plan's critical path). The grab's
                    // round trip then overlaps the producer's last k-blocks of this list.
                    while ((int32_t)(pub_units - atomicOr(prod_units, 0u)) > args.grab_ahead) {}
                    const uint32_t nxt = atomicAdd(grab, 1u) - base;
                    if (nxt >= G) {
                        // no more lists of step k for us: take the first grab of step k + 1
                        // now, so its round trip overlaps the publication / ordering polls.
                        // (Its slot's previous round completed long ago: the counter is at
                        // the new round's base, and no work starts before those polls.)
                        pre = atomicAdd(&args.dq->grab[(k + 1) % kQueue], 1u) - grab_base(k + 1);
                        have_pre = true;
                    }
                    idx = nxt;
                }
            }
        }
    } else if (warp == 0) {
        // ---------------- TMA producer ----------------
        // Whole warp, uniform control flow on broadcast item fields, one elected lane issues
        // (tensor-map pointers and coordinates in uniform registers: see warp_uni).
        if (has_gemm || has_gemv) {
            int stage = 0;
            uint32_t phase = 0;
            // GEMV rows are streamed by the 4 epilogue warps with 16-byte loads (~32 KB in flight
            // per SM: latency-bound at ~2.5 TB/s); one bulk L2 prefetch per row range, issued for
            // every GEMV item of the list before any other work, keeps HBM streaming at full rate
            // and turns the warps' loads into L2 hits.
            auto prefetch_gemv = [&](const StepView& v) {
                auto one = [&](const WorkItem& it) {
                    if (item_kind(it.type) != kItemGemv || it.kb1 > 0) return;   // staged rows stream by TMA
                    const DevProblem* P = v.probs + it.problem;
                    const char* w = reinterpret_cast<const char*>(P->in0);
                    const int64_t esz = P->in_dt == GMX_ST_F32 ? 4 : 2;
                    const int64_t row = (int64_t)P->cols * esz, pitch = P->ld_in0 * esz;
                    if (row == pitch) {   // contiguous rows: one range
                        prefetch_l2_range(w + it.row0 * pitch, (it.col0 - it.row0) * pitch);
                    } else {
                        for (int r = it.row0; r < it.col0; ++r) prefetch_l2_range(w + r * pitch, row);
                    }
                };
                if (lane != 0) return;
                if (v.inl_n == 0) {
                    for (int i = v.beg; i < v.end; ++i) one(v.items[i - v.ibase]);
                } else {
                    ItemCursor c = item_begin(v);
                    WorkItem it;
                    while (next_item(v, c, it)) one(it);
                }
            };
            auto issue_list = [&](const StepView& v) {
                prefetch_gemv(v);
                __syncwarp();
                for_each_item(v, [&](const WorkItem& it, int i) {
                    const int32_t type = warp_uni((int32_t)it.type);
                    const int32_t kb0 = warp_uni(it.kb0), kb1 = warp_uni(it.kb1);
                    const DevProblem* P = reinterpret_cast<const DevProblem*>(
                        warp_uni(reinterpret_cast<uint64_t>(v.probs + it.problem)));
                    if (item_kind(type) == kItemGemv && kb1 > 0) {
                        // staged GEMV: W as tensor boxes (two per stage), consumed by the epilogue warps
                        const bool f32 = warp_uni(P->in_dt) == GMX_ST_F32;
                        const int R = gv_box_rows(f32);
                        const int nck = (warp_uni(P->cols) + kGvStageCols - 1) / kGvStageCols;
                        const int32_t row0 = warp_uni(it.row0);
                        const uint32_t box_bytes = (uint32_t)(kGvBoxCols * R * (f32 ? 4 : 2));
                        for (int st = 0; st < kb1; ++st) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            const int rb = st / nck, cc = st % nck;
                            uint8_t* tile = smem + stage * kStageBytes;
                            if (elect_one()) {
                                mbar_expect_tx(&full[stage], 2 * box_bytes);   // OOB parts arrive zero-filled
                                tma_load_2d(tile, &P->tm_rows, &full[stage], cc * kGvStageCols, row0 + rb * R);
                                tma_load_2d(tile + box_bytes, &P->tm_rows, &full[stage], cc * kGvStageCols + kGvBoxCols,
                                            row0 + rb * R);
                            }
                            __syncwarp();
                            if (++stage == kStages) { stage = 0; phase ^= 1; }
                        }
                        return;
                    }
                    if (item_kind(type) != kItemGemm) return;
                    const int32_t row0 = warp_uni(it.row0), col0 = warp_uni(it.col0);
                    const uint32_t bytes = kStageA + warp_uni((uint32_t)it.bn) * (kBlockK * 2);
                    const int kel = kblock_elems(type & kItemTf32);
                    if (args.trace && lane == 0) args.trace[8 * i + 0] = global_timer_ns();
                    if (elect_one()) {
                        tma_prefetch_desc(&P->tm_rows);   // descriptor fetch overlaps the slot wait
                        tma_prefetch_desc(&P->tm_cols);
                    }
                    __syncwarp();
                    for (int kb = kb0; kb < kb1; ++kb) {
                        timed(ic, kIPEmpty, true, [&] { mbar_wait(&empty[stage], phase ^ 1); });
                        GMX_INSTR_INC(kIPStages);
                        uint8_t* tile = smem + stage * kStageBytes;
                        if (elect_one()) {
                            mbar_expect_tx(&full[stage], bytes);
                            tma_load_2d(tile, &P->tm_rows, &full[stage], kb * kel, row0);
                            tma_load_2d(tile + kStageA, &P->tm_cols, &full[stage], kb * kel, col0);
                        }
                        __syncwarp();
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }, [&] {
                    __syncwarp();
                    if (lane == 0) release_unit();
                });
            };
            for (bool first = true;; first = false) {
                const Unit* u;
                timed(ic, kIPUnit, !first, [&] { u = next_unit(first); });
                const int32_t uidx = warp_uni(u->idx);
                const int64_t uk = u->k;
                if (lane == 0) atomicAdd(prod_units, 1u);   // the list scheduler paces its grabs on this
                if (uidx >= 0) {
                    issue_list(unit_view(u));   // releases the unit after reading its last item
                } else {
                    __syncwarp();
                    if (lane == 0) release_unit();
                }
                advance_unit();
                if (uidx == kUnitStop) {
                    if (lane == 0) {
                        instr_dump(args, ic, kIPUnit, kIPEmpty + 1);
                        instr_dump(args, ic, kIPStages, kIPStages + 1);
                    }
                    break;
                }
                if (uidx >= 0 && args.rtrace && uk < args.rtrace_steps && lane == 0)
                    args.rtrace[(uk * gridDim.x + blockIdx.x) * 8 + 1] = global_timer_ns();
            }
        }
    } else if (warp == 1) {
        // ---------------- UMMA issuer ----------------
        // The whole warp runs the loop (uniform control flow on broadcast values) and one
        // elected lane issues: the descriptors then live in uniform registers and consecutive
        // UTCHMMAs issue back to back.
        if (has_gemm) {
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            const uint32_t tbase = warp_uni(tmem_base);
            for (bool first = true;; first = false) {
                const Unit* u;
                timed(ic, kIMUnit, !first, [&] { u = next_unit(first); });
                const int32_t uidx = warp_uni(u->idx);
                if (uidx < 0) {
                    __syncwarp();
                    if (lane == 0) release_unit();
                    advance_unit();
                    if (uidx == kUnitStop) {
                        if (lane == 0) instr_dump(args, ic, kIMUnit, kIMFull + 1);
                        break;
                    }
                    continue;
                }
                const StepView v = unit_view(u);
                for_each_item(v, [&](const WorkItem& it, int i) {
                    const int32_t type = warp_uni((int32_t)it.type);
                    const int32_t kb0 = warp_uni(it.kb0), kb1 = warp_uni(it.kb1);
                    if (item_kind(type) == kItemGemv) {
                        // staged GEMV: its ring stages are the epilogue's. Still wait for each one to
                        // be filled: a role that skipped stages without waiting could run more than
                        // one lap ahead of the producer, and a parity wait cannot tell lap L from
                        // lap L + 2 (it would take a GEMV stage's data for its next k-block).
                        for (int st = 0; st < kb1; ++st) {
                            mbar_wait(&full[stage], phase);
                            if (++stage == kStages) { stage = 0; phase ^= 1; }
                        }
                        return;
                    }
                    if (item_kind(type) != kItemGemm) return;
                    const bool tf32 = type & kItemTf32;
                    const uint32_t bn = warp_uni((uint32_t)it.bn);
                    const uint32_t idesc = tf32 ? idesc_tf32_m128(bn) : idesc_bf16_m128(bn);
                    timed(ic, kIMTempty, true, [&] { mbar_wait(&tempty[acc], acc_phase ^ 1); });
                    tc_fence_after();
                    const uint32_t d_tmem = tbase + (uint32_t)acc * kMaxBN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        timed(ic, kIMFull, true, [&] { mbar_wait(&full[stage], phase); });
                        tc_fence_after();
                        const uint8_t* tile = smem + stage * kStageBytes;
                        const uint64_t a_desc = smem_desc_sw128(tile);
                        const uint64_t b_desc = smem_desc_sw128(tile + kStageA);
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < kBlockK / 16; ++kk) {   // UMMA K steps of 32 B (16 bf16 / 8 tf32)
                                if (args.dbg & 4) continue;
                                const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
                                if (tf32)
                                    umma_tf32(d_tmem, a_desc + 2 * kk, b_desc + 2 * kk, idesc, accum);
                                else
                                    umma_bf16(d_tmem, a_desc + 2 * kk, b_desc + 2 * kk, idesc, accum);
                            }
                            umma_commit(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) umma_commit(&tfull[acc]);
                    __syncwarp();
                    if (args.trace && lane == 0) args.trace[8 * i + 1] = global_timer_ns();
                    if (++acc == kAcc) { acc = 0; acc_phase ^= 1; }
                }, [&] {
                    __syncwarp();
                    if (lane == 0) release_unit();
                });
                advance_unit();
            }
        }
    } else if (warp >= 2 && warp <= 5) {
        // ---------------- epilogue / CUDA-core items ----------------
        const int ew = warp - 2;                 // 0..3
        const int lgrp = warp & 3;               // TMEM lane quarter this warp may access
        const int trow = lgrp * 32 + lane;       // tile row owned by this thread
        const int etid = ew * 32 + lane;         // 0..127
        int acc = 0;
        uint32_t acc_phase = 0;
        Staging S{stg, kStageOut / Cfg::stage_bufs, Cfg::stage_bufs, 0u};
        uint32_t groups = 0;                     // bulk groups committed by etid 0 (tracked by all)
        int pend = -1, pend_age = 0;             // split item whose completion is deferred
        WorkItem pend_it{};
        StepView v{};
        int rstage = 0;                          // TMA ring position (staged GEMV items read from it)
        uint32_t rphase = 0;
        auto complete_pending_body = [&]() {
            const WorkItem pt = pend_it;
            int32_t* counter = v.counters + pt.tile_slot;
            asm volatile("fence.acq_rel.gpu;" ::: "memory");   // this thread's reductions have landed
            named_bar_sync(1, 128);
            if (etid == 0) {
                int32_t prev;
                asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
                const int last = prev == pt.nsplit - 1;
                if (last) {
                    *counter = 0;   // re-arm for the next launch of this plan
                    fence_proxy_async_global();   // the other splits' sums, for the bulk loads
                }
                *split_flag = last;
                if (args.trace) args.trace[8 * pend + 5] = global_timer_ns();
            }
            named_bar_sync(1, 128);
            const bool last = *split_flag != 0;
            named_bar_sync(1, 128);   // split_flag read by all before it can be rewritten
            if (last) {
                groups += split_finalize(load_epi(v.probs + pt.problem), pt.row0, pt.col0,
                                         v.ws + (int64_t)pt.ws_blk * kWsBlock, S, trow, etid);
                if (args.trace && etid == 0) args.trace[8 * pend + 6] = global_timer_ns();
            }
            pend = -1;
        };
        auto complete_pending = [&]() { timed(ic, kIEComplete, true, [&] { complete_pending_body(); }); };
        // Resident accounting: a list counts into its step's done counter once its writes (generic
        // and TMA stores) are complete. To keep the TMA-store round trip off the critical path it
        // is deferred until the CTA finished its next list (then only the older list's store
        // groups are waited for); at the end of a step (no more lists for this CTA) it is flushed,
        // since a later step may wait for this one.
        int64_t acct_k = -1;      // step of the finished lists not yet counted
        uint32_t acct_n = 0;      // how many of them (a CTA's lists of one step are counted together)
        uint32_t acct_groups = 0;
        int aslot = 0;
        uint32_t aphase = 0;
        auto hand_over = [&](int64_t kk, uint32_t n) {   // etid 0: the accountant counts n lists of step kk (or stops, kk < 0)
            mbar_wait(&aempty[aslot], aphase ^ 1);
            aq[aslot] = kk < 0 ? kk : (kk | ((int64_t)n << 48));
            mbar_arrive(&afull[aslot]);   // release.cta: the epilogue's writes happen-before the count
            if (++aslot == kAcctQ) { aslot = 0; aphase ^= 1; }
        };
        auto account_body = [&](int64_t kk, uint32_t n, uint32_t newer_groups) {
            timed(ic, kIABar, true, [&] { named_bar_sync(1, 128); });   // all epilogue writes happen-before etid 0's release
            if (etid == 0) {
                timed(ic, kIAWait, true, [&] {
                    bulk_wait_upto(newer_groups);   // TMA stores of that list have landed
                    fence_proxy_async_global();
                });
                timed(ic, kIARed, true, [&] {
                    if (accountant)
                        hand_over(kk, n);
                    else
                        count_list_done(args, kk, n);
                });
                if (args.rtrace && kk < args.rtrace_steps)
                    args.rtrace[(kk * gridDim.x + blockIdx.x) * 8 + 3] = global_timer_ns();
            }
        };
        auto account = [&](int64_t kk, uint32_t n, uint32_t newer_groups) {
            timed(ic, kIEAcct, true, [&] { account_body(kk, n, newer_groups); });
        };
        for (bool first = true;; first = false) {
            const Unit* up;   // every epilogue thread waits on the unit barrier
            timed(ic, kIEUnit, !first, [&] { up = next_unit(first); });
            struct { int64_t k; int32_t idx, last; } u{up->k, up->idx, up->last};
            if (u.idx < 0) {   // end of a step for this CTA, or stop: flush the pending count
                __syncwarp();   // the warp has read the unit
                if (lane == 0) release_unit();
                advance_unit();
                if (acct_k >= 0) {
                    account(acct_k, acct_n, 0);
                    acct_k = -1;
                }
                if (u.idx == kUnitStop) {
                    if (etid == 0 && accountant) hand_over(-1, 0);
                    if (etid == 0) {
                        instr_dump(args, ic, kIEUnit, kIETfull + 1);
                        instr_dump(args, ic, kIEStaged, kIXIssue + 1);
                    }
                    break;
                }
                continue;
            }
            v = unit_view(up);
            uint64_t* rt = (args.rtrace && u.k < args.rtrace_steps) ? args.rtrace + (u.k * gridDim.x + blockIdx.x) * 8 : nullptr;
            if (rt && etid == 0) {
                rt[2] = global_timer_ns();
                rt[4] = (uint64_t)(v.end - v.beg);
            }
            for_each_item(v, [&](const WorkItem& it, int i) {
                const DevProblem* Pg = v.probs + it.problem;
                if (args.trace && etid == 0 && item_kind(it.type) != kItemGemm) args.trace[8 * i + 0] = global_timer_ns();
                if (item_kind(it.type) == kItemGemm) {
                    for (int kb = it.kb0; kb < it.kb1; ++kb)   // the MMA's stages: keep the ring position
                        if (++rstage == kStages) { rstage = 0; rphase ^= 1; }
                    const EpiParams E = load_epi(Pg);
                    timed(ic, kIETfull, true, [&] { mbar_wait(&tfull[acc], acc_phase); });
                    tc_fence_after();
                    if (args.trace && etid == 0) args.trace[8 * i + 2] = global_timer_ns();
                    const uint32_t taddr = tmem_base + ((uint32_t)(lgrp * 32) << 16) + (uint32_t)acc * kMaxBN;
                    const int nchunks = E.bn / 32;
                    const bool split = it.nsplit > 1;
                    if (args.dbg & 2) {   // experiment: no epilogue (bounds the load/MMA side)
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                    } else if (!split && E.tma_out && !(args.dbg & 8)) {
                        timed(ic, kIEStaged, true, [&] {
                            groups += epilogue_staged(E, it.row0, it.col0, S, trow, etid, taddr, &tempty[acc],
                                                      args.trace ? args.trace + 8 * i : nullptr, ic);
                        });
                    } else if (!split) {
                        for (int c = 0; c < nchunks; ++c) {
                            float vv[32];
                            tmem_ld32(taddr + (uint32_t)(c * 32), vv);
                            store_tile_chunk(E, it.row0, it.col0, trow, c, vv);
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                    } else {
                        // split-K (planner only splits TMA-store problems): reduce now, complete later
                        if (pend >= 0) complete_pending();   // at most one split in flight
                        float* acc_tile = v.ws + (int64_t)it.ws_blk * kWsBlock;
                        timed(ic, kIESplit, true, [&] { split_reduce(E, acc_tile, trow, taddr, &tempty[acc]); });
                        if (args.trace && etid == 0) args.trace[8 * i + 4] = global_timer_ns();
                        pend = i;
                        pend_it = it;
                        pend_age = 0;
                    }
                    if (++acc == kAcc) { acc = 0; acc_phase ^= 1; }
                } else if (it.type == kItemGemv && it.kb1 > 0) {
                    uint32_t rs;
                    if (Pg->in_dt == GMX_ST_F32)
                        rs = gemv_staged<float>(Pg, it, ew, etid, smem, full, empty, rstage, rphase, kStages);
                    else
                        rs = gemv_staged<__nv_bfloat16>(Pg, it, ew, etid, smem, full, empty, rstage, rphase, kStages);
                    rstage = (int)(rs & 0xFFFFu);
                    rphase = rs >> 16;
                } else if (it.type == kItemGemv) {
                    if (Pg->in_dt == GMX_ST_F32)
                        gemv_rows<float>(Pg, it.row0, it.col0, ew);
                    else
                        gemv_rows<__nv_bfloat16>(Pg, it.row0, it.col0, ew);
                } else {
                    if (Pg->in_dt == GMX_ST_F32)
                        eltwise_range<float>(Pg, it.row0, it.col0, etid, 128);
                    else
                        eltwise_range<__nv_bfloat16>(Pg, it.row0, it.col0, etid, 128);
                }
                if (args.trace) {
                    named_bar_sync(2, 128);
                    if (etid == 0) args.trace[8 * i + 3] = global_timer_ns();
                }
                if (pend >= 0 && pend != i && ++pend_age >= 1) complete_pending();
            }, [&] {
                __syncwarp();   // the warp has read the unit's last item
                if (lane == 0) release_unit();
            });
            if (pend >= 0) complete_pending();
            advance_unit();
            if (rt && etid == 0) rt[7] = global_timer_ns();
            if (args.resident && u.last) {
                if (acct_k == u.k) {   // another list of the pending step: counted with it
                    ++acct_n;
                } else {
                    if (acct_k >= 0) account(acct_k, acct_n, groups - acct_groups);   // the previous step's lists
                    acct_k = u.k;
                    acct_n = 1;
                }
                acct_groups = groups;
            }
        }
        // TMA stores must have read their smem before the CTA exits; their global writes
        // complete with the grid (a dependent launch's griddepcontrol.wait covers them)
        if (etid == 0) bulk_wait_read0();
    }

    if (ktr && warp == 2 && lane == 0) ktr[2] = global_timer_ns();
    tc_fence_before();
    __syncthreads();
    // this CTA's work is done: the next step may start taking SMs
    if (!args.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 1 && has_gemm) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::tmem_cols);
    }
    if (ktr && threadIdx.x == 32) ktr[3] = global_timer_ns();
}

// ------------------------------------------------------------------ host side

static thread_local std::string g_err;

static int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}

#define GMX_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) return fail(GMX_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

using StreamWriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWriteValue32Fn stream_write_fn() {
    static StreamWriteValue32Fn fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<StreamWriteValue32Fn>(p);
        return (StreamWriteValue32Fn) nullptr;
    }();
    return fn;
}

// experiment knob GMX_L2_PROMO=0|64|128|256 (default 256): L2 sector promotion of operand loads
static CUtensorMapL2promotion l2_promotion() {
    static CUtensorMapL2promotion v = [] {
        const char* e = std::getenv("GMX_L2_PROMO");
        const int x = e ? std::atoi(e) : 256;
        return x == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : x == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : x == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    return v;
}

// bf16 or fp32 [rows x K] row-major operand, leading dim `ld` elements, boxes of one 128-byte
// swizzle row (64 bf16 / 32 fp32) of K x box_rows.
static int make_tmap(CUtensorMap* map, const void* ptr, int64_t rows, int64_t K, int64_t ld, int box_rows,
                     bool f32) {
    auto fn = encode_fn();
    if (!fn) return fail(GMX_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * (f32 ? 4 : 2))};
    cuuint32_t box[2] = {(cuuint32_t)kblock_elems(f32), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GMX_EINVAL, "cuTensorMapEncodeTiled failed (alignment/stride?) code " + std::to_string((int)r));
    return GMX_OK;
}

// UMMA N of a problem: 64 for narrow outputs, else 128 (multiples of 64 keep every output
// TMA box inside its own tile).
static int choose_bn(int64_t cols) { return cols <= 64 ? 64 : kMaxBN; }

struct HostProblem {
    DevProblem dev;
    gmx_problem_desc desc;
    bool live = false;
    int64_t op_bytes = 0;   // algorithmic bytes (each operand + result once)
    int64_t flops = 0;
};

// Device buffers of a plan come from the stream-ordered allocator (cudaMallocAsync) and are
// released with cudaFreeAsync on the stream of the plan's last launch, so evicting a plan
// whose launch is still queued is safe and no eviction ever synchronizes the device.
constexpr size_t kPinZeros = (size_t)4 << 20;   // residency pinned staging: leading zero block

// Plan flavours of one slot set: per-step launches, resident steps queued behind others
// (throughput: coarse split), and resident steps entering an idle device (latency: the step runs
// alone, so its critical path is its longest list; finer split).
enum : int8_t { kPlanStep = 0, kPlanResident = 1, kPlanIdle = 2 };

struct Plan {
    std::vector<int32_t> key;       // sorted slot list this plan was built for
    int64_t res_seq = -1;           // resident: last step (seq) that used this plan, in residency res_epoch
    int64_t res_epoch = -1;
    std::vector<WorkItem> items;
    std::vector<int32_t> cta_off;   // cta_off[grid + 1] then cta_flags[grid]
    void* d_buf = nullptr;          // items + offsets/flags
    void* d_state = nullptr;        // split-K accumulators + counters (zeroed, re-armed by the kernel)
    WorkItem* d_items = nullptr;
    int32_t* d_off = nullptr;
    float* d_ws = nullptr;
    int32_t* d_counters = nullptr;
    bool uploaded = false;
    bool in_arena = false;          // device memory is the residency arena's (never freed per plan)
    int8_t mode = 0;                // kPlanStep (split_pct_step), kPlanResident (split_pct) or kPlanIdle (split_pct_idle)
    int64_t ws_floats = 0;
    int32_t n_counters = 0;
    cudaStream_t stream = nullptr;  // stream of the last launch
    cudaEvent_t done_ev = nullptr;  // multi-stream mode: recorded after each launch of the plan
    uint64_t last_use = 0;          // LRU clock
    gmx_plan_stats stats{};
    ~Plan() {
        if (d_buf && !in_arena) cudaFreeAsync(d_buf, stream);
        if (d_state && !in_arena) cudaFreeAsync(d_state, stream);
        if (done_ev) cudaEventDestroy(done_ev);
    }
};

}  // namespace gmx

struct gmx_exec {
    int device = 0;
    int num_sms = 148;
    std::vector<gmx::HostProblem> probs;
    gmx::DevProblem* d_probs = nullptr;
    size_t d_cap = 0;
    bool table_dirty = false;
    std::unordered_map<uint64_t, std::vector<std::unique_ptr<gmx::Plan>>> plans;   // hash(slots) -> plans
    size_t n_plans = 0;
    size_t plan_capacity = 4096;
    uint64_t clock = 0;
    std::vector<int32_t> key_scratch;
    gmx::Plan* last = nullptr;
    std::unique_ptr<gmx::Plan> uncached;
    float* ws = nullptr;
    int64_t ws_cap = 0;
    int32_t* counters = nullptr;
    int32_t counters_cap = 0;
    int64_t max_split = 32;
    int64_t split_pct = 400;     // split a tile into pieces of about this % of the per-CTA share
    // per-step launches run a step alone (no next step overlaps its tail), so their plans split
    // finer: a lone C2 step 27.5 -> 23.5 us (CUDA events, queued), held resident steps keep the
    // coarse split (5.96 vs 6.19 us at 200 %)
    int64_t split_pct_step = 200;
    // resident steps published while no earlier step is in flight run alone (the first step of
    // a serving burst): their plans split like this (0: same plan as any resident step). Lone
    // C2 step, publish -> completion seen by the host (tools/resident_lone.py): 32.2 us on the
    // resident plan (400 %), 28.8 at 200 %, 29.4 at 100 %, 32.8 at 50 %
    int64_t split_pct_idle = 200;
    // GEMV rows through the TMA ring (bulk copies) when stageable. Off by default: faster for a
    // held batch of C1 steps (11.7 vs 13.3 us/step) but slower lone and live-fed (C1 through the
    // resident runtime 17.7 vs 11.6 us per round; tools/c1_kernel.py, tools/ab_c1.sh)
    bool gemv_staged = true;              // option "gemv_staged": W as tensor boxes through the ring
    int ctas_per_sm = 1;         // 1, or 2 CTAs of the coalesced kernel per SM (the latter runs as 2 waves)
    bool cache_plans = true;
    bool attr_set = false;
    bool tracing = false;
    bool pdl = true;
    bool early_trigger = true;
    bool multi_stream = false;   // launches may come from several streams (realtime runtime)
    int occupancy[2] = {0, 0};   // measured resident CTAs/SM of the 1- and 2-CTA kernel shapes
    bool inline_plans = false;   // option "inline_plans": first-seen slot sets run as inline steps
    int inline_promote = 1;      // sightings before a slot set gets a cached plan
    std::vector<std::pair<uint64_t, int32_t>> inline_seen = std::vector<std::pair<uint64_t, int32_t>>(4096);
    int64_t inline_launches = 0;
    int32_t dbg = 0;
    const gmx::Plan* recent[3] = {nullptr, nullptr, nullptr};   // plans of the last launches
    // per-step launches: slots written / read by launches since the last fully ordered launch
    std::vector<uint8_t> hz_wr, hz_rd;
    std::vector<int32_t> hz_touched;
    uint64_t* trace = nullptr;
    int64_t trace_cap = 0;
    int64_t trace_items = 0;
    // resident (persistent) mode
    struct Resident {
        bool active = false;
        cudaStream_t stream = nullptr;        // stream of the persistent launch
        cudaStream_t upload = nullptr;        // non-blocking stream for plan/table uploads
        gmx::StepDesc* hring = nullptr;       // pinned, device-mapped
        int64_t* hpub = nullptr;              // pinned, device-mapped: [0] published count
        int64_t* hdone = nullptr;             // pinned, device-mapped: [kQueue] seq + 1 per slot
        gmx::StepDesc* hring_d = nullptr;     // device aliases of the three above
        int64_t* hpub_d = nullptr;
        int64_t* hdone_d = nullptr;
        gmx::DevQueue* dq = nullptr;
        int64_t seq = 0;                      // steps enqueued in this residency
        int grid = 0;
        int64_t epoch = 0;                     // residency counter (validates Plan::res_seq)
        std::vector<int64_t> last_write;       // per slot: last step (seq) that wrote its output
        std::vector<int64_t> last_read;        // per slot: last step (seq) that read its output (WAR)
        std::vector<void*> graveyard;          // device tables retired during residency
        std::vector<uint8_t> zeros;            // host zeros for copy-engine clears while resident
        // plans first built DURING a residency: device memory from a bump arena allocated before the
        // persistent launch (no stream-ordered allocation behind the kernel), uploaded on `upload`
        // without blocking the serving thread; the step waits on the device for a copy-engine
        // stream write of plan_ready (cuStreamWriteValue32 after the copies)
        char* arena = nullptr;
        size_t arena_size = 0, arena_used = 0;
        // pinned staging for those uploads (a pageable source can make cudaMemcpyAsync wait): a
        // zero block for copy-engine clears, then a bump region reset at each resident_begin (the
        // previous residency's copies completed before its kernel did)
        char* pin = nullptr;
        size_t pin_size = 0, pin_used = 0;
        int window = 16;                       // max steps a CTA may run ahead (option "resident_window")
        int64_t wait_ns = 0, waits = 0, pub_ns = 0, pubs = 0, up_ns = 0, ups = 0, wr_ns = 0;   // diagnostics (dbg bit 16)
        int grab_ahead = 1;                    // option "grab_ahead": see KernelArgs::grab_ahead
        int64_t relay_ns = 0;                  // last residency: release -> last relay (diagnostic)
        int32_t rtrace_steps = 0;              // option "rtrace": stamp this many steps
        uint64_t* rtrace = nullptr;
    } res;
};

namespace gmx {

static int ensure_table(gmx_exec* ex, cudaStream_t stream) {
    if (!ex->table_dirty) return GMX_OK;
    std::vector<DevProblem> host(ex->probs.size());
    for (size_t i = 0; i < host.size(); ++i) host[i] = ex->probs[i].dev;
    if (ex->res.active) {
        // the persistent kernel may still read the current table through queued steps: write a
        // fresh copy (upload stream, waited here) and retire the old one until residency ends
        const size_t cap = std::max<size_t>(64, ex->probs.size());
        DevProblem* fresh = nullptr;
        GMX_CUDA(cudaMallocAsync(&fresh, cap * sizeof(DevProblem), ex->res.upload));
        GMX_CUDA(cudaMemcpyAsync(fresh, host.data(), host.size() * sizeof(DevProblem), cudaMemcpyHostToDevice,
                                 ex->res.upload));
        GMX_CUDA(cudaStreamSynchronize(ex->res.upload));
        if (ex->d_probs) ex->res.graveyard.push_back(ex->d_probs);
        ex->d_probs = fresh;
        ex->d_cap = cap;
        ex->table_dirty = false;
        return GMX_OK;
    }
    if (ex->probs.size() > ex->d_cap) {
        size_t cap = std::max<size_t>(64, ex->d_cap);
        while (cap < ex->probs.size()) cap *= 2;
        if (ex->d_probs) GMX_CUDA(cudaFree(ex->d_probs));
        GMX_CUDA(cudaMalloc(&ex->d_probs, cap * sizeof(DevProblem)));
        ex->d_cap = cap;
    }
    GMX_CUDA(cudaMemcpy(ex->d_probs, host.data(), host.size() * sizeof(DevProblem), cudaMemcpyHostToDevice));
    ex->table_dirty = false;
    (void)stream;
    return GMX_OK;
}

// Planner cost model, in ns of one SM, calibrated from %globaltimer traces of C2 steps on B200
// (tools/trace_c2.py): with every SM streaming, TMA delivers ~50 GB/s per SM (the step is HBM
// bound), a 128 x BN epilogue costs ~0.6 us, a split-K partial (RED + arrival) ~2 us and the
// last split's finalize ~2.2 us.
constexpr double kNsPerKB = 20.0;
constexpr double kTileFixedNs = 600.0;
constexpr double kSplitNs = 800.0;   // epilogue-side reduce issue; the L2 round trips are deferred
constexpr double kCudaCoreFixedNs = 400.0;

static double gemm_tile_cost(const DevProblem& P, int kb) {
    return (double)kb * (kTileRows + P.bn) * kBlockK * 2.0 / 1024.0 * kNsPerKB + kTileFixedNs;
}

static int build_plan(gmx_exec* ex, const std::vector<int32_t>& slots, Plan& plan, int mode) {
    struct Cand {
        WorkItem it;
        double cost;
    };
    std::vector<Cand> cands;
    double total = 0.0;
    gmx_plan_stats st{};
    // pass 1: base items (no split) to size the per-SM target
    struct TileRef { int32_t slot; int32_t r0, c0; double cost; };
    std::vector<TileRef> tiles;
    for (int32_t s : slots) {
        const HostProblem& hp = ex->probs[s];
        const DevProblem& P = hp.dev;
        st.operand_bytes += hp.op_bytes;
        st.flops += hp.flops;
        if (P.kind == kItemGemm) {
            for (int r0 = 0; r0 < P.rows; r0 += kTileRows)
                for (int c0 = 0; c0 < P.cols; c0 += P.bn) {
                    const double c = gemm_tile_cost(P, P.kblocks);
                    tiles.push_back({s, r0, c0, c});
                    total += c;
                    st.tile_load_bytes += (int64_t)P.kblocks * (kTileRows + P.bn) * kBlockK * 2;
                }
        } else {
            total += (double)hp.op_bytes / 1024.0 * kNsPerKB + kCudaCoreFixedNs;
        }
    }
    const int slots_total = ex->num_sms * ex->ctas_per_sm;   // resident CTAs of one launch
    // per-CTA share; with 2 CTAs/SM each streams at about half an SM's rate
    const double target = std::max(total * ex->ctas_per_sm / slots_total, 2000.0);
    // GEMM tiles, split along K when one tile exceeds the per-SM share
    int32_t n_counters = 0;
    int64_t ws_blocks = 0;
    for (const TileRef& t : tiles) {
        const DevProblem& P = ex->probs[t.slot].dev;
        int nsplit = 1;
        const double piece = target * (double)(mode == kPlanResident ? ex->split_pct
                                               : mode == kPlanIdle ? ex->split_pct_idle : ex->split_pct_step) / 100.0;
        if (t.cost > piece && P.kblocks >= 2 && P.tma_out) {
            nsplit = (int)std::min<int64_t>({(int64_t)std::ceil(t.cost / piece), (int64_t)P.kblocks, ex->max_split, 255});
            // splitting only pays when a piece plus the fixup beats the whole tile
            if (gemm_tile_cost(P, (P.kblocks + nsplit - 1) / nsplit) + kSplitNs >= t.cost) nsplit = 1;
        }
        ++st.n_gemm_tiles;
        int32_t slot = -1, blk = 0;
        if (nsplit > 1) {
            slot = n_counters++;
            blk = (int32_t)ws_blocks;
            ws_blocks += ((int64_t)kTileRows * P.bn + kWsBlock - 1) / kWsBlock;   // one fp32 accumulator tile
        }
        for (int sp = 0; sp < nsplit; ++sp) {
            WorkItem it{};
            it.problem = t.slot;
            it.type = kItemGemm | (P.in_dt == GMX_ST_F32 ? kItemTf32 : 0);
            it.nsplit = (uint8_t)nsplit;
            it.split = (uint8_t)sp;
            it.row0 = t.r0;
            it.col0 = t.c0;
            it.kb0 = (int32_t)((int64_t)P.kblocks * sp / nsplit);
            it.kb1 = (int32_t)((int64_t)P.kblocks * (sp + 1) / nsplit);
            it.bn = (uint8_t)P.bn;
            it.tile_slot = slot;
            it.ws_blk = blk;
            const double c = gemm_tile_cost(P, it.kb1 - it.kb0) + (nsplit > 1 ? kSplitNs : 0.0);
            cands.push_back({it, c});
            if (nsplit > 1) ++st.n_split_items;
        }
    }
    // CUDA-core items: chunk so no item exceeds about half the per-SM share
    for (int32_t s : slots) {
        const HostProblem& hp = ex->probs[s];
        const DevProblem& P = hp.dev;
        if (P.kind == kItemGemv) {
            const double row_bytes = (double)P.cols * (P.in_dt == GMX_ST_F32 ? 4 : 2);
            const double item_bytes = std::max(32768.0, (target * 0.5 - kCudaCoreFixedNs) / kNsPerKB * 1024.0);
            // whole row blocks: 16 rows (4 epilogue warps x 4 rows in flight, gemv_rows) or the
            // staged path's R-row tensor boxes
            const bool f32 = P.in_dt == GMX_ST_F32;
            const bool staged = ex->gemv_staged && P.bn != 0;
            const int blk = staged ? gv_box_rows(f32) : 16;
            int rows_per = (int)std::max((double)blk, std::floor(item_bytes / row_bytes));
            rows_per = std::max(blk, (rows_per / blk) * blk);
            for (int r0 = 0; r0 < P.rows; r0 += rows_per) {
                WorkItem it{};
                it.problem = s;
                it.type = kItemGemv;
                it.row0 = r0;
                it.col0 = std::min(P.rows, r0 + rows_per);
                it.kb1 = staged ? gv_stages(it.col0 - it.row0, P.cols, f32) : 0;   // ring stages (0: unstaged)
                cands.push_back({it, row_bytes * (it.col0 - it.row0) / 1024.0 * kNsPerKB + kCudaCoreFixedNs});
                ++st.n_gemv_items;
            }
        } else if (P.kind == kItemEltwise) {
            const int esz = P.in_dt == GMX_ST_F32 ? 4 : 2;
            int64_t per = (int64_t)std::max(32768.0, (target * 0.5 - kCudaCoreFixedNs) / kNsPerKB * 1024.0) / (2 * esz);
            per = std::max<int64_t>(1024, (per / 1024) * 1024);
            for (int64_t e0 = 0; e0 < P.rows; e0 += per) {
                WorkItem it{};
                it.problem = s;
                it.type = kItemEltwise;
                it.row0 = (int32_t)e0;
                it.col0 = (int32_t)std::min<int64_t>(P.rows, e0 + per);
                cands.push_back({it, 2.0 * esz * (it.col0 - it.row0) / 1024.0 * kNsPerKB + kCudaCoreFixedNs});
                ++st.n_eltwise_items;
            }
        }
    }
    // LPT: longest item first onto the least-loaded CTA
    std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.cost > b.cost; });
    const int grid = (int)std::max<size_t>(1, std::min<size_t>((size_t)slots_total, cands.size()));
    std::vector<std::vector<int32_t>> per_cta(grid);
    std::vector<double> load(grid, 0.0);
    using QE = std::pair<double, int>;
    std::priority_queue<QE, std::vector<QE>, std::greater<QE>> heap;
    for (int c = 0; c < grid; ++c) heap.push({0.0, c});
    for (size_t i = 0; i < cands.size(); ++i) {
        QE top = heap.top();
        heap.pop();
        per_cta[top.second].push_back((int32_t)i);
        load[top.second] += cands[i].cost;
        heap.push({load[top.second], top.second});
    }
    plan.items.clear();
    plan.cta_off.assign(1, 0);
    std::vector<int32_t> flags(grid, 0);
    for (int c = 0; c < grid; ++c) {
        // split pieces first: their deferred completion then overlaps the CTA's other items
        std::stable_partition(per_cta[c].begin(), per_cta[c].end(),
                              [&](int32_t idx) { return cands[idx].it.nsplit > 1; });
        for (int32_t idx : per_cta[c]) {
            plan.items.push_back(cands[idx].it);
            if (item_kind(cands[idx].it.type) == kItemGemm) flags[c] |= 1;
            if (item_kind(cands[idx].it.type) == kItemGemv) flags[c] |= 2;
        }
        plan.cta_off.push_back((int32_t)plan.items.size());
    }
    if (plan.items.empty()) {   // keep the device arrays non-empty
        plan.cta_off.assign(2, 0);
        flags.assign(1, 0);
    }
    // device layout: cta_off[grid + 1] followed by cta_flags[grid]
    plan.cta_off.insert(plan.cta_off.end(), flags.begin(), flags.end());
    st.grid = grid;
    st.n_items = (int32_t)plan.items.size();
    st.max_cta_cost = *std::max_element(load.begin(), load.end());
    st.mean_cta_cost = std::accumulate(load.begin(), load.end(), 0.0) / grid;
    plan.stats = st;
    plan.ws_floats = ws_blocks * kWsBlock;
    plan.n_counters = n_counters;
    return GMX_OK;
}

// Upload the plan (one stream-ordered allocation + one copy) and allocate its split-K state.
// Split-K state is owned by the plan, so steps of different plans that overlap under PDL never
// share accumulators; a plan launched again while a recent launch of it may still run waits.
// Bump allocation from the residency arena (256-byte aligned); nullptr when it is full.
static void* arena_alloc(gmx_exec* ex, size_t bytes) {
    auto& r = ex->res;
    const size_t b = (bytes + 255) & ~size_t(255);
    if (!r.arena || r.arena_used + b > r.arena_size) return nullptr;
    void* p = r.arena + r.arena_used;
    r.arena_used += b;
    return p;
}

static int upload_plan(gmx_exec* ex, Plan& plan, cudaStream_t stream) {
    if (plan.uploaded) return GMX_OK;
    auto& r = ex->res;
    const size_t items_bytes = std::max<size_t>(1, plan.items.size()) * sizeof(WorkItem);
    const size_t off_bytes = plan.cta_off.size() * sizeof(int32_t);
    const size_t nstage = items_bytes + off_bytes, nal = (nstage + 255) & ~size_t(255);
    const size_t ws_bytes = (size_t)plan.ws_floats * sizeof(float);
    const size_t state = (plan.ws_floats > 0 || plan.n_counters > 0)
                             ? ws_bytes + (size_t)std::max(1, 2 * plan.n_counters) * sizeof(int32_t) : 0;
    auto fill = [&](uint8_t* dst) {
        if (!plan.items.empty()) std::memcpy(dst, plan.items.data(), plan.items.size() * sizeof(WorkItem));
        std::memcpy(dst + items_bytes, plan.cta_off.data(), off_bytes);
    };
    auto finish = [&]() {
        plan.d_items = reinterpret_cast<WorkItem*>(plan.d_buf);
        plan.d_off = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(plan.d_buf) + items_bytes);
        if (state) {
            plan.d_ws = reinterpret_cast<float*>(plan.d_state);
            plan.d_counters = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(plan.d_state) + ws_bytes);
        }
        plan.stream = stream;
        plan.uploaded = true;
        return GMX_OK;
    };
    // during a residency: one block of the arena (plan + split-K state), the plan filled by ONE
    // copy from pinned staging — no stream-ordered allocation, no pageable staging, no host wait.
    // The arena is zeroed whenever it is (re)started and the kernel re-arms split-K state after
    // use, so a new plan's state needs no clearing.
    const size_t span = nal;
    if (r.active && r.pin && r.pin_used + span <= r.pin_size) {
        if (char* blk = static_cast<char*>(arena_alloc(ex, nal + state))) {
            uint8_t* stg = reinterpret_cast<uint8_t*>(r.pin + r.pin_used);
            r.pin_used += span;
            fill(stg);
            GMX_CUDA(cudaMemcpyAsync(blk, stg, nstage, cudaMemcpyHostToDevice, stream));
            plan.d_buf = blk;
            plan.d_state = state ? blk + nal : nullptr;
            plan.in_arena = true;
            return finish();
        }
    }
    // general path: stream-ordered allocations
    std::vector<uint8_t> staging(nstage);
    fill(staging.data());
    GMX_CUDA(cudaMallocAsync(&plan.d_buf, nstage, stream));
    GMX_CUDA(cudaMemcpyAsync(plan.d_buf, staging.data(), nstage, cudaMemcpyHostToDevice, stream));
    if (state) {
        GMX_CUDA(cudaMallocAsync(&plan.d_state, state, stream));
        if (r.active) {
            // a memset KERNEL could not get an SM while the persistent kernel holds them all:
            // zero through the copy engine instead
            const void* zsrc = r.pin;
            if (!r.pin || state > kPinZeros) {
                r.zeros.resize(std::max(r.zeros.size(), state));
                zsrc = r.zeros.data();
            }
            GMX_CUDA(cudaMemcpyAsync(plan.d_state, zsrc, state, cudaMemcpyHostToDevice, stream));
        } else {
            GMX_CUDA(cudaMemsetAsync(plan.d_state, 0, state, stream));
        }
    }
    return finish();
}

// Least-recently-used eighth of the cache goes when it is full (stream-ordered frees).
static void evict_plans(gmx_exec* ex) {
    std::vector<std::pair<uint64_t, Plan*>> all;
    for (auto& kv : ex->plans)
        for (auto& p : kv.second) all.push_back({p->last_use, p.get()});
    std::sort(all.begin(), all.end());
    const size_t drop = std::max<size_t>(1, all.size() / 8);
    std::unordered_map<const Plan*, bool> doomed;
    for (size_t i = 0; i < drop && i < all.size(); ++i) doomed[all[i].second] = true;
    for (auto& kv : ex->plans) {
        auto& bucket = kv.second;
        for (size_t i = 0; i < bucket.size();) {
            if (doomed.count(bucket[i].get())) {
                if (ex->last == bucket[i].get()) ex->last = nullptr;
                for (auto& r : ex->recent)
                    if (r == bucket[i].get()) r = nullptr;
                bucket.erase(bucket.begin() + i);
                --ex->n_plans;
            } else {
                ++i;
            }
        }
    }
}

// Drop every plan living in the residency arena and rewind the arena (only when no kernel can
// still read it: called at resident_begin once the previous persistent launch has completed).
static void recycle_arena(gmx_exec* ex) {
    for (auto& kv : ex->plans) {
        auto& bucket = kv.second;
        for (size_t i = 0; i < bucket.size();) {
            if (bucket[i]->in_arena) {
                if (ex->last == bucket[i].get()) ex->last = nullptr;
                for (auto& r : ex->recent)
                    if (r == bucket[i].get()) r = nullptr;
                bucket.erase(bucket.begin() + i);
                --ex->n_plans;
            } else {
                ++i;
            }
        }
    }
    ex->res.arena_used = 0;
}

}  // namespace gmx

namespace gmx {

static int set_kernel_attrs(gmx_exec* ex) {
    if (ex->attr_set) return GMX_OK;
    // maximum shared-memory carveout, so two 2-CTA/SM blocks really fit one SM
    GMX_CUDA(cudaFuncSetAttribute(coalesced_step_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<1>()));
    GMX_CUDA(cudaFuncSetAttribute(coalesced_step_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<2>()));
    GMX_CUDA(cudaFuncSetAttribute(coalesced_step_kernel<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    GMX_CUDA(cudaFuncSetAttribute(coalesced_step_kernel<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int occ1 = 0, occ2 = 0;
    GMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, coalesced_step_kernel<1>, kThreads, smem_bytes<1>()));
    GMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, coalesced_step_kernel<2>, kThreads, smem_bytes<2>()));
    ex->occupancy[0] = occ1;
    ex->occupancy[1] = occ2;
    // tcgen05.alloc users are placed one CTA per SM by the runtime (occupancy reports 1 for both
    // shapes), so the 2-CTA shape runs as extra waves, and resident mode uses the 1-CTA shape
    if (occ1 < 1) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, coalesced_step_kernel<2>);
        int smem_sm = 0, smem_blk = 0, regs_sm = 0, resv = 0;
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ex->device);
        cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, ex->device);
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, ex->device);
        cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, ex->device);
        return fail(GMX_ECUDA, "occupancy: 1-CTA shape " + std::to_string(occ1) + "/SM, 2-CTA shape " +
                                   std::to_string(occ2) + "/SM (need 1 and 2); regs " + std::to_string(fa.numRegs) +
                                   " static smem " + std::to_string(fa.sharedSizeBytes) + " dyn " +
                                   std::to_string(smem_bytes<2>()) + " smem/SM " + std::to_string(smem_sm) +
                                   " optin/blk " + std::to_string(smem_blk) + " reserved/blk " + std::to_string(resv) +
                                   " regs/SM " + std::to_string(regs_sm));
    }
    ex->attr_set = true;
    return GMX_OK;
}

// Virtual work items of an inline step over `key` (see next_item).
static int64_t inline_item_count(const gmx_exec* ex, const std::vector<int32_t>& key) {
    int64_t total = 0;
    for (int32_t sl : key) {
        const DevProblem& P = ex->probs[sl].dev;
        if (P.kind == kItemGemm)
            total += (int64_t)((P.rows + kTileRows - 1) / kTileRows) * ((P.cols + P.bn - 1) / P.bn);
        else if (P.kind == kItemGemv)
            total += (P.rows + kInlineGemvRows - 1) / kInlineGemvRows;
        else
            total += (P.rows + kInlineEltwise - 1) / kInlineEltwise;
    }
    return total;
}


// Spin until host ring slot `slot` is free again (its previous step completed on the device).
static int wait_slot_free(gmx_exec* ex, int64_t seq) {
    auto& r = ex->res;
    if (seq < kQueue) return GMX_OK;
    const int64_t need = seq - kQueue + 1;
    volatile int64_t* d = r.hdone + (seq % kQueue);
    for (uint64_t spins = 0; *d < need; ++spins) {
        if ((spins & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(r.stream);
            if (e != cudaErrorNotReady && e != cudaSuccess) return fail(GMX_ECUDA, std::string("resident kernel: ") + cudaGetErrorString(e));
            if (e == cudaSuccess && *d < need) return fail(GMX_ESTATE, "resident kernel exited early");
        }
    }
    return GMX_OK;
}

static int64_t host_ns() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (int64_t)t.tv_sec * 1000000000 + t.tv_nsec;
}

static int publish_step(gmx_exec* ex, const StepDesc& d) {
    auto& r = ex->res;
    int rc;
    if (ex->dbg & 16) {
        const int64_t t0 = host_ns();
        const volatile int64_t* hd = r.hdone + (r.seq % kQueue);
        const bool blocked = r.seq >= kQueue && *hd < r.seq - kQueue + 1;
        if ((rc = wait_slot_free(ex, r.seq))) return rc;
        if (blocked) { r.wait_ns += host_ns() - t0; ++r.waits; }
    } else if ((rc = wait_slot_free(ex, r.seq))) {
        return rc;
    }
    StepDesc* slot = r.hring + (r.seq % kQueue);
    const int64_t tp = (ex->dbg & 16) ? host_ns() : 0;
    std::memcpy(slot, &d, sizeof d);
    __atomic_store_n(r.hpub, r.seq + 1, __ATOMIC_RELEASE);   // x86: ordered after the entry
    if (ex->dbg & 16) r.wr_ns += host_ns() - tp;
    ++r.seq;
    return GMX_OK;
}

// Resident mode: the step goes to the persistent kernel's queue instead of a launch.
static int enqueue_resident_impl(gmx_exec* ex, Plan* plan, const std::vector<int32_t>& key, const int32_t* dep_slots,
                                 int32_t ndep, int32_t flags, bool cached, int64_t* seq_out);
static int enqueue_resident(gmx_exec* ex, Plan* plan, const std::vector<int32_t>& key, const int32_t* dep_slots,
                            int32_t ndep, int32_t flags, bool cached, int64_t* seq_out) {
    if (!(ex->dbg & 16)) return enqueue_resident_impl(ex, plan, key, dep_slots, ndep, flags, cached, seq_out);
    const int64_t t0 = host_ns();
    const int rc = enqueue_resident_impl(ex, plan, key, dep_slots, ndep, flags, cached, seq_out);
    ex->res.pub_ns += host_ns() - t0;
    ++ex->res.pubs;
    return rc;
}
static int enqueue_resident_impl(gmx_exec* ex, Plan* plan, const std::vector<int32_t>& key, const int32_t* dep_slots,
                                 int32_t ndep, int32_t flags, bool cached, int64_t* seq_out) {
    auto& r = ex->res;
    int rc;
    bool pending = false;   // plan uploaded by this call: the step waits on the device for its flag
    if (plan && !plan->uploaded) {
        const int64_t tu = (ex->dbg & 16) ? host_ns() : 0;
        if ((rc = upload_plan(ex, *plan, r.upload))) return rc;
        if (ex->dbg & 16) { r.up_ns += host_ns() - tu; ++r.ups; }
        if (plan->in_arena && stream_write_fn()) {
            pending = true;
        } else {
            GMX_CUDA(cudaStreamSynchronize(r.upload));
        }
    }
    if (plan) {
        plan->stream = r.stream;   // later frees are ordered after the persistent kernel
        plan->last_use = ++ex->clock;
    }
    // Ordering. Steps <= seq - window are complete before this one starts anyway. Inside the
    // window wait for: the producers of the inputs (dep_slots: the last step that wrote each),
    // and the latest step sharing this plan (split-K state) or a slot (outputs). Without
    // dependency information a non-independent step waits for every earlier step.
    const int64_t seq = r.seq;
    const int64_t oldest = seq - r.window + 1;
    bool wait_all = (flags & GMX_LAUNCH_INDEPENDENT) == 0 && ndep == 0;
    int64_t waits[4];
    int nw = 0;
    auto need = [&](int64_t j) {
        if (wait_all || j < oldest || j >= seq) return;
        for (int q = 0; q < nw; ++q)
            if (waits[q] == j) return;
        if (nw == 4) { wait_all = true; return; }
        waits[nw++] = j;
    };
    if (r.last_write.size() < ex->probs.size()) r.last_write.resize(ex->probs.size(), -1);
    if (r.last_read.size() < ex->probs.size()) r.last_read.resize(ex->probs.size(), -1);
    for (int32_t i = 0; i < ndep; ++i) {
        const int32_t sl = dep_slots[i];
        if (sl >= 0 && sl < (int32_t)r.last_write.size()) need(r.last_write[sl]);
    }
    // outputs: the last step that wrote (WAW) or read (WAR) each member slot; split-K state:
    // the last step of this plan
    for (int32_t sl : key) {
        need(r.last_write[sl]);
        need(r.last_read[sl]);
    }
    if (plan && plan->res_epoch == r.epoch) need(plan->res_seq);
    StepDesc d{};
    d.probs = ex->d_probs;
    if (plan) {
        d.items = plan->d_items;
        d.cta_off = plan->d_off;
        d.ws = plan->d_ws;
        d.counters = plan->d_counters;
        d.grid = plan->stats.grid;
    } else {   // inline step: list i (< #items) enumerates the members' items g with g % grid == i
        d.grid = (int32_t)std::max<int64_t>(1, std::min<int64_t>(r.grid, inline_item_count(ex, key)));
        d.inline_n = (int32_t)key.size();
        for (size_t i = 0; i < key.size(); ++i) d.inline_slots[i] = key[i];
    }
    d.wait_all = wait_all ? 1 : 0;
    if (pending) {   // copy-engine write of seq + 1 after the plan's copies, on the same stream
        d.stop = 2;
        const CUresult cr = stream_write_fn()(r.upload, reinterpret_cast<CUdeviceptr>(&r.dq->plan_ready[seq % kQueue]),
                                              (cuuint32_t)(seq + 1), 0);
        if (cr != CUDA_SUCCESS) return fail(GMX_ECUDA, "cuStreamWriteValue32 failed: " + std::to_string((int)cr));
    }
    // nwait -1: no wait, only the proxy fence (inputs of already-observed producers)
    d.nwait = wait_all ? 0 : (nw == 0 && ((flags & GMX_LAUNCH_FENCE) || ndep > 0) ? -1 : nw);
    for (int q = 0; q < nw; ++q) d.wait_steps[q] = waits[q];
    if (d.grid > r.grid) return fail(GMX_ESTATE, "plan grid exceeds the resident grid");
    if ((rc = publish_step(ex, d))) return rc;
    for (int32_t sl : key) r.last_write[sl] = seq;
    for (int32_t i = 0; i < ndep; ++i)
        if (dep_slots[i] >= 0 && dep_slots[i] < (int32_t)r.last_read.size()) r.last_read[dep_slots[i]] = seq;
    if (plan) {
        plan->res_seq = seq;
        plan->res_epoch = r.epoch;
    }
    if (plan) {
        plan->stats.cached = cached;
        ex->last = plan;
    }
    if (seq_out) *seq_out = seq;
    return GMX_OK;
}

// Per-step launches: true if this launch writes a slot read or written, or reads a slot written,
// by a launch since the last fully ordered one (PDL launches of independent steps may overlap).
// A hazard resets the window to this launch (it will be launched fully ordered).
static bool per_step_hazard(gmx_exec* ex, const std::vector<int32_t>& key, const int32_t* dep_slots, int32_t ndep) {
    const size_t ns = ex->probs.size();
    if (ex->hz_wr.size() < ns) {
        ex->hz_wr.resize(ns, 0);
        ex->hz_rd.resize(ns, 0);
    }
    bool hazard = false;
    for (int32_t sl : key) hazard |= ex->hz_wr[sl] || ex->hz_rd[sl];
    for (int32_t i = 0; i < ndep; ++i) {
        const int32_t sl = dep_slots[i];
        if (sl >= 0 && (size_t)sl < ns) hazard |= ex->hz_wr[sl] != 0;
    }
    if (hazard) {
        for (int32_t sl : ex->hz_touched) ex->hz_wr[sl] = ex->hz_rd[sl] = 0;
        ex->hz_touched.clear();
    }
    for (int32_t sl : key) {
        if (!ex->hz_wr[sl] && !ex->hz_rd[sl]) ex->hz_touched.push_back(sl);
        ex->hz_wr[sl] = 1;
    }
    for (int32_t i = 0; i < ndep; ++i) {
        const int32_t sl = dep_slots[i];
        if (sl < 0 || (size_t)sl >= ns) continue;
        if (!ex->hz_wr[sl] && !ex->hz_rd[sl]) ex->hz_touched.push_back(sl);
        ex->hz_rd[sl] = 1;
    }
    return hazard;
}

}  // namespace gmx

using namespace gmx;

extern "C" {

int gmx_exec_resident_begin(gmx_exec* ex, void* stream_ptr) { return gmx_exec_resident_begin_ex(ex, stream_ptr, 0); }

int gmx_exec_resident_begin_ex(gmx_exec* ex, void* stream_ptr, int32_t hold) {
    if (!ex) return fail(GMX_EINVAL, "null argument");
    auto& r = ex->res;
    if (r.active) return fail(GMX_ESTATE, "already resident");
    if (ex->tracing) return fail(GMX_ESTATE, "tracing is not supported in resident mode");
    if (!ex->cache_plans) return fail(GMX_ESTATE, "resident mode needs cache_plans");
    if (ex->ctas_per_sm != 1) return fail(GMX_ESTATE, "resident mode needs ctas_per_sm = 1 (all CTAs co-resident)");
    if (!r.hring) {
        GMX_CUDA(cudaHostAlloc(&r.hring, kQueue * sizeof(StepDesc), cudaHostAllocMapped));
        GMX_CUDA(cudaHostAlloc(&r.hpub, 64, cudaHostAllocMapped));
        GMX_CUDA(cudaHostAlloc(&r.hdone, kQueue * sizeof(int64_t), cudaHostAllocMapped));
        GMX_CUDA(cudaHostGetDevicePointer((void**)&r.hring_d, r.hring, 0));
        GMX_CUDA(cudaHostGetDevicePointer((void**)&r.hpub_d, r.hpub, 0));
        GMX_CUDA(cudaHostGetDevicePointer((void**)&r.hdone_d, r.hdone, 0));
        GMX_CUDA(cudaMalloc(&r.dq, sizeof(DevQueue)));
        GMX_CUDA(cudaStreamCreateWithFlags(&r.upload, cudaStreamNonBlocking));
        r.arena_size = (size_t)1 << 30;      // 1 GB of the 180: wall-clock serving builds ~2000 plans per 0.3 s
        GMX_CUDA(cudaMalloc(&r.arena, r.arena_size));
        GMX_CUDA(cudaMemset(r.arena, 0, r.arena_size));
        r.pin_size = (size_t)64 << 20;
        GMX_CUDA(cudaHostAlloc(&r.pin, r.pin_size, cudaHostAllocDefault));
        std::memset(r.pin, 0, kPinZeros);
    }
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    int rc;
    if ((rc = ensure_table(ex, stream))) return rc;
    // ring entries are read only once published (hpub), so neither ring needs clearing; the
    // completion flags and the device counters restart from zero with the new residency's seq
    std::memset(r.hdone, 0, kQueue * sizeof(int64_t));
    __atomic_store_n(r.hpub, (int64_t)0, __ATOMIC_RELEASE);
    __atomic_store_n(r.hpub + 1, (int64_t)(hold ? 0 : 1), __ATOMIC_RELEASE);   // go flag
    GMX_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(r.dq) + offsetof(DevQueue, published), 0,
                             sizeof(DevQueue) - offsetof(DevQueue, published), stream));
    if ((rc = set_kernel_attrs(ex))) return rc;
    r.grid = ex->num_sms * ex->ctas_per_sm;
    // plans first built in earlier residencies live in the arena: once it is half full and the
    // previous persistent launch has finished (nothing can read them), drop them and rewind
    if (r.arena_used > r.arena_size / 2 && (!r.stream || cudaStreamQuery(r.stream) == cudaSuccess)) {
        GMX_CUDA(cudaMemsetAsync(r.arena, 0, r.arena_used, stream));   // ordered before the launch below
        recycle_arena(ex);
    }
    r.seq = 0;
    r.pin_used = kPinZeros;
    r.stream = stream;
    ++r.epoch;
    r.last_write.assign(ex->probs.size(), -1);
    r.last_read.assign(ex->probs.size(), -1);
    KernelArgs args{};
    args.dbg = ex->dbg;
    args.independent = 1;
    args.early_trigger = 0;
    args.resident = 1;
    args.dq = r.dq;
    args.hring = r.hring_d;
    args.hpub = r.hpub_d;
    args.hdone = r.hdone_d;
    args.window = r.window;
    args.grab_ahead = ex->res.grab_ahead;
    if (r.rtrace_steps > 0) {
        // (step, CTA) stamps + one row of relay stamps + one row of host-report stamps
        const size_t nb = ((size_t)r.rtrace_steps * r.grid * 8 + 2 * (size_t)r.rtrace_steps) * sizeof(uint64_t);
        if (!r.rtrace) GMX_CUDA(cudaMalloc(&r.rtrace, nb));
        GMX_CUDA(cudaMemsetAsync(r.rtrace, 0, nb, stream));
        args.rtrace = r.rtrace;
        args.rtrace_steps = r.rtrace_steps;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(r.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = ex->ctas_per_sm == 2 ? smem_bytes<2>() : smem_bytes<1>();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident, or the launch fails
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ex->ctas_per_sm == 2)
        GMX_CUDA(cudaLaunchKernelEx(&cfg, coalesced_step_kernel<2>, args));
    else
        GMX_CUDA(cudaLaunchKernelEx(&cfg, coalesced_step_kernel<1>, args));
    r.active = true;
    return GMX_OK;
}

int gmx_exec_resident_release(gmx_exec* ex) {
    if (!ex) return fail(GMX_EINVAL, "null argument");
    if (!ex->res.hpub) return fail(GMX_ESTATE, "not resident");
    __atomic_store_n(ex->res.hpub + 1, (int64_t)1, __ATOMIC_RELEASE);
    return GMX_OK;
}

int gmx_exec_resident_device_ns(gmx_exec* ex, int64_t* out) {
    if (!ex || !out) return fail(GMX_EINVAL, "null argument");
    if (!ex->res.dq) return fail(GMX_ESTATE, "never resident");
    uint64_t t[3];
    GMX_CUDA(cudaMemcpy(t, &ex->res.dq->t_first, sizeof t, cudaMemcpyDeviceToHost));
    *out = (int64_t)(t[1] - t[0]);
    ex->res.relay_ns = (int64_t)(t[2] - t[0]);
    return GMX_OK;
}

int gmx_exec_resident_read_rtrace(gmx_exec* ex, uint64_t* out, int64_t capacity, int32_t* grid) {
    if (!ex || !grid) return fail(GMX_EINVAL, "null argument");
    auto& r = ex->res;
    *grid = r.grid;
    const int64_t n = (int64_t)r.rtrace_steps * r.grid * 8 + 2 * (int64_t)r.rtrace_steps;
    if (!r.rtrace || capacity < n) return fail(GMX_EINVAL, "no rtrace or capacity too small");
    GMX_CUDA(cudaDeviceSynchronize());
    GMX_CUDA(cudaMemcpy(out, r.rtrace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return GMX_OK;
}

int gmx_exec_resident_active(const gmx_exec* ex) { return ex && ex->res.active ? 1 : 0; }

int gmx_exec_resident_step_done(gmx_exec* ex, int64_t seq) {
    if (!ex || seq < 0) return 0;
    auto& r = ex->res;
    if (!r.hdone) return 0;
    if (seq < r.seq - kQueue) return 1;   // its ring slot was recycled, so it completed
    return ((volatile int64_t*)r.hdone)[seq % kQueue] >= seq + 1 ? 1 : 0;
}

int gmx_exec_resident_sm_clock(gmx_exec* ex, double* mhz, int64_t* span_ns) {
    if (!ex || !mhz) return fail(GMX_EINVAL, "null argument");
    if (!ex->res.dq) return fail(GMX_ESTATE, "never resident");
    if (ex->res.active) return fail(GMX_ESTATE, "residency still active");
    uint64_t t[6];   // t_first t_last t_relay t_stop c_first c_stop
    GMX_CUDA(cudaMemcpy(t, &ex->res.dq->t_first, sizeof t, cudaMemcpyDeviceToHost));
    const double dt = (double)(t[3] - t[0]);
    *mhz = dt > 0 ? (double)(t[5] - t[4]) / dt * 1e3 : 0.0;
    if (span_ns) *span_ns = (int64_t)dt;
    return GMX_OK;
}

int gmx_exec_resident_relay_ns(gmx_exec* ex, int64_t* out) {
    if (!ex || !out) return fail(GMX_EINVAL, "null argument");
    *out = ex->res.relay_ns;
    return GMX_OK;
}

int gmx_exec_resident_end(gmx_exec* ex) {
    if (!ex) return fail(GMX_EINVAL, "null argument");
    auto& r = ex->res;
    if (!r.active) return fail(GMX_ESTATE, "not resident");
    if (ex->dbg & 16) {
        std::fprintf(stderr, "[gmx resident] steps %lld, host blocked on a full ring %lld times, %.3f ms; enqueue %.3f ms over %lld; plan uploads %lld, %.3f ms\n",
                     (long long)r.seq, (long long)r.waits, r.wait_ns / 1e6, r.pub_ns / 1e6, (long long)r.pubs,
                     (long long)r.ups, r.up_ns / 1e6);
        std::fprintf(stderr, "[gmx resident] ring entry writes %.3f ms\n", r.wr_ns / 1e6);
        r.wait_ns = r.waits = r.pub_ns = r.pubs = r.up_ns = r.ups = r.wr_ns = 0;
    }
    __atomic_store_n(r.hpub + 1, (int64_t)1, __ATOMIC_RELEASE);   // a held start is released
    StepDesc d{};
    d.stop = 1;
    d.nwait = 0;
    int rc = publish_step(ex, d);
    r.active = false;
    for (void* p : r.graveyard) cudaFreeAsync(p, r.stream);   // after the persistent kernel
    r.graveyard.clear();
    return rc;
}

int gmx_exec_resident_completed(gmx_exec* ex, int64_t* out) {
    if (!ex || !out) return fail(GMX_EINVAL, "null argument");
    auto& r = ex->res;
    // steps complete out of order; report the longest completed prefix
    int64_t done = 0;
    const int64_t lo = std::max<int64_t>(0, r.seq - kQueue);
    done = lo;
    for (int64_t q = lo; q < r.seq; ++q) {
        if (((volatile int64_t*)r.hdone)[q % kQueue] >= q + 1) done = q + 1; else break;
    }
    *out = done;
    return GMX_OK;
}

int gmx_exec_create(int32_t device, gmx_exec** out) {
    if (!out) return fail(GMX_EINVAL, "null argument");
    int ndev = 0;
    GMX_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(GMX_EINVAL, "no such CUDA device");
    cudaDeviceProp prop;
    GMX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(GMX_ECUDA, std::string("executor targets sm_100a; device is ") + prop.name);
    GMX_CUDA(cudaSetDevice(device));
    {   // keep freed plan memory in the stream-ordered pool (plans churn on dynamic workloads)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t threshold = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
        }
    }
    auto* ex = new gmx_exec();
    ex->device = device;
    ex->num_sms = prop.multiProcessorCount;
    *out = ex;
    return GMX_OK;
}

void gmx_exec_destroy(gmx_exec* ex) {
    if (!ex) return;
    cudaSetDevice(ex->device);
    if (ex->res.active) {
        gmx_exec_resident_end(ex);
        cudaStreamSynchronize(ex->res.stream);
    }
    if (ex->res.hring) {
        cudaDeviceSynchronize();
        cudaFreeHost(ex->res.hring);
        cudaFreeHost(ex->res.hpub);
        cudaFreeHost(ex->res.hdone);
        cudaFree(ex->res.dq);
        cudaStreamDestroy(ex->res.upload);
    }
    ex->plans.clear();
    ex->uncached.reset();
    if (ex->res.arena) cudaFree(ex->res.arena);   // after the plans that may live in it
    if (ex->res.pin) cudaFreeHost(ex->res.pin);
    if (ex->d_probs) cudaFree(ex->d_probs);
    if (ex->ws) cudaFree(ex->ws);
    if (ex->counters) cudaFree(ex->counters);
    delete ex;
}

int gmx_exec_num_sms(const gmx_exec* ex, int32_t* out) {
    if (!ex || !out) return fail(GMX_EINVAL, "null argument");
    *out = ex->num_sms;
    return GMX_OK;
}

int gmx_exec_register(gmx_exec* ex, const gmx_problem_desc* d, int32_t* out_slot) {
    if (!ex || !d || !out_slot) return fail(GMX_EINVAL, "null argument");
    HostProblem hp;
    hp.desc = *d;
    DevProblem& P = hp.dev;
    std::memset(&P, 0, sizeof P);
    P.out = d->c;
    P.bias = d->bias;
    P.act = d->activation;
    P.in_dt = d->in_dtype;
    P.out_dt = d->out_dtype;
    P.ld_out = d->ldc;
    if (d->activation < GMX_ACT_NONE || d->activation > GMX_ACT_GELU) return fail(GMX_EINVAL, "unknown activation");
    if ((d->in_dtype != GMX_ST_BF16 && d->in_dtype != GMX_ST_F32) ||
        (d->out_dtype != GMX_ST_BF16 && d->out_dtype != GMX_ST_F32))
        return fail(GMX_EINVAL, "unknown storage dtype");
    if (!d->a || !d->c) return fail(GMX_EINVAL, "operand pointer is NULL");
    const int64_t isz = d->in_dtype == GMX_ST_F32 ? 4 : 2, osz = d->out_dtype == GMX_ST_F32 ? 4 : 2;
    if (d->op == GMX_OP_GEMM) {
        if (d->m < 1 || d->n < 1 || d->k < 1) return fail(GMX_EINVAL, "gemm dims must be >= 1");
        if (d->m >= (1 << 30) || d->n >= (1 << 30) || d->k >= (1 << 30)) return fail(GMX_EINVAL, "gemm dims too large");
        if (!d->b) return fail(GMX_EINVAL, "gemm B operand is NULL");
        if (d->lda < d->k || d->ldb < d->k || d->ldc < d->n) return fail(GMX_EINVAL, "leading dimension too small");
        if ((d->lda * isz) % 16 || (d->ldb * isz) % 16)
            return fail(GMX_EINVAL, "lda/ldb rows must be multiples of 16 bytes (TMA strides)");
        if ((reinterpret_cast<uintptr_t>(d->a) | reinterpret_cast<uintptr_t>(d->b)) & 15)
            return fail(GMX_EINVAL, "A/B must be 16-byte aligned");
        // orientation: the side that needs fewer (128 + BN) x K tile loads goes on UMMA-M
        auto traffic = [](int64_t R, int64_t Cc) {
            const int bn = choose_bn(Cc);
            return ((R + kTileRows - 1) / kTileRows) * ((Cc + bn - 1) / bn) * (int64_t)(kTileRows + bn);
        };
        const bool swap = traffic(d->n, d->m) < traffic(d->m, d->n);
        P.kind = kItemGemm;
        P.swap = swap;
        P.rows = (int32_t)(swap ? d->n : d->m);
        P.cols = (int32_t)(swap ? d->m : d->n);
        P.K = (int32_t)d->k;
        P.bn = choose_bn(P.cols);
        if (d->tile_n != 0) {   // tuned tile (autotune.py); multiples of 64 keep output boxes per tile
            if (d->tile_n != 64 && d->tile_n != 128) return fail(GMX_EINVAL, "tile_n must be 0, 64 or 128");
            P.bn = d->tile_n;
        }
        const bool f32 = d->in_dtype == GMX_ST_F32;   // fp32 operands: tf32 UMMA
        P.kblocks = (int32_t)((d->k + kblock_elems(f32) - 1) / kblock_elems(f32));
        const void* rows_ptr = swap ? d->b : d->a;
        const void* cols_ptr = swap ? d->a : d->b;
        const int64_t rows_ld = swap ? d->ldb : d->lda, cols_ld = swap ? d->lda : d->ldb;
        int rc;
        if ((rc = make_tmap(&P.tm_rows, rows_ptr, P.rows, d->k, rows_ld, kTileRows, f32)) ||
            (rc = make_tmap(&P.tm_cols, cols_ptr, P.cols, d->k, cols_ld, P.bn, f32)))
            return rc;
        // output tensor map (TMA-store epilogue) when C allows 16-byte-aligned rows
        P.tma_out = 0;
        if ((reinterpret_cast<uintptr_t>(d->c) & 15) == 0 && (d->ldc * osz) % 16 == 0) {
            auto fn = encode_fn();
            const int inner = (int)(128 / osz);
            cuuint64_t dims[2] = {(cuuint64_t)d->n, (cuuint64_t)d->m};
            cuuint64_t strides[1] = {(cuuint64_t)(d->ldc * osz)};
            // swapped tiles store a whole epilogue pass per box: 16 KB staging / (32 x 128 B) rows
            cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)(swap ? 32 * (16384 / (128 * 32 * (int)osz)) : kTileRows)};
            cuuint32_t estr[2] = {1, 1};
            if (fn && fn(&P.tm_out, d->out_dtype == GMX_ST_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         2, d->c, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                P.tma_out = 1;
        }
        hp.op_bytes = isz * (d->m * d->k + d->k * d->n) + osz * d->m * d->n;
        hp.flops = 2 * d->m * d->n * d->k;
    } else if (d->op == GMX_OP_GEMV) {
        if (d->m < 1 || d->n < 1 || d->m >= (1 << 30) || d->n >= (1 << 30)) return fail(GMX_EINVAL, "bad gemv dims");
        if (!d->b) return fail(GMX_EINVAL, "gemv x operand is NULL");
        if (d->lda < d->n) return fail(GMX_EINVAL, "leading dimension too small");
        P.kind = kItemGemv;
        P.rows = (int32_t)d->m;
        P.cols = (int32_t)d->n;
        P.in0 = d->a;
        P.in1 = d->b;
        P.ld_in0 = d->lda;
        // W as a 2D tensor ({256-element x R-row} boxes, no swizzle) for the staged path
        P.bn = 0;
        const bool f32 = d->in_dtype == GMX_ST_F32;
        if (((reinterpret_cast<uintptr_t>(d->a) | reinterpret_cast<uintptr_t>(d->b)) & 15) == 0 &&
            (d->lda * isz) % 16 == 0 && d->n % (16 / isz) == 0) {
            auto fn = encode_fn();
            cuuint64_t dims[2] = {(cuuint64_t)d->n, (cuuint64_t)d->m};
            cuuint64_t strides[1] = {(cuuint64_t)(d->lda * isz)};
            cuuint32_t box[2] = {(cuuint32_t)kGvBoxCols, (cuuint32_t)gv_box_rows(f32)};
            cuuint32_t estr[2] = {1, 1};
            if (fn && fn(&P.tm_rows, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                         const_cast<void*>(d->a), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                P.bn = 1;
        }
        hp.op_bytes = isz * (d->m * d->n + d->n) + osz * d->m;
        hp.flops = 2 * d->m * d->n;
    } else if (d->op == GMX_OP_ELEMENTWISE) {
        if (d->m < 1 || d->m >= ((int64_t)1 << 31)) return fail(GMX_EINVAL, "bad elementwise length");
        if (d->in_dtype != d->out_dtype) return fail(GMX_EINVAL, "elementwise keeps its dtype");
        P.kind = kItemEltwise;
        P.rows = (int32_t)d->m;
        P.in0 = d->a;
        hp.op_bytes = isz * d->m + osz * d->m;
        hp.flops = d->m;
    } else {
        return fail(GMX_EINVAL, "unknown op");
    }
    hp.live = true;
    int32_t slot = -1;
    for (size_t i = 0; i < ex->probs.size(); ++i)
        if (!ex->probs[i].live) { slot = (int32_t)i; break; }
    if (slot < 0) {
        slot = (int32_t)ex->probs.size();
        ex->probs.push_back(hp);
    } else {
        ex->probs[slot] = hp;
    }
    ex->table_dirty = true;
    *out_slot = slot;
    return GMX_OK;
}

int gmx_exec_unregister(gmx_exec* ex, int32_t slot) {
    if (!ex || slot < 0 || slot >= (int32_t)ex->probs.size() || !ex->probs[slot].live)
        return fail(GMX_EINVAL, "bad slot");
    ex->probs[slot].live = false;
    // plans referencing the slot become invalid
    for (auto& kv : ex->plans) {
        auto& bucket = kv.second;
        for (size_t i = 0; i < bucket.size();) {
            if (std::binary_search(bucket[i]->key.begin(), bucket[i]->key.end(), slot)) {
                if (ex->last == bucket[i].get()) ex->last = nullptr;
                bucket.erase(bucket.begin() + i);
                --ex->n_plans;
            } else {
                ++i;
            }
        }
    }
    return GMX_OK;
}

int gmx_exec_launch(gmx_exec* ex, const int32_t* slots, int32_t n, void* stream_ptr) {
    return gmx_exec_launch_ex(ex, slots, n, stream_ptr, 0);
}

int gmx_exec_launch_ex(gmx_exec* ex, const int32_t* slots, int32_t n, void* stream_ptr, int32_t flags) {
    return gmx_exec_launch_deps(ex, slots, n, nullptr, 0, stream_ptr, flags, nullptr);
}

int gmx_exec_launch_deps(gmx_exec* ex, const int32_t* slots, int32_t n, const int32_t* dep_slots, int32_t ndep,
                         void* stream_ptr, int32_t flags, int64_t* step_seq) {
    if (!ex || (n > 0 && !slots) || (ndep > 0 && !dep_slots)) return fail(GMX_EINVAL, "null argument");
    if (step_seq) *step_seq = -1;
    if (n == 0) return GMX_OK;
    if (ndep > 0) flags &= ~GMX_LAUNCH_INDEPENDENT;   // reads earlier outputs
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_ptr);
    std::vector<int32_t>& key = ex->key_scratch;
    key.assign(slots, slots + n);
    std::sort(key.begin(), key.end());
    uint64_t h = 0x6A09E667F3BCC909ull ^ (uint64_t)n;
    for (int32_t s : key) {
        if (s < 0 || s >= (int32_t)ex->probs.size() || !ex->probs[s].live) return fail(GMX_EINVAL, "bad slot");
        h = mix64(h ^ (uint64_t)(uint32_t)s);
    }
    int rc;
    if ((rc = ensure_table(ex, stream))) return rc;
    if (ex->inline_plans && !ex->tracing && n <= kInlineMaxMembers) {
        // a slot set seen for the first time (wall-clock serving: most step compositions are
        // one-offs) runs as an INLINE step — the device enumerates the work items — instead of
        // paying for a host plan build + upload; a recurring one gets a cached LPT plan
        bool hit = false;
        auto pit = ex->plans.find(h);
        if (pit != ex->plans.end())
            for (auto& p : pit->second) hit |= p->key == key;
        if (!hit) {
            // sightings per slot set: a direct-mapped table (no rehash / clear pauses on the
            // serving path); a collision just restarts that set's count
            auto& e = ex->inline_seen[h & (kSeenSlots - 1)];
            if (e.first != h) e = {h, 0};
            if (e.second++ < ex->inline_promote) {
                const int64_t total = inline_item_count(ex, key);
                const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ex->num_sms, total));
                if (ex->res.active) {   // resident: the slots ride in the step descriptor
                    ++ex->inline_launches;
                    return enqueue_resident(ex, nullptr, key, dep_slots, ndep, flags, false, step_seq);
                }
                if ((total + grid - 1) / grid <= kInlineMaxItems) {
                    if ((rc = set_kernel_attrs(ex))) return rc;
                    const bool hazard = per_step_hazard(ex, key, dep_slots, ndep);
                    KernelArgs args{};
                    args.probs = ex->d_probs;
                    args.dbg = ex->dbg;
                    args.independent = (flags & GMX_LAUNCH_INDEPENDENT) != 0 ? 1 : 0;
                    args.early_trigger = ex->early_trigger ? 1 : 0;
                    args.inline_n = n;
                    for (int32_t i = 0; i < n; ++i) args.inline_slots[i] = key[i];
                    cudaLaunchConfig_t cfg{};
                    cfg.gridDim = dim3((unsigned)grid);
                    cfg.blockDim = dim3(kThreadsPerStep);
                    cfg.dynamicSmemBytes = smem_bytes<1>();
                    cfg.stream = stream;
                    cudaLaunchAttribute attr[1];
                    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    attr[0].val.programmaticStreamSerializationAllowed = ex->pdl && !hazard ? 1 : 0;
                    cfg.attrs = attr;
                    cfg.numAttrs = 1;
                    GMX_CUDA(cudaLaunchKernelEx(&cfg, coalesced_step_kernel<1>, args));
                    ++ex->inline_launches;
                    return GMX_OK;
                }
            }
        }
    }
    Plan* plan = nullptr;
    bool cached = false;
    if (ex->cache_plans) {
        // per-mode split (split_pct*): a resident step entering an idle device (nothing published
        // earlier still in flight) takes the latency plan
        int mode = ex->res.active ? kPlanResident : kPlanStep;
        if (ex->res.active && ex->split_pct_idle > 0 &&
            (ex->res.seq == 0 || gmx_exec_resident_step_done(ex, ex->res.seq - 1)))
            mode = kPlanIdle;
        auto& bucket = ex->plans[h];
        for (auto& p : bucket)
            if (p->key == key && p->mode == mode) {
                plan = p.get();
                cached = true;
                break;
            }
        if (!plan) {
            // no eviction while resident: queued steps may still reference any cached plan
            if (ex->n_plans >= ex->plan_capacity && !ex->res.active) evict_plans(ex);
            auto p = std::make_unique<Plan>();
            if ((rc = build_plan(ex, key, *p, mode))) return rc;
            p->key = key;
            p->mode = (int8_t)mode;
            plan = p.get();
            ex->plans[h].push_back(std::move(p));
            ++ex->n_plans;
        }
    } else {
        if (ex->res.active) return fail(GMX_ESTATE, "resident mode needs cache_plans");
        ex->uncached = std::make_unique<Plan>();   // the previous one is freed stream-ordered
        if ((rc = build_plan(ex, key, *ex->uncached, kPlanStep))) return rc;
        plan = ex->uncached.get();
    }
    if (ex->res.active) return enqueue_resident(ex, plan, key, dep_slots, ndep, flags, cached, step_seq);
    // multi-stream: a plan's split-K state and outputs must not be used by two launches at once
    if (ex->multi_stream && plan->done_ev && plan->stream != stream)
        GMX_CUDA(cudaStreamWaitEvent(stream, plan->done_ev, 0));
    if ((rc = upload_plan(ex, *plan, stream))) return rc;
    plan->stream = stream;
    plan->last_use = ++ex->clock;
    if ((rc = set_kernel_attrs(ex))) return rc;
    if (ex->tracing && (int64_t)plan->items.size() > ex->trace_cap) {
        if (ex->trace) GMX_CUDA(cudaFree(ex->trace));
        ex->trace_cap = std::max<int64_t>(1024, (int64_t)plan->items.size());
        // item rows + one row of kernel stamps per CTA
        GMX_CUDA(cudaMalloc(&ex->trace, (ex->trace_cap + 2 * kMaxGrid) * 8 * sizeof(uint64_t)));
    }
    if (ex->tracing) {
        GMX_CUDA(cudaMemsetAsync(ex->trace, 0, plan->items.size() * 8 * sizeof(uint64_t), stream));
        ex->trace_items = (int64_t)plan->items.size();
    }
    // independent only if the caller says so AND this plan's split-K state is not possibly in
    // use by a still-running recent launch
    bool independent = (flags & GMX_LAUNCH_INDEPENDENT) != 0 && !ex->tracing;
    for (const Plan* r : ex->recent) independent &= (r != plan);
    // a slot hazard with any launch since the last fully ordered one: launch fully ordered
    const bool hazard = per_step_hazard(ex, key, dep_slots, ndep);
    KernelArgs args{ex->d_probs, plan->d_items, plan->d_off, plan->d_off + plan->stats.grid + 1, plan->d_ws,
                    plan->d_counters, ex->tracing ? ex->trace : nullptr, ex->dbg, independent ? 1 : 0,
                    ex->early_trigger ? 1 : 0};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(plan->stats.grid);
    cfg.blockDim = dim3(kThreadsPerStep);
    cfg.dynamicSmemBytes = ex->ctas_per_sm == 2 ? smem_bytes<2>() : smem_bytes<1>();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = ex->pdl && !hazard ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ex->ctas_per_sm == 2)
        GMX_CUDA(cudaLaunchKernelEx(&cfg, coalesced_step_kernel<2>, args));
    else
        GMX_CUDA(cudaLaunchKernelEx(&cfg, coalesced_step_kernel<1>, args));
    if (ex->multi_stream) {
        if (!plan->done_ev) GMX_CUDA(cudaEventCreateWithFlags(&plan->done_ev, cudaEventDisableTiming));
        GMX_CUDA(cudaEventRecord(plan->done_ev, stream));
    }
    ex->recent[2] = ex->recent[1];
    ex->recent[1] = ex->recent[0];
    ex->recent[0] = plan;
    plan->stats.cached = cached;
    ex->last = plan;
    return GMX_OK;
}

int gmx_exec_last_plan(const gmx_exec* ex, gmx_plan_stats* out) {
    if (!ex || !out) return fail(GMX_EINVAL, "null argument");
    if (!ex->last) return fail(GMX_ESTATE, "no launch yet");
    *out = ex->last->stats;
    return GMX_OK;
}

int gmx_exec_clear_plans(gmx_exec* ex) {
    if (!ex) return fail(GMX_EINVAL, "null argument");
    ex->plans.clear();
    ex->n_plans = 0;
    ex->last = nullptr;
    return GMX_OK;
}

int gmx_exec_set_option(gmx_exec* ex, const char* name, int64_t value) {
    if (!ex || !name) return fail(GMX_EINVAL, "null argument");
    const std::string n(name);
    if (ex->res.active) return fail(GMX_ESTATE, "options cannot change while resident");
    if (n == "max_split") {
        if (value < 1 || value > 255) return fail(GMX_EINVAL, "max_split must be in [1, 255]");
        ex->max_split = value;
    } else if (n == "rtrace") {
        if (value < 0 || value > 100000) return fail(GMX_EINVAL, "rtrace must be in [0, 100000]");
        if (ex->res.rtrace) { cudaFree(ex->res.rtrace); ex->res.rtrace = nullptr; }
        ex->res.rtrace_steps = (int32_t)value;
        return GMX_OK;
    } else if (n == "inline_plans") {
        if (ex->ctas_per_sm != 1 && value) return fail(GMX_EINVAL, "inline steps use the 1-CTA kernel shape");
        ex->inline_plans = value != 0;
        return GMX_OK;
    } else if (n == "inline_promote") {
        if (value < 0 || value > 1000000) return fail(GMX_EINVAL, "inline_promote must be >= 0");
        ex->inline_promote = (int)value;
        return GMX_OK;
    } else if (n == "grab_ahead") {
        if (value < 0 || value > 64) return fail(GMX_EINVAL, "grab_ahead must be in [0, 64]");
        ex->res.grab_ahead = (int)value;
        return GMX_OK;
    } else if (n == "resident_window") {
        if (value < 1 || value > kMaxWindow) return fail(GMX_EINVAL, "resident_window must be in [1, 512]");
        ex->res.window = (int)value;
        return GMX_OK;
    } else if (n == "ctas_per_sm") {
        if (value != 1 && value != 2) return fail(GMX_EINVAL, "ctas_per_sm must be 1 or 2");
        ex->ctas_per_sm = (int)value;
    } else if (n == "gemv_staged") {
        ex->gemv_staged = value != 0;   // applies to plans built afterwards (clear_plans)
    } else if (n == "split_pct" || n == "split_pct_step") {   // split_pct sets both modes
        if (value < 10 || value > 2000) return fail(GMX_EINVAL, "split_pct must be in [10, 2000]");
        if (n == "split_pct") ex->split_pct = value;
        ex->split_pct_step = value;
    } else if (n == "split_pct_idle") {   // 0: idle-device resident steps use the resident plan
        if (value != 0 && (value < 10 || value > 2000)) return fail(GMX_EINVAL, "split_pct_idle must be 0 or in [10, 2000]");
        ex->split_pct_idle = value;
    } else if (n == "cache_plans") {
        ex->cache_plans = value != 0;
    } else if (n == "plan_capacity") {
        if (value < 1) return fail(GMX_EINVAL, "plan_capacity must be >= 1");
        ex->plan_capacity = (size_t)value;
    } else if (n == "multi_stream") {
        ex->multi_stream = value != 0;
        return GMX_OK;
    } else if (n == "early_trigger") {
        ex->early_trigger = value != 0;
        return GMX_OK;
    } else if (n == "pdl") {
        ex->pdl = value != 0;
        return GMX_OK;
    } else if (n == "dbg") {
        ex->dbg = (int32_t)value;
        return GMX_OK;
    } else if (n == "trace") {
        ex->tracing = value != 0;
        return GMX_OK;
    } else {
        return fail(GMX_EINVAL, "unknown option " + n);
    }
    ex->plans.clear();
    ex->n_plans = 0;
    ex->last = nullptr;
    return GMX_OK;
}

const char* gmx_exec_last_error(void) { return g_err.c_str(); }

int gmx_exec_stream_retired(gmx_exec* ex, void* stream_ptr) {
    if (!ex) return fail(GMX_EINVAL, "null argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_ptr);
    GMX_CUDA(cudaStreamSynchronize(st));
    for (auto& kv : ex->plans)
        for (auto& p : kv.second)
            if (p->stream == st) p->stream = nullptr;   // later frees go to the legacy stream
    if (ex->uncached && ex->uncached->stream == st) ex->uncached->stream = nullptr;
    return GMX_OK;
}

int gmx_exec_read_trace(const gmx_exec* ex, uint64_t* stamps, int32_t* items, int32_t* cta_off,
                        int32_t capacity, int32_t* n_items, int32_t* grid) {
    if (!ex || !n_items || !grid) return fail(GMX_EINVAL, "null argument");
    if (!ex->tracing || !ex->last) return fail(GMX_ESTATE, "tracing off or no launch");
    const int32_t n = (int32_t)ex->trace_items;
    *n_items = n;
    *grid = ex->last->stats.grid;
    if (capacity < n) return GMX_OK;
    GMX_CUDA(cudaDeviceSynchronize());
    // capacity >= n + grid: the per-CTA kernel stamp rows (entry, prologue done, loops done, exit) too
    const int64_t rows = capacity >= n + *grid ? (int64_t)n + *grid : n;
    GMX_CUDA(cudaMemcpy(stamps, ex->trace, (size_t)rows * 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < n; ++i) std::memcpy(items + 8 * i, &ex->last->items[i], sizeof(WorkItem));
    for (int32_t c = 0; c <= ex->last->stats.grid; ++c) cta_off[c] = ex->last->cta_off[c];
    return GMX_OK;
}

}  // extern "C"
