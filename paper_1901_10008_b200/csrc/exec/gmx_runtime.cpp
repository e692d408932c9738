// gmx_runtime.cpp — native event loop driving the decision core and the executor.
//
// engine.py:320-367 restated: one scheduler step per distinct timestamp after draining every
// event at that time (COMPLETE < ARRIVAL < WAKEUP, ascending id); each step's dispatches become
// ONE coalesced launch. Storage is flat (pooled request records, kernel/dependency arenas,
// open-addressing id maps) so a steady-state round performs no heap allocation.

#include "../../../include/gmx_runtime.h"
#include "../core/flatmap.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <deque>
#include <queue>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}

enum : int32_t { kComplete = 0, kArrival = 1, kWakeup = 2 };
constexpr int32_t kHasDeps = 1 << 30;

struct Event {
    int64_t time;
    int32_t kind;
    int64_t id;
    bool operator>(const Event& o) const {
        if (time != o.time) return time > o.time;
        if (kind != o.kind) return kind > o.kind;
        return id > o.id;
    }
};

struct Pending {                 // one submitted request, pooled
    int64_t request_id;
    int32_t stream;
    int64_t arrival, deadline;
    int32_t k_off, n;            // kernels in the kernel arena
    int32_t d_off;               // dependency CSR: offsets in off_arena[d_off .. d_off + n]
    bool arrived;
};

}  // namespace

struct gmx_runtime {
    gmx_sched* sched;
    gmx_exec* ex;
    int32_t mode;
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> heap;
    // Arrivals submitted in (time, id) order — the common case, requests are queued ahead —
    // wait in a FIFO instead of the heap, which then only holds completions and wakeups; an
    // out-of-order arrival goes to the heap. The event order is unchanged (merge of the two).
    // FIFO as a vector + head (no chunk allocation per push/pop; reset whenever it drains)
    struct Fifo {
        std::vector<Event> v;
        size_t head = 0;
        bool empty() const { return head == v.size(); }
        const Event& front() const { return v[head]; }
        const Event& back() const { return v.back(); }
        void push_back(const Event& e) {
            if (empty()) { v.clear(); head = 0; }
            v.push_back(e);
        }
        void pop_front() {
            if (++head == v.size()) { v.clear(); head = 0; }
        }
    } arrivals;
    std::vector<Pending> pool;
    std::vector<int32_t> pool_free;
    gmx::IdMap req_index;                 // request id -> pool index (until the request finishes)
    gmx::IdMap slot_of;                   // kernel id -> executor slot (until dispatched)
    gmx::IdMap depslots_of;               // kernel id -> offset in depslot_arena (kernels with deps)
    std::vector<int32_t> depslot_arena;   // [count, producer slot...] per kernel with deps
    std::vector<int32_t> launch_deps;     // producer slots of one launch
    std::vector<gmx_kernel_desc> k_arena; // compacted when the pool drains
    std::vector<int64_t> dep_arena;
    std::vector<int32_t> off_arena;
    std::vector<int64_t> done_ids, done_times;
    std::vector<int64_t> pred;
    std::vector<int32_t> launch_slots;
    int64_t wake_seq = 0;
    int64_t live_requests = 0;
    gmx_runtime_stats st{};
    // realtime mode
    bool origin_set = false;
    int64_t origin_ns = 0;
    struct InFlight {
        cudaEvent_t ev;                  // launch per step: event after the launch
        std::vector<int64_t> dispatch_ids;
        int64_t seq;                     // resident executor: step queue position (ev unused)
        int64_t start;                   // runtime clock at launch (measured durations)
    };
    std::deque<InFlight> inflight;
    std::vector<cudaStream_t> streams;   // realtime: launches round-robin over these
    int64_t prof_ns[4] = {0, 0, 0, 0};   // host time in add_request / step / complete / launch
    bool prof_on = false;                // gmx_runtime_set_profiling (clock reads cost ~1 us/round)
    bool measured_ratios = false;        // realtime: straggler windows get observed durations
    int64_t last_seq = -1;               // resident executor: queue position of the last step
    gmx::IdMap cancelled;                // dispatch ids cancelled by straggler eviction
    std::vector<int32_t> straggler_buf;
    size_t next_stream = 0;
    std::vector<cudaEvent_t> event_pool;
    std::vector<gmx_replay_rec> log;
    std::vector<int64_t> log_kids;
};

static int64_t steady_ns() {
    return (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

static void log_rec(gmx_runtime* rt, int32_t kind, int64_t t, int64_t a, int32_t n = 0, int64_t off = 0) {
    rt->log.push_back(gmx_replay_rec{kind, n, t, a, off});
}

// purge: an evicted request's undispatched kernels never reach a launch, so their slot and
// producer-slot entries are dropped here (a finished request's were consumed at dispatch)
static void release_request(gmx_runtime* rt, int64_t rid, bool purge = false, int32_t known_pi = -1) {
    const int32_t pi = known_pi >= 0 ? known_pi : rt->req_index.find(rid);
    if (pi < 0) return;
    if (purge) {
        const Pending& p = rt->pool[pi];
        for (int32_t i = 0; i < p.n; ++i) {
            const int64_t kid = rt->k_arena[p.k_off + i].kernel_id;
            rt->slot_of.erase(kid);
            rt->depslots_of.erase(kid);
        }
    }
    rt->req_index.erase(rid);
    rt->pool_free.push_back(pi);
    if (--rt->live_requests == 0) {   // nothing outstanding: recycle the arenas
        rt->k_arena.clear();
        rt->dep_arena.clear();
        rt->off_arena.clear();
        rt->depslot_arena.clear();
        rt->depslots_of.clear();
    }
}

extern "C" {

const char* gmx_runtime_last_error(void) { return g_err.c_str(); }

int gmx_runtime_create(gmx_sched* sched, gmx_exec* ex, int32_t mode, gmx_runtime** out) {
    if (!sched || !out) return fail(GMX_EINVAL, "null argument");
    if (mode != GMX_RT_LOCKSTEP && mode != GMX_RT_REALTIME) return fail(GMX_EINVAL, "unsupported runtime mode");
    if (!ex && mode == GMX_RT_REALTIME) return fail(GMX_EINVAL, "wall-clock mode needs an executor");
    // wall-clock serving: most step compositions are one-offs, so first sightings run as inline
    // steps (device-enumerated work items) instead of paying a host plan build + upload
    if (ex && mode == GMX_RT_REALTIME) {
        gmx_exec_set_option(ex, "inline_plans", 1);
        gmx_exec_set_option(ex, "inline_promote", 1 << 20);   // plans only for steps too big to inline
    }
    auto* rt = new gmx_runtime();
    rt->sched = sched;
    rt->ex = ex;
    rt->mode = mode;
    *out = rt;
    return GMX_OK;
}

void gmx_runtime_destroy(gmx_runtime* rt) {
    if (!rt) return;
    for (cudaStream_t st : rt->streams) {
        gmx_exec_stream_retired(rt->ex, st);
        cudaStreamDestroy(st);
    }
    for (auto& f : rt->inflight) cudaEventDestroy(f.ev);
    for (cudaEvent_t e : rt->event_pool) cudaEventDestroy(e);
    delete rt;
}

int gmx_runtime_set_streams(gmx_runtime* rt, int32_t n) {
    if (!rt || n < 1 || n > 64) return fail(GMX_EINVAL, "stream count must be in [1, 64]");
    for (cudaStream_t st : rt->streams) {
        gmx_exec_stream_retired(rt->ex, st);
        cudaStreamDestroy(st);
    }
    rt->streams.clear();
    for (int32_t i = 0; i < n; ++i) {
        cudaStream_t st;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            return fail(GMX_ECUDA, "cudaStreamCreate failed");
        rt->streams.push_back(st);
    }
    return gmx_exec_set_option(rt->ex, "multi_stream", n > 1 ? 1 : 0);
}

int gmx_runtime_set_origin(gmx_runtime* rt, int64_t ns) {
    if (!rt) return fail(GMX_EINVAL, "null argument");
    rt->origin_ns = ns;
    rt->origin_set = true;
    return GMX_OK;
}

int gmx_runtime_set_measured_stragglers(gmx_runtime* rt, int32_t on) {
    if (!rt) return fail(GMX_EINVAL, "null argument");
    rt->measured_ratios = on != 0;
    return GMX_OK;
}

int gmx_runtime_set_profiling(gmx_runtime* rt, int32_t on) {
    if (!rt) return fail(GMX_EINVAL, "null argument");
    rt->prof_on = on != 0;
    return GMX_OK;
}

int gmx_runtime_host_profile(const gmx_runtime* rt, int64_t* out4) {
    if (!rt || !out4) return fail(GMX_EINVAL, "null argument");
    for (int i = 0; i < 4; ++i) out4[i] = rt->prof_ns[i];
    return GMX_OK;
}

int64_t gmx_runtime_clock_ns(const gmx_runtime* rt) {
    if (!rt || !rt->origin_set) return 0;
    return steady_ns() - rt->origin_ns;
}

int gmx_runtime_submit(gmx_runtime* rt, int64_t rid, int32_t stream, int64_t arrival, int64_t deadline,
                       const gmx_kernel_desc* ks, int32_t n, const int64_t* dep_ids, const int32_t* dep_off,
                       const int32_t* slots) {
    if (!rt || (n > 0 && (!ks || !dep_off || !slots))) return fail(GMX_EINVAL, "null argument");
    if (rt->req_index.find(rid) >= 0) return fail(GMX_EINVAL, "request id already pending");
    int32_t pi;
    if (!rt->pool_free.empty()) {
        pi = rt->pool_free.back();
        rt->pool_free.pop_back();
    } else {
        pi = (int32_t)rt->pool.size();
        rt->pool.emplace_back();
    }
    Pending& p = rt->pool[pi];
    p.request_id = rid;
    p.stream = stream;
    p.arrival = arrival;
    p.deadline = deadline;
    p.k_off = (int32_t)rt->k_arena.size();
    p.n = n;
    p.d_off = (int32_t)rt->off_arena.size();
    p.arrived = false;
    rt->k_arena.insert(rt->k_arena.end(), ks, ks + n);
    const int32_t dep_base = (int32_t)rt->dep_arena.size();
    for (int32_t i = 0; i <= n; ++i) rt->off_arena.push_back(n > 0 ? dep_off[i] : 0);
    if (n > 0 && dep_off[n] > 0) rt->dep_arena.insert(rt->dep_arena.end(), dep_ids, dep_ids + dep_off[n]);
    // the n+1 CSR offsets are relative to this request's first dependency; a trailing
    // sentinel records where those dependencies start in dep_arena
    rt->off_arena.push_back(dep_base);
    // executor slot per kernel; bit 30 marks kernels with dependencies (they may read what an
    // earlier launch wrote, so their launch must not overlap it)
    for (int32_t i = 0; i < n; ++i)
        rt->slot_of.put(ks[i].kernel_id, slots[i] | ((n > 0 && dep_off[i + 1] > dep_off[i]) ? kHasDeps : 0));
    // producers' executor slots per dependent kernel (deps name kernels of the same request,
    // kernels.py:95-124), so a launch can tell the executor exactly which outputs it reads
    for (int32_t i = 0; i < n; ++i) {
        if (dep_off[i + 1] <= dep_off[i]) continue;
        const int32_t off = (int32_t)rt->depslot_arena.size();
        rt->depslot_arena.push_back(0);
        for (int32_t j = dep_off[i]; j < dep_off[i + 1]; ++j)
            for (int32_t q = 0; q < n; ++q)
                if (ks[q].kernel_id == dep_ids[j]) {
                    rt->depslot_arena.push_back(slots[q]);
                    ++rt->depslot_arena[off];
                    break;
                }
        rt->depslots_of.put(ks[i].kernel_id, off);
    }
    rt->req_index.put(rid, pi);
    ++rt->live_requests;
    const Event ev{arrival, kArrival, rid};
    if (rt->arrivals.empty() || !(rt->arrivals.back() > ev))
        rt->arrivals.push_back(ev);
    else
        rt->heap.push(ev);
    return GMX_OK;
}

// engine.py:345-351: after the events at `now` are drained and before the step, every stream
// whose straggler ratio exceeds the threshold is evicted; its cancelled dispatches' completion
// events are ignored and its requests leave (evicted, not completed).
static int evict_stragglers(gmx_runtime* rt, int64_t now) {
    int32_t n = 0;
    int rc = gmx_sched_find_stragglers(rt->sched, nullptr, 0, &n);
    if (rc || n == 0) return rc ? fail(rc, std::string("stragglers: ") + gmx_last_error()) : GMX_OK;
    rt->straggler_buf.resize((size_t)n);
    if ((rc = gmx_sched_find_stragglers(rt->sched, rt->straggler_buf.data(), n, &n)))
        return fail(rc, std::string("stragglers: ") + gmx_last_error());
    for (int32_t st : rt->straggler_buf) {
        gmx_evict_view ev;
        if ((rc = gmx_sched_evict_stream(rt->sched, st, now, &ev))) return fail(rc, std::string("evict: ") + gmx_last_error());
        for (int32_t i = 0; i < ev.n_cancelled; ++i) {
            rt->cancelled.put(ev.cancelled_dispatch_ids[i], 1);
            ++rt->st.cancelled_dispatches;
        }
        for (int32_t i = 0; i < ev.n_evicted; ++i) {
            ++rt->st.evicted_requests;
            release_request(rt, ev.evicted_request_ids[i], true);
        }
        log_rec(rt, 6, now, st);
    }
    return GMX_OK;
}

static int on_finished(gmx_runtime* rt, const gmx_complete_view& cv, int64_t now) {
    for (int32_t i = 0; i < cv.n_finished; ++i) {
        const int64_t r = cv.finished_request_ids[i];
        rt->done_ids.push_back(r);
        rt->done_times.push_back(now);
        ++rt->st.completed_requests;
        const int32_t pi = rt->req_index.find(r);
        if (pi >= 0) {
            if (now > rt->pool[pi].deadline) ++rt->st.slo_misses;
            release_request(rt, r, false, pi);
        }
    }
    return GMX_OK;
}

static int on_arrival(gmx_runtime* rt, int64_t rid) {
    const int32_t pi = rt->req_index.find(rid);
    if (pi < 0 || rt->pool[pi].arrived) return GMX_OK;
    Pending& p = rt->pool[pi];
    p.arrived = true;
    rt->pred.resize((size_t)std::max(1, p.n));
    const int32_t dep_base = rt->off_arena[p.d_off + p.n + 1];
    int32_t accepted = 0;
    const int64_t t_add = rt->prof_on ? steady_ns() : 0;
    int rc = gmx_sched_add_request(rt->sched, rid, p.stream, p.arrival, rt->k_arena.data() + p.k_off, p.n,
                                   rt->dep_arena.data() + dep_base, rt->off_arena.data() + p.d_off,
                                   rt->pred.data(), &accepted);
    if (rt->prof_on) rt->prof_ns[0] += steady_ns() - t_add;
    if (rc) return fail(rc, std::string("add_request: ") + gmx_last_error());
    if (!accepted) {   // stream already evicted (engine.py:338-342, "stream-evicted")
        ++rt->st.evicted_requests;
        release_request(rt, rid, true);
    }
    return GMX_OK;
}

// One scheduler step at `now` and ONE launch for all of its dispatches. In realtime mode the
// dispatch ids of the launch are returned in `ids` (completion is observed, not scheduled).
static int step_and_launch(gmx_runtime* rt, int64_t now, void* stream, bool realtime, std::vector<int64_t>* ids) {
    gmx_step_view v;
    const int64_t t_step = rt->prof_on ? steady_ns() : 0;
    int rc = gmx_sched_step(rt->sched, now, &v);
    if (rt->prof_on) rt->prof_ns[1] += steady_ns() - t_step;
    if (rc) return fail(rc, std::string("step: ") + gmx_last_error());
    ++rt->st.steps;
    rt->st.withheld += v.n_withheld;
    if (realtime) {
        log_rec(rt, 5, now, 0);
        for (int32_t d = 0; d < v.n_dispatches; ++d) {
            const gmx_dispatch_rec& r = v.dispatches[d];
            log_rec(rt, 2, now, r.dispatch_id, r.n_kernels, (int64_t)rt->log_kids.size());
            rt->log_kids.insert(rt->log_kids.end(), v.dispatch_kernel_ids + r.kernel_offset,
                                v.dispatch_kernel_ids + r.kernel_offset + r.n_kernels);
        }
        for (int32_t w = 0; w < v.n_withheld; ++w) {
            const int32_t a = v.withheld_offsets[w], b = v.withheld_offsets[w + 1];
            log_rec(rt, 3, now, 0, b - a, (int64_t)rt->log_kids.size());
            rt->log_kids.insert(rt->log_kids.end(), v.withheld_kernel_ids + a, v.withheld_kernel_ids + b);
        }
        log_rec(rt, 4, now, v.has_wakeup ? v.wakeup : -1);
    }
    if (v.n_dispatches > 0) {
        rt->launch_slots.clear();
        rt->launch_deps.clear();
        bool independent = true;
        for (int32_t d = 0; d < v.n_dispatches; ++d) {
            const gmx_dispatch_rec& r = v.dispatches[d];
            for (int32_t j = 0; j < r.n_kernels; ++j) {
                const int64_t kid = v.dispatch_kernel_ids[r.kernel_offset + j];
                const int64_t taken = rt->slot_of.take(kid);
                const int32_t slot = taken == gmx::IdMap::kAbsent ? -1 : (int32_t)taken;
                if (slot < 0 && rt->ex) return fail(GMX_ESTATE, "dispatched kernel has no operands bound");
                independent &= (slot & kHasDeps) == 0;
                rt->launch_slots.push_back(slot & ~kHasDeps);
                if (slot & kHasDeps) {
                    const int64_t off = rt->depslots_of.take(kid);
                    if (off != gmx::IdMap::kAbsent) {
                        const int32_t cnt = rt->depslot_arena[off];
                        rt->launch_deps.insert(rt->launch_deps.end(), rt->depslot_arena.begin() + off + 1,
                                               rt->depslot_arena.begin() + off + 1 + cnt);
                    }
                }
            }
            if (realtime)
                ids->push_back(r.dispatch_id);
            else
                rt->heap.push({r.end, kComplete, r.dispatch_id});
            rt->st.useful_flops += r.useful_flops;
            rt->st.kernels += r.n_kernels;
        }
        const int64_t t_l = rt->prof_on ? steady_ns() : 0;
        // dependencies go to the executor as the producers' slots: a per-step launch becomes
        // dependent, a resident step waits only for the steps that wrote those slots
        int64_t seq = -1;
        // wall clock: a member became ready only after its producers' completion was OBSERVED, so
        // the launch carries no ordering against earlier steps (it must not wait for unrelated
        // work queued before it)
        int32_t lflags = 0;
        if (realtime) {   // ... but its TMA loads still need the proxy fence (resident mode)
            if (!independent) lflags |= GMX_LAUNCH_FENCE;
            rt->launch_deps.clear();
            independent = true;
        }
        if (independent) lflags |= GMX_LAUNCH_INDEPENDENT;
        rc = rt->ex ? gmx_exec_launch_deps(rt->ex, rt->launch_slots.data(), (int32_t)rt->launch_slots.size(),
                                           rt->launch_deps.data(), (int32_t)rt->launch_deps.size(), stream,
                                           lflags, &seq)
                    : GMX_OK;   // decisions-only runtime (no executor): nothing to launch
        rt->last_seq = seq;
        if (rt->prof_on) rt->prof_ns[3] += steady_ns() - t_l;
        if (rc) return fail(rc, std::string("launch: ") + gmx_exec_last_error());
        ++rt->st.launches;
        rt->st.dispatches += v.n_dispatches;
    }
    if (v.has_wakeup) rt->heap.push({v.wakeup, kWakeup, ++rt->wake_seq});
    rt->st.now = now;
    return GMX_OK;
}

// Earliest pending event (heap and arrival FIFO merged); nullptr when none.
static const Event* peek_event(const gmx_runtime* rt) {
    const Event* h = rt->heap.empty() ? nullptr : &rt->heap.top();
    const Event* a = rt->arrivals.empty() ? nullptr : &rt->arrivals.front();
    if (!h) return a;
    if (!a) return h;
    return (*h > *a) ? a : h;
}
static Event pop_event(gmx_runtime* rt) {
    const Event* e = peek_event(rt);
    const Event out = *e;
    if (!rt->arrivals.empty() && e == &rt->arrivals.front())
        rt->arrivals.pop_front();
    else
        rt->heap.pop();
    return out;
}

// Wall-clock loop: returns when every submitted request has finished and nothing is in flight,
// or when the clock passes `until`.
static int run_realtime(gmx_runtime* rt, int64_t until, void* stream, gmx_runtime_stats* out) {
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (!rt->origin_set) {
        rt->origin_ns = steady_ns();
        rt->origin_set = true;
    }
    std::vector<int64_t> ids;
    for (;;) {
        const int64_t now = steady_ns() - rt->origin_ns;
        bool any = false;
        // COMPLETE: any launch whose event has completed (launches on several streams may
        // retire out of order; each launch's dispatches complete in dispatch-id order)
        for (size_t i = 0; i < rt->inflight.size();) {
            if (rt->inflight[i].seq >= 0) {   // resident: the executor's host-mapped completion flags
                if (!gmx_exec_resident_step_done(rt->ex, rt->inflight[i].seq)) {
                    ++i;
                    continue;
                }
            } else {
                const cudaError_t q = cudaEventQuery(rt->inflight[i].ev);
                if (q == cudaErrorNotReady) {
                    ++i;
                    continue;
                }
                if (q != cudaSuccess) return fail(GMX_ECUDA, std::string("launch failed: ") + cudaGetErrorString(q));
            }
            for (int64_t did : rt->inflight[i].dispatch_ids) {
                if (rt->cancelled.find(did) >= 0) {
                    rt->cancelled.erase(did);
                    continue;
                }
                gmx_complete_view cv;
                const int64_t measured = rt->measured_ratios ? now - rt->inflight[i].start : -1;
                int rc = gmx_sched_complete_measured(rt->sched, did, now, measured, &cv);
                if (rc) return fail(rc, std::string("complete: ") + gmx_last_error());
                log_rec(rt, 0, now, did, 0, measured);
                on_finished(rt, cv, now);
            }
            if (rt->inflight[i].seq < 0) rt->event_pool.push_back(rt->inflight[i].ev);
            rt->inflight.erase(rt->inflight.begin() + (long)i);
            any = true;
        }
        // ARRIVAL then WAKEUP events that are due (heap order: time, kind, id)
        while (peek_event(rt) && peek_event(rt)->time <= now) {
            const Event e = pop_event(rt);
            if (e.kind == kArrival) {
                log_rec(rt, 1, now, e.id);
                int rc = on_arrival(rt, e.id);
                if (rc) return rc;
            }
            any = true;
        }
        if (any) {
            int rc0 = evict_stragglers(rt, now);
            if (rc0) return rc0;
            ids.clear();
            void* launch_stream = stream;
            if (!rt->streams.empty()) {
                cs = rt->streams[rt->next_stream];
                launch_stream = cs;
            }
            int rc = step_and_launch(rt, now, launch_stream, true, &ids);
            if (rc) return rc;
            if (!ids.empty() && rt->last_seq >= 0) {   // resident executor: no events needed
                rt->inflight.push_back({nullptr, ids, rt->last_seq, now});
            } else if (!ids.empty()) {
                cudaEvent_t ev;
                if (!rt->event_pool.empty()) {
                    ev = rt->event_pool.back();
                    rt->event_pool.pop_back();
                } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
                    return fail(GMX_ECUDA, "cudaEventCreate failed");
                }
                if (cudaEventRecord(ev, cs) != cudaSuccess) return fail(GMX_ECUDA, "cudaEventRecord failed");
                rt->inflight.push_back({ev, ids, -1, now});
                if (!rt->streams.empty()) rt->next_stream = (rt->next_stream + 1) % rt->streams.size();
            }
            continue;
        }
        if (!peek_event(rt) && rt->inflight.empty()) break;   // drained
        if (now > until) break;
    }
    rt->st.now = steady_ns() - rt->origin_ns;
    if (out) *out = rt->st;
    return GMX_OK;
}

int gmx_runtime_run(gmx_runtime* rt, int64_t until, void* stream, gmx_runtime_stats* out) {
    if (!rt) return fail(GMX_EINVAL, "null argument");
    if (rt->mode == GMX_RT_REALTIME) return run_realtime(rt, until, stream, out);
    while (peek_event(rt) && peek_event(rt)->time <= until) {
        const int64_t now = peek_event(rt)->time;
        while (peek_event(rt) && peek_event(rt)->time == now) {
            const Event e = pop_event(rt);
            if (e.kind == kComplete) {
                if (rt->cancelled.find(e.id) >= 0) {   // engine.py:326-327
                    rt->cancelled.erase(e.id);
                    continue;
                }
                gmx_complete_view cv;
                const int64_t t_c = rt->prof_on ? steady_ns() : 0;
                int rc = gmx_sched_complete(rt->sched, e.id, now, &cv);
                if (rt->prof_on) rt->prof_ns[2] += steady_ns() - t_c;
                if (rc) return fail(rc, std::string("complete: ") + gmx_last_error());
                on_finished(rt, cv, now);
            } else if (e.kind == kArrival) {
                int rc = on_arrival(rt, e.id);
                if (rc) return rc;
            }
        }
        int rc = evict_stragglers(rt, now);
        if (rc) return rc;
        // a step with no ready kernel decides nothing (every policy): skip it (most of a C2
        // round's completion events leave the ready set empty)
        if (gmx_sched_ready_count(rt->sched) == 0) {
            rt->st.now = now;
            continue;
        }
        rc = step_and_launch(rt, now, stream, false, nullptr);
        if (rc) return rc;
    }
    if (out) *out = rt->st;
    return GMX_OK;
}

int gmx_runtime_replay_log(const gmx_runtime* rt, gmx_replay_rec* recs, int64_t cap, int64_t* n_out,
                           int64_t* kids, int64_t kid_cap, int64_t* n_kids) {
    if (!rt || !n_out || !n_kids) return fail(GMX_EINVAL, "null argument");
    *n_out = (int64_t)rt->log.size();
    *n_kids = (int64_t)rt->log_kids.size();
    if (recs) std::copy(rt->log.begin(), rt->log.begin() + std::min<int64_t>(cap, *n_out), recs);
    if (kids) std::copy(rt->log_kids.begin(), rt->log_kids.begin() + std::min<int64_t>(kid_cap, *n_kids), kids);
    return GMX_OK;
}

int gmx_runtime_drain_completions(gmx_runtime* rt, int64_t* ids, int64_t* times, int32_t cap, int32_t* n_out) {
    if (!rt || !n_out) return fail(GMX_EINVAL, "null argument");
    const int32_t n = (int32_t)std::min<size_t>((size_t)cap, rt->done_ids.size());
    for (int32_t i = 0; i < n; ++i) {
        ids[i] = rt->done_ids[i];
        times[i] = rt->done_times[i];
    }
    rt->done_ids.erase(rt->done_ids.begin(), rt->done_ids.begin() + n);
    rt->done_times.erase(rt->done_times.begin(), rt->done_times.begin() + n);
    *n_out = n;
    return GMX_OK;
}

}  // extern "C"
