// gmx_runtime.cpp — native event loop driving the decision core and the executor.
//
// engine.py:320-367 restated: one scheduler step per distinct timestamp after draining every
// event at that time; each step's dispatches become ONE coalesced launch.

#include "../../../include/gmx_runtime.h"

#include <algorithm>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}

enum : int32_t { kComplete = 0, kArrival = 1, kWakeup = 2 };

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

struct PendingRequest {
    int32_t stream;
    int64_t arrival, deadline;
    std::vector<gmx_kernel_desc> kernels;
    std::vector<int64_t> dep_ids;
    std::vector<int32_t> dep_off;
};

}  // namespace

struct gmx_runtime {
    gmx_sched* sched;
    gmx_exec* ex;
    int32_t mode;
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> heap;
    std::unordered_map<int64_t, PendingRequest> pending;     // request id -> not yet arrived
    std::unordered_map<int64_t, int32_t> slot_of;            // kernel id -> executor slot
    std::unordered_map<int64_t, int64_t> deadline_of;        // request id -> absolute deadline
    std::unordered_map<int64_t, int64_t> flops_of;           // dispatch id -> useful flops
    std::vector<int64_t> done_ids, done_times;
    int64_t wake_seq = 0;
    gmx_runtime_stats st{};
    std::vector<int32_t> launch_slots;
};

extern "C" {

const char* gmx_runtime_last_error(void) { return g_err.c_str(); }

int gmx_runtime_create(gmx_sched* sched, gmx_exec* ex, int32_t mode, gmx_runtime** out) {
    if (!sched || !ex || !out) return fail(GMX_EINVAL, "null argument");
    if (mode != GMX_RT_LOCKSTEP) return fail(GMX_EINVAL, "unsupported runtime mode");
    auto* rt = new gmx_runtime();
    rt->sched = sched;
    rt->ex = ex;
    rt->mode = mode;
    *out = rt;
    return GMX_OK;
}

void gmx_runtime_destroy(gmx_runtime* rt) { delete rt; }

int gmx_runtime_submit(gmx_runtime* rt, int64_t rid, int32_t stream, int64_t arrival, int64_t deadline,
                       const gmx_kernel_desc* ks, int32_t n, const int64_t* dep_ids, const int32_t* dep_off,
                       const int32_t* slots) {
    if (!rt || (n > 0 && (!ks || !dep_off || !slots))) return fail(GMX_EINVAL, "null argument");
    PendingRequest p;
    p.stream = stream;
    p.arrival = arrival;
    p.deadline = deadline;
    p.kernels.assign(ks, ks + n);
    p.dep_off.assign(dep_off, dep_off + n + 1);
    if (n > 0 && dep_off[n] > 0) p.dep_ids.assign(dep_ids, dep_ids + dep_off[n]);
    for (int32_t i = 0; i < n; ++i) rt->slot_of[ks[i].kernel_id] = slots[i];
    rt->pending[rid] = std::move(p);
    rt->deadline_of[rid] = deadline;
    rt->heap.push({arrival, kArrival, rid});
    return GMX_OK;
}

int gmx_runtime_run(gmx_runtime* rt, int64_t until, void* stream, gmx_runtime_stats* out) {
    if (!rt) return fail(GMX_EINVAL, "null argument");
    std::vector<int64_t> pred;
    while (!rt->heap.empty() && rt->heap.top().time <= until) {
        const int64_t now = rt->heap.top().time;
        while (!rt->heap.empty() && rt->heap.top().time == now) {
            const Event e = rt->heap.top();
            rt->heap.pop();
            if (e.kind == kComplete) {
                gmx_complete_view cv;
                int rc = gmx_sched_complete(rt->sched, e.id, now, &cv);
                if (rc) return fail(rc, std::string("complete: ") + gmx_last_error());
                for (int32_t i = 0; i < cv.n_finished; ++i) {
                    const int64_t r = cv.finished_request_ids[i];
                    rt->done_ids.push_back(r);
                    rt->done_times.push_back(now);
                    ++rt->st.completed_requests;
                    auto it = rt->deadline_of.find(r);
                    if (it != rt->deadline_of.end()) {
                        if (now > it->second) ++rt->st.slo_misses;
                        rt->deadline_of.erase(it);
                    }
                }
            } else if (e.kind == kArrival) {
                auto it = rt->pending.find(e.id);
                if (it == rt->pending.end()) continue;
                PendingRequest& p = it->second;
                const int32_t n = (int32_t)p.kernels.size();
                pred.resize(std::max(1, n));
                int32_t accepted = 0;
                int rc = gmx_sched_add_request(rt->sched, e.id, p.stream, p.arrival, p.kernels.data(), n,
                                               p.dep_ids.empty() ? nullptr : p.dep_ids.data(), p.dep_off.data(),
                                               pred.data(), &accepted);
                if (rc) return fail(rc, std::string("add_request: ") + gmx_last_error());
                rt->pending.erase(it);
            }
        }
        gmx_step_view v;
        int rc = gmx_sched_step(rt->sched, now, &v);
        if (rc) return fail(rc, std::string("step: ") + gmx_last_error());
        ++rt->st.steps;
        rt->st.withheld += v.n_withheld;
        if (v.n_dispatches > 0) {
            rt->launch_slots.clear();
            for (int32_t d = 0; d < v.n_dispatches; ++d) {
                const gmx_dispatch_rec& r = v.dispatches[d];
                for (int32_t j = 0; j < r.n_kernels; ++j) {
                    auto it = rt->slot_of.find(v.dispatch_kernel_ids[r.kernel_offset + j]);
                    if (it == rt->slot_of.end()) return fail(GMX_ESTATE, "dispatched kernel has no operands bound");
                    rt->launch_slots.push_back(it->second);
                    rt->slot_of.erase(it);
                }
                rt->heap.push({r.end, kComplete, r.dispatch_id});
                rt->st.useful_flops += r.useful_flops;
                rt->st.kernels += r.n_kernels;
            }
            rc = gmx_exec_launch(rt->ex, rt->launch_slots.data(), (int32_t)rt->launch_slots.size(), stream);
            if (rc) return fail(rc, std::string("launch: ") + gmx_exec_last_error());
            ++rt->st.launches;
            rt->st.dispatches += v.n_dispatches;
        }
        if (v.has_wakeup) rt->heap.push({v.wakeup, kWakeup, ++rt->wake_seq});
        rt->st.now = now;
    }
    if (out) *out = rt->st;
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
