/* Host cost of the native decision path for C2 rounds (16 tenants, ooo, b200 profile):
 * add_request x16 -> step (withhold) -> step at wakeup (dispatch) -> complete all. */
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include "../include/gmx_core.h"

static const int64_t SH[13][3] = {{64,3136,147},{64,3136,64},{64,3136,576},{256,3136,64},{128,784,256},
  {128,784,1152},{512,784,128},{256,196,512},{256,196,2304},{1024,196,256},{512,49,1024},{512,49,4608},{2048,49,512}};

static double now_us(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e6 + t.tv_nsec / 1e3; }

int main(int argc, char** argv) {
    int rounds = argc > 1 ? atoi(argv[1]) : 20000;
    int tenants = argc > 2 ? atoi(argv[2]) : 16;
    gmx_profile p = {148, 8, 1639.6e12, 74.4e12, 6543.1e9, 4000};
    gmx_policy_params pp = {0.25, 0.5, 2.0, 32, 8, 0.15, 10000, 0.0};
    gmx_sched* s;
    if (gmx_sched_create(&p, GMX_POLICY_OOO, &pp, NULL, 0.6, 0.4, 0, &s)) return 1;
    if (argc > 3) gmx_sched_set_retire(s, atoi(argv[3]));
    int32_t codes[1024];
    char name[32];
    for (int i = 0; i < tenants; ++i) { snprintf(name, sizeof name, "t%03d", i); gmx_sched_intern_stream(s, name, &codes[i]); }
    double t0 = 0; int64_t dispatched = 0; double ta = 0, ts = 0, tc = 0;
    for (int r = 0; r < rounds + 100; ++r) {
        if (r == 100) t0 = now_us();
        int64_t base = (int64_t)r * 1000000;
        double q0 = now_us();
        for (int i = 0; i < tenants; ++i) {
            gmx_kernel_desc k = {0};
            k.kernel_id = (int64_t)r * tenants + i; k.stream = codes[i]; k.op = GMX_OP_GEMM; k.dtype = GMX_DT_FP16;
            k.ndims = 3; k.dims[0] = SH[i % 13][0]; k.dims[1] = SH[i % 13][1]; k.dims[2] = SH[i % 13][2];
            k.arrival = base; k.deadline = base + 10000000;
            int32_t off[2] = {0, 0}; int64_t pred; int32_t acc;
            gmx_sched_add_request(s, k.kernel_id, codes[i], base, &k, 1, NULL, off, &pred, &acc);
        }
        double q1 = now_us();
        int64_t t = base; int left = tenants;
        /* lockstep virtual time: dispatches complete at their model end; SM-gated clusters
           dispatch after completions free SMs (engine.py:320-367 order) */
        int64_t pend_id[4096], pend_end[4096]; int npend = 0; int64_t wake = -1;
        while (left > 0) {
            gmx_step_view v;
            gmx_sched_step(s, t, &v);
            for (int d = 0; d < v.n_dispatches; ++d) {
                pend_id[npend] = v.dispatches[d].dispatch_id; pend_end[npend++] = v.dispatches[d].end;
                left -= v.dispatches[d].n_kernels; dispatched++;
            }
            wake = v.has_wakeup ? v.wakeup : -1;
            if (left <= 0) break;
            int64_t next = wake;
            for (int d = 0; d < npend; ++d) if (pend_id[d] >= 0 && (next < 0 || pend_end[d] < next)) next = pend_end[d];
            if (next < 0) next = t + 1;
            t = next;
            for (int d = 0; d < npend; ++d) if (pend_id[d] >= 0 && pend_end[d] <= t) {
                gmx_complete_view cv; gmx_sched_complete(s, pend_id[d], t, &cv); pend_id[d] = -1; }
        }
        double q2 = now_us();
        for (int d = 0; d < npend; ++d) if (pend_id[d] >= 0) { gmx_complete_view cv; gmx_sched_complete(s, pend_id[d], t + 100000, &cv); }
        double q3 = now_us();
        if (r >= 100) { ta += q1 - q0; ts += q2 - q1; tc += q3 - q2; }
    }
    double el = now_us() - t0;
    printf("%d tenants: %.2f us per round (%.2f dispatches/round) add %.2f step %.2f complete %.2f\n", tenants, el / rounds, (double)dispatched / (rounds + 100), ta / rounds, ts / rounds, tc / rounds);
    gmx_sched_destroy(s);
    return 0;
}
