/* Host cost of the native serving loop (decisions only: no executor) for C2 rounds, the
 * bench.py timed region without the GPU: 16 tenants x 1 request per round, then
 * gmx_runtime_run over the rounds (arrivals -> add_request -> step -> complete ...).
 *
 *   bench_runtime [rounds=700] [reps=1] [window=0] [tenants=16]
 *
 * window 0: every round submitted up front, one run over all of them (large id tables);
 * window W: like bench.py's serving loop, W rounds are submitted, then run, and so on (only the
 * runs are timed; the tables stay small).
 * build: gcc -O2 -I include tools/bench_runtime.c -L paper_1901_10008_b200/lib -lgmx_exec -lgmx_core */
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
#include "../include/gmx_runtime.h"

static const int64_t SH[13][3] = {{64,3136,147},{64,3136,64},{64,3136,576},{256,3136,64},{128,784,256},
  {128,784,1152},{512,784,128},{256,196,512},{256,196,2304},{1024,196,256},{512,49,1024},{512,49,4608},{2048,49,512}};
static double now_us(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e6 + t.tv_nsec / 1e3; }

static int tenants = 16;   /* C2; 512 = C5 */
static const int64_t RNS = 1000000, SLO = 10000000;

static int submit_rounds(gmx_runtime* rt, const int32_t* codes, int r0, int r1) {
    for (int r = r0; r < r1; ++r)
        for (int i = 0; i < tenants; ++i) {
            gmx_kernel_desc k = {0};
            k.kernel_id = (int64_t)r * tenants + i; k.stream = codes[i]; k.op = GMX_OP_GEMM; k.dtype = GMX_DT_FP16;
            k.ndims = 3; k.dims[0] = SH[i % 13][0]; k.dims[1] = SH[i % 13][1]; k.dims[2] = SH[i % 13][2];
            k.arrival = (int64_t)r * RNS; k.deadline = k.arrival + SLO;
            int32_t off[2] = {0, 0}, slot = 0;
            if (gmx_runtime_submit(rt, k.kernel_id, codes[i], k.arrival, k.deadline, &k, 1, NULL, off, &slot)) {
                printf("submit: %s\n", gmx_last_error()); return 1; }
        }
    return 0;
}

int main(int argc, char** argv) {
    const int rounds = argc > 1 ? atoi(argv[1]) : 700;
    const int reps = argc > 2 ? atoi(argv[2]) : 1;   /* fresh runtime per repetition (profiling) */
    const int window = argc > 3 ? atoi(argv[3]) : 0;
    if (argc > 4) tenants = atoi(argv[4]);
    if (tenants < 1 || tenants > 4096) return 1;
    const int warm = 200;
    double best = 1e30;
    for (int rep = 0; rep < reps; ++rep) {
    gmx_profile p = {148, 8, 1639.6e12, 74.4e12, 6543.1e9, 4000};
    gmx_policy_params pp = {0.25, 0.5, 2.0, 32, 8, 0.15, 10000, 0.0};
    gmx_sched* s;
    if (gmx_sched_create(&p, GMX_POLICY_OOO, &pp, NULL, 0.6, 0.4, 0, &s)) return 1;
    gmx_sched_set_retire(s, 1);
    static int32_t codes[4096];
    char name[32];
    for (int i = 0; i < tenants; ++i) { snprintf(name, sizeof name, "t%03d", i); gmx_sched_intern_stream(s, name, &codes[i]); }
    gmx_runtime* rt;
    if (gmx_runtime_create(s, NULL, GMX_RT_LOCKSTEP, &rt)) { printf("create: %s\n", gmx_last_error()); return 1; }
    gmx_runtime_stats st;
    double el = 0;
    if (window <= 0) {
        if (submit_rounds(rt, codes, 0, rounds)) return 1;
        gmx_runtime_run(rt, (int64_t)warm * RNS - 1, NULL, &st);
        if (getenv("GMX_PROF")) gmx_runtime_set_profiling(rt, 1);
        double t0 = now_us();
        gmx_runtime_run(rt, (int64_t)rounds * RNS - 1, NULL, &st);
        el = now_us() - t0;
    } else {
        for (int r = 0; r < rounds; r += window) {
            const int r1 = r + window < rounds ? r + window : rounds;
            if (submit_rounds(rt, codes, r, r1)) return 1;
            if (r == warm && getenv("GMX_PROF")) gmx_runtime_set_profiling(rt, 1);
            double t0 = now_us();
            gmx_runtime_run(rt, (int64_t)r1 * RNS - 1, NULL, &st);
            if (r >= warm) el += now_us() - t0;
        }
    }
    if (el / (rounds - warm) < best) best = el / (rounds - warm);
    if (rep == reps - 1 && getenv("GMX_PROF")) {
        int64_t p[4];
        gmx_runtime_host_profile(rt, p);
        printf("per round (us): add_request %.3f step %.3f complete %.3f launch %.3f\n", p[0] / 1e3 / (rounds - warm),
               p[1] / 1e3 / (rounds - warm), p[2] / 1e3 / (rounds - warm), p[3] / 1e3 / (rounds - warm));
    }
    if (rep == reps - 1)
        printf("%.3f us per round, best of %d (%lld steps, %lld dispatches over %d rounds, window %d)\n", best, reps,
               (long long)st.steps, (long long)st.dispatches, rounds, window);
    gmx_runtime_destroy(rt);
    gmx_sched_destroy(s);
    }
    return 0;
}
