// Host-side cost of touching cudaHostAlloc'd (pinned, device-mapped) memory vs malloc'd memory:
// 256-byte memcpy (a resident step descriptor) and 8-byte reads (completion flags).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void run(const char* name, char* buf) {
    char src[256];
    memset(src, 1, sizeof src);
    const int N = 100000;
    double t0 = now();
    for (int i = 0; i < N; ++i) { src[0] = (char)i; memcpy(buf + (i % 1024) * 256, src, 256); }
    double t1 = now();
    volatile long long* f = (volatile long long*)buf;
    long long acc = 0;
    for (int i = 0; i < N; ++i) acc += f[(i * 32) % (1024 * 32)];
    double t2 = now();
    printf("%-28s memcpy 256 B: %.3f us   read 8 B: %.3f us   (%lld)\n", name, (t1 - t0) / N, (t2 - t1) / N, acc & 1);
}
int main() {
    char* h;
    cudaHostAlloc(&h, 1024 * 256, cudaHostAllocMapped); run("cudaHostAlloc(Mapped)", h);
    char* h2; cudaHostAlloc(&h2, 1024 * 256, cudaHostAllocDefault); run("cudaHostAlloc(Default)", h2);
    char* h3; cudaHostAlloc(&h3, 1024 * 256, cudaHostAllocMapped | cudaHostAllocWriteCombined); run("cudaHostAlloc(Mapped|WC)", h3);
    char* m = (char*)malloc(1024 * 256); run("malloc", m);
    char* r = (char*)aligned_alloc(4096, 1024 * 256); cudaHostRegister(r, 1024 * 256, cudaHostRegisterMapped); run("malloc+cudaHostRegister", r);
    return 0;
}
