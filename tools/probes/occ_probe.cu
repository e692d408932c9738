// Probe: what limits two 192-thread CTAs per SM (smem granularity, registers, tcgen05 use).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(192, 2) k_plain(int* p) { extern __shared__ int s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); p[threadIdx.x] = s[191 - threadIdx.x]; }
__global__ void __maxnreg__(160) k_regs(float* p, int n) {
    float v[150];
#pragma unroll
    for (int i = 0; i < 150; ++i) v[i] = p[i * n + threadIdx.x];
    float acc = 0;
#pragma unroll
    for (int i = 0; i < 150; ++i) acc += v[i] * v[149 - i];
    p[threadIdx.x] = acc;
}
__global__ void __launch_bounds__(192, 2) k_tmem(uint32_t* p) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
    p[threadIdx.x] = slot;
}
template <typename F>
void probe(const char* name, F f, int b) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, 192, b);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, f);
    printf("%-8s dyn %d: %d/SM (regs %d static %zu) %s\n", name, b, n, fa.numRegs, fa.sharedSizeBytes, cudaGetErrorString(e));
}
int main() {
    for (int b : {100 * 1024, 112 * 1024, 114944, 115712}) {
        probe("plain", k_plain, b);
        probe("regs160", k_regs, b);
        probe("tmem", k_tmem, b);
    }
    return 0;
}
