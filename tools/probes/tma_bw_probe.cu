// Probe: aggregate TMA (cp.async.bulk global->shared) throughput on B200, to tell whether the
// coalesced step is bound by L2->SM delivery (L2-resident re-reads) or by DRAM.
//   mode 0: every CTA streams a distinct slice of a buffer larger than L2 (DRAM-bound)
//   mode 1: every CTA streams a slice of an L2-resident buffer (L2 hit path)
//   mode 2: half the chunks DRAM-streamed, half L2 hits (the coalesced step's mix)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw_probe tma_bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(b)),
        "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b))
                 : "memory");
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) probe(const char* big, size_t big_bytes, const char* small, size_t small_bytes,
                                            int mode, int iters, unsigned long long* sink) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ uint64_t bar[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t nbig = big_bytes / CHUNK, nsmall = small_bytes / CHUNK;
    unsigned long long acc = 0;
    auto src_of = [&](int i) -> const char* {
        size_t g = (size_t)i * gridDim.x + blockIdx.x;
        bool hit = mode == 1 || (mode == 2 && (i & 1));
        return hit ? small + (g % nsmall) * CHUNK : big + (g % nbig) * CHUNK;
    };
    for (int i = 0; i < STAGES && i < iters; ++i) {
        mbar_expect(&bar[i], CHUNK);
        bulk_g2s(smem + i * CHUNK, src_of(i), CHUNK, &bar[i]);
    }
    for (int i = 0; i < iters; ++i) {
        int s = i % STAGES;
        mbar_wait(&bar[s], (i / STAGES) & 1);
        acc += *(volatile unsigned*)(smem + s * CHUNK);
        int j = i + STAGES;
        if (j < iters) {
            mbar_expect(&bar[s], CHUNK);
            bulk_g2s(smem + s * CHUNK, src_of(j), CHUNK, &bar[s]);
        }
    }
    sink[blockIdx.x] = acc;
}

// mode 3: 2D tensor TMA (SWIZZLE_128B, box 64 x 128 bf16 = 16 KB, the executor's operand box)
// streaming 128-row panels of a [rows x K] matrix k-block by k-block, 2 boxes per 32 KB stage.
__global__ void __launch_bounds__(32) probe2d(const __grid_constant__ CUtensorMap map, int64_t rows, int64_t K,
                                              int stages, int panels_per_cta, unsigned long long* sink) {
    extern __shared__ __align__(1024) char smem_raw[];
    char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar[16];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int kb = (int)(K / 64), npan = (int)(rows / 128);
    const int per_stage = 2;
    const int steps = panels_per_cta * kb / per_stage;
    auto issue = [&](int i, int s) {
        mbar_expect(&bar[s], 32768);
        for (int q = 0; q < per_stage; ++q) {
            int lin = i * per_stage + q;
            int pan = ((lin / kb) * gridDim.x + blockIdx.x) % npan, kk = lin % kb;
            uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + s * 32768 + q * 16384);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
                "l"(&map), "r"((uint32_t)__cvta_generic_to_shared(&bar[s])), "r"(kk * 64), "r"(pan * 128)
                : "memory");
        }
    };
    unsigned long long acc = 0;
    for (int i = 0; i < stages && i < steps; ++i) issue(i, i);
    for (int i = 0; i < steps; ++i) {
        int s = i % stages;
        mbar_wait(&bar[s], (i / stages) & 1);
        acc += *(volatile unsigned*)(smem + s * 32768);
        if (i + stages < steps) issue(i + stages, s);
    }
    sink[blockIdx.x] = acc;
}

void run2d(char* big, size_t bb, int64_t K, int stages, unsigned long long* sink, int nsm) {
    int64_t rows = (int64_t)(bb / (K * 2)) / 128 * 128;
    CUtensorMap map;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(K * 2)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, big, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = stages * 32768 + 1024;
    cudaFuncSetAttribute(probe2d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // 256 MB per launch in total
    int panels = (int)(((size_t)256 << 20) / ((size_t)128 * K * 2) / nsm);
    if (panels < 1) panels = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe2d<<<nsm, 32, smem>>>(map, rows, K, stages, panels, sink);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) probe2d<<<nsm, 32, smem>>>(map, rows, K, stages, panels, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)panels * 128 * K * 2 * nsm * reps;
    printf("{\"mode\": 3, \"K\": %lld, \"stages\": %d, \"GBps\": %.1f}\n", (long long)K, stages,
           bytes / (ms * 1e-3) / 1e9);
}

template <int STAGES, int CHUNK>
void run(const char* big, size_t bb, const char* small, size_t sb, unsigned long long* sink, int nsm, int mode) {
    const int smem = STAGES * CHUNK;
    cudaFuncSetAttribute(probe<STAGES, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = (int)((size_t)256 << 20) / (CHUNK * nsm);   // 256 MB in total
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<STAGES, CHUNK><<<nsm, 32, smem>>>(big, bb, small, sb, mode, iters, sink);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) probe<STAGES, CHUNK><<<nsm, 32, smem>>>(big, bb, small, sb, mode, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)iters * CHUNK * nsm * reps;
    printf("{\"mode\": %d, \"stages\": %d, \"chunk\": %d, \"GBps\": %.1f, \"per_sm_GBps\": %.1f}\n", mode, STAGES, CHUNK,
           bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / nsm);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    size_t bb = (size_t)2 << 30, sb = (size_t)16 << 20;
    char *big, *small;
    unsigned long long* sink;
    cudaMalloc(&big, bb);
    cudaMalloc(&small, sb);
    cudaMalloc(&sink, 4096 * 8);
    cudaMemset(big, 1, bb);
    cudaMemset(small, 1, sb);
    for (int mode = 0; mode < 3; ++mode) {
        run<2, 32768>(big, bb, small, sb, sink, nsm, mode);
        run<4, 32768>(big, bb, small, sb, sink, nsm, mode);
        run<6, 32768>(big, bb, small, sb, sink, nsm, mode);
        run<12, 16384>(big, bb, small, sb, sink, nsm, mode);
        run<6, 16384>(big, bb, small, sb, sink, nsm, mode);
    }
    for (int64_t K : {64, 128, 256, 576, 1152, 4608})
        for (int st : {4, 6})
            run2d(big, bb, K, st, sink, nsm);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
