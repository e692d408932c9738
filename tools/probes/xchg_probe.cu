// Probe: cost of exchanging fp32 split-K partials between SMs on B200.
//   (a) DSMEM: cluster of 2/4, thread st.shared::cluster.v4 to the peer, cluster barrier
//   (b) DSMEM: cp.async.bulk smem -> peer smem (mbarrier complete_tx)
//   (c) L2: plain st.global.v4 + fence + flag, peer polls flag then loads
// plus cudaOccupancyMaxActiveClusters for the executor's smem footprint.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <int BYTES>
__global__ void __launch_bounds__(128) dsmem_st(uint64_t* out, int reps) {
    extern __shared__ uint4 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const unsigned peer = rank ^ 1;
    uint4* remote = cl.map_shared_rank(sm, peer);
    cl.sync();
    uint64_t t0 = gt();
    for (int r = 0; r < reps; ++r) {
        for (int i = threadIdx.x; i < BYTES / 16; i += 128) remote[i] = make_uint4(i, r, 1, 2);
        cl.sync();
    }
    uint64_t t1 = gt();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void __launch_bounds__(128) dsmem_bulk(uint64_t* out, int reps, int bytes) {
    extern __shared__ __align__(128) uint8_t smb[];
    __shared__ __align__(8) uint64_t bar;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const unsigned peer = rank ^ 1;
    uint8_t* src = smb;
    uint8_t* dst = smb + bytes;
    uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cl.sync();
    uint32_t ph = 0;
    uint64_t t0 = gt();
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(bytes));
        }
        cl.sync();   // peer's expect_tx posted before our copy lands
        if (threadIdx.x == 0) {
            uint32_t dst_local = (uint32_t)__cvta_generic_to_shared(dst);
            uint32_t dst_remote, bar_remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst_remote) : "r"(dst_local), "r"(peer));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar_remote) : "r"(bar_a), "r"(peer));
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst_remote), "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes), "r"(bar_remote) : "memory");
            uint32_t ok = 0;
            while (!ok) {
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                             : "=r"(ok) : "r"(bar_a), "r"(ph));
            }
        }
        ph ^= 1;
        __syncthreads();
    }
    cl.sync();
    uint64_t t1 = gt();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

// L2 exchange between CTA pairs (2b, 2b+1): store partial, fence, flag; peer waits, loads.
__global__ void __launch_bounds__(128) l2_xchg(float4* ws, int* flags, uint64_t* out, int reps, int bytes) {
    const int pair = blockIdx.x >> 1, me = blockIdx.x & 1;
    float4* mine = ws + (size_t)blockIdx.x * (bytes / 16);
    float4* theirs = ws + (size_t)(blockIdx.x ^ 1) * (bytes / 16);
    int* myflag = flags + blockIdx.x;
    int* theirflag = flags + (blockIdx.x ^ 1);
    (void)pair; (void)me;
    float acc = 0;
    uint64_t t0 = gt();
    for (int r = 1; r <= reps; ++r) {
        for (int i = threadIdx.x; i < bytes / 16; i += 128) mine[i] = make_float4(r, i, 0, 0);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(myflag), "r"(r) : "memory");
        if (threadIdx.x == 0) {
            int v = 0;
            do { asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(theirflag) : "memory"); } while (v < r);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < bytes / 16; i += 128) { float4 x = __ldcg(theirs + i); acc += x.x; }
        __syncthreads();
    }
    uint64_t t1 = gt();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps + (acc == -1.f);
}

int main() {
    int dev = 0; cudaSetDevice(dev);
    cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    printf("%s SMs %d\n", p.name, p.multiProcessorCount);
    uint64_t* d_out; cudaMalloc(&d_out, 4096 * 8);
    uint64_t h[4096];
    // occupancy: clusters of the executor's footprint (192 threads, ~225 KB smem)
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = 225 * 1024;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        cudaFuncSetAttribute(dsmem_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dsmem_bulk, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    const int reps = 50;
    {
        cudaFuncSetAttribute(dsmem_st<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 32768;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, dsmem_st<32768>, d_out, reps);
        cudaLaunchKernelEx(&cfg, dsmem_st<32768>, d_out, reps);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, 148 * 8, cudaMemcpyDeviceToHost);
        printf("dsmem st.v4 32KB to peer + cluster.sync: %llu ns (%s) all-148\n", (unsigned long long)h[0], cudaGetErrorString(e));
    }
    for (int bytes : {8192, 16384, 32768, 65536}) {
        cudaFuncSetAttribute(dsmem_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 2 * bytes;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, dsmem_bulk, d_out, reps, bytes);
        cudaLaunchKernelEx(&cfg, dsmem_bulk, d_out, reps, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, 148 * 8, cudaMemcpyDeviceToHost);
        printf("dsmem bulk %d B to peer (+2 cluster syncs): %llu ns  (%s)\n", bytes, (unsigned long long)h[0], cudaGetErrorString(e));
    }
    float4* ws; int* flags;
    cudaMalloc(&ws, 148 * 65536); cudaMalloc(&flags, 148 * 4);
    for (int bytes : {16384, 32768, 65536}) {
        cudaMemset(flags, 0, 148 * 4);
        l2_xchg<<<148, 128>>>(ws, flags, d_out, reps, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, 148 * 8, cudaMemcpyDeviceToHost);
        printf("L2 store+fence+flag+load %d B: %llu ns (%s) [idle GPU]\n", bytes, (unsigned long long)h[0], cudaGetErrorString(e));
    }
    return 0;
}
