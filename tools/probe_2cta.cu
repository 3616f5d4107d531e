// tcgen05 MMA rate with a CTA pair (cta_group::2, M=256) vs one CTA (M=128),
// SS and TS, N = 64 / 128 / 256 (tools only, not part of the product).
// Question: does the pair lift the N=64 products the S2 kernels are built on
// (48 cyc SS / 45.6 cyc TS per M=128 MMA on one SM) toward the 32-cycle ideal?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_2cta tools/probe_2cta.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2407_17678_b200/csrc/kernels/sm100_ptx.cuh"

using namespace s2dev;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int PAIR, int TS>
__global__ void __launch_bounds__(128, 1) probe(int N, int iters, long long* out) {
    constexpr int ts = TS;
    extern __shared__ __align__(1024) uint8_t smem[];
    // no static shared memory: the dynamic window stays 1024-B aligned (SW128 atoms)
    uint64_t& bar = *reinterpret_cast<uint64_t*>(smem + 160 * 1024);
    uint32_t& tbase = *reinterpret_cast<uint32_t*>(smem + 160 * 1024 + 8);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = PAIR ? cluster_rank() : 0;
    // operands: zeros (timing only); A 128 x 16 slices at 0, B at 64 KB
    if (tid == 0 && (smem_u32(smem) & 1023u)) __trap();
    for (int i = tid; i < 160 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t M = PAIR ? 256 : 128;
    const uint32_t idesc = umma_idesc_bf16(M, N, 0, 0);
    const uint64_t da = umma_desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t db = umma_desc_sw128(smem_u32(smem) + 32768, 16, 1024);
    if (rank == 0 && tid == 0) {
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // walk the 4 K slices of a 64-wide SW128 atom (+32 B)
                if constexpr (PAIR) {
                    if constexpr (TS)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                                     "r"(tmem + 256 + kk * 8), "l"(db + kk * 2), "r"(idesc), "r"(1u)
                                     : "memory");
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                     "l"(da + kk * 2), "l"(db + kk * 2), "r"(idesc), "r"(1u)
                                     : "memory");
                } else {
                    if constexpr (TS)
                        mma_ts(tmem, tmem + 256 + kk * 8, db + kk * 2, idesc, 1u);
                    else
                        mma_ss(tmem, da + kk * 2, db + kk * 2, idesc, 1u);
                }
            }
        }
        const long long t1 = clock64();
        if (PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             smem_u32(&bar)),
                         "h"(static_cast<uint16_t>(3))
                         : "memory");
        else
            mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    if (PAIR && rank != 0 && tid == 0) mbar_wait(smem_u32(&bar), 0);  // the multicast commit lands here too
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    const int iters = 4096, smem = 160 * 1024 + 64;
    cudaFuncSetAttribute(probe<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ts = 0; ts < 2; ++ts)
        for (int N : {64, 128, 256}) {
            for (int pair = 0; pair < 2; ++pair) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(pair ? 2 : 1);
                cfg.blockDim = dim3(128);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = pair ? 2 : 1;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cudaError_t e = pair ? (ts ? cudaLaunchKernelEx(&cfg, probe<1, 1>, N, iters, d)
                                           : cudaLaunchKernelEx(&cfg, probe<1, 0>, N, iters, d))
                                     : (ts ? cudaLaunchKernelEx(&cfg, probe<0, 1>, N, iters, d)
                                           : cudaLaunchKernelEx(&cfg, probe<0, 0>, N, iters, d));
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
                long long h[2] = {0, 0};
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const double cyc = double(h[1]) / iters;
                const double ideal = 128.0 * N / 256.0;  // per SM: 128 rows x N per MMA
                printf("%s M=%d N=%3d: %6.1f cyc/MMA (issue %6.1f), ideal per SM %5.1f -> %3.0f%%  [%s]\n",
                       ts ? "TS" : "SS", pair ? 256 : 128, N, cyc, double(h[0]) / iters, ideal, 100.0 * ideal / cyc,
                       cudaGetErrorString(e));
                if (e != cudaSuccess) return 1;
            }
        }
    return 0;
}
