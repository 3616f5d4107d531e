// Shared-memory contention probe (tools only): the dK/dV step's four MMAs
// (S^T, dP^T: SS M=128 N=128 K=128; dV, dK: TS M=128 N=128 K=128) issued back to
// back on one SM, alone and with a concurrent TMA stream writing 64 KB per step
// into shared memory, on one CTA and on a CTA pair (cta_group::2, M=256: each SM
// reads only half of every B operand).  Reports cycles per step (ideal 2048).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_smem_bw tools/probe_smem_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2407_17678_b200/csrc/kernels/sm100_ptx.cuh"
#include "../paper_2407_17678_b200/csrc/tma_host.hpp"

using namespace s2dev;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}

// smem: [0,64K) K|V (A operands), [64K,128K) Q|dO (B operands), [128K, 192K) TMA sink
template <int PAIR>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap m, int steps, int tma, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196608);
    uint32_t& tbase = *reinterpret_cast<uint32_t*>(smem + 196608 + 64);
    volatile int& done = *reinterpret_cast<volatile int*>(smem + 196608 + 72);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = PAIR ? cluster_rank() : 0;
    for (int i = tid; i < 131072 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar[0]), 1);
        mbar_init(smem_u32(&bar[1]), 1);
        fence_mbar_init();
        done = 0;
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc(smem_u32(&tbase), 512);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t s0 = smem_u32(smem);
    constexpr uint32_t M = PAIR ? 256 : 128;
    const uint32_t idS = umma_idesc_bf16(M, 128, 0, 0), idA = umma_idesc_bf16(M, 128, 0, 1);
    if (rank == 0 && tid == 0) {
        const uint64_t dK = umma_desc_sw128(s0, 16, 1024), dV = umma_desc_sw128(s0 + 32768, 16, 1024);
        // one CTA: B = full 128-row tiles; pair: each SM holds 64 rows of the B of S^T / dP^T,
        // and 64 of the D columns of the B of dV / dK
        const uint64_t dQ = umma_desc_sw128(s0 + 65536, 16, 1024), ddO = umma_desc_sw128(s0 + 98304, 16, 1024);
        const uint64_t dQmn = umma_desc_sw128(s0 + 65536, 16384, 1024), ddOmn = umma_desc_sw128(s0 + 98304, 16384, 1024);
        const long long t0 = clock64();
        for (int n = 0; n < steps; ++n) {
            const uint32_t reg = (n & 1) * 128;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                if (PAIR) mma2_ss(tmem + reg, dK + o, dQ + o, idS, kk > 0);
                else mma_ss(tmem + reg, dK + o, dQ + o, idS, kk > 0);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (PAIR) mma2_ts(tmem + 256, tmem + reg + kk * 8, ddOmn + ((kk * 2048) >> 4), idA, 1);
                else mma_ts(tmem + 256, tmem + reg + kk * 8, ddOmn + ((kk * 2048) >> 4), idA, 1);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                if (PAIR) mma2_ss(tmem + reg, dV + o, ddO + o, idS, kk > 0);
                else mma_ss(tmem + reg, dV + o, ddO + o, idS, kk > 0);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (PAIR) mma2_ts(tmem + 384, tmem + reg + kk * 8, dQmn + ((kk * 2048) >> 4), idA, 1);
                else mma_ts(tmem + 384, tmem + reg + kk * 8, dQmn + ((kk * 2048) >> 4), idA, 1);
            }
        }
        if (PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             smem_u32(&bar[0])), "h"(static_cast<uint16_t>(3)) : "memory");
        else
            mma_commit(smem_u32(&bar[0]));
        mbar_wait(smem_u32(&bar[0]), 0);
        out[0] = clock64() - t0;
        done = 1;
    }
    if (PAIR && rank != 0 && tid == 0) {
        mbar_wait(smem_u32(&bar[0]), 0);
        done = 1;
    }
    if (tma && warp == 1 && (tid & 31) == 0) {  // 64 KB per `tma` cycles into the sink, while the MMAs run
        uint32_t ph = 0;
        long long bytes = 0;
        const long long t0 = clock64();
        for (int it = 0; !done; ++it) {
            mbar_expect_tx(smem_u32(&bar[1]), 65536);
            tma_load_rows(s0 + 131072, &m, smem_u32(&bar[1]), (it * 128) % 8192, 0);
            tma_load_rows(s0 + 131072 + 32768, &m, smem_u32(&bar[1]), (it * 128 + 128) % 8192, 0);
            mbar_wait(smem_u32(&bar[1]), ph);
            ph ^= 1;
            bytes += 65536;
            while (clock64() - t0 < (it + 1) * static_cast<long long>(tma) && !done) {
            }
        }
        out[1 + rank] = bytes;
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else tmem_dealloc(tmem, 512);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 32);
    void* src;
    cudaMalloc(&src, 8192 * 256);
    cudaMemset(src, 0, 8192 * 256);
    const CUtensorMap m = s2host::make_map_bf16_kmajor(src, 128, 8192, 1, 128);
    const int smem = 196608 + 128, steps = 512;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int pair = 0; pair < 2; ++pair)
        for (int tma : {0, 4000, 2048, 1500, 1}) {
            cudaMemset(d, 0, 32);
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
            cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, probe<1>, m, steps, tma, d)
                                 : cudaLaunchKernelEx(&cfg, probe<0>, m, steps, tma, d);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            long long h[4] = {0, 0, 0, 0};
            cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
            const double cyc = double(h[0]) / steps;
            printf("%s tma every %5d cyc: %6.0f cyc/step (ideal 2048, %3.0f%%); TMA into SM0 %5.1f B/cyc  [%s]\n",
                   pair ? "pair M=256" : "one  M=128", tma, cyc, 100.0 * 2048 / cyc, double(h[1]) / h[0],
                   cudaGetErrorString(e));
        }
    return 0;
}
