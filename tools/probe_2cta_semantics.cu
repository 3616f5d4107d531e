// cta_group::2 operand semantics check (tools only): one M=256 MMA over a CTA
// pair.  Expectation tested: A rows [128r, 128r+128) come from CTA r's shared
// memory, B's N columns [N/2 r, N/2 r + N/2) from CTA r's shared memory, and CTA r's
// TMEM receives D rows [128r, 128r+128) x all N columns.  Both SS (K-major A and
// B) and TS (A from each CTA's TMEM, B MN-major) forms.  Also a cta_group::2
// TMA-free operand fill: every CTA writes its own operands with st.shared.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

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
// SW128 K-major tile of R rows x 64 bf16: element (row, col) at row*128 + ((col/8) ^ (row%8))*16 + (col%8)*2
__device__ __forceinline__ uint32_t sw128(int row, int col) {
    return row * 128 + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2;
}

// A: [256][64] (M x K, K-major), B (SS): [N][64] K-major; D = A B^T.
// TS: P in TMEM (A, 128 x K=64 per CTA), B = V [K=64][N] MN-major.
__global__ void __launch_bounds__(128, 1) k(const float* A, const float* B, const float* V, float* D_ss, float* D_ts,
                                            int N) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 98304);
    uint32_t& tbase = *reinterpret_cast<uint32_t*>(smem + 98304 + 16);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t r = cluster_rank();
    __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(smem);           // 128 x 64 (this CTA's rows)
    __nv_bfloat16* sB = reinterpret_cast<__nv_bfloat16*>(smem + 16384);   // N/2 x 64 (this CTA's B rows)
    __nv_bfloat16* sV = reinterpret_cast<__nv_bfloat16*>(smem + 32768);   // K=64 x N/2 (this CTA's V columns, MN-major)
    for (int i = tid; i < 128 * 64; i += 128) {
        const int row = i / 64, col = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(smem + sw128(row, col)) = __float2bfloat16(A[(128 * r + row) * 64 + col]);
    }
    for (int i = tid; i < (N / 2) * 64; i += 128) {
        const int row = i / 64, col = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(smem + 16384 + sw128(row, col)) =
            __float2bfloat16(B[(N / 2 * r + row) * 64 + col]);
    }
    // V [K=64 keys][N]: this CTA's N/2 columns, MN-major SW128: key row kr, column n -> sw128(kr, n) (N/2 <= 64)
    for (int i = tid; i < 64 * (N / 2); i += 128) {
        const int kr = i / (N / 2), n = i % (N / 2);
        *reinterpret_cast<__nv_bfloat16*>(smem + 32768 + sw128(kr, n)) = __float2bfloat16(V[kr * N + N / 2 * r + n]);
    }
    (void)sA; (void)sB; (void)sV;
    fence_proxy_async_smem();
    if (tid == 0) {
        mbar_init(smem_u32(&bar[0]), 1);
        mbar_init(smem_u32(&bar[1]), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tbase;
    // P for TS: this CTA's A rows as bf16 pairs into TMEM columns [256, 288) (K=64 -> 32 cols)
    {
        const int row = tid;  // lane
        uint32_t pk[32];
        for (int c = 0; c < 32; ++c) {
            const float a0 = A[(128 * r + row) * 64 + 2 * c], a1 = A[(128 * r + row) * 64 + 2 * c + 1];
            pk[c] = pack_bf16(a0, a1);
        }
        tmem_st32(tmem + 256 + ((static_cast<uint32_t>(warp) * 32) << 16), pk);
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (r == 0 && tid == 0) {
        const uint32_t idS = umma_idesc_bf16(256, N, 0, 0), idT = umma_idesc_bf16(256, N, 0, 1);
        const uint64_t da = umma_desc_sw128(smem_u32(smem), 16, 1024), db = umma_desc_sw128(smem_u32(smem) + 16384, 16, 1024);
        const uint64_t dv = umma_desc_sw128(smem_u32(smem) + 32768, 8192, 1024);
        for (int kk = 0; kk < 4; ++kk)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da + kk * 2), "l"(db + kk * 2), "r"(idS), "r"(kk > 0 ? 1u : 0u) : "memory");
        for (int kk = 0; kk < 4; ++kk)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 128),
                         "r"(tmem + 256 + kk * 8), "l"(dv + ((kk * 2048) >> 4)), "r"(idT), "r"(kk > 0 ? 1u : 0u)
                         : "memory");
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&bar[0])), "h"(static_cast<uint16_t>(3)) : "memory");
    }
    mbar_wait(smem_u32(&bar[0]), 0);
    tc_fence_after();
    {
        const int row = tid;
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t u[32];
            tmem_ld32(tmem + c0 + ((static_cast<uint32_t>(warp) * 32) << 16), u);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) D_ss[(128 * r + row) * N + c0 + j] = __uint_as_float(u[j]);
            tmem_ld32(tmem + 128 + c0 + ((static_cast<uint32_t>(warp) * 32) << 16), u);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) D_ts[(128 * r + row) * N + c0 + j] = __uint_as_float(u[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

static float bfr(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
    for (int N : {64, 128}) {
        const int M = 256, K = 64;
        float *A, *B, *V, *Dss, *Dts;
        cudaMallocManaged(&A, M * K * 4);
        cudaMallocManaged(&B, N * K * 4);
        cudaMallocManaged(&V, K * N * 4);
        cudaMallocManaged(&Dss, M * N * 4);
        cudaMallocManaged(&Dts, M * N * 4);
        srand(1);
        for (int i = 0; i < M * K; ++i) A[i] = bfr((rand() % 17 - 8) / 8.f);
        for (int i = 0; i < N * K; ++i) B[i] = bfr((rand() % 17 - 8) / 8.f);
        for (int i = 0; i < K * N; ++i) V[i] = bfr((rand() % 17 - 8) / 8.f);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = 98304 + 64;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 64);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, (const float*)A, (const float*)B, (const float*)V, Dss, Dts, N);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        double ess = 0, ets = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0, t = 0;
                for (int kk = 0; kk < K; ++kk) {
                    s += double(A[m * K + kk]) * B[n * K + kk];
                    t += double(A[m * K + kk]) * V[kk * N + n];
                }
                ess = fmax(ess, fabs(s - Dss[m * N + n]));
                ets = fmax(ets, fabs(t - Dts[m * N + n]));
            }
        printf("N=%d: SS max|err| %.3g  TS max|err| %.3g  [%s]\n", N, ess, ets, cudaGetErrorString(e));
    }
    return 0;
}
