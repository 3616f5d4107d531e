// Test-only probes of the sm_100a building blocks used by the attention
// kernels: TMA (3-D, SW128) -> smem -> tcgen05.mma (SS and TS forms) -> TMEM
// -> tcgen05.ld.  Compared against torch matmul in tests/test_gpu_probe.py.
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>

#include "../../paper_2407_17678_b200/csrc/kernels/sm100_ptx.cuh"
#include "../../paper_2407_17678_b200/csrc/tma_host.hpp"

using namespace s2dev;

// D[128 x N] = A[128 x K] * B[N x K]^T, both K-major bf16.
__global__ void __launch_bounds__(128, 1)
    probe_ss_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                    int N, int K, float* D) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[2];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32;
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = sA + (K / 64) * 16384;
    if (tid == 0) {
        mbar_init(smem_u32(&bars[0]), 1);
        mbar_init(smem_u32(&bars[1]), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_s;
    if (tid == 0) {
        const uint32_t bar = smem_u32(&bars[0]);
        mbar_expect_tx(bar, (K / 64) * (16384 + N * 128));
        for (int s = 0; s < K / 64; ++s) {
            tma_load_3d(sA + s * 16384, &mA, bar, s * 64, 0, 0);
            tma_load_3d(sB + s * N * 128, &mB, bar, s * 64, 0, 0);
        }
        mbar_wait(bar, 0);
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
        for (int kk = 0; kk < K / 16; ++kk) {
            const int sub = kk / 4, off = (kk % 4) * 32;
            const uint64_t ad = umma_desc_sw128(sA + sub * 16384 + off, 16, 1024);
            const uint64_t bd = umma_desc_sw128(sB + sub * N * 128 + off, 16, 1024);
            mma_ss(tbase, ad, bd, idesc, kk > 0);
        }
        mma_commit(smem_u32(&bars[1]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bars[1]), 0);
    tc_fence_after();
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + ((warp * 32) << 16) + c, r);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[tid * N + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

// O[128 x Dv] = P[128 x KK] (fp32 in, rounded to bf16, placed in TMEM) *
//               V[KK x Dv] (bf16, Dv contiguous = MN-major B operand).
__global__ void __launch_bounds__(128, 1)
    probe_ts_kernel(const float* P, const __grid_constant__ CUtensorMap mV, int KK, int Dv,
                    float* O) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[3];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32;
    const uint32_t sV = smem_u32(smem);
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(smem_u32(&bars[i]), i == 2 ? 128 : 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_s;
    const uint32_t tP = tbase + 256;
    // every thread writes its P row as packed bf16 pairs
    for (int c = 0; c < KK / 2; c += 16) {
        uint32_t r[16];
        for (int j = 0; j < 16; ++j)
            r[j] = pack_bf16(P[tid * KK + 2 * (c + j)], P[tid * KK + 2 * (c + j) + 1]);
        tmem_st16(tP + ((warp * 32) << 16) + c, r);
    }
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(smem_u32(&bars[2]));
    if (tid == 0) {
        const uint32_t bar = smem_u32(&bars[0]);
        mbar_expect_tx(bar, (Dv / 64) * KK * 128);
        for (int s = 0; s < Dv / 64; ++s) tma_load_3d(sV + s * KK * 128, &mV, bar, s * 64, 0, 0);
        mbar_wait(bar, 0);
        mbar_wait(smem_u32(&bars[2]), 0);
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, Dv, 0, 1);
        for (int kk = 0; kk < KK / 16; ++kk) {
            const uint64_t bd = umma_desc_sw128(sV + kk * 16 * 128, KK * 128, 1024);
            mma_ts(tbase, tP + kk * 8, bd, idesc, kk > 0);
        }
        mma_commit(smem_u32(&bars[1]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bars[1]), 0);
    tc_fence_after();
    for (int c = 0; c < Dv; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + ((warp * 32) << 16) + c, r);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) O[tid * Dv + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

static thread_local char g_msg[512];

extern "C" const char* probe_last_error() { return g_msg; }

// A: device bf16 [128][K]; B: device bf16 [N][K]; D: device f32 [128][N].
extern "C" int probe_ss(const void* A, const void* B, int N, int K, float* D) {
    try {
        const CUtensorMap mA = s2host::make_map_bf16_3d(A, K, 128, 1, 64, 128);
        const CUtensorMap mB = s2host::make_map_bf16_3d(B, K, N, 1, 64, N);
        const int smem = 1024 + (K / 64) * (16384 + N * 128);
        cudaFuncSetAttribute(probe_ss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_ss_kernel<<<1, 128, smem>>>(mA, mB, N, K, D);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            snprintf(g_msg, sizeof g_msg, "%s", cudaGetErrorString(e));
            return 2;
        }
        return 0;
    } catch (const std::exception& ex) {
        snprintf(g_msg, sizeof g_msg, "%s", ex.what());
        return 1;
    }
}

// P: device f32 [128][KK]; V: device bf16 [KK][Dv]; O: device f32 [128][Dv].
extern "C" int probe_ts(const float* P, const void* V, int KK, int Dv, float* O) {
    try {
        const CUtensorMap mV = s2host::make_map_bf16_3d(V, Dv, KK, 1, 64, KK);
        const int smem = 1024 + (Dv / 64) * KK * 128;
        cudaFuncSetAttribute(probe_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_ts_kernel<<<1, 128, smem>>>(P, mV, KK, Dv, O);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            snprintf(g_msg, sizeof g_msg, "%s", cudaGetErrorString(e));
            return 2;
        }
        return 0;
    } catch (const std::exception& ex) {
        snprintf(g_msg, sizeof g_msg, "%s", ex.what());
        return 1;
    }
}
