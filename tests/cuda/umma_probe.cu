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
                    int N, int K, float* D, int a_in_tmem) {
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
            if (a_in_tmem) {
                // A's K slice kk: smem (SW128 K-major) -> TMEM columns 256 + 8kk (128 lanes x 256 bit)
                asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tbase + 256 + kk * 8), "l"(ad)
                             : "memory");
                mma_ts(tbase, tbase + 256 + kk * 8, bd, idesc, kk > 0);
            } else {
                mma_ss(tbase, ad, bd, idesc, kk > 0);
            }
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
extern "C" int probe_ss_tmem_a(const void* A, const void* B, int N, int K, float* D, int a_in_tmem);
extern "C" int probe_ss(const void* A, const void* B, int N, int K, float* D) {
    return probe_ss_tmem_a(A, B, N, K, D, 0);
}
// a_in_tmem: A staged smem -> TMEM with tcgen05.cp.128x256b, then TS MMAs
extern "C" int probe_ss_tmem_a(const void* A, const void* B, int N, int K, float* D, int a_in_tmem) {
    try {
        const CUtensorMap mA = s2host::make_map_bf16_3d(A, K, 128, 1, 64, 128);
        const CUtensorMap mB = s2host::make_map_bf16_3d(B, K, N, 1, 64, N);
        const int smem = 1024 + (K / 64) * (16384 + N * 128);
        cudaFuncSetAttribute(probe_ss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        probe_ss_kernel<<<1, 128, smem>>>(mA, mB, N, K, D, a_in_tmem);
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

// ---- throughput probe: back-to-back MMAs on resident operands -------------
// kind 0: SS  (A smem K-major 128 x 64, B smem K-major N x 64)
// kind 1: TS  (A tmem, B smem MN-major 16 x N rows)
__global__ void __launch_bounds__(128, 1) probe_rate_kernel(int kind, int N, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base_s;
    if (tid == 0) {
        const uint32_t sA = smem_u32(smem), sB = sA + 32768;
        const long long t0 = clock64();
        if (kind == 0) {
            const uint32_t id = umma_idesc_bf16(128, N, 0, 0);
            for (int i = 0; i < iters; ++i) {
                const int kk = i & 3;
                mma_ss(tb, umma_desc_sw128(sA + kk * 32, 16, 1024), umma_desc_sw128(sB + kk * 32, 16, 1024), id, 1);
            }
        } else {
            const uint32_t id = umma_idesc_bf16(128, N, 0, 1);
            for (int i = 0; i < iters; ++i) {
                const int kk = i & 3;
                mma_ts(tb, tb + 256 + kk * 8, umma_desc_sw128(sB + kk * 2048, 8192, 1024), id, 1);
            }
        }
        const long long t1 = clock64();
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int probe_rate(int kind, int N, int iters, long long* host_out) {
    long long* d;
    cudaMalloc(&d, 16);
    const int smem = 1024 + 65536;
    cudaFuncSetAttribute(probe_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_rate_kernel<<<1, 128, smem>>>(kind, N, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) {
        snprintf(g_msg, sizeof g_msg, "%s", cudaGetErrorString(e));
        return 2;
    }
    return 0;
}

__device__ __forceinline__ bool lane_is_zero() { return (threadIdx.x & 31) == 0; }

// ---- the dK/dV step's MMA sequence alone (no TMA, no elementwise) ----------
// per step: S^T (SS N=64 x 8), dP^T (SS N=64 x 8), dV (TS N=128 x 4), dK (TS N=128 x 4)
__global__ void __launch_bounds__(256, 1) probe_dkv_seq_kernel(int steps, int variant, long long* out, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2[2];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 131072 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar2[0]), 1);
        mbar_init(smem_u32(&bar2[1]), 1);
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base_s;
    if (tid == 0) {
        const uint32_t sK0 = smem_u32(smem);
        const uint32_t idS = umma_idesc_bf16(128, 64, 0, 0), idA = umma_idesc_bf16(128, 128, 0, 1);
        const long long t0 = clock64();
        for (int n = 0; n < steps; ++n) {
            const int b = n & 1;
            const uint32_t sK = sK0, sV = sK0 + 32768;
            const uint32_t rot = variant == 11 ? (n % 2) * 32768 : 0;  // rotate Q/dO stage
            const uint32_t sQ = sK0 + 65536 + rot - (variant == 11 ? 0 : 0), sdO = sQ + 16384;
            if (variant != 2) {
                for (int kk = 0; kk < 8; ++kk) {
                    const int sub = kk >> 2, off = (kk & 3) * 32;
                    mma_ss(tb + b * 64, umma_desc_sw128(sK + sub * 16384 + off, 16, 1024),
                           umma_desc_sw128(sQ + sub * 8192 + off, 16, 1024), idS, kk > 0);
                    mma_ss(tb + 128 + b * 64, umma_desc_sw128(sV + sub * 16384 + off, 16, 1024),
                           umma_desc_sw128(sdO + sub * 8192 + off, 16, 1024), idS, kk > 0);
                }
            }
            if (variant == 7 || variant == 8) mma_commit(smem_u32(&bar2[0]));
            if (variant == 9) tc_fence_after();
            if (variant == 10) {
                mma_commit(smem_u32(&bar2[0]));
                mbar_wait(smem_u32(&bar2[0]), n & 1);  // wait for the group, like waiting S before PV
                tc_fence_after();
            }
            if (variant != 1) {
                for (int kk = 0; kk < 4; ++kk) {
                    mma_ts(tb + 256, tb + b * 64 + kk * 8, umma_desc_sw128(sdO + kk * 2048, 8192, 1024), idA, 1);
                    mma_ts(tb + 384, tb + 128 + b * 64 + kk * 8, umma_desc_sw128(sQ + kk * 2048, 8192, 1024), idA, 1);
                }
            }
            if (variant == 8) mma_commit(smem_u32(&bar2[1]));
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        out[0] = clock64() - t0;
        atomicExch(reinterpret_cast<int*>(&tmem_base_s) + 0, tb);  // keep
        *reinterpret_cast<volatile int*>(out + 1) = 1;  // done flag
    }
    if (warp == 4 && variant == 5 && lane_is_zero()) {
        // contention: TMA bulk copies of 32 KB per ~1000 cycles into a spare region
        __shared__ uint64_t tbar;
        mbar_init(smem_u32(&tbar), 1);
        fence_mbar_init();
        const uint32_t dst = smem_u32(smem) + 131072 - 32768;
        uint32_t ph = 0;
        int it = 0;
        while (*reinterpret_cast<volatile int*>(out + 1) == 0 && it < 100000) {
            mbar_expect_tx(smem_u32(&tbar), 32768);
            for (int c = 0; c < 4; ++c)
                bulk_load(dst + c * 8192, gsrc + (static_cast<size_t>(it % 64) * 32768) + c * 8192, 8192, smem_u32(&tbar));
            mbar_wait(smem_u32(&tbar), ph);
            ph ^= 1;
            ++it;
        }
    }
    if (warp >= 1 && variant == 6) {
        // issue contention: every other warp runs an FMA/MUFU mix until done
        float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.f;
        int it = 0;
        while (*reinterpret_cast<volatile int*>(out + 1) == 0 && it < 2000000) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                a = fmaf(a, b, 1e-7f);
                c += fast_exp2(a);
            }
            ++it;
        }
        if (c == 12345.f) out[2] = 1;
    }
    if (warp >= 4 && variant >= 3 && variant <= 4) {
        // contention: load S^T/dP^T-sized chunks and store P-sized chunks like the elementwise WG
        const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
        uint32_t r[32];
        int it = 0;
        while (*reinterpret_cast<volatile int*>(out + 1) == 0 && it < 200000) {
            tmem_ld32(tb + lo + (it & 1) * 64, r);
            tmem_ld32(tb + lo + 128 + (it & 1) * 64, r);
            tmem_ld_wait();
            if (variant == 4) {
                uint32_t w[16];
                for (int j = 0; j < 16; ++j) w[j] = r[j] + 1;
                tmem_st16(tb + lo + 200, w);
                tmem_st_wait();
            }
            ++it;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

__device__ __forceinline__ bool lane_is_zero_dummy() { return true; }
extern "C" int probe_dkv_seq(int steps, int variant, long long* host_out) {
    long long* d;
    cudaMalloc(&d, 32);
    static uint8_t* gsrc = nullptr;
    if (!gsrc) {
        cudaMalloc(&gsrc, 64 * 32768);
        cudaMemset(gsrc, 0, 64 * 32768);
    }
    const int smem = 1024 + 131072;
    cudaFuncSetAttribute(probe_dkv_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(d, 0, 32);
    probe_dkv_seq_kernel<<<1, 256, smem>>>(steps, variant, d, gsrc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : 2;
}

// ---- issue-order probe: 16 MMAs per iteration in a given arrangement --------
// mode 0: SS N=64, one accumulator, one A region (k-slices cycle)
// mode 1: SS N=64, two accumulators / two A regions, interleaved (S, dP, S, dP ...)
// mode 2: SS N=64, two accumulators, grouped (8 x S then 8 x dP)
// mode 3: SS N=128 interleaved        mode 4: SS N=128 grouped
// mode 5: TS N=128 two accumulators interleaved (dV, dK)
// mode 6: SS N=256 interleaved        mode 7: mode 1 with accumulate=0 on each group's first MMA
// mode 8: mode 2 with accumulate=0 on each group's first MMA
template <int mode>
__global__ void __launch_bounds__(128, 1) probe_mix_kernel(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 131072 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base_s;
    if (tid == 0) {
        const uint32_t s0 = smem_u32(smem);
        const uint32_t sA0 = s0, sA1 = s0 + 32768, sB0 = s0 + 65536, sB1 = s0 + 98304;
        constexpr int N = (mode == 3 || mode == 4 || mode == 5) ? 128 : (mode == 6 ? 256 : 64);
        constexpr uint32_t id = umma_idesc_bf16(128, N, 0, mode == 5 ? 1 : 0);
        const uint32_t acc1 = mode == 6 ? 256 : 128;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                int which, kk;
                if (mode == 0) { which = 0; kk = j & 7; }
                else if (mode == 1 || mode == 3 || mode == 5 || mode == 6 || mode == 7) { which = j & 1; kk = j >> 1; }
                else { which = j >> 3; kk = j & 7; }
                const int sub = kk >> 2, off = (kk & 3) * 32;
                const uint32_t acc = ((mode == 7 || mode == 8) && kk == 0) ? 0u : 1u;
                if (mode == 5) {
                    mma_ts(tb + 256 + which * 128 - (which ? 0 : 0), tb + which * 64 + kk * 8,
                           umma_desc_sw128((which ? sB1 : sB0) + kk * 2048, 8192, 1024), id, acc);
                } else {
                    mma_ss(tb + which * acc1, umma_desc_sw128((which ? sA1 : sA0) + sub * 16384 + off, 16, 1024),
                           umma_desc_sw128((which ? sB1 : sB0) + sub * 16384 + off, 16, 1024), id, acc);
                }
            }
        }
        const long long t1 = clock64();
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        out[0] = t1 - t0;
        out[1] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int probe_mix(int mode, int iters, long long* host_out) {
    long long* d;
    cudaMalloc(&d, 16);
    const int smem = 1024 + 131072;
#define PM(M)                                                                                  \
    if (mode == M) {                                                                           \
        cudaFuncSetAttribute(probe_mix_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        probe_mix_kernel<M><<<1, 128, smem>>>(iters, d);                                       \
    }
    PM(0) PM(1) PM(2) PM(3) PM(4) PM(5) PM(7) PM(8)
#undef PM
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : 2;
}

// ---- the dK/dV step's MMA sequence, unrolled issue, with optional contention --
// V bit 0: S^T/dP^T (16 x SS N=64)   bit 1: dV/dK (8 x TS N=128)
// bit 2: warps 4-7 stream TMEM loads of the S/dP columns + P stores (the elementwise WG's traffic)
// bit 3: warp 2 streams 32 KB TMA bulk loads into a spare smem region
template <int V>
__global__ void __launch_bounds__(256, 1) probe_dkv2_kernel(int steps, long long* out, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, tbar;
    __shared__ uint32_t tmem_base_s;
    __shared__ volatile int done;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 163840 / 4; i += 256) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&tbar), 1);
        fence_mbar_init();
        done = 0;
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base_s;
    if (tid == 0) {
        const uint32_t sK = smem_u32(smem), sV = sK + 32768, sQ = sK + 65536, sdO = sQ + 16384;
        constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0), idA = umma_idesc_bf16(128, 128, 0, 1);
        const long long t0 = clock64();
        for (int n = 0; n < steps; ++n) {
            const int b = n & 1;
            if (V & 1) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int sub = kk >> 2, off = (kk & 3) * 32;
                    mma_ss(tb + b * 64, umma_desc_sw128(sK + sub * 16384 + off, 16, 1024),
                           umma_desc_sw128(sQ + sub * 8192 + off, 16, 1024), idS, kk > 0);
                    mma_ss(tb + 128 + b * 64, umma_desc_sw128(sV + sub * 16384 + off, 16, 1024),
                           umma_desc_sw128(sdO + sub * 8192 + off, 16, 1024), idS, kk > 0);
                }
            }
            if (V & 2) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    mma_ts(tb + 256, tb + b * 64 + kk * 8, umma_desc_sw128(sdO + kk * 2048, 8192, 1024), idA, 1);
                    mma_ts(tb + 384, tb + 128 + b * 64 + kk * 8, umma_desc_sw128(sQ + kk * 2048, 8192, 1024), idA, 1);
                }
            }
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        out[0] = clock64() - t0;
        done = 1;
    }
    if ((V & 8) && warp == 2 && (tid & 31) == 0) {
        const uint32_t dst = smem_u32(smem) + 131072;
        uint32_t ph = 0;
        for (int it = 0; it < 100000 && !done; ++it) {
            mbar_expect_tx(smem_u32(&tbar), 32768);
            for (int c = 0; c < 4; ++c)
                bulk_load(dst + c * 8192, gsrc + (static_cast<size_t>(it % 64) * 32768) + c * 8192, 8192, smem_u32(&tbar));
            mbar_wait(smem_u32(&tbar), ph);
            ph ^= 1;
        }
    }
    if ((V & 4) && warp >= 4) {
        const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
        for (int it = 0; it < 400000 && !done; ++it) {
            uint32_t r[32], d[32];
            tmem_ld32(tb + lo + (it & 1) * 64, r);
            tmem_ld32(tb + lo + 128 + (it & 1) * 64, d);
            tmem_ld_wait();
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j] = r[j] ^ d[j + 16];
            tmem_st16(tb + lo + 200, w);
            tmem_st16(tb + lo + 232, w);
            tmem_st_wait();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int probe_dkv2(int steps, int variant, long long* host_out) {
    long long* d;
    cudaMalloc(&d, 16);
    static uint8_t* gsrc = nullptr;
    if (!gsrc) {
        cudaMalloc(&gsrc, 64 * 32768);
        cudaMemset(gsrc, 0, 64 * 32768);
    }
    const int smem = 1024 + 163840;
#define PD(M)                                                                                         \
    if (variant == M) {                                                                               \
        cudaFuncSetAttribute(probe_dkv2_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        probe_dkv2_kernel<M><<<1, 256, smem>>>(steps, d, gsrc);                                       \
    }
    PD(1) PD(2) PD(3) PD(7) PD(11) PD(15)
#undef PD
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : 2;
}

// ---- TMEM load bandwidth: `nw` warps each issue `iters` x (4 x tcgen05.ld.32x32b.x32)
// then wait; reports cycles of the slowest warp.
__global__ void __launch_bounds__(512, 1) probe_tmem_ld_kernel(int nw, int iters, long long* out) {
    __shared__ uint32_t tmem_base_s;
    __shared__ unsigned long long tmax;
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    if (tid == 0) tmax = 0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base_s;
    if (warp < nw) {
        const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
        uint32_t acc = 0;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            uint32_t r0[32], r1[32], r2[32], r3[32];
            const uint32_t col = ((warp >> 2) * 128 + (i & 1) * 0) & 511;
            tmem_ld32(tb + lo + col, r0);
            tmem_ld32(tb + lo + col + 32, r1);
            tmem_ld32(tb + lo + col + 64, r2);
            tmem_ld32(tb + lo + col + 96, r3);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += r0[j] ^ r1[j] ^ r2[j] ^ r3[j];
        }
        const long long t1 = clock64();
        if ((tid & 31) == 0) atomicMax(&tmax, static_cast<unsigned long long>(t1 - t0));
        if (acc == 0x12345678u) out[1] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) out[0] = static_cast<long long>(tmax);
    if (warp == 0) tmem_dealloc(tb, 512);
}

extern "C" int probe_tmem_ld(int nw, int iters, long long* host_out) {
    long long* d;
    cudaMalloc(&d, 16);
    probe_tmem_ld_kernel<<<1, 512>>>(nw, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(host_out, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : 2;
}
