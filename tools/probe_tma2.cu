// TMA tensor-load throughput per SM, kernel-like layout (tools only).
// Variants: box rows {64,128}, stage bytes, stages, barrier placement, L2 hint.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2407_17678_b200/csrc/tma_host.hpp"
#include "../paper_2407_17678_b200/csrc/kernels/sm100_ptx.cuh"
using namespace s2dev;

// 4-D map [outer][rows][2 halves][64]: one box {64, box_rows, 2} = both 128-B column
// halves of box_rows rows, landing as [half][row][64] (the SW128 K-major sub-slices).
static CUtensorMap make_map_4d(const void* base, uint64_t rows, uint64_t outer, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {64, rows, 2, outer};
    const cuuint64_t strides[3] = {256, 128, rows * 256};
    const cuuint32_t box[4] = {64, box_rows, 2, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = s2host::tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                                                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("4d encode failed %d\n", int(r));
    return m;
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__global__ void __launch_bounds__(128, 1) k4(const __grid_constant__ CUtensorMap m, int outer, int rows, int box_rows,
                                             int steps, int nst, int stage_bytes, int seq, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
    uint64_t* empty = full + 16;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(smem_u32(&full[i]), 1);
            mbar_init(smem_u32(&empty[i]), 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const int box_bytes = box_rows * 256, per = stage_bytes / box_bytes;
    if (tid == 0) {
        uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
        int row = 0, o = blockIdx.x % outer;
        for (int s = 0; s < steps; ++s) {
            const int st = s % nst;
            if (s >= nst) mbar_wait(smem_u32(&empty[st]), ((s / nst) + 1) & 1);
            const uint32_t bar = smem_u32(&full[st]);
            mbar_expect_tx(bar, stage_bytes);
            for (int kk = 0; kk < per; ++kk) {
                if (seq) {
                    row = (row + box_rows) % rows;
                } else {
                    x = x * 6364136223846793005ull + 1442695040888963407ull;
                    row = int((x >> 40) % (rows / box_rows)) * box_rows;
                    o = int((x >> 20) % outer);
                }
                tma_load_4d(smem_u32(smem + st * stage_bytes + kk * box_bytes), &m, bar, 0, row, 0, o);
            }
        }
    } else if (tid == 32) {
        for (int s = 0; s < steps; ++s) {
            const int st = s % nst;
            mbar_wait(smem_u32(&full[st]), (s / nst) & 1);
            mbar_arrive(smem_u32(&empty[st]));
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap m, int outer, int rows, int box_rows,
                                            int steps, int nst, int stage_bytes, int hint, int seq, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
    uint64_t* empty = full + 16;
    const int tid = threadIdx.x;
    if (tid == 0) {
        if (smem_u32(smem) & 1023) __trap();
        for (int i = 0; i < nst; ++i) {
            mbar_init(smem_u32(&full[i]), 1);
            mbar_init(smem_u32(&empty[i]), 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const int box_bytes = box_rows * 128, per = stage_bytes / box_bytes;
    if (tid == 0) {
        const uint64_t pol = policy_evict_last();
        uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
        int row = 0, o = blockIdx.x % outer;
        for (int s = 0; s < steps; ++s) {
            const int st = s % nst;
            if (s >= nst) mbar_wait(smem_u32(&empty[st]), ((s / nst) + 1) & 1);
            const uint32_t bar = smem_u32(&full[st]);
            mbar_expect_tx(bar, stage_bytes);
            for (int kk = 0; kk < per; kk += 2) {
                if (seq) {
                    row = (row + box_rows) % rows;
                } else {
                    x = x * 6364136223846793005ull + 1442695040888963407ull;
                    row = int((x >> 40) % (rows / box_rows)) * box_rows;
                    o = int((x >> 20) % outer);
                }
                for (int h = 0; h < 2 && kk + h < per; ++h) {
                    const uint32_t dst = smem_u32(smem + st * stage_bytes + (kk + h) * box_bytes);
                    if (hint) tma_load_3d_hint(dst, &m, bar, h * 64, row, o, pol);
                    else tma_load_3d(dst, &m, bar, h * 64, row, o);
                }
            }
        }
    } else if (tid == 32) {
        for (int s = 0; s < steps; ++s) {
            const int st = s % nst;
            mbar_wait(smem_u32(&full[st]), (s / nst) & 1);
            mbar_arrive(smem_u32(&empty[st]));
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

int main(int argc, char** argv) {
    const size_t foot = argc > 1 ? strtoull(argv[1], 0, 0) : (512ull << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* src;
    cudaMalloc(&src, foot);
    cudaMemset(src, 0, foot);
    long long* cyc;
    cudaMalloc(&cyc, sms * sizeof(long long));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const int rows = 32768;
    const int outer = int(foot / (size_t(rows) * 256));
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int box_rows : {64, 128})
        for (int seq : {1, 0}) {
            const CUtensorMap m = make_map_4d(src, rows, outer, box_rows);
            const int cfg[][2] = {{32768, 4}, {65536, 2}, {65536, 3}};
            for (auto& c : cfg) {
                const int sb = c[0], nst = c[1];
                const int steps = int((1024ll << 20) / sms / sb);
                const int smem = sb * nst + 512;
                k4<<<sms, 128, smem>>>(m, outer, rows, box_rows, 4, nst, sb, seq, cyc);
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                k4<<<sms, 128, smem>>>(m, outer, rows, box_rows, steps, nst, sb, seq, cyc);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                long long h[256];
                cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
                double mc = 0;
                for (int i = 0; i < sms; ++i) mc += h[i];
                mc /= sms;
                const double bytes = double(steps) * sb * sms;
                printf("4D box 64x%3dx2 %s stage %6d x %d: %6.2f TB/s %5.1f B/SM-cyc (%4.0f MHz) %s\n", box_rows,
                       seq ? "seq" : "rnd", sb, nst, bytes / ms / 1e9, bytes / sms / mc, mc / (ms * 1e3),
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    for (int box_rows : {64, 128})
        for (int seq : {1, 0})
            for (int hint : {0}) {
                const CUtensorMap m = s2host::make_map_bf16_3d(src, 128, rows, outer, 64, box_rows);
                const int cfg[][2] = {{32768, 4}, {65536, 2}, {65536, 3}, {16384, 8}};
                for (auto& c : cfg) {
                    const int sb = c[0], nst = c[1];
                    if (sb < 2 * box_rows * 128) continue;
                    const int steps = int((1024ll << 20) / sms / sb);
                    const int smem = sb * nst + 512;
                    k<<<sms, 128, smem>>>(m, outer, rows, box_rows, 4, nst, sb, hint, seq, cyc);
                    cudaEvent_t a, b;
                    cudaEventCreate(&a);
                    cudaEventCreate(&b);
                    cudaEventRecord(a);
                    k<<<sms, 128, smem>>>(m, outer, rows, box_rows, steps, nst, sb, hint, seq, cyc);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    long long h[256];
                    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
                    double mc = 0;
                    for (int i = 0; i < sms; ++i) mc += h[i];
                    mc /= sms;
                    const double bytes = double(steps) * sb * sms;
                    printf("box 64x%3d %s hint=%d stage %6d x %d: %6.2f TB/s %5.1f B/SM-cyc (%4.0f MHz) %s\n", box_rows,
                           seq ? "seq" : "rnd", hint, sb, nst, bytes / ms / 1e9, bytes / sms / mc, mc / (ms * 1e3),
                           cudaGetErrorString(cudaGetLastError()));
                }
            }
    return 0;
}
