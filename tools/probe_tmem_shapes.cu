// tcgen05.ld / st .16x256b fragment layout probe (tools only): TMEM filled with
// value = lane * 1000 + column through 32x32b stores; each thread of warp 0
// loads one 16x256b.x2 fragment at lane offset 0 and 16 and prints what it got.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2407_17678_b200/csrc/kernels/sm100_ptx.cuh"
using namespace s2dev;

__global__ void k(int* out) {
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) { tmem_alloc(smem_u32(&tbase), 128); tmem_relinquish(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t t = tbase;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = tid * 1000 + c;
    tmem_st32(t + ((warp * 32) << 16), v);
    for (int c = 0; c < 32; ++c) v[c] = tid * 1000 + 32 + c;
    tmem_st32(t + 32 + ((warp * 32) << 16), v);
    tmem_st_wait();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    for (int h = 0; h < 2; ++h) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(t + (((warp * 32) + 16 * h) << 16)));
        tmem_ld_wait();
        for (int i = 0; i < 8; ++i) out[(h * 128 + tid) * 8 + i] = r[i];
    }
    // st 16x256b.x1 of (tid*10 + i) at lane offset 0, cols 64.., read back with 32x32b
    {
        uint32_t r[4] = {uint32_t(tid * 10), uint32_t(tid * 10 + 1), uint32_t(tid * 10 + 2), uint32_t(tid * 10 + 3)};
        asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(t + 64 + ((warp * 32) << 16)),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
        tmem_st_wait();
        uint32_t u[32];
        tmem_ld32(t + 64 + ((warp * 32) << 16), u);
        tmem_ld_wait();
        for (int i = 0; i < 8; ++i) out[(256 + tid) * 8 + i] = u[i];
    }
    // st 16x128b.x2 of (tid*10 + i) at lane offset 16, cols 96..103, read back with 32x32b
    {
        uint32_t r[4] = {uint32_t(tid * 10), uint32_t(tid * 10 + 1), uint32_t(tid * 10 + 2), uint32_t(tid * 10 + 3)};
        asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(t + 96 + ((warp * 32 + 16) << 16)),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
        tmem_st_wait();
        uint32_t u[32];
        tmem_ld32(t + 96 + ((warp * 32) << 16), u);
        tmem_ld_wait();
        for (int i = 0; i < 8; ++i) out[(384 + tid) * 8 + i] = u[i];
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc(t, 128);
}

int main() {
    int* d; cudaMallocManaged(&d, 512 * 8 * 4);
    k<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(e));
    for (int h = 0; h < 2; ++h)
        for (int t = 0; t < 32; t += 1) {
            printf("ld16x256b.x2 h=%d thread %2d:", h, t);
            for (int i = 0; i < 8; ++i) printf(" %6d", d[(h * 128 + t) * 8 + i]);
            printf("\n");
        }
    for (int t = 0; t < 16; ++t) {
        printf("st16x256b.x1 -> lane %2d cols 64..71:", t);
        for (int i = 0; i < 8; ++i) printf(" %4d", d[(256 + t) * 8 + i]);
        printf("\n");
    }
    for (int t = 16; t < 32; ++t) {
        printf("st16x128b.x2 @lane16 -> lane %2d cols 96..103:", t);
        for (int i = 0; i < 8; ++i) printf(" %4d", d[(384 + t) * 8 + i]);
        printf("\n");
    }
    return 0;
}
