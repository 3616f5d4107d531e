// L2 reduce-add throughput probe (tools only, not part of the product).
// Question it answers: can 148 SMs each push one 64 x 128 fp32 dQ partial
// (32 KB) per backward step into HBM-resident accumulators fast enough for
// an in-kernel dQ (FA-style) dK/dV kernel?  Each CTA loops: fill a smem
// tile, issue a bulk reduce-add (or a plain bulk store, or red.global.v4)
// into a pseudo-random 32 KB tile of a 512 MB accumulator; report GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_reduce tools/probe_reduce.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 32768;
__constant__ int kTiles;  // accumulator size in 32 KB tiles

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(128) probe(float* acc, int steps, int nbuf) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* buf = reinterpret_cast<float*>(smem);
    const int tid = threadIdx.x;
    for (int s = 0; s < steps; ++s) {
        const int b = s % nbuf;
        float* sb = buf + b * (kTile / 4);
        const uint32_t tile = (blockIdx.x * 7919u + s * 104729u) % kTiles;
        if (MODE == 2) {
            float4* dst = reinterpret_cast<float4*>(acc + static_cast<size_t>(tile) * (kTile / 4));
            for (int i = tid; i < kTile / 16; i += 128)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "f"(1.f),
                             "f"(1.f), "f"(1.f), "f"(1.f)
                             : "memory");
            continue;
        }
        // the buffer about to be overwritten must have been read by its bulk op
        if (tid == 0) {
            if (nbuf == 2)
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
        for (int i = tid; i < kTile / 16; i += 128)
            reinterpret_cast<float4*>(sb)[i] = make_float4(1.f, 1.f, 1.f, 1.f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            float* dst = acc + static_cast<size_t>(tile) * (kTile / 4);
            if (MODE == 0)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                                 dst),
                             "r"(su32(sb)), "r"(kTile)
                             : "memory");
            else
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(sb)),
                             "r"(kTile)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE>
void run(const char* name, float* acc, int grid, int steps, int nbuf) {
    auto k = probe<MODE>;
    const int sm = MODE == 2 ? 0 : nbuf * kTile;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k<<<grid, 128, sm>>>(acc, steps, nbuf);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<grid, 128, sm>>>(acc, steps, nbuf);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 5.0 * grid * steps * kTile;
    printf("%-12s grid=%4d nbuf=%d  %.3f ms  %.0f GB/s of partials (%s)\n", name, grid, nbuf, ms / 5,
           bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float* acc;
    cudaMalloc(&acc, static_cast<size_t>(kTile) * 16384);
    cudaMemset(acc, 0, static_cast<size_t>(kTile) * 16384);
    for (int tiles : {512, 2048, 4096, 16384}) {
        cudaMemcpyToSymbol(kTiles, &tiles, sizeof(int));
        printf("accumulator %d MB\n", tiles / 32);
        run<0>("bulk_reduce", acc, 148, 400, 2);
        run<1>("bulk_store", acc, 148, 400, 2);
        run<2>("red.v4", acc, 148, 400, 1);
    }
    cudaFree(acc);
    return 0;
}
