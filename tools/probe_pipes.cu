// Per-SM throughput of the elementwise instructions of the attention kernels
// (tools only): ex2.approx.f32 (MUFU), cvt.rn.bf16x2.f32 (F2FP pack), the
// integer round-and-pack alternative, FFMA2.  16 warps on one SM, independent
// chains; reports results per SM-cycle.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int OP>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, long long* cyc) {
    float a[8];
    uint32_t u[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 1e-3f + j; u[j] = threadIdx.x + j; }
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
            if (OP == 1) {  // pack two floats
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[j]), "f"(a[(j + 1) & 7]));
                u[j] ^= r;
                a[j] = __uint_as_float(__float_as_uint(a[j]) + 1u);
            }
            if (OP == 2) {  // integer round-to-nearest pack: 2 IADD + 1 PRMT
                const uint32_t x0 = __float_as_uint(a[j]) + 0x8000u, x1 = __float_as_uint(a[(j + 1) & 7]) + 0x8000u;
                uint32_t r;
                asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(x0), "r"(x1));
                u[j] ^= r;
                a[j] = __uint_as_float(__float_as_uint(a[j]) + 1u);
            }
            if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[j]));
            if (OP == 4) {  // cvt.rn.bf16x2 only (no extra ALU)
                uint32_t r;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[j]), "f"(a[(j + 3) & 7]));
                u[j] += r;
            }
        }
    }
    const long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j] + u[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 148 * 512 * 4);
    cudaMalloc(&c, 148 * 8);
    const char* names[] = {"ex2.approx.f32 (MUFU)", "cvt.rn.bf16x2 + iadd", "iadd x2 + prmt pack + iadd", "ffma",
                           "cvt.rn.bf16x2.f32 + iadd"};
    const int iters = 4096;
    for (int op = 0; op < 5; ++op) {
        for (int w : {8, 16}) {
            void (*kern)(float*, int, long long*) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
            kern<<<1, 32 * w>>>(o, iters, c);
            cudaDeviceSynchronize();
            long long h;
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("%-30s %2d warps: %6.2f ops per SM-cycle\n", names[op], w, double(iters) * 8 * 32 * w / h);
        }
    }
    return 0;
}
