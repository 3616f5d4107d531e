// S2-Attention forward, reference-precision path (fp32 storage, fp32 FFMA).
//
// Serves S2_DTYPE_F32 (cfg1 of BASELINE.json: fp32 parity at 1e-4, which TF32
// tensor cores cannot meet — SURVEY §7 hard part 3) and any block_size /
// head_dim the tcgen05 kernel does not tile (block_size % 16 != 0, D not in
// {64,128}).  Same walk as process_query_block (attention.cpp:26-98): per
// query row, ascending CSR row blocks, online softmax; one warp per row, lanes
// split keys for the scores and head_dim for the output accumulator.
// Unattended keys are never read, the visit order is fixed, and no value is
// reduced across warps, so results are deterministic and exact under the
// reference's exactness tests (test_attention.cpp:196-257).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <type_traits>
#include <stdint.h>

namespace s2dev {

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

struct SimtParams {
    const int* bh_list;   // [num_bh] data index of each query head processed
    const int* head_of;   // [num_bh] layout head
    const int* row_ptr;   // [H][B+1]
    const int* col_idx;   // concatenated
    const int64_t* col_off;  // [H]
    int num_bh, N, D, S, B, hpg;
    float scale;
};

// head_dim <= 32 * DPL: instantiated for DPL 8 / 16 / 64 (head_dim <= 256 / 512 / 2048)
constexpr int kMaxHeadDim = 2048;

template <typename T, int DPL>
__global__ void __launch_bounds__(128) s2_fwd_simt_kernel(const T* __restrict__ q,
                                                          const T* __restrict__ k,
                                                          const T* __restrict__ v,
                                                          T* __restrict__ out,
                                                          float* __restrict__ lse,
                                                          const SimtParams p) {
    extern __shared__ float sq[];  // [4 warps][D]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qb = blockIdx.x;
    const int slot = blockIdx.y;
    const int bh = p.bh_list[slot];
    const int head = p.head_of[slot];
    const int kvbh = bh / p.hpg;
    const int N = p.N, D = p.D, S = p.S;
    const T* Q = q + static_cast<size_t>(bh) * N * D;
    const T* K = k + static_cast<size_t>(kvbh) * N * D;
    const T* V = v + static_cast<size_t>(kvbh) * N * D;
    const int* rp = p.row_ptr + static_cast<size_t>(head) * (p.B + 1);
    const int* ci = p.col_idx + p.col_off[head];
    float* qs = sq + warp * D;
    const int q_begin = qb * S;
    const int q_end = min(q_begin + S, N);
    const int nd = (D + 31) / 32;

    for (int i = q_begin + warp; i < q_end; i += 4) {
        for (int x = lane; x < D; x += 32) qs[x] = to_f(Q[static_cast<size_t>(i) * D + x]);
        __syncwarp();
        float m = -INFINITY, l = 0.f;
        float acc[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
        for (int ptr = rp[qb]; ptr < rp[qb + 1]; ++ptr) {
            const int k_begin = ci[ptr] * S;
            const int k_end = min(min(k_begin + S, N), i + 1);
            for (int kc = k_begin; kc < k_end; kc += 32) {
                const int key = kc + lane;
                float s = -INFINITY;
                if (key < k_end) {
                    const T* kr = K + static_cast<size_t>(key) * D;
                    float dot = 0.f;
                    for (int x = 0; x < D; ++x) dot = fmaf(qs[x], to_f(kr[x]), dot);
                    s = dot * p.scale;
                }
                float cm = s;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
                const float m_new = fmaxf(m, cm);
                const float alpha = expf(m - m_new);
                const float pv = (key < k_end) ? expf(s - m_new) : 0.f;
                float ps = pv;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
                l = l * alpha + ps;
#pragma unroll
                for (int e = 0; e < DPL; ++e) acc[e] *= alpha;
                const int nk = min(32, k_end - kc);
                for (int kk = 0; kk < nk; ++kk) {
                    const float w = __shfl_sync(0xffffffffu, pv, kk);
                    const T* vr = V + static_cast<size_t>(kc + kk) * D;
#pragma unroll
                    for (int e = 0; e < DPL; ++e) {
                        const int x = lane + 32 * e;
                        if (e < nd && x < D) acc[e] = fmaf(w, to_f(vr[x]), acc[e]);
                    }
                }
                m = m_new;
            }
        }
        const float inv = 1.0f / l;
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
            const int x = lane + 32 * e;
            if (e < nd && x < D) out[static_cast<size_t>(bh) * N * D + static_cast<size_t>(i) * D + x] = from_f<T>(acc[e] * inv);
        }
        if (lane == 0) lse[static_cast<size_t>(bh) * N + i] = m + logf(l);
        __syncwarp();
    }
}

}  // namespace s2dev

cudaError_t s2_launch_fwd_simt(bool bf16, const void* q, const void* k, const void* v, void* out,
                               float* lse, const int* bh_list, const int* head_of, int num_bh,
                               const int* row_ptr, const int* col_idx, const int64_t* col_off,
                               int N, int D, int S, int B, int hpg, float scale,
                               cudaStream_t stream) {
    if (num_bh == 0) return cudaSuccess;
    if (D > s2dev::kMaxHeadDim) return cudaErrorInvalidValue;
    s2dev::SimtParams p{bh_list, head_of, row_ptr, col_idx, col_off, num_bh, N, D, S, B, hpg, scale};
    dim3 grid(B, num_bh);
    const size_t smem = 4 * D * sizeof(float);  // <= 32 KB
    auto launch = [&](auto tag) {
        constexpr int DPL = decltype(tag)::value;
        if (bf16)
            s2dev::s2_fwd_simt_kernel<__nv_bfloat16, DPL><<<grid, 128, smem, stream>>>(
                static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
                static_cast<const __nv_bfloat16*>(v), static_cast<__nv_bfloat16*>(out), lse, p);
        else
            s2dev::s2_fwd_simt_kernel<float, DPL><<<grid, 128, smem, stream>>>(
                static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v),
                static_cast<float*>(out), lse, p);
    };
    if (D <= 256)
        launch(std::integral_constant<int, 8>{});
    else if (D <= 512)
        launch(std::integral_constant<int, 16>{});
    else
        launch(std::integral_constant<int, 64>{});
    return cudaGetLastError();
}
