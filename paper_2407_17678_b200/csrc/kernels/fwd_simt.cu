// S2-Attention forward, reference-precision path (fp32 arithmetic, FFMA).
//
// Serves S2_DTYPE_F32 (cfg1 of BASELINE.json: fp32 parity at 1e-4, which TF32
// tensor cores cannot meet -- SURVEY §7 hard part 3) and the bf16 shapes the
// tcgen05 kernels do not tile (block_size % 16 != 0, head_dim not in {64, 128};
// their backward is S2_ERR_UNSUPPORTED).  Two kernels, both walking
// process_query_block (attention.cpp:26-98): ascending CSR row blocks, online
// softmax.
//   s2_fwd_tile_kernel   head_dim <= 256: 64-row query tiles, K / V chunks staged
//                        in shared memory, 4x4 register blocking (below)
//   s2_fwd_simt_kernel   head_dim <= 2048: one warp per row, lanes split keys for
//                        the scores and head_dim for the output accumulator
// Unattended keys are never read, the visit order is fixed, and no value is
// reduced across CTAs, so results are deterministic and exact under the
// reference's exactness tests (test_attention.cpp:196-257).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
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
    // flat 1-D grid (no 65535 cap on batch x heads): late (long-row) blocks first
    const int qb = p.B - 1 - static_cast<int>(blockIdx.x / p.num_bh);
    const int slot = static_cast<int>(blockIdx.x % p.num_bh);
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


// ---------------------------------------------------------------------------
// Tiled reference-precision forward (fp32 FFMA from shared memory), D <= 256.
// One CTA = 64 query rows of one query block (blocks larger than 64 rows are
// split into 64-row sub-tiles) x one query head; 256 threads as a 16 x 16 grid,
// thread (ty, tx) owns rows 4ty..4ty+3 and, per 64-key chunk, keys 4tx..4tx+3
// of S and output columns [tx DT/16, (tx+1) DT/16).  Q and each K chunk are
// staged transposed ([x][row], coalesced loads, conflict-free float4 reads), V
// row-major.  Per chunk the walk is process_query_block's
// (/root/reference/proj/src/attention.cpp:39-84): scores scaled once, the
// block max, alpha = exp(m - m_new), p = exp(s - m_new), l = alpha l + sum p,
// acc = alpha acc + p V -- in fp32 where the reference accumulates in double
// (BASELINE cfg1 parity is 1e-4).  Unattended keys are never read and nothing
// is reduced across CTAs: deterministic, shard-isolated.
template <typename T, int DT>
__global__ void __launch_bounds__(256) s2_fwd_tile_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                          const T* __restrict__ v, T* __restrict__ out,
                                                          float* __restrict__ lse, const SimtParams p) {
    constexpr int CW = DT / 16;  // output columns per thread
    extern __shared__ __align__(16) float sm[];
    float* Qt = sm;              // [DT][64]
    float* Kt = Qt + DT * 64;    // [DT][64]
    float* Vs = Kt + DT * 64;    // [64][DT]
    float* Ps = Vs + 64 * DT;    // [64][68]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = p.N, D = p.D, S = p.S;
    const int nsub = (S + 63) >> 6;
    // flat 1-D grid (no 65535 cap on batch x heads): late (long-row) query blocks first
    const int xb = p.B * nsub - 1 - static_cast<int>(blockIdx.x / p.num_bh);
    const int qb = xb / nsub, sub = xb - qb * nsub;
    const int slot = static_cast<int>(blockIdx.x % p.num_bh);
    const int bh = p.bh_list[slot], head = p.head_of[slot], kvbh = bh / p.hpg;
    const int r0 = qb * S + sub * 64;
    const int r_end = min(min(qb * S + S, N), r0 + 64);
    if (r0 >= r_end) return;
    const T* Q = q + static_cast<size_t>(bh) * N * D;
    const T* K = k + static_cast<size_t>(kvbh) * N * D;
    const T* V = v + static_cast<size_t>(kvbh) * N * D;
    const int* rp = p.row_ptr + static_cast<size_t>(head) * (p.B + 1);
    const int* ci = p.col_idx + p.col_off[head];

    // Q tile, transposed; rows past the tile and columns past D are zero
    for (int e = tid; e < 64 * DT; e += 256) {
        const int r = e & 63, x = e >> 6;
        Qt[x * 64 + r] = (r0 + r < r_end && x < D) ? to_f(Q[static_cast<size_t>(r0 + r) * D + x]) : 0.f;
    }
    float m[4], l[4], o[4][CW];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int j = 0; j < CW; ++j) o[i][j] = 0.f;
    }
    const int row_last = r_end - 1;
    for (int ptr = rp[qb]; ptr < rp[qb + 1]; ++ptr) {
        const int kb0 = ci[ptr] * S;
        const int kb_end = min(min(kb0 + S, N), row_last + 1);  // in-block causality bounds the chunk
        for (int k0 = kb0; k0 < kb_end; k0 += 64) {
            const int nk = min(64, kb_end - k0);
            __syncthreads();  // the previous chunk's K / V / P reads are done
            for (int e = tid; e < 64 * DT; e += 256) {
                const int c = e & 63, x = e >> 6;
                Kt[x * 64 + c] = (c < nk && x < D) ? to_f(K[static_cast<size_t>(k0 + c) * D + x]) : 0.f;
            }
            for (int e = tid; e < 64 * DT; e += 256) {
                const int x = e % DT, c = e / DT;
                Vs[c * DT + x] = (c < nk && x < D) ? to_f(V[static_cast<size_t>(k0 + c) * D + x]) : 0.f;
            }
            __syncthreads();
            float s[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 4
            for (int x = 0; x < D; ++x) {
                const float4 a = *reinterpret_cast<const float4*>(Qt + x * 64 + 4 * ty);
                const float4 b = *reinterpret_cast<const float4*>(Kt + x * 64 + 4 * tx);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) s[i][j] = fmaf(av[i], bv[j], s[i][j]);
            }
            float alpha[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = r0 + 4 * ty + i;
                float bm = -INFINITY;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int key = k0 + 4 * tx + j;
                    s[i][j] = (4 * tx + j < nk && key <= row) ? s[i][j] * p.scale : -INFINITY;
                    bm = fmaxf(bm, s[i][j]);
                }
#pragma unroll
                for (int off = 1; off < 16; off <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
                const float m_new = fmaxf(m[i], bm);
                // a row with nothing admitted so far keeps m = -inf: alpha 1, p 0
                const float mb = m_new == -INFINITY ? 0.f : m_new;
                alpha[i] = m[i] == -INFINITY ? (m_new == -INFINITY ? 1.f : 0.f) : expf(m[i] - m_new);
                float bs = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    s[i][j] = expf(s[i][j] - mb);
                    bs += s[i][j];
                }
#pragma unroll
                for (int off = 1; off < 16; off <<= 1) bs += __shfl_xor_sync(0xffffffffu, bs, off);
                l[i] = alpha[i] * l[i] + bs;
                m[i] = m_new;
                *reinterpret_cast<float4*>(Ps + (4 * ty + i) * 68 + 4 * tx) = make_float4(s[i][0], s[i][1], s[i][2], s[i][3]);
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CW; ++j) o[i][j] *= alpha[i];
#pragma unroll 2
            for (int c = 0; c < nk; ++c) {
                float pv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) pv[i] = Ps[(4 * ty + i) * 68 + c];
#pragma unroll
                for (int j4 = 0; j4 < CW; j4 += 4) {
                    const float4 w = *reinterpret_cast<const float4*>(Vs + c * DT + tx * CW + j4);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        o[i][j4 + 0] = fmaf(pv[i], w.x, o[i][j4 + 0]);
                        o[i][j4 + 1] = fmaf(pv[i], w.y, o[i][j4 + 1]);
                        o[i][j4 + 2] = fmaf(pv[i], w.z, o[i][j4 + 2]);
                        o[i][j4 + 3] = fmaf(pv[i], w.w, o[i][j4 + 3]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = r0 + 4 * ty + i;
        if (row >= r_end) continue;
        const float inv = 1.0f / l[i];  // l = 0 (no admitted key): NaN, the reference's acc / l
        T* orow = out + static_cast<size_t>(bh) * N * D + static_cast<size_t>(row) * D;
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            const int x = tx * CW + j;
            if (x < D) orow[x] = from_f<T>(o[i][j] * inv);
        }
        if (tx == 0) lse[static_cast<size_t>(bh) * N + row] = m[i] + logf(l[i]);
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
    if (D <= 256 && std::getenv("S2_SIMT_ROWWISE") == nullptr) {
        // tiled kernel: 64-row sub-tiles of every query block
        const dim3 grid(static_cast<unsigned>(B) * ((S + 63) / 64) * num_bh);
        auto launch = [&](auto tag) {
            constexpr int DT = decltype(tag)::value;
            const size_t smem = (3 * DT * 64 + 64 * 68) * sizeof(float);
            auto go = [&](auto kern, auto* qq, auto* kk, auto* vv, auto* oo) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                kern<<<grid, 256, smem, stream>>>(qq, kk, vv, oo, lse, p);
            };
            if (bf16)
                go(s2dev::s2_fwd_tile_kernel<__nv_bfloat16, DT>, static_cast<const __nv_bfloat16*>(q),
                   static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
                   static_cast<__nv_bfloat16*>(out));
            else
                go(s2dev::s2_fwd_tile_kernel<float, DT>, static_cast<const float*>(q), static_cast<const float*>(k),
                   static_cast<const float*>(v), static_cast<float*>(out));
        };
        if (D <= 64)
            launch(std::integral_constant<int, 64>{});
        else if (D <= 128)
            launch(std::integral_constant<int, 128>{});
        else
            launch(std::integral_constant<int, 256>{});
        return cudaGetLastError();
    }
    // row-wise kernel: head_dim up to 2048 (S2_SIMT_ROWWISE=1 forces it for any D)
    const dim3 grid(static_cast<unsigned>(B) * num_bh);
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
