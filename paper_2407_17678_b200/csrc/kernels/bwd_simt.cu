// S2-Attention backward, reference-precision path (fp32 arithmetic, FFMA).
//
// Serves the shapes the tcgen05 backward does not tile: S2_DTYPE_F32 (BASELINE
// cfg1's precision, parity at 1e-4) and bf16 with head_dim not in {64, 128} or
// block_size % 16 != 0, for head_dim <= 128.  The gradient is the one the oracle
// restates (oracle/s2_oracle.c: s2o_attn_bwd) of the forward's admitted set
// (/root/reference/proj/src/reference.cpp:28-36: the row block's CSR blocks, keys
// <= the query position):
//   P = exp(scale q.k - lse), Delta_i = dO_i . O_i, dS = P (dO.v - Delta),
//   dQ = scale sum_j dS_ij k_j, dK = scale sum_i dS_ij q_i, dV = sum_i P_ij dO_i.
// Three kernels, all in fixed visit orders with no atomics (deterministic):
//   s2_bwd_simt_prep     Delta per row (one warp per row)
//   s2_bwd_dq_tile       64 query rows x one query head per CTA, walking the row
//                        block's CSR list (as the forward tile kernel does)
//   s2_bwd_dkv_tile      64 keys x one kv head per CTA, walking the key block's CSC
//                        list over every query head of the GQA group
// The tile kernels use the forward tile kernel's 16 x 16 thread grid with 4 x 4
// register blocks; operands of the score products are staged transposed
// ([x][64], float4 reads), operands of the accumulating products row-major.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdint.h>

#include <type_traits>

#include "sm100_ptx.cuh"

namespace s2dev {
namespace bsimt {

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T>
__device__ __forceinline__ T cvt(float x);
template <>
__device__ __forceinline__ float cvt<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

struct Params {
    const int* bh_list;      // [num_bh] data index of each query head (slot = unit * hpg + j)
    const int* head_of;      // [num_bh] layout head
    const int* row_ptr;      // [H][B+1] CSR
    const int* col_idx;
    const int64_t* col_off;  // [H]
    const int* col_ptr;      // [H][B+1] CSC (key block -> query blocks)
    const int* row_idx;
    const int64_t* row_off;  // [H]
    const float* lse;        // [bh][N], natural log (the forward's)
    float* delta;            // [num_bh][Npad] workspace
    int num_bh, N, Npad, D, S, B, hpg;
    float scale;
};

// stage rows [row0, row0 + n) of a [N][D] head into smem, transposed ([x][64],
// zero past n / D) and/or row-major ([64][DT])
template <typename T, int DT>
__device__ __forceinline__ void stage_t(float* dst, const T* src, int row0, int n, int D) {
    for (int e = threadIdx.x; e < 64 * DT; e += 256) {
        const int c = e & 63, x = e >> 6;
        dst[x * 64 + c] = (c < n && x < D) ? ld(src + static_cast<size_t>(row0 + c) * D + x) : 0.f;
    }
}
template <typename T, int DT>
__device__ __forceinline__ void stage_r(float* dst, const T* src, int row0, int n, int D) {
    for (int e = threadIdx.x; e < 64 * DT; e += 256) {
        const int x = e % DT, c = e / DT;
        dst[c * DT + x] = (c < n && x < D) ? ld(src + static_cast<size_t>(row0 + c) * D + x) : 0.f;
    }
}

// Delta_i = sum_x dO_ix O_ix; 0 for rows without an admitted key (lse -inf, O NaN)
template <typename T>
__global__ void __launch_bounds__(256) s2_bwd_simt_prep(const T* __restrict__ out, const T* __restrict__ dout,
                                                        const Params p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // flat 1-D grid (no 65535 cap on batch x heads)
    const int row = static_cast<int>(blockIdx.x / p.num_bh) * 8 + warp;
    const int slot = static_cast<int>(blockIdx.x % p.num_bh);
    if (row >= p.N) return;
    const int bh = p.bh_list[slot];
    const size_t base = (static_cast<size_t>(bh) * p.N + row) * p.D;
    float acc = 0.f;
    for (int x = lane; x < p.D; x += 32) acc = fmaf(ld(dout + base + x), ld(out + base + x), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        const bool live = p.lse[static_cast<size_t>(bh) * p.N + row] != -INFINITY;
        p.delta[static_cast<size_t>(slot) * p.Npad + row] = live ? acc : 0.f;
    }
}

// Cluster reduction of per-thread accumulators (the SPLIT > 1 kernels): ranks > 0
// park theirs in thread-private shared-memory slots, rank 0 adds them rank by rank
// (a fixed order: deterministic).  Returns whether this CTA stores the result.
template <int SPLIT, int CW>
__device__ __forceinline__ bool cluster_sum(float (&a)[4][CW], float (&b)[4][CW], float* sm, bool two) {
    if (SPLIT == 1) return true;
    const int crank = static_cast<int>(blockIdx.x % SPLIT);
    __syncthreads();  // the staging buffers are free
    float* park = sm + static_cast<size_t>(threadIdx.x) * (8 * CW);
    if (crank != 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                park[i * CW + j] = a[i][j];
                if (two) park[4 * CW + i * CW + j] = b[i][j];
            }
    }
    s2dev::cluster_sync();
    if (crank == 0) {
        for (int rr = 1; rr < SPLIT; ++rr) {
            const uint32_t remote = s2dev::mapa_shared(s2dev::smem_u32(park), rr);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    float x, y = 0.f;
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(remote + 4u * (i * CW + j)));
                    if (two)
                        asm volatile("ld.shared::cluster.f32 %0, [%1];"
                                     : "=f"(y)
                                     : "r"(remote + 4u * (4 * CW + i * CW + j)));
                    a[i][j] += x;
                    b[i][j] += y;
                }
        }
    }
    s2dev::cluster_sync();  // the parked slots outlive rank 0's reads
    return crank == 0;
}

// dQ: one CTA = 64 query rows (a 64-row sub-tile of one query block) x one query
// head.  SPLIT > 1: a cluster shares the tile, rank r taking key chunks with
// (chunk index % SPLIT) == r, summed into rank 0 by cluster_sum.
template <typename T, int DT, int SPLIT>
__global__ void __launch_bounds__(256) s2_bwd_dq_tile(const T* __restrict__ q, const T* __restrict__ k,
                                                      const T* __restrict__ v, const T* __restrict__ dout,
                                                      T* __restrict__ dq, const Params p) {
    constexpr int CW = DT / 16;
    extern __shared__ __align__(16) float sm[];
    float* Qt = sm;              // [DT][64]
    float* dOt = Qt + DT * 64;   // [DT][64]
    float* Kt = dOt + DT * 64;   // [DT][64]
    float* Vt = Kt + DT * 64;    // [DT][64]
    float* Ks = Vt + DT * 64;    // [64][DT]
    float* dSs = Ks + 64 * DT;   // [64][68]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = p.N, D = p.D, S = p.S;
    const int nsub = (S + 63) >> 6;
    // flat 1-D grid (no 65535 cap on batch x heads): late (long-row) query blocks first
    const int crank = SPLIT > 1 ? static_cast<int>(blockIdx.x % SPLIT) : 0;
    const int cid = static_cast<int>(blockIdx.x / SPLIT);
    const int xb = p.B * nsub - 1 - cid / p.num_bh;
    const int qb = xb / nsub, sub = xb - qb * nsub;
    const int slot = cid % p.num_bh;
    const int bh = p.bh_list[slot], head = p.head_of[slot], kvbh = bh / p.hpg;
    const int r0 = qb * S + sub * 64;
    const int r_end = min(min(qb * S + S, N), r0 + 64);
    if (r0 >= r_end) return;  // (uniform across the cluster)
    const T* Q = q + static_cast<size_t>(bh) * N * D;
    const T* dO = dout + static_cast<size_t>(bh) * N * D;
    const T* K = k + static_cast<size_t>(kvbh) * N * D;
    const T* V = v + static_cast<size_t>(kvbh) * N * D;
    const int* rp = p.row_ptr + static_cast<size_t>(head) * (p.B + 1);
    const int* ci = p.col_idx + p.col_off[head];

    stage_t<T, DT>(Qt, Q, r0, r_end - r0, D);
    stage_t<T, DT>(dOt, dO, r0, r_end - r0, D);
    // P = exp2(scale log2e s - lse log2e); rows past the tile or without an admitted
    // key get lse2 = +inf (P = 0) and Delta = 0
    float lse2[4], dl[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = r0 + 4 * ty + i;
        const float l = row < r_end ? p.lse[static_cast<size_t>(bh) * N + row] : -INFINITY;
        lse2[i] = l == -INFINITY ? INFINITY : l * 1.4426950408889634f;
        dl[i] = row < r_end ? p.delta[static_cast<size_t>(slot) * p.Npad + row] : 0.f;
    }
    const float sl2 = p.scale * 1.4426950408889634f;
    float acc[4][CW];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CW; ++j) acc[i][j] = 0.f;
    const int row_last = r_end - 1;
    int kc = 0;  // key chunk index over the walk (SPLIT: this rank's share)
    for (int ptr = rp[qb]; ptr < rp[qb + 1]; ++ptr) {
        const int kb0 = ci[ptr] * S;
        const int kb_end = min(min(kb0 + S, N), row_last + 1);
        for (int k0 = kb0; k0 < kb_end; k0 += 64) {
            if (SPLIT > 1 && (kc++ % SPLIT) != crank) continue;
            const int nk = min(64, kb_end - k0);
            __syncthreads();  // the previous chunk's reads are done
            stage_t<T, DT>(Kt, K, k0, nk, D);
            stage_t<T, DT>(Vt, V, k0, nk, D);
            stage_r<T, DT>(Ks, K, k0, nk, D);
            __syncthreads();
            float s[4][4], dp[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) s[i][j] = dp[i][j] = 0.f;
#pragma unroll 2
            for (int x = 0; x < D; ++x) {
                const float4 a = *reinterpret_cast<const float4*>(Qt + x * 64 + 4 * ty);
                const float4 b = *reinterpret_cast<const float4*>(Kt + x * 64 + 4 * tx);
                const float4 c = *reinterpret_cast<const float4*>(dOt + x * 64 + 4 * ty);
                const float4 d = *reinterpret_cast<const float4*>(Vt + x * 64 + 4 * tx);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
                const float cv[4] = {c.x, c.y, c.z, c.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        s[i][j] = fmaf(av[i], bv[j], s[i][j]);
                        dp[i][j] = fmaf(cv[i], dv[j], dp[i][j]);
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = r0 + 4 * ty + i;
                float ds[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int key = k0 + 4 * tx + j;
                    const bool ok = 4 * tx + j < nk && key <= row;
                    const float pr = ok ? exp2f(fmaf(s[i][j], sl2, -lse2[i])) : 0.f;
                    ds[j] = pr * (dp[i][j] - dl[i]);
                }
                *reinterpret_cast<float4*>(dSs + (4 * ty + i) * 68 + 4 * tx) = make_float4(ds[0], ds[1], ds[2], ds[3]);
            }
            __syncthreads();
#pragma unroll 2
            for (int c = 0; c < nk; ++c) {
                float dv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) dv[i] = dSs[(4 * ty + i) * 68 + c];
#pragma unroll
                for (int j4 = 0; j4 < CW; j4 += 4) {
                    const float4 w = *reinterpret_cast<const float4*>(Ks + c * DT + tx * CW + j4);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        acc[i][j4 + 0] = fmaf(dv[i], w.x, acc[i][j4 + 0]);
                        acc[i][j4 + 1] = fmaf(dv[i], w.y, acc[i][j4 + 1]);
                        acc[i][j4 + 2] = fmaf(dv[i], w.z, acc[i][j4 + 2]);
                        acc[i][j4 + 3] = fmaf(dv[i], w.w, acc[i][j4 + 3]);
                    }
                }
            }
        }
    }
    if (!cluster_sum<SPLIT, CW>(acc, acc, sm, false)) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = r0 + 4 * ty + i;
        if (row >= r_end) continue;
        T* o = dq + static_cast<size_t>(bh) * N * D + static_cast<size_t>(row) * D;
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            const int x = tx * CW + j;
            if (x < D) o[x] = cvt<T>(acc[i][j] * p.scale);
        }
    }
}

// dK / dV: one CTA = 64 keys (a 64-key sub-tile of one key block) x one kv head; it
// walks, for every query head of the group in order, the key block's CSC list
// (ascending query blocks) in 64-row query chunks.  SPLIT = 2: a cluster of two CTAs
// shares the tile -- CTA rank r takes the chunks with (chunk index % 2) == r -- and
// rank 0 adds rank 1's accumulators (read through distributed shared memory) to its
// own before the store: a fixed order, so still deterministic.  A stripe key block,
// which every later query block attends, has a list up to B long while a local-only
// one has a few entries; splitting halves the longest CTA.
template <typename T, int DT, int SPLIT>
__global__ void __launch_bounds__(256) s2_bwd_dkv_tile(const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, const T* __restrict__ dout,
                                                       T* __restrict__ dk, T* __restrict__ dv, const Params p) {
    constexpr int CW = DT / 16;
    extern __shared__ __align__(16) float sm[];
    float* Kt = sm;              // [DT][64]
    float* Vt = Kt + DT * 64;    // [DT][64]
    float* Qt = Vt + DT * 64;    // [DT][64]
    float* dOt = Qt + DT * 64;   // [DT][64]
    float* Qs = dOt + DT * 64;   // [64][DT]
    float* dOs = Qs + 64 * DT;   // [64][DT]
    float* Ps = dOs + 64 * DT;   // [64][68]
    float* dSs = Ps + 64 * 68;   // [64][68]
    float* Ls = dSs + 64 * 68;   // [64] lse2 of the chunk's rows
    float* Ds = Ls + 64;         // [64] Delta of the chunk's rows
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = p.N, D = p.D, S = p.S;
    const int nsub = (S + 63) >> 6;
    // flat 1-D grid: early key blocks (the longest transposed lists) first
    const int nunits = p.num_bh / p.hpg;
    const int crank = SPLIT > 1 ? static_cast<int>(blockIdx.x % SPLIT) : 0;  // cluster rank (1-D clusters)
    const int cid = static_cast<int>(blockIdx.x / SPLIT);
    const int xb = cid / nunits;
    const int kb = xb / nsub, sub = xb - kb * nsub;
    const int unit = cid % nunits;
    const int k0 = kb * S + sub * 64;
    const int k_end = min(min(kb * S + S, N), k0 + 64);
    if (k0 >= k_end) return;  // (uniform across the cluster: both ranks share the tile)
    const int kvbh = p.bh_list[unit * p.hpg] / p.hpg;
    const T* K = k + static_cast<size_t>(kvbh) * N * D;
    const T* V = v + static_cast<size_t>(kvbh) * N * D;
    stage_t<T, DT>(Kt, K, k0, k_end - k0, D);
    stage_t<T, DT>(Vt, V, k0, k_end - k0, D);
    const float sl2 = p.scale * 1.4426950408889634f;
    float ak[4][CW], av[4][CW];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CW; ++j) ak[i][j] = av[i][j] = 0.f;
    int qc = 0;  // query chunk index over the whole walk (SPLIT: this rank's share)
    for (int hj = 0; hj < p.hpg; ++hj) {
        const int slot = unit * p.hpg + hj;
        const int bh = p.bh_list[slot], head = p.head_of[slot];
        const T* Q = q + static_cast<size_t>(bh) * N * D;
        const T* dO = dout + static_cast<size_t>(bh) * N * D;
        const int* cp = p.col_ptr + static_cast<size_t>(head) * (p.B + 1);
        const int* ri = p.row_idx + p.row_off[head];
        for (int ptr = cp[kb]; ptr < cp[kb + 1]; ++ptr) {
            const int qb = ri[ptr];
            const int q_end = min(qb * S + S, N);
            // rows before the tile's first key admit none of its keys
            for (int r0 = max(qb * S, k0); r0 < q_end; r0 += 64) {
                if (SPLIT > 1 && (qc++ % SPLIT) != crank) continue;
                const int nq = min(64, q_end - r0);
                __syncthreads();  // the previous chunk's reads are done
                stage_t<T, DT>(Qt, Q, r0, nq, D);
                stage_t<T, DT>(dOt, dO, r0, nq, D);
                stage_r<T, DT>(Qs, Q, r0, nq, D);
                stage_r<T, DT>(dOs, dO, r0, nq, D);
                if (tid < 64) {
                    const int row = r0 + tid;
                    const float l = tid < nq ? p.lse[static_cast<size_t>(bh) * N + row] : -INFINITY;
                    Ls[tid] = l == -INFINITY ? INFINITY : l * 1.4426950408889634f;
                    Ds[tid] = tid < nq ? p.delta[static_cast<size_t>(slot) * p.Npad + row] : 0.f;
                }
                __syncthreads();
                float s[4][4], dp[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) s[i][j] = dp[i][j] = 0.f;
#pragma unroll 2
                for (int x = 0; x < D; ++x) {
                    const float4 a = *reinterpret_cast<const float4*>(Kt + x * 64 + 4 * ty);
                    const float4 b = *reinterpret_cast<const float4*>(Qt + x * 64 + 4 * tx);
                    const float4 c = *reinterpret_cast<const float4*>(Vt + x * 64 + 4 * ty);
                    const float4 d = *reinterpret_cast<const float4*>(dOt + x * 64 + 4 * tx);
                    const float avv[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
                    const float cv[4] = {c.x, c.y, c.z, c.w}, dvv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            s[i][j] = fmaf(avv[i], bv[j], s[i][j]);
                            dp[i][j] = fmaf(cv[i], dvv[j], dp[i][j]);
                        }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // S^T row: key 4ty+i; columns: query rows 4tx+j
                    const int key = k0 + 4 * ty + i;
                    float pr[4], ds[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c = 4 * tx + j;
                        const bool ok = key < k_end && c < nq && r0 + c >= key;
                        pr[j] = ok ? exp2f(fmaf(s[i][j], sl2, -Ls[c])) : 0.f;
                        ds[j] = pr[j] * (dp[i][j] - Ds[c]);
                    }
                    *reinterpret_cast<float4*>(Ps + (4 * ty + i) * 68 + 4 * tx) = make_float4(pr[0], pr[1], pr[2], pr[3]);
                    *reinterpret_cast<float4*>(dSs + (4 * ty + i) * 68 + 4 * tx) = make_float4(ds[0], ds[1], ds[2], ds[3]);
                }
                __syncthreads();
#pragma unroll 2
                for (int c = 0; c < nq; ++c) {
                    float pv[4], dsv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        pv[i] = Ps[(4 * ty + i) * 68 + c];
                        dsv[i] = dSs[(4 * ty + i) * 68 + c];
                    }
#pragma unroll
                    for (int j4 = 0; j4 < CW; j4 += 4) {
                        const float4 wo = *reinterpret_cast<const float4*>(dOs + c * DT + tx * CW + j4);
                        const float4 wq = *reinterpret_cast<const float4*>(Qs + c * DT + tx * CW + j4);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            av[i][j4 + 0] = fmaf(pv[i], wo.x, av[i][j4 + 0]);
                            av[i][j4 + 1] = fmaf(pv[i], wo.y, av[i][j4 + 1]);
                            av[i][j4 + 2] = fmaf(pv[i], wo.z, av[i][j4 + 2]);
                            av[i][j4 + 3] = fmaf(pv[i], wo.w, av[i][j4 + 3]);
                            ak[i][j4 + 0] = fmaf(dsv[i], wq.x, ak[i][j4 + 0]);
                            ak[i][j4 + 1] = fmaf(dsv[i], wq.y, ak[i][j4 + 1]);
                            ak[i][j4 + 2] = fmaf(dsv[i], wq.z, ak[i][j4 + 2]);
                            ak[i][j4 + 3] = fmaf(dsv[i], wq.w, ak[i][j4 + 3]);
                        }
                    }
                }
            }
        }
    }
    if (!cluster_sum<SPLIT, CW>(ak, av, sm, true)) return;
    // every key of the tile is written: 0 for keys no query attends
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int key = k0 + 4 * ty + i;
        if (key >= k_end) continue;
        const size_t o = (static_cast<size_t>(kvbh) * N + key) * D;
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            const int x = tx * CW + j;
            if (x < D) {
                dk[o + x] = cvt<T>(ak[i][j] * p.scale);
                dv[o + x] = cvt<T>(av[i][j]);
            }
        }
    }
}

}  // namespace bsimt
}  // namespace s2dev

// query-chunk split of the dK/dV tiles over a cluster (1: none).  A/B at cfg1's shape
// (fp32, N=2048, H=8, D=64): backward 0.684 ms (1), 0.454 (2), 0.600 (4), 1.43 (8);
// N=8192 D=128: 6.54 / 5.33 / 7.00 / 13.9 ms
#ifndef S2_SIMT_DKV_SPLIT
#define S2_SIMT_DKV_SPLIT 2
#endif
static constexpr int kDkvSplit = S2_SIMT_DKV_SPLIT;
// dQ: the same split over key chunks does not pay (cfg1 shape 0.462 vs 0.453 ms,
// N=8192 D=128 5.64 vs 5.33 ms): a query block's list is at most local + stripe long
#ifndef S2_SIMT_DQ_SPLIT
#define S2_SIMT_DQ_SPLIT 1
#endif
static constexpr int kDqSplit = S2_SIMT_DQ_SPLIT;

// One backward over the plan's CSR / CSC (device arrays as s2_launch_fwd_simt's):
// prep, dQ, dK/dV on `stream`.  bh_list / head_of: num_bh = num_units * hpg slots,
// unit-major.  delta: [num_bh][Npad] floats of workspace.  head_dim <= 128.
cudaError_t s2_launch_bwd_simt(bool bf16, const void* q, const void* k, const void* v, const void* out,
                               const float* lse, const void* dout, void* dq, void* dk, void* dv,
                               const int* bh_list, const int* head_of, int num_bh, const int* row_ptr,
                               const int* col_idx, const int64_t* col_off, const int* col_ptr,
                               const int* row_idx, const int64_t* row_off, float* delta, int N, int Npad,
                               int D, int S, int B, int hpg, float scale, cudaStream_t stream) {
    using namespace s2dev::bsimt;
    if (num_bh == 0 || N == 0) return cudaSuccess;
    if (D > 128) return cudaErrorInvalidValue;
    const Params p{bh_list, head_of, row_ptr, col_idx, col_off, col_ptr, row_idx, row_off, lse, delta,
                   num_bh, N, Npad, D, S, B, hpg, scale};
    const int nsub = (S + 63) / 64;
    auto run = [&](auto tag, auto dtag) -> cudaError_t {
        constexpr int DT = decltype(dtag)::value;
        using T = typename decltype(tag)::type;
        const T* tq = static_cast<const T*>(q);
        const T* tk = static_cast<const T*>(k);
        const T* tv = static_cast<const T*>(v);
        const T* to = static_cast<const T*>(out);
        const T* tdo = static_cast<const T*>(dout);
        s2_bwd_simt_prep<T><<<dim3(static_cast<unsigned>((N + 7) / 8) * num_bh), 256, 0, stream>>>(to, tdo, p);
        const int smem_q = (5 * DT * 64 + 64 * 68) * 4;
        const int smem_kv = (6 * DT * 64 + 2 * 64 * 68 + 128) * 4;
        cudaError_t e;
        auto dqk = s2_bwd_dq_tile<T, DT, kDqSplit>;
        auto dkv = s2_bwd_dkv_tile<T, DT, kDkvSplit>;
        if ((e = cudaFuncSetAttribute(dqk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(dkv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv)) != cudaSuccess)
            return e;
        // both tile kernels in 1-D clusters of kDqSplit / kDkvSplit CTAs
        auto cluster_launch = [&](auto kern, unsigned ctas, int split, int smem, auto... args) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctas * split);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = split;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, kern, args...);
        };
        if ((e = cluster_launch(dqk, static_cast<unsigned>(B) * nsub * num_bh, kDqSplit, smem_q, tq, tk, tv, tdo,
                                static_cast<T*>(dq), p)) != cudaSuccess ||
            (e = cluster_launch(dkv, static_cast<unsigned>(B) * nsub * (num_bh / hpg), kDkvSplit, smem_kv, tq, tk, tv,
                                tdo, static_cast<T*>(dk), static_cast<T*>(dv), p)) != cudaSuccess)
            return e;
        return cudaGetLastError();
    };
    struct F32 { using type = float; };
    struct BF16 { using type = __nv_bfloat16; };
    if (bf16)
        return D <= 64 ? run(BF16{}, std::integral_constant<int, 64>{}) : run(BF16{}, std::integral_constant<int, 128>{});
    return D <= 64 ? run(F32{}, std::integral_constant<int, 64>{}) : run(F32{}, std::integral_constant<int, 128>{});
}
