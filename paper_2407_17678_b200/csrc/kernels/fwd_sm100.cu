// S2-Attention forward, sm_100a: TMA-staged Q/K/V tiles, tcgen05.mma with
// fp32 accumulators in TMEM, online softmax with one thread per query row.
//
// Replaces the reference's streaming kernel process_query_block
// (/root/reference/proj/src/attention.cpp:26-98): a 128-row query tile walks
// only the 64-key chunks its rows attend (the union of two layout row
// blocks when block_size = 64), two chunks (gathered, need not be adjacent)
// per 128-key MMA tile.  Masked scores are -inf, so P = 0 exactly and no
// value row outside the shard ever contributes (test_attention.cpp:196-215).
// The visit order is fixed per tile and nothing is reduced across CTAs, so
// results are deterministic and independent of head position.
//
// Warp roles (256 threads, 1 CTA / SM):
//   warp 0      TMA producer (Q once, K/V chunk pairs into an NST-deep ring)
//   warp 1      MMA issuer: S_n = Q K_n^T (SS), O += P_{n-1} V_{n-1} (TS)
//   warp 2      TMEM allocator
//   warps 4..7  softmax (thread = query row = TMEM lane), lazy O rescale,
//               epilogue (O / l -> bf16, lse)
// TMEM columns: S double buffer [0,256), O [256, 256+D), P (bf16x2) double
// buffer [384, 512).
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {

struct FwdParams {
    const FwdItem* items;
    const int2* chunks;  // {chunk, mask}
    __nv_bfloat16* out;
    float* lse;
    int seq_len;
    int hpg;
    float scale_log2;
};

template <int D, int NST>
struct FwdSmem {
    static constexpr int kSub = D / 64;                  // 64-column swizzle subtiles
    static constexpr int kQBytes = kSub * 16384;         // 128 rows
    static constexpr int kKVBytes = kSub * 16384;        // 128 keys
    static constexpr int kStageBytes = 2 * kKVBytes;     // K + V
    static constexpr int kTotal = 1024 + kQBytes + NST * kStageBytes;
};

template <int D, int NST>
__global__ void __launch_bounds__(256, 1)
    s2_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
    using L = FwdSmem<D, NST>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q, bar_k[NST], bar_v[NST], bar_empty[NST];
    __shared__ uint64_t bar_s[2], bar_p[2], bar_pv[2];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const FwdItem item = p.items[blockIdx.x];
    const int cnt = item.chunk_cnt;
    const int T = (cnt + 1) >> 1;  // 128-key MMA tiles
    const int2* ch = p.chunks + item.chunk_off;
    const int kvbh = item.bh / p.hpg;

    const uint32_t sQ = smem_u32(smem);
    const uint32_t sKV = sQ + L::kQBytes;

    if (tid == 0) {
        mbar_init(smem_u32(&bar_q), 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_k[i]), 1);
            mbar_init(smem_u32(&bar_v[i]), 1);
            mbar_init(smem_u32(&bar_empty[i]), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_s[i]), 1);
            mbar_init(smem_u32(&bar_p[i]), 128);
            mbar_init(smem_u32(&bar_pv[i]), 1);
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc(smem_u32(&tmem_base_s), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tS = tmem, tO = tmem + 256, tP = tmem + 384;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const uint64_t keep = policy_evict_last();
            mbar_expect_tx(smem_u32(&bar_q), L::kQBytes);
            for (int s = 0; s < L::kSub; ++s)
                tma_load_3d(sQ + s * 16384, &tmQ, smem_u32(&bar_q), s * 64, item.qtile * 128,
                            item.bh);
            for (int n = 0; n < T; ++n) {
                const int st = n % NST;
                if (n >= NST) mbar_wait(smem_u32(&bar_empty[st]), ((n / NST) + 1) & 1);
                const int nc = (2 * n + 1 < cnt) ? 2 : 1;
                const uint32_t sK = sKV + st * L::kStageBytes;
                const uint32_t sV = sK + L::kKVBytes;
                mbar_expect_tx(smem_u32(&bar_k[st]), nc * L::kSub * 8192);
                for (int h = 0; h < nc; ++h) {
                    const int c = ch[2 * n + h].x;
                    for (int s = 0; s < L::kSub; ++s)
                        tma_load_3d_hint(sK + s * 16384 + h * 8192, &tmK, smem_u32(&bar_k[st]),
                                         s * 64, c * 64, kvbh, keep);
                }
                mbar_expect_tx(smem_u32(&bar_v[st]), nc * L::kSub * 8192);
                for (int h = 0; h < nc; ++h) {
                    const int c = ch[2 * n + h].x;
                    for (int s = 0; s < L::kSub; ++s)
                        tma_load_3d_hint(sV + s * 16384 + h * 8192, &tmV, smem_u32(&bar_v[st]),
                                         s * 64, c * 64, kvbh, keep);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t idS128 = umma_idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idS64 = umma_idesc_bf16(128, 64, 0, 0);
            constexpr uint32_t idO = umma_idesc_bf16(128, D, 0, 1);
            mbar_wait(smem_u32(&bar_q), 0);
            tc_fence_after();
            for (int n = 0; n <= T; ++n) {
                if (n < T) {
                    const int st = n % NST, b = n & 1;
                    const int nc = (2 * n + 1 < cnt) ? 2 : 1;
                    const uint32_t sK = sKV + st * L::kStageBytes;
                    mbar_wait(smem_u32(&bar_k[st]), (n / NST) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const int sub = kk >> 2, off = (kk & 3) * 32;
                        const uint64_t ad = umma_desc_sw128(sQ + sub * 16384 + off, 16, 1024);
                        const uint64_t bd = umma_desc_sw128(sK + sub * 16384 + off, 16, 1024);
                        mma_ss(tS + b * 128, ad, bd, nc == 2 ? idS128 : idS64, kk > 0);
                    }
                    mma_commit(smem_u32(&bar_s[b]));
                }
                if (n >= 1) {
                    const int m = n - 1, st = m % NST, b = m & 1;
                    const int nc = (2 * m + 1 < cnt) ? 2 : 1;
                    const uint32_t sV = sKV + st * L::kStageBytes + L::kKVBytes;
                    mbar_wait(smem_u32(&bar_v[st]), (m / NST) & 1);
                    mbar_wait(smem_u32(&bar_p[b]), (m >> 1) & 1);
                    tc_fence_after();
                    for (int kk = 0; kk < nc * 4; ++kk) {
                        const uint64_t bd = umma_desc_sw128(sV + kk * 2048, 16384, 1024);
                        mma_ts(tO, tP + b * 64 + kk * 8, bd, idO, (m > 0 || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(smem_u32(&bar_pv[b]));
                    mma_commit(smem_u32(&bar_empty[st]));
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------- softmax
        const int r = tid - 128;                  // row in tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int q_pos = item.qtile * 128 + r;
        const int rg = r >> 4;
        const float sl2 = p.scale_log2;
        float m_run = -INFINITY, l_run = 0.f;
        for (int n = 0; n < T; ++n) {
            const int b = n & 1;
            const int nc = (2 * n + 1 < cnt) ? 2 : 1;
            mbar_wait(smem_u32(&bar_s[b]), (n >> 1) & 1);
            tc_fence_after();
            float s[128];
            {
                uint32_t u[32];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (c < nc * 2) {
                        tmem_ld32(tS + b * 128 + c * 32 + lane_off, u);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(u[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) s[c * 32 + j] = -INFINITY;
                    }
                }
            }
            // block-level mask (16x16 granularity) + token causality
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h < nc) {
                    const int2 e = ch[2 * n + h];
                    const uint32_t bits = (static_cast<uint32_t>(e.y) >> (rg * 4)) & 0xFu;
                    const int key0 = e.x * 64;
                    const bool diag = key0 + 63 > item.qtile * 128;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const bool on = (bits >> g) & 1u;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int c = h * 64 + g * 16 + j;
                            if (!on || (diag && key0 + g * 16 + j > q_pos)) s[c] = -INFINITY;
                        }
                    }
                }
            }
            float mx = s[0];
#pragma unroll
            for (int j = 1; j < 128; ++j) mx = fmaxf(mx, s[j]);
            const float m_tile = mx * sl2;
            float m_use = m_run;
            bool rescale = false;
            if (m_tile > m_run) {
                if (m_run == -INFINITY) {
                    m_use = m_tile;
                } else if (m_tile > m_run + 8.0f) {
                    m_use = m_tile;
                    rescale = true;
                }
            }
            if (__any_sync(0xffffffffu, rescale)) {
                // O of this row must be stable: PV_{n-1} complete.
                mbar_wait(smem_u32(&bar_pv[(n - 1) & 1]), ((n - 1) >> 1) & 1);
                tc_fence_after();
                const float alpha = rescale ? fast_exp2(m_run - m_use) : 1.0f;
                l_run *= alpha;
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t u[32];
                    tmem_ld32(tO + c * 32 + lane_off, u);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * alpha);
                    tmem_st32(tO + c * 32 + lane_off, u);
                }
            }
            const float base = (m_use == -INFINITY) ? 0.f : m_use;
            float sum = 0.f;
            uint32_t pk[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const float p0 = fast_exp2(fmaf(s[2 * j], sl2, -base));
                const float p1 = fast_exp2(fmaf(s[2 * j + 1], sl2, -base));
                sum += p0 + p1;
                pk[j] = pack_bf16(p0, p1);
            }
            l_run += sum;
            m_run = m_use;
            // P buffer b was last read by PV_{n-2}.
            if (n >= 2) mbar_wait(smem_u32(&bar_pv[b]), ((n - 2) >> 1) & 1);
            tc_fence_after();
            {
                uint32_t u[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) u[j] = pk[j];
                tmem_st32(tP + b * 64 + lane_off, u);
                if (nc == 2) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) u[j] = pk[32 + j];
                    tmem_st32(tP + b * 64 + 32 + lane_off, u);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_p[b]));
        }
        // ---------------------------------------------------- epilogue
        mbar_wait(smem_u32(&bar_pv[(T - 1) & 1]), ((T - 1) >> 1) & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l_run;
        const bool valid = q_pos < p.seq_len;
        __nv_bfloat16* orow = p.out + (static_cast<size_t>(item.bh) * p.seq_len + q_pos) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(tO + c * 32 + lane_off, u);
            tmem_ld_wait();
            if (valid) {
                uint4 w[4];
                uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    wp[j] = pack_bf16(__uint_as_float(u[2 * j]) * inv_l,
                                      __uint_as_float(u[2 * j + 1]) * inv_l);
                uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[j] = w[j];
            }
        }
        if (valid)
            p.lse[static_cast<size_t>(item.bh) * p.seq_len + q_pos] =
                (m_run + __log2f(l_run)) * 0.69314718055994530942f;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int D, int NST>
static cudaError_t launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                          const FwdParams& p, int num_items, cudaStream_t stream) {
    using L = FwdSmem<D, NST>;
    auto kern = s2_fwd_sm100_kernel<D, NST>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (e != cudaSuccess) return e;
    kern<<<num_items, 256, L::kTotal, stream>>>(q, k, v, p);
    return cudaGetLastError();
}

}  // namespace s2dev

// Host entry used by capi.cpp.
cudaError_t s2_launch_fwd_sm100(int head_dim, const CUtensorMap& q, const CUtensorMap& k,
                                const CUtensorMap& v, const s2dev::FwdItem* items, int num_items,
                                const int2* chunks, __nv_bfloat16* out, float* lse, int seq_len,
                                int hpg, float scale_log2, cudaStream_t stream) {
    s2dev::FwdParams p{items, chunks, out, lse, seq_len, hpg, scale_log2};
    if (num_items == 0) return cudaSuccess;
    if (head_dim == 128) return s2dev::launch<128, 2>(q, k, v, p, num_items, stream);
    if (head_dim == 64) return s2dev::launch<64, 4>(q, k, v, p, num_items, stream);
    return cudaErrorInvalidValue;
}
