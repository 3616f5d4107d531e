// S2 sparse decode over a per-(batch, kv-head) COMPACTED KV cache, sm_100a.
//
// The reference has no decode kernel; its only decode logic is the cache
// simulator simulate_decode_cache (/root/reference/proj/src/analysis.cpp:
// 57-104): key block j is retained while the decode row bt <= evict_after[j]
// (:76-82), and for KV-efficient masks (verify.cpp:53-72) the retained set is
// exactly row bt of the mask (test_analysis.cpp:148-161).  The cache below
// stores only those blocks: every kv head has a slot pool; a block keeps one
// slot from generation until eviction; the decode row is a list of slots.
//
//  * s2_kv_compact_kernel: dense prefix [B,Hkv,T,D] -> slots of retained blocks
//  * s2_kv_append_kernel:  one new token per (b, kv head)
//  * s2_decode_split_kernel: split-KV attention of all query heads of a GQA
//    group at position t over a contiguous range of the row's slots; K/V
//    64-token blocks streamed by TMA (128-byte swizzle, conflict-free smem
//    reads) through an NST-deep ring; fp32 math on CUDA cores (the step is
//    HBM-bound: ~0.25 FMA/byte); partial (o, lse) per split.
//  * s2_decode_combine_kernel: lse-weighted merge of the splits.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {


template <int HPG, int D>
__global__ void __launch_bounds__(128) s2_decode_split_kernel(const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV,
                                                              const DecodeParams p) {
    constexpr int NST = 3;
    constexpr int SUB = D / 64;
    constexpr int BLK_BYTES = SUB * 8192;  // 64 tokens x D bf16
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_full[NST];
    __shared__ float sq[HPG][D];           // q of the group's heads, pre-scaled (log2)
    __shared__ float sp[HPG][64];          // probabilities of the current block
    __shared__ float smax[2][HPG];
    const int tid = threadIdx.x;
    const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
    const int64_t roff = p.row_ptr[static_cast<size_t>(g) * (p.NB + 1) + p.bt];
    const int len = static_cast<int>(p.row_ptr[static_cast<size_t>(g) * (p.NB + 1) + p.bt + 1] - roff);
    const int first = split * p.blocks_per_split;
    const int nblk = max(0, min(p.blocks_per_split, len - first));
    const int* slots = p.slot_idx + roff + first;
    const int kvbh = b * p.Hkv + g;

    for (int i = tid; i < HPG * D; i += 128) {
        const int h = i / D, x = i % D;
        sq[h][x] = __bfloat162float(p.q[(static_cast<size_t>(b) * p.H + g * HPG + h) * D + x]) *
                   p.scale_log2;
    }
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) mbar_init(smem_u32(&bar_full[i]), 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t sbase = smem_u32(smem);
    auto issue = [&](int i) {
        const int st = i % NST;
        const uint32_t dst = sbase + st * 2 * BLK_BYTES;
        const uint32_t bar = smem_u32(&bar_full[st]);
        mbar_expect_tx(bar, 2 * BLK_BYTES);
        const int row = slots[i] * 64;
#pragma unroll
        for (int s = 0; s < SUB; ++s) {
            tma_load_3d(dst + s * 8192, &tmK, bar, s * 64, row, kvbh);
            tma_load_3d(dst + BLK_BYTES + s * 8192, &tmV, bar, s * 64, row, kvbh);
        }
    };
    if (tid == 0)
        for (int i = 0; i < NST && i < nblk; ++i) issue(i);

    // score mapping: token = tid % 64, heads hs*NHT .. of hs = tid / 64
    constexpr int NHT = HPG >= 2 ? HPG / 2 : 1;
    const int tok = tid & 63, hs = tid >> 6;
    const bool score_thread = HPG >= 2 || hs == 0;
    // PV mapping: 16-byte d-chunk c = tid % (D/8), token group tg = tid / (D/8)
    constexpr int NCH = D / 8;             // 16B chunks per row
    constexpr int NTG = 128 / NCH;         // token groups
    const int c = tid % NCH, tg = tid / NCH;
    float acc[HPG][8];
#pragma unroll
    for (int h = 0; h < HPG; ++h)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[h][e] = 0.f;
    float m_run[HPG], l_run[HPG];
#pragma unroll
    for (int h = 0; h < HPG; ++h) {
        m_run[h] = -INFINITY;
        l_run[h] = 0.f;
    }

    for (int i = 0; i < nblk; ++i) {
        const int st = i % NST;
        mbar_wait(smem_u32(&bar_full[st]), (i / NST) & 1);
        const uint8_t* sK = smem + st * 2 * BLK_BYTES;
        const uint8_t* sV = sK + BLK_BYTES;
        const int valid = (first + i == len - 1) ? p.last_tokens : 64;
        // ---- scores
        float s[NHT];
#pragma unroll
        for (int h = 0; h < NHT; ++h) s[h] = 0.f;
        if (score_thread) {
#pragma unroll
            for (int sub = 0; sub < SUB; ++sub)
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    const uint4 kv = *reinterpret_cast<const uint4*>(
                        sK + sub * 8192 + tok * 128 + ((ch ^ (tok & 7)) << 4));
                    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
                    float kf[8];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        kf[2 * e] = __low2float(k2[e]);
                        kf[2 * e + 1] = __high2float(k2[e]);
                    }
                    const int x0 = sub * 64 + ch * 8;
#pragma unroll
                    for (int h = 0; h < NHT; ++h) {
                        const float* qh = sq[hs * NHT + h] + x0;
#pragma unroll
                        for (int e = 0; e < 8; ++e) s[h] = fmaf(qh[e], kf[e], s[h]);
                    }
                }
            if (tok >= valid)
#pragma unroll
                for (int h = 0; h < NHT; ++h) s[h] = -INFINITY;
        }
        // ---- block max per head (two warps per head set)
#pragma unroll
        for (int h = 0; h < NHT; ++h) {
            float mx = s[h];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((tid & 31) == 0 && score_thread) smax[(tid >> 5) & 1][hs * NHT + h] = mx;
        }
        __syncthreads();
        float alpha[HPG];
#pragma unroll
        for (int h = 0; h < HPG; ++h) {
            const float mb = fmaxf(smax[0][h], smax[1][h]);
            const float mn = fmaxf(m_run[h], mb);
            alpha[h] = (m_run[h] == -INFINITY) ? 0.f : fast_exp2(m_run[h] - mn);
            m_run[h] = mn;
        }
        if (score_thread)
#pragma unroll
            for (int h = 0; h < NHT; ++h) sp[hs * NHT + h][tok] = fast_exp2(s[h] - m_run[hs * NHT + h]);
        __syncthreads();
        // ---- l and PV
#pragma unroll
        for (int h = 0; h < HPG; ++h) {
            float ps = 0.f;
            for (int t = 0; t < 64; ++t) ps += sp[h][t];
            l_run[h] = l_run[h] * alpha[h] + ps;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[h][e] *= alpha[h];
        }
        const int sub = c / 8, ch = c % 8;
        for (int t = tg; t < 64; t += NTG) {
            const uint4 vv = *reinterpret_cast<const uint4*>(sV + sub * 8192 + t * 128 + ((ch ^ (t & 7)) << 4));
            const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vv);
            float vf[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                vf[2 * e] = __low2float(v2[e]);
                vf[2 * e + 1] = __high2float(v2[e]);
            }
#pragma unroll
            for (int h = 0; h < HPG; ++h) {
                const float ph = sp[h][t];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[h][e] = fmaf(ph, vf[e], acc[h][e]);
            }
        }
        __syncthreads();
        if (tid == 0 && i + NST < nblk) issue(i + NST);
    }
    // ---- reduce the token groups through shared memory (reuse the ring)
    float* red = reinterpret_cast<float*>(smem);  // [NTG][HPG][D]
    __syncthreads();
#pragma unroll
    for (int h = 0; h < HPG; ++h)
#pragma unroll
        for (int e = 0; e < 8; ++e) red[(tg * HPG + h) * D + c * 8 + e] = acc[h][e];
    __syncthreads();
    for (int i = tid; i < HPG * D; i += 128) {
        const int h = i / D, x = i % D;
        float o = 0.f;
        for (int t = 0; t < NTG; ++t) o += red[(t * HPG + h) * D + x];
        const size_t row = (static_cast<size_t>(b) * p.H + g * HPG + h) * p.splits + split;
        const float l = l_run[h];
        p.o_part[row * D + x] = nblk > 0 && l > 0.f ? o / l : 0.f;
        if (x == 0) p.lse_part[row] = nblk > 0 && l > 0.f ? m_run[h] + __log2f(l) : -INFINITY;
    }
}

__global__ void s2_decode_combine_kernel(const float* __restrict__ o_part,
                                         const float* __restrict__ lse_part, int splits, int D,
                                         __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
    const int bh = blockIdx.x;
    const float* lp = lse_part + static_cast<size_t>(bh) * splits;
    float m = -INFINITY;
    for (int s = 0; s < splits; ++s) m = fmaxf(m, lp[s]);
    float den = 0.f;
    for (int s = 0; s < splits; ++s) den += lp[s] == -INFINITY ? 0.f : exp2f(lp[s] - m);
    for (int x = threadIdx.x; x < D; x += blockDim.x) {
        float num = 0.f;
        for (int s = 0; s < splits; ++s)
            if (lp[s] != -INFINITY)
                num += exp2f(lp[s] - m) * o_part[(static_cast<size_t>(bh) * splits + s) * D + x];
        out[static_cast<size_t>(bh) * D + x] = __float2bfloat16_rn(num / den);
    }
    if (threadIdx.x == 0 && lse) lse[bh] = (m + log2f(den)) * 0.69314718055994530942f;
}

// dense [B, Hkv, T, D] -> pool [B, Hkv, cap*S, D]: one CTA per (retained block, b)
__global__ void s2_kv_compact_kernel(const __nv_bfloat16* __restrict__ k,
                                     const __nv_bfloat16* __restrict__ v,
                                     __nv_bfloat16* __restrict__ kp, __nv_bfloat16* __restrict__ vp,
                                     const int4* __restrict__ items, int Hkv, int T, int S, int D,
                                     int cap) {
    const int4 item = items[blockIdx.x];  // {g, key block, slot, -}
    const int2 it = make_int2(item.y, item.z);
    const int g = item.x, b = blockIdx.y;
    const size_t src = ((static_cast<size_t>(b) * Hkv + g) * T + static_cast<size_t>(it.x) * S) * D;
    const size_t dst = ((static_cast<size_t>(b) * Hkv + g) * cap * S + static_cast<size_t>(it.y) * S) * D;
    const int ntok = min(S, T - it.x * S);
    const int n16 = ntok * D / 8;
    const uint4* ks = reinterpret_cast<const uint4*>(k + src);
    const uint4* vs = reinterpret_cast<const uint4*>(v + src);
    uint4* kd = reinterpret_cast<uint4*>(kp + dst);
    uint4* vd = reinterpret_cast<uint4*>(vp + dst);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) {
        kd[i] = ks[i];
        vd[i] = vs[i];
    }
}

__global__ void s2_kv_append_kernel(const __nv_bfloat16* __restrict__ k,
                                    const __nv_bfloat16* __restrict__ v,
                                    __nv_bfloat16* __restrict__ kp, __nv_bfloat16* __restrict__ vp,
                                    const int* __restrict__ slot_of, int NB, int bt, int Hkv, int S,
                                    int D, int cap, int pos_in_block) {
    const int bg = blockIdx.x;  // b*Hkv + g
    const int g = bg % Hkv;
    const int slot = slot_of[static_cast<size_t>(g) * NB + bt];
    const size_t dst = (static_cast<size_t>(bg) * cap * S + static_cast<size_t>(slot) * S +
                        pos_in_block) * D;
    for (int x = threadIdx.x; x < D; x += blockDim.x) {
        kp[dst + x] = k[static_cast<size_t>(bg) * D + x];
        vp[dst + x] = v[static_cast<size_t>(bg) * D + x];
    }
}

}  // namespace s2dev

using namespace s2dev;

template <int HPG, int D>
static cudaError_t launch_decode(const CUtensorMap& mk, const CUtensorMap& mv,
                                 const DecodeParams& p, int batch, cudaStream_t st) {
    const int smem = 1024 + 3 * 2 * (D / 64) * 8192;
    auto kern = s2_decode_split_kernel<HPG, D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(p.splits, p.Hkv, batch), 128, smem, st>>>(mk, mv, p);
    return cudaGetLastError();
}

cudaError_t s2_launch_decode(const CUtensorMap& mk, const CUtensorMap& mv, const DecodeParams& p,
                             int batch, cudaStream_t st) {
#define S2_DEC(HP, DD) \
    if (p.hpg == HP && p.D == DD) return launch_decode<HP, DD>(mk, mv, p, batch, st);
    S2_DEC(1, 64) S2_DEC(2, 64) S2_DEC(4, 64) S2_DEC(8, 64)
    S2_DEC(1, 128) S2_DEC(2, 128) S2_DEC(4, 128) S2_DEC(8, 128)
#undef S2_DEC
    return cudaErrorInvalidValue;
}

cudaError_t s2_launch_decode_combine(const float* o_part, const float* lse_part, int splits, int D,
                                     int num_bh, __nv_bfloat16* out, float* lse, cudaStream_t st) {
    s2_decode_combine_kernel<<<num_bh, 128, 0, st>>>(o_part, lse_part, splits, D, out, lse);
    return cudaGetLastError();
}

cudaError_t s2_launch_kv_compact(const void* k, const void* v, void* kp, void* vp,
                                 const int4* items, int num_items, int batch, int Hkv, int T, int S,
                                 int D, int cap, cudaStream_t st) {
    if (num_items == 0) return cudaSuccess;
    s2_kv_compact_kernel<<<dim3(num_items, batch), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
        static_cast<__nv_bfloat16*>(kp), static_cast<__nv_bfloat16*>(vp), items, Hkv, T, S, D, cap);
    return cudaGetLastError();
}

cudaError_t s2_launch_kv_append(const void* k, const void* v, void* kp, void* vp,
                                const int* slot_of, int NB, int bt, int batch, int Hkv, int S,
                                int D, int cap, int pos_in_block, cudaStream_t st) {
    s2_kv_append_kernel<<<batch * Hkv, 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v),
        static_cast<__nv_bfloat16*>(kp), static_cast<__nv_bfloat16*>(vp), slot_of, NB, bt, Hkv, S,
        D, cap, pos_in_block);
    return cudaGetLastError();
}
