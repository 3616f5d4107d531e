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
//    64-token blocks streamed by TMA (128-byte swizzle) through an NST-deep
//    ring by a producer warp; QK^T and PV on the tensor cores (mma.sync, the
//    group's heads as the M rows), fp32 online softmax; partial (o, lse) per
//    split.
//  * s2_decode_combine_kernel: lse-weighted merge of the splits.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {


__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D(16x8, f32) += A(16x16, bf16, rows 8..15 zero) * B(16x8, bf16)
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                          uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
        "{%8, %9}, {%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// Split-KV decode of one (batch, kv head, split).  Warp 4 streams the
// split's 64-token K/V blocks by TMA (128-byte swizzle) through an NST ring;
// warps 0-3 each own 16 tokens of every block and run the block on the
// tensor cores (mma.sync m16n8k16: the GQA group's query heads are the M
// rows, so one K/V read serves every head of the group):
//   S(heads x 16 tok) = Q K^T   (K fragments by ldmatrix)
//   P = exp2(S*scale - m)        online softmax per warp (quad shuffles)
//   O(heads x D) += P V          (P re-used from the S accumulators as the A
//                                 fragment; V fragments by ldmatrix.trans)
// The four per-warp states (m, l, O) are merged through shared memory and
// written as the split's partial (o, lse); s2_decode_combine_kernel merges
// the splits.  The step is HBM-bound; the MMAs only keep the SM's issue
// slots free so the ring stays full.
template <int HPG, int D>
__global__ void __launch_bounds__(160) s2_decode_split_kernel(const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV,
                                                              const DecodeParams p) {
    constexpr int NST = 3;
    constexpr int SUB = D / 64;
    constexpr int BLK_BYTES = SUB * 8192;  // 64 tokens x D bf16
    constexpr int KSTEPS = D / 16;
    constexpr int NT = D / 8;  // n-tiles of the PV product
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_full[NST], bar_empty[NST];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, g = blockIdx.y, b = blockIdx.z;
    const int64_t roff = p.row_ptr[static_cast<size_t>(g) * (p.NB + 1) + p.bt];
    const int len = static_cast<int>(p.row_ptr[static_cast<size_t>(g) * (p.NB + 1) + p.bt + 1] - roff);
    const int first = split * p.blocks_per_split;
    const int nblk = max(0, min(p.blocks_per_split, len - first));
    const int* slots = p.slot_idx + roff + first;
    const int kvbh = b * p.Hkv + g;
    const uint32_t sbase = smem_u32(smem);

    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_full[i]), 1);
            mbar_init(smem_u32(&bar_empty[i]), 4);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // programmatic dependent launch: the combine's CTAs may be scheduled from here;
    // q, the cache and o_part / lse_part (read by the previous combine) are only
    // touched after the previous kernel in the stream has completed
    pdl_launch_dependents();
    pdl_wait();

    if (warp == 4) {
        // ---------------------------------------------------------- producer
        if (lane == 0) {
            const uint64_t stream = policy_evict_first();
            for (int i = 0; i < nblk; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(smem_u32(&bar_empty[st]), ((i / NST) + 1) & 1);
                const uint32_t dst = sbase + st * 2 * BLK_BYTES;
                const uint32_t bar = smem_u32(&bar_full[st]);
                mbar_expect_tx(bar, 2 * BLK_BYTES);
                const int row = slots[i] * 64;
#pragma unroll
                for (int s = 0; s < SUB; ++s) {
                    tma_load_3d_hint(dst + s * 8192, &tmK, bar, s * 64, row, kvbh, stream);
                    tma_load_3d_hint(dst + BLK_BYTES + s * 8192, &tmV, bar, s * 64, row, kvbh, stream);
                }
            }
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    const int gq = lane >> 2, tg = lane & 3;  // fragment row (head) / column pair
    const bool head_ok = gq < HPG;
    // A fragments of Q (rows = heads, rows 8..15 are zero): a0 = cols 2tg.., a2 = cols 2tg+8..
    uint32_t qa[KSTEPS][2];
    {
        const __nv_bfloat16* qrow = p.q + (static_cast<size_t>(b) * p.H + g * HPG + (head_ok ? gq : 0)) * D;
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
            qa[kk][0] = head_ok ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * tg) : 0u;
            qa[kk][1] = head_ok ? *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 8 + 2 * tg) : 0u;
        }
    }
    float o[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = p.scale_log2;
    const int tok0 = warp * 16;  // this warp's tokens within each block
    // ldmatrix row addresses (swizzled: 16-byte chunk c of token r sits at c ^ (r & 7))
    const int mi = lane >> 3, r8 = lane & 7;
    const int k_tok = tok0 + (mi >> 1) * 8 + r8, k_chk = mi & 1;   // K: {n-tile, k-half}
    const int v_tok = tok0 + (mi & 1) * 8 + r8, v_chk = mi >> 1;   // V: {k-half, n-tile}

    for (int i = 0; i < nblk; ++i) {
        const int st = i % NST;
        mbar_wait(smem_u32(&bar_full[st]), (i / NST) & 1);
        const uint32_t sK = sbase + st * 2 * BLK_BYTES, sV = sK + BLK_BYTES;
        const int valid = (first + i == len - 1) ? p.last_tokens : 64;
        // ---- S = Q K^T for 16 tokens (two n-tiles)
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < KSTEPS; ++kk) {
            const int c = 2 * kk + k_chk;  // 16-byte chunk along D
            const uint32_t addr = sK + (c >> 3) * 8192 + k_tok * 128 + (((c & 7) ^ (k_tok & 7)) << 4);
            uint32_t b00, b01, b10, b11;
            ldsm_x4(addr, b00, b01, b10, b11);
            mma_16816(sc[0], qa[kk][0], qa[kk][1], b00, b01);
            mma_16816(sc[1], qa[kk][0], qa[kk][1], b10, b11);
        }
        // ---- online softmax (row = head gq; its 16 scores live in the quad)
        float s[4] = {sc[0][0] * sl2, sc[0][1] * sl2, sc[1][0] * sl2, sc[1][1] * sl2};
        if (valid < 64) {
            const int t0 = tok0 + 2 * tg;
            if (t0 >= valid) s[0] = -INFINITY;
            if (t0 + 1 >= valid) s[1] = -INFINITY;
            if (t0 + 8 >= valid) s[2] = -INFINITY;
            if (t0 + 9 >= valid) s[3] = -INFINITY;
        }
        float mx = fmaxf(fmaxf(s[0], s[1]), fmaxf(s[2], s[3]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);
        const float base = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = fast_exp2(m_run - base);
        float pr[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) pr[e] = fast_exp2(s[e] - base);
        l_run = l_run * alpha + (pr[0] + pr[1]) + (pr[2] + pr[3]);
        m_run = m_new;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            o[j][0] *= alpha;
            o[j][1] *= alpha;
        }
        const uint32_t pa0 = pack_bf16(pr[0], pr[1]), pa2 = pack_bf16(pr[2], pr[3]);
        // ---- O += P V (V fragments transposed out of the token-major tile)
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
            const int c = j + v_chk;
            const uint32_t addr = sV + (c >> 3) * 8192 + v_tok * 128 + (((c & 7) ^ (v_tok & 7)) << 4);
            uint32_t b0a, b1a, b0b, b1b;
            ldsm_x4_t(addr, b0a, b1a, b0b, b1b);
            mma_16816(o[j], pa0, pa2, b0a, b1a);
            mma_16816(o[j + 1], pa0, pa2, b0b, b1b);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_empty[st]));
    }
    // quad-reduce l (each lane summed its own 4 columns)
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);

    // ---- merge the four warps' states (reuse the ring: every stage was consumed)
    named_bar_sync(1, 128);
    float* red_o = reinterpret_cast<float*>(smem);   // [4][HPG][D]
    float* red_m = red_o + 4 * HPG * D;              // [4][HPG]
    float* red_l = red_m + 4 * HPG;                  // [4][HPG]
    if (head_ok) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            float* dst = red_o + (warp * HPG + gq) * D + j * 8 + 2 * tg;
            dst[0] = o[j][0];
            dst[1] = o[j][1];
        }
        if (tg == 0) {
            red_m[warp * HPG + gq] = m_run;
            red_l[warp * HPG + gq] = l_run;
        }
    }
    named_bar_sync(1, 128);
    for (int idx = tid; idx < HPG * D; idx += 128) {
        const int h = idx / D, x = idx % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, red_m[w * HPG + h]);
        float num = 0.f, den = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float f = fast_exp2(red_m[w * HPG + h] - M);
                num += f * red_o[(w * HPG + h) * D + x];
                den += f * red_l[w * HPG + h];
            }
        }
        const size_t row = (static_cast<size_t>(b) * p.H + g * HPG + h) * p.splits + split;
        const bool ok = den > 0.f;
        p.o_part[row * D + x] = ok ? num / den : 0.f;
        if (x == 0) p.lse_part[row] = ok ? M + __log2f(den) : -INFINITY;
    }
}

__global__ void s2_decode_combine_kernel(const float* __restrict__ o_part,
                                         const float* __restrict__ lse_part, int splits, int D,
                                         __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
    const int bh = blockIdx.x;
    pdl_wait();  // the split kernel's partials are complete and visible
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
    static_assert(4 * HPG * D * 4 + 8 * HPG * 4 <= 3 * 2 * (D / 64) * 8192, "merge buffer fits the ring");
    auto kern = s2_decode_split_kernel<HPG, D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(p.splits, p.Hkv, batch), dim3(160), smem, st, mk, mv, p);
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
    return launch_pdl(s2_decode_combine_kernel, dim3(num_bh), dim3(128), 0, st, o_part, lse_part, splits, D, out,
                      lse);
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
