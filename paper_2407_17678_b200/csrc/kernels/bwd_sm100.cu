// S2-Attention backward, sm_100a (no reference symbol: SPEC.md:262).
//
// Gradient of out = softmax_masked(scale * Q K^T) V over the same admitted
// set as the forward (reference.cpp:28-36): P = exp(scale*S - lse),
// dP = dO V^T, dS = P o (dP - Delta), Delta = rowsum(dO o O),
// dV = P^T dO, dK = scale * dS^T Q, dQ = scale * dS K.
//
//  * s2_bwd_prep_kernel: Delta and lse*log2(e) into row-padded workspaces.
//  * s2_bwd_dkv_kernel:  one CTA owns a 128-key tile (two 64-key chunks,
//    paired by similar q-tile lists) of one kv head and walks the TRANSPOSED
//    tile list (every q tile of every query head of its GQA group that
//    attends it) in 64-row halves.  dK/dV accumulate in TMEM and are written
//    once: no atomics, deterministic.
//  * s2_bwd_dq_kernel:   one CTA owns a 128-row query tile and walks its
//    CSR chunk list, dQ accumulating in TMEM.
//
// Both use the same warp layout (384 threads): warp 0 TMA producer, warp 1
// MMA issuer, warp 2 TMEM allocator, warps 4-7 / 8-11 two elementwise
// warpgroups that split the 64 columns of each score tile (32 each), with
// S/dP double-buffered in TMEM so the elementwise pass of step n overlaps
// the MMAs of steps n-1 and n+1.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {

// ------------------------------------------------------------------ prep
#ifndef S2_PREP_ROWS
#define S2_PREP_ROWS 1
#endif
// Delta = rowsum(dO o O) and lse*log2(e) per row; HBM-bound (reads O and dO
// once).  D/8 lanes own a row (16-byte loads), 256 / (D/8) rows per 256-thread
// block iteration, grid-stride over rows.
#ifndef S2_DKV_L2HINT
#define S2_DKV_L2HINT 1
#endif

template <int D>
__global__ void __launch_bounds__(256) s2_bwd_prep_kernel(const __nv_bfloat16* __restrict__ out,
                                                          const __nv_bfloat16* __restrict__ dout,
                                                          const float* __restrict__ lse,
                                                          float* __restrict__ delta,
                                                          float* __restrict__ lse2, int num_bh,
                                                          int N, int Npad) {
    // Rows in 32-bit arithmetic (the host checks num_bh * Npad < 2^31): a 64-bit
    // divide / modulo per row made this kernel issue-bound, not HBM-bound.
    pdl_launch_dependents();
    pdl_wait();
    constexpr int LPR = D / 8;  // lanes per row
    constexpr int kRows = S2_PREP_ROWS;  // rows per thread per sweep (2 x kRows 16-byte loads in flight)
    const uint32_t total = static_cast<uint32_t>(num_bh) * static_cast<uint32_t>(Npad);
    const uint32_t sub = threadIdx.x % LPR;
    const uint32_t stride = gridDim.x * blockDim.x / LPR;  // rows per sweep
    for (uint32_t row0 = (blockIdx.x * blockDim.x + threadIdx.x) / LPR; row0 < total; row0 += kRows * stride) {
        uint4 a[kRows], b[kRows];
        uint32_t bh[kRows], t[kRows];
#pragma unroll
        for (int u = 0; u < kRows; ++u) {  // issue every load first
            const uint32_t row = row0 + u * stride;
            bh[u] = row / static_cast<uint32_t>(Npad);
            t[u] = row - bh[u] * static_cast<uint32_t>(Npad);
            a[u] = b[u] = make_uint4(0u, 0u, 0u, 0u);
            if (row < total && t[u] < static_cast<uint32_t>(N)) {
                const size_t off = (static_cast<size_t>(bh[u]) * N + t[u]) * D + sub * 8;
                a[u] = __ldg(reinterpret_cast<const uint4*>(out + off));
                b[u] = __ldg(reinterpret_cast<const uint4*>(dout + off));
            }
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const uint32_t row = row0 + u * stride;
            const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 x = __bfloat1622float2(a2[j]), y = __bfloat1622float2(b2[j]);
                acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
            }
#pragma unroll
            for (int s = LPR / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
            if (sub == 0 && row < total) {
                // padded rows and rows without an admitted key (lse -inf, O NaN):
                // lse2 = +inf makes P = 0 and delta = 0 keeps dS = 0 * (dP - delta) finite
                const float l = t[u] < static_cast<uint32_t>(N) ? lse[static_cast<size_t>(bh[u]) * N + t[u]]
                                                                : -INFINITY;
                const bool live = l > -INFINITY;
                delta[row] = live ? acc : 0.f;
                lse2[row] = live ? l * 1.4426950408889634f : INFINITY;
            }
        }
    }
}

struct BwdParams {
    const void* items;
    const int* sched;     // [grid + 1] item range of each CTA (host-side schedule)
    const void* entries;  // BwdEntry (dkv) or int2 chunks (dq)
    const float* lse2;    // [num_qbh][Npad], log2 domain, +inf padding
    const float* delta;   // [num_qbh][Npad]
    __nv_bfloat16* g0;    // dkv: dK ; dq: dQ
    __nv_bfloat16* g1;    // dkv: dV
    int N, Npad, hpg;
    float scale_log2, scale;
    long long* trace;  // debug: per-step clock64 of CTA 0 (nullptr = off)
    int debug;         // debug ablations (0 in production)
    // dQ kernel with the prep fused (s2_bwd_dq_kernel only): it computes Delta and
    // lse2 of its tile's rows from O, dO and lse and writes them to the workspace
    // rows (lse2 / delta above) that the dK/dV kernel, launched after it, reads
    const __nv_bfloat16* o;    // nullptr: not fused (the prep kernel ran)
    const __nv_bfloat16* dout;
    const float* lse;          // the forward's lse (natural log) [num_qbh][N]
    float* delta_w;            // = delta / lse2 above, writable (fused prep only)
    float* lse2_w;
};

#define S2TRACE(slot, n)                                                       \
    do {                                                                       \
        if (p.trace && blockIdx.x == 0 && (n) < 2048)  /* 16 slots x 2048 */   \
            p.trace[(slot) * 2048 + (n)] = clock64();                          \
    } while (0)

template <int D>
struct BwdCfg {
    static constexpr int kSub = D / 64;
    static constexpr int kTile128 = kSub * 16384;  // 128 rows x D bf16
    static constexpr int kTile64 = kSub * 8192;    // 64 rows x D bf16
    // dkv: resident K (128 keys) in 2 buffers (the next item's K loads under
    // this item; a finished item's dead K tile stages its epilogue's TMA
    // stores), V in 1 buffer (it is copied into TMEM at item start, so the
    // next item's V can land right after); kNSTkv stages of Q64, dO64
    // (1024-B aligned SW128 tiles), an aux slot per stage (lse2[64], delta[64],
    // meta) and the barriers.  No static shared memory and no alignment slack:
    // the dynamic window is declared 1024-B aligned (checked at run time).
#ifndef S2_DKV_NST
#define S2_DKV_NST 4
#endif
    static constexpr int kNSTkv = S2_DKV_NST;
    static constexpr int kDkvStage = 2 * kTile64;
    static constexpr int kAux = 528;
    static constexpr int kDkvBars = 256;
    static constexpr int kDkvSmem = 3 * kTile128 + kNSTkv * kDkvStage + kNSTkv * kAux + kDkvBars;
    // dq: Q, dO (128 rows) in one buffer (they are copied into TMEM at item
    // start, so the next item's tiles land right after), a dQ staging tile for
    // the epilogue's TMA store, kNSTq stages of K64, V64 and the barriers.
#ifndef S2_DQ_NST
#define S2_DQ_NST 4
#endif

    static constexpr int kNSTq = S2_DQ_NST;
    static constexpr int kDqStage = 2 * kTile64;
    static constexpr int kDqBars = 256 + 1024;  // barriers | fused prep: 2 x 128 partial row dots
    static constexpr int kDqSmem = 3 * kTile128 + kNSTq * kDqStage + kDqBars;
};

// Stage layout of the dK/dV kernel: Q rows [64][D] | dO rows [64][D], and the
// stage's aux slot: lse2[64] | delta[64] | meta (4 x u32: first q row, chunk-0 /
// chunk-1 masks of this 64-row half (row groups 0..3), query data index).  The producer writes meta
// with a plain shared store before its expect_tx arrive (release), so whoever
// observes the stage's full barrier sees it: the MMA issuer and the
// elementwise warps never touch the global entry list.
template <int D>
__global__ void __launch_bounds__(384, 1)
    s2_bwd_dkv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                      const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
                      const BwdParams p) {
    using C = BwdCfg<D>;
    constexpr int NST = C::kNSTkv;
    constexpr int kMeta = 512;  // byte offset of the meta in a stage's aux slot
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1024-B alignment
    // bar_kvf[kb]: K buffer kb and the V buffer hold the item's tiles.
    // bar_kve[kb]: K buffer kb is free (its item's last S^T MMA done AND the
    // epilogue TMA stores staged in it have read it): count 2.
    // bar_vcp: the item's V has been copied into TMEM.  bar_ve (count 2): the V
    // buffer may be refilled -- the copy is done AND the previous item's
    // epilogue, which stages dK in the V buffer, has been stored.
    // bar_dpf: the elementwise warps have read dP^T (its single TMEM buffer is free).
    struct Bars {
        uint64_t kvf[2], kve[2], ve, vcp, sf[NST], se[NST], s[2], p[2], af, ae, dpf;
        uint32_t tmem_base;
    };
    static_assert(sizeof(Bars) <= C::kDkvBars, "barrier block");
    Bars& bars = *reinterpret_cast<Bars*>(smem + 3 * C::kTile128 + NST * (C::kDkvStage + C::kAux));
    auto& bar_kvf = bars.kvf;
    auto& bar_kve = bars.kve;
    auto& bar_ve = bars.ve;
    auto& bar_vcp = bars.vcp;
    auto& bar_sf = bars.sf;
    auto& bar_se = bars.se;
    auto& bar_s = bars.s;
    auto& bar_p = bars.p;
    auto& bar_af = bars.af;
    auto& bar_ae = bars.ae;
    auto& bar_dpf = bars.dpf;
    auto& tmem_base_s = bars.tmem_base;
    // K buffer kb at sK + kb * kTile128, the V buffer after both
    const uint32_t sK = smem_u32(smem), sV = sK + 2 * C::kTile128;
    const uint32_t sSt = sK + 3 * C::kTile128;
    const uint32_t sAux = sSt + NST * C::kDkvStage;
    uint8_t* const gAux = smem + (sAux - sK);  // generic pointer to aux 0
    const BwdItem* items = static_cast<const BwdItem*>(p.items);
    const BwdEntry* ents = static_cast<const BwdEntry*>(p.entries);

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_kvf[i]), 1);
            mbar_init(smem_u32(&bar_kve[i]), 2);
        }
        mbar_init(smem_u32(&bar_ve), 2);
        mbar_init(smem_u32(&bar_vcp), 1);
        mbar_init(smem_u32(&bar_af), 1);
        mbar_init(smem_u32(&bar_ae), 256);
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_sf[i]), 1);
            mbar_init(smem_u32(&bar_se[i]), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_s[i]), 1);
            mbar_init(smem_u32(&bar_p[i]), 256);
        }
        mbar_init(smem_u32(&bar_dpf), 256);
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
    pdl_launch_dependents();
    pdl_wait();  // the previous kernel's outputs are visible from here on
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x] = globaltimer_ns();  // debug: CTA start
    // TMEM: V at 0 (the dP^T A operand: copied in once per item with tcgen05.cp, so
    // the per-step dP^T MMAs read only the 2 KB dO slices from shared memory),
    // S^T[b] at 64+64b (the elementwise warps write P^T and dS^T back into it: warp
    // group w's 32 columns hold P^T at +0..15 and dS^T at +16..31), dP^T at 192
    // (single buffer: read into registers at the start of each elementwise pass),
    // dV at 256, dK at 384.
    const int i_beg = p.sched[blockIdx.x], i_end = p.sched[blockIdx.x + 1];

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
        if (warp == 0 && lane == 0) {
            // ---------------------------------------------------- producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmdO);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            uint32_t it_cnt = 0, st_it = 0;
            // S2_DKV_L2HINT: Q / dO rows are re-streamed by every key tile of the head
            // (keep them in L2); a key tile's K / V are read once (stream them)
            const uint64_t keep = policy_evict_last(), once = policy_evict_first();
            for (int i = i_beg; i < i_end; ++i, ++it_cnt) {
                const BwdItem it = items[i];
                const int kb = it_cnt & 1;
                if (it_cnt >= 2) mbar_wait(smem_u32(&bar_kve[kb]), ((it_cnt >> 1) - 1) & 1);
                const int nc = it.c1 >= 0 ? 2 : 1;
                const uint32_t kvbar = smem_u32(&bar_kvf[kb]), kvoff = kb * C::kTile128;
                mbar_expect_tx(kvbar, 2 * nc * C::kSub * 8192);
                for (int h = 0; h < nc; ++h)
                    for (int s = 0; s < C::kSub; ++s) {
                        const int row = (h ? it.c1 : it.c0) * 64;
                        if (S2_DKV_L2HINT)
                            tma_load_3d_hint(sK + kvoff + s * 16384 + h * 8192, &tmK, kvbar, s * 64, row, it.kvbh, once);
                        else
                            tma_load_3d(sK + kvoff + s * 16384 + h * 8192, &tmK, kvbar, s * 64, row, it.kvbh);
                    }
                if (it_cnt >= 1) mbar_wait(smem_u32(&bar_ve), (it_cnt - 1) & 1);
                for (int h = 0; h < nc; ++h)
                    for (int s = 0; s < C::kSub; ++s) {
                        const int row = (h ? it.c1 : it.c0) * 64;
                        if (S2_DKV_L2HINT)
                            tma_load_3d_hint(sV + s * 16384 + h * 8192, &tmV, kvbar, s * 64, row, it.kvbh, once);
                        else
                            tma_load_3d(sV + s * 16384 + h * 8192, &tmV, kvbar, s * 64, row, it.kvbh);
                    }
                for (int j = 0; j < p.hpg; ++j) {
                    const int qbh = it.kvbh * p.hpg + j;
                    // q tiles descending: every stripe tile of a head ends at the last q
                    // tile, so tiles of one head running together meet on the same Q/dO
                    // rows in L2 (3% faster than ascending at cfg3)
                    for (int e = it.count - 1; e >= 0; --e) {
                        const BwdEntry en = ents[it.offset + e];
                        for (int half = 0; half < 2; ++half) {
                            const uint32_t m0 = (en.mask0 >> (16 * half)) & 0xFFFFu;
                            const uint32_t m1 = (en.mask1 >> (16 * half)) & 0xFFFFu;
                            if ((m0 | m1) == 0) continue;
                            const int st = st_it % NST;
                            if (st_it >= NST) mbar_wait(smem_u32(&bar_se[st]), ((st_it / NST) + 1) & 1);
                            const uint32_t base = sSt + st * C::kDkvStage;
                            const uint32_t bar = smem_u32(&bar_sf[st]);
                            const int row0 = en.qtile * 128 + half * 64;
                            *reinterpret_cast<uint4*>(gAux + st * C::kAux + kMeta) =
                                make_uint4(static_cast<uint32_t>(row0), m0, m1, static_cast<uint32_t>(qbh));
                            // debug 16 (timing experiments only, wrong results): skip the dO tile
                            const bool half_bytes = (p.debug & 16) != 0;
                            mbar_expect_tx(bar, (half_bytes ? 1 : 2) * C::kTile64 + 512);
                            if (S2_DKV_L2HINT) {
                                tma_load_rows_hint(base, &tmQ, bar, row0, qbh, keep);
                                if (!half_bytes) tma_load_rows_hint(base + C::kTile64, &tmdO, bar, row0, qbh, keep);
                            } else {
                                tma_load_rows(base, &tmQ, bar, row0, qbh);
                                if (!half_bytes) tma_load_rows(base + C::kTile64, &tmdO, bar, row0, qbh);
                            }
                            const size_t lo = static_cast<size_t>(qbh) * p.Npad + row0;
                            bulk_load(sAux + st * C::kAux, p.lse2 + lo, 256, bar);
                            bulk_load(sAux + st * C::kAux + 256, p.delta + lo, 256, bar);
                            ++st_it;
                        }
                    }
                }
            }
        } else if (warp == 1) {
            // ---------------------------------------------------- MMA issuer
            // The whole warp runs the loop on warp-uniform values; one elected
            // lane issues (keeps descriptors in uniform registers: no
            // per-MMA waterfall loop).  Per step n: S^T(n), dP^T(n) into TMEM
            // buffer n&1, then dV, dK += the previous step's P^T, dS^T.
            constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0);
            constexpr uint32_t idA = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            // SW128 K-major advance along K = +32 B per 16 elements (+2 in the desc)
            const uint64_t dK0 = umma_desc_sw128(sK, 16, 1024), dV0 = umma_desc_sw128(sV, 16, 1024);
            const uint64_t dSt0 = umma_desc_sw128(sSt, 16, 1024);
            const uint64_t dStMN0 = umma_desc_sw128(sSt, 8192, 1024);
            uint32_t it_cnt = 0, st_it = 0;
            for (int i = i_beg; i < i_end; ++i, ++it_cnt) {
                const int nsteps = warp_uniform(items[i].nsteps);
                const int kb = it_cnt & 1;
                const uint32_t kvoff = (kb * C::kTile128) >> 4;
                mbar_wait(smem_u32(&bar_kvf[kb]), (it_cnt >> 1) & 1);
                if (leader) {  // V -> TMEM, after the previous item's last dP^T (issue order)
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        tmem_cp_128x256b(tmem + kk * 8, dV0 + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4));
                    mma_commit(smem_u32(&bar_vcp));  // V is in TMEM
                    mma_commit(smem_u32(&bar_ve));   // (+ the previous epilogue's dK store)
                }
                __syncwarp();
                auto accumulate = [&](uint32_t n, int st, bool first) {
                    const int b = n & 1;
                    S2TRACE(3, n);
                    mbar_wait(smem_u32(&bar_p[b]), (n >> 1) & 1);
                    S2TRACE(4, n);
                    if (first && it_cnt > 0) {
                        S2TRACE(11, it_cnt);
                        mbar_wait(smem_u32(&bar_ae), (it_cnt - 1) & 1);
                        S2TRACE(12, it_cnt);
                    }
                    tc_fence_after();  // A operands (P^T, dS^T) were written to TMEM by tcgen05.st
                    const uint64_t dst = dStMN0 + static_cast<uint64_t>((st * C::kDkvStage) >> 4);
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < ((p.debug & 2) ? 0 : 4); ++kk) {
                            const uint32_t acc = (first && kk == 0) ? 0u : 1u;
                            // K slice kk of P^T / dS^T: WG (kk >> 1) stored it at 32*(kk>>1) + 8*(kk&1)
                            // (+16 for dS^T) of the step's S^T buffer
                            const uint32_t ac = 64 + b * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                            // dV += P^T dO ; dK += dS^T Q   (B operands MN-major)
                            mma_ts(tmem + 256, tmem + ac, dst + ((C::kTile64 + kk * 2048) >> 4), idA, acc);
                            mma_ts(tmem + 384, tmem + ac + 16, dst + ((kk * 2048) >> 4), idA, acc);
                        }
                        mma_commit(smem_u32(&bar_se[st]));
                    }
                    __syncwarp();
                };
                for (int s = 0; s < nsteps; ++s) {
                    const uint32_t n = st_it;
                    const int st = st_it % NST;
                    S2TRACE(0, n);
                    mbar_wait(smem_u32(&bar_sf[st]), (st_it / NST) & 1);
                    S2TRACE(1, n);
                    const uint64_t dst = dSt0 + static_cast<uint64_t>((st * C::kDkvStage) >> 4);
                    const int b = n & 1;
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {  // S^T = K Q^T  (K-major x K-major)
                            const uint32_t ao = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                            const uint32_t bo = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                            mma_ss(tmem + 64 + b * 64, dK0 + kvoff + ao, dst + bo, idS, kk > 0);
                        }
                    }
                    __syncwarp();
                    // dP^T(n) overwrites dP^T(n-1): the elementwise pass n-1 must have read it
                    if (n > 0) mbar_wait(smem_u32(&bar_dpf), (n - 1) & 1);
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {  // dP^T = V dO^T  (V from TMEM)
                            const uint32_t bo = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                            mma_ts(tmem + 192, tmem + kk * 8, dst + ((C::kTile64 >> 4) + bo), idS, kk > 0);
                        }
                        mma_commit(smem_u32(&bar_s[b]));
                        // K is read by the S^T MMAs only: release it after the item's
                        // last ones (the epilogue stores staged in it arrive too).
                        if (s == nsteps - 1) mma_commit(smem_u32(&bar_kve[kb]));
                    }
                    __syncwarp();
                    S2TRACE(2, n);
                    if (s > 0) accumulate(n - 1, (st_it - 1) % NST, s == 1);
                    ++st_it;
                }
                accumulate(st_it - 1, (st_it - 1) % NST, nsteps == 1);
                if (leader) mma_commit(smem_u32(&bar_af));
                __syncwarp();
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
        // -------------------------------------------------------- elementwise
        const int wg = (warp >> 2) - 1;  // column half of the 64 q columns
        const int kr = tid & 127;         // key row == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const float sl2 = p.scale_log2;
        const int cg = (kr & 63) >> 4;
        const int hk = kr >> 6;
        uint32_t it_cnt = 0, st_it = 0;
        int release = -1;  // WG leader: K buffer (and the V buffer) whose epilogue stores are in flight
        if (tid == 128) mbar_arrive(smem_u32(&bar_ve));  // no epilogue before the first item
        for (int i = i_beg; i < i_end; ++i, ++it_cnt) {
            const BwdItem it = items[i];
            const int chunk = hk ? it.c1 : it.c0;
            const int key_pos = chunk * 64 + (kr & 63);
            const bool key_ok = chunk >= 0 && key_pos < p.N;
            for (int s = 0; s < it.nsteps; ++s, ++st_it) {
                const int st = st_it % NST;
                const int b = st_it & 1;
                // lse2 / delta / meta of this stage first (shared-space vector loads,
                // broadcast), while S^T / dP^T are still being computed.  They were
                // written by a bulk copy / the producer: observe the stage barrier
                // ourselves (the stage cannot be refilled before our P arrives).
                mbar_wait(smem_u32(&bar_sf[st]), (st_it / NST) & 1);
                const uint4 meta = *reinterpret_cast<const uint4*>(gAux + st * C::kAux + kMeta);
                const uint32_t m = key_ok ? (hk ? meta.z : meta.y) : 0u;
                const uint32_t sl = sAux + st * C::kAux + wg * 128;
                const bool on0 = (m >> (wg * 8 + cg)) & 1u;
                const bool on1 = (m >> (wg * 8 + 4 + cg)) & 1u;
                const int q0 = static_cast<int>(meta.x) + wg * 32;
                float l2v[32], dlv[32];
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 a = lds_f4(sl + c * 4), d4 = lds_f4(sl + 256 + c * 4);
                    l2v[c] = a.x; l2v[c + 1] = a.y; l2v[c + 2] = a.z; l2v[c + 3] = a.w;
                    dlv[c] = d4.x; dlv[c + 1] = d4.y; dlv[c + 2] = d4.z; dlv[c + 3] = d4.w;
                }
                if (tid == 128) S2TRACE(5, st_it);
                mbar_wait(smem_u32(&bar_s[b]), (st_it >> 1) & 1);
                if (tid == 128) S2TRACE(6, st_it);
                tc_fence_after();
                if (p.debug & 1) {
                    tc_fence_before();
                    mbar_arrive(smem_u32(&bar_dpf));
                    mbar_arrive(smem_u32(&bar_p[b]));
                    continue;
                }
                uint32_t su[32], du[32];
                tmem_ld32(tmem + 64 + b * 64 + wg * 32 + lane_off, su);
                tmem_ld32(tmem + 192 + wg * 32 + lane_off, du);
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive(smem_u32(&bar_dpf));  // dP^T is in registers: the next dP^T may land
                uint32_t pk[16], dk[16];
                if (on0 && on1 && key_pos <= q0) {
                    // fully attended 32 columns, no causal cut: no per-element masking
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float p0 = fast_exp2(fmaf(__uint_as_float(su[c]), sl2, -l2v[c]));
                        const float p1 = fast_exp2(fmaf(__uint_as_float(su[c + 1]), sl2, -l2v[c + 1]));
                        pk[c >> 1] = pack_bf16(p0, p1);
                        dk[c >> 1] = pack_bf16(p0 * (__uint_as_float(du[c]) - dlv[c]),
                                               p1 * (__uint_as_float(du[c + 1]) - dlv[c + 1]));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        float pv[2], dv[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int cc = c + u;
                            const bool ok = (cc < 16 ? on0 : on1) && key_pos <= q0 + cc;
                            const float pe = fast_exp2(fmaf(__uint_as_float(su[cc]), sl2, -l2v[cc]));
                            pv[u] = ok ? pe : 0.f;
                            dv[u] = ok ? pe * (__uint_as_float(du[cc]) - dlv[cc]) : 0.f;
                        }
                        pk[c >> 1] = pack_bf16(pv[0], pv[1]);
                        dk[c >> 1] = pack_bf16(dv[0], dv[1]);
                    }
                }
                // P^T / dS^T of my 32 q columns go into the 32 S^T columns I read
                // (never into the other WG's unread columns)
                tmem_st16(tmem + 64 + b * 64 + wg * 32 + lane_off, pk);
                tmem_st16(tmem + 64 + b * 64 + wg * 32 + 16 + lane_off, dk);
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(smem_u32(&bar_p[b]));
                if (tid == 128) S2TRACE(7, st_it);
                if (release >= 0) {  // the previous item's stores read their staging long ago
                    bulk_wait_read0();
                    mbar_arrive(smem_u32(&bar_kve[release]));
                    mbar_arrive(smem_u32(&bar_ve));
                    release = -1;
                }
            }
            // ---------------------------------------------------- epilogue
            // TMEM -> registers (then the accumulators are released); dV, then dK,
            // as bf16 into the swizzled staging tile over the item's dead K tile
            // (warp group wg converts the row's 16-byte chunks [wg*D/16, (wg+1)*D/16)),
            // TMA stores (one 64 x 64 box per chunk and D/64 slice; rows past seq_len
            // are clipped by the tensor map).
            if (tid == 128) S2TRACE(8, it_cnt);
            mbar_wait(smem_u32(&bar_af), it_cnt & 1);
            if (tid == 128) S2TRACE(9, it_cnt);
            tc_fence_after();
            constexpr int kHalf = D / 2;  // columns per warp group (a multiple of 32)
            uint32_t av[kHalf], ak[kHalf];
#pragma unroll
            for (int c = 0; c < kHalf / 32; ++c) {
                tmem_ld32(tmem + 256 + wg * kHalf + c * 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(av + 32 * c));
                tmem_ld32(tmem + 384 + wg * kHalf + c * 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(ak + 32 * c));
            }
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_ae));
            const bool st_leader = tid == 128;
            if (release >= 0) {  // (an item without steps: release here at the latest)
                bulk_wait_read0();
                mbar_arrive(smem_u32(&bar_kve[release]));
                mbar_arrive(smem_u32(&bar_ve));
                release = -1;
            }
            const bool has_next = i + 1 < i_end;
            // bar_af: every MMA of the item is done, so its K tile is dead: dV is
            // staged there.  dK goes to the V buffer once the next item's V has been
            // copied into TMEM (the producer refills it only after these stores).
#pragma unroll
            for (int ph = 0; ph < 2; ++ph) {  // 0: dV, 1: dK (scaled)
                const uint32_t* acc = ph ? ak : av;
                const float mul = ph ? p.scale : 1.0f;
                const uint32_t sOut = ph ? sV : sK + (it_cnt & 1) * C::kTile128;
                const uint32_t so = sOut + hk * (C::kSub * 8192) + (kr & 63) * 128;
                if (ph == 1 && has_next) mbar_wait(smem_u32(&bar_vcp), (it_cnt + 1) & 1);
#pragma unroll
                for (int j = 0; j < D / 16; ++j) {
                    const int c = wg * (D / 16) + j;  // 16-byte chunk of the row: D/64 slice c>>3
                    const uint32_t w0 = pack_bf16(__uint_as_float(acc[8 * j]) * mul, __uint_as_float(acc[8 * j + 1]) * mul);
                    const uint32_t w1 = pack_bf16(__uint_as_float(acc[8 * j + 2]) * mul, __uint_as_float(acc[8 * j + 3]) * mul);
                    const uint32_t w2 = pack_bf16(__uint_as_float(acc[8 * j + 4]) * mul, __uint_as_float(acc[8 * j + 5]) * mul);
                    const uint32_t w3 = pack_bf16(__uint_as_float(acc[8 * j + 6]) * mul, __uint_as_float(acc[8 * j + 7]) * mul);
                    sts_u4(so + (c >> 3) * 8192 + (((c & 7) ^ (kr & 7)) << 4), w0, w1, w2, w3);
                }
                fence_proxy_async_smem();
                named_bar_sync(1, 256);
                if (st_leader) {
                    const CUtensorMap* tm = ph ? &tmdK : &tmdV;
                    for (int h = 0; h < 2; ++h) {
                        const int ch = h ? it.c1 : it.c0;
                        if (ch < 0) continue;
#pragma unroll
                        for (int sb = 0; sb < C::kSub; ++sb)
                            tma_store_3d(tm, sOut + h * (C::kSub * 8192) + sb * 8192, sb * 64, ch * 64, it.kvbh);
                    }
                    bulk_commit();
                }
            }
            if (st_leader) release = static_cast<int>(it_cnt & 1);  // arrive on bar_kve / bar_ve once read
            if (tid == 128) S2TRACE(10, it_cnt);
        }
        if (tid == 128) bulk_wait0();  // staging tiles must outlive the stores
        (void)release;
    }
    tc_fence_before();
    __syncthreads();
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x + 1] = globaltimer_ns();  // debug: CTA end
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int D>
__global__ void __launch_bounds__(384, 1)
    s2_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmdQ, const __grid_constant__ CUtensorMap /*unused*/,
                     const BwdParams p) {
    using C = BwdCfg<D>;
    constexpr int NST = C::kNSTq;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1024-B alignment
    // bar_qf / bar_qe: the Q/dO buffer holds the item's tiles / has been copied
    // into TMEM (the buffer may be refilled)
    struct Bars {
        uint64_t qf, qe, sf[NST], se[NST], s[2], p[2], af, ae;
        uint32_t tmem_base;
    };
    static_assert(sizeof(Bars) <= 256, "barrier block");
    Bars& bars = *reinterpret_cast<Bars*>(smem + 3 * C::kTile128 + NST * C::kDqStage);
    auto& bar_qf = bars.qf;
    auto& bar_qe = bars.qe;
    auto& bar_sf = bars.sf;
    auto& bar_se = bars.se;
    auto& bar_s = bars.s;
    auto& bar_p = bars.p;
    auto& bar_af = bars.af;
    auto& bar_ae = bars.ae;
    auto& tmem_base_s = bars.tmem_base;
    // Q at sQ, dO after it, the dQ staging tile after that, then the stages
    const uint32_t sQ = smem_u32(smem), sdO = sQ + C::kTile128, sOut = sQ + 2 * C::kTile128;
    const uint32_t sSt = sQ + 3 * C::kTile128;
    const FwdItem* items = static_cast<const FwdItem*>(p.items);
    const int2* chunks = static_cast<const int2*>(p.entries);

    if (tid == 0) {
        mbar_init(smem_u32(&bar_qf), 1);
        mbar_init(smem_u32(&bar_qe), 1);
        mbar_init(smem_u32(&bar_af), 1);
        mbar_init(smem_u32(&bar_ae), 256);
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_sf[i]), 1);
            mbar_init(smem_u32(&bar_se[i]), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_s[i]), 1);
            mbar_init(smem_u32(&bar_p[i]), 256);
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
    pdl_launch_dependents();
    pdl_wait();  // the previous kernel's outputs are visible from here on
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x] = globaltimer_ns();  // debug: CTA start
    // TMEM: Q at 0 and dO at 64 (the S / dP A operands, copied in with tcgen05.cp once
    // per item: the per-step MMAs then read only the 2 KB K / V slices from shared
    // memory), S[b] at 128+64b, dP[b] at 256+64b, dQ at 384.

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
        if (warp == 0 && lane == 0) {
            tma_prefetch(&tmQ);
            tma_prefetch(&tmdO);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const uint64_t keep = policy_evict_last();
            uint32_t it_cnt = 0, st_it = 0;
            for (int i = p.sched[blockIdx.x]; i < p.sched[blockIdx.x + 1]; ++i, ++it_cnt) {
                const FwdItem it = items[i];
                const int kvbh = it.bh / p.hpg;
                if (it_cnt >= 1) mbar_wait(smem_u32(&bar_qe), (it_cnt - 1) & 1);
                const uint32_t qbar = smem_u32(&bar_qf);
                mbar_expect_tx(qbar, 2 * C::kTile128);
                tma_load_rows(sQ, &tmQ, qbar, it.qtile * 128, it.bh);
                tma_load_rows(sdO, &tmdO, qbar, it.qtile * 128, it.bh);
                for (int n = 0; n < it.chunk_cnt; ++n, ++st_it) {
                    const int st = st_it % NST;
                    if (st_it >= NST) mbar_wait(smem_u32(&bar_se[st]), ((st_it / NST) + 1) & 1);
                    const uint32_t base = sSt + st * C::kDqStage;
                    const uint32_t bar = smem_u32(&bar_sf[st]);
                    const int row = chunks[it.chunk_off + n].x * 64;
                    mbar_expect_tx(bar, 2 * C::kTile64);
                    tma_load_rows_hint(base, &tmK, bar, row, kvbh, keep);
                    tma_load_rows_hint(base + C::kTile64, &tmV, bar, row, kvbh, keep);
                }
            }
        } else if (warp == 1) {
            // whole-warp issuer, elected lane (see the dK/dV kernel)
            constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0);
            constexpr uint32_t idA = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            const uint64_t dQ0 = umma_desc_sw128(sQ, 16, 1024), ddO0 = umma_desc_sw128(sdO, 16, 1024);
            const uint64_t dSt0 = umma_desc_sw128(sSt, 16, 1024);
            const uint64_t dStMN0 = umma_desc_sw128(sSt, 8192, 1024);
            uint32_t it_cnt = 0, st_it = 0, n_glob = 0;
            const int i_end = p.sched[blockIdx.x + 1];
            for (int i = p.sched[blockIdx.x]; i < i_end; ++i, ++it_cnt) {
                const int chunk_cnt = warp_uniform(items[i].chunk_cnt);
                S2TRACE(13, it_cnt);
                mbar_wait(smem_u32(&bar_qf), it_cnt & 1);
                S2TRACE(14, it_cnt);
                if (leader) {  // after the previous item's last S / dP MMAs (issue order)
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t ao = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        tmem_cp_128x256b(tmem + kk * 8, dQ0 + ao);
                        tmem_cp_128x256b(tmem + 64 + kk * 8, ddO0 + ao);
                    }
                    // Q / dO now live in TMEM: the buffer may be refilled once the copies are done
                    mma_commit(smem_u32(&bar_qe));
                }
                __syncwarp();
                bool first = true;
                auto accumulate = [&](uint32_t n, int st) {
                    const int b = n & 1;
                    S2TRACE(3, n);
                    mbar_wait(smem_u32(&bar_p[b]), (n >> 1) & 1);
                    S2TRACE(4, n);
                    if (first && it_cnt > 0) mbar_wait(smem_u32(&bar_ae), (it_cnt - 1) & 1);
                    tc_fence_after();  // A operand (dS) was written to TMEM by tcgen05.st
                    const uint64_t dst = dStMN0 + static_cast<uint64_t>((st * C::kDqStage) >> 4);
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)  // dQ += dS K  (K chunk as MN-major B)
                            mma_ts(tmem + 384, tmem + 256 + b * 64 + (kk >> 1) * 32 + (kk & 1) * 8,
                                   dst + ((kk * 2048) >> 4), idA, (first && kk == 0) ? 0u : 1u);
                        mma_commit(smem_u32(&bar_se[st]));
                    }
                    __syncwarp();
                    first = false;
                };
                int prev_st = -1;
                uint32_t prev_n = 0;
                for (int n = 0; n < chunk_cnt; ++n, ++st_it, ++n_glob) {
                    const int st = st_it % NST;
                    S2TRACE(0, n_glob);
                    mbar_wait(smem_u32(&bar_sf[st]), (st_it / NST) & 1);
                    S2TRACE(1, n_glob);
                    const uint64_t dst = dSt0 + static_cast<uint64_t>((st * C::kDqStage) >> 4);
                    const int b = n_glob & 1;
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t bo = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                            // S = Q K^T, dP = dO V^T with Q / dO from TMEM (TS)
                            mma_ts(tmem + 128 + b * 64, tmem + kk * 8, dst + bo, idS, kk > 0);
                            mma_ts(tmem + 256 + b * 64, tmem + 64 + kk * 8, dst + ((C::kTile64 >> 4) + bo), idS,
                                   kk > 0);
                        }
                        mma_commit(smem_u32(&bar_s[b]));
                    }
                    __syncwarp();
                    S2TRACE(2, n_glob);
                    if (prev_st >= 0) accumulate(prev_n, prev_st);
                    prev_st = st;
                    prev_n = n_glob;
                }
                if (prev_st >= 0) accumulate(prev_n, prev_st);
                if (leader) {
                    mma_commit(smem_u32(&bar_af));
                }
                __syncwarp();
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
        const int wg = (warp >> 2) - 1;  // key-column half of each 64-key chunk
        const int r = tid & 127;          // query row == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const float sl2 = p.scale_log2;
        uint32_t it_cnt = 0, n_glob = 0;
        for (int i = p.sched[blockIdx.x]; i < p.sched[blockIdx.x + 1]; ++i, ++it_cnt) {
            const FwdItem it = items[i];
            const int q_pos = it.qtile * 128 + r;
            const size_t lrow = static_cast<size_t>(it.bh) * p.Npad + q_pos;
            float l2, dl;
            if (p.o) {
                // fused prep (s2_bwd_prep_kernel's rule): Delta = rowsum(dO o O) over
                // this warpgroup's D/2 columns, the halves combined through shared
                // memory; rows past seq_len and rows without an admitted key get
                // lse2 = +inf, Delta = 0 (P = 0, dS finite)
                float* part = reinterpret_cast<float*>(smem + 3 * C::kTile128 + NST * C::kDqStage + 256);
                float acc = 0.f, l = -INFINITY;
                if (q_pos < p.N) {
                    const size_t off = (static_cast<size_t>(it.bh) * p.N + q_pos) * D + wg * (D / 2);
                    const uint4* a4 = reinterpret_cast<const uint4*>(p.o + off);
                    const uint4* b4 = reinterpret_cast<const uint4*>(p.dout + off);
#pragma unroll
                    for (int c = 0; c < D / 16; ++c) {
                        const uint4 a = __ldg(a4 + c), b = __ldg(b4 + c);
                        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
                        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 x = __bfloat1622float2(a2[j]), y = __bfloat1622float2(b2[j]);
                            acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
                        }
                    }
                    l = p.lse[static_cast<size_t>(it.bh) * p.N + q_pos];
                }
                part[wg * 128 + r] = acc;
                named_bar_sync(1, 256);
                const float dot = part[r] + part[128 + r];
                const bool live = l > -INFINITY;
                dl = live ? dot : 0.f;
                l2 = live ? l * 1.4426950408889634f : INFINITY;
                if (wg == 0) {
                    p.delta_w[lrow] = dl;
                    p.lse2_w[lrow] = l2;
                }
            } else {
                l2 = p.lse2[lrow];
                dl = p.delta[lrow];
            }
            const int rg = r >> 4;
            for (int n = 0; n < it.chunk_cnt; ++n, ++n_glob) {
                const int2 ch = chunks[it.chunk_off + n];
                const int b = n_glob & 1;
                if (tid == 128) S2TRACE(5, n_glob);
                mbar_wait(smem_u32(&bar_s[b]), (n_glob >> 1) & 1);
                if (tid == 128) S2TRACE(6, n_glob);
                tc_fence_after();
                uint32_t su[32], du[32];
                tmem_ld32(tmem + 128 + b * 64 + wg * 32 + lane_off, su);
                tmem_ld32(tmem + 256 + b * 64 + wg * 32 + lane_off, du);
                const uint32_t bits = (static_cast<uint32_t>(ch.y) >> (rg * 4)) & 0xFu;
                const bool on0 = (bits >> (wg * 2)) & 1u, on1 = (bits >> (wg * 2 + 1)) & 1u;
                const int k0 = ch.x * 64 + wg * 32;
                tmem_ld_wait();
                uint32_t dk[16];
                if (on0 && on1 && k0 + 31 <= q_pos) {
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float p0 = fast_exp2(fmaf(__uint_as_float(su[c]), sl2, -l2));
                        const float p1 = fast_exp2(fmaf(__uint_as_float(su[c + 1]), sl2, -l2));
                        dk[c >> 1] = pack_bf16(p0 * (__uint_as_float(du[c]) - dl),
                                               p1 * (__uint_as_float(du[c + 1]) - dl));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        float dv[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int cc = c + u;
                            const bool ok = (cc < 16 ? on0 : on1) && k0 + cc <= q_pos;
                            const float pe = fast_exp2(fmaf(__uint_as_float(su[cc]), sl2, -l2));
                            dv[u] = ok ? pe * (__uint_as_float(du[cc]) - dl) : 0.f;
                        }
                        dk[c >> 1] = pack_bf16(dv[0], dv[1]);
                    }
                }
                tmem_st16(tmem + 256 + b * 64 + wg * 32 + lane_off, dk);  // own columns only
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(smem_u32(&bar_p[b]));
                if (tid == 128) S2TRACE(7, n_glob);
            }
            mbar_wait(smem_u32(&bar_af), it_cnt & 1);
            tc_fence_after();
            // TMEM -> registers (accumulator released), bf16 into the swizzled
            // staging tile, TMA store of the 128 x D tile (rows past seq_len clipped)
            uint32_t acc[D / 2];
#pragma unroll
            for (int c = 0; c < D / 64; ++c)
                tmem_ld32(tmem + 384 + wg * (D / 2) + c * 32 + lane_off,
                          *reinterpret_cast<uint32_t(*)[32]>(acc + 32 * c));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_ae));
            // the previous item's store has read the staging tile (long ago)
            if (tid == 128) bulk_wait_read0();
            named_bar_sync(1, 256);
            const float sc = it.chunk_cnt > 0 ? p.scale : 0.f;  // no chunks: dQ = 0
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {  // my 16-byte chunks: global chunk index g
                const int g = wg * (D / 16) + c;
                const uint32_t w0 = pack_bf16(__uint_as_float(acc[8 * c]) * sc, __uint_as_float(acc[8 * c + 1]) * sc);
                const uint32_t w1 = pack_bf16(__uint_as_float(acc[8 * c + 2]) * sc, __uint_as_float(acc[8 * c + 3]) * sc);
                const uint32_t w2 = pack_bf16(__uint_as_float(acc[8 * c + 4]) * sc, __uint_as_float(acc[8 * c + 5]) * sc);
                const uint32_t w3 = pack_bf16(__uint_as_float(acc[8 * c + 6]) * sc, __uint_as_float(acc[8 * c + 7]) * sc);
                sts_u4(sOut + (g >> 3) * 16384 + r * 128 + (((g & 7) ^ (r & 7)) << 4), w0, w1, w2, w3);
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 256);
            if (tid == 128) {
#pragma unroll
                for (int sb = 0; sb < C::kSub; ++sb)
                    tma_store_3d(&tmdQ, sOut + sb * 16384, sb * 64, it.qtile * 128, it.bh);
                bulk_commit();
            }
        }
        if (tid == 128) bulk_wait0();  // the staging tile must outlive the store
    }
    tc_fence_before();
    __syncthreads();
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x + 1] = globaltimer_ns();  // debug: CTA end
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------- dQ, 128-key steps
// One CTA owns a 128-row query tile and walks its chunk list two chunks (128
// keys) per step, so S = Q K^T and dP = dO V^T are M=128 x N=128 MMAs (an
// N=64 MMA has a ~45-cycle floor against 32 ideal; N=128 runs at the full
// rate).  TMEM holds Q and dO (the TS A operands, copied in once per item),
// ONE S, ONE dP and the dQ accumulator: 64+64+128+128+128 = 512 columns, so
// S and dP are single-buffered and the overlap comes from the issue order of
// the single MMA warp, which the tensor pipe executes in order:
//     S(n+1) | dQ(n) += dS(n) K(n) | dP(n+1)
// S(n+1) needs only that the elementwise warps have READ S(n); dP(n+1)
// overwrites the dS(n) that dQ(n) reads, which is safe because it is issued
// after it.  The elementwise pass of step n (exp, dS) thus runs while the pipe
// computes dP(n) and S(n+1).  A third warpgroup drains the dQ accumulator and
// stores it, so item boundaries do not stall the elementwise warps.
//
// Warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue,
// 8-11 / 12-15 elementwise (thread = query row = TMEM lane; warpgroup w owns
// the 64 keys of chunk w of each step).  Shared memory (D = 128): Q | dO |
// dQ staging (32 KB each) | 2 stages of K (128 keys) | V (128 keys).
template <int D>
struct Dq2Cfg {
    static constexpr int kSub = D / 64;
    static constexpr int kTile = kSub * 16384;  // 128 rows x D bf16, [D/64][128][64] SW128
    static constexpr int kNST = D == 128 ? 2 : 4;
    static constexpr int kStage = 2 * kTile;  // K rows 0..127 (chunk h at +h*8 KB per slice) | V
    static constexpr int kBars = 512;
    static constexpr int kSmem = 3 * kTile + kNST * kStage + kBars;
    // TMEM columns
    static constexpr uint32_t tQ = 0, tdO = D / 2, tS = D, tdP = D + 128, tAcc = D + 256;
};

template <int D>
__global__ void __launch_bounds__(512, 1)
    s2_bwd_dq2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                      const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmdQ, const __grid_constant__ CUtensorMap /*unused*/,
                      const BwdParams p) {
    using C = Dq2Cfg<D>;
    constexpr int NST = C::kNST;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1024-B alignment
    // qf / qe: the Q/dO buffer holds the item's tiles / has been copied into TMEM.
    // kvf / kve: K/V stage full / free (after the step's dQ MMA).
    // sf: S in TMEM; sfr: the elementwise warps have read S (S may be overwritten);
    // dpf: dP in TMEM; dsf: dS written over dP; af / ae: dQ accumulator full / drained.
    struct Bars {
        uint64_t qf, qe, kvf[NST], kve[NST], sf, sfr, dpf, dsf, af, ae;
        uint32_t tmem_base;
    };
    static_assert(sizeof(Bars) <= C::kBars, "barrier block");
    Bars& bars = *reinterpret_cast<Bars*>(smem + 3 * C::kTile + NST * C::kStage);
    const uint32_t sQ = smem_u32(smem), sdO = sQ + C::kTile, sOut = sQ + 2 * C::kTile;
    const uint32_t sSt = sQ + 3 * C::kTile;
    const FwdItem* items = static_cast<const FwdItem*>(p.items);
    const int2* chunks = static_cast<const int2*>(p.entries);
    const int i_beg = p.sched[blockIdx.x], i_end = p.sched[blockIdx.x + 1];

    if (tid == 0) {
        mbar_init(smem_u32(&bars.qf), 1);
        mbar_init(smem_u32(&bars.qe), 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bars.kvf[i]), 1);
            mbar_init(smem_u32(&bars.kve[i]), 1);
        }
        mbar_init(smem_u32(&bars.sf), 1);
        mbar_init(smem_u32(&bars.sfr), 256);
        mbar_init(smem_u32(&bars.dpf), 1);
        mbar_init(smem_u32(&bars.dsf), 256);
        mbar_init(smem_u32(&bars.af), 1);
        mbar_init(smem_u32(&bars.ae), 128);
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc(smem_u32(&bars.tmem_base), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    pdl_launch_dependents();
    pdl_wait();  // the previous kernel's outputs are visible from here on
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x] = globaltimer_ns();  // debug: CTA start

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
        if (warp == 0 && lane == 0) {
            // ---------------------------------------------------------- producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmdO);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const uint64_t keep = policy_evict_last();
            uint32_t g = 0, qc = 0;
            for (int i = i_beg; i < i_end; ++i) {
                const FwdItem it = items[i];
                if (it.chunk_cnt == 0) continue;
                const int kvbh = it.bh / p.hpg;
                if (qc >= 1) mbar_wait(smem_u32(&bars.qe), (qc - 1) & 1);
                const uint32_t qbar = smem_u32(&bars.qf);
                mbar_expect_tx(qbar, 2 * C::kTile);
                tma_load_rows(sQ, &tmQ, qbar, it.qtile * 128, it.bh);
                tma_load_rows(sdO, &tmdO, qbar, it.qtile * 128, it.bh);
                ++qc;
                const int nsteps = (it.chunk_cnt + 1) / 2;
                for (int n = 0; n < nsteps; ++n, ++g) {
                    const int st = g % NST;
                    if (g >= NST) mbar_wait(smem_u32(&bars.kve[st]), ((g / NST) + 1) & 1);
                    const int nch = 2 * n + 1 < it.chunk_cnt ? 2 : 1;
                    const uint32_t base = sSt + st * C::kStage;
                    const uint32_t bar = smem_u32(&bars.kvf[st]);
                    mbar_expect_tx(bar, nch * 2 * C::kSub * 8192);
                    for (int h = 0; h < nch; ++h) {
                        const int row = chunks[it.chunk_off + 2 * n + h].x * 64;
                        for (int s = 0; s < C::kSub; ++s) {
                            tma_load_3d_hint(base + s * 16384 + h * 8192, &tmK, bar, s * 64, row, kvbh, keep);
                            tma_load_3d_hint(base + C::kTile + s * 16384 + h * 8192, &tmV, bar, s * 64, row, kvbh,
                                             keep);
                        }
                    }
                }
            }
        } else if (warp == 1) {
            // -------------------------------------------------------- MMA issuer
            // whole warp on warp-uniform values, one elected lane issues
            constexpr uint32_t idS128 = umma_idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idS64 = umma_idesc_bf16(128, 64, 0, 0);
            constexpr uint32_t idQ = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            const uint64_t dQs = umma_desc_sw128(sQ, 16, 1024), ddOs = umma_desc_sw128(sdO, 16, 1024);
            const uint64_t dK0 = umma_desc_sw128(sSt, 16, 1024);            // K-major K (B of S)
            const uint64_t dV0 = umma_desc_sw128(sSt + C::kTile, 16, 1024);  // K-major V (B of dP)
            const uint64_t dKmn = umma_desc_sw128(sSt, 16384, 1024);         // MN-major K (B of dQ)
            uint32_t g = 0, qc = 0, ac = 0;
            bool pend = false, pfirst = false, plast = false;
            uint32_t pg = 0, pst = 0, pnk = 0, pac = 0;
            // dQ(pg) += dS(pg) K(pg): once the elementwise warps wrote dS (and, for an
            // item's first step, the epilogue drained the previous item's accumulator)
            auto issue_dq = [&]() {
                S2TRACE(3, pg);
                mbar_wait(smem_u32(&bars.dsf), pg & 1);
                if (pfirst && pac > 0) mbar_wait(smem_u32(&bars.ae), (pac - 1) & 1);
                S2TRACE(4, pg);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = dKmn + static_cast<uint64_t>((pst * C::kStage) >> 4);
                    for (uint32_t kk = 0; kk < pnk / 16; ++kk)
                        mma_ts(tmem + C::tAcc, tmem + C::tdP + (kk >> 2) * 64 + (kk & 3) * 8,
                               b0 + ((kk * 2048) >> 4), idQ, (pfirst && kk == 0) ? 0u : 1u);
                    mma_commit(smem_u32(&bars.kve[pst]));
                    if (plast) mma_commit(smem_u32(&bars.af));
                }
                __syncwarp();
            };
            for (int i = i_beg; i < i_end; ++i) {
                const int cnt = warp_uniform(items[i].chunk_cnt);
                if (cnt == 0) continue;
                mbar_wait(smem_u32(&bars.qf), qc & 1);
                if (leader) {  // Q / dO -> TMEM, after every earlier S / dP MMA (issue order)
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t ao = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        tmem_cp_128x256b(tmem + C::tQ + kk * 8, dQs + ao);
                        tmem_cp_128x256b(tmem + C::tdO + kk * 8, ddOs + ao);
                    }
                    mma_commit(smem_u32(&bars.qe));  // the buffer may be refilled once copied
                }
                __syncwarp();
                ++qc;
                const int nsteps = (cnt + 1) / 2;
                for (int n = 0; n < nsteps; ++n, ++g) {
                    const uint32_t st = g % NST;
                    const bool two = 2 * n + 1 < cnt;
                    const uint32_t idS = two ? idS128 : idS64;
                    S2TRACE(0, g);
                    mbar_wait(smem_u32(&bars.kvf[st]), (g / NST) & 1);
                    S2TRACE(8, g);
                    if (g > 0) mbar_wait(smem_u32(&bars.sfr), (g - 1) & 1);
                    S2TRACE(1, g);
                    tc_fence_after();
                    const uint64_t so = static_cast<uint64_t>((st * C::kStage) >> 4);
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {  // S = Q K^T (Q from TMEM)
                            const uint32_t bo = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                            mma_ts(tmem + C::tS, tmem + C::tQ + kk * 8, dK0 + so + bo, idS, kk > 0);
                        }
                        mma_commit(smem_u32(&bars.sf));
                    }
                    __syncwarp();
                    if (pend) issue_dq();
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {  // dP = dO V^T (dO from TMEM)
                            const uint32_t bo = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                            mma_ts(tmem + C::tdP, tmem + C::tdO + kk * 8, dV0 + so + bo, idS, kk > 0);
                        }
                        mma_commit(smem_u32(&bars.dpf));
                    }
                    __syncwarp();
                    S2TRACE(2, g);
                    pend = true;
                    pg = g;
                    pst = st;
                    pnk = two ? 128 : 64;
                    pfirst = n == 0;
                    plast = n == nsteps - 1;
                    pac = ac;
                }
                ++ac;
            }
            if (pend) issue_dq();
        }
    } else if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 120;" ::: "memory");
        // ---------------------------------------------------------------- epilogue
        // TMEM -> registers as bf16 (the accumulator is released as soon as it is
        // read), x scale, into the swizzled staging tile, TMA store of the 128 x D
        // tile (rows past seq_len clipped by the tensor map).
        const int r = tid & 127;
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const bool st_leader = tid == 128;
        uint32_t ac = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const FwdItem it = items[i];
            uint32_t pk[D / 2];
            if (it.chunk_cnt > 0) {
                mbar_wait(smem_u32(&bars.af), ac & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t u[32];
                    tmem_ld32(tmem + C::tAcc + c * 32 + lane_off, u);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        pk[c * 16 + j] = pack_bf16(__uint_as_float(u[2 * j]) * p.scale,
                                                   __uint_as_float(u[2 * j + 1]) * p.scale);
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&bars.ae));
                ++ac;
            } else {  // no chunk: dQ = 0
#pragma unroll
                for (int j = 0; j < D / 2; ++j) pk[j] = 0u;
            }
            if (st_leader) bulk_wait_read0();  // the previous store has read the staging tile
            named_bar_sync(1, 128);
#pragma unroll
            for (int c = 0; c < D / 8; ++c)  // 16-byte chunk c of the row: D/64 slice c >> 3
                sts_u4(sOut + (c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4), pk[4 * c],
                       pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (st_leader) {
#pragma unroll
                for (int sb = 0; sb < C::kSub; ++sb)
                    tma_store_3d(&tmdQ, sOut + sb * 16384, sb * 64, it.qtile * 128, it.bh);
                bulk_commit();
            }
        }
        if (st_leader) bulk_wait0();  // the staging tile must outlive the store
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;" ::: "memory");
        // ------------------------------------------------------------- elementwise
        const int w = (warp >> 2) - 2;  // chunk w of each step (its 64 keys)
        const int r = tid & 127;        // query row == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + C::tS + 64 * w + lane_off, tdP = tmem + C::tdP + 64 * w + lane_off;
        const float sl2 = p.scale_log2;
        const int rg = r >> 4;
        uint32_t g = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const FwdItem it = items[i];
            if (it.chunk_cnt == 0) continue;
            const int q_pos = it.qtile * 128 + r;
            const size_t lrow = static_cast<size_t>(it.bh) * p.Npad + q_pos;
            const float l2 = p.lse2[lrow];  // +inf / 0 for rows without keys (prep)
            const float dl = p.delta[lrow];
            const int nsteps = (it.chunk_cnt + 1) / 2;
            for (int n = 0; n < nsteps; ++n, ++g) {
                const int idx = 2 * n + w;
                const bool has = idx < it.chunk_cnt;
                const int2 ch = has ? chunks[it.chunk_off + idx] : make_int2(0, 0);
                if (tid == 256) S2TRACE(5, g);
                mbar_wait(smem_u32(&bars.sf), g & 1);
                if (tid == 256) S2TRACE(6, g);
                tc_fence_after();
                float sv[64];
                if (has) {
                    tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(sv));
                    tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
                    tmem_ld_wait();
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&bars.sfr));  // S may be overwritten by S(n+1)
                if (has) {
                    const uint32_t bits = (static_cast<uint32_t>(ch.y) >> (rg * 4)) & 0xFu;
                    const int k0 = ch.x * 64;
                    if (bits == 0xFu && k0 + 63 <= q_pos) {
#pragma unroll
                        for (int j = 0; j < 64; ++j) sv[j] = fast_exp2(fmaf(sv[j], sl2, -l2));
                    } else {
#pragma unroll
                        for (int j = 0; j < 64; ++j) {
                            const bool ok = ((bits >> (j >> 4)) & 1u) && k0 + j <= q_pos;
                            const float pe = fast_exp2(fmaf(sv[j], sl2, -l2));
                            sv[j] = ok ? pe : 0.f;
                        }
                    }
                }
                mbar_wait(smem_u32(&bars.dpf), g & 1);
                tc_fence_after();
                if (has) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t du[32], dk[16];
                        tmem_ld32(tdP + h * 32, du);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 32; c += 2)
                            dk[c >> 1] = pack_bf16(sv[h * 32 + c] * (__uint_as_float(du[c]) - dl),
                                                   sv[h * 32 + c + 1] * (__uint_as_float(du[c + 1]) - dl));
                        // dS of keys [32h, 32h+32) into columns [16h, 16h+16) of my dP
                        // region: columns this thread has already read
                        tmem_st16(tdP + h * 16, dk);
                    }
                    tmem_st_wait();
                }
                tc_fence_before();
                mbar_arrive(smem_u32(&bars.dsf));
                if (tid == 256) S2TRACE(7, g);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x + 1] = globaltimer_ns();  // debug: CTA end
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------- dK/dV, 128-row q steps
// One CTA owns a 128-key tile (two 64-key chunks) of one kv head and walks its
// transposed list one 128-row q tile per step, so S^T = K Q^T and dP^T = V dO^T
// are M=128 x N=128 MMAs (full rate; the 64-row steps of s2_bwd_dkv_kernel are
// N=64, ~45 cycles against 32).  TMEM: two 128-column step regions and the dV,
// dK accumulators (512 columns).  Step n owns region n & 1 for its whole life:
// S^T(n) lands there; once the elementwise warps have read it, dP^T(n) is
// computed over it; they read dP^T(n) and write dS^T(n) and P^T(n) (bf16)
// back into the same columns, which dV(n) and dK(n) then consume.  The single
// MMA warp issues, per step n,
//     S^T(n+1) | dV(n) += P^T(n) dO(n) | dP^T(n+1) | dK(n) += dS^T(n) Q(n)
// and the tensor pipe executes them in order, so S^T(n+1) overwrites region
// (n+1)&1 only after dV(n-1), dK(n-1) read it, the exponentials of step n+1
// run while the pipe computes dV(n), dP^T(n+1), dK(n), and dP^T(n+1) is ready
// before they end.  K and V stay in shared memory (SS MMAs), single-buffered:
// K is free after an item's last S^T, one step before the next item's first
// S^T needs the next K (V likewise).  Q (3 slots), dO (2 slots) and lse2 /
// delta (2 slots) stream in rings sized to the issue order: Q(n) is last read
// by dK(n), dO(n) by dV(n).  A fourth warpgroup drains dV / dK from TMEM and
// stores them (row stores; no shared memory is left for a staging tile).  No
// atomics: deterministic.
//
// Warps (768 threads): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7
// epilogue, 8-23 elementwise: four warpgroups (thread = key row = TMEM lane;
// warpgroup w owns q columns [32w, 32w+32) of each step), so each SMSP holds
// four elementwise warps to hide the exp / TMEM latencies of the others.
#ifndef S2_DKV2_ALT
#define S2_DKV2_ALT 0
#endif
// MMA issue order: 2 = dP^T-first (default), 0 = S^T-first (the original order).
// (Two issuers, and a dynamic choice between dP^T and the previous step's dV / dK,
// measured slower: DESIGN.md section 7.)
#ifndef S2_DKV2_SPLIT
#define S2_DKV2_SPLIT 2
#endif
template <int D>
struct Dkv2Cfg {
    static constexpr int kSub = D / 64;
    static constexpr int kT = kSub * 16384;  // 128 rows x D bf16: [D/64][128][64] SW128
    static constexpr int kNQ = 3, kNO = 2, kNA = 2;
    static constexpr int kAux = 1024;  // lse2[128] | delta[128]
    static constexpr int kBars = 512;
    static constexpr int kSmem = (2 + kNQ + kNO) * kT + kNA * kAux + kBars;
    static constexpr uint32_t tR = 0, tdV = 256, tdK = 256 + D;  // step regions at tR + 128 * (n & 1)
};

template <int D>
__global__ void __launch_bounds__(768, 1)
    s2_bwd_dkv2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                       const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ CUtensorMap /*unused*/, const __grid_constant__ CUtensorMap /*unused*/,
                       const BwdParams p) {
    using C = Dkv2Cfg<D>;
    constexpr int NQ = C::kNQ, NO = C::kNO, NA = C::kNA;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1024-B alignment
    struct Bars {
        uint64_t kf, vf, kfree, vfree, qf[NQ], qe[NQ], of[NO], oe[NO], af[NA], ae[NA];
        uint64_t sf, sfr, dpf, pds, accf, acce;
        uint4 meta[NA];  // per aux slot: first q row, chunk-0 / chunk-1 masks, query data index
        uint32_t tmem_base;
    };
    static_assert(sizeof(Bars) <= C::kBars, "barrier block");
    const uint32_t sK = smem_u32(smem), sV = sK + C::kT, sQ0 = sK + 2 * C::kT;
    const uint32_t sdO0 = sQ0 + NQ * C::kT, sAux = sdO0 + NO * C::kT;
    Bars& bars = *reinterpret_cast<Bars*>(smem + (sAux - sK) + NA * C::kAux);
    const BwdItem* items = static_cast<const BwdItem*>(p.items);
    const BwdEntry* ents = static_cast<const BwdEntry*>(p.entries);
    const int i_beg = p.sched[blockIdx.x], i_end = p.sched[blockIdx.x + 1];

    if (tid == 0) {
        mbar_init(smem_u32(&bars.kf), 1);
        mbar_init(smem_u32(&bars.vf), 1);
        mbar_init(smem_u32(&bars.kfree), 1);
        mbar_init(smem_u32(&bars.vfree), 1);
        for (int i = 0; i < NQ; ++i) {
            mbar_init(smem_u32(&bars.qf[i]), 1);
            mbar_init(smem_u32(&bars.qe[i]), 1);
        }
        for (int i = 0; i < NO; ++i) {
            mbar_init(smem_u32(&bars.of[i]), 1);
            mbar_init(smem_u32(&bars.oe[i]), 1);
        }
        for (int i = 0; i < NA; ++i) {
            mbar_init(smem_u32(&bars.af[i]), 1);
            mbar_init(smem_u32(&bars.ae[i]), 16);
        }
        mbar_init(smem_u32(&bars.sf), 1);
        mbar_init(smem_u32(&bars.sfr), 16);  // one arrival per elementwise warp
        mbar_init(smem_u32(&bars.dpf), 1);
        mbar_init(smem_u32(&bars.pds), 16);
        mbar_init(smem_u32(&bars.accf), 1);
        mbar_init(smem_u32(&bars.acce), 4);
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc(smem_u32(&bars.tmem_base), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    pdl_launch_dependents();
    pdl_wait();  // the previous kernel's outputs are visible from here on
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x] = globaltimer_ns();  // debug: CTA start
    const int nchunk_pad = (p.N + 63) / 64 * 64;  // a row coordinate past the tensor: TMA fills zeros

    if (warp < 4) {
        // registers: 768 threads launch with 80 each (61440); 40 + 48 + 4 x 96 per
        // warpgroup fits that pool (setmaxnreg.inc blocks until the pool has them)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
        if (warp == 0 && lane == 0) {
            // ---------------------------------------------------------- producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmdO);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            uint32_t ic = 0, g = 0;
            for (int i = i_beg; i < i_end; ++i) {
                const BwdItem it = items[i];
                if (it.nsteps128 == 0) continue;
                // K, V tiles: chunk h of the pair in rows [64h, 64h+64) of every D/64 slice
                // (a missing second chunk reads past the tensor: zeros)
                const int r0 = it.c0 * 64, r1 = it.c1 >= 0 ? it.c1 * 64 : nchunk_pad;
                if (ic >= 1) mbar_wait(smem_u32(&bars.kfree), (ic - 1) & 1);
                mbar_expect_tx(smem_u32(&bars.kf), C::kT);
                for (int s = 0; s < C::kSub; ++s) {
                    tma_load_3d(sK + s * 16384, &tmK, smem_u32(&bars.kf), s * 64, r0, it.kvbh);
                    tma_load_3d(sK + s * 16384 + 8192, &tmK, smem_u32(&bars.kf), s * 64, r1, it.kvbh);
                }
                if (ic >= 1) mbar_wait(smem_u32(&bars.vfree), (ic - 1) & 1);
                mbar_expect_tx(smem_u32(&bars.vf), C::kT);
                for (int s = 0; s < C::kSub; ++s) {
                    tma_load_3d(sV + s * 16384, &tmV, smem_u32(&bars.vf), s * 64, r0, it.kvbh);
                    tma_load_3d(sV + s * 16384 + 8192, &tmV, smem_u32(&bars.vf), s * 64, r1, it.kvbh);
                }
                ++ic;
                for (int j = 0; j < p.hpg; ++j) {
                    const int qbh = it.kvbh * p.hpg + j;
                    // q tiles descending (as s2_bwd_dkv_kernel: tiles of one head running
                    // together meet on the same Q / dO rows in L2)
                    for (int e = it.count - 1; e >= 0; --e) {
                        const BwdEntry en = ents[it.offset + e];
                        if ((en.mask0 | en.mask1) == 0) continue;
                        const int row0 = en.qtile * 128;
                        const int qs = g % NQ, os = g % NO, as = g % NA;
                        if (g >= NQ) mbar_wait(smem_u32(&bars.qe[qs]), ((g / NQ) + 1) & 1);
                        mbar_expect_tx(smem_u32(&bars.qf[qs]), C::kT);
                        tma_load_rows(sQ0 + qs * C::kT, &tmQ, smem_u32(&bars.qf[qs]), row0, qbh);
                        if (g >= NA) mbar_wait(smem_u32(&bars.ae[as]), ((g / NA) + 1) & 1);
                        bars.meta[as] = make_uint4(static_cast<uint32_t>(row0), en.mask0, en.mask1,
                                                   static_cast<uint32_t>(qbh));
                        mbar_expect_tx(smem_u32(&bars.af[as]), 1024);
                        const size_t lo = static_cast<size_t>(qbh) * p.Npad + row0;
                        bulk_load(sAux + as * C::kAux, p.lse2 + lo, 512, smem_u32(&bars.af[as]));
                        bulk_load(sAux + as * C::kAux + 512, p.delta + lo, 512, smem_u32(&bars.af[as]));
                        if (g >= NO) mbar_wait(smem_u32(&bars.oe[os]), ((g / NO) + 1) & 1);
                        mbar_expect_tx(smem_u32(&bars.of[os]), C::kT);
                        tma_load_rows(sdO0 + os * C::kT, &tmdO, smem_u32(&bars.of[os]), row0, qbh);
                        ++g;
                    }
                }
            }
        } else if (warp == 1 && S2_DKV2_SPLIT == 2) {
            // ---------------------------------- MMA issuer, dP^T-first order (default)
            // Per step g:  dP^T(g) | dV(g-1) | dK(g-1) | S^T(g+1).  dP^T(g) goes to the
            // pipe as soon as the elementwise warps have read S^T(g), ahead of the
            // previous step's dV / dK, so it completes while they exponentiate; S^T(g+1)
            // overwrites region (g+1)&1 right after dK(g-1) read it (in-order pipe).
            constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idA = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            const uint64_t dK0 = umma_desc_sw128(sK, 16, 1024), dV0 = umma_desc_sw128(sV, 16, 1024);
            const uint64_t dQ0 = umma_desc_sw128(sQ0, 16, 1024), ddO0 = umma_desc_sw128(sdO0, 16, 1024);
            const uint64_t dQmn = umma_desc_sw128(sQ0, 16384, 1024), ddOmn = umma_desc_sw128(sdO0, 16384, 1024);
            auto issue_s = [&](uint32_t gs, bool first, bool last, uint32_t ic) {
                const uint32_t qs = gs % NQ;
                mbar_wait(smem_u32(&bars.qf[qs]), (gs / NQ) & 1);
                if (first) mbar_wait(smem_u32(&bars.kf), ic & 1);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = dQ0 + static_cast<uint64_t>((qs * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        mma_ss(tmem + C::tR + 128 * (gs & 1), dK0 + o, b0 + o, idS, kk > 0);
                    }
                    mma_commit(smem_u32(&bars.sf));
                    if (last) mma_commit(smem_u32(&bars.kfree));
                }
                __syncwarp();
            };
            auto issue_dp = [&](uint32_t gs, bool first, bool last, uint32_t ic) {
                const uint32_t os = gs % NO;
                mbar_wait(smem_u32(&bars.of[os]), (gs / NO) & 1);
                if (first) mbar_wait(smem_u32(&bars.vf), ic & 1);
                mbar_wait(smem_u32(&bars.sfr), gs & 1);
                S2TRACE(13, gs);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = ddO0 + static_cast<uint64_t>((os * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        mma_ss(tmem + C::tR + 128 * (gs & 1), dV0 + o, b0 + o, idS, kk > 0);
                    }
                    mma_commit(smem_u32(&bars.dpf));
                    if (last) mma_commit(smem_u32(&bars.vfree));
                }
                __syncwarp();
            };
            auto issue_acc = [&](uint32_t gs, bool first, bool last, uint32_t ic) {
                mbar_wait(smem_u32(&bars.pds), gs & 1);  // P^T(gs), dS^T(gs) in TMEM
                if (first && ic > 0) mbar_wait(smem_u32(&bars.acce), (ic - 1) & 1);
                S2TRACE(2, gs);
                tc_fence_after();
                const uint32_t reg = C::tR + 128 * (gs & 1);
                const uint32_t os = gs % NO, qs = gs % NQ;
                if (leader) {
                    const uint64_t bo = ddOmn + static_cast<uint64_t>((os * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)  // K-dim: the step's 128 q rows; P^T at +16
                        mma_ts(tmem + C::tdV, tmem + reg + (kk >> 1) * 32 + 16 + (kk & 1) * 8,
                               bo + ((kk * 2048) >> 4), idA, (!first || kk > 0) ? 1u : 0u);
                    mma_commit(smem_u32(&bars.oe[os]));  // dO(gs) read (dP^T(gs), dV(gs))
                    const uint64_t bq = dQmn + static_cast<uint64_t>((qs * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)  // dS^T at +0
                        mma_ts(tmem + C::tdK, tmem + reg + (kk >> 1) * 32 + (kk & 1) * 8,
                               bq + ((kk * 2048) >> 4), idA, (!first || kk > 0) ? 1u : 0u);
                    mma_commit(smem_u32(&bars.qe[qs]));  // Q(gs) read (S^T(gs), dK(gs))
                    if (last) mma_commit(smem_u32(&bars.accf));
                }
                __syncwarp();
                S2TRACE(3, gs);
            };
            // the previous step's (first, last, item index) for its dV / dK
            bool p_first = false, p_last = false, have_prev = false;
            uint32_t p_ic = 0, g = 0, ic = 0;
            int i = i_beg;
            while (i < i_end && warp_uniform(items[i].nsteps128) == 0) ++i;
            if (i < i_end) {
                int ns = warp_uniform(items[i].nsteps128);
                issue_s(0, true, ns == 1, 0);
                while (true) {
                    for (int n = 0; n < ns; ++n, ++g) {
                        S2TRACE(0, g);
                        issue_dp(g, n == 0, n == ns - 1, ic);
                        if (have_prev) issue_acc(g - 1, p_first, p_last, p_ic);
                        // the next step: n+1 of this item, or the first of the next item
                        int ni = i, nn = n + 1, nns = ns;
                        uint32_t nic = ic;
                        if (nn == ns) {
                            ni = i + 1;
                            while (ni < i_end && warp_uniform(items[ni].nsteps128) == 0) ++ni;
                            nn = 0;
                            nic = ic + 1;
                            nns = ni < i_end ? warp_uniform(items[ni].nsteps128) : 0;
                        }
                        if (ni < i_end) issue_s(g + 1, nn == 0, nn == nns - 1, nic);
                        S2TRACE(1, g);
                        have_prev = true;
                        p_first = n == 0;
                        p_last = n == ns - 1;
                        p_ic = ic;
                    }
                    ++ic;
                    ++i;
                    while (i < i_end && warp_uniform(items[i].nsteps128) == 0) ++i;
                    if (i >= i_end) break;
                    ns = warp_uniform(items[i].nsteps128);
                }
                issue_acc(g - 1, p_first, p_last, p_ic);
            }
        } else if (warp == 1) {  // single issuer (S2_DKV2_SPLIT=0)
            // -------------------------------------------------------- MMA issuer
            constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);
            constexpr uint32_t idA = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            const uint64_t dK0 = umma_desc_sw128(sK, 16, 1024), dV0 = umma_desc_sw128(sV, 16, 1024);
            const uint64_t dQ0 = umma_desc_sw128(sQ0, 16, 1024), ddO0 = umma_desc_sw128(sdO0, 16, 1024);
            const uint64_t dQmn = umma_desc_sw128(sQ0, 16384, 1024), ddOmn = umma_desc_sw128(sdO0, 16384, 1024);
            // S^T(g) = K Q(g)^T / dP^T(g) = V dO(g)^T; `first` / `last`: the step opens /
            // closes its item (ic: the item's index among this CTA's items)
            auto issue_s = [&](uint32_t g, bool first, bool last, uint32_t ic) {
                const uint32_t qs = g % NQ;
                mbar_wait(smem_u32(&bars.qf[qs]), (g / NQ) & 1);
                if (first) mbar_wait(smem_u32(&bars.kf), ic & 1);
                S2TRACE(4, g - 1);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = dQ0 + static_cast<uint64_t>((qs * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        mma_ss(tmem + C::tR + 128 * (g & 1), dK0 + o, b0 + o, idS, kk > 0);
                    }
                    mma_commit(smem_u32(&bars.sf));
                    if (last) mma_commit(smem_u32(&bars.kfree));  // the item's K is read by S^T only
                }
                __syncwarp();
            };
            // dP^T(g) over S^T(g) in region g & 1, once the elementwise warps have read S^T(g)
            auto issue_dp = [&](uint32_t g, bool first, bool last, uint32_t ic) {
                const uint32_t os = g % NO;
                mbar_wait(smem_u32(&bars.of[os]), (g / NO) & 1);
                if (first) mbar_wait(smem_u32(&bars.vf), ic & 1);
                mbar_wait(smem_u32(&bars.sfr), g & 1);
                S2TRACE(13, g - 1);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = ddO0 + static_cast<uint64_t>((os * C::kT) >> 4);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t o = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        mma_ss(tmem + C::tR + 128 * (g & 1), dV0 + o, b0 + o, idS, kk > 0);
                    }
                    mma_commit(smem_u32(&bars.dpf));
                    if (last) mma_commit(smem_u32(&bars.vfree));  // V is read by dP^T only
                }
                __syncwarp();
            };
            // first item with steps
            int i = i_beg;
            while (i < i_end && warp_uniform(items[i].nsteps128) == 0) ++i;
            if (i < i_end) {
                int ns = warp_uniform(items[i].nsteps128);
                uint32_t g = 0, ic = 0;
                issue_s(0, true, ns == 1, 0);
                issue_dp(0, true, ns == 1, 0);  // (waits for the elementwise warps to read S^T(0))
                while (true) {
                    for (int n = 0; n < ns; ++n, ++g) {
                        // the step after g: n+1 of this item, or the first of the next item
                        bool has_next = true, nfirst = false;
                        int nns = ns, ni = i;
                        if (n + 1 == ns) {
                            ni = i + 1;
                            while (ni < i_end && warp_uniform(items[ni].nsteps128) == 0) ++ni;
                            has_next = ni < i_end;
                            nfirst = true;
                            nns = has_next ? warp_uniform(items[ni].nsteps128) : 0;
                        }
                        const int nn = nfirst ? 0 : n + 1;
                        const uint32_t nic = nfirst ? ic + 1 : ic;
                        const bool nlast = nn == nns - 1;
                        S2TRACE(0, g);
                        if (has_next) issue_s(g + 1, nfirst, nlast, nic);  // region (g+1)&1: dK(g-1) read it
                        S2TRACE(1, g);
                        mbar_wait(smem_u32(&bars.pds), g & 1);  // P^T(g), dS^T(g) in TMEM
                        if (n == 0 && ic > 0) mbar_wait(smem_u32(&bars.acce), (ic - 1) & 1);
                        S2TRACE(2, g);
                        tc_fence_after();
                        const uint32_t reg = C::tR + 128 * (g & 1);
                        const uint32_t os = g % NO, qs = g % NQ;
                        if (leader) {
                            const uint64_t bo = ddOmn + static_cast<uint64_t>((os * C::kT) >> 4);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)  // K-dim: the step's 128 q rows; P^T at +16
                                mma_ts(tmem + C::tdV, tmem + reg + (kk >> 1) * 32 + 16 + (kk & 1) * 8,
                                       bo + ((kk * 2048) >> 4), idA, (n > 0 || kk > 0) ? 1u : 0u);
                            mma_commit(smem_u32(&bars.oe[os]));  // dO(g) read (dP^T(g), dV(g))
                        }
                        __syncwarp();
                        S2TRACE(8, g);
                        if (has_next) issue_dp(g + 1, nfirst, nlast, nic);
                        S2TRACE(14, g);
                        if (leader) {
                            const uint64_t bq = dQmn + static_cast<uint64_t>((qs * C::kT) >> 4);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)  // dS^T at +0
                                mma_ts(tmem + C::tdK, tmem + reg + (kk >> 1) * 32 + (kk & 1) * 8,
                                       bq + ((kk * 2048) >> 4), idA, (n > 0 || kk > 0) ? 1u : 0u);
                            mma_commit(smem_u32(&bars.qe[qs]));  // Q(g) read (S^T(g), dK(g))
                            if (n == ns - 1) mma_commit(smem_u32(&bars.accf));
                        }
                        __syncwarp();
                        S2TRACE(3, g);
                    }
                    ++ic;
                    ++i;
                    while (i < i_end && warp_uniform(items[i].nsteps128) == 0) ++i;
                    if (i >= i_end) break;
                    ns = warp_uniform(items[i].nsteps128);
                }
            }
        }
    } else if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 48;" ::: "memory");
        // ---------------------------------------------------------------- epilogue
        // dV, dK (x scale) TMEM -> registers -> bf16 row stores; the accumulators are
        // released once read (the next item's first dV / dK overwrite them)
        const int kr = tid & 127;
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        uint32_t ic = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const BwdItem it = items[i];
            if (it.nsteps128 == 0) continue;
            const int chunk = kr < 64 ? it.c0 : it.c1;
            const int key = chunk * 64 + (kr & 63);
            const bool ok = chunk >= 0 && key < p.N;
            const size_t row = (static_cast<size_t>(it.kvbh) * p.N + (ok ? key : 0)) * D;
            mbar_wait(smem_u32(&bars.accf), ic & 1);
            tc_fence_after();
#pragma unroll
            for (int ph = 0; ph < 2; ++ph) {  // 0: dV, 1: dK
                __nv_bfloat16* dst = (ph ? p.g0 : p.g1) + row;
                const float mul = ph ? p.scale : 1.0f;
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t u[32];
                    tmem_ld32(tmem + (ph ? C::tdK : C::tdV) + c * 32 + lane_off, u);
                    tmem_ld_wait();
                    if (ph == 1 && c == D / 32 - 1) {  // every accumulator column read
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(smem_u32(&bars.acce));
                    }
                    if (ok) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            uint4 w;
                            w.x = pack_bf16(__uint_as_float(u[8 * q4 + 0]) * mul, __uint_as_float(u[8 * q4 + 1]) * mul);
                            w.y = pack_bf16(__uint_as_float(u[8 * q4 + 2]) * mul, __uint_as_float(u[8 * q4 + 3]) * mul);
                            w.z = pack_bf16(__uint_as_float(u[8 * q4 + 4]) * mul, __uint_as_float(u[8 * q4 + 5]) * mul);
                            w.w = pack_bf16(__uint_as_float(u[8 * q4 + 6]) * mul, __uint_as_float(u[8 * q4 + 7]) * mul);
                            *reinterpret_cast<uint4*>(dst + c * 32 + q4 * 8) = w;
                        }
                    }
                }
            }
            ++ic;
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 96;" ::: "memory");
        // ------------------------------------------------------------- elementwise
        const int w = (warp >> 2) - 2;  // q columns [32w, 32w+32) of each step
        const int kr = tid & 127;       // key row == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const float sl2 = p.scale_log2;
        const uint64_t sl2v = f2_pack(sl2, sl2);
        const int cg = (kr & 63) >> 4;
        uint32_t g = 0, g_done = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const BwdItem it = items[i];
            if (it.nsteps128 == 0) continue;
            const int chunk = kr < 64 ? it.c0 : it.c1;
            const int key = chunk * 64 + (kr & 63);
            const bool key_ok = chunk >= 0 && key < p.N;
            for (int n = 0; n < it.nsteps128; ++n, ++g) {
                const uint32_t as = g % NA;
                mbar_wait(smem_u32(&bars.af[as]), (g / NA) & 1);
                const uint4 meta = bars.meta[as];
                const uint32_t m = key_ok ? (kr < 64 ? meta.y : meta.z) : 0u;
                const int q0 = static_cast<int>(meta.x) + 32 * w;
                // my 2 q row groups (16 rows each) x my key column group
                const uint32_t bits = ((m >> (8 * w + cg)) & 1u) | (((m >> (8 * w + 4 + cg)) & 1u) << 1);
                const uint32_t sl = sAux + as * C::kAux + w * 128;  // lse2[32w..], delta at +512
                const uint32_t tR = tmem + C::tR + 128 * (g & 1) + 32 * w + lane_off;
                if (tid == 256) S2TRACE(5, g);
                mbar_wait(smem_u32(&bars.sf), g & 1);
                if (tid == 256) S2TRACE(6, g);
                tc_fence_after();
                float sv[32];
                tmem_ld32(tR, *reinterpret_cast<uint32_t(*)[32]>(sv));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars.sfr));  // dP^T(n) may now be computed over S^T(n)
                // The two halves of the elementwise warps (X: q columns [64X, 64X+64))
                // take turns on the exponentials -- X0(n), X1(n), X0(n+1), ... -- so each
                // runs with the MUFU pipe to itself while the other does its dS / P
                // packing (all 16 warps exponentiating together was MUFU-bound for
                // ~1.3K cycles, then issue-bound for ~0.9K, per step)
                const int X = w >> 1;
                if (S2_DKV2_ALT) {
                    if (X == 1) named_bar_sync(2, 512);
                    else if (g_done > 0) named_bar_sync(3, 512);
                }
                if (tid == 256) S2TRACE(9, g);
                const int dbg = p.debug;  // timing ablations (wrong results when != 0)
                if (dbg & 64) {
                    // no exponentials
                } else if (bits == 0x3u && key <= q0) {  // every (q, key) of my 32 columns admitted
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 l = (dbg & 32) ? make_float4(1.f, 2.f, 3.f, 4.f) : lds_f4(sl + c * 4);
                        const uint64_t x0 = ffma2(f2_pack(sv[c], sv[c + 1]), sl2v, f2_pack(-l.x, -l.y));
                        const uint64_t x1 = ffma2(f2_pack(sv[c + 2], sv[c + 3]), sl2v, f2_pack(-l.z, -l.w));
                        float a0, a1;
                        f2_unpack(x0, a0, a1);
                        sv[c] = fast_exp2(a0);
                        sv[c + 1] = fast_exp2(a1);
                        if ((c & 12) == 12) {  // 1 pair in 4 on the FMA pipe (cubic 2^x): MUFU paces this loop
                            f2_unpack(exp2_poly2(x1), sv[c + 2], sv[c + 3]);
                        } else {
                            f2_unpack(x1, a0, a1);
                            sv[c + 2] = fast_exp2(a0);
                            sv[c + 3] = fast_exp2(a1);
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 l = lds_f4(sl + c * 4);
                        const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const bool ok = ((bits >> (c >> 4)) & 1u) && key <= q0 + c + u;
                            const float pe = fast_exp2(fmaf(sv[c + u], sl2, -lv[u]));
                            sv[c + u] = ok ? pe : 0.f;
                        }
                    }
                }
                if (S2_DKV2_ALT) named_bar_arrive(2 + X, 512);
                ++g_done;
                if (tid == 256) S2TRACE(10, g);
                mbar_wait(smem_u32(&bars.dpf), g & 1);
                if (tid == 256) S2TRACE(11, g);
                tc_fence_after();
                float dp[32];
                tmem_ld32(tR, *reinterpret_cast<uint32_t(*)[32]>(dp));
                tmem_ld_wait();
                if (tid == 256) S2TRACE(12, g);
                uint32_t ds[16], pk[16];
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 d4 = (dbg & 32) ? make_float4(1.f, 2.f, 3.f, 4.f) : lds_f4(sl + 512 + c * 4);
                    ds[c >> 1] = pack_bf16(sv[c] * (dp[c] - d4.x), sv[c + 1] * (dp[c + 1] - d4.y));
                    ds[(c >> 1) + 1] = pack_bf16(sv[c + 2] * (dp[c + 2] - d4.z), sv[c + 3] * (dp[c + 3] - d4.w));
                    pk[c >> 1] = pack_bf16(sv[c], sv[c + 1]);
                    pk[(c >> 1) + 1] = pack_bf16(sv[c + 2], sv[c + 3]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars.ae[as]));  // lse2 / delta / meta of the slot read
                // dS^T into columns [0,16) and P^T into [16,32) of my columns (all read)
                if (!(dbg & 128)) {
                    tmem_st16(tR, ds);
                    tmem_st16(tR + 16, pk);
                    tmem_st_wait();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars.pds));
                if (tid == 256) S2TRACE(7, g);
            }
        }
        if (S2_DKV2_ALT && (w >> 1) == 0 && g_done > 0) named_bar_sync(3, 512);  // X1's last arrival
    }
    tc_fence_before();
    __syncthreads();
    if (p.trace && tid == 0) p.trace[15 * 2048 + 2 * blockIdx.x + 1] = globaltimer_ns();  // debug: CTA end
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace s2dev

using namespace s2dev;

static long long* g_trace = nullptr;
static int g_debug = 0;
extern "C" void s2_debug_set_mode(int m) { g_debug = m; }
// Debug hook (not in s2attn.h): a device buffer of 8 x 2048 int64 for CTA-0 step timestamps.
extern "C" void s2_debug_set_trace(void* dev_buf) { g_trace = static_cast<long long*>(dev_buf); }
long long* s2_debug_trace_buffer() { return g_trace; }

cudaError_t s2_launch_bwd_prep(const __nv_bfloat16* out, const __nv_bfloat16* dout,
                               const float* lse, float* delta, float* lse2, int num_bh, int N,
                               int Npad, int D, cudaStream_t stream) {
    const long long rows = static_cast<long long>(num_bh) * Npad;
    if (rows >= (1ll << 31)) return cudaErrorInvalidValue;  // the kernel indexes rows in 32 bits
    const int per_block = 256 / (D / 8);
    const long long need = (rows + per_block - 1) / per_block;
    const int blocks = static_cast<int>(std::min<long long>(need, 148LL * 8));
    if (D == 128)
        return launch_pdl(s2_bwd_prep_kernel<128>, dim3(blocks), dim3(256), 0, stream, out, dout, lse, delta, lse2,
                          num_bh, N, Npad);
    else if (D == 64)
        return launch_pdl(s2_bwd_prep_kernel<64>, dim3(blocks), dim3(256), 0, stream, out, dout, lse, delta, lse2,
                          num_bh, N, Npad);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

template <class K>
static cudaError_t launch_bwd(K kern, int smem, int grid, const CUtensorMap& q,
                              const CUtensorMap& dout, const CUtensorMap& k, const CUtensorMap& v,
                              const CUtensorMap& o0, const CUtensorMap& o1, const BwdParams& p,
                              cudaStream_t stream, int threads = 384) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(grid), dim3(threads), smem, stream, q, dout, k, v, o0, o1, p);
}

// which = 0: dK/dV kernel (q/do: 64-row boxes; o0 = dK, o1 = dV maps with 64-row
// boxes); which = 1: dQ kernel (q/do: 128-row boxes; o0 = dQ map, 128-row boxes).
// k/v: 64-row boxes.
cudaError_t s2_launch_bwd_sm100(int which, int D, const CUtensorMap& q, const CUtensorMap& dout,
                                const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o0,
                                const CUtensorMap& o1, const void* items, const int* sched, int grid,
                                const void* entries, const float* lse2, const float* delta,
                                int N, int Npad, int hpg, float scale, cudaStream_t stream,
                                void* g0, void* g1, const void* fused_o, const void* fused_dout,
                                const float* fused_lse, float* fused_delta, float* fused_lse2) {
    if (grid == 0) return cudaSuccess;
    const float sl2 = scale * 1.4426950408889634f;
    // debug bit 8 selects which kernel records the trace (0: dK/dV, 8: dQ)
    long long* tr = ((g_debug & 8) != 0) == (which == 1 || which == 2) ? g_trace : nullptr;
    BwdParams pp{items, sched, entries, lse2, delta, static_cast<__nv_bfloat16*>(g0), static_cast<__nv_bfloat16*>(g1),
                 N, Npad, hpg, sl2, scale, tr, g_debug & ~8,
                 which == 1 ? static_cast<const __nv_bfloat16*>(fused_o) : nullptr,
                 static_cast<const __nv_bfloat16*>(fused_dout), fused_lse, fused_delta, fused_lse2};
    if (g_debug & 4) grid = 1;  // debug: isolate one CTA from memory-system contention
    if (which == 3) {  // dK/dV over 128-row q steps (q/do: 4-D 128-row maps; g0 = dK, g1 = dV)
        if (D == 128)
            return launch_bwd(s2_bwd_dkv2_kernel<128>, Dkv2Cfg<128>::kSmem, grid, q, dout, k, v, o0, o1, pp, stream,
                              768);
        if (D == 64)
            return launch_bwd(s2_bwd_dkv2_kernel<64>, Dkv2Cfg<64>::kSmem, grid, q, dout, k, v, o0, o1, pp, stream,
                              768);
        return cudaErrorInvalidValue;
    }
    if (which == 2) {  // dQ over 128-key steps (q/do: 128-row boxes; o0 = dQ map)
        if (D == 128)
            return launch_bwd(s2_bwd_dq2_kernel<128>, Dq2Cfg<128>::kSmem, grid, q, dout, k, v, o0, o1, pp, stream,
                              512);
        if (D == 64)
            return launch_bwd(s2_bwd_dq2_kernel<64>, Dq2Cfg<64>::kSmem, grid, q, dout, k, v, o0, o1, pp, stream,
                              512);
        return cudaErrorInvalidValue;
    }
    if (D == 128)
        return which == 0 ? launch_bwd(s2_bwd_dkv_kernel<128>, BwdCfg<128>::kDkvSmem, grid, q, dout, k, v, o0, o1, pp, stream)
                          : launch_bwd(s2_bwd_dq_kernel<128>, BwdCfg<128>::kDqSmem, grid, q, dout, k, v, o0, o1, pp, stream);
    if (D == 64)
        return which == 0 ? launch_bwd(s2_bwd_dkv_kernel<64>, BwdCfg<64>::kDkvSmem, grid, q, dout, k, v, o0, o1, pp, stream)
                          : launch_bwd(s2_bwd_dq_kernel<64>, BwdCfg<64>::kDqSmem, grid, q, dout, k, v, o0, o1, pp, stream);
    return cudaErrorInvalidValue;
}
