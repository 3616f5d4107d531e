// S2-Attention forward on CTA pairs (cta_group::2), sm_100a, head_dim 128.
//
// Replaces the reference's streaming kernel process_query_block
// (/root/reference/proj/src/attention.cpp:26-98) and its OpenMP driver
// run_streaming (:100-118), like fwd_sm100.cu, with N=128 score products.
//
// A cluster of two CTAs (one TPC) owns a work item = a PAIR of adjacent
// 128-row query tiles of one (batch, head): CTA r holds tile 2*qpair + r.
// Both walk the union of the two tiles' chunk lists, two 64-key chunks per
// step (PairStep {c0, c1}), and the leader CTA issues every MMA for both:
//   S  = Q K^T   M=256 (tile r's rows from CTA r's Q), N=128 keys: CTA 0
//                holds chunk c0's K, CTA 1 chunk c1's; SS, 8 x K=16
//   O += P V     M=256, N=128 (= D): CTA r holds V[c0 | c1][64r, 64r+64),
//                A = P from each CTA's TMEM; TS, 8 x K=16 keys
// so each MMA runs at the full M=128 x N=128 per-SM rate, where the 1-CTA
// kernel's N=64 S products take ~45 instead of 32 cycles (profiles/r1e).
// Each CTA streams 32 KB per 128-key step (half of the pair's K and V): the
// same L2 -> SM bytes per query row as the 1-CTA pair kernel.
//
// Visit order is fixed per item and nothing is reduced across clusters:
// deterministic and independent of head position (test_attention.cpp:217-257).
// A tile's masked-out chunk of a step gives -inf scores, so P = 0 exactly and
// no key outside the shard contributes (test_attention.cpp:196-215).
//
// Warp roles (512 threads per CTA, 1 CTA / SM):
//   warp 0      TMA producer (both CTAs): Q tile, per step K(c_r) and the
//               CTA's D half of V(c0), V(c1); completion counted on the
//               leader's barriers (.cta_group::2 TMA)
//   warp 1      S issuer (leader): S(k) into TMEM buffer k % 3 once the P V
//               that last read that buffer is complete
//   warp 2      TMEM allocator (both CTAs, cta_group::2)
//   warp 3      P V issuer (leader): O += P(k) V(k) once both CTAs' P(k) is in
//               TMEM; releases the K/V stage, signals O final per item
//   warps 4-11  softmax: two warpgroups, each with 16 rows of every warp
//               quarter (16-lane TMEM shapes), 128 columns per step
//   warps 12-15 epilogue: O -> registers (TMEM released at once), x 1/l,
//               swizzled staging, TMA store; overlaps the next item's softmax
// TMEM (512 columns per CTA): S buffers at 0 / 128 / 256 (P of a step
// overwrites the first 64 columns of its buffer as bf16x2), O at 384.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "fwd_mask.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {

struct P2Item {  // = the pair kernel's PairItem (capi.cpp)
    int32_t bh;
    int32_t qpair;
    int32_t nsteps;
    int32_t has_b;
    int64_t step_off;
};
struct P2Step {  // = PairStep: chunks c0, c1 (-1: none) and the two tiles' masks
    int32_t c0, c1;
    uint32_t a0, a1, b0, b1;
};

struct P2Params {
    const P2Item* items;
    const int* sched;  // [clusters + 1] item range of each cluster
    const P2Step* steps;
    float* lse;
    int seq_len;
    int hpg;
    float scale_log2;
    long long* trace;  // debug: per-step clock64 of cluster 0 (nullptr = off)
};

// debug trace (tools/trace_fwd2.py): slot + 24 * rank of cluster 0's CTAs
#define S2P2TRACE(slot, n)                                                          \
    do {                                                                            \
        if (p.trace && blockIdx.x < 2 && (n) < 2048)                                \
            p.trace[((slot) + 24 * blockIdx.x) * 2048 + (n)] = clock64();           \
    } while (0)

namespace p2 {
constexpr int kQBytes = 32768;  // 128 rows x 128 bf16: 2 SW128 slices [64 cols][128 rows]
constexpr int kKBytes = 16384;  // 64 keys x 128: 2 slices [64 cols][64 rows]
constexpr int kVBytes = 16384;  // 128 keys x this CTA's 64 columns (MN-major SW128)
constexpr int kStage = kKBytes + kVBytes;
#ifndef S2_P2_NST
#define S2_P2_NST 4
#endif
constexpr int kNST = S2_P2_NST;
constexpr int kStgBytes = 32768;  // O staging: 2 x [128 rows][64 cols]
constexpr int kSmem = 1024 + kQBytes + kNST * kStage + kStgBytes;
constexpr int kNS = 3;            // S buffers
constexpr uint32_t kOCol = 384;
// exp2 on the FMA pipe (cubic) for 1 in (mask+1) pairs; -1: all on MUFU.EX2
// softmax warpgroups alternate their non-MUFU phases (named barriers 2 / 3)
#ifndef S2_P2_ALTERNATE
#define S2_P2_ALTERNATE 1
#endif
#ifndef S2_P2_POLY_MASK
#define S2_P2_POLY_MASK -1
#endif
}  // namespace p2

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    s2_fwd_pair2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                        const P2Params p) {
    using namespace p2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // Same offsets in both CTAs.  Barriers the leader's MMA warps wait on count
    // both CTAs: bar_qf / bar_kf (TMA bytes of both), bar_pf (8 warps of each
    // CTA), bar_oe (4).  MMA completions (bar_qe, bar_ke, bar_sf, bar_pv,
    // bar_of) arrive in both CTAs (multicast commit).
    __shared__ uint64_t bar_qf, bar_qe, bar_kf[kNST], bar_ke[kNST];
    __shared__ uint64_t bar_sf[kNS], bar_pf[kNS], bar_pv[kNS], bar_of, bar_oe, bar_stf, bar_ste;
    __shared__ float st_l[128], st_m[128];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cl = blockIdx.x >> 1;
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sKV = sQ + kQBytes;
    const uint32_t sStg = sKV + kNST * kStage;

    if (tid == 0) {
        mbar_init(smem_u32(&bar_qf), 1);
        mbar_init(smem_u32(&bar_qe), 1);
        for (int i = 0; i < kNST; ++i) {
            mbar_init(smem_u32(&bar_kf[i]), 1);
            mbar_init(smem_u32(&bar_ke[i]), 1);
        }
        for (int i = 0; i < kNS; ++i) {
            mbar_init(smem_u32(&bar_sf[i]), 1);
            mbar_init(smem_u32(&bar_pf[i]), 16);
            mbar_init(smem_u32(&bar_pv[i]), 1);
        }
        mbar_init(smem_u32(&bar_of), 1);
        mbar_init(smem_u32(&bar_oe), 8);
        mbar_init(smem_u32(&bar_stf), 256);
        mbar_init(smem_u32(&bar_ste), 128);
        fence_mbar_init();
    }
    if (warp == 2) {
        tmem_alloc_2cta(smem_u32(&tmem_base_s), 512);
        tmem_relinquish_2cta();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's barriers are initialised before anyone signals them
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    pdl_launch_dependents();
    pdl_wait();

    const int i_beg = p.sched[cl], i_end = p.sched[cl + 1];
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------------ producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const uint64_t keep = policy_evict_last();
            const uint32_t qf_l = mapa_shared(smem_u32(&bar_qf), 0);
            uint32_t kv_it = 0, q_use = 0;
            for (int i = i_beg; i < i_end; ++i) {
                const P2Item it = p.items[i];
                const int kvbh = it.bh / p.hpg;
                if (q_use > 0) mbar_wait(smem_u32(&bar_qe), (q_use - 1) & 1);
                if (leader) mbar_expect_tx(smem_u32(&bar_qf), 2 * kQBytes);
                tma_load_rows_2cta(sQ, &tmQ, qf_l, (2 * it.qpair + static_cast<int>(rank)) * 128, it.bh, keep);
                ++q_use;
                const P2Step* steps = p.steps + it.step_off;
                for (int n = 0; n < it.nsteps; ++n) {
                    const P2Step ps = steps[n];
                    const int c0 = ps.c0, c1 = ps.c1 < 0 ? ps.c0 : ps.c1;
                    const int st = kv_it % kNST;
                    S2P2TRACE(9, kv_it);
                    if (kv_it >= kNST) mbar_wait(smem_u32(&bar_ke[st]), ((kv_it / kNST) + 1) & 1);
                    S2P2TRACE(10, kv_it);
                    const uint32_t sK = sKV + st * kStage, sV = sK + kKBytes;
                    if (leader) mbar_expect_tx(smem_u32(&bar_kf[st]), 2 * kStage);
                    const uint32_t bar = mapa_shared(smem_u32(&bar_kf[st]), 0);
                    tma_load_rows_2cta(sK, &tmK, bar, (rank ? c1 : c0) * 64, kvbh, keep);
                    tma_load_3d_2cta(sV, &tmV, bar, 64 * static_cast<int>(rank), c0 * 64, kvbh, keep);
                    tma_load_3d_2cta(sV + 8192, &tmV, bar, 64 * static_cast<int>(rank), c1 * 64, kvbh, keep);
                    ++kv_it;
                }
            }
        } else if (warp == 1 && leader) {
            // ------------------------------------------------------ S issuer
            constexpr uint32_t idS = umma_idesc_bf16(256, 128, 0, 0);
            const bool el = elect_one();
            const uint64_t dQ0 = umma_desc_sw128(sQ, 16, 1024);
            const uint64_t dKV0 = umma_desc_sw128(sKV, 16, 1024);
            uint32_t kv_it = 0, q_use = 0, k = 0;
            for (int i = i_beg; i < i_end; ++i) {
                const int nsteps = warp_uniform(p.items[i].nsteps);
                mbar_wait(smem_u32(&bar_qf), q_use & 1);
                for (int n = 0; n < nsteps; ++n) {
                    const int st = kv_it % kNST;
                    S2P2TRACE(0, k);
                    mbar_wait(smem_u32(&bar_kf[st]), (kv_it / kNST) & 1);
                    S2P2TRACE(1, k);
                    const uint32_t b = k % kNS, u = k / kNS;
                    if (u > 0) mbar_wait(smem_u32(&bar_pv[b]), (u - 1) & 1);  // buffer b's last P V read it
                    S2P2TRACE(2, k);
                    tc_fence_after();
                    const uint64_t dk = dKV0 + static_cast<uint64_t>((st * kStage) >> 4);
                    if (el) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint32_t oq = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                            const uint32_t ok = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                            mma_ss_2cta(tmem + b * 128, dQ0 + oq, dk + ok, idS, kk > 0);
                        }
                        mma_commit_2cta(smem_u32(&bar_sf[b]));
                    }
                    __syncwarp();
                    ++kv_it;
                    ++k;
                }
                // every S of the item is issued: both Q tiles are free once they complete
                if (el) mma_commit_2cta(smem_u32(&bar_qe));
                __syncwarp();
                ++q_use;
            }
        } else if (warp == 3 && leader) {
            // ------------------------------------------------------ P V issuer
            constexpr uint32_t idO = umma_idesc_bf16(256, 128, 0, 1);
            const bool el = elect_one();
            const uint64_t dV0 = umma_desc_sw128(sKV + kKBytes, 8192, 1024);
            uint32_t kv_it = 0, k = 0, o_use = 0;
            for (int i = i_beg; i < i_end; ++i) {
                const int nsteps = warp_uniform(p.items[i].nsteps);
                for (int n = 0; n < nsteps; ++n) {
                    const int st = kv_it % kNST;
                    const uint32_t b = k % kNS, u = k / kNS;
                    S2P2TRACE(3, k);
                    mbar_wait(smem_u32(&bar_pf[b]), u & 1);
                    S2P2TRACE(4, k);
                    if (n == 0 && o_use > 0) mbar_wait(smem_u32(&bar_oe), (o_use - 1) & 1);
                    S2P2TRACE(11, k);
                    tc_fence_after();  // P was written to both CTAs' TMEM by tcgen05.st
                    const uint64_t dv = dV0 + static_cast<uint64_t>((st * kStage) >> 4);
                    if (el) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            mma_ts_2cta(tmem + kOCol, tmem + b * 128 + kk * 8, dv + ((kk * 2048) >> 4), idO,
                                        (n > 0 || kk > 0) ? 1u : 0u);
                        mma_commit_2cta(smem_u32(&bar_pv[b]));
                        mma_commit_2cta(smem_u32(&bar_ke[st]));  // K read by S(k) (complete: P(k) exists), V by this
                        if (n == nsteps - 1) mma_commit_2cta(smem_u32(&bar_of));
                    }
                    __syncwarp();
                    ++kv_it;
                    ++k;
                }
                if (nsteps == 0) {  // no attended chunk: O is never written (out = NaN rows below)
                    if (o_use > 0) mbar_wait(smem_u32(&bar_oe), (o_use - 1) & 1);
                    if (el) mma_commit_2cta(smem_u32(&bar_of));
                    __syncwarp();
                }
                ++o_use;
            }
        }
    } else if (warp < 12) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 168;" ::: "memory");
        // ----------------------------------------------------------- softmax
        // Warpgroup h takes lanes [16h, 16h+16) of each warp's quarter (16-lane
        // TMEM shapes): thread t holds rows A = L + t/4 and B = A + 8 of the
        // step's 128 columns, 32 each (columns 8j + 2(t%4) + {0,1}); the four
        // threads of a row combine maxima / sums with two shuffles.  The two
        // warpgroups run independently, so one's loads and maxima overlap the
        // other's exponentials.  (A single warpgroup over all 128 columns was
        // latency-bound: 2.2K cycles per step for 1K of MUFU work; a column
        // split needs a cross-warpgroup max exchange every step.)
        const int h = warp >= 8;
        const int L = 32 * (warp & 3) + 16 * h;  // first TMEM lane (tile row) of the warp
        const int LA = L + (lane >> 2);          // row A; row B = LA + 8
        const uint32_t lane_off = static_cast<uint32_t>(L) << 16;
        const uint32_t tS0 = tmem + lane_off, tO = tmem + lane_off + kOCol;
        const int rg = L >> 4;                   // 16-row mask group of both rows
        const int cq = 2 * (lane & 3);
        const float sl2 = p.scale_log2;
        uint32_t pf_l[kNS];
#pragma unroll
        for (int b = 0; b < kNS; ++b) pf_l[b] = mapa_shared(smem_u32(&bar_pf[b]), 0);
        uint32_t k = 0, icnt = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const P2Item it = p.items[i];
            const P2Step* steps = p.steps + it.step_off;
            const int row0 = (2 * it.qpair + static_cast<int>(rank)) * 128;
            const int qA = row0 + LA, qB = qA + 8;
            float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
            P2Step nxt = steps[0];
            for (int n = 0; n < it.nsteps; ++n) {
                const P2Step s = nxt;
                if (n + 1 < it.nsteps) nxt = steps[n + 1];
                const uint32_t b = k % kNS, u = k / kNS;
                // the two warpgroups alternate their load / mask / max phases, so each
                // one's exponentials have the MUFU pipe to themselves
                if (S2_P2_ALTERNATE) {
                    if (h == 1) named_bar_sync(2, 256);  // warpgroup 0 has its maxima of step k
                    else if (k > 0) named_bar_sync(3, 256);  // warpgroup 1 has its maxima of step k-1
                }
                if (lane == 0 && warp == 4 + 4 * h) S2P2TRACE(5 + 12 * h, k);
                mbar_wait(smem_u32(&bar_sf[b]), u & 1);
                if (lane == 0 && warp == 4 + 4 * h) S2P2TRACE(6 + 12 * h, k);
                tc_fence_after();
                // warp-uniform mask words of this step's two chunks (uniform branch
                // below: masked steps get their own copy of the step body, so the
                // common unmasked step carries no select / register-copy work)
                const int c1 = s.c1 < 0 ? s.c0 : s.c1;
                const uint32_t bits0 = warp_uniform(((rank ? s.b0 : s.a0) >> (rg * 4)) & 0xFu);
                const uint32_t bits1 = warp_uniform(((s.c1 < 0 ? 0u : (rank ? s.b1 : s.a1)) >> (rg * 4)) & 0xFu);
                const int key00 = warp_uniform(s.c0 * 64), key01 = warp_uniform(c1 * 64);
                const bool diag0 = key00 + 63 > row0, diag1 = key01 + 63 > row0;
                const bool need_mask = bits0 != 0xFu || bits1 != 0xFu || diag0 || diag1;
                auto step = [&](auto masked) {
                    constexpr bool MASK = decltype(masked)::value;
                    float sv[64];
                    tmem_ld_16x256b_x16(tS0 + b * 128, *reinterpret_cast<uint32_t(*)[64]>(sv));
                    tmem_ld_wait();
                    if (MASK) {
                        // fwd_mask.cuh semantics: 16-column groups of each chunk, and
                        // in-block causality on the diagonal chunk
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const uint32_t bits = hh ? bits1 : bits0;
                            const int key0 = hh ? key01 : key00;
                            const bool diag = hh ? diag1 : diag0;
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                const bool on = (bits >> (jj >> 1)) & 1u;
                                const int j = 8 * hh + jj;
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int key = key0 + 8 * jj + cq + e;
                                    sv[4 * j + e] = (!on || (diag && key > qA)) ? -INFINITY : sv[4 * j + e];
                                    sv[4 * j + 2 + e] = (!on || (diag && key > qB)) ? -INFINITY : sv[4 * j + 2 + e];
                                }
                            }
                        }
                    }
                    float xa = fmaxf(sv[0], sv[1]), xb = fmaxf(sv[2], sv[3]);
                    float ya = fmaxf(sv[4], sv[5]), yb = fmaxf(sv[6], sv[7]);
    #pragma unroll
                    for (int j = 2; j < 16; j += 2) {  // 3-input FMNMX
                        xa = fmaxf(xa, fmaxf(sv[4 * j], sv[4 * j + 1]));
                        xb = fmaxf(xb, fmaxf(sv[4 * j + 2], sv[4 * j + 3]));
                        ya = fmaxf(ya, fmaxf(sv[4 * j + 4], sv[4 * j + 5]));
                        yb = fmaxf(yb, fmaxf(sv[4 * j + 6], sv[4 * j + 7]));
                    }
                    float mxA = fmaxf(xa, ya), mxB = fmaxf(xb, yb);
                    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
                    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
                    mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
                    mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
                    // lazy rescale: O and l keep a stale max until the new one exceeds it by 2^8
                    const float tA = mxA * sl2, tB = mxB * sl2;
                    float uA = mA, uB = mB;
                    bool rA = false, rB = false;
                    if (tA > mA) {
                        if (mA == -INFINITY) uA = tA;
                        else if (tA > mA + 8.0f) { uA = tA; rA = true; }
                    }
                    if (tB > mB) {
                        if (mB == -INFINITY) uB = tB;
                        else if (tB > mB + 8.0f) { uB = tB; rB = true; }
                    }
                    if (__any_sync(0xffffffffu, rA || rB)) {
                        // O must hold every earlier step's P V (the last: step k-1) before it is rescaled
                        mbar_wait(smem_u32(&bar_pv[(k - 1) % kNS]), ((k - 1) / kNS) & 1);
                        tc_fence_after();
                        const float aA = rA ? fast_exp2(mA - uA) : 1.0f, aB = rB ? fast_exp2(mB - uB) : 1.0f;
                        lA *= aA;
                        lB *= aB;
    #pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            uint32_t w[32];
                            tmem_ld_16x256b_x8(tO + c * 64, w);
                            tmem_ld_wait();
    #pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                w[4 * j] = __float_as_uint(__uint_as_float(w[4 * j]) * aA);
                                w[4 * j + 1] = __float_as_uint(__uint_as_float(w[4 * j + 1]) * aA);
                                w[4 * j + 2] = __float_as_uint(__uint_as_float(w[4 * j + 2]) * aB);
                                w[4 * j + 3] = __float_as_uint(__uint_as_float(w[4 * j + 3]) * aB);
                            }
                            tmem_st_16x256b_x8(tO + c * 64, w);
                        }
                    }
                    mA = uA;
                    mB = uB;
                    if (S2_P2_ALTERNATE) named_bar_arrive(2 + h, 256);
                    if (lane == 0 && warp == 4 + 4 * h) S2P2TRACE(7 + 12 * h, k);
                    const float bA = (uA == -INFINITY) ? 0.f : uA, bB = (uB == -INFINITY) ? 0.f : uB;
                    const uint64_t sl2v = f2_pack(sl2, sl2), nbA = f2_pack(-bA, -bA), nbB = f2_pack(-bB, -bB);
                    uint64_t accA[2] = {0ull, 0ull}, accB[2] = {0ull, 0ull};
                    uint32_t pk[32];
    #pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint64_t xA = ffma2(f2_pack(sv[4 * j], sv[4 * j + 1]), sl2v, nbA);
                        const uint64_t xB = ffma2(f2_pack(sv[4 * j + 2], sv[4 * j + 3]), sl2v, nbB);
                        uint64_t pA, pB;
                        if (S2_P2_POLY_MASK >= 0 && (j & S2_P2_POLY_MASK) == S2_P2_POLY_MASK) {
                            pA = exp2_poly2(xA);
                            pB = exp2_poly2(xB);
                        } else {
                            float x0, x1;
                            f2_unpack(xA, x0, x1);
                            pA = f2_pack(fast_exp2(x0), fast_exp2(x1));
                            f2_unpack(xB, x0, x1);
                            pB = f2_pack(fast_exp2(x0), fast_exp2(x1));
                        }
                        accA[j & 1] = fadd2(accA[j & 1], pA);
                        accB[j & 1] = fadd2(accB[j & 1], pB);
                        float p0, p1;
                        f2_unpack(pA, p0, p1);
                        pk[2 * j] = pack_bf16(p0, p1);  // P column 4j + t%4 (keys 8j + cq, +1) of row A
                        f2_unpack(pB, p0, p1);
                        pk[2 * j + 1] = pack_bf16(p0, p1);
                    }
                    // P as bf16x2 into columns [0, 64) of the buffer (this warp's rows only)
                    tmem_st_16x128b_x16(tS0 + b * 128, pk);
                    {
                        float a0, a1;
                        f2_unpack(fadd2(accA[0], accA[1]), a0, a1);
                        lA += a0 + a1;
                        f2_unpack(fadd2(accB[0], accB[1]), a0, a1);
                        lB += a0 + a1;
                    }
                };
                if (need_mask) step(std::true_type{});
                else step(std::false_type{});
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(pf_l[b]);
                if (lane == 0 && warp == 4 + 4 * h) S2P2TRACE(8 + 12 * h, k);
                ++k;
            }
            // row statistics for the epilogue warpgroup (sums over the 4 threads of a row)
            lA += __shfl_xor_sync(0xffffffffu, lA, 1);
            lB += __shfl_xor_sync(0xffffffffu, lB, 1);
            lA += __shfl_xor_sync(0xffffffffu, lA, 2);
            lB += __shfl_xor_sync(0xffffffffu, lB, 2);
            if (icnt > 0) mbar_wait(smem_u32(&bar_ste), (icnt - 1) & 1);
            if ((lane & 3) == 0) {
                st_l[LA] = lA;
                st_l[LA + 8] = lB;
                st_m[LA] = mA;
                st_m[LA + 8] = mB;
            }
            mbar_arrive(smem_u32(&bar_stf));
            ++icnt;
        }
        if (S2_P2_ALTERNATE && h == 0 && k > 0) named_bar_sync(3, 256);  // warpgroup 1's last arrival
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 120;" ::: "memory");
        // ---------------------------------------------------------- epilogue
        const int r = tid & 127;
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tO = tmem + lane_off + kOCol;
        const uint32_t oe_l = mapa_shared(smem_u32(&bar_oe), 0);
        uint32_t o_cnt = 0;
        for (int i = i_beg; i < i_end; ++i) {
            const P2Item it = p.items[i];
            const int row0 = (2 * it.qpair + static_cast<int>(rank)) * 128;
            const int q_pos = row0 + r;
            mbar_wait(smem_u32(&bar_stf), o_cnt & 1);
            const float l_run = st_l[r], m_run = st_m[r];
            mbar_arrive(smem_u32(&bar_ste));
            // a row with no admitted key: out = 0/0 = NaN, lse = -inf (the reference's acc / l)
            const float inv_l = l_run > 0.f ? 1.0f / l_run : __int_as_float(0x7fc00000);
            mbar_wait(smem_u32(&bar_of), o_cnt & 1);
            tc_fence_after();
            if (r == 0) bulk_wait_read0();  // the previous item's stores have read the staging tile
            named_bar_sync(1, 128);
            // O in two 64-column halves (registers), released after the second load
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                uint32_t ov[64];
                tmem_ld32(tO + j * 64, *reinterpret_cast<uint32_t(*)[32]>(ov));
                tmem_ld32(tO + j * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(ov + 32));
                tmem_ld_wait();
                if (j == 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(oe_l);  // O of this CTA may be overwritten
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t* w = ov + c * 8;
                    sts_u4(sStg + j * 16384 + r * 128 + ((c ^ (r & 7)) << 4),
                           pack_bf16(__uint_as_float(w[0]) * inv_l, __uint_as_float(w[1]) * inv_l),
                           pack_bf16(__uint_as_float(w[2]) * inv_l, __uint_as_float(w[3]) * inv_l),
                           pack_bf16(__uint_as_float(w[4]) * inv_l, __uint_as_float(w[5]) * inv_l),
                           pack_bf16(__uint_as_float(w[6]) * inv_l, __uint_as_float(w[7]) * inv_l));
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (r == 0) {  // rows past seq_len are clipped by the tensor map
                tma_store_3d(&tmO, sStg, 0, row0, it.bh);
                tma_store_3d(&tmO, sStg + 16384, 64, row0, it.bh);
                bulk_commit();
            }
            if (q_pos < p.seq_len)
                p.lse[static_cast<size_t>(it.bh) * p.seq_len + q_pos] = (m_run + __log2f(l_run)) * 0.69314718055994530942f;
            ++o_cnt;
        }
        if (r == 0) bulk_wait0();  // the staging tile must outlive the stores
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no CTA leaves while its peer may still signal its barriers
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2cta(tmem, 512);
    }
}

}  // namespace s2dev

// Clusters of the persistent grid: pairs that can be co-resident (at most
// one per TPC).
int s2_fwd_pair2_clusters() {
    static int n = -1;
    if (n >= 0) return n;
    auto kern = s2dev::s2_fwd_pair2_kernel;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, s2dev::p2::kSmem) != cudaSuccess) {
        n = 0;
        return n;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms & ~1);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = s2dev::p2::kSmem;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess) c = 0;
    cudaGetLastError();
    n = std::min(c, sms / 2);
    return n;
}

long long* s2_debug_trace_buffer();
cudaError_t s2_launch_fwd_pair2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                                const CUtensorMap& o, const void* items, const int* sched, int clusters,
                                const void* steps, float* lse, int seq_len, int hpg, float scale_log2,
                                cudaStream_t stream) {
    if (clusters == 0) return cudaSuccess;
    s2dev::P2Params p{static_cast<const s2dev::P2Item*>(items), sched, static_cast<const s2dev::P2Step*>(steps),
                      lse, seq_len, hpg, scale_log2, s2_debug_trace_buffer()};
    auto kern = s2dev::s2_fwd_pair2_kernel;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, s2dev::p2::kSmem);
    if (e != cudaSuccess) return e;
    return s2dev::launch_pdl(kern, dim3(2 * clusters), dim3(512), s2dev::p2::kSmem, stream, q, k, v, o, p);
}
