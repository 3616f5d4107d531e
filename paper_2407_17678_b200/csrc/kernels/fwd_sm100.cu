// S2-Attention forward, sm_100a.  Persistent CTAs; each work item is a PAIR
// of adjacent 128-row query tiles of one (batch, head) that share every K/V
// load (the union of their chunk lists), with one softmax warpgroup per tile.
//
// Replaces the reference's streaming kernel process_query_block
// (/root/reference/proj/src/attention.cpp:26-98) and its OpenMP driver
// run_streaming (:100-118).  Only the 64-key chunks a tile's rows attend are
// visited; masked scores are -inf, so P = 0 exactly and no value row outside
// the shard ever contributes (test_attention.cpp:196-215).  Visit order is
// fixed per item and nothing is reduced across CTAs: deterministic, and
// independent of head position (test_attention.cpp:217-257).
//
// Chunk-granular pipeline: every step is one 64-key chunk.  Each tile's 128
// S columns hold TWO chunk scores (S(k) in half k&1), so the MMA warp issues
// S_t(k+1) before O_t += P_t(k) V(k): the next scores are computed while the
// softmax of this chunk runs, instead of after it.
//
// Warp roles (384 threads, 1 CTA / SM; setmaxnreg moves registers from the
// control warpgroup (72/thread) to the two softmax warpgroups (216/thread)):
//   warp 0      TMA producer: Q tiles, one K/V chunk per NST ring stage
//   warp 1      S issuer:   S_t(j) = Q_t K(j)^T for both tiles (SS, N=64), into
//               S half j & 1 once the P V that last read that half is complete
//   warp 2      TMEM allocator
//   warp 3      P V issuer: O_t += P_t(j) V(j) (TS, K=64) as soon as P_t(j) is in
//               TMEM; releases the K/V stage.  (tcgen05.mma issue blocks for about
//               the MMA's execution time, so one warp that also waited for P left
//               the pipe idle meanwhile: two issuers, 6-7% faster.)
//   warps 4-7   softmax of tile 0 (thread = query row = TMEM lane), epilogue
//   warps 8-11  softmax of tile 1
// TMEM (512 columns): tile t owns [256t, 256t+256): S halves at +0 / +64 (P
// of a chunk overwrites the first 32 columns of its half as bf16x2), O at +128.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "fwd_mask.cuh"
#include "sm100_ptx.cuh"

namespace s2dev {

struct PairItem {
    int32_t bh;      // data index of the query head
    int32_t qpair;   // query tiles 2*qpair, 2*qpair+1
    int32_t nsteps;
    int32_t has_b;   // tile 2*qpair+1 exists
    int64_t step_off;
};
struct PairStep {
    int32_t c0, c1;
    uint32_t a0, a1, b0, b1;
};

constexpr int kMaxPeers = 8;

struct Fwd2Params {
    const PairItem* items;
    const int* sched;  // [grid + 1] item range of each CTA (host-side schedule)
    const PairStep* steps;
    __nv_bfloat16* out;
    float* lse;
    int seq_len;
    int hpg;
    float scale_log2;
    long long* trace;  // debug: per-step clock64 of CTA 0 (nullptr = off)
};

// Fused output exchange (head-parallel multi-GPU, s2_attn_fwd_peers): every
// finished O tile is also TMA-stored into each rank's full output buffer (peer
// memory over NVLink) and its lse rows written there -- the forward and the
// all-gather in one kernel.  num_peers = 0: off.  A separate __grid_constant__
// parameter: folding it into Fwd2Params (2.6 KB, all grid-constant) cost the
// forward ~10%.
struct FwdPeers {
    int num_peers;
    const int* unit_global;           // local unit index -> global unit index
    float* peer_lse[kMaxPeers];       // [total_units * hpg][seq_len] per rank
    CUtensorMap peer_o[kMaxPeers];    // bf16 [total_units * hpg][seq_len][D], boxes {64, 128}
};
// the plain forward's instantiation carries no exchange parameters at all
struct NoPeers {
    static constexpr int num_peers = 0;
    const int* unit_global;
    float* peer_lse[1];
    CUtensorMap peer_o[1];
};

#define S2FTRACE(slot, n)                                                      \
    do {                                                                       \
        if (p.trace && blockIdx.x == 0 && (n) < 2048)                          \
            p.trace[(slot) * 2048 + (n)] = clock64();                          \
    } while (0)

template <int D>
struct Fwd2Cfg {
    static constexpr int kSub = D / 64;
    static constexpr int kQBytes = kSub * 16384;  // 128 rows
    static constexpr int kCBytes = kSub * 8192;   // one 64-key chunk of K (or V)
// exp2 on the FMA pipe (cubic) for 1 in (mask+1) pairs; -1: all on MUFU.EX2.
// The two tiles' softmax warps on one SM sub-partition share its MUFU (4 lanes per
// cycle); a small share on the FMA pipe shortens their exponential phases, a
// large one only adds instructions.  Same-box A/B (r2g): 1 in 16 0.677 vs 0.683 ms
// and 0.715 vs 0.727; 1 in 8 0.678-0.680; 1 in 4 0.688.  (Making the two warps take
// turns on the MUFU instead lost: 0.78 ms.)
#ifndef S2_FWD_POLY_MASK
#define S2_FWD_POLY_MASK 15
#endif
#ifndef S2_FWD_NST
#define S2_FWD_NST 4
#endif

    static constexpr int kNST = D == 128 ? S2_FWD_NST : 8;
    static constexpr int kStageBytes = 2 * kCBytes;
    // per tile, a 128-row x 64-column bf16 staging slice for the O epilogue's TMA stores
    static constexpr int kStgBytes = 16384;
    static constexpr int kSmem = 1024 + 2 * kQBytes + kNST * kStageBytes + 2 * kStgBytes;
};

template <int D, bool PEERS>
__global__ void __launch_bounds__(384, 1)
    s2_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmO, const Fwd2Params p,
                        const __grid_constant__ std::conditional_t<PEERS, FwdPeers, NoPeers> px) {
    using C = Fwd2Cfg<D>;
    constexpr int NST = C::kNST;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_qf[2], bar_qe[2], bar_kf[NST], bar_ke[NST];
    // bar_pv[t][h]: completes once per P V of tile t that read S half h (P V #m
    // reads half m & 1).  The S issuer waits on it before overwriting that half
    // (two MMA-issuing warps: no issue-order guarantee between them), the
    // softmax before rescaling O.  S / P barriers are per (tile, S half) too:
    // with two chunks in flight per tile, a single barrier could complete two
    // phases ahead of a waiter.
    __shared__ uint64_t bar_sf[2][2], bar_pf[2][2], bar_of[2], bar_oe[2], bar_pv[2][2];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t sQ0 = smem_u32(smem);
    const uint32_t sKV = sQ0 + 2 * C::kQBytes;
    const uint32_t sStg = sKV + NST * C::kStageBytes;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bar_qf[i]), 1);
            mbar_init(smem_u32(&bar_qe[i]), 1);
            for (int j = 0; j < 2; ++j) {
                mbar_init(smem_u32(&bar_sf[i][j]), 1);
                mbar_init(smem_u32(&bar_pf[i][j]), 128);
            }
            mbar_init(smem_u32(&bar_of[i]), 1);
            mbar_init(smem_u32(&bar_oe[i]), 128);
            mbar_init(smem_u32(&bar_pv[i][0]), 1);
            mbar_init(smem_u32(&bar_pv[i][1]), 1);
        }
        for (int i = 0; i < NST; ++i) {
            mbar_init(smem_u32(&bar_kf[i]), 1);
            mbar_init(smem_u32(&bar_ke[i]), 1);
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

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;" ::: "memory");
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------------ producer
            tma_prefetch(&tmQ);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const uint64_t keep = policy_evict_last();
            uint32_t kv_it = 0, q_use[2] = {0, 0};
            for (int i = p.sched[blockIdx.x]; i < p.sched[blockIdx.x + 1]; ++i) {
                const PairItem it = p.items[i];
                const int kvbh = it.bh / p.hpg;
                for (int t = 0; t < 2; ++t) {
                    if (t == 1 && !it.has_b) continue;
                    if (q_use[t] > 0) mbar_wait(smem_u32(&bar_qe[t]), (q_use[t] - 1) & 1);
                    const uint32_t sQ = sQ0 + t * C::kQBytes;
                    mbar_expect_tx(smem_u32(&bar_qf[t]), C::kQBytes);
                    tma_load_rows(sQ, &tmQ, smem_u32(&bar_qf[t]), (2 * it.qpair + t) * 128, it.bh);
                    ++q_use[t];
                }
                const PairStep* steps = p.steps + it.step_off;
                for (int n = 0; n < it.nsteps; ++n) {
                    const PairStep ps = steps[n];
                    for (int h = 0; h < 2; ++h) {
                        const int chunk = h ? ps.c1 : ps.c0;
                        if (chunk < 0) continue;
                        const int st = kv_it % NST;
                        if (kv_it >= NST) mbar_wait(smem_u32(&bar_ke[st]), ((kv_it / NST) + 1) & 1);
                        const uint32_t sK = sKV + st * C::kStageBytes, sV = sK + C::kCBytes;
                        const uint32_t bar = smem_u32(&bar_kf[st]);
                        mbar_expect_tx(bar, 2 * C::kCBytes);
                        tma_load_rows_hint(sK, &tmK, bar, chunk * 64, kvbh, keep);
                        tma_load_rows_hint(sV, &tmV, bar, chunk * 64, kvbh, keep);
                        ++kv_it;
                    }
                }
            }
        } else if (warp == 1) {
            // ------------------------------------------------------ S issuer
            // tcgen05.mma issue runs at about the rate the pipe executes it, so a
            // warp that also waits for P leaves the pipe idle meanwhile.  S and
            // P V therefore have their own issuing warps (1 and 3); the pipe is
            // fed whenever either has work.  Whole warp on warp-uniform values,
            // one elected lane issues (descriptors in uniform registers).
            constexpr uint32_t idS = umma_idesc_bf16(128, 64, 0, 0);
            const bool leader = elect_one();
            const uint64_t dQ0 = umma_desc_sw128(sQ0, 16, 1024);
            const uint64_t dKV0 = umma_desc_sw128(sKV, 16, 1024);
            uint32_t kv_it = 0, q_use[2] = {0, 0};
            uint32_t k_cnt[2] = {0, 0};  // S of tile t issued so far (global): its S half
            const int i_end = p.sched[blockIdx.x + 1];
            for (int i = p.sched[blockIdx.x]; i < i_end; ++i) {
                const int nsteps = warp_uniform(p.items[i].nsteps);
                const bool has_b = warp_uniform(p.items[i].has_b) != 0;
                const PairStep* steps = p.steps + p.items[i].step_off;
                const bool has[2] = {true, has_b};
                for (int t = 0; t < 2; ++t)
                    if (has[t]) mbar_wait(smem_u32(&bar_qf[t]), q_use[t] & 1);
                PairStep nxt = steps[0];
                for (int n = 0; n < nsteps; ++n) {
                    const PairStep ps = nxt;
                    if (n + 1 < nsteps) nxt = steps[n + 1];
                    for (int h = 0; h < 2; ++h) {
                        const int chunk = warp_uniform(h ? ps.c1 : ps.c0);
                        if (chunk < 0) continue;
                        const uint32_t mk[2] = {warp_uniform(h ? ps.a1 : ps.a0), warp_uniform(h ? ps.b1 : ps.b0)};
                        const int st = kv_it % NST;
                        S2FTRACE(0, kv_it);
                        mbar_wait(smem_u32(&bar_kf[st]), (kv_it / NST) & 1);
                        S2FTRACE(1, kv_it);
                        const uint64_t dk = dKV0 + static_cast<uint64_t>((st * C::kStageBytes) >> 4);
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            if (!has[t] || !mk[t]) continue;
                            const uint32_t kc = k_cnt[t]++;
                            const uint32_t half = kc & 1;
                            // the half holds P of S #kc-2: its P V must be complete
                            if (kc >= 2) mbar_wait(smem_u32(&bar_pv[t][half]), ((kc - 2) >> 1) & 1);
                            const uint32_t tS = tmem + t * 256 + half * 64;
                            const uint64_t dq = dQ0 + static_cast<uint64_t>((t * C::kQBytes) >> 4);
                            if (leader) {
#pragma unroll
                                for (int kk = 0; kk < D / 16; ++kk) {
                                    const uint32_t oq = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                                    const uint32_t ok = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                                    mma_ss(tS, dq + oq, dk + ok, idS, kk > 0);
                                }
                                mma_commit(smem_u32(&bar_sf[t][half]));
                            }
                            __syncwarp();
                        }
                        S2FTRACE(2, kv_it);
                        ++kv_it;
                    }
                }
                // every S of the item is issued: the Q tiles are free once they complete
                // (the next item's Q loads overlap the last softmax, P V and epilogue)
                if (leader)
                    for (int t = 0; t < 2; ++t)
                        if (has[t]) mma_commit(smem_u32(&bar_qe[t]));
                __syncwarp();
                for (int t = 0; t < 2; ++t)
                    if (has[t]) ++q_use[t];
            }
        } else if (warp == 3) {
            // ------------------------------------------------------ P V issuer
            constexpr uint32_t idO = umma_idesc_bf16(128, D, 0, 1);
            const bool leader = elect_one();
            const uint64_t dVmn0 = umma_desc_sw128(sKV + C::kCBytes, 8192, 1024);
            uint32_t kv_it = 0, p_cnt[2] = {0, 0}, o_use[2] = {0, 0};
            const int i_end = p.sched[blockIdx.x + 1];
            for (int i = p.sched[blockIdx.x]; i < i_end; ++i) {
                const int nsteps = warp_uniform(p.items[i].nsteps);
                const bool has_b = warp_uniform(p.items[i].has_b) != 0;
                const PairStep* steps = p.steps + p.items[i].step_off;
                const bool has[2] = {true, has_b};
                bool first_pv[2] = {true, true};
                int last_chunk[2] = {-1, -1};  // this item's last attended chunk per tile
                for (int n = 0; n < nsteps; ++n) {
                    const PairStep ps = steps[n];
                    for (int h = 0; h < 2; ++h) {
                        const int chunk = h ? ps.c1 : ps.c0;
                        if (chunk < 0) continue;
                        const int kc = n * 2 + h;
                        if (has[0] && (h ? ps.a1 : ps.a0)) last_chunk[0] = kc;
                        if (has[1] && (h ? ps.b1 : ps.b0)) last_chunk[1] = kc;
                    }
                }
                last_chunk[0] = warp_uniform(last_chunk[0]);
                last_chunk[1] = warp_uniform(last_chunk[1]);
                PairStep nxt = steps[0];
                for (int n = 0; n < nsteps; ++n) {
                    const PairStep ps = nxt;
                    if (n + 1 < nsteps) nxt = steps[n + 1];
                    for (int h = 0; h < 2; ++h) {
                        const int chunk = warp_uniform(h ? ps.c1 : ps.c0);
                        if (chunk < 0) continue;
                        const uint32_t mk[2] = {warp_uniform(h ? ps.a1 : ps.a0), warp_uniform(h ? ps.b1 : ps.b0)};
                        const int st = kv_it % NST;
                        const uint64_t dv = dVmn0 + static_cast<uint64_t>((st * C::kStageBytes) >> 4);
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            if (!has[t] || !mk[t]) continue;
                            const uint32_t m = p_cnt[t]++;
                            const uint32_t half = m & 1;
                            const uint32_t tS = tmem + t * 256 + half * 64, tO = tmem + t * 256 + 128;
                            S2FTRACE(3 + 10 * t, m);
                            mbar_wait(smem_u32(&bar_pf[t][half]), (m >> 1) & 1);
                            S2FTRACE(12 + 2 * t, m);
                            if (first_pv[t] && o_use[t] > 0) mbar_wait(smem_u32(&bar_oe[t]), (o_use[t] - 1) & 1);
                            tc_fence_after();  // P was written to TMEM by tcgen05.st
                            if (leader) {
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    mma_ts(tO, tS + kk * 8, dv + ((kk * 2048) >> 4), idO,
                                           (first_pv[t] && kk == 0) ? 0u : 1u);
                                mma_commit(smem_u32(&bar_pv[t][half]));
                                // O of tile t is final after its last P V of the item
                                if (n * 2 + h == last_chunk[t]) mma_commit(smem_u32(&bar_of[t]));
                            }
                            __syncwarp();
                            first_pv[t] = false;
                        }
                        // stage st: K was read by the S MMAs (complete: their P existed),
                        // V by the P V just issued
                        if (leader) mma_commit(smem_u32(&bar_ke[st]));
                        __syncwarp();
                        ++kv_it;
                    }
                }
                for (int t = 0; t < 2; ++t)
                    if (has[t]) {
                        if (last_chunk[t] < 0) {  // (a tile with no attended chunk: O is never written)
                            if (leader) mma_commit(smem_u32(&bar_of[t]));
                            __syncwarp();
                        }
                        ++o_use[t];
                    }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;" ::: "memory");
        // ------------------------------------------------------- softmax WGs
        const int t = (warp >> 2) - 1;         // tile 0: warps 4-7, tile 1: warps 8-11
        const int r = tid & 127;               // row in tile == TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 256 + lane_off, tO = tS + 128;
        const int rg = r >> 4;
        const float sl2 = p.scale_log2;
        uint32_t s_cnt = 0, o_cnt = 0, k_cnt = 0;
        for (int i = p.sched[blockIdx.x]; i < p.sched[blockIdx.x + 1]; ++i) {
            const PairItem it = p.items[i];
            if (t == 1 && !it.has_b) continue;
            const PairStep* steps = p.steps + it.step_off;
            const int row0 = (2 * it.qpair + t) * 128;
            const int q_pos = row0 + r;
            float m_run = -INFINITY, l_run = 0.f;
            PairStep nxt = steps[0];  // software-pipelined: step n+1 loads during step n
            for (int n = 0; n < it.nsteps; ++n) {
                const PairStep s = nxt;
                if (n + 1 < it.nsteps) nxt = steps[n + 1];
                for (int hh = 0; hh < 2; ++hh) {
                    const int chunk = hh ? s.c1 : s.c0;
                    const uint32_t msk = t ? (hh ? s.b1 : s.b0) : (hh ? s.a1 : s.a0);
                    if (chunk < 0 || !msk) continue;
                    const uint32_t half = k_cnt & 1;  // S half of this chunk
                    const uint32_t k_here = k_cnt++;
                    if (r == 0) S2FTRACE(4 + 2 * t, s_cnt);
                    mbar_wait(smem_u32(&bar_sf[t][half]), (k_here >> 1) & 1);
                    if (r == 0) S2FTRACE(5 + 2 * t, s_cnt);
                    ++s_cnt;
                    tc_fence_after();
                    float sv[64];
                    {
                        uint32_t* u = reinterpret_cast<uint32_t*>(sv);
                        tmem_ld32(tS + half * 64, *reinterpret_cast<uint32_t(*)[32]>(u));
                        tmem_ld32(tS + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32));
                        tmem_ld_wait();
                    }
                    if (r == 0 && t == 0) S2FTRACE(16, s_cnt - 1);
                    apply_mask(sv, chunk, msk, rg, q_pos, row0);
                    float mxa[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) mxa[k] = fmaxf(sv[k], sv[k + 8]);
#pragma unroll
                    for (int j = 16; j < 64; j += 16)
#pragma unroll
                        for (int k = 0; k < 8; ++k) mxa[k] = fmaxf(mxa[k], fmaxf(sv[j + k], sv[j + k + 8]));
                    const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                                           fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
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
                    if (r == 0 && t == 0) S2FTRACE(17, s_cnt - 1);
                    if (__any_sync(0xffffffffu, rescale)) {
                        // O must hold every earlier chunk's P V before it is rescaled: the
                        // last one issued is this tile's chunk k_here-1 (its (k_here-1)-th
                        // P V overall), still possibly in flight
                        if (k_here > 0)
                            mbar_wait(smem_u32(&bar_pv[t][(k_here - 1) & 1]), ((k_here - 1) >> 1) & 1);
                        tc_fence_after();
                        const float alpha = rescale ? fast_exp2(m_run - m_use) : 1.0f;
                        l_run *= alpha;
#pragma unroll
                        for (int c = 0; c < D / 32; ++c) {
                            uint32_t u[32];
                            tmem_ld32(tO + c * 32, u);
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * alpha);
                            tmem_st32(tO + c * 32, u);
                        }
                    }
                    m_run = m_use;
                    const float base = (m_use == -INFINITY) ? 0.f : m_use;
                    const uint64_t sl2v = f2_pack(sl2, sl2), nbase = f2_pack(-base, -base);
                    uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const uint64_t x = ffma2(f2_pack(sv[c * 32 + 2 * j], sv[c * 32 + 2 * j + 1]), sl2v, nbase);
                            uint64_t pr;
#ifdef S2_FWD_ABLATE_EXP  // timing experiments only (wrong results): no exponentials
                            if (true) {
                                pr = x;
                            } else
#endif
                            if (S2_FWD_POLY_MASK >= 0 && (j & S2_FWD_POLY_MASK) == S2_FWD_POLY_MASK) {  // 1 in (mask+1) on the FMA pipe
                                pr = exp2_poly2(x);
                            } else {
                                float x0, x1;
                                f2_unpack(x, x0, x1);
                                pr = f2_pack(fast_exp2(x0), fast_exp2(x1));
                            }
                            acc[j & 3] = fadd2(acc[j & 3], pr);
                            float p0, p1;
                            f2_unpack(pr, p0, p1);
                            pk[j] = pack_bf16(p0, p1);
                        }
                        tmem_st16(tS + half * 64 + c * 16, pk);
                    }
                    {
                        float a0, a1;
                        f2_unpack(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])), a0, a1);
                        l_run += a0 + a1;
                    }
                    if (r == 0 && t == 0) S2FTRACE(18, s_cnt - 1);
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(smem_u32(&bar_pf[t][half]));
                    if (r == 0 && t == 0) S2FTRACE(8, s_cnt - 1);
                }
            }
            // ---------------------------------------------------- epilogue
            // O -> registers (then its TMEM is released to the next item), x 1/l as
            // bf16 into this tile's swizzled staging slice, one TMA store per 64
            // columns (rows past seq_len are clipped by the tensor map)
            if (r == 0 && t == 0) S2FTRACE(9, o_cnt);
            mbar_wait(smem_u32(&bar_of[t]), o_cnt & 1);
            if (r == 0 && t == 0) S2FTRACE(10, o_cnt);
            tc_fence_after();
            uint32_t ov[D];
#pragma unroll
            for (int c = 0; c < D / 32; ++c) tmem_ld32(tO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(ov + 32 * c));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(smem_u32(&bar_oe[t]));
            // a row with no admitted key: out = 0/0 = NaN, lse = -inf (the reference's
            // acc / l); explicit, since a tile without any chunk never wrote its O
            const float inv_l = l_run > 0.f ? 1.0f / l_run : __int_as_float(0x7fc00000);
            const uint32_t stg = sStg + t * C::kStgBytes;
            // data index of this tile's head in the ranks' full outputs (fused exchange)
            const int bh_out = px.num_peers ? px.unit_global[it.bh / p.hpg] * p.hpg + it.bh % p.hpg : it.bh;
#pragma unroll
            for (int j = 0; j < D / 64; ++j) {
                if (r == 0) bulk_wait_read0();  // the previous store has read the slice
                named_bar_sync(1 + t, 128);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t* u = ov + j * 64 + c * 8;
                    sts_u4(stg + r * 128 + ((c ^ (r & 7)) << 4),
                           pack_bf16(__uint_as_float(u[0]) * inv_l, __uint_as_float(u[1]) * inv_l),
                           pack_bf16(__uint_as_float(u[2]) * inv_l, __uint_as_float(u[3]) * inv_l),
                           pack_bf16(__uint_as_float(u[4]) * inv_l, __uint_as_float(u[5]) * inv_l),
                           pack_bf16(__uint_as_float(u[6]) * inv_l, __uint_as_float(u[7]) * inv_l));
                }
                fence_proxy_async_smem();
                named_bar_sync(1 + t, 128);
                if (r == 0) {
                    tma_store_3d(&tmO, stg, j * 64, row0, it.bh);
                    for (int pr = 0; pr < px.num_peers; ++pr)  // the same tile into every rank's output
                        tma_store_3d(&px.peer_o[pr], stg, j * 64, row0, bh_out);
                    bulk_commit();
                }
            }
            if (q_pos < p.seq_len) {
                const float lse_v = (m_run + __log2f(l_run)) * 0.69314718055994530942f;
                p.lse[static_cast<size_t>(it.bh) * p.seq_len + q_pos] = lse_v;
                for (int pr = 0; pr < px.num_peers; ++pr)
                    px.peer_lse[pr][static_cast<size_t>(bh_out) * p.seq_len + q_pos] = lse_v;
            }
            if (r == 0 && t == 0) S2FTRACE(11, o_cnt);
            ++o_cnt;
        }
        if (r == 0) bulk_wait0();  // the staging slice must outlive the stores
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
static cudaError_t launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                          const CUtensorMap& o, const Fwd2Params& p, const FwdPeers& px, int grid,
                          cudaStream_t stream) {
    if (px.num_peers == 0) {
        auto kern = s2_fwd_sm100_kernel<D, false>;
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg<D>::kSmem);
        if (e != cudaSuccess) return e;
        return launch_pdl(kern, dim3(grid), dim3(384), Fwd2Cfg<D>::kSmem, stream, q, k, v, o, p, NoPeers{});
    }
    auto kern = s2_fwd_sm100_kernel<D, true>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg<D>::kSmem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(grid), dim3(384), Fwd2Cfg<D>::kSmem, stream, q, k, v, o, p, px);
}

}  // namespace s2dev

// Host entry used by capi.cpp: items grouped per CTA, sched = [grid + 1] offsets.
long long* s2_debug_trace_buffer();
cudaError_t s2_launch_fwd_sm100(int head_dim, const CUtensorMap& q, const CUtensorMap& k,
                                const CUtensorMap& v, const CUtensorMap& o, const void* items, const int* sched,
                                int grid, const void* steps, __nv_bfloat16* out, float* lse,
                                int seq_len, int hpg, float scale_log2, cudaStream_t stream,
                                int num_peers, const int* unit_global, float* const* peer_lse,
                                const CUtensorMap* peer_o) {
    if (grid == 0) return cudaSuccess;
    if (num_peers < 0 || num_peers > s2dev::kMaxPeers) return cudaErrorInvalidValue;
    s2dev::Fwd2Params p{static_cast<const s2dev::PairItem*>(items), sched,
                        static_cast<const s2dev::PairStep*>(steps), out, lse, seq_len, hpg,
                        scale_log2, s2_debug_trace_buffer()};
    s2dev::FwdPeers px{};
    px.num_peers = num_peers;
    px.unit_global = unit_global;
    for (int r = 0; r < num_peers; ++r) {
        px.peer_lse[r] = peer_lse[r];
        px.peer_o[r] = peer_o[r];
    }
    if (head_dim == 128) return s2dev::launch<128>(q, k, v, o, p, px, grid, stream);
    if (head_dim == 64) return s2dev::launch<64>(q, k, v, o, p, px, grid, stream);
    return cudaErrorInvalidValue;
}
