// C ABI of include/s2attn.h: layout builder, plans, forward, partitioner.
// (backward: capi_bwd.cpp, decode: capi_decode.cpp)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>

#include "capi_internal.hpp"
#include "tma_host.hpp"

cudaError_t s2_launch_fwd_sm100(int head_dim, const CUtensorMap& q, const CUtensorMap& k,
                                const CUtensorMap& v, const CUtensorMap& o, const void* items, const int* sched,
                                int grid, const void* steps, __nv_bfloat16* out, float* lse,
                                int seq_len, int hpg, float scale_log2, cudaStream_t stream,
                                int num_peers, const int* unit_global, float* const* peer_lse,
                                const CUtensorMap* peer_o);
int s2_fwd_pair2_clusters();
cudaError_t s2_launch_fwd_pair2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                                const CUtensorMap& o, const void* items, const int* sched, int clusters,
                                const void* steps, float* lse, int seq_len, int hpg, float scale_log2,
                                cudaStream_t stream);
cudaError_t s2_launch_fwd_simt(bool bf16, const void* q, const void* k, const void* v, void* out,
                               float* lse, const int* bh_list, const int* head_of, int num_bh,
                               const int* row_ptr, const int* col_idx, const int64_t* col_off,
                               int N, int D, int S, int B, int hpg, float scale,
                               cudaStream_t stream);

namespace s2 {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? S2_ERR_OUT_OF_MEMORY : S2_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

cudaError_t upload(DevBuf& buf, const void* host, size_t bytes) {
    if (buf.ptr) {
        cudaFree(buf.ptr);
        buf.ptr = nullptr;
    }
    cudaGetDevice(&buf.device);
    buf.bytes = bytes;
    cudaError_t e = cudaMalloc(&buf.ptr, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return e;
    if (bytes) e = cudaMemcpy(buf.ptr, host, bytes, cudaMemcpyHostToDevice);
    return e;
}

static std::string check_cfg_ptr(const s2_pattern_config* cfg) {
    if (!cfg) return "config is null";
    if (cfg->num_segments < 0 || cfg->num_segments > S2_MAX_SEGMENTS)
        return "num_segments must lie in [0, S2_MAX_SEGMENTS]";
    for (int s = 0; s < cfg->num_segments; ++s)
        if (cfg->segments[s].num_offsets > 0 && !cfg->segments[s].offsets)
            return "segment offsets pointer is null";
    return "";
}

#define S2_CHECK_CFG(cfg)                                             \
    do {                                                              \
        std::string m_ = check_cfg_ptr(cfg);                          \
        if (m_.empty()) m_ = validate(from_c(cfg));                   \
        if (!m_.empty()) return fail(S2_ERR_INVALID_ARGUMENT, m_);    \
    } while (0)

int ensure_csr_uploaded(s2_plan* p) {
    if (int rc = check_device(p)) return rc;
    if (p->device < 0) cudaGetDevice(&p->device);
    if (p->csr_uploaded) return S2_OK;
    const int H = p->num_heads, B = p->num_blocks;
    std::vector<int> rp(static_cast<size_t>(H) * (B + 1));
    std::vector<int> ci;
    for (int h = 0; h < H; ++h) {
        std::copy(p->csr[h].ptr.begin(), p->csr[h].ptr.end(), rp.begin() + static_cast<size_t>(h) * (B + 1));
        ci.insert(ci.end(), p->csr[h].idx.begin(), p->csr[h].idx.end());
    }
    cudaError_t e;
    if ((e = upload(p->d_row_ptr, rp.data(), rp.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(p->d_col_idx, ci.data(), ci.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(p->d_col_off, p->col_off.data(), p->col_off.size() * sizeof(int64_t))) !=
            cudaSuccess)
        return cuda_fail(e, "uploading CSR");
    p->csr_uploaded = true;
    return S2_OK;
}

// the transposed lists of every head (ascending query blocks per key block), as
// s2_layout_build_csc / the reference's to_csr of the transposed mask
int ensure_csc_uploaded(s2_plan* p) {
    if (int rc = check_device(p)) return rc;
    if (p->device < 0) cudaGetDevice(&p->device);
    if (p->csc_uploaded) return S2_OK;
    const int H = p->num_heads, B = p->num_blocks;
    std::vector<int> cp(static_cast<size_t>(H) * (B + 1), 0);
    std::vector<int> ri;
    std::vector<int64_t> off(H);
    for (int h = 0; h < H; ++h) {
        const Csr& c = p->csr[h];
        int* col = cp.data() + static_cast<size_t>(h) * (B + 1);
        for (int x : c.idx) ++col[x + 1];
        for (int b = 0; b < B; ++b) col[b + 1] += col[b];
        off[h] = static_cast<int64_t>(ri.size());
        ri.resize(ri.size() + c.idx.size());
        std::vector<int> fill(col, col + B);
        for (int r = 0; r < B; ++r)  // rows ascending -> each column's rows ascending
            for (int e = c.ptr[r]; e < c.ptr[r + 1]; ++e) ri[off[h] + fill[c.idx[e]]++] = r;
    }
    cudaError_t e;
    if ((e = upload(p->d_col_ptr, cp.data(), cp.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(p->d_row_idx, ri.data(), ri.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(p->d_row_off, off.data(), off.size() * sizeof(int64_t))) != cudaSuccess)
        return cuda_fail(e, "uploading CSC");
    p->csc_uploaded = true;
    return S2_OK;
}

int check_device(const s2_plan* p) {
    if (p->device < 0) return S2_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != p->device)
        return fail(S2_ERR_INVALID_ARGUMENT, "plan was first used on device " + std::to_string(p->device) +
                                                 "; its device-side lists cannot serve device " +
                                                 std::to_string(cur) + " (create one plan per device)");
    return S2_OK;
}

Lists* get_lists(s2_plan* p, int seq_len, int* status) {
    if ((*status = check_device(p)) != S2_OK) return nullptr;
    if (p->device < 0) cudaGetDevice(&p->device);
    auto it = p->lists.find(seq_len);
    Lists* L;
    if (it == p->lists.end()) {
        auto nl = std::make_unique<Lists>();
        nl->tiled = p->block_size % 16 == 0;
        if (nl->tiled) {
            nl->fwd = build_fwd_list(p->csr, seq_len, p->block_size);
            nl->pairs = build_pair_list(nl->fwd, p->num_heads);
            nl->bwd = build_bwd_list(nl->fwd, p->num_heads, p->num_kv_heads, seq_len);
        }
        L = nl.get();
        p->lists[seq_len] = std::move(nl);
    } else {
        L = it->second.get();
    }
    if (L->tiled && !L->uploaded) {
        static_assert(sizeof(ChunkEntry) == 8, "ChunkEntry layout");
        static_assert(sizeof(BwdEntry) == sizeof(s2dev::BwdEntry), "BwdEntry layout");
        cudaError_t e;
        static_assert(sizeof(PairStep) == 24, "PairStep layout");
        if ((e = upload(L->d_chunks, L->fwd.chunks.data(), L->fwd.chunks.size() * 8)) != cudaSuccess ||
            (e = upload(L->d_steps, L->pairs.steps.data(), L->pairs.steps.size() * sizeof(PairStep))) !=
                cudaSuccess ||
            (e = upload(L->d_entries, L->bwd.entries.data(),
                        L->bwd.entries.size() * sizeof(BwdEntry))) != cudaSuccess) {
            *status = cuda_fail(e, "uploading tile lists");
            return nullptr;
        }
        L->uploaded = true;
    }
    *status = S2_OK;
    return L;
}

// Static persistent-CTA schedule (greedy list scheduling: each item goes to
// the CTA whose queue finishes earliest).  Items are visited in cost
// classes, heaviest class first (LPT: the tail is made of the lightest
// items), and head-major inside a class, so CTAs sweep the heads of one class
// together and a head's K/V (or Q/dO) stays L2-resident while they do.  A
// class spans a factor of 2^(1/4) in cost.  `overhead` is the fixed per-item
// cost (operand loads, epilogue) in the same unit as `cost`.  Returns the
// items regrouped per CTA plus offsets [grid + 1].
template <class T, class Cost, class Key>
static std::vector<int32_t> schedule_items(std::vector<T>& items, int grid, Cost cost, Key key,
                                           int64_t overhead, int key_group = 0) {
    auto cls = [&](const T& a) {
        const double c = static_cast<double>(cost(a) + overhead);
        return static_cast<int>(std::floor(4.0 * std::log2(std::max(1.0, c))));
    };
    // key_group > 0: keys (heads) are swept in groups of key_group, LPT inside a group
    // (bounds the L2 working set of streamed operands to a group's heads)
    auto grp = [&](const T& a) { return key_group > 0 ? static_cast<int64_t>(key(a)) / key_group : 0; };
    std::stable_sort(items.begin(), items.end(), [&](const T& a, const T& b) {
        const auto ga = grp(a), gb = grp(b);
        if (ga != gb) return ga < gb;
        const int ca = cls(a), cb = cls(b);
        if (ca != cb) return ca > cb;
        const auto ka = key(a), kb = key(b);
        if (ka != kb) return ka < kb;
        return cost(a) > cost(b);
    });
    std::vector<std::vector<T>> per(grid);
    std::vector<std::pair<int64_t, int>> heap;  // (finish time, cta) min-heap
    for (int c = 0; c < grid; ++c) heap.push_back({0, c});
    std::make_heap(heap.begin(), heap.end(), std::greater<>());
    for (const T& it : items) {
        std::pop_heap(heap.begin(), heap.end(), std::greater<>());
        auto& top = heap.back();
        per[top.second].push_back(it);
        top.first += cost(it) + overhead;
        std::push_heap(heap.begin(), heap.end(), std::greater<>());
    }
    std::vector<int32_t> off(grid + 1, 0);
    items.clear();
    for (int c = 0; c < grid; ++c) {
        items.insert(items.end(), per[c].begin(), per[c].end());
        off[c + 1] = static_cast<int32_t>(items.size());
    }
    return off;
}

// The CTA-pair forward (fwd_pair2.cu) serves head_dim 128 when S2_FWD_2CTA=1
// (opt-in until it beats the 1-CTA pair kernel on cfg3).
static bool pair2_enabled() {
    const char* e = getenv("S2_FWD_2CTA");
    return e && e[0] == '1';
}

// dK/dV schedule: units (kv heads) are swept in groups, LPT inside a group, so the
// Q / dO rows the CTAs stream concurrently belong to fewer heads and stay in L2.
// Default: two halves once there are 16+ units (cfg3: dK/dV 1.26 -> 1.23 ms; four or
// more groups lose to the LPT imbalance at group boundaries).  S2_DKV_GROUP=<units
// per group> overrides, 0 = one group.
static int dkv_group(int num_units) {
    const char* e = getenv("S2_DKV_GROUP");
    if (e) return atoi(e);
    return num_units >= 16 ? (num_units + 1) / 2 : 0;
}

// per-item overhead of the LPT cost model, in step units (tuning knob: env
// S2_SCHED_OVH_<kind>)
static int64_t sched_overhead(const char* env, int64_t dflt) {
    const char* e = getenv(env);
    return e ? atoll(e) : dflt;
}

// Units are (batch, kv-group); local data index of query head j of the
// ui-th listed unit is ui*hpg + j (= b*H + h when every unit is listed).
WorkItems* get_items(s2_plan* p, Lists* L, int batch, int num_units, const int* unit_ids,
                     int* status) {
    // the forward fills every SM; the backward kernels leave s2_set_sm_reserve SMs
    // to the collective that overlaps them (the all-gather of O)
    const int grid_fwd = num_sms(), grid = persistent_grid();
    std::string key = std::to_string(batch) + ":g" + std::to_string(grid_fwd) + "/" + std::to_string(grid) +
                      (pair2_enabled() ? "p2" : "") + ":";
    std::vector<int> units;
    if (unit_ids) {
        units.assign(unit_ids, unit_ids + num_units);
        for (int u : units) key += std::to_string(u) + ",";
    } else {
        units.resize(static_cast<size_t>(batch) * p->num_kv_heads);
        std::iota(units.begin(), units.end(), 0);
        key += "all";
    }
    auto it = L->items.find(key);
    if (it != L->items.end()) {
        *status = S2_OK;
        return it->second.get();
    }
    auto w = std::make_unique<WorkItems>();
    const int hpg = p->num_heads / p->num_kv_heads;
    std::vector<int> bh, head;
    for (size_t ui = 0; ui < units.size(); ++ui) {
        const int g = units[ui] % p->num_kv_heads;
        for (int j = 0; j < hpg; ++j) {
            bh.push_back(static_cast<int>(ui) * hpg + j);
            head.push_back(g * hpg + j);
        }
    }
    cudaError_t e;
    w->num_bh = static_cast<int>(bh.size());
    if ((e = upload(w->simt_bh, bh.data(), bh.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(w->simt_head, head.data(), head.size() * sizeof(int))) != cudaSuccess) {
        *status = cuda_fail(e, "uploading work items");
        return nullptr;
    }
    if (L->tiled) {
        const int nt = L->fwd.num_qtiles;
        std::vector<s2dev::FwdItem> fi;
        fi.reserve(bh.size() * nt);
        for (size_t i = 0; i < bh.size(); ++i)
            for (int t = 0; t < nt; ++t) {
                const size_t w_ = static_cast<size_t>(head[i]) * nt + t;
                const int64_t off = L->fwd.offset[w_];
                const int cnt = static_cast<int>(L->fwd.offset[w_ + 1] - off);
                fi.push_back({bh[i], head[i], t, cnt, off});
            }
        const std::vector<int32_t> off_fwd = schedule_items(
            fi, grid, [](const s2dev::FwdItem& a) { return int64_t(a.chunk_cnt); },
            [](const s2dev::FwdItem& a) { return a.bh; }, sched_overhead("S2_SCHED_OVH_DQ", 2));
        struct PairItem {
            int32_t bh, qpair, nsteps, has_b;
            int64_t step_off;
        };
        std::vector<PairItem> pi;
        const int np = L->pairs.num_pairs;
        for (size_t i = 0; i < bh.size(); ++i)
            for (int q = 0; q < np; ++q) {
                const size_t w_ = static_cast<size_t>(head[i]) * np + q;
                const int64_t off = L->pairs.offset[w_];
                pi.push_back({bh[i], q, static_cast<int32_t>(L->pairs.offset[w_ + 1] - off),
                              2 * q + 1 < nt ? 1 : 0, off});
            }
        // CTA-pair forward: both tiles of a pair are computed whatever their masks
        std::vector<PairItem> pi2;
        const int clusters = pair2_enabled() ? s2_fwd_pair2_clusters() : 0;
        if (clusters > 0) {
            pi2 = pi;
            const std::vector<int32_t> off2 = schedule_items(
                pi2, clusters, [](const PairItem& a) { return int64_t(a.nsteps) * 2; },
                [](const PairItem& a) { return a.bh; }, sched_overhead("S2_SCHED_OVH_FWD2", 3));
            w->clusters = clusters;
            w->num_pair2 = static_cast<int>(pi2.size());
            if ((e = upload(w->pair2, pi2.data(), pi2.size() * sizeof(PairItem))) != cudaSuccess ||
                (e = upload(w->pair2_sched, off2.data(), off2.size() * sizeof(int32_t))) != cudaSuccess) {
                *status = cuda_fail(e, "uploading work items");
                return nullptr;
            }
        }
        const std::vector<int32_t> off_pair = schedule_items(
            pi, grid_fwd, [](const PairItem& a) { return int64_t(a.nsteps) * (1 + a.has_b); },
            [](const PairItem& a) { return a.bh; }, sched_overhead("S2_SCHED_OVH_FWD", 4));
        w->num_pair = static_cast<int>(pi.size());
        if ((e = upload(w->pair, pi.data(), pi.size() * sizeof(PairItem))) != cudaSuccess ||
            (e = upload(w->pair_sched, off_pair.data(), off_pair.size() * sizeof(int32_t))) != cudaSuccess ||
            (e = upload(w->fwd_sched, off_fwd.data(), off_fwd.size() * sizeof(int32_t))) != cudaSuccess) {
            *status = cuda_fail(e, "uploading work items");
            return nullptr;
        }
        std::vector<s2dev::BwdItem> bi;
        for (size_t ui = 0; ui < units.size(); ++ui) {
            const int g = units[ui] % p->num_kv_heads;
            for (const BwdTile& t : L->bwd.tiles)
                if (t.group == g) bi.push_back({static_cast<int>(ui), t.c0, t.c1, t.count, t.offset, 0, 0});
        }
        // dK/dV cost: 64-row q halves the kernel steps through (a half with
        // no mask bit in either chunk is skipped) for every head of the group.
        std::unordered_map<int64_t, int64_t> halves;  // tile entry offset -> active halves
        for (const BwdTile& t : L->bwd.tiles) {
            int64_t h = 0;
            for (int e = 0; e < t.count; ++e) {
                const BwdEntry& en = L->bwd.entries[t.offset + e];
                const uint32_t m = en.mask0 | en.mask1;
                h += ((m & 0xFFFFu) != 0) + ((m >> 16) != 0);
            }
            halves[t.offset] = h;
        }
        // 128-row kernel: q tiles with a mask bit in either chunk
        std::unordered_map<int64_t, int64_t> tiles;
        for (const BwdTile& t : L->bwd.tiles) {
            int64_t n = 0;
            for (int e = 0; e < t.count; ++e) {
                const BwdEntry& en = L->bwd.entries[t.offset + e];
                n += (en.mask0 | en.mask1) != 0;
            }
            tiles[t.offset] = n;
        }
        for (auto& it : bi) {
            it.nsteps = static_cast<int32_t>(halves.at(it.offset) * hpg);
            it.nsteps128 = static_cast<int32_t>(tiles.at(it.offset) * hpg);
        }
        const size_t nb_all = bi.size();
        bi.erase(std::remove_if(bi.begin(), bi.end(), [](const s2dev::BwdItem& a) { return a.nsteps == 0; }),
                 bi.end());
        w->bwd_dropped = bi.size() != nb_all;
        auto bwd_cost = [](const s2dev::BwdItem& a) { return int64_t(a.nsteps); };
        const std::vector<int32_t> off_bwd = schedule_items(
            bi, grid, bwd_cost, [](const s2dev::BwdItem& a) { return a.kvbh; }, sched_overhead("S2_SCHED_OVH_DKV", 4),
            dkv_group(static_cast<int>(units.size())));
        w->num_fwd = static_cast<int>(fi.size());
        w->num_bwd = static_cast<int>(bi.size());
        w->grid = grid;
        w->grid_fwd = grid_fwd;
        if ((e = upload(w->fwd, fi.data(), fi.size() * sizeof(s2dev::FwdItem))) != cudaSuccess ||
            (e = upload(w->bwd, bi.data(), bi.size() * sizeof(s2dev::BwdItem))) != cudaSuccess ||
            (e = upload(w->bwd_sched, off_bwd.data(), off_bwd.size() * sizeof(int32_t))) != cudaSuccess) {
            *status = cuda_fail(e, "uploading work items");
            return nullptr;
        }
    }
    WorkItems* out = w.get();
    L->items[key] = std::move(w);
    *status = S2_OK;
    return out;
}

// Shared validation of s2_attn_args against the plan (kernel_common.hpp:20-32,
// attention.cpp:102-110).
int check_args(const s2_plan* p, const s2_attn_args* a) {
    if (!p) return fail(S2_ERR_INVALID_ARGUMENT, "plan is null");
    if (!a) return fail(S2_ERR_INVALID_ARGUMENT, "args is null");
    if (a->batch < 1 || a->num_heads < 1 || a->seq_len < 1 || a->head_dim < 1)
        return fail(S2_ERR_INVALID_ARGUMENT, "tensor dimensions must be positive");
    if (a->num_heads != p->num_heads) return fail(S2_ERR_INVALID_ARGUMENT, "one mask per head required");
    const int hkv = a->num_kv_heads > 0 ? a->num_kv_heads : a->num_heads;
    if (hkv != p->num_kv_heads)
        return fail(S2_ERR_INVALID_ARGUMENT, "num_kv_heads does not match the plan");
    if ((a->seq_len + p->block_size - 1) / p->block_size != p->num_blocks)
        return fail(S2_ERR_INVALID_ARGUMENT,
                    "mask block count does not match ceil(seq_len/block_size)");
    if (a->num_splits < 1 || a->head_dim % a->num_splits != 0)
        return fail(S2_ERR_INVALID_ARGUMENT, "num_splits must divide head_dim");
    if (a->dtype != S2_DTYPE_BF16 && a->dtype != S2_DTYPE_F32)
        return fail(S2_ERR_INVALID_ARGUMENT, "unknown dtype");
    if (!a->q || !a->k || !a->v || !a->out || !a->lse)
        return fail(S2_ERR_INVALID_ARGUMENT, "q/k/v/out/lse must be non-null device pointers");
    if (a->unit_ids) {
        if (a->num_units < 1) return fail(S2_ERR_INVALID_ARGUMENT, "num_units must be positive");
        for (int i = 0; i < a->num_units; ++i)
            if (a->unit_ids[i] < 0 || a->unit_ids[i] >= a->batch * p->num_kv_heads)
                return fail(S2_ERR_INVALID_ARGUMENT, "unit id outside [0, batch*num_kv_heads)");
    }
    return S2_OK;
}

int num_sms() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

static std::atomic<int> g_sm_reserve{0};

// CTAs of the persistent tcgen05 kernels: one per SM minus the SMs left to
// concurrent work (NCCL's all-gather CTAs on a communication stream), so a
// static schedule never waits for an SM that a collective occupies.
int persistent_grid() { return std::max(1, num_sms() - g_sm_reserve.load()); }

bool use_tcgen05(const s2_plan* p, const s2_attn_args* a) {
    return a->dtype == S2_DTYPE_BF16 && p->block_size % 16 == 0 &&
           (a->head_dim == 64 || a->head_dim == 128);
}

static s2_plan* new_plan_from_csr(std::vector<Csr> csr, int H, int Hkv, int N, int S) {
    auto* p = new s2_plan();
    p->num_heads = H;
    p->num_kv_heads = Hkv;
    p->seq_len = N;
    p->block_size = S;
    p->num_blocks = (N + S - 1) / S;
    p->csr = std::move(csr);
    p->col_off.resize(H);
    int64_t off = 0;
    for (int h = 0; h < H; ++h) {
        p->col_off[h] = off;
        off += p->csr[h].nnz();
    }
    return p;
}

}  // namespace s2

using namespace s2;

extern "C" {

const char* s2_last_error(void) { return g_last_error.c_str(); }

int s2_set_sm_reserve(int sms) {
    if (sms < 0) return fail(S2_ERR_INVALID_ARGUMENT, "sm reserve must be >= 0");
    g_sm_reserve.store(sms);
    return S2_OK;
}
int s2_abi_version(void) { return S2_ABI_VERSION; }

int s2_make_single_stride_config(int seq_len, int block_size, int num_heads, int local_blocks,
                                 int remote_stride, int local_stride, s2_pattern_config* cfg) {
    if (!cfg) return fail(S2_ERR_INVALID_ARGUMENT, "config is null");
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->seq_len = seq_len;
    cfg->block_size = block_size;
    cfg->num_heads = num_heads;
    cfg->num_kv_heads = num_heads;
    cfg->local_blocks = local_blocks;
    cfg->local_stride = local_stride;
    const int B = block_size > 0 ? static_cast<int>((static_cast<long long>(seq_len) + block_size - 1) / block_size) : 0;
    if (local_blocks < B) {
        cfg->num_segments = 1;
        cfg->segments[0].start_block_distance = local_blocks;
        cfg->segments[0].end_block_distance = B;
        cfg->segments[0].stride = remote_stride;
    }
    S2_CHECK_CFG(cfg);
    return S2_OK;
}

int s2_pattern_validate(const s2_pattern_config* cfg) {
    S2_CHECK_CFG(cfg);
    return S2_OK;
}

int s2_pattern_num_blocks(const s2_pattern_config* cfg) {
    return cfg && cfg->block_size > 0 ? from_c(cfg).num_blocks() : 0;
}

int s2_pattern_offset_for(const s2_pattern_config* cfg, int segment, int head, int* offset) {
    S2_CHECK_CFG(cfg);
    if (segment < 0 || segment >= cfg->num_segments)
        return fail(S2_ERR_INVALID_ARGUMENT, "segment index out of range");
    if (head < 0 || head >= cfg->num_heads)
        return fail(S2_ERR_INVALID_ARGUMENT, "head index outside [0, num_heads)");
    *offset = from_c(cfg).offset_for(segment, head);
    return S2_OK;
}

static int check_head(const s2_pattern_config* cfg, int head) {
    if (head < 0 || head >= cfg->num_heads)
        return fail(S2_ERR_INVALID_ARGUMENT,
                    "head index " + std::to_string(head) + " outside [0, num_heads)");
    return S2_OK;
}

int s2_layout_nnz(const s2_pattern_config* cfg, int head, int64_t* nnz) {
    S2_CHECK_CFG(cfg);
    if (int rc = check_head(cfg, head)) return rc;
    const Pattern p = from_c(cfg);
    std::vector<int> row;
    int64_t n = 0;
    for (int i = 0; i < p.num_blocks(); ++i) {
        row_blocks(p, head, i, row);
        n += static_cast<int64_t>(row.size());
    }
    *nnz = n;
    return S2_OK;
}

int s2_layout_build_csr(const s2_pattern_config* cfg, int head, int* row_ptr, int* col_idx) {
    S2_CHECK_CFG(cfg);
    if (int rc = check_head(cfg, head)) return rc;
    if (!row_ptr || !col_idx) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    const Csr c = build_csr(from_c(cfg), head);
    std::copy(c.ptr.begin(), c.ptr.end(), row_ptr);
    std::copy(c.idx.begin(), c.idx.end(), col_idx);
    return S2_OK;
}

int s2_layout_build_csc(const s2_pattern_config* cfg, int head, int* col_ptr, int* row_idx) {
    S2_CHECK_CFG(cfg);
    if (int rc = check_head(cfg, head)) return rc;
    if (!col_ptr || !row_idx) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    const Csr c = transpose(build_csr(from_c(cfg), head));
    std::copy(c.ptr.begin(), c.ptr.end(), col_ptr);
    std::copy(c.idx.begin(), c.idx.end(), row_idx);
    return S2_OK;
}

int s2_layout_evict_after(const s2_pattern_config* cfg, int head, int* ev) {
    S2_CHECK_CFG(cfg);
    if (int rc = check_head(cfg, head)) return rc;
    if (!ev) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    const std::vector<int> e = evict_after(transpose(build_csr(from_c(cfg), head)));
    std::copy(e.begin(), e.end(), ev);
    return S2_OK;
}

int s2_layout_kv_efficient(const s2_pattern_config* cfg, int head, int* ok) {
    S2_CHECK_CFG(cfg);
    if (int rc = check_head(cfg, head)) return rc;
    *ok = kv_efficient(transpose(build_csr(from_c(cfg), head))) ? 1 : 0;
    return S2_OK;
}

int s2_csr_validate(int num_blocks, const int* row_ptr, const int* col_idx, int64_t nnz) {
    const std::string m = validate_csr(num_blocks, row_ptr, col_idx, nnz);
    return m.empty() ? S2_OK : fail(S2_ERR_INVALID_ARGUMENT, m);
}

int s2_plan_create(const s2_pattern_config* cfg, s2_plan** out) {
    S2_CHECK_CFG(cfg);
    if (!out) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    try {
        const Pattern pat = from_c(cfg);
        std::vector<Csr> csr(pat.num_heads);
#pragma omp parallel for schedule(dynamic)
        for (int h = 0; h < pat.num_heads; ++h) csr[h] = build_csr(pat, h);
        s2_plan* p = new_plan_from_csr(std::move(csr), pat.num_heads, pat.kv_heads(), pat.seq_len,
                                       pat.block_size);
        p->has_pattern = true;
        p->pattern = pat;
        *out = p;
    } catch (const std::bad_alloc&) {
        return fail(S2_ERR_OUT_OF_MEMORY, "host allocation failed building the layout");
    }
    return S2_OK;
}

int s2_plan_create_from_csr(int num_heads, int num_kv_heads, int seq_len, int block_size,
                            const int* const* row_ptr, const int* const* col_idx, s2_plan** out) {
    if (!out) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    if (num_heads < 1) return fail(S2_ERR_INVALID_ARGUMENT, "csr list is empty");
    if (seq_len < 1) return fail(S2_ERR_INVALID_ARGUMENT, "tensor dimensions must be positive");
    if (block_size < 1) return fail(S2_ERR_INVALID_ARGUMENT, "block_size must be positive");
    const int hkv = num_kv_heads > 0 ? num_kv_heads : num_heads;
    if (num_heads % hkv != 0) return fail(S2_ERR_INVALID_ARGUMENT, "num_kv_heads must divide num_heads");
    if (!row_ptr || !col_idx) return fail(S2_ERR_INVALID_ARGUMENT, "csr pointers are null");
    const int B = (seq_len + block_size - 1) / block_size;
    std::vector<Csr> csr(num_heads);
    for (int h = 0; h < num_heads; ++h) {
        if (!row_ptr[h]) return fail(S2_ERR_INVALID_ARGUMENT, "row_ptr must have num_blocks + 1 entries");
        const int64_t nnz = row_ptr[h][B];
        const std::string m = validate_csr(B, row_ptr[h], col_idx[h], nnz);
        if (!m.empty()) return fail(S2_ERR_INVALID_ARGUMENT, m);
        csr[h].num_blocks = B;
        csr[h].ptr.assign(row_ptr[h], row_ptr[h] + B + 1);
        csr[h].idx.assign(col_idx[h], col_idx[h] + nnz);
    }
    const int hpg = num_heads / hkv;
    for (int h = 0; h < num_heads; ++h) {
        const int lead = (h / hpg) * hpg;
        if (csr[h].ptr != csr[lead].ptr || csr[h].idx != csr[lead].idx)
            return fail(S2_ERR_INVALID_ARGUMENT, "heads of one kv group must share the same mask");
    }
    *out = new_plan_from_csr(std::move(csr), num_heads, hkv, seq_len, block_size);
    return S2_OK;
}

void s2_plan_destroy(s2_plan* plan) { delete plan; }

int s2_plan_get_stats(const s2_plan* cplan, s2_plan_stats* st) {
    if (!cplan || !st) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    auto* p = const_cast<s2_plan*>(cplan);
    std::lock_guard<std::mutex> lk(p->mu);
    std::memset(st, 0, sizeof(*st));
    st->num_heads = p->num_heads;
    st->num_kv_heads = p->num_kv_heads;
    st->seq_len = p->seq_len;
    st->block_size = p->block_size;
    st->num_blocks = p->num_blocks;
    const int64_t B = p->num_blocks;
    for (const Csr& c : p->csr) {
        st->nnz_total += c.nnz();
        st->dense_pairs += B * (B + 1) / 2;
        for (int i = 0; i < c.num_blocks; ++i)
            st->max_row_len = std::max(st->max_row_len, c.ptr[i + 1] - c.ptr[i]);
        const Csr t = transpose(c);
        for (int j = 0; j < t.num_blocks; ++j)
            st->max_col_len = std::max(st->max_col_len, t.ptr[j + 1] - t.ptr[j]);
    }
    if (p->block_size % 16 == 0) {
        auto it = p->lists.find(p->seq_len);
        Lists* L;
        std::unique_ptr<Lists> tmp;
        if (it != p->lists.end()) {
            L = it->second.get();
        } else {
            tmp = std::make_unique<Lists>();
            tmp->fwd = build_fwd_list(p->csr, p->seq_len, p->block_size);
            tmp->bwd = build_bwd_list(tmp->fwd, p->num_heads, p->num_kv_heads, p->seq_len);
            L = tmp.get();
        }
        st->fwd_tiles = static_cast<int64_t>(p->num_heads) * L->fwd.num_qtiles;
        st->fwd_chunk_visits = static_cast<int64_t>(L->fwd.chunks.size());
        st->bwd_tiles = static_cast<int64_t>(L->bwd.tiles.size());
        st->bwd_qtile_visits = static_cast<int64_t>(L->bwd.entries.size());
    }
    return S2_OK;
}

int s2_plan_fwd_tiles(s2_plan* p, int* num_qtiles, int64_t* num_entries, int64_t* offsets,
                      int32_t* chunks, uint32_t* masks) {
    if (!p || !num_qtiles || !num_entries) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (p->block_size % 16 != 0)
        return fail(S2_ERR_UNSUPPORTED, "tile lists need block_size % 16 == 0");
    std::lock_guard<std::mutex> lk(p->mu);
    auto it = p->lists.find(p->seq_len);
    if (it == p->lists.end()) {
        // the same complete entry get_lists() builds (a later forward reuses it)
        auto nl = std::make_unique<Lists>();
        nl->tiled = true;
        nl->fwd = build_fwd_list(p->csr, p->seq_len, p->block_size);
        nl->pairs = build_pair_list(nl->fwd, p->num_heads);
        nl->bwd = build_bwd_list(nl->fwd, p->num_heads, p->num_kv_heads, p->seq_len);
        it = p->lists.emplace(p->seq_len, std::move(nl)).first;
    }
    const FwdList& f = it->second->fwd;
    *num_qtiles = f.num_qtiles;
    *num_entries = static_cast<int64_t>(f.chunks.size());
    if (offsets) std::copy(f.offset.begin(), f.offset.end(), offsets);
    if (chunks)
        for (size_t i = 0; i < f.chunks.size(); ++i) chunks[i] = f.chunks[i].chunk;
    if (masks)
        for (size_t i = 0; i < f.chunks.size(); ++i) masks[i] = f.chunks[i].mask;
    return S2_OK;
}

int s2_plan_bwd_tiles(s2_plan* p, int64_t* num_tiles, int64_t* num_entries, int64_t* tiles,
                      int64_t* entries) {
    if (!p || !num_tiles || !num_entries) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    int nq = 0;
    int64_t ne = 0;
    if (int rc = s2_plan_fwd_tiles(p, &nq, &ne, nullptr, nullptr, nullptr)) return rc;
    std::lock_guard<std::mutex> lk(p->mu);
    const BwdList& b = p->lists.at(p->seq_len)->bwd;
    *num_tiles = static_cast<int64_t>(b.tiles.size());
    *num_entries = static_cast<int64_t>(b.entries.size());
    if (tiles)
        for (size_t i = 0; i < b.tiles.size(); ++i) {
            tiles[5 * i + 0] = b.tiles[i].group;
            tiles[5 * i + 1] = b.tiles[i].c0;
            tiles[5 * i + 2] = b.tiles[i].c1;
            tiles[5 * i + 3] = b.tiles[i].offset;
            tiles[5 * i + 4] = b.tiles[i].count;
        }
    if (entries)
        for (size_t i = 0; i < b.entries.size(); ++i) {
            entries[3 * i + 0] = b.entries[i].qtile;
            entries[3 * i + 1] = b.entries[i].mask0;
            entries[3 * i + 2] = b.entries[i].mask1;
        }
    return S2_OK;
}

int s2_plan_head_nnz(const s2_plan* p, int head, int64_t* nnz) {
    if (!p || !nnz) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (head < 0 || head >= p->num_heads) return fail(S2_ERR_INVALID_ARGUMENT, "head out of range");
    *nnz = p->csr[head].nnz();
    return S2_OK;
}

int s2_plan_fwd_flops(const s2_plan* p, int batch, int head_dim, double* active, double* dense) {
    if (!p) return fail(S2_ERR_INVALID_ARGUMENT, "plan is null");
    if (batch < 1 || head_dim < 1) return fail(S2_ERR_INVALID_ARGUMENT, "head_dim must be positive");
    const double per_pair = 4.0 * head_dim * double(p->block_size) * p->block_size;  // analysis.cpp:29-31
    int64_t nnz = 0;
    for (const Csr& c : p->csr) nnz += c.nnz();
    const double B = p->num_blocks;
    if (active) *active = per_pair * double(nnz) * batch;
    if (dense) *dense = per_pair * B * (B + 1) / 2.0 * p->num_heads * batch;
    return S2_OK;
}

int s2_plan_unit_weights(const s2_plan* p, int batch, int64_t* w) {
    if (!p || !w) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (batch < 1) return fail(S2_ERR_INVALID_ARGUMENT, "batch must be positive");
    const int hpg = p->num_heads / p->num_kv_heads;
    for (int b = 0; b < batch; ++b)
        for (int g = 0; g < p->num_kv_heads; ++g) {
            int64_t s = 0;
            for (int j = 0; j < hpg; ++j) s += p->csr[g * hpg + j].nnz();
            w[b * p->num_kv_heads + g] = s;
        }
    return S2_OK;
}

int s2_partition_lpt(int num_units, const int64_t* weights, int num_ranks, int* owner,
                     int64_t* load) {
    if (num_units < 0 || num_ranks < 1) return fail(S2_ERR_INVALID_ARGUMENT, "bad unit/rank count");
    if (num_units > 0 && (!weights || !owner)) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    partition_lpt(num_units, weights, num_ranks, owner, load);
    return S2_OK;
}

static int attn_fwd_impl(s2_plan* p, const s2_attn_args* a, int num_peers, void* const* peer_out,
                         float* const* peer_lse, const int* unit_global, int total_units,
                         s2_stream_t stream) {
    if (int rc = check_args(p, a)) return rc;
    std::lock_guard<std::mutex> lk(p->mu);
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const double scale = resolve_scale(a->scale, a->head_dim);
    const int hpg = p->num_heads / p->num_kv_heads;
    int rc = S2_OK;
    Lists* L = get_lists(p, a->seq_len, &rc);
    if (!L) return rc;
    WorkItems* w = get_items(p, L, a->batch, a->num_units, a->unit_ids, &rc);
    if (!w) return rc;
    const int nu = a->unit_ids ? a->num_units : a->batch * p->num_kv_heads;
    cudaError_t e;
    if (num_peers > 0 && !use_tcgen05(p, a))
        return fail(S2_ERR_UNSUPPORTED, "the fused output exchange needs the bf16 tcgen05 path");
    if (use_tcgen05(p, a)) {
        try {
            const uint64_t N = a->seq_len, D = a->head_dim;
            // loads: whole-row 4-D boxes (one TMA per 128-row Q tile / 64-key chunk)
            const CUtensorMap mq = s2host::make_map_bf16_kmajor(a->q, D, N, uint64_t(nu) * hpg, 128);
            const CUtensorMap mk = s2host::make_map_bf16_kmajor(a->k, D, N, nu, 64);
            const CUtensorMap mv = s2host::make_map_bf16_kmajor(a->v, D, N, nu, 64);
            const CUtensorMap mo = s2host::make_map_bf16_3d(a->out, D, N, uint64_t(nu) * hpg, 64, 128);
            CUtensorMap peer_maps[8];
            for (int r = 0; r < num_peers; ++r)
                peer_maps[r] = s2host::make_map_bf16_3d(peer_out[r], D, N, uint64_t(total_units) * hpg, 64, 128);
            if (num_peers == 0 && D == 128 && w->clusters > 0) {
                // CTA pairs: V as 64-column boxes (each CTA holds its D half of a chunk)
                const CUtensorMap mv2 = s2host::make_map_bf16_3d(a->v, D, N, nu, 64, 64);
                ProfScope prof("fwd_sm100", st);
                e = s2_launch_fwd_pair2(mq, mk, mv2, mo, w->pair2.ptr, w->pair2_sched.as<int>(), w->clusters,
                                        L->d_steps.ptr, a->lse, a->seq_len, hpg, float(scale * M_LOG2E), st);
                if (e != cudaSuccess) return cuda_fail(e, "s2_attn_fwd launch");
                return S2_OK;
            }
            ProfScope prof("fwd_sm100", st);
            e = s2_launch_fwd_sm100(a->head_dim, mq, mk, mv, mo, w->pair.ptr, w->pair_sched.as<int>(),
                                    w->grid_fwd, L->d_steps.ptr, static_cast<__nv_bfloat16*>(a->out),
                                    a->lse, a->seq_len, hpg, float(scale * M_LOG2E), st, num_peers,
                                    unit_global, peer_lse, peer_maps);
        } catch (const std::exception& ex) {
            return fail(S2_ERR_CUDA, ex.what());
        }
    } else {
        if (a->head_dim > 2048)
            return fail(S2_ERR_UNSUPPORTED, "head_dim > 2048 is not supported");
        if ((rc = ensure_csr_uploaded(p))) return rc;
        ProfScope prof("fwd_simt", st);
        e = s2_launch_fwd_simt(a->dtype == S2_DTYPE_BF16, a->q, a->k, a->v, a->out, a->lse,
                               w->simt_bh.as<int>(), w->simt_head.as<int>(), w->num_bh,
                               p->d_row_ptr.as<int>(), p->d_col_idx.as<int>(),
                               p->d_col_off.as<int64_t>(), a->seq_len, a->head_dim, p->block_size,
                               p->num_blocks, hpg, float(scale), st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "s2_attn_fwd launch");
    return S2_OK;
}

int s2_attn_fwd(s2_plan* p, const s2_attn_args* a, s2_stream_t stream) {
    return attn_fwd_impl(p, a, 0, nullptr, nullptr, nullptr, 0, stream);
}

int s2_attn_fwd_peers(s2_plan* p, const s2_attn_args* a, int num_peers, void* const* peer_out,
                      float* const* peer_lse, const int* unit_global, int total_units,
                      s2_stream_t stream) {
    if (num_peers < 1 || num_peers > 8)
        return fail(S2_ERR_INVALID_ARGUMENT, "num_peers must be in [1, 8]");
    if (!peer_out || !peer_lse || !unit_global || !a || !a->unit_ids)
        return fail(S2_ERR_INVALID_ARGUMENT,
                    "peer_out, peer_lse, unit_global and the local unit_ids are required");
    if (total_units < a->num_units)
        return fail(S2_ERR_INVALID_ARGUMENT, "total_units is smaller than the local unit count");
    for (int r = 0; r < num_peers; ++r)
        if (!peer_out[r] || !peer_lse[r])
            return fail(S2_ERR_INVALID_ARGUMENT, "null peer buffer");
    return attn_fwd_impl(p, a, num_peers, peer_out, peer_lse, unit_global, total_units, stream);
}

}  // extern "C"
