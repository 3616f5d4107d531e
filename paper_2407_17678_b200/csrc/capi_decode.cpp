// C ABI: compacted KV cache + sparse decode (s2_kvcache_*, s2_attn_decode*).
//
// Slot bookkeeping follows simulate_decode_cache (analysis.cpp:57-104): key
// block j is stored from its generation (row j) until row evict_after[j]
// (:76-82); afterwards its slot is reused.  Only KV-efficient masks
// (verify.cpp:53-72, e.g. any single-stride config with local_stride 1) are
// accepted, for which the stored set at row bt is exactly row bt of the mask.
#include <algorithm>
#include <cmath>
#include <queue>
#include <vector>

#include "capi_internal.hpp"
#include "tma_host.hpp"

namespace s2dev {
}  // namespace s2dev

cudaError_t s2_launch_decode(const CUtensorMap& mk, const CUtensorMap& mv,
                             const s2dev::DecodeParams& p, int batch, cudaStream_t st);
cudaError_t s2_launch_decode_combine(const float* o_part, const float* lse_part, int splits, int D,
                                     int num_bh, __nv_bfloat16* out, float* lse, cudaStream_t st);
cudaError_t s2_launch_kv_compact(const void* k, const void* v, void* kp, void* vp,
                                 const int4* items, int num_items, int batch, int Hkv, int T, int S,
                                 int D, int cap, cudaStream_t st);
cudaError_t s2_launch_kv_append(const void* k, const void* v, void* kp, void* vp,
                                const int* slot_of, int NB, int bt, int batch, int Hkv, int S,
                                int D, int cap, int pos_in_block, cudaStream_t st);

using namespace s2;

static constexpr int kMaxSplits = 32;

struct s2_kvcache {
    s2_plan* plan = nullptr;
    int batch = 0, D = 0, H = 0, Hkv = 0, hpg = 0, S = 0, NB = 0, N = 0, cap = 0;
    int length = 0;
    std::vector<int> slot_of;       // [Hkv][NB]
    std::vector<int64_t> row_ptr;   // [Hkv][NB+1]
    std::vector<int> slot_idx;      // per row, ascending key block
    std::vector<int> row_blocks;    // key block of each slot_idx entry
    DevBuf d_slot_of, d_row_ptr, d_slot_idx, kpool, vpool, d_items;
    CUtensorMap mk{}, mv{};
};

namespace {
int check_cache(const s2_kvcache* c) {
    if (!c) return fail(S2_ERR_INVALID_ARGUMENT, "cache is null");
    return S2_OK;
}
int64_t retained_tokens(const s2_kvcache* c, int g) {
    if (c->length == 0) return 0;
    const int t = c->length - 1, bt = t / c->S;
    const int64_t a = c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt];
    const int64_t b = c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt + 1];
    int64_t n = 0;
    for (int64_t i = a; i < b; ++i) n += c->row_blocks[i] < bt ? c->S : (t - bt * c->S + 1);
    return n;
}
// Split-KV factor: every split CTA streams about the same number of blocks,
// so the launch runs in waves of 2 CTAs / SM.  Take the smallest split
// count giving at least two waves whose last wave is >= 95% full (else the
// fullest), keeping >= 4 blocks per split.
int choose_splits(const s2_kvcache* c, int max_len) {
    const double units = static_cast<double>(c->batch) * c->Hkv;
    const double slots = 2.0 * num_sms();
    const int s_max = std::max(1, std::min(kMaxSplits, max_len / 4));
    int best = 1;
    double best_eff = -1.0;
    for (int s = 1; s <= s_max; ++s) {
        const double waves = units * s / slots;
        const double eff = waves / std::ceil(waves);
        if (waves >= 2.0 && eff >= 0.95) return s;
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
    }
    return best;
}
}  // namespace

extern "C" {

int s2_kvcache_create(s2_plan* p, int batch, int head_dim, int dtype, s2_kvcache** out) {
    if (!p || !out) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (batch < 1 || head_dim < 1) return fail(S2_ERR_INVALID_ARGUMENT, "tensor dimensions must be positive");
    if (dtype != S2_DTYPE_BF16) return fail(S2_ERR_UNSUPPORTED, "the decode cache stores bf16");
    if (head_dim != 64 && head_dim != 128) return fail(S2_ERR_UNSUPPORTED, "decode needs head_dim 64 or 128");
    if (p->block_size != 64) return fail(S2_ERR_UNSUPPORTED, "decode needs block_size 64");
    const int hpg = p->num_heads / p->num_kv_heads;
    if (hpg != 1 && hpg != 2 && hpg != 4 && hpg != 8)
        return fail(S2_ERR_UNSUPPORTED, "decode supports 1, 2, 4 or 8 query heads per kv head");
    auto* c = new s2_kvcache();
    c->plan = p;
    c->batch = batch;
    c->D = head_dim;
    c->H = p->num_heads;
    c->Hkv = p->num_kv_heads;
    c->hpg = hpg;
    c->S = p->block_size;
    c->NB = p->num_blocks;
    c->N = p->seq_len;
    c->slot_of.assign(static_cast<size_t>(c->Hkv) * c->NB, -1);
    c->row_ptr.assign(static_cast<size_t>(c->Hkv) * (c->NB + 1), 0);
    for (int g = 0; g < c->Hkv; ++g) {
        const Csr& csr = p->csr[g * hpg];
        const Csr csc = transpose(csr);
        if (!kv_efficient(csc)) {
            delete c;
            return fail(S2_ERR_UNSUPPORTED,
                        "mask is not KV-cache efficient (verify.cpp:53-72): a compacted cache "
                        "cannot serve it");
        }
        const std::vector<int> ev = evict_after(csc);
        std::vector<std::vector<int>> expire(c->NB);
        for (int j = 0; j < c->NB; ++j) expire[ev[j]].push_back(j);
        std::priority_queue<int, std::vector<int>, std::greater<int>> free_slots;
        int used = 0;
        for (int bt = 0; bt < c->NB; ++bt) {
            if (bt > 0)
                for (int j : expire[bt - 1]) free_slots.push(c->slot_of[static_cast<size_t>(g) * c->NB + j]);
            int s;
            if (!free_slots.empty()) {
                s = free_slots.top();
                free_slots.pop();
            } else {
                s = used++;
            }
            c->slot_of[static_cast<size_t>(g) * c->NB + bt] = s;
        }
        c->cap = std::max(c->cap, used);
        for (int bt = 0; bt < c->NB; ++bt) {
            c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt] = static_cast<int64_t>(c->slot_idx.size());
            for (int q = csr.ptr[bt]; q < csr.ptr[bt + 1]; ++q) {
                c->slot_idx.push_back(c->slot_of[static_cast<size_t>(g) * c->NB + csr.idx[q]]);
                c->row_blocks.push_back(csr.idx[q]);
            }
        }
        c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + c->NB] = static_cast<int64_t>(c->slot_idx.size());
    }
    cudaError_t e;
    const size_t pool = static_cast<size_t>(batch) * c->Hkv * c->cap * c->S * c->D * 2;
    if ((e = upload(c->d_slot_of, c->slot_of.data(), c->slot_of.size() * sizeof(int))) != cudaSuccess ||
        (e = upload(c->d_row_ptr, c->row_ptr.data(), c->row_ptr.size() * sizeof(int64_t))) != cudaSuccess ||
        (e = upload(c->d_slot_idx, c->slot_idx.data(), c->slot_idx.size() * sizeof(int))) != cudaSuccess) {
        delete c;
        return cuda_fail(e, "uploading cache tables");
    }
    cudaGetDevice(&c->kpool.device);
    c->vpool.device = c->kpool.device;
    if ((e = cudaMalloc(&c->kpool.ptr, pool)) != cudaSuccess || (e = cudaMalloc(&c->vpool.ptr, pool)) != cudaSuccess) {
        delete c;
        return cuda_fail(e, "allocating the KV pool");
    }
    c->kpool.bytes = c->vpool.bytes = pool;
    cudaMemset(c->kpool.ptr, 0, pool);
    cudaMemset(c->vpool.ptr, 0, pool);
    try {
        c->mk = s2host::make_map_bf16_3d(c->kpool.ptr, c->D, static_cast<uint64_t>(c->cap) * c->S,
                                         static_cast<uint64_t>(batch) * c->Hkv, 64, 64);
        c->mv = s2host::make_map_bf16_3d(c->vpool.ptr, c->D, static_cast<uint64_t>(c->cap) * c->S,
                                         static_cast<uint64_t>(batch) * c->Hkv, 64, 64);
    } catch (const std::exception& ex) {
        delete c;
        return fail(S2_ERR_CUDA, ex.what());
    }
    *out = c;
    return S2_OK;
}

void s2_kvcache_destroy(s2_kvcache* c) { delete c; }

int s2_kvcache_length(const s2_kvcache* c, int* length) {
    if (int rc = check_cache(c)) return rc;
    if (!length) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    *length = c->length;
    return S2_OK;
}

int s2_kvcache_bytes(const s2_kvcache* c, int64_t* pool_bytes, int64_t* dense_bytes) {
    if (int rc = check_cache(c)) return rc;
    if (pool_bytes) *pool_bytes = static_cast<int64_t>(c->kpool.bytes + c->vpool.bytes);
    if (dense_bytes)
        *dense_bytes = 2LL * c->batch * c->Hkv * static_cast<int64_t>(c->N) * c->D * 2;
    return S2_OK;
}

int s2_kvcache_retained_tokens(const s2_kvcache* c, int kv_head, int64_t* tokens) {
    if (int rc = check_cache(c)) return rc;
    if (kv_head < 0 || kv_head >= c->Hkv || !tokens) return fail(S2_ERR_INVALID_ARGUMENT, "bad kv head");
    *tokens = retained_tokens(c, kv_head);
    return S2_OK;
}

int s2_kvcache_prefill(s2_kvcache* c, const void* k, const void* v, int T, s2_stream_t stream) {
    if (int rc = check_cache(c)) return rc;
    if (T < 0 || T > c->N) return fail(S2_ERR_INVALID_ARGUMENT, "num_tokens must lie in [0, seq_len]");
    if (T > 0 && (!k || !v)) return fail(S2_ERR_INVALID_ARGUMENT, "k/v must be non-null");
    c->length = T;
    if (T == 0) return S2_OK;
    const int bt = (T - 1) / c->S;
    std::vector<int4> items;
    for (int g = 0; g < c->Hkv; ++g)
        for (int64_t i = c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt];
             i < c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt + 1]; ++i)
            items.push_back(make_int4(g, c->row_blocks[i], c->slot_idx[i], 0));
    cudaError_t e = upload(c->d_items, items.data(), items.size() * sizeof(int4));
    if (e != cudaSuccess) return cuda_fail(e, "uploading compaction items");
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ProfScope prof("kv_compact", st);
    e = s2_launch_kv_compact(k, v, c->kpool.ptr, c->vpool.ptr, c->d_items.as<int4>(),
                             static_cast<int>(items.size()), c->batch, c->Hkv, T, c->S, c->D, c->cap, st);
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "kv_compact launch");
}

int s2_kvcache_append(s2_kvcache* c, const void* k, const void* v, s2_stream_t stream) {
    if (int rc = check_cache(c)) return rc;
    if (!k || !v) return fail(S2_ERR_INVALID_ARGUMENT, "k/v must be non-null");
    if (c->length >= c->N) return fail(S2_ERR_INVALID_ARGUMENT, "cache is full (seq_len reached)");
    const int t = c->length;
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    ProfScope prof("kv_append", st);
    cudaError_t e = s2_launch_kv_append(k, v, c->kpool.ptr, c->vpool.ptr, c->d_slot_of.as<int>(),
                                        c->NB, t / c->S, c->batch, c->Hkv, c->S, c->D, c->cap,
                                        t % c->S, st);
    if (e != cudaSuccess) return cuda_fail(e, "kv_append launch");
    ++c->length;
    return S2_OK;
}

int s2_attn_decode_workspace_size(const s2_kvcache* c, size_t* bytes) {
    if (int rc = check_cache(c)) return rc;
    if (!bytes) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    *bytes = static_cast<size_t>(c->batch) * c->H * kMaxSplits * (c->D + 1) * sizeof(float);
    return S2_OK;
}

int s2_attn_decode_bytes(const s2_kvcache* c, int64_t* bytes) {
    if (int rc = check_cache(c)) return rc;
    if (!bytes) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    int64_t tok = 0;
    for (int g = 0; g < c->Hkv; ++g) tok += retained_tokens(c, g);
    *bytes = tok * c->batch * c->D * 2 * 2 + 2LL * c->batch * c->H * c->D * 2;
    return S2_OK;
}

int s2_attn_decode(s2_kvcache* c, const void* q, void* out, float* lse, double scale,
                   void* workspace, size_t workspace_bytes, s2_stream_t stream) {
    if (int rc = check_cache(c)) return rc;
    if (!q || !out) return fail(S2_ERR_INVALID_ARGUMENT, "q/out must be non-null");
    if (c->length < 1) return fail(S2_ERR_INVALID_ARGUMENT, "decode needs at least one cached token");
    size_t need = 0;
    s2_attn_decode_workspace_size(c, &need);
    if (!workspace || workspace_bytes < need)
        return fail(S2_ERR_INVALID_ARGUMENT, "workspace too small (s2_attn_decode_workspace_size)");
    const int t = c->length - 1, bt = t / c->S;
    int max_len = 0;
    for (int g = 0; g < c->Hkv; ++g)
        max_len = std::max<int>(max_len, static_cast<int>(c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt + 1] -
                                                          c->row_ptr[static_cast<size_t>(g) * (c->NB + 1) + bt]));
    const int splits = choose_splits(c, max_len);
    const double sc = resolve_scale(scale, c->D);
    float* o_part = static_cast<float*>(workspace);
    float* lse_part = o_part + static_cast<size_t>(c->batch) * c->H * kMaxSplits * c->D;
    s2dev::DecodeParams p{static_cast<const __nv_bfloat16*>(q), c->d_row_ptr.as<int64_t>(),
                          c->d_slot_idx.as<int>(), c->NB, bt, t - bt * c->S + 1, splits,
                          (max_len + splits - 1) / splits, c->H, c->Hkv, c->D, c->hpg,
                          float(sc * M_LOG2E), o_part, lse_part};
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    {
        ProfScope prof("decode_split", st);
        e = s2_launch_decode(c->mk, c->mv, p, c->batch, st);
    }
    if (e == cudaSuccess) {
        ProfScope prof("decode_combine", st);
        e = s2_launch_decode_combine(o_part, lse_part, splits, c->D, c->batch * c->H,
                                     static_cast<__nv_bfloat16*>(out), lse, st);
    }
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "s2_attn_decode launch");
}

}  // extern "C"
