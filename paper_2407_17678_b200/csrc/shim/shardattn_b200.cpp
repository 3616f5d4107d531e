// libshardattn_b200.so: the reference's C++ API (include/shardattn_b200/shardattn/*.hpp)
// implemented over the C ABI of include/s2attn.h.  Host data in, host data out,
// same validation order and std::invalid_argument conditions as the reference
// (pattern.cpp:36-79, csr.cpp:11-33, kernel_common.hpp:20-41, attention.cpp:100-118,146-152).
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "s2attn.h"
#include "shardattn/attention.hpp"
#include "shardattn/csr.hpp"
#include "shardattn/pattern.hpp"

namespace shardattn {
namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = s2_last_error();
    if (rc == S2_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error("s2attn: " + msg);
}
void ck(int rc) {
    if (rc != S2_OK) raise(rc);
}

// PatternConfig -> s2_pattern_config (offsets stay owned by `cfg`).
struct CConfig {
    s2_pattern_config c{};
    explicit CConfig(const PatternConfig& cfg) {
        c.seq_len = cfg.seq_len;
        c.block_size = cfg.block_size;
        c.num_heads = cfg.num_heads;
        c.num_kv_heads = cfg.num_kv_heads;
        c.local_blocks = cfg.local_blocks;
        c.local_stride = cfg.local_stride;
        if (cfg.stride_segments.size() > S2_MAX_SEGMENTS)
            throw std::invalid_argument("too many stride segments");
        c.num_segments = static_cast<int>(cfg.stride_segments.size());
        for (int s = 0; s < c.num_segments; ++s) {
            const StrideSegment& seg = cfg.stride_segments[s];
            c.segments[s] = {seg.start_block_distance, seg.end_block_distance, seg.stride,
                             static_cast<int>(seg.offsets.size()),
                             seg.offsets.empty() ? nullptr : seg.offsets.data()};
        }
    }
};

// Device buffer owned for the duration of one call.
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) { ck(s2_device_malloc(&p, bytes)); }
    ~Dev() {
        if (p) s2_device_free(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

struct Plan {
    s2_plan* p = nullptr;
    ~Plan() { s2_plan_destroy(p); }
};

void check_shapes(const AttentionTensors& t, std::size_t masks, int mask_blocks, int block_size) {
    if (t.num_heads < 1 || t.seq_len < 1 || t.head_dim < 1)
        throw std::invalid_argument("tensor dimensions must be positive");
    const std::size_t n = static_cast<std::size_t>(t.num_heads) * t.seq_len * t.head_dim;
    if (t.q.size() != n || t.k.size() != n || t.v.size() != n)
        throw std::invalid_argument("q/k/v sizes do not match [heads, seq, dim]");
    if (masks != static_cast<std::size_t>(t.num_heads))
        throw std::invalid_argument("one mask per head required");
    if (block_size < 1) throw std::invalid_argument("block_size must be positive");
    if (mask_blocks != (t.seq_len + block_size - 1) / block_size)
        throw std::invalid_argument("mask block count does not match ceil(seq_len/block_size)");
}

Plan make_plan(const std::vector<CsrMask>& csr, int seq_len, int block_size) {
    std::vector<const int*> rp, ci;
    static const int kZero = 0;
    for (const CsrMask& c : csr) {
        rp.push_back(c.row_ptr.data());
        ci.push_back(c.col_idx.empty() ? &kZero : c.col_idx.data());
    }
    Plan plan;
    ck(s2_plan_create_from_csr(static_cast<int>(csr.size()), 0, seq_len, block_size, rp.data(),
                               ci.data(), &plan.p));
    return plan;
}

// The GPU forward on host tensors (fp32 kernel), filling t.out / t.lse like
// prepare_outputs (kernel_common.hpp:43-46) + the streaming kernel.
void gpu_forward(AttentionTensors& t, const std::vector<CsrMask>& csr, int block_size,
                 int num_splits) {
    Plan plan = make_plan(csr, t.seq_len, block_size);
    const size_t n = t.q.size();
    const size_t rows = static_cast<size_t>(t.num_heads) * t.seq_len;
    Dev q(n * 4), k(n * 4), v(n * 4), o(n * 4), l(rows * 4);
    ck(s2_memcpy_h2d(q.p, t.q.data(), n * 4, nullptr));
    ck(s2_memcpy_h2d(k.p, t.k.data(), n * 4, nullptr));
    ck(s2_memcpy_h2d(v.p, t.v.data(), n * 4, nullptr));
    s2_attn_args a{};
    a.dtype = S2_DTYPE_F32;
    a.batch = 1;
    a.num_heads = t.num_heads;
    a.num_kv_heads = t.num_heads;
    a.seq_len = t.seq_len;
    a.head_dim = t.head_dim;
    a.scale = t.scale == 0.0 ? S2_SCALE_ZERO : t.scale;  // the reference applies scale literally
    a.num_splits = num_splits;
    a.q = q.p;
    a.k = k.p;
    a.v = v.p;
    a.out = o.p;
    a.lse = static_cast<float*>(l.p);
    ck(s2_attn_fwd(plan.p, &a, nullptr));
    t.out.assign(n, 0.0f);
    std::vector<float> lse(rows);
    ck(s2_memcpy_d2h(t.out.data(), o.p, n * 4, nullptr));
    ck(s2_memcpy_d2h(lse.data(), l.p, rows * 4, nullptr));
    ck(s2_stream_synchronize(nullptr));
    t.lse.assign(lse.begin(), lse.end());
}

}  // namespace

// ------------------------------------------------------------------ pattern
int PatternConfig::num_blocks() const {
    return static_cast<int>((static_cast<long long>(seq_len) + block_size - 1) / block_size);
}

int PatternConfig::offset_for(std::size_t segment, int head) const {
    const StrideSegment& seg = stride_segments.at(segment);
    int raw = group_of(head);
    if (!seg.offsets.empty())
        raw = seg.offsets.size() == static_cast<std::size_t>(num_heads) ? seg.offsets[head]
                                                                         : seg.offsets[group_of(head)];
    return raw % seg.stride;
}

void PatternConfig::validate() const {
    CConfig c(*this);
    ck(s2_pattern_validate(&c.c));
}

HeadBlockMask::HeadBlockMask(int head_index, int num_blocks)
    : head_index_(head_index), num_blocks_(num_blocks),
      bits_(static_cast<std::size_t>(num_blocks) * num_blocks, 0) {}

bool HeadBlockMask::is_causal() const {
    for (int i = 0; i < num_blocks_; ++i)
        for (int j = i + 1; j < num_blocks_; ++j)
            if (at(i, j)) return false;
    return true;
}

bool HeadBlockMask::has_full_diagonal() const {
    for (int i = 0; i < num_blocks_; ++i)
        if (!at(i, i)) return false;
    return true;
}

std::size_t HeadBlockMask::popcount() const {
    std::size_t n = 0;
    for (std::uint8_t b : bits_) n += b;
    return n;
}

std::vector<int> HeadBlockMask::row(int query_block) const {
    std::vector<int> r;
    for (int j = 0; j < num_blocks_; ++j)
        if (at(query_block, j)) r.push_back(j);
    return r;
}

bool same_bits(const HeadBlockMask& a, const HeadBlockMask& b) {
    if (a.num_blocks() != b.num_blocks()) return false;
    for (int i = 0; i < a.num_blocks(); ++i)
        for (int j = 0; j < a.num_blocks(); ++j)
            if (a.at(i, j) != b.at(i, j)) return false;
    return true;
}

void LayerSchedule::validate() const {
    if (num_layers < 1) throw std::invalid_argument("num_layers must be positive");
    for (int id : dense_layer_ids)
        if (id < 0 || id >= num_layers)
            throw std::invalid_argument("dense layer id " + std::to_string(id) +
                                        " outside [0, num_layers)");
    sparse_pattern.validate();
}

HeadBlockMask build_head_mask(const PatternConfig& config, int head) {
    CConfig c(config);
    ck(s2_pattern_validate(&c.c));
    if (head < 0 || head >= config.num_heads)
        throw std::invalid_argument("head index " + std::to_string(head) +
                                    " outside [0, num_heads)");
    int64_t n = 0;
    ck(s2_layout_nnz(&c.c, head, &n));
    const int B = config.num_blocks();
    std::vector<int> rp(B + 1), ci(static_cast<size_t>(std::max<int64_t>(n, 1)));
    ck(s2_layout_build_csr(&c.c, head, rp.data(), ci.data()));
    HeadBlockMask m(head, B);
    for (int i = 0; i < B; ++i)
        for (int p = rp[i]; p < rp[i + 1]; ++p) m.set(i, ci[p], true);
    return m;
}

std::vector<HeadBlockMask> build_all_masks(const PatternConfig& config) {
    config.validate();
    std::vector<HeadBlockMask> masks;
    masks.reserve(config.num_heads);
    for (int h = 0; h < config.num_heads; ++h) masks.push_back(build_head_mask(config, h));
    return masks;
}

std::vector<std::vector<HeadBlockMask>> build_layer_masks(const LayerSchedule& schedule) {
    schedule.validate();
    const std::vector<HeadBlockMask> sparse = build_all_masks(schedule.sparse_pattern);
    std::vector<HeadBlockMask> dense;
    for (std::size_t h = 0; h < sparse.size(); ++h)
        dense.push_back(dense_causal_mask(schedule.sparse_pattern.num_blocks(), static_cast<int>(h)));
    std::vector<std::vector<HeadBlockMask>> out;
    for (int l = 0; l < schedule.num_layers; ++l)
        out.push_back(schedule.dense_layer_ids.count(l) ? dense : sparse);
    return out;
}

HeadBlockMask dense_causal_mask(int num_blocks, int head_index) {
    HeadBlockMask m(head_index, num_blocks);
    for (int i = 0; i < num_blocks; ++i)
        for (int j = 0; j <= i; ++j) m.set(i, j, true);
    return m;
}

static PatternConfig base_config(int seq_len, int block_size, int num_heads, int local_blocks,
                                 int local_stride) {
    PatternConfig c;
    c.seq_len = seq_len;
    c.block_size = block_size;
    c.num_heads = num_heads;
    c.num_kv_heads = num_heads;
    c.local_blocks = local_blocks;
    c.local_stride = local_stride;
    return c;
}

PatternConfig make_single_stride_config(int seq_len, int block_size, int num_heads,
                                        int local_blocks, int remote_stride, int local_stride) {
    PatternConfig c = base_config(seq_len, block_size, num_heads, local_blocks, local_stride);
    if (local_blocks < c.num_blocks())
        c.stride_segments.push_back({local_blocks, c.num_blocks(), remote_stride, {}});
    c.validate();
    return c;
}

PatternConfig make_multi_stride_config(int seq_len, int block_size, int num_heads,
                                       int local_blocks, int mid_block_distance, int stride1,
                                       int stride2) {
    PatternConfig c = base_config(seq_len, block_size, num_heads, local_blocks, 1);
    c.stride_segments.push_back({local_blocks, mid_block_distance, stride1, {}});
    c.stride_segments.push_back({mid_block_distance, c.num_blocks(), stride2, {}});
    c.validate();
    return c;
}

PatternConfig make_sliding_window_config(int seq_len, int block_size, int num_heads,
                                         int window_blocks) {
    PatternConfig c = base_config(seq_len, block_size, num_heads, window_blocks, 1);
    c.validate();
    return c;
}

PatternConfig make_dense_config(int seq_len, int block_size, int num_heads) {
    return make_single_stride_config(seq_len, block_size, num_heads, 1, 1);
}

// ---------------------------------------------------------------------- csr
void CsrMask::validate() const {
    if (num_blocks < 1) throw std::invalid_argument("csr num_blocks must be positive");
    if (row_ptr.size() != static_cast<std::size_t>(num_blocks) + 1)
        throw std::invalid_argument("row_ptr must have num_blocks + 1 entries");
    if (row_ptr.front() != 0) throw std::invalid_argument("row_ptr[0] must be 0");
    if (row_ptr.back() != static_cast<int>(col_idx.size()))
        throw std::invalid_argument("row_ptr[B] must equal col_idx length");
    static const int kZero = 0;
    ck(s2_csr_validate(num_blocks, row_ptr.data(), col_idx.empty() ? &kZero : col_idx.data(),
                       static_cast<int64_t>(col_idx.size())));
}

CsrMask to_csr(const HeadBlockMask& mask) {
    CsrMask c;
    c.head_index = mask.head_index();
    c.num_blocks = mask.num_blocks();
    c.row_ptr.push_back(0);
    for (int i = 0; i < c.num_blocks; ++i) {
        for (int j = 0; j <= i; ++j)
            if (mask.at(i, j)) c.col_idx.push_back(j);
        c.row_ptr.push_back(static_cast<int>(c.col_idx.size()));
    }
    return c;
}

std::vector<CsrMask> to_csr(const std::vector<HeadBlockMask>& masks) {
    std::vector<CsrMask> out;
    for (const HeadBlockMask& m : masks) out.push_back(to_csr(m));
    return out;
}

HeadBlockMask from_csr(const CsrMask& csr, int num_blocks) {
    if (csr.num_blocks != num_blocks)
        throw std::invalid_argument("csr block count does not match requested num_blocks");
    csr.validate();
    HeadBlockMask m(csr.head_index, num_blocks);
    for (int i = 0; i < num_blocks; ++i)
        for (int p = csr.row_ptr[i]; p < csr.row_ptr[i + 1]; ++p) m.set(i, csr.col_idx[p], true);
    return m;
}

std::size_t nnz(const CsrMask& csr) { return csr.col_idx.size(); }

// ---------------------------------------------------------------- attention
AttentionTensors AttentionTensors::zeros(int num_heads, int seq_len, int head_dim) {
    AttentionTensors t;
    t.num_heads = num_heads;
    t.seq_len = seq_len;
    t.head_dim = head_dim;
    t.scale = 1.0 / std::sqrt(static_cast<double>(head_dim));
    const std::size_t n = static_cast<std::size_t>(num_heads) * seq_len * head_dim;
    t.q.assign(n, 0.0f);
    t.k.assign(n, 0.0f);
    t.v.assign(n, 0.0f);
    return t;
}

AttentionTensors AttentionTensors::random(int num_heads, int seq_len, int head_dim,
                                          std::uint64_t seed) {
    AttentionTensors t = zeros(num_heads, seq_len, head_dim);
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<float> u(-1.0f, 1.0f);
    for (auto* vec : {&t.q, &t.k, &t.v})
        for (float& x : *vec) x = u(gen);
    return t;
}

void dsplit_attention(AttentionTensors& t, const std::vector<CsrMask>& csr, int block_size,
                      int num_splits) {
    if (csr.empty()) throw std::invalid_argument("csr list is empty");
    check_shapes(t, csr.size(), csr.front().num_blocks, block_size);
    for (const CsrMask& c : csr) {
        c.validate();
        if (c.num_blocks != csr.front().num_blocks)
            throw std::invalid_argument("csr masks differ in block count");
    }
    if (num_splits < 1 || t.head_dim % num_splits != 0)
        throw std::invalid_argument("num_splits must divide head_dim");
    gpu_forward(t, csr, block_size, num_splits);
}

void streaming_sharded_attention(AttentionTensors& t, const std::vector<CsrMask>& csr,
                                 int block_size) {
    dsplit_attention(t, csr, block_size, 1);
}

void naive_masked_attention(AttentionTensors& t, const std::vector<HeadBlockMask>& masks,
                            int block_size) {
    check_shapes(t, masks.size(), masks.empty() ? -1 : masks.front().num_blocks(), block_size);
    gpu_forward(t, to_csr(masks), block_size, 1);
}

void dense_masked_attention(AttentionTensors& t, const std::vector<HeadBlockMask>& masks,
                            int block_size) {
    check_shapes(t, masks.size(), masks.empty() ? -1 : masks.front().num_blocks(), block_size);
    for (const HeadBlockMask& m : masks)
        if (!m.is_causal() || !m.has_full_diagonal())
            throw std::invalid_argument("masks must be causal with a full diagonal");
    for (const auto* vec : {&t.q, &t.k, &t.v})
        for (float x : *vec)
            if (!std::isfinite(x))
                throw std::invalid_argument(vec == &t.q ? "non-finite entry in q"
                                            : vec == &t.k ? "non-finite entry in k"
                                                          : "non-finite entry in v");
    gpu_forward(t, to_csr(masks), block_size, 1);
}

void streaming_sharded_attention_backward(const AttentionTensors& t,
                                          const std::vector<CsrMask>& csr, int block_size,
                                          const std::vector<float>& dout, AttentionGrads& grads) {
    if (csr.empty()) throw std::invalid_argument("csr list is empty");
    check_shapes(t, csr.size(), csr.front().num_blocks, block_size);
    for (const CsrMask& c : csr) c.validate();
    const size_t n = t.q.size();
    if (dout.size() != n) throw std::invalid_argument("dout size does not match [heads, seq, dim]");
    if (t.head_dim > 128) throw std::invalid_argument("backward supports head_dim <= 128");
    // fp32 end to end, like the forward: the reference-precision backward kernels
    // (bwd_simt.cu; head_dim <= 128, else S2_ERR_UNSUPPORTED -> invalid_argument)
    Plan plan = make_plan(csr, t.seq_len, block_size);
    const size_t rows = static_cast<size_t>(t.num_heads) * t.seq_len;
    Dev q(n * 4), k(n * 4), v(n * 4), o(n * 4), l(rows * 4), g(n * 4), dq(n * 4), dk(n * 4), dv(n * 4);
    ck(s2_memcpy_h2d(q.p, t.q.data(), n * 4, nullptr));
    ck(s2_memcpy_h2d(k.p, t.k.data(), n * 4, nullptr));
    ck(s2_memcpy_h2d(v.p, t.v.data(), n * 4, nullptr));
    ck(s2_memcpy_h2d(g.p, dout.data(), n * 4, nullptr));
    s2_attn_bwd_args a{};
    a.fwd.dtype = S2_DTYPE_F32;
    a.fwd.batch = 1;
    a.fwd.num_heads = t.num_heads;
    a.fwd.num_kv_heads = t.num_heads;
    a.fwd.seq_len = t.seq_len;
    a.fwd.head_dim = t.head_dim;
    a.fwd.scale = t.scale == 0.0 ? S2_SCALE_ZERO : t.scale;
    a.fwd.num_splits = 1;
    a.fwd.q = q.p;
    a.fwd.k = k.p;
    a.fwd.v = v.p;
    a.fwd.out = o.p;
    a.fwd.lse = static_cast<float*>(l.p);
    a.dout = g.p;
    a.dq = dq.p;
    a.dk = dk.p;
    a.dv = dv.p;
    ck(s2_attn_fwd(plan.p, &a.fwd, nullptr));
    size_t ws = 0;
    ck(s2_attn_bwd_workspace_size(plan.p, &a, &ws));
    Dev w(ws);
    ck(s2_attn_bwd(plan.p, &a, w.p, ws, nullptr));
    grads.dq.resize(n);
    grads.dk.resize(n);
    grads.dv.resize(n);
    ck(s2_memcpy_d2h(grads.dq.data(), dq.p, n * 4, nullptr));
    ck(s2_memcpy_d2h(grads.dk.data(), dk.p, n * 4, nullptr));
    ck(s2_memcpy_d2h(grads.dv.data(), dv.p, n * 4, nullptr));
    ck(s2_stream_synchronize(nullptr));
}

void sharded_decode(AttentionTensors& t, const std::vector<CsrMask>& csr, int block_size, int position) {
    if (csr.empty()) throw std::invalid_argument("csr list is empty");
    check_shapes(t, csr.size(), csr.front().num_blocks, block_size);
    for (const CsrMask& c : csr) {
        c.validate();
        if (c.num_blocks != csr.front().num_blocks)
            throw std::invalid_argument("csr masks differ in block count");
    }
    if (position < 0 || position >= t.seq_len)
        throw std::invalid_argument("decode position outside [0, seq_len)");
    auto bf16 = [](float x) {
        uint32_t u;
        std::memcpy(&u, &x, 4);
        return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    };
    const int H = t.num_heads, d = t.head_dim, T = position + 1;
    Plan plan = make_plan(csr, t.seq_len, block_size);
    struct Cache {
        s2_kvcache* c = nullptr;
        ~Cache() { s2_kvcache_destroy(c); }
    } cache;
    ck(s2_kvcache_create(plan.p, 1, d, S2_DTYPE_BF16, &cache.c));
    // the prefix [H, T, d] of k / v, bf16
    const size_t nkv = static_cast<size_t>(H) * T * d;
    std::vector<uint16_t> hk(nkv), hv(nkv), hq(static_cast<size_t>(H) * d);
    for (int h = 0; h < H; ++h)
        for (int s = 0; s < T; ++s)
            for (int c = 0; c < d; ++c) {
                const size_t dst = (static_cast<size_t>(h) * T + s) * d + c;
                hk[dst] = bf16(t.k[t.idx(h, s, c)]);
                hv[dst] = bf16(t.v[t.idx(h, s, c)]);
            }
    for (int h = 0; h < H; ++h)
        for (int c = 0; c < d; ++c) hq[static_cast<size_t>(h) * d + c] = bf16(t.q[t.idx(h, position, c)]);
    Dev k(nkv * 2), v(nkv * 2), q(hq.size() * 2), o(hq.size() * 2), l(static_cast<size_t>(H) * 4);
    ck(s2_memcpy_h2d(k.p, hk.data(), nkv * 2, nullptr));
    ck(s2_memcpy_h2d(v.p, hv.data(), nkv * 2, nullptr));
    ck(s2_memcpy_h2d(q.p, hq.data(), hq.size() * 2, nullptr));
    ck(s2_kvcache_prefill(cache.c, k.p, v.p, T, nullptr));
    size_t ws = 0;
    ck(s2_attn_decode_workspace_size(cache.c, &ws));
    Dev w(ws);
    ck(s2_attn_decode(cache.c, q.p, o.p, static_cast<float*>(l.p), t.scale == 0.0 ? S2_SCALE_ZERO : t.scale, w.p,
                      ws, nullptr));
    std::vector<uint16_t> ho(hq.size());
    std::vector<float> hl(H);
    ck(s2_memcpy_d2h(ho.data(), o.p, ho.size() * 2, nullptr));
    ck(s2_memcpy_d2h(hl.data(), l.p, hl.size() * 4, nullptr));
    ck(s2_stream_synchronize(nullptr));
    t.out.assign(t.q.size(), 0.0f);
    t.lse.assign(static_cast<size_t>(H) * t.seq_len, -std::numeric_limits<double>::infinity());
    for (int h = 0; h < H; ++h) {
        for (int c = 0; c < d; ++c) {
            const uint32_t u = static_cast<uint32_t>(ho[static_cast<size_t>(h) * d + c]) << 16;
            std::memcpy(&t.out[t.idx(h, position, c)], &u, 4);
        }
        t.lse[t.row_index(h, position)] = hl[h];
    }
}

}  // namespace shardattn
