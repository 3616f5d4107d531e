// ORACLE / TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
//
// extern "C" wrapper over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled from where the sources lie by
// oracle/Makefile into oracle/_ref/libshardattn_ref.so).  It lets pytest
// (ctypes) drive the reference's own layout builder, streaming/naive/dense
// attention kernels, decode-cache simulator and RNG, so the C restatement in
// oracle/s2_oracle.c and the golden fixtures can be pinned to the reference.
// Only the reference's public headers (proj/include/shardattn) are used.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "s2attn.h"
#include "shardattn/analysis.hpp"
#include "shardattn/attention.hpp"
#include "shardattn/csr.hpp"
#include "shardattn/pattern.hpp"
#include "shardattn/selftest.hpp"
#include "shardattn/serialize.hpp"
#include "shardattn/verify.hpp"

using namespace shardattn;

namespace {
thread_local std::string g_err;

PatternConfig to_cfg(const s2_pattern_config* c) {
    PatternConfig cfg;
    cfg.seq_len = c->seq_len;
    cfg.block_size = c->block_size;
    cfg.num_heads = c->num_heads;
    cfg.num_kv_heads = c->num_kv_heads;
    cfg.local_blocks = c->local_blocks;
    cfg.local_stride = c->local_stride;
    for (int s = 0; s < c->num_segments; ++s) {
        StrideSegment seg;
        seg.start_block_distance = c->segments[s].start_block_distance;
        seg.end_block_distance = c->segments[s].end_block_distance;
        seg.stride = c->segments[s].stride;
        for (int i = 0; i < c->segments[s].num_offsets; ++i)
            seg.offsets.push_back(c->segments[s].offsets[i]);
        cfg.stride_segments.push_back(seg);
    }
    return cfg;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

AttentionTensors make_tensors(int H, int N, int d, double scale, const float* q, const float* k,
                              const float* v) {
    AttentionTensors t = AttentionTensors::zeros(H, N, d);
    if (scale != 0.0) t.scale = scale;
    const std::size_t n = static_cast<std::size_t>(H) * N * d;
    std::memcpy(t.q.data(), q, n * sizeof(float));
    std::memcpy(t.k.data(), k, n * sizeof(float));
    std::memcpy(t.v.data(), v, n * sizeof(float));
    return t;
}

void copy_out(const AttentionTensors& t, float* out, double* lse) {
    std::memcpy(out, t.out.data(), t.out.size() * sizeof(float));
    std::memcpy(lse, t.lse.data(), t.lse.size() * sizeof(double));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(const s2_pattern_config* c) {
    return guarded([&] { to_cfg(c).validate(); });
}

// to_csr(build_head_mask(cfg, head)); row_ptr may be NULL to query nnz only.
int ref_build_csr(const s2_pattern_config* c, int head, int* row_ptr, int* col_idx,
                  int64_t* nnz) {
    return guarded([&] {
        const CsrMask csr = to_csr(build_head_mask(to_cfg(c), head));
        *nnz = static_cast<int64_t>(csr.col_idx.size());
        if (row_ptr) {
            std::memcpy(row_ptr, csr.row_ptr.data(), csr.row_ptr.size() * sizeof(int));
            std::memcpy(col_idx, csr.col_idx.data(), csr.col_idx.size() * sizeof(int));
        }
    });
}

// build_all_masks -> to_csr for every head, concatenated (row_ptr: H*(B+1)).
int ref_build_all_csr(const s2_pattern_config* c, int* row_ptr, int* col_idx, int64_t* nnz) {
    return guarded([&] {
        const std::vector<CsrMask> all = to_csr(build_all_masks(to_cfg(c)));
        int64_t total = 0;
        for (const CsrMask& m : all) total += static_cast<int64_t>(m.col_idx.size());
        *nnz = total;
        if (!row_ptr) return;
        std::size_t rp = 0, ci = 0;
        for (const CsrMask& m : all) {
            std::memcpy(row_ptr + rp, m.row_ptr.data(), m.row_ptr.size() * sizeof(int));
            std::memcpy(col_idx + ci, m.col_idx.data(), m.col_idx.size() * sizeof(int));
            rp += m.row_ptr.size();
            ci += m.col_idx.size();
        }
    });
}

int ref_csr_validate(int num_blocks, const int* row_ptr, const int* col_idx, int64_t nnz) {
    return guarded([&] {
        CsrMask m;
        m.num_blocks = num_blocks;
        m.row_ptr.assign(row_ptr, row_ptr + (num_blocks >= 0 ? num_blocks + 1 : 0));
        m.col_idx.assign(col_idx, col_idx + nnz);
        m.validate();
    });
}

int ref_random_tensors(int H, int N, int d, uint64_t seed, float* q, float* k, float* v) {
    return guarded([&] {
        const AttentionTensors t = AttentionTensors::random(H, N, d, seed);
        const std::size_t n = t.q.size() * sizeof(float);
        std::memcpy(q, t.q.data(), n);
        std::memcpy(k, t.k.data(), n);
        std::memcpy(v, t.v.data(), n);
    });
}

static std::vector<CsrMask> csr_list(int H, int B, const int* row_ptr, const int* col_idx) {
    std::vector<CsrMask> v(H);
    std::size_t ci = 0;
    for (int h = 0; h < H; ++h) {
        v[h].head_index = h;
        v[h].num_blocks = B;
        v[h].row_ptr.assign(row_ptr + static_cast<std::size_t>(h) * (B + 1),
                            row_ptr + static_cast<std::size_t>(h + 1) * (B + 1));
        const int n = v[h].row_ptr.back();
        v[h].col_idx.assign(col_idx + ci, col_idx + ci + n);
        ci += n;
    }
    return v;
}

// streaming_sharded_attention / dsplit_attention on concatenated CSR lists.
int ref_streaming(int H, int N, int d, int S, double scale, const float* q, const float* k,
                  const float* v, int B, const int* row_ptr, const int* col_idx,
                  int num_splits, float* out, double* lse) {
    return guarded([&] {
        AttentionTensors t = make_tensors(H, N, d, scale, q, k, v);
        const std::vector<CsrMask> csr = csr_list(H, B, row_ptr, col_idx);
        if (num_splits <= 0)
            streaming_sharded_attention(t, csr, S);
        else
            dsplit_attention(t, csr, S, num_splits);
        copy_out(t, out, lse);
    });
}

int ref_naive(const s2_pattern_config* c, int d, double scale, const float* q, const float* k,
              const float* v, float* out, double* lse) {
    return guarded([&] {
        const PatternConfig cfg = to_cfg(c);
        AttentionTensors t = make_tensors(cfg.num_heads, cfg.seq_len, d, scale, q, k, v);
        naive_masked_attention(t, build_all_masks(cfg), cfg.block_size);
        copy_out(t, out, lse);
    });
}

int ref_dense(const s2_pattern_config* c, int d, double scale, const float* q, const float* k,
              const float* v, float* out, double* lse) {
    return guarded([&] {
        const PatternConfig cfg = to_cfg(c);
        AttentionTensors t = make_tensors(cfg.num_heads, cfg.seq_len, d, scale, q, k, v);
        dense_masked_attention(t, build_all_masks(cfg), cfg.block_size);
        copy_out(t, out, lse);
    });
}

// simulate_decode_cache: evict_after of one head + final-step occupancy.
int ref_decode_cache(const s2_pattern_config* c, int total_tokens, int head, int* evict_after,
                     int64_t* occupancy_last, int* dead_total) {
    return guarded([&] {
        const CacheSchedule s = simulate_decode_cache(to_cfg(c), total_tokens);
        const HeadCacheSchedule& h = s.heads.at(head);
        std::memcpy(evict_after, h.evict_after.data(), h.evict_after.size() * sizeof(int));
        *occupancy_last = h.occupancy.back();
        int dead = 0;
        for (int x : h.dead_blocks) dead += x;
        *dead_total = dead;
    });
}

int ref_kv_efficient(const s2_pattern_config* c, int head, int* ok) {
    return guarded([&] {
        *ok = check_kv_cache_efficiency(build_head_mask(to_cfg(c), head)).ok ? 1 : 0;
    });
}

int ref_exact_flops(const s2_pattern_config* c, int head_dim, double* dense, double* sparse,
                    int64_t* nnz_per_head) {
    return guarded([&] {
        const FlopsReport r = exact_flops(to_cfg(c), head_dim);
        *dense = r.dense_flops;
        *sparse = r.sparse_flops;
        for (std::size_t h = 0; h < r.nnz_per_head.size(); ++h)
            nnz_per_head[h] = static_cast<int64_t>(r.nnz_per_head[h]);
    });
}

double ref_max_relative_error_f(const float* a, const float* b, int64_t n) {
    return max_relative_error(std::vector<float>(a, a + n), std::vector<float>(b, b + n));
}

double ref_max_relative_error_d(const double* a, const double* b, int64_t n) {
    return max_relative_error(std::vector<double>(a, a + n), std::vector<double>(b, b + n));
}


// ---- serialize.cpp / analysis.cpp (fixtures for tests/test_serialize.py) ----
static int put_str(const std::string& s, char* buf, int cap) {
    if (!buf || cap < static_cast<int>(s.size()) + 1) throw std::length_error("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

int ref_config_json(const s2_pattern_config* c, char* buf, int cap) {
    return guarded([&] { put_str(to_json(to_cfg(c)).dump(), buf, cap); });
}

int ref_config_hash(const s2_pattern_config* c, uint64_t* h) {
    return guarded([&] { *h = config_hash(to_cfg(c)); });
}

// load_config_file: canonical pattern / schedule documents, report fields.
int ref_load_config(const char* path, char* pattern, char* schedule, char* out, char* format, int cap) {
    return guarded([&] {
        const CliConfigFile f = load_config_file(path);
        put_str(to_json(f.pattern).dump(), pattern, cap);
        put_str(f.schedule ? to_json(*f.schedule).dump() : std::string(), schedule, cap);
        put_str(f.out, out, cap);
        put_str(f.format, format, cap);
    });
}

int ref_kv_reduction(const s2_pattern_config* c, int num_layers, const int* dense, int ndense,
                     double* pct) {
    return guarded([&] {
        LayerSchedule s;
        s.num_layers = num_layers;
        for (int i = 0; i < ndense; ++i) s.dense_layer_ids.insert(dense[i]);
        s.sparse_pattern = to_cfg(c);
        *pct = kv_reduction(s);
    });
}

int ref_decode_cache_full(const s2_pattern_config* c, int total_tokens, int head, int* evict_after,
                          int64_t* occupancy, int* dead, int64_t* peak, double* mean) {
    return guarded([&] {
        const CacheSchedule cs = simulate_decode_cache(to_cfg(c), total_tokens);
        const HeadCacheSchedule& h = cs.heads.at(head);
        std::copy(h.evict_after.begin(), h.evict_after.end(), evict_after);
        std::copy(h.occupancy.begin(), h.occupancy.end(), occupancy);
        std::copy(h.dead_blocks.begin(), h.dead_blocks.end(), dead);
        *peak = h.peak_tokens;
        *mean = h.mean_tokens;
    });
}

int ref_analytic(double seq_len, double local_window, double stride, int heads, double* eq,
                 double* red, double* upper) {
    return guarded([&] {
        *eq = equivalent_context_length(seq_len, local_window, stride);
        *red = analytic_flops_reduction(seq_len, local_window, stride);
        *upper = speedup_upper_bound(heads, seq_len, local_window);
    });
}
}  // extern "C"
