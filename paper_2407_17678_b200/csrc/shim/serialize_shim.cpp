// shardattn:: serialize.hpp / analysis.hpp over the C ABI (part of
// libshardattn_b200.so).  Host-only: no device is touched.
#include <stdexcept>
#include <string>
#include <vector>

#include "s2attn.h"
#include "shardattn/analysis.hpp"
#include "shardattn/serialize.hpp"

namespace shardattn {
namespace {

void ck(int rc) {
    if (rc == S2_OK) return;
    const std::string msg = s2_last_error();
    if (rc == S2_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

struct CConfig {
    s2_pattern_config c{};
    explicit CConfig(const PatternConfig& cfg) {
        c.seq_len = cfg.seq_len;
        c.block_size = cfg.block_size;
        c.num_heads = cfg.num_heads;
        c.num_kv_heads = cfg.num_kv_heads;
        c.local_blocks = cfg.local_blocks;
        c.local_stride = cfg.local_stride;
        if (cfg.stride_segments.size() > S2_MAX_SEGMENTS) throw std::invalid_argument("too many stride segments");
        c.num_segments = static_cast<int>(cfg.stride_segments.size());
        for (int s = 0; s < c.num_segments; ++s) {
            const StrideSegment& seg = cfg.stride_segments[s];
            c.segments[s] = {seg.start_block_distance, seg.end_block_distance, seg.stride,
                             static_cast<int>(seg.offsets.size()),
                             seg.offsets.empty() ? nullptr : seg.offsets.data()};
        }
    }
};

PatternConfig from_c(const s2_pattern_config& c) {
    PatternConfig p;
    p.seq_len = c.seq_len;
    p.block_size = c.block_size;
    p.num_heads = c.num_heads;
    p.num_kv_heads = c.num_kv_heads;
    p.local_blocks = c.local_blocks;
    p.local_stride = c.local_stride;
    for (int s = 0; s < c.num_segments; ++s) {
        StrideSegment seg;
        seg.start_block_distance = c.segments[s].start_block_distance;
        seg.end_block_distance = c.segments[s].end_block_distance;
        seg.stride = c.segments[s].stride;
        if (c.segments[s].num_offsets > 0)
            seg.offsets.assign(c.segments[s].offsets, c.segments[s].offsets + c.segments[s].num_offsets);
        p.stride_segments.push_back(std::move(seg));
    }
    return p;
}

struct CSchedule {
    std::vector<int> ids;
    CConfig cfg;
    s2_layer_schedule s{};
    explicit CSchedule(const LayerSchedule& ls) : ids(ls.dense_layer_ids.begin(), ls.dense_layer_ids.end()), cfg(ls.sparse_pattern) {
        s.num_layers = ls.num_layers;
        s.num_dense = static_cast<int>(ids.size());
        s.dense_layer_ids = ids.empty() ? nullptr : ids.data();
        s.sparse_pattern = cfg.c;
    }
};

template <class F>
std::string text_of(F&& f) {
    size_t n = 0;
    ck(f(nullptr, 0, &n));
    std::string out(n + 1, '\0');
    ck(f(out.data(), out.size(), &n));
    out.resize(n);
    return out;
}

LayerSchedule schedule_from_c(const s2_layer_schedule& s) {
    LayerSchedule ls;
    ls.num_layers = s.num_layers;
    for (int i = 0; i < s.num_dense; ++i) ls.dense_layer_ids.insert(s.dense_layer_ids[i]);
    ls.sparse_pattern = from_c(s.sparse_pattern);
    return ls;
}

}  // namespace

nlohmann::json to_json(const PatternConfig& config) {
    CConfig c(config);
    return nlohmann::json::parse(text_of([&](char* b, size_t cap, size_t* n) { return s2_pattern_to_json(&c.c, b, cap, n); }));
}

nlohmann::json to_json(const LayerSchedule& schedule) {
    CSchedule c(schedule);
    return nlohmann::json::parse(text_of([&](char* b, size_t cap, size_t* n) { return s2_schedule_to_json(&c.s, b, cap, n); }));
}

nlohmann::json to_json(const CsrMask& csr) {
    return nlohmann::json::parse(text_of([&](char* b, size_t cap, size_t* n) {
        return s2_csr_to_json(csr.head_index, csr.num_blocks, csr.row_ptr.data(), csr.col_idx.data(), b, cap, n);
    }));
}

PatternConfig pattern_config_from_json(const nlohmann::json& j) {
    s2_pattern_config c{};
    std::vector<int> offs(4096);
    ck(s2_pattern_from_json(j.dump().c_str(), &c, offs.data(), static_cast<int>(offs.size())));
    return from_c(c);
}

LayerSchedule layer_schedule_from_json(const nlohmann::json& j, const PatternConfig& default_pattern) {
    CConfig def(default_pattern);
    s2_layer_schedule s{};
    std::vector<int> dense(4096), offs(4096);
    ck(s2_schedule_from_json(j.dump().c_str(), &def.c, &s, dense.data(), static_cast<int>(dense.size()),
                             offs.data(), static_cast<int>(offs.size())));
    return schedule_from_c(s);
}

CsrMask csr_from_json(const nlohmann::json& j) {
    const std::string t = j.dump();
    int head = 0, nb = 0;
    int64_t nnz = 0;
    ck(s2_csr_from_json(t.c_str(), &head, &nb, nullptr, 0, nullptr, 0, &nnz));
    CsrMask m;
    m.head_index = head;
    m.num_blocks = nb;
    m.row_ptr.resize(nb + 1);
    m.col_idx.resize(static_cast<size_t>(nnz));
    ck(s2_csr_from_json(t.c_str(), &head, &nb, m.row_ptr.data(), nb + 1, m.col_idx.data(), nnz, &nnz));
    return m;
}

CliConfigFile load_config_file(const std::string& path) {
    s2_config_file f{};
    std::vector<int> dense(4096), offs(8192);
    const int rc = s2_config_file_load(path.c_str(), &f, dense.data(), static_cast<int>(dense.size()),
                                       offs.data(), static_cast<int>(offs.size()));
    if (rc != S2_OK) throw std::runtime_error(s2_last_error());
    CliConfigFile out;
    out.pattern = from_c(f.pattern);
    if (f.has_schedule) out.schedule = schedule_from_c(f.schedule);
    out.out = f.out;
    out.format = f.format;
    return out;
}

std::uint64_t config_hash(const PatternConfig& config) {
    CConfig c(config);
    uint64_t h = 0;
    ck(s2_pattern_hash(&c.c, &h));
    return h;
}

double equivalent_context_length(double seq_len, double local_window, double stride) {
    double v = 0;
    ck(s2_equivalent_context_length(seq_len, local_window, stride, &v));
    return v;
}

double analytic_flops_reduction(double seq_len, double local_window, double stride) {
    double v = 0;
    ck(s2_analytic_flops_reduction(seq_len, local_window, stride, &v));
    return v;
}

double speedup_upper_bound(int num_heads, double seq_len, double local_window) {
    double v = 0;
    ck(s2_speedup_upper_bound(num_heads, seq_len, local_window, &v));
    return v;
}

double flops_per_block_pair(int head_dim, int block_size) {
    return 4.0 * head_dim * static_cast<double>(block_size) * block_size;
}

FlopsReport exact_flops(const PatternConfig& config, int head_dim) {
    CConfig c(config);
    s2_flops_report r{};
    std::vector<int64_t> nph(std::max(1, config.num_heads));
    ck(s2_exact_flops(&c.c, head_dim, &r, nph.data()));
    FlopsReport out;
    out.dense_flops = r.dense_flops;
    out.sparse_flops = r.sparse_flops;
    out.reduction_factor = r.reduction_factor;
    out.equivalent_context = r.equivalent_context;
    for (int h = 0; h < config.num_heads; ++h) out.nnz_per_head.push_back(static_cast<std::size_t>(nph[h]));
    return out;
}

CacheSchedule simulate_decode_cache(const PatternConfig& config, int total_tokens) {
    CConfig c(config);
    ck(s2_pattern_validate(&c.c));
    CacheSchedule cs;
    cs.block_size = config.block_size;
    cs.num_blocks = config.num_blocks();
    cs.total_tokens = total_tokens;
    for (int h = 0; h < config.num_heads; ++h) {
        HeadCacheSchedule hs;
        hs.head_index = h;
        hs.evict_after.resize(cs.num_blocks);
        hs.occupancy.resize(std::max(0, total_tokens));
        hs.dead_blocks.resize(std::max(0, total_tokens));
        ck(s2_simulate_decode_cache(&c.c, total_tokens, h, hs.evict_after.data(), hs.occupancy.data(),
                                    hs.dead_blocks.data(), &hs.peak_tokens, &hs.mean_tokens));
        cs.heads.push_back(std::move(hs));
    }
    return cs;
}

double kv_reduction(const LayerSchedule& schedule) {
    CSchedule c(schedule);
    double v = 0;
    ck(s2_kv_reduction(&c.s, &v));
    return v;
}

}  // namespace shardattn
