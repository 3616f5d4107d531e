// C ABI: JSON documents of the layout policy / CSR masks / layer schedule and
// the config-file loader (reference serialize.hpp, serialize.cpp), plus the
// layout analysis that needs no device (reference analysis.hpp, analysis.cpp).
//
// Documents are built with nlohmann::json (the same header-only library the
// reference uses, taken from the image); its default object type keeps keys
// sorted and dump() is compact, which is the reference's canonical encoding,
// so s2_pattern_hash == shardattn::config_hash bit for bit (pinned by
// tests/test_serialize.py against fixtures made by the reference itself).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "capi_internal.hpp"
#include "layout.hpp"

using nlohmann::json;

namespace s2 {
namespace {

int kv_heads_of(const s2_pattern_config* c) { return c->num_kv_heads > 0 ? c->num_kv_heads : c->num_heads; }

json pattern_doc(const s2_pattern_config* c) {
    json segments = json::array();
    for (int s = 0; s < c->num_segments; ++s) {
        const s2_stride_segment& g = c->segments[s];
        json seg{{"start_block_distance", g.start_block_distance},
                 {"end_block_distance", g.end_block_distance},
                 {"stride", g.stride}};
        if (g.offsets && g.num_offsets > 0)
            seg["offsets"] = std::vector<int>(g.offsets, g.offsets + g.num_offsets);
        segments.push_back(std::move(seg));
    }
    return json{{"seq_len", c->seq_len},
                {"block_size", c->block_size},
                {"num_heads", c->num_heads},
                {"num_kv_heads", kv_heads_of(c)},
                {"local_blocks", c->local_blocks},
                {"local_stride", c->local_stride},
                {"stride_segments", segments},
                {"offset_scheme", "head_mod_stride"}};
}

// Throws std::invalid_argument (validation) or json::exception (shape).
void pattern_from_doc(const json& j, s2_pattern_config* c, int* offsets_buf, int offsets_cap) {
    std::memset(c, 0, sizeof(*c));
    c->seq_len = j.at("seq_len").get<int>();
    c->block_size = j.at("block_size").get<int>();
    c->num_heads = j.at("num_heads").get<int>();
    c->num_kv_heads = j.value("num_kv_heads", c->num_heads);
    c->local_blocks = j.value("local_blocks", 1);
    c->local_stride = j.value("local_stride", 1);
    int used = 0;
    if (j.contains("stride_segments")) {
        const json& segs = j.at("stride_segments");
        if (segs.size() > static_cast<size_t>(S2_MAX_SEGMENTS))
            throw std::invalid_argument("at most " + std::to_string(S2_MAX_SEGMENTS) +
                                        " stride_segments are supported");
        for (const json& sj : segs) {
            s2_stride_segment& g = c->segments[c->num_segments++];
            g.start_block_distance = sj.at("start_block_distance").get<int>();
            g.end_block_distance = sj.at("end_block_distance").get<int>();
            g.stride = sj.at("stride").get<int>();
            if (sj.contains("offsets")) {
                const std::vector<int> o = sj.at("offsets").get<std::vector<int>>();
                if (used + static_cast<int>(o.size()) > offsets_cap || (!offsets_buf && !o.empty()))
                    throw std::length_error("offsets buffer too small");
                std::copy(o.begin(), o.end(), offsets_buf + used);
                g.offsets = offsets_buf + used;
                g.num_offsets = static_cast<int>(o.size());
                used += g.num_offsets;
            }
        }
    }
    const std::string scheme = j.value("offset_scheme", std::string("head_mod_stride"));
    if (scheme != "head_mod_stride") throw std::invalid_argument("unknown offset_scheme '" + scheme + "'");
    const std::string msg = validate(from_c(c));
    if (!msg.empty()) throw std::invalid_argument(msg);
}

std::string schedule_msg(const s2_layer_schedule* s) {
    if (s->num_layers < 1) return "num_layers must be positive";
    for (int i = 0; i < s->num_dense; ++i)
        if (s->dense_layer_ids[i] < 0 || s->dense_layer_ids[i] >= s->num_layers)
            return "dense layer id " + std::to_string(s->dense_layer_ids[i]) + " outside [0, num_layers)";
    return validate(from_c(&s->sparse_pattern));
}

json schedule_doc(const s2_layer_schedule* s) {
    std::set<int> ids(s->dense_layer_ids, s->dense_layer_ids + s->num_dense);
    return json{{"num_layers", s->num_layers},
                {"dense_layer_ids", std::vector<int>(ids.begin(), ids.end())},
                {"sparse_pattern", pattern_doc(&s->sparse_pattern)}};
}

void schedule_from_doc(const json& j, const s2_pattern_config* def, s2_layer_schedule* s, int* dense_buf,
                       int dense_cap, int* offsets_buf, int offsets_cap) {
    std::memset(s, 0, sizeof(*s));
    s->num_layers = j.at("num_layers").get<int>();
    std::set<int> ids;
    if (j.contains("dense_layer_ids"))
        for (const json& id : j.at("dense_layer_ids")) ids.insert(id.get<int>());
    if (static_cast<int>(ids.size()) > dense_cap || (!dense_buf && !ids.empty()))
        throw std::length_error("dense layer buffer too small");
    int n = 0;
    for (int id : ids) dense_buf[n++] = id;
    s->num_dense = n;
    s->dense_layer_ids = dense_buf;
    if (j.contains("sparse_pattern")) {
        pattern_from_doc(j.at("sparse_pattern"), &s->sparse_pattern, offsets_buf, offsets_cap);
    } else {
        if (!def) throw std::invalid_argument("schedule has no sparse_pattern and no default pattern");
        s->sparse_pattern = *def;  // offsets (if any) stay the caller's
    }
    const std::string msg = schedule_msg(s);
    if (!msg.empty()) throw std::invalid_argument(msg);
}

int emit(const json& doc, char* buf, size_t cap, size_t* len) {
    const std::string out = doc.dump();
    if (len) *len = out.size();
    if (!buf) return S2_OK;
    if (cap < out.size() + 1) return fail(S2_ERR_BUFFER_TOO_SMALL, "output buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
    return S2_OK;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::length_error& e) {
        return fail(S2_ERR_BUFFER_TOO_SMALL, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(S2_ERR_INVALID_ARGUMENT, e.what());
    } catch (const json::exception& e) {
        return fail(S2_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return fail(S2_ERR_INVALID_ARGUMENT, e.what());
    }
}

// Retained-set bookkeeping of one head from its CSC (analysis.cpp:57-104):
// key block j is kept for decode rows (j, evict_after[j]]; a difference array
// gives the retained-block count of every row in O(B).
struct HeadCache {
    std::vector<int> ev;         // evict_after
    std::vector<int> kept_prev;  // retained blocks j < bt at row bt
    std::vector<int> row_len;    // |row(bt)|
};

HeadCache head_cache(const Pattern& p, int head) {
    const Csr csr = build_csr(p, head);
    const Csr csc = transpose(csr);
    HeadCache hc;
    hc.ev = evict_after(csc);
    const int B = p.num_blocks();
    std::vector<int> diff(B + 1, 0);
    for (int j = 0; j < B; ++j)
        if (hc.ev[j] > j) {
            diff[j + 1] += 1;
            diff[hc.ev[j] + 1 <= B ? hc.ev[j] + 1 : B] -= 1;
        }
    hc.kept_prev.assign(B, 0);
    int run = 0;
    for (int bt = 0; bt < B; ++bt) {
        run += diff[bt];
        hc.kept_prev[bt] = run;
    }
    hc.row_len.resize(B);
    for (int bt = 0; bt < B; ++bt) hc.row_len[bt] = csr.ptr[bt + 1] - csr.ptr[bt];
    return hc;
}

}  // namespace
}  // namespace s2

using namespace s2;

extern "C" {

int s2_pattern_to_json(const s2_pattern_config* cfg, char* buf, size_t cap, size_t* len) {
    if (!cfg) return fail(S2_ERR_INVALID_ARGUMENT, "config is null");
    return guarded([&]() -> int { return emit(pattern_doc(cfg), buf, cap, len); });
}

int s2_pattern_from_json(const char* text, s2_pattern_config* cfg, int* offsets_buf, int offsets_cap) {
    if (!text || !cfg) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        pattern_from_doc(json::parse(text), cfg, offsets_buf, offsets_cap);
        return S2_OK;
    });
}

int s2_pattern_hash(const s2_pattern_config* cfg, uint64_t* hash) {
    if (!cfg || !hash) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        const std::string doc = pattern_doc(cfg).dump();
        uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a 64
        for (unsigned char ch : doc) {
            h ^= ch;
            h *= 0x100000001b3ull;
        }
        *hash = h;
        return S2_OK;
    });
}

int s2_csr_to_json(int head_index, int num_blocks, const int* row_ptr, const int* col_idx, char* buf,
                   size_t cap, size_t* len) {
    if (num_blocks < 0 || !row_ptr) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        const int nnz = row_ptr[num_blocks];
        if (nnz > 0 && !col_idx) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
        const json doc{{"head_index", head_index},
                       {"num_blocks", num_blocks},
                       {"row_ptr", std::vector<int>(row_ptr, row_ptr + num_blocks + 1)},
                       {"col_idx", std::vector<int>(col_idx, col_idx + nnz)}};
        return emit(doc, buf, cap, len);
    });
}

int s2_csr_from_json(const char* text, int* head_index, int* num_blocks, int* row_ptr, int row_cap,
                     int* col_idx, int64_t col_cap, int64_t* nnz) {
    if (!text) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        const json j = json::parse(text);
        const int nb = j.at("num_blocks").get<int>();
        const std::vector<int> rp = j.at("row_ptr").get<std::vector<int>>();
        const std::vector<int> ci = j.at("col_idx").get<std::vector<int>>();
        const std::string msg = validate_csr(nb, rp.data(), ci.data(), static_cast<int64_t>(ci.size()));
        if (!msg.empty() || static_cast<int>(rp.size()) != nb + 1)
            throw std::invalid_argument(msg.empty() ? "row_ptr must have num_blocks + 1 entries" : msg);
        if (head_index) *head_index = j.value("head_index", 0);
        if (num_blocks) *num_blocks = nb;
        if (nnz) *nnz = static_cast<int64_t>(ci.size());
        if (row_ptr) {
            if (row_cap < nb + 1) return fail(S2_ERR_BUFFER_TOO_SMALL, "row_ptr buffer too small");
            std::copy(rp.begin(), rp.end(), row_ptr);
        }
        if (col_idx) {
            if (col_cap < static_cast<int64_t>(ci.size()))
                return fail(S2_ERR_BUFFER_TOO_SMALL, "col_idx buffer too small");
            std::copy(ci.begin(), ci.end(), col_idx);
        }
        return S2_OK;
    });
}

int s2_schedule_validate(const s2_layer_schedule* schedule) {
    if (!schedule) return fail(S2_ERR_INVALID_ARGUMENT, "schedule is null");
    if (schedule->num_dense > 0 && !schedule->dense_layer_ids)
        return fail(S2_ERR_INVALID_ARGUMENT, "dense_layer_ids is null");
    const std::string msg = schedule_msg(schedule);
    return msg.empty() ? S2_OK : fail(S2_ERR_INVALID_ARGUMENT, msg);
}

int s2_schedule_to_json(const s2_layer_schedule* schedule, char* buf, size_t cap, size_t* len) {
    if (int rc = s2_schedule_validate(schedule)) return rc;
    return guarded([&]() -> int { return emit(schedule_doc(schedule), buf, cap, len); });
}

int s2_schedule_from_json(const char* text, const s2_pattern_config* default_pattern,
                          s2_layer_schedule* schedule, int* dense_buf, int dense_cap, int* offsets_buf,
                          int offsets_cap) {
    if (!text || !schedule) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        schedule_from_doc(json::parse(text), default_pattern, schedule, dense_buf, dense_cap, offsets_buf,
                          offsets_cap);
        return S2_OK;
    });
}

int s2_config_file_load(const char* path, s2_config_file* file, int* dense_buf, int dense_cap,
                        int* offsets_buf, int offsets_cap) {
    if (!path || !file) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    std::memset(file, 0, sizeof(*file));
    std::ifstream in(path);
    if (!in) return fail(S2_ERR_CONFIG, std::string("cannot open config file '") + path + "'");
    json j;
    try {
        in >> j;
    } catch (const json::parse_error& e) {
        return fail(S2_ERR_CONFIG, std::string("config '") + path + "': " + e.what());
    }
    try {
        const json& pj = j.contains("pattern") ? j.at("pattern") : j;
        pattern_from_doc(pj, &file->pattern, offsets_buf, offsets_cap);
        int used = 0;
        for (int s = 0; s < file->pattern.num_segments; ++s) used += file->pattern.segments[s].num_offsets;
        if (j.contains("schedule")) {
            schedule_from_doc(j.at("schedule"), &file->pattern, &file->schedule, dense_buf, dense_cap,
                              offsets_buf ? offsets_buf + used : nullptr, offsets_cap - used);
            file->has_schedule = 1;
        }
        if (j.contains("report")) {
            const std::string out = j.at("report").value("out", std::string());
            const std::string fmt = j.at("report").value("format", std::string());
            if (out.size() >= sizeof(file->out) || fmt.size() >= sizeof(file->format))
                throw std::invalid_argument("report out/format too long");
            std::memcpy(file->out, out.c_str(), out.size() + 1);
            std::memcpy(file->format, fmt.c_str(), fmt.size() + 1);
        }
        return S2_OK;
    } catch (const std::length_error& e) {
        return fail(S2_ERR_BUFFER_TOO_SMALL, e.what());
    } catch (const std::exception& e) {
        return fail(S2_ERR_CONFIG, std::string("config '") + path + "': " + e.what());
    }
}

int s2_equivalent_context_length(double seq_len, double local_window, double stride, double* out) {
    if (!out) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (local_window < 1.0 || local_window > seq_len)
        return fail(S2_ERR_INVALID_ARGUMENT, "local_window must lie in [1, seq_len]");
    if (stride < 1.0) return fail(S2_ERR_INVALID_ARGUMENT, "stride must be >= 1");
    *out = local_window + (seq_len - local_window) / stride;
    return S2_OK;
}

int s2_analytic_flops_reduction(double seq_len, double local_window, double stride, double* out) {
    double eq = 0.0;
    if (int rc = s2_equivalent_context_length(seq_len, local_window, stride, &eq)) return rc;
    *out = seq_len / eq;
    return S2_OK;
}

int s2_speedup_upper_bound(int num_heads, double seq_len, double local_window, double* out) {
    if (num_heads < 1) return fail(S2_ERR_INVALID_ARGUMENT, "num_heads must be positive");
    return s2_analytic_flops_reduction(seq_len, local_window, num_heads, out);
}

int s2_exact_flops(const s2_pattern_config* cfg, int head_dim, s2_flops_report* report, int64_t* nnz_per_head) {
    if (!cfg || !report) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    const Pattern p = from_c(cfg);
    const std::string msg = validate(p);
    if (!msg.empty()) return fail(S2_ERR_INVALID_ARGUMENT, msg);
    if (head_dim < 1) return fail(S2_ERR_INVALID_ARGUMENT, "head_dim must be positive");
    const double per_pair = 4.0 * head_dim * static_cast<double>(p.block_size) * p.block_size;
    const double B = p.num_blocks();
    int64_t total = 0;
    for (int h = 0; h < p.num_heads; ++h) {
        const int64_t n = build_csr(p, h).nnz();
        if (nnz_per_head) nnz_per_head[h] = n;
        total += n;
    }
    report->dense_flops = per_pair * (B * (B + 1) / 2.0) * p.num_heads;
    report->sparse_flops = per_pair * static_cast<double>(total);
    report->reduction_factor = report->dense_flops / report->sparse_flops;
    report->equivalent_context = p.seq_len / report->reduction_factor;
    return S2_OK;
}

int s2_simulate_decode_cache(const s2_pattern_config* cfg, int total_tokens, int head, int* evict_after_out,
                             int64_t* occupancy, int* dead_blocks, int64_t* peak_tokens, double* mean_tokens) {
    if (!cfg) return fail(S2_ERR_INVALID_ARGUMENT, "config is null");
    const Pattern p = from_c(cfg);
    const std::string msg = validate(p);
    if (!msg.empty()) return fail(S2_ERR_INVALID_ARGUMENT, msg);
    if (total_tokens < 1 || total_tokens > p.seq_len)
        return fail(S2_ERR_INVALID_ARGUMENT, "total_tokens must lie in [1, seq_len]");
    if (head < 0 || head >= p.num_heads) return fail(S2_ERR_INVALID_ARGUMENT, "head index out of range");
    const HeadCache hc = head_cache(p, head);
    if (evict_after_out) std::copy(hc.ev.begin(), hc.ev.end(), evict_after_out);
    const int S = p.block_size;
    int64_t peak = 0;
    double sum = 0.0;
    for (int t = 0; t < total_tokens; ++t) {
        const int bt = t / S;
        // retained: the kept earlier blocks plus block bt itself (its diagonal keeps it)
        const int64_t tokens = static_cast<int64_t>(hc.kept_prev[bt]) * S + (t - bt * S + 1);
        if (occupancy) occupancy[t] = tokens;
        // row(bt) is a subset of the retained set; every other retained block is dead
        if (dead_blocks) dead_blocks[t] = hc.kept_prev[bt] + 1 - hc.row_len[bt];
        peak = std::max(peak, tokens);
        sum += static_cast<double>(tokens);
    }
    if (peak_tokens) *peak_tokens = peak;
    if (mean_tokens) *mean_tokens = sum / total_tokens;
    return S2_OK;
}

int s2_kv_reduction(const s2_layer_schedule* schedule, double* percent) {
    if (int rc = s2_schedule_validate(schedule)) return rc;
    if (!percent) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    const Pattern p = from_c(&schedule->sparse_pattern);
    const int N = p.seq_len, S = p.block_size, bt = (N - 1) / S;
    double frac = 0.0;
    for (int h = 0; h < p.num_heads; ++h) {
        const HeadCache hc = head_cache(p, h);
        frac += static_cast<double>(static_cast<int64_t>(hc.kept_prev[bt]) * S + (N - 1 - bt * S + 1)) / N;
    }
    frac /= p.num_heads;
    const std::set<int> dense(schedule->dense_layer_ids, schedule->dense_layer_ids + schedule->num_dense);
    double retained = 0.0;
    for (int l = 0; l < schedule->num_layers; ++l) retained += dense.count(l) ? 1.0 : frac;
    retained /= schedule->num_layers;
    *percent = 100.0 * (1.0 - retained);
    return S2_OK;
}

}  // extern "C"
