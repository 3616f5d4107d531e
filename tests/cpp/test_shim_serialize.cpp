// C++ drop-in check (host only): the reference's serialize.hpp / analysis.hpp
// API from include/shardattn_b200, exercised the way
// /root/reference/proj/tests/test_serialize.cpp and test_analysis.cpp use it.
// Argument 1: a directory for temporary config files.
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>

#include "shardattn/analysis.hpp"
#include "shardattn/serialize.hpp"

using namespace shardattn;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)

template <class E, class F>
static bool throws_with(F&& f, const std::string& needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    }
    return false;
}

static std::string write(const std::string& dir, const std::string& name, const std::string& body) {
    const std::string path = dir + "/" + name;
    std::ofstream(path) << body;
    return path;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    // pattern round trip with offsets and GQA (test_serialize.cpp:30-49)
    PatternConfig cfg = make_multi_stride_config(256, 16, 8, 2, 8, 3, 6);
    cfg.num_kv_heads = 4;
    cfg.stride_segments[0].offsets = {0, 1, 2, 0};
    cfg.validate();
    const nlohmann::json doc = to_json(cfg);
    for (const char* key : {"seq_len", "block_size", "num_heads", "num_kv_heads", "local_blocks",
                            "local_stride", "stride_segments", "offset_scheme"})
        CHECK(doc.contains(key));
    const PatternConfig back = pattern_config_from_json(doc);
    CHECK(to_json(back) == doc);
    CHECK(config_hash(back) == config_hash(cfg));

    // schedule round trip + inheritance (:51-67)
    LayerSchedule schedule;
    schedule.num_layers = 24;
    schedule.dense_layer_ids = {0, 1};
    schedule.sparse_pattern = make_single_stride_config(512, 64, 4, 1, 4);
    const LayerSchedule sback = layer_schedule_from_json(to_json(schedule), schedule.sparse_pattern);
    CHECK(sback.num_layers == 24);
    CHECK(sback.dense_layer_ids == std::set<int>({0, 1}));
    const LayerSchedule inh = layer_schedule_from_json(nlohmann::json{{"num_layers", 8}}, schedule.sparse_pattern);
    CHECK(inh.dense_layer_ids.empty());
    CHECK(to_json(inh.sparse_pattern) == to_json(schedule.sparse_pattern));

    // csr round trip (:88-94)
    const CsrMask csr = to_csr(build_head_mask(make_single_stride_config(8, 1, 4, 2, 3), 1));
    const CsrMask cback = csr_from_json(to_json(csr));
    CHECK(cback.row_ptr == csr.row_ptr && cback.col_idx == csr.col_idx && cback.head_index == csr.head_index);

    // config files (:96-111) and diagnostics (:113-133)
    const CliConfigFile f = load_config_file(write(dir, "a.json", R"({
        "pattern": {"seq_len": 512, "block_size": 64, "num_heads": 4, "local_blocks": 1,
                    "stride_segments": [{"start_block_distance": 1, "end_block_distance": 8, "stride": 2}]},
        "schedule": {"num_layers": 12, "dense_layer_ids": [0]},
        "report": {"out": "r.csv", "format": "csv"}})"));
    CHECK(f.pattern.num_heads == 4 && f.pattern.kv_heads() == 4);
    CHECK(f.schedule.has_value() && f.schedule->num_layers == 12);
    CHECK(to_json(f.schedule->sparse_pattern) == to_json(f.pattern));
    CHECK(f.out == "r.csv" && f.format == "csv");
    const CliConfigFile plain = load_config_file(write(dir, "b.json", R"({"seq_len": 64, "block_size": 8, "num_heads": 2})"));
    CHECK(plain.pattern.num_blocks() == 8 && !plain.schedule.has_value());
    CHECK(throws_with<std::runtime_error>([&] { load_config_file(write(dir, "c.json", R"({"pattern": {"block_size": 64, "num_heads": 4}})")); }, "seq_len"));
    CHECK(throws_with<std::runtime_error>([&] { load_config_file(write(dir, "d.json", R"({"seq_len": 64, "block_size": 8, "num_heads": 4,
        "stride_segments": [{"start_block_distance": 1, "end_block_distance": 8, "stride": 0}]})")); }, "stride"));
    CHECK(throws_with<std::runtime_error>([&] { load_config_file(write(dir, "e.json", R"({"seq_len": 64, "block_size": 8, "num_heads": 4, "offset_scheme": "mystery"})")); }, "offset_scheme"));
    CHECK(throws_with<std::runtime_error>([&] { load_config_file("does_not_exist.json"); }, "cannot open"));

    // hash stability (:135-141)
    const PatternConfig a = make_single_stride_config(512, 64, 4, 1, 4);
    PatternConfig b = a;
    CHECK(config_hash(a) == config_hash(b));
    b.stride_segments[0].stride = 5;
    CHECK(config_hash(a) != config_hash(b));

    // analysis (test_analysis.cpp): closed forms, exact flops, cache schedule, kv reduction
    CHECK(equivalent_context_length(1024, 64, 4) == 64 + 960 / 4.0);
    CHECK(throws_with<std::invalid_argument>([] { equivalent_context_length(100, 0, 2); }, "local_window"));
    const FlopsReport fr = exact_flops(make_single_stride_config(512, 64, 4, 1, 4), 128);
    CHECK(fr.nnz_per_head.size() == 4 && fr.reduction_factor == fr.dense_flops / fr.sparse_flops);
    const PatternConfig dc = make_single_stride_config(4096, 64, 8, 2, 4);
    const CacheSchedule cs = simulate_decode_cache(dc, 4096);
    CHECK(cs.heads.size() == 8 && cs.heads[0].occupancy.size() == 4096);
    for (const HeadCacheSchedule& h : cs.heads) CHECK(h.dead_blocks.back() == 0);  // KV-efficient: nothing dead
    LayerSchedule ls;
    ls.num_layers = 24;
    ls.dense_layer_ids = {0, 1};
    ls.sparse_pattern = make_single_stride_config(8192, 64, 16, 1, 15);
    CHECK(kv_reduction(ls) > 80.0 && kv_reduction(ls) < 90.0);

    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
