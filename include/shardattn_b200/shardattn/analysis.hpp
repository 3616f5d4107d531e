// Drop-in for the reference's shardattn/analysis.hpp over the C ABI
// (s2_exact_flops, s2_simulate_decode_cache, s2_kv_reduction, ...).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "shardattn/pattern.hpp"

namespace shardattn {

double equivalent_context_length(double seq_len, double local_window, double stride);
double analytic_flops_reduction(double seq_len, double local_window, double stride);
double speedup_upper_bound(int num_heads, double seq_len, double local_window);
double flops_per_block_pair(int head_dim, int block_size);

struct FlopsReport {
    double dense_flops = 0.0;
    double sparse_flops = 0.0;
    double reduction_factor = 0.0;
    double equivalent_context = 0.0;
    std::vector<std::size_t> nnz_per_head;
};
FlopsReport exact_flops(const PatternConfig& config, int head_dim);

struct HeadCacheSchedule {
    int head_index = 0;
    std::vector<int> evict_after;
    std::vector<std::int64_t> occupancy;
    std::vector<int> dead_blocks;
    std::int64_t peak_tokens = 0;
    double mean_tokens = 0.0;
};

struct CacheSchedule {
    int block_size = 0;
    int num_blocks = 0;
    int total_tokens = 0;
    std::vector<HeadCacheSchedule> heads;
};
CacheSchedule simulate_decode_cache(const PatternConfig& config, int total_tokens);

double kv_reduction(const LayerSchedule& schedule);

}  // namespace shardattn
