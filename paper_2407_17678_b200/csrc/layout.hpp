// Host-side S2 layout builder: policy -> per-head CSR (forward) and CSC
// (backward), emitted analytically in O(nnz) instead of the reference's
// O(B^2) mask materialisation (pattern.cpp:127-158 + csr.cpp:35-47), and the
// tile work lists the sm_100a kernels consume.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/s2attn.h"

namespace s2 {

struct Segment {
    int start = 0, end = 0, stride = 1;
    std::vector<int> offsets;
};

// Owned, normalised copy of s2_pattern_config (pattern.hpp:37-60).
struct Pattern {
    int seq_len = 0, block_size = 1, num_heads = 1, num_kv_heads = 0;
    int local_blocks = 1, local_stride = 1;
    std::vector<Segment> segments;

    int num_blocks() const {
        return static_cast<int>((static_cast<long long>(seq_len) + block_size - 1) / block_size);
    }
    int kv_heads() const { return num_kv_heads > 0 ? num_kv_heads : num_heads; }
    int heads_per_group() const { return num_heads / kv_heads(); }
    int group_of(int h) const { return h / heads_per_group(); }
    int offset_for(int s, int head) const;  // pattern.cpp:16-34
};

Pattern from_c(const s2_pattern_config* c);
// "" when valid, else the reference's std::invalid_argument message
// (pattern.cpp:36-79).
std::string validate(const Pattern& p);

// Key blocks of row i of head `head`, ascending (analytic).
void row_blocks(const Pattern& p, int head, int i, std::vector<int>& out);

struct Csr {
    int num_blocks = 0;
    std::vector<int> ptr;  // B+1
    std::vector<int> idx;  // nnz
    int64_t nnz() const { return static_cast<int64_t>(idx.size()); }
};

Csr build_csr(const Pattern& p, int head);
Csr transpose(const Csr& csr);  // CSR <-> CSC of the same bits
// "" or the CsrMask::validate message (csr.cpp:11-33).
std::string validate_csr(int num_blocks, const int* ptr, const int* idx, int64_t nnz);
// evict_after from the CSC (analysis.cpp:76-82): last attending row.
std::vector<int> evict_after(const Csr& csc);
// check_kv_cache_efficiency (verify.cpp:53-72) from the CSC.
bool kv_efficient(const Csr& csc);

// ---------------------------------------------------------------------------
// Tile work lists.
//
// Token granularity of the masks: 16x16 squares.  A 128-row query tile is 8
// row groups; a 64-key chunk is 4 column groups; bit (g*4 + c) of a chunk mask
// says whether row group g may attend column group c (block-level bit; token
// causality is applied in-kernel).  Valid whenever block_size % 16 == 0, so the
// tcgen05 kernels serve every such block size, not just 64.
constexpr int kTileQ = 128;
constexpr int kChunk = 64;

struct ChunkEntry {
    int32_t chunk;  // key chunk index (keys chunk*64 .. +63)
    uint32_t mask;  // 8 row groups x 4 column groups
};

// Forward / dQ: per (head, q tile) the ascending list of key chunks.
struct FwdList {
    int num_qtiles = 0;
    std::vector<int64_t> offset;     // [H * num_qtiles + 1]
    std::vector<ChunkEntry> chunks;  // concatenated
};
FwdList build_fwd_list(const std::vector<Csr>& csr, int seq_len, int block_size);

// Forward / dQ steps for a PAIR of adjacent query tiles (2p, 2p+1) sharing
// every K/V load: the union of both tiles' chunk lists, two chunks per step,
// with each tile's masks (0 = the tile skips that chunk).
struct PairStep {
    int32_t c0, c1;      // chunks (c1 = -1 when the step holds one chunk)
    uint32_t a0, a1;     // tile 2p   masks for c0 / c1
    uint32_t b0, b1;     // tile 2p+1 masks for c0 / c1
};
struct PairList {
    int num_pairs = 0;
    std::vector<int64_t> offset;  // [H * num_pairs + 1]
    std::vector<PairStep> steps;
};
PairList build_pair_list(const FwdList& fwd, int num_heads);

// dK/dV: per (kv group, key tile) a pair of chunks (c1 may be -1) and the
// ascending list of q tiles with the two chunk masks.  Chunks of one group
// are paired by similarity of their q-tile lists so stripe blocks pair with
// stripe blocks (SURVEY §7 hard part 2).
struct BwdTile {
    int32_t group;  // representative head = group * hpg
    int32_t c0, c1;
    int64_t offset;
    int32_t count;
};
struct BwdEntry {
    int32_t qtile;
    uint32_t mask0, mask1;
};
struct BwdList {
    std::vector<BwdTile> tiles;
    std::vector<BwdEntry> entries;
    // some 64-key chunk of some kv group has no attending query, so no tile
    // covers it: its dK / dV are 0 and must be written as such (zero-filled)
    bool uncovered = false;
};
BwdList build_bwd_list(const FwdList& fwd, int num_heads, int num_kv_heads, int seq_len);

// LPT partition (no reference symbol).
void partition_lpt(int num_units, const int64_t* weights, int num_ranks, int* owner,
                   int64_t* load);

}  // namespace s2
