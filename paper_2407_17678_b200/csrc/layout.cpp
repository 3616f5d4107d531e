#include "layout.hpp"

#include <algorithm>
#include <numeric>

namespace s2 {

int Pattern::offset_for(int s, int head) const {
    const Segment& seg = segments[s];
    int raw;
    if (!seg.offsets.empty())
        raw = static_cast<int>(seg.offsets.size()) == num_heads ? seg.offsets[head]
                                                                : seg.offsets[group_of(head)];
    else
        raw = group_of(head);  // OffsetScheme::HeadModStride
    return raw % seg.stride;
}

Pattern from_c(const s2_pattern_config* c) {
    Pattern p;
    p.seq_len = c->seq_len;
    p.block_size = c->block_size;
    p.num_heads = c->num_heads;
    p.num_kv_heads = c->num_kv_heads;
    p.local_blocks = c->local_blocks;
    p.local_stride = c->local_stride;
    const int ns = std::max(0, std::min(c->num_segments, S2_MAX_SEGMENTS));
    for (int s = 0; s < ns; ++s) {
        Segment seg;
        seg.start = c->segments[s].start_block_distance;
        seg.end = c->segments[s].end_block_distance;
        seg.stride = c->segments[s].stride;
        if (c->segments[s].offsets && c->segments[s].num_offsets > 0)
            seg.offsets.assign(c->segments[s].offsets,
                               c->segments[s].offsets + c->segments[s].num_offsets);
        p.segments.push_back(std::move(seg));
    }
    return p;
}

std::string validate(const Pattern& p) {
    if (p.seq_len < 1) return "seq_len must be positive";
    if (p.block_size < 1) return "block_size must be positive";
    if (p.num_heads < 1) return "num_heads must be positive";
    if (p.num_kv_heads < 0) return "num_kv_heads must be positive";
    if (p.num_heads % p.kv_heads() != 0) return "num_kv_heads must divide num_heads";
    if (p.local_blocks < 1) return "local_blocks must be >= 1";
    if (p.local_stride < 1) return "local_stride must be >= 1";
    const int blocks = p.num_blocks();
    int prev_end = p.local_blocks;
    for (std::size_t s = 0; s < p.segments.size(); ++s) {
        const Segment& seg = p.segments[s];
        if (seg.stride < 1) return "segment stride must be >= 1";
        if (seg.start < p.local_blocks) return "segment start must be >= local_blocks";
        if (seg.end > blocks) return "segment end must be <= num_blocks";
        if (seg.start >= seg.end) return "segment range must be non-empty";
        if (seg.start < prev_end && s > 0) return "segments must be ordered and non-overlapping";
        prev_end = seg.end;
        if (!seg.offsets.empty()) {
            const int n = static_cast<int>(seg.offsets.size());
            if (n != p.num_heads && n != p.kv_heads())
                return "segment offsets must list one entry per head or per kv head";
            for (int o : seg.offsets)
                if (o < 0) return "offsets must be non-negative";
            if (n == p.num_heads)
                for (int h = 0; h < p.num_heads; ++h) {
                    const int lead = p.group_of(h) * p.heads_per_group();
                    if (seg.offsets[h] % seg.stride != seg.offsets[lead] % seg.stride)
                        return "offsets must agree within each kv group";
                }
        }
    }
    return "";
}

// Row i = (strided members of every segment, farthest segment first) then the
// local window, which is exactly ascending key order because validated
// segments are ordered by distance and start at or beyond local_blocks.
// Equivalent to scanning j <= i with the bit rule of pattern.cpp:138-155.
void row_blocks(const Pattern& p, int head, int i, std::vector<int>& out) {
    out.clear();
    for (int s = static_cast<int>(p.segments.size()) - 1; s >= 0; --s) {
        const Segment& seg = p.segments[s];
        const int lo = std::max(0, i - seg.end + 1);
        const int hi = i - seg.start;
        if (hi < lo) continue;
        const int o = p.offset_for(s, head);
        int j = std::max(lo, o);
        const int rem = (j - o) % seg.stride;
        if (rem) j += seg.stride - rem;
        for (; j <= hi; j += seg.stride) out.push_back(j);
    }
    for (int d = std::min(p.local_blocks - 1, i); d >= 0; --d)
        if (d % p.local_stride == 0) out.push_back(i - d);
}

Csr build_csr(const Pattern& p, int head) {
    Csr c;
    c.num_blocks = p.num_blocks();
    c.ptr.assign(c.num_blocks + 1, 0);
    std::vector<int> row;
    for (int i = 0; i < c.num_blocks; ++i) {
        row_blocks(p, head, i, row);
        c.idx.insert(c.idx.end(), row.begin(), row.end());
        c.ptr[i + 1] = static_cast<int>(c.idx.size());
    }
    return c;
}

Csr transpose(const Csr& csr) {
    Csr t;
    const int B = csr.num_blocks;
    t.num_blocks = B;
    t.ptr.assign(B + 1, 0);
    t.idx.resize(csr.idx.size());
    for (int j : csr.idx) t.ptr[j + 1]++;
    for (int j = 0; j < B; ++j) t.ptr[j + 1] += t.ptr[j];
    std::vector<int> fill(t.ptr.begin(), t.ptr.end() - 1);
    for (int i = 0; i < B; ++i)
        for (int q = csr.ptr[i]; q < csr.ptr[i + 1]; ++q) t.idx[fill[csr.idx[q]]++] = i;
    return t;
}

std::string validate_csr(int num_blocks, const int* ptr, const int* idx, int64_t nnz) {
    if (num_blocks < 1) return "csr num_blocks must be positive";
    if (!ptr || (nnz > 0 && !idx)) return "row_ptr must have num_blocks + 1 entries";
    if (ptr[0] != 0) return "row_ptr[0] must be 0";
    if (ptr[num_blocks] != nnz) return "row_ptr[B] must equal col_idx length";
    for (int i = 0; i < num_blocks; ++i) {
        if (ptr[i] > ptr[i + 1]) return "row_ptr must be non-decreasing";
        for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
            if (q < 0 || q >= nnz) return "row_ptr must be non-decreasing";
            const int col = idx[q];
            if (col < 0 || col >= num_blocks)
                return "column index " + std::to_string(col) + " outside [0, num_blocks)";
            if (col > i)
                return "column " + std::to_string(col) + " above the diagonal in row " +
                       std::to_string(i);
            if (q > ptr[i] && idx[q - 1] >= col)
                return "columns must be strictly ascending within a row";
        }
    }
    return "";
}

std::vector<int> evict_after(const Csr& csc) {
    std::vector<int> ev(csc.num_blocks);
    for (int j = 0; j < csc.num_blocks; ++j)
        ev[j] = csc.ptr[j + 1] > csc.ptr[j] ? std::max(j, csc.idx[csc.ptr[j + 1] - 1]) : j;
    return ev;
}

bool kv_efficient(const Csr& csc) {
    for (int j = 0; j < csc.num_blocks; ++j) {
        const int n = csc.ptr[j + 1] - csc.ptr[j];
        if (n == 0) continue;
        if (csc.idx[csc.ptr[j]] != j) return false;  // diagonal is always first
        if (csc.idx[csc.ptr[j + 1] - 1] != j + n - 1) return false;
    }
    return true;
}

FwdList build_fwd_list(const std::vector<Csr>& csr, int seq_len, int block_size) {
    FwdList f;
    const int H = static_cast<int>(csr.size());
    f.num_qtiles = (seq_len + kTileQ - 1) / kTileQ;
    const int nchunks = (seq_len + kChunk - 1) / kChunk;
    std::vector<std::vector<ChunkEntry>> per(static_cast<std::size_t>(H) * f.num_qtiles);
#pragma omp parallel
    {
        std::vector<uint32_t> m(nchunks, 0);
        std::vector<int> touched;
#pragma omp for schedule(dynamic)
        for (int h = 0; h < H; ++h) {
            const Csr& c = csr[h];
            for (int t = 0; t < f.num_qtiles; ++t) {
                touched.clear();
                for (int g = 0; g < 8; ++g) {
                    const int r0 = t * kTileQ + g * 16;
                    if (r0 >= seq_len) break;
                    const int qb = r0 / block_size;
                    for (int q = c.ptr[qb]; q < c.ptr[qb + 1]; ++q) {
                        const int k0 = c.idx[q] * block_size;
                        const int k1 = std::min(k0 + block_size, seq_len);
                        for (int k = k0; k < k1; k += 16) {
                            const int ch = k / kChunk;
                            if (!m[ch]) touched.push_back(ch);
                            m[ch] |= 1u << (g * 4 + (k % kChunk) / 16);
                        }
                    }
                }
                std::sort(touched.begin(), touched.end());
                auto& out = per[static_cast<std::size_t>(h) * f.num_qtiles + t];
                out.reserve(touched.size());
                for (int ch : touched) {
                    out.push_back({ch, m[ch]});
                    m[ch] = 0;
                }
            }
        }
    }
    f.offset.assign(per.size() + 1, 0);
    for (std::size_t i = 0; i < per.size(); ++i) f.offset[i + 1] = f.offset[i] + per[i].size();
    f.chunks.resize(f.offset.back());
    for (std::size_t i = 0; i < per.size(); ++i)
        std::copy(per[i].begin(), per[i].end(), f.chunks.begin() + f.offset[i]);
    return f;
}

PairList build_pair_list(const FwdList& fwd, int num_heads) {
    PairList pl;
    pl.num_pairs = (fwd.num_qtiles + 1) / 2;
    pl.offset.assign(static_cast<size_t>(num_heads) * pl.num_pairs + 1, 0);
    struct U {
        int32_t c;
        uint32_t a, b;
    };
    std::vector<U> uni;
    for (int h = 0; h < num_heads; ++h)
        for (int p = 0; p < pl.num_pairs; ++p) {
            uni.clear();
            const size_t wa = static_cast<size_t>(h) * fwd.num_qtiles + 2 * p;
            const bool has_b = 2 * p + 1 < fwd.num_qtiles;
            int64_t ia = fwd.offset[wa], ea = fwd.offset[wa + 1];
            int64_t ib = has_b ? fwd.offset[wa + 1] : 0, eb = has_b ? fwd.offset[wa + 2] : 0;
            while (ia < ea || ib < eb) {
                if (ib >= eb || (ia < ea && fwd.chunks[ia].chunk < fwd.chunks[ib].chunk)) {
                    uni.push_back({fwd.chunks[ia].chunk, fwd.chunks[ia].mask, 0u});
                    ++ia;
                } else if (ia >= ea || fwd.chunks[ib].chunk < fwd.chunks[ia].chunk) {
                    uni.push_back({fwd.chunks[ib].chunk, 0u, fwd.chunks[ib].mask});
                    ++ib;
                } else {
                    uni.push_back({fwd.chunks[ia].chunk, fwd.chunks[ia].mask, fwd.chunks[ib].mask});
                    ++ia;
                    ++ib;
                }
            }
            for (size_t i = 0; i < uni.size(); i += 2) {
                PairStep s{uni[i].c, -1, uni[i].a, 0u, uni[i].b, 0u};
                if (i + 1 < uni.size()) {
                    s.c1 = uni[i + 1].c;
                    s.a1 = uni[i + 1].a;
                    s.b1 = uni[i + 1].b;
                }
                pl.steps.push_back(s);
            }
            pl.offset[static_cast<size_t>(h) * pl.num_pairs + p + 1] = static_cast<int64_t>(pl.steps.size());
        }
    return pl;
}

BwdList build_bwd_list(const FwdList& fwd, int num_heads, int num_kv_heads, int seq_len) {
    BwdList b;
    const int hpg = num_heads / num_kv_heads;
    const int nchunks = (seq_len + kChunk - 1) / kChunk;
    struct QE {
        int32_t t;
        uint32_t m;
    };
    std::vector<std::vector<QE>> lists(nchunks);
    for (int g = 0; g < num_kv_heads; ++g) {
        const int h = g * hpg;
        for (auto& l : lists) l.clear();
        for (int t = 0; t < fwd.num_qtiles; ++t) {
            const std::size_t w = static_cast<std::size_t>(h) * fwd.num_qtiles + t;
            for (int64_t e = fwd.offset[w]; e < fwd.offset[w + 1]; ++e)
                lists[fwd.chunks[e].chunk].push_back({t, fwd.chunks[e].mask});
        }
        std::vector<int> order;
        for (int c = 0; c < nchunks; ++c) {
            if (!lists[c].empty())
                order.push_back(c);
            else
                b.uncovered = true;  // no tile will write this chunk's dK / dV
        }
        std::sort(order.begin(), order.end(), [&](int a, int c) {
            if (lists[a].size() != lists[c].size()) return lists[a].size() > lists[c].size();
            if (lists[a][0].t != lists[c][0].t) return lists[a][0].t < lists[c][0].t;
            return a < c;
        });
        for (std::size_t i = 0; i < order.size(); i += 2) {
            const int c0 = order[i];
            const int c1 = i + 1 < order.size() ? order[i + 1] : -1;
            BwdTile tile{g, c0, c1, static_cast<int64_t>(b.entries.size()), 0};
            const auto& L0 = lists[c0];
            static const std::vector<QE> kEmpty;
            const auto& L1 = c1 >= 0 ? lists[c1] : kEmpty;
            std::size_t a = 0, z = 0;
            while (a < L0.size() || z < L1.size()) {
                BwdEntry e{0, 0u, 0u};
                if (z >= L1.size() || (a < L0.size() && L0[a].t < L1[z].t)) {
                    e = {L0[a].t, L0[a].m, 0u};
                    ++a;
                } else if (a >= L0.size() || L1[z].t < L0[a].t) {
                    e = {L1[z].t, 0u, L1[z].m};
                    ++z;
                } else {
                    e = {L0[a].t, L0[a].m, L1[z].m};
                    ++a;
                    ++z;
                }
                b.entries.push_back(e);
            }
            tile.count = static_cast<int32_t>(b.entries.size() - tile.offset);
            b.tiles.push_back(tile);
        }
    }
    return b;
}

void partition_lpt(int num_units, const int64_t* weights, int num_ranks, int* owner,
                   int64_t* load) {
    std::vector<int> order(num_units);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return weights[a] > weights[b]; });
    std::vector<int64_t> l(num_ranks, 0);
    for (int u : order) {
        int best = 0;
        for (int r = 1; r < num_ranks; ++r)
            if (l[r] < l[best]) best = r;
        owner[u] = best;
        l[best] += weights[u];
    }
    if (load)
        for (int r = 0; r < num_ranks; ++r) load[r] = l[r];
}

}  // namespace s2
