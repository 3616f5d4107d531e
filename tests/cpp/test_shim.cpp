// C++ drop-in check: the reference's own API (shardattn::, include/shardattn_b200)
// backed by the B200 kernels, exercised the way /root/reference/proj/tests use it.
// Restates test_attention.cpp:72-294 and test_csr.cpp:30-42; the comparison
// oracle is the C restatement (oracle/s2_oracle.c, linked here as test infra).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "shardattn/attention.hpp"
#include "shardattn/csr.hpp"
#include "shardattn/pattern.hpp"

extern "C" void s2o_attn_fwd(int, int, int, int, int, int, double, const float*, const float*,
                             const float*, const int*, const int*, float*, double*);
extern "C" void s2o_attn_bwd(int, int, int, int, int, int, double, const float*, const float*,
                             const float*, const float*, const int*, const int*, float*, float*,
                             float*);

using namespace shardattn;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                               \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(c)) {                                                            \
            ++g_fail;                                                          \
            std::fprintf(stderr, "FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);  \
        }                                                                      \
    } while (0)
#define CHECK_THROWS(stmt)                                    \
    do {                                                      \
        bool thrown = false;                                  \
        try {                                                 \
            stmt;                                             \
        } catch (const std::invalid_argument&) {              \
            thrown = true;                                    \
        }                                                     \
        CHECK(thrown);                                        \
    } while (0)

struct Inst {
    PatternConfig cfg;
    std::vector<HeadBlockMask> masks;
    std::vector<CsrMask> csr;
    AttentionTensors t;
};

static Inst make(int heads, int n, int d, int s, int stride, std::uint64_t seed, int local = 1) {
    Inst i;
    i.cfg = make_single_stride_config(n, s, heads, local, stride);
    i.masks = build_all_masks(i.cfg);
    i.csr = to_csr(i.masks);
    i.t = AttentionTensors::random(heads, n, d, seed);
    return i;
}

static void oracle_fwd(const Inst& in, std::vector<float>& out, std::vector<double>& lse) {
    std::vector<int> rp, ci;
    for (const CsrMask& c : in.csr) {
        rp.insert(rp.end(), c.row_ptr.begin(), c.row_ptr.end());
        ci.insert(ci.end(), c.col_idx.begin(), c.col_idx.end());
    }
    const AttentionTensors& t = in.t;
    out.assign(t.q.size(), 0.f);
    lse.assign(static_cast<size_t>(t.num_heads) * t.seq_len, 0.0);
    s2o_attn_fwd(1, t.num_heads, t.num_heads, t.seq_len, t.head_dim, in.cfg.block_size, t.scale,
                 t.q.data(), t.k.data(), t.v.data(), rp.data(), ci.data(), out.data(), lse.data());
}

template <class T>
static bool close(const std::vector<T>& a, const std::vector<T>& b, double tol) {
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (std::fabs(double(a[i]) - double(b[i])) > tol + tol * std::fabs(double(b[i]))) return false;
    return true;
}

int main() {
    // golden compressed form (test_csr.cpp:30-42)
    {
        const CsrMask c = to_csr(build_head_mask(make_single_stride_config(8, 1, 4, 2, 3), 1));
        CHECK((c.row_ptr == std::vector<int>{0, 1, 3, 5, 8, 11, 14, 18, 22}));
        CHECK((c.col_idx == std::vector<int>{0, 0, 1, 1, 2, 1, 2, 3, 1, 3, 4, 1, 4, 5, 1, 4, 5, 6, 1,
                                             4, 6, 7}));
    }
    // a single token attends only itself (test_attention.cpp:72-79)
    {
        Inst in = make(2, 1, 8, 4, 1, 3);
        dense_masked_attention(in.t, in.masks, 4);
        for (size_t i = 0; i < in.t.v.size(); ++i) CHECK(in.t.out[i] == in.t.v[i]);
    }
    // zero values -> zero output, finite lse (:81-87)
    {
        Inst in = make(2, 32, 8, 8, 2, 5);
        std::fill(in.t.v.begin(), in.t.v.end(), 0.0f);
        streaming_sharded_attention(in.t, in.csr, 8);
        for (float x : in.t.out) CHECK(x == 0.0f);
        for (double l : in.t.lse) CHECK(std::isfinite(l));
    }
    // randomized strided instances vs the oracle (:98-122), fp32 tolerance 1e-4
    {
        std::mt19937 rng(31);
        for (int trial = 0; trial < 12; ++trial) {
            const int heads = 1 + rng() % 4, n = 8 + rng() % 120, d = rng() % 2 ? 16 : 8;
            const int s = 1 << (2 + rng() % 3), stride = 1 + rng() % 4;
            Inst in = make(heads, n, d, s, stride, 1000 + trial);
            std::vector<float> ro;
            std::vector<double> rl;
            oracle_fwd(in, ro, rl);
            AttentionTensors a = in.t;
            streaming_sharded_attention(a, in.csr, s);
            CHECK(close(a.out, ro, 1e-4));
            CHECK(close(a.lse, rl, 1e-4));
            AttentionTensors b = in.t;
            dsplit_attention(b, in.csr, s, 2);
            CHECK(close(b.out, ro, 1e-4));
        }
    }
    // dsplit(1) == streaming bit for bit (:124-132)
    {
        Inst in = make(3, 96, 16, 16, 3, 17);
        AttentionTensors a = in.t, b = in.t;
        streaming_sharded_attention(a, in.csr, 16);
        dsplit_attention(b, in.csr, 16, 1);
        CHECK(a.out == b.out);
        CHECK(a.lse == b.lse);
    }
    // unattended value rows change nothing, exactly (:196-215)
    {
        std::mt19937 rng(43);
        for (int trial = 0; trial < 3; ++trial) {
            Inst in = make(2, 40, 8, 8, 3, 4000 + trial);
            AttentionTensors base = in.t;
            streaming_sharded_attention(base, in.csr, 8);
            const int h = rng() % 2, i = rng() % 40;
            AttentionTensors poked = in.t;
            for (int j = 0; j < 40; ++j) {
                if (j <= i && in.masks[h].at(i / 8, j / 8)) continue;
                for (int x = 0; x < 8; ++x) poked.v[poked.idx(h, j, x)] += 1000.0f;
            }
            streaming_sharded_attention(poked, in.csr, 8);
            for (int x = 0; x < 8; ++x) CHECK(poked.out[poked.idx(h, i, x)] == base.out[base.idx(h, i, x)]);
        }
    }
    // permuting heads permutes outputs exactly (:217-240)
    {
        Inst in = make(4, 32, 8, 8, 4, 47);
        AttentionTensors base = in.t;
        streaming_sharded_attention(base, in.csr, 8);
        const int perm[4] = {2, 0, 3, 1};
        AttentionTensors sh = AttentionTensors::zeros(4, 32, 8);
        std::vector<CsrMask> csr(4);
        for (int h = 0; h < 4; ++h) {
            csr[h] = in.csr[perm[h]];
            for (int i = 0; i < 32; ++i)
                for (int x = 0; x < 8; ++x) {
                    sh.q[sh.idx(h, i, x)] = in.t.q[in.t.idx(perm[h], i, x)];
                    sh.k[sh.idx(h, i, x)] = in.t.k[in.t.idx(perm[h], i, x)];
                    sh.v[sh.idx(h, i, x)] = in.t.v[in.t.idx(perm[h], i, x)];
                }
        }
        streaming_sharded_attention(sh, csr, 8);
        for (int h = 0; h < 4; ++h)
            for (int i = 0; i < 32; ++i)
                for (int x = 0; x < 8; ++x)
                    CHECK(sh.out[sh.idx(h, i, x)] == base.out[base.idx(perm[h], i, x)]);
    }
    // error contract (:143-147, 259-282)
    {
        Inst in = make(2, 16, 6, 8, 1, 23);
        CHECK_THROWS(dsplit_attention(in.t, in.csr, 8, 4));
        CHECK_THROWS(dsplit_attention(in.t, in.csr, 8, 0));
        Inst j = make(2, 16, 8, 8, 1, 59);
        std::vector<HeadBlockMask> one(j.masks.begin(), j.masks.begin() + 1);
        CHECK_THROWS(dense_masked_attention(j.t, one, 8));
        CHECK_THROWS(streaming_sharded_attention(j.t, j.csr, 4));
        AttentionTensors bad = j.t;
        bad.k[3] = std::numeric_limits<float>::quiet_NaN();
        CHECK_THROWS(dense_masked_attention(bad, j.masks, 8));
        bad = j.t;
        bad.q.pop_back();
        CHECK_THROWS(streaming_sharded_attention(bad, j.csr, 8));
        PatternConfig cfg = make_single_stride_config(8, 1, 4, 2, 3);
        CHECK_THROWS(build_head_mask(cfg, 4));
        cfg.stride_segments[0].stride = 0;
        CHECK_THROWS(cfg.validate());
    }
    // ragged tails (:284-294)
    {
        Inst in = make(2, 45, 8, 8, 2, 61);
        std::vector<float> ro;
        std::vector<double> rl;
        oracle_fwd(in, ro, rl);
        AttentionTensors a = in.t;
        naive_masked_attention(a, in.masks, 8);
        CHECK(close(a.out, ro, 1e-4));
    }
    // extension: backward (fp32, like the forward) vs the fp64 oracle at 1e-4, at a
    // tensor-core shape and at an odd one (block 24, head_dim 40)
    for (const auto& [H, N, D, S] : {std::array<int, 4>{2, 300, 64, 64}, std::array<int, 4>{3, 250, 40, 24}}) {
        Inst in = make(H, N, D, S, 2, 7, 2);
        std::vector<float> dout(in.t.q.size());
        std::mt19937_64 g(5);
        std::uniform_real_distribution<float> u(-1.f, 1.f);
        for (float& x : dout) x = u(g);
        AttentionGrads gr;
        streaming_sharded_attention_backward(in.t, in.csr, S, dout, gr);
        std::vector<int> rp, ci;
        for (const CsrMask& c : in.csr) {
            rp.insert(rp.end(), c.row_ptr.begin(), c.row_ptr.end());
            ci.insert(ci.end(), c.col_idx.begin(), c.col_idx.end());
        }
        std::vector<float> dq(dout.size()), dk(dout.size()), dv(dout.size());
        s2o_attn_bwd(1, H, H, N, D, S, in.t.scale, in.t.q.data(), in.t.k.data(), in.t.v.data(),
                     dout.data(), rp.data(), ci.data(), dq.data(), dk.data(), dv.data());
        CHECK(close(gr.dq, dq, 1e-4));
        CHECK(close(gr.dk, dk, 1e-4));
        CHECK(close(gr.dv, dv, 1e-4));
    }
    {  // head_dim > 128 has no backward: the reference's exception type
        Inst in = make(1, 100, 160, 64, 1, 3, 2);
        AttentionGrads gr;
        CHECK_THROWS(streaming_sharded_attention_backward(in.t, in.csr, 64, std::vector<float>(in.t.q.size()), gr));
    }
    // extension: decode of one position over the compacted cache == that row of the
    // forward (bf16 operands: 2e-2), rows <= position only; other rows zero / -inf
    {
        Inst in = make(4, 1000, 128, 64, 3, 71, 2);
        std::vector<float> ro;
        std::vector<double> rl;
        oracle_fwd(in, ro, rl);
        for (int pos : {0, 63, 64, 500, 999}) {
            AttentionTensors a = in.t;
            sharded_decode(a, in.csr, 64, pos);
            bool ok = true;
            for (int h = 0; h < 4; ++h) {
                for (int x = 0; x < 128; ++x) {
                    const double got = a.out[a.idx(h, pos, x)], ref = ro[a.idx(h, pos, x)];
                    ok = ok && std::fabs(got - ref) <= 2e-2 + 2e-2 * std::fabs(ref);
                }
                ok = ok && std::fabs(a.lse[a.row_index(h, pos)] - rl[a.row_index(h, pos)]) <= 2e-2;
                const int other = pos == 0 ? 1 : 0;
                ok = ok && a.out[a.idx(h, other, 0)] == 0.0f && std::isinf(a.lse[a.row_index(h, other)]);
            }
            CHECK(ok);
        }
        CHECK_THROWS(sharded_decode(in.t, in.csr, 64, 1000));
        CHECK_THROWS(sharded_decode(in.t, in.csr, 64, -1));
    }
    // a literal zero scale (AttentionTensors' default member value, attention.hpp:23)
    // is applied as given: uniform weights over the admitted keys
    {
        Inst in = make(2, 200, 16, 8, 3, 83);
        in.t.scale = 0.0;
        std::vector<float> ro;
        std::vector<double> rl;
        oracle_fwd(in, ro, rl);
        AttentionTensors a = in.t;
        streaming_sharded_attention(a, in.csr, 8);
        CHECK(close(a.out, ro, 1e-4));
        CHECK(close(a.lse, rl, 1e-4));
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
