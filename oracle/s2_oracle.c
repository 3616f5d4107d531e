/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement of the reference S2-Attention algorithm
 * (/root/reference/proj, `shardattn`).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * Each function cites the reference file:line it restates.  The
 * restatement is pinned to the reference itself (oracle/_ref, built from the
 * reference sources by oracle/Makefile) by tests/test_oracle.py, and to the
 * committed golden fixtures in tests/golden/ (made by
 * oracle/make_golden.py), so it can travel to the GPU box where
 * /root/reference does not exist.
 *
 * Forward: fp32 storage, fp64 accumulation, the same operation order as
 * process_query_block (attention.cpp:26-98), so it is bit-identical to the
 * reference's streaming kernel (tested).
 * Backward / decode: the reference has none; these restate the
 * gradient / single-row forms of the same definition (reference.cpp:28-50,
 * p_ij = exp(scale*q_i.k_j - lse_i) over admitted j <= i) in fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/s2attn.h"

/* ---------------------------------------------------------------- pattern */

/* PatternConfig::num_blocks, pattern.cpp:12-14 */
int s2o_num_blocks(const s2_pattern_config* c) {
    return (int)(((long long)c->seq_len + c->block_size - 1) / c->block_size);
}

static int kv_heads(const s2_pattern_config* c) {
    return c->num_kv_heads > 0 ? c->num_kv_heads : c->num_heads;
}
static int group_of(const s2_pattern_config* c, int h) {
    return h / (c->num_heads / kv_heads(c));
}

/* PatternConfig::offset_for, pattern.cpp:16-34 */
int s2o_offset_for(const s2_pattern_config* c, int s, int head) {
    const s2_stride_segment* seg = &c->segments[s];
    int raw;
    if (seg->num_offsets > 0) {
        raw = seg->num_offsets == c->num_heads ? seg->offsets[head] : seg->offsets[group_of(c, head)];
    } else {
        raw = group_of(c, head); /* OffsetScheme::HeadModStride */
    }
    return raw % seg->stride;
}

/* PatternConfig::validate, pattern.cpp:36-79.  Returns 0 or 1 (+message). */
int s2o_validate(const s2_pattern_config* c, char* msg, int msglen) {
#define FAIL(m)                                   \
    do {                                          \
        if (msg) snprintf(msg, (size_t)msglen, "%s", m); \
        return 1;                                 \
    } while (0)
    if (c->seq_len < 1) FAIL("seq_len must be positive");
    if (c->block_size < 1) FAIL("block_size must be positive");
    if (c->num_heads < 1) FAIL("num_heads must be positive");
    if (c->num_kv_heads < 0) FAIL("num_kv_heads must be positive");
    if (c->num_heads % kv_heads(c) != 0) FAIL("num_kv_heads must divide num_heads");
    if (c->local_blocks < 1) FAIL("local_blocks must be >= 1");
    if (c->local_stride < 1) FAIL("local_stride must be >= 1");
    if (c->num_segments < 0 || c->num_segments > S2_MAX_SEGMENTS) FAIL("too many segments");
    const int blocks = s2o_num_blocks(c);
    int prev_end = c->local_blocks;
    for (int s = 0; s < c->num_segments; ++s) {
        const s2_stride_segment* seg = &c->segments[s];
        if (seg->stride < 1) FAIL("segment stride must be >= 1");
        if (seg->start_block_distance < c->local_blocks) FAIL("segment start must be >= local_blocks");
        if (seg->end_block_distance > blocks) FAIL("segment end must be <= num_blocks");
        if (seg->start_block_distance >= seg->end_block_distance) FAIL("segment range must be non-empty");
        if (seg->start_block_distance < prev_end && s > 0)
            FAIL("segments must be ordered and non-overlapping");
        prev_end = seg->end_block_distance;
        if (seg->num_offsets > 0) {
            if (seg->num_offsets != c->num_heads && seg->num_offsets != kv_heads(c))
                FAIL("segment offsets must list one entry per head or per kv head");
            for (int i = 0; i < seg->num_offsets; ++i)
                if (seg->offsets[i] < 0) FAIL("offsets must be non-negative");
            if (seg->num_offsets == c->num_heads) {
                const int hpg = c->num_heads / kv_heads(c);
                for (int h = 0; h < c->num_heads; ++h) {
                    const int lead = group_of(c, h) * hpg;
                    if (seg->offsets[h] % seg->stride != seg->offsets[lead] % seg->stride)
                        FAIL("offsets must agree within each kv group");
                }
            }
        }
    }
    return 0;
#undef FAIL
}

/* One bit of build_head_mask, pattern.cpp:138-155 (the formula_bit of
 * test_pattern.cpp:17-29). */
int s2o_mask_bit(const s2_pattern_config* c, int head, int i, int j) {
    if (j > i) return 0;
    if (j == i) return 1; /* diagonal forced, pattern.cpp:155 */
    const int dist = i - j;
    if (dist < c->local_blocks && dist % c->local_stride == 0) return 1;
    for (int s = 0; s < c->num_segments; ++s) {
        const s2_stride_segment* seg = &c->segments[s];
        if (dist < seg->start_block_distance || dist >= seg->end_block_distance) continue;
        const int r = j - s2o_offset_for(c, s, head);
        return r >= 0 && r % seg->stride == 0; /* segments disjoint: first decides */
    }
    return 0;
}

/* to_csr(build_head_mask(cfg, head)): csr.cpp:35-47 scans j <= i per row.
 * row_ptr == NULL only counts.  Returns nnz. */
int64_t s2o_build_csr(const s2_pattern_config* c, int head, int* row_ptr, int* col_idx) {
    const int B = s2o_num_blocks(c);
    int64_t n = 0;
    if (row_ptr) row_ptr[0] = 0;
    for (int i = 0; i < B; ++i) {
        for (int j = 0; j <= i; ++j)
            if (s2o_mask_bit(c, head, i, j)) {
                if (col_idx) col_idx[n] = j;
                ++n;
            }
        if (row_ptr) row_ptr[i + 1] = (int)n;
    }
    return n;
}

/* Column form of the same bits (no reference symbol). */
void s2o_csc_from_csr(int B, const int* row_ptr, const int* col_idx, int* col_ptr, int* row_idx) {
    memset(col_ptr, 0, sizeof(int) * (size_t)(B + 1));
    for (int p = 0; p < row_ptr[B]; ++p) col_ptr[col_idx[p] + 1]++;
    for (int j = 0; j < B; ++j) col_ptr[j + 1] += col_ptr[j];
    int* fill = (int*)malloc(sizeof(int) * (size_t)B);
    memcpy(fill, col_ptr, sizeof(int) * (size_t)B);
    for (int i = 0; i < B; ++i)
        for (int p = row_ptr[i]; p < row_ptr[i + 1]; ++p) row_idx[fill[col_idx[p]]++] = i;
    free(fill);
}

/* HeadCacheSchedule::evict_after, analysis.cpp:76-82. */
void s2o_evict_after(const s2_pattern_config* c, int head, int* ev) {
    const int B = s2o_num_blocks(c);
    for (int j = 0; j < B; ++j) {
        int last = j;
        for (int i = j; i < B; ++i)
            if (s2o_mask_bit(c, head, i, j)) last = i;
        ev[j] = last;
    }
}

/* check_kv_cache_efficiency, verify.cpp:53-72. */
int s2o_kv_efficient(const s2_pattern_config* c, int head) {
    const int B = s2o_num_blocks(c);
    for (int j = 0; j < B; ++j) {
        int gap = 0;
        for (int i = j; i < B; ++i) {
            if (!s2o_mask_bit(c, head, i, j)) gap = 1;
            else if (gap) return 0;
        }
    }
    return 1;
}

/* ------------------------------------------------------------------ RNG */
/* AttentionTensors::random (attention.cpp:135-144): std::mt19937_64(seed),
 * std::uniform_real_distribution<float>(-1, 1), filling q then k then v.
 * mt19937_64 is fully specified by the C++ standard; the float mapping is
 * libstdc++'s generate_canonical<float, 24> (one 64-bit draw / 2^64, clamped
 * below 1) followed by a + (b - a) * u. */
typedef struct {
    uint64_t mt[312];
    int idx;
} s2o_mt64;

static void mt64_seed(s2o_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(s2o_mt64* s) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            s->mt[i] = s->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

static float mt64_uniform_m1_1(s2o_mt64* s) {
    const float sum = (float)mt64_next(s);
    float u = sum / 18446744073709551616.0f;
    if (u >= 1.0f) u = nextafterf(1.0f, 0.0f);
    return u * 2.0f + -1.0f;
}

void s2o_random_tensors(int H, int N, int d, uint64_t seed, float* q, float* k, float* v) {
    s2o_mt64 st;
    mt64_seed(&st, seed);
    const size_t n = (size_t)H * N * d;
    for (size_t i = 0; i < n; ++i) q[i] = mt64_uniform_m1_1(&st);
    for (size_t i = 0; i < n; ++i) k[i] = mt64_uniform_m1_1(&st);
    for (size_t i = 0; i < n; ++i) v[i] = mt64_uniform_m1_1(&st);
}

/* ------------------------------------------------------------- forward */

static void head_offsets(int H, int B, const int* row_ptr, int64_t* col_off) {
    int64_t off = 0;
    for (int h = 0; h < H; ++h) {
        col_off[h] = off;
        off += row_ptr[(size_t)h * (B + 1) + B];
    }
}

/* process_query_block (attention.cpp:26-98) for one (batch*head, q-block)
 * task, num_splits == 1, identical operation order; batch and GQA folded in
 * by index arithmetic. */
static void fwd_task(int N, int D, int S, double scale, const float* q, const float* k,
                     const float* v, const int* rp, const int* ci, int qb, float* out,
                     double* lse, double* m, double* l, double* acc, double* p) {
    const int q_begin = qb * S;
    const int q_end = q_begin + S < N ? q_begin + S : N;
    const int rows = q_end - q_begin;
    for (int r = 0; r < rows; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.0;
    }
    memset(acc, 0, sizeof(double) * (size_t)rows * D);
    for (int ptr = rp[qb]; ptr < rp[qb + 1]; ++ptr) {
        const int kb = ci[ptr];
        const int k_begin = kb * S;
        const int k_end = k_begin + S < N ? k_begin + S : N;
        for (int r = 0; r < rows; ++r) {
            const int i = q_begin + r;
            const int c_end = k_end < i + 1 ? k_end : i + 1;
            const int cols = c_end - k_begin;
            if (cols <= 0) continue;
            const float* q_row = q + (size_t)i * D;
            for (int c = 0; c < cols; ++c) {
                const float* k_row = k + (size_t)(k_begin + c) * D;
                double dot = 0.0; /* dot_full, kernel_common.hpp:48-52 */
                for (int x = 0; x < D; ++x) dot += (double)q_row[x] * k_row[x];
                p[c] = 0.0 + dot;
            }
            double block_max = -INFINITY;
            for (int c = 0; c < cols; ++c) {
                p[c] *= scale;
                if (p[c] > block_max) block_max = p[c];
            }
            const double m_new = m[r] > block_max ? m[r] : block_max;
            const double alpha = exp(m[r] - m_new);
            double block_sum = 0.0;
            for (int c = 0; c < cols; ++c) {
                p[c] = exp(p[c] - m_new);
                block_sum += p[c];
            }
            l[r] = alpha * l[r] + block_sum;
            double* a = acc + (size_t)r * D;
            for (int x = 0; x < D; ++x) a[x] *= alpha;
            for (int c = 0; c < cols; ++c) {
                const float* v_row = v + (size_t)(k_begin + c) * D;
                const double w = p[c];
                for (int x = 0; x < D; ++x) a[x] += w * v_row[x];
            }
            m[r] = m_new;
        }
    }
    for (int r = 0; r < rows; ++r) {
        const int i = q_begin + r;
        const double inv = 1.0 / l[r];
        const double* a = acc + (size_t)r * D;
        float* o = out + (size_t)i * D;
        for (int x = 0; x < D; ++x) o[x] = (float)(a[x] * inv);
        lse[i] = m[r] + log(l[r]);
    }
}

/* streaming_sharded_attention (attention.cpp:100-118,190-193) over
 * q/out [batch,H,N,D], k/v [batch,Hkv,N,D]; row_ptr H*(B+1) and the
 * concatenated col_idx of every head.  OpenMP over (unit, q-block) exactly
 * like run_streaming. */
void s2o_attn_fwd(int batch, int H, int Hkv, int N, int D, int S, double scale, const float* q,
                  const float* k, const float* v, const int* row_ptr, const int* col_idx,
                  float* out, double* lse) {
    const int B = (N + S - 1) / S;
    const int hpg = H / Hkv;
    int64_t* col_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)H);
    head_offsets(H, B, row_ptr, col_off);
    const int units = batch * H;
#pragma omp parallel
    {
        double* m = (double*)malloc(sizeof(double) * (size_t)S);
        double* l = (double*)malloc(sizeof(double) * (size_t)S);
        double* acc = (double*)malloc(sizeof(double) * (size_t)S * D);
        double* p = (double*)malloc(sizeof(double) * (size_t)S);
#pragma omp for collapse(2) schedule(dynamic)
        for (int u = 0; u < units; ++u)
            for (int qb = 0; qb < B; ++qb) {
                const int b = u / H, h = u % H;
                const size_t qo = (size_t)u * N * D;
                const size_t ko = ((size_t)b * Hkv + h / hpg) * N * D;
                fwd_task(N, D, S, scale, q + qo, k + ko, v + ko, row_ptr + (size_t)h * (B + 1),
                         col_idx + col_off[h], qb, out + qo, lse + (size_t)u * N, m, l, acc, p);
            }
        free(m);
        free(l);
        free(acc);
        free(p);
    }
    free(col_off);
}

/* ------------------------------------------------------------ backward */

/* Gradient of out = softmax_masked(scale*Q K^T) V with the admitted set of
 * reference.cpp:28-36 (block mask of row block + token causality).  fp64.
 * Recomputes the forward (m, z two-pass as reference.cpp:28-45) per row.
 * Parallel over (batch, kv-group) units so dK/dV accumulation is race-free;
 * the order inside a unit is fixed (deterministic). */
void s2o_attn_bwd(int batch, int H, int Hkv, int N, int D, int S, double scale, const float* q,
                  const float* k, const float* v, const float* dout, const int* row_ptr,
                  const int* col_idx, float* dq, float* dk, float* dv) {
    const int B = (N + S - 1) / S;
    const int hpg = H / Hkv;
    int64_t* col_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)H);
    head_offsets(H, B, row_ptr, col_off);
    const int units = batch * Hkv;
#pragma omp parallel
    {
        double* sc = (double*)malloc(sizeof(double) * (size_t)N);
        double* o = (double*)malloc(sizeof(double) * (size_t)D);
        double* gq = (double*)malloc(sizeof(double) * (size_t)D);
        double* gk = (double*)malloc(sizeof(double) * (size_t)N * D);
        double* gv = (double*)malloc(sizeof(double) * (size_t)N * D);
#pragma omp for schedule(dynamic)
        for (int u = 0; u < units; ++u) {
            const int b = u / Hkv, g = u % Hkv;
            const float* K = k + (size_t)u * N * D;
            const float* V = v + (size_t)u * N * D;
            memset(gk, 0, sizeof(double) * (size_t)N * D);
            memset(gv, 0, sizeof(double) * (size_t)N * D);
            for (int hh = 0; hh < hpg; ++hh) {
                const int h = g * hpg + hh;
                const size_t qo = ((size_t)b * H + h) * N * D;
                const int* rp = row_ptr + (size_t)h * (B + 1);
                const int* ci = col_idx + col_off[h];
                for (int i = 0; i < N; ++i) {
                    const int bi = i / S;
                    const float* qi = q + qo + (size_t)i * D;
                    const float* doi = dout + qo + (size_t)i * D;
                    double mx = -INFINITY;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            double dot = 0.0;
                            for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
                            sc[j] = scale * dot;
                            if (sc[j] > mx) mx = sc[j];
                        }
                    }
                    double z = 0.0;
                    for (int x = 0; x < D; ++x) o[x] = 0.0;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            sc[j] = exp(sc[j] - mx);
                            z += sc[j];
                            for (int x = 0; x < D; ++x) o[x] += sc[j] * V[(size_t)j * D + x];
                        }
                    }
                    double delta = 0.0;
                    for (int x = 0; x < D; ++x) {
                        o[x] /= z;
                        delta += (double)doi[x] * o[x];
                    }
                    for (int x = 0; x < D; ++x) gq[x] = 0.0;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            const double pij = sc[j] / z;
                            double dp = 0.0;
                            for (int x = 0; x < D; ++x) dp += (double)doi[x] * V[(size_t)j * D + x];
                            const double ds = pij * (dp - delta);
                            for (int x = 0; x < D; ++x) {
                                gq[x] += ds * K[(size_t)j * D + x];
                                gk[(size_t)j * D + x] += ds * qi[x];
                                gv[(size_t)j * D + x] += pij * doi[x];
                            }
                        }
                    }
                    for (int x = 0; x < D; ++x) dq[qo + (size_t)i * D + x] = (float)(scale * gq[x]);
                }
            }
            for (size_t e = 0; e < (size_t)N * D; ++e) {
                dk[(size_t)u * N * D + e] = (float)(scale * gk[e]);
                dv[(size_t)u * N * D + e] = (float)gv[e];
            }
        }
        free(sc);
        free(o);
        free(gq);
        free(gk);
        free(gv);
    }
    free(col_off);
}

/* s2o_attn_bwd, parallel inside a (batch, kv-group) unit: bit-identical results,
 * for the CPU baseline legs of bench.py (one unit is a single thread's work in
 * s2o_attn_bwd).  Pass 1, parallel over query rows: each row's max, sum, delta
 * and dQ, computed exactly as s2o_attn_bwd does.  Pass 2, parallel over key
 * blocks: dK / dV of each key summed over (query head of the group, attending
 * row) in ascending order -- s2o_attn_bwd's accumulation order -- with p and dp
 * recomputed from the same expressions.  Test infrastructure only. */
void s2o_attn_bwd_par(int batch, int H, int Hkv, int N, int D, int S, double scale, const float* q,
                      const float* k, const float* v, const float* dout, const int* row_ptr,
                      const int* col_idx, float* dq, float* dk, float* dv) {
    const int B = (N + S - 1) / S;
    const int hpg = H / Hkv;
    int64_t* col_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)H);
    head_offsets(H, B, row_ptr, col_off);
    double* mrow = (double*)malloc(sizeof(double) * (size_t)N * hpg);
    double* zrow = (double*)malloc(sizeof(double) * (size_t)N * hpg);
    double* drow = (double*)malloc(sizeof(double) * (size_t)N * hpg);
    /* per head of a group: for each key block, the row blocks listing it (ascending) */
    int* cptr = (int*)malloc(sizeof(int) * (size_t)(B + 1) * hpg);
    int* crow = NULL;
    for (int u = 0; u < batch * Hkv; ++u) {
        const int b = u / Hkv, g = u % Hkv;
        const float* K = k + (size_t)u * N * D;
        const float* V = v + (size_t)u * N * D;
        int64_t nnz_g = 0;
        for (int hh = 0; hh < hpg; ++hh) {
            const int* rp = row_ptr + (size_t)(g * hpg + hh) * (B + 1);
            nnz_g += rp[B];
        }
        crow = (int*)realloc(crow, sizeof(int) * (size_t)(nnz_g > 0 ? nnz_g : 1));
        int64_t base = 0;
        for (int hh = 0; hh < hpg; ++hh) {
            const int h = g * hpg + hh;
            const int* rp = row_ptr + (size_t)h * (B + 1);
            const int* ci = col_idx + col_off[h];
            int* cp = cptr + (size_t)hh * (B + 1);
            for (int c = 0; c <= B; ++c) cp[c] = 0;
            for (int e = 0; e < rp[B]; ++e) cp[ci[e] + 1]++;
            for (int c = 0; c < B; ++c) cp[c + 1] += cp[c];
            int* fill = (int*)malloc(sizeof(int) * (size_t)B);
            for (int c = 0; c < B; ++c) fill[c] = cp[c];
            for (int bi = 0; bi < B; ++bi)  /* ascending rows per column */
                for (int e = rp[bi]; e < rp[bi + 1]; ++e) crow[base + fill[ci[e]]++] = bi;
            free(fill);
            for (int c = 0; c <= B; ++c) cp[c] += (int)base;
            base += rp[B];
        }
        /* pass 1: rows */
        for (int hh = 0; hh < hpg; ++hh) {
            const int h = g * hpg + hh;
            const size_t qo = ((size_t)b * H + h) * N * D;
            const int* rp = row_ptr + (size_t)h * (B + 1);
            const int* ci = col_idx + col_off[h];
#pragma omp parallel
            {
                double* sc = (double*)malloc(sizeof(double) * (size_t)N);
                double* o = (double*)malloc(sizeof(double) * (size_t)D);
                double* gq = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
                for (int i = 0; i < N; ++i) {
                    const int bi = i / S;
                    const float* qi = q + qo + (size_t)i * D;
                    const float* doi = dout + qo + (size_t)i * D;
                    double mx = -INFINITY;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            double dot = 0.0;
                            for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
                            sc[j] = scale * dot;
                            if (sc[j] > mx) mx = sc[j];
                        }
                    }
                    double z = 0.0;
                    for (int x = 0; x < D; ++x) o[x] = 0.0;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            sc[j] = exp(sc[j] - mx);
                            z += sc[j];
                            for (int x = 0; x < D; ++x) o[x] += sc[j] * V[(size_t)j * D + x];
                        }
                    }
                    double delta = 0.0;
                    for (int x = 0; x < D; ++x) {
                        o[x] /= z;
                        delta += (double)doi[x] * o[x];
                    }
                    for (int x = 0; x < D; ++x) gq[x] = 0.0;
                    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr) {
                        const int j0 = ci[ptr] * S;
                        for (int j = j0; j < j0 + S && j <= i; ++j) {
                            const double pij = sc[j] / z;
                            double dp = 0.0;
                            for (int x = 0; x < D; ++x) dp += (double)doi[x] * V[(size_t)j * D + x];
                            const double ds = pij * (dp - delta);
                            for (int x = 0; x < D; ++x) gq[x] += ds * K[(size_t)j * D + x];
                        }
                    }
                    for (int x = 0; x < D; ++x) dq[qo + (size_t)i * D + x] = (float)(scale * gq[x]);
                    mrow[(size_t)hh * N + i] = mx;
                    zrow[(size_t)hh * N + i] = z;
                    drow[(size_t)hh * N + i] = delta;
                }
                free(sc);
                free(o);
                free(gq);
            }
        }
        /* pass 2: key blocks */
#pragma omp parallel
        {
            double* gk = (double*)malloc(sizeof(double) * (size_t)D);
            double* gv = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic)
            for (int cb = 0; cb < B; ++cb) {
                for (int j = cb * S; j < cb * S + S && j < N; ++j) {
                    for (int x = 0; x < D; ++x) gk[x] = gv[x] = 0.0;
                    for (int hh = 0; hh < hpg; ++hh) {
                        const int h = g * hpg + hh;
                        const size_t qo = ((size_t)b * H + h) * N * D;
                        const int* cp = cptr + (size_t)hh * (B + 1);
                        for (int e = cp[cb]; e < cp[cb + 1]; ++e) {
                            const int bi = crow[e];
                            for (int i = bi * S; i < bi * S + S && i < N; ++i) {
                                if (j > i) continue;
                                const float* qi = q + qo + (size_t)i * D;
                                const float* doi = dout + qo + (size_t)i * D;
                                double dot = 0.0;
                                for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
                                const double pij = exp(scale * dot - mrow[(size_t)hh * N + i]) / zrow[(size_t)hh * N + i];
                                double dp = 0.0;
                                for (int x = 0; x < D; ++x) dp += (double)doi[x] * V[(size_t)j * D + x];
                                const double ds = pij * (dp - drow[(size_t)hh * N + i]);
                                for (int x = 0; x < D; ++x) {
                                    gk[x] += ds * qi[x];
                                    gv[x] += pij * doi[x];
                                }
                            }
                        }
                    }
                    for (int x = 0; x < D; ++x) {
                        dk[(size_t)u * N * D + (size_t)j * D + x] = (float)(scale * gk[x]);
                        dv[(size_t)u * N * D + (size_t)j * D + x] = (float)gv[x];
                    }
                }
            }
            free(gk);
            free(gv);
        }
    }
    free(crow);
    free(cptr);
    free(mrow);
    free(zrow);
    free(drow);
    free(col_off);
}

/* ------------------------------------------------- sampled backward rows */

/* Row statistics of query row i (reference.cpp:28-45 two-pass): max m, sum z
 * of exp(scale*q_i.k_j - m) over the admitted keys, and delta = dO_i . O_i. */
static void row_stats(const float* qi, const float* doi, const float* K, const float* V,
                      const int* rp, const int* ci, int i, int S, int D, double scale,
                      double* m_out, double* z_out, double* delta_out) {
    const int bi = i / S;
    double mx = -INFINITY;
    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr)
        for (int j = ci[ptr] * S; j < ci[ptr] * S + S && j <= i; ++j) {
            double dot = 0.0;
            for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
            if (scale * dot > mx) mx = scale * dot;
        }
    double z = 0.0, dl = 0.0;
    for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr)
        for (int j = ci[ptr] * S; j < ci[ptr] * S + S && j <= i; ++j) {
            double dot = 0.0, dp = 0.0;
            for (int x = 0; x < D; ++x) {
                dot += (double)qi[x] * K[(size_t)j * D + x];
                dp += (double)doi[x] * V[(size_t)j * D + x];
            }
            const double w = exp(scale * dot - mx);
            z += w;
            dl += w * dp;  /* sum_j p_ij (dO_i . v_j) * z  ==  z * (dO_i . O_i) */
        }
    *m_out = mx;
    *z_out = z;
    *delta_out = dl / z;
}

/* Does row block bi list key block bj?  (CSR rows are strictly ascending) */
static int row_has_block(const int* rp, const int* ci, int bi, int bj) {
    int lo = rp[bi], hi = rp[bi + 1];
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (ci[mid] < bj) lo = mid + 1;
        else hi = mid;
    }
    return lo < rp[bi + 1] && ci[lo] == bj;
}

/* The gradient of s2o_attn_bwd at sampled rows, for full-size parity checks
 * (it is the same definition: p_ij = exp(scale q_i.k_j - m_i)/z_i over the
 * admitted set, dS_ij = p_ij (dO_i.v_j - delta_i)):
 *   qsel[2n] = (u = b*H + h, i)    -> dq_out[n*D]  = scale * sum_j dS_ij k_j
 *   ksel[2n] = (g = b*Hkv + kv, j) -> dk_out[n*D]  = scale * sum_{h in group, i} dS_ij q_i
 *                                     dv_out[n*D]  = sum_{h in group, i} p_ij dO_i
 * Key rows visit every admitted query row of the group's heads (rows whose
 * block row lists j's block, i >= j), in parallel over i. */
void s2o_bwd_sample(int batch, int H, int Hkv, int N, int D, int S, double scale, const float* q,
                    const float* k, const float* v, const float* dout, const int* row_ptr,
                    const int* col_idx, int nq, const int* qsel, float* dq_out, int nk,
                    const int* ksel, float* dk_out, float* dv_out) {
    const int B = (N + S - 1) / S;
    const int hpg = H / Hkv;
    (void)batch;  /* rows are addressed by their (batch, head) unit index */
    int64_t* col_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)H);
    head_offsets(H, B, row_ptr, col_off);
#pragma omp parallel for schedule(dynamic)
    for (int n = 0; n < nq; ++n) {
        const int u = qsel[2 * n], i = qsel[2 * n + 1];
        const int b = u / H, h = u % H, bi = i / S;
        const size_t qo = (size_t)u * N * D;
        const float* qi = q + qo + (size_t)i * D;
        const float* doi = dout + qo + (size_t)i * D;
        const float* K = k + ((size_t)b * Hkv + h / hpg) * (size_t)N * D;
        const float* V = v + ((size_t)b * Hkv + h / hpg) * (size_t)N * D;
        const int* rp = row_ptr + (size_t)h * (B + 1);
        const int* ci = col_idx + col_off[h];
        double mx, z, delta;
        row_stats(qi, doi, K, V, rp, ci, i, S, D, scale, &mx, &z, &delta);
        double* gq = (double*)calloc((size_t)D, sizeof(double));
        for (int ptr = rp[bi]; ptr < rp[bi + 1]; ++ptr)
            for (int j = ci[ptr] * S; j < ci[ptr] * S + S && j <= i; ++j) {
                double dot = 0.0, dp = 0.0;
                for (int x = 0; x < D; ++x) {
                    dot += (double)qi[x] * K[(size_t)j * D + x];
                    dp += (double)doi[x] * V[(size_t)j * D + x];
                }
                const double ds = exp(scale * dot - mx) / z * (dp - delta);
                for (int x = 0; x < D; ++x) gq[x] += ds * K[(size_t)j * D + x];
            }
        for (int x = 0; x < D; ++x) dq_out[(size_t)n * D + x] = (float)(scale * gq[x]);
        free(gq);
    }
    for (int n = 0; n < nk; ++n) {
        const int g = ksel[2 * n], j = ksel[2 * n + 1];
        const int b = g / Hkv, kv = g % Hkv, bj = j / S;
        const float* K = k + (size_t)g * N * D;
        const float* V = v + (size_t)g * N * D;
        double* gk = (double*)calloc((size_t)D, sizeof(double));
        double* gv = (double*)calloc((size_t)D, sizeof(double));
        for (int hh = 0; hh < hpg; ++hh) {
            const int h = kv * hpg + hh;
            const size_t qo = ((size_t)b * H + h) * N * D;
            const int* rp = row_ptr + (size_t)h * (B + 1);
            const int* ci = col_idx + col_off[h];
#pragma omp parallel
            {
                double* lk = (double*)calloc((size_t)D, sizeof(double));
                double* lv = (double*)calloc((size_t)D, sizeof(double));
#pragma omp for schedule(dynamic, 64)
                for (int i = j; i < N; ++i) {
                    if (!row_has_block(rp, ci, i / S, bj)) continue;
                    const float* qi = q + qo + (size_t)i * D;
                    const float* doi = dout + qo + (size_t)i * D;
                    double mx, z, delta;
                    row_stats(qi, doi, K, V, rp, ci, i, S, D, scale, &mx, &z, &delta);
                    double dot = 0.0, dp = 0.0;
                    for (int x = 0; x < D; ++x) {
                        dot += (double)qi[x] * K[(size_t)j * D + x];
                        dp += (double)doi[x] * V[(size_t)j * D + x];
                    }
                    const double pij = exp(scale * dot - mx) / z;
                    const double ds = pij * (dp - delta);
                    for (int x = 0; x < D; ++x) {
                        lk[x] += ds * qi[x];
                        lv[x] += pij * doi[x];
                    }
                }
#pragma omp critical
                for (int x = 0; x < D; ++x) {
                    gk[x] += lk[x];
                    gv[x] += lv[x];
                }
                free(lk);
                free(lv);
            }
        }
        for (int x = 0; x < D; ++x) {
            dk_out[(size_t)n * D + x] = (float)(scale * gk[x]);
            dv_out[(size_t)n * D + x] = (float)gv[x];
        }
        free(gk);
        free(gv);
    }
    free(col_off);
}

/* -------------------------------------------------------------- decode */

/* Single query row at position t for every (batch, head): the row form of
 * naive_masked_attention (reference.cpp:28-50): admitted keys are j <= t in
 * the blocks of mask row bt = t / S.  k/v are dense [batch, Hkv, T, D] with
 * T > t; q/out [batch, H, D]; lse [batch, H].  fp64 two-pass. */
void s2o_decode(int batch, int H, int Hkv, int T, int D, int S, int t, double scale,
                const float* q, const float* k, const float* v, const int* row_ptr,
                const int* col_idx, int B, float* out, double* lse) {
    const int hpg = H / Hkv;
    int64_t* col_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)H);
    head_offsets(H, B, row_ptr, col_off);
    const int bt = t / S;
#pragma omp parallel for schedule(dynamic)
    for (int u = 0; u < batch * H; ++u) {
        const int b = u / H, h = u % H;
        const float* qi = q + (size_t)u * D;
        const float* K = k + ((size_t)b * Hkv + h / hpg) * (size_t)T * D;
        const float* V = v + ((size_t)b * Hkv + h / hpg) * (size_t)T * D;
        const int* rp = row_ptr + (size_t)h * (B + 1);
        const int* ci = col_idx + col_off[h];
        double mx = -INFINITY;
        for (int ptr = rp[bt]; ptr < rp[bt + 1]; ++ptr)
            for (int j = ci[ptr] * S; j < ci[ptr] * S + S && j <= t; ++j) {
                double dot = 0.0;
                for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
                if (scale * dot > mx) mx = scale * dot;
            }
        double z = 0.0;
        double* acc = (double*)calloc((size_t)D, sizeof(double));
        for (int ptr = rp[bt]; ptr < rp[bt + 1]; ++ptr)
            for (int j = ci[ptr] * S; j < ci[ptr] * S + S && j <= t; ++j) {
                double dot = 0.0;
                for (int x = 0; x < D; ++x) dot += (double)qi[x] * K[(size_t)j * D + x];
                const double w = exp(scale * dot - mx);
                z += w;
                for (int x = 0; x < D; ++x) acc[x] += w * V[(size_t)j * D + x];
            }
        for (int x = 0; x < D; ++x) out[(size_t)u * D + x] = (float)(acc[x] / z);
        if (lse) lse[u] = mx + log(z);
        free(acc);
    }
    free(col_off);
}

/* ------------------------------------------------------------- metrics */

/* max_relative_error, selftest.cpp:19-30: max |a-b| / max(|a|,|b|), 0/0 skipped. */
double s2o_max_rel_f(const float* a, const float* b, int64_t n) {
    double worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double x = a[i], y = b[i];
        const double s = fabs(x) > fabs(y) ? fabs(x) : fabs(y);
        if (s == 0.0) continue;
        const double e = fabs(x - y) / s;
        if (e > worst) worst = e;
    }
    return worst;
}

double s2o_max_rel_d(const double* a, const double* b, int64_t n) {
    double worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double s = fabs(a[i]) > fabs(b[i]) ? fabs(a[i]) : fabs(b[i]);
        if (s == 0.0) continue;
        const double e = fabs(a[i] - b[i]) / s;
        if (e > worst) worst = e;
    }
    return worst;
}

/* FNV-1a 64 over 32-bit words (test infrastructure: fingerprint of a CSR array,
 * the same fold as oracle/make_golden.py::fnv_fast; C so 128K layouts of every
 * head are fingerprinted in milliseconds). */
uint64_t s2o_fnv1a64_u32(const uint32_t* a, int64_t n) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (int64_t i = 0; i < n; ++i) h = (h ^ (uint64_t)a[i]) * 0x100000001B3ull;
    return h;
}
