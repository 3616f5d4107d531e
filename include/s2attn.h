/*
 * s2attn.h — C ABI of the B200-native S2-Attention hot path.
 *
 * This is the drop-in boundary. The reference
 * (`shardattn`, /root/reference/proj) exposes a C++ API with std::vector and
 * exceptions and no FFI; every entry point below replaces one reference
 * symbol (cited per function) with a plain-C equivalent: POD structs, plain
 * pointers and sizes, int status codes, a thread-local error string, caller-
 * owned device buffers and an explicit CUDA stream.  The C++ shim in
 * include/shardattn_b200/ rebuilds the reference's exact `shardattn::`
 * signatures on top of this header.
 *
 * Tensor layouts (device memory, row-major, contiguous):
 *   q, out, dq, dout : [batch, num_heads,    seq_len, head_dim]
 *   k, v, dk, dv     : [batch, num_kv_heads, seq_len, head_dim]
 *   lse              : [batch, num_heads, seq_len] float32, natural log
 * The reference has no batch and no GQA in its tensors
 * (attention.hpp:17-37, idx=(h*N+t)*d+c); batch=1, num_kv_heads=num_heads
 * reproduces that layout exactly.
 */
#ifndef S2ATTN_H_
#define S2ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2_ABI_VERSION 1
#define S2_MAX_SEGMENTS 8

/* ---- status codes ------------------------------------------------------ */
/* The reference throws std::invalid_argument for every contract violation
 * (pattern.cpp:36-79, csr.cpp:11-33, kernel_common.hpp:20-41,
 * attention.cpp:102-110).  Those all map to S2_ERR_INVALID_ARGUMENT here;
 * the shim turns that code back into std::invalid_argument. */
enum {
    S2_OK = 0,
    S2_ERR_INVALID_ARGUMENT = 1,
    S2_ERR_CUDA = 2,
    S2_ERR_UNSUPPORTED = 3,
    S2_ERR_NO_DEVICE = 4,
    S2_ERR_OUT_OF_MEMORY = 5,
    /* load_config_file's std::runtime_error (serialize.cpp:123-146): the file
     * cannot be opened / parsed, or a field is missing or invalid; the
     * message names the file and the offending field. */
    S2_ERR_CONFIG = 6,
    /* a caller-provided output buffer is too small; the *len / count outputs
     * carry the size needed */
    S2_ERR_BUFFER_TOO_SMALL = 7
};

/* SMs the persistent backward kernels (dK/dV, dQ) leave free for concurrent
 * work: NCCL's all-gather of O on a communication stream overlaps the
 * backward, so their grid becomes (SM count - sms).  The forward, which has no
 * collective to overlap, keeps every SM.  Process-wide; 0 default. */
int s2_set_sm_reserve(int sms);

/* Message for the last non-zero status returned on this thread. */
const char* s2_last_error(void);
int s2_abi_version(void);

/* ---- element types ----------------------------------------------------- */
enum {
    S2_DTYPE_BF16 = 0, /* tcgen05 path: bf16 operands, fp32 accumulate in TMEM */
    S2_DTYPE_F32 = 1   /* reference-precision path: fp32 storage, fp32 FFMA   */
};

typedef struct CUstream_st* s2_stream_t; /* == cudaStream_t */

/* ---- layout policy ----------------------------------------------------- */
/* POD mirror of shardattn::StrideSegment / PatternConfig
 * (pattern.hpp:17-60).  offsets == NULL / num_offsets == 0 means the
 * HeadModStride scheme (o_h = group_of(h) mod stride, pattern.cpp:25-33). */
typedef struct s2_stride_segment {
    int start_block_distance;
    int end_block_distance;
    int stride;
    int num_offsets;    /* 0, num_heads or num_kv_heads */
    const int* offsets; /* host pointer, read during the call only */
} s2_stride_segment;

typedef struct s2_pattern_config {
    int seq_len;      /* N tokens */
    int block_size;   /* S tokens per block; B = ceil(N/S) */
    int num_heads;    /* H */
    int num_kv_heads; /* 0 means num_heads */
    int local_blocks;
    int local_stride;
    int num_segments;
    s2_stride_segment segments[S2_MAX_SEGMENTS];
} s2_pattern_config;

/* Fills cfg like make_single_stride_config (pattern.cpp:190-204): one segment
 * {local_blocks, B, remote_stride} when local_blocks < B.  Validates. */
int s2_make_single_stride_config(int seq_len, int block_size, int num_heads, int local_blocks,
                                 int remote_stride, int local_stride, s2_pattern_config* cfg);

/* PatternConfig::validate (pattern.cpp:36-79). */
int s2_pattern_validate(const s2_pattern_config* cfg);
/* PatternConfig::num_blocks (pattern.cpp:12-14). */
int s2_pattern_num_blocks(const s2_pattern_config* cfg);
/* PatternConfig::offset_for (pattern.cpp:16-34). */
int s2_pattern_offset_for(const s2_pattern_config* cfg, int segment, int head, int* offset);

/* ---- host layout builder (analytic, O(nnz)) ----------------------------- */
/* Bit-exact to to_csr(build_head_mask(cfg, head)) (csr.cpp:35-47,
 * pattern.cpp:127-158) without materialising the B x B mask. */
int s2_layout_nnz(const s2_pattern_config* cfg, int head, int64_t* nnz);
/* row_ptr: B+1 ints; col_idx: nnz ints, ascending within each row. */
int s2_layout_build_csr(const s2_pattern_config* cfg, int head, int* row_ptr, int* col_idx);
/* Transpose of the same bits (no reference symbol; backward layout):
 * col_ptr: B+1 ints; row_idx: nnz ints, ascending within each column. */
int s2_layout_build_csc(const s2_pattern_config* cfg, int head, int* col_ptr, int* row_idx);
/* HeadCacheSchedule::evict_after (analysis.cpp:76-82): per key block the last
 * query block attending it.  evict_after: B ints. */
int s2_layout_evict_after(const s2_pattern_config* cfg, int head, int* evict_after);
/* check_kv_cache_efficiency (verify.cpp:53-72): *ok = 1 when every column's
 * attending rows form one interval starting at the diagonal. */
int s2_layout_kv_efficient(const s2_pattern_config* cfg, int head, int* ok);
/* CsrMask::validate (csr.cpp:11-33). */
int s2_csr_validate(int num_blocks, const int* row_ptr, const int* col_idx, int64_t nnz);

/* ---- plans: device-resident layout + tile work lists -------------------- */
typedef struct s2_plan s2_plan;

/* From a policy (the north_star path). */
int s2_plan_create(const s2_pattern_config* cfg, s2_plan** plan);
/* From caller CSR lists, one per head (the shim path for
 * streaming_sharded_attention(t, vector<CsrMask>, block_size),
 * attention.cpp:100-118, with the same validation). row_ptr[h]: B+1 ints,
 * col_idx[h]: row_ptr[h][B] ints.  GQA heads of a group must share bits. */
int s2_plan_create_from_csr(int num_heads, int num_kv_heads, int seq_len, int block_size,
                            const int* const* row_ptr, const int* const* col_idx,
                            s2_plan** plan);
void s2_plan_destroy(s2_plan* plan);

typedef struct s2_plan_stats {
    int num_heads, num_kv_heads, seq_len, block_size, num_blocks;
    int64_t nnz_total;        /* sum over heads of active block pairs */
    int64_t dense_pairs;      /* B(B+1)/2 per head, summed */
    int max_row_len, max_col_len;
    int64_t fwd_tiles;        /* (head, 128-row q tile) work items */
    int64_t fwd_chunk_visits; /* 64-key chunks visited by the fwd kernel */
    int64_t bwd_tiles;        /* (kv-group, 128-key tile) work items */
    int64_t bwd_qtile_visits; /* q tiles visited by the dK/dV kernel */
} s2_plan_stats;
int s2_plan_get_stats(const s2_plan* plan, s2_plan_stats* stats);
/* Introspection of the tile work lists (tests, tooling).  Pass NULL arrays to
 * query the sizes.  fwd: offsets [H * num_qtiles + 1], chunk / mask per entry.
 * bwd: tiles [5 * num_tiles] = {group, c0, c1, offset, count},
 * entries [3 * num_entries] = {qtile, mask0, mask1}. */
int s2_plan_fwd_tiles(s2_plan* plan, int* num_qtiles, int64_t* num_entries, int64_t* offsets,
                      int32_t* chunks, uint32_t* masks);
int s2_plan_bwd_tiles(s2_plan* plan, int64_t* num_tiles, int64_t* num_entries, int64_t* tiles,
                      int64_t* entries);
/* Active block pairs of one head (exact_flops' nnz_per_head, analysis.cpp:46-48). */
int s2_plan_head_nnz(const s2_plan* plan, int head, int64_t* nnz);

/* ---- forward ------------------------------------------------------------ */
/* Replaces streaming_sharded_attention / dsplit_attention
 * (attention.cpp:190-198).  num_splits is validated exactly like the
 * reference (>= 1 and divides head_dim, attention.cpp:109-110); the GPU
 * kernel's accumulation order does not depend on it, so dsplit(1) and
 * streaming are bit-identical as the reference requires
 * (test_attention.cpp:124-132).
 *
 * Kernels: bf16 with head_dim 64 / 128 and block_size % 16 == 0 runs the
 * tcgen05 kernel; every other bf16 / fp32 case runs an fp32-FFMA kernel --
 * shared-memory tiles for head_dim <= 256, one warp per row up to 2048 -- with
 * no tensor cores; head_dim > 2048 fails with S2_ERR_UNSUPPORTED.  s2_attn_bwd
 * follows the same split, its fp32-FFMA kernels taking head_dim <= 128
 * (S2_ERR_UNSUPPORTED above).
 *
 * Units: the head-parallel partitioner works on (batch, kv-group) units,
 * u = b*num_kv_heads + g.  unit_ids == NULL processes every unit and the
 * tensors have the full layout above; otherwise the tensors hold only the
 * listed units, packed unit-major: q/out [num_units, H/Hkv, N, D],
 * k/v [num_units, N, D], lse [num_units, H/Hkv, N]. */
/* Literal zero softmax scale (negative zero; +0.0 selects the default). */
#define S2_SCALE_ZERO (-0.0)

typedef struct s2_attn_args {
    int dtype;
    int batch, num_heads, num_kv_heads, seq_len, head_dim;
    double scale; /* +0.0 => 1/sqrt(head_dim) as AttentionTensors::zeros;
                     S2_SCALE_ZERO (-0.0) => a literal 0 (uniform weights, as the
                     reference computes for scale == 0) */
    int num_splits;
    int num_units;       /* ignored when unit_ids == NULL */
    const int* unit_ids; /* host */
    const void* q;
    const void* k;
    const void* v;
    void* out;
    float* lse;
} s2_attn_args;
int s2_attn_fwd(s2_plan* plan, const s2_attn_args* args, s2_stream_t stream);

/* Forward with the head-parallel output exchange fused in (no reference
 * symbol): besides args->out / args->lse (this rank's packed
 * units), every finished O tile is TMA-stored into each of the num_peers
 * ranks' FULL output buffers, and its lse rows written there.  The forward and
 * the all-gather become one kernel; peer memory is reached over NVLink P2P
 * (buffers mapped with CUDA IPC or symmetric memory).
 *   peer_out[r]  bf16 [total_units, H/Hkv, N, D] of rank r (device pointer valid here)
 *   peer_lse[r]  fp32 [total_units, H/Hkv, N]
 *   unit_global  device int[num_units]: global unit index of each local unit
 *                (the full layouts are unit-major, as with unit_ids == NULL)
 * Requires the bf16 tcgen05 path and args->unit_ids; 1 <= num_peers <= 8.
 * The caller orders the ranks' completion (e.g. a barrier after the kernel)
 * before reading the full buffers. */
int s2_attn_fwd_peers(s2_plan* plan, const s2_attn_args* args, int num_peers, void* const* peer_out,
                      float* const* peer_lse, const int* unit_global, int total_units,
                      s2_stream_t stream);

/* ---- backward (no reference symbol: SPEC.md:262) ------------------------ */
/* dQ kernel walks the CSR tile list, dK/dV kernel walks the transposed (CSC)
 * tile list; every dK/dV tile is owned by exactly one CTA (no atomics).
 * bf16, head_dim 64 / 128, block_size % 16 == 0: tcgen05 kernels (bwd_sm100.cu);
 * other bf16 / fp32 shapes with head_dim <= 128: fp32-FFMA tile kernels over
 * the plan's CSR / CSC (bwd_simt.cu); head_dim > 128 otherwise:
 * S2_ERR_UNSUPPORTED. */
typedef struct s2_attn_bwd_args {
    s2_attn_args fwd; /* q, k, v, out (forward output), lse as written by fwd */
    const void* dout;
    void* dq;
    void* dk;
    void* dv;
} s2_attn_bwd_args;
int s2_attn_bwd_workspace_size(const s2_plan* plan, const s2_attn_bwd_args* args, size_t* bytes);
int s2_attn_bwd(s2_plan* plan, const s2_attn_bwd_args* args, void* workspace,
                size_t workspace_bytes, s2_stream_t stream);

/* ---- one layer's forward + backward on HOST buffers -------------------------
 * The reference's data path (AttentionTensors in host memory, attention.hpp:
 * 17-37), for the shapes s2_attn_bwd takes (bf16 or fp32): every pointer in
 * `args` (q, k, v, dout in; out, lse, dq, dk, dv out) is HOST memory, ideally
 * pinned.  The (batch, kv-group) units are cut
 * into num_chunks chunks whose H2D copy, forward + backward and D2H copy are
 * pipelined on three streams (heads are independent, test_attention.cpp:
 * 217-240), so the PCIe transfers overlap each other and the kernels.
 * workspace: device memory of s2_attn_fwd_bwd_host_workspace_size bytes.
 * Completion is ordered on `stream`. */
int s2_attn_fwd_bwd_host_workspace_size(const s2_plan* plan, const s2_attn_bwd_args* args,
                                        int num_chunks, size_t* bytes);
int s2_attn_fwd_bwd_host(s2_plan* plan, const s2_attn_bwd_args* args, int num_chunks,
                         void* workspace, size_t workspace_bytes, s2_stream_t stream);

/* ---- decode over a per-(batch, kv-head) compacted KV cache --------------- */
/* Cache contents follow simulate_decode_cache (analysis.cpp:57-104): key
 * block j is kept while the decode row bt <= evict_after[j]; for KV-efficient
 * masks (verify.cpp:53-72) the kept set is exactly row bt of the mask, so the
 * cache stores only the blocks each head can attend.  Non-efficient masks are
 * rejected with S2_ERR_UNSUPPORTED. */
typedef struct s2_kvcache s2_kvcache;
int s2_kvcache_create(s2_plan* plan, int batch, int head_dim, int dtype, s2_kvcache** cache);
void s2_kvcache_destroy(s2_kvcache* cache);
/* Number of tokens currently held per sequence (= next position). */
int s2_kvcache_length(const s2_kvcache* cache, int* length);
/* Physical device bytes of the pool and the bytes a dense cache would need. */
int s2_kvcache_bytes(const s2_kvcache* cache, int64_t* pool_bytes, int64_t* dense_bytes);
/* Retained tokens per sequence per kv head at the current length. */
int s2_kvcache_retained_tokens(const s2_kvcache* cache, int kv_head, int64_t* tokens);
/* Compacts a dense prefix k/v [batch, Hkv, num_tokens, D] (device) into the
 * cache (kv_compact kernel); resets the length to num_tokens. */
int s2_kvcache_prefill(s2_kvcache* cache, const void* k, const void* v, int num_tokens,
                       s2_stream_t stream);
/* Appends one token per sequence, k/v [batch, Hkv, D] (kv_append kernel). */
int s2_kvcache_append(s2_kvcache* cache, const void* k, const void* v, s2_stream_t stream);
/* One query row per (batch, head) at position length-1: q/out [batch, H, D],
 * lse [batch, H] (may be NULL).  Split-KV kernel + lse-weighted combine. */
int s2_attn_decode_workspace_size(const s2_kvcache* cache, size_t* bytes);
int s2_attn_decode(s2_kvcache* cache, const void* q, void* out, float* lse, double scale,
                   void* workspace, size_t workspace_bytes, s2_stream_t stream);
/* Bytes the decode step must read from HBM at the current length (K,V of the
 * retained tokens + q + out): the roofline numerator. */
int s2_attn_decode_bytes(const s2_kvcache* cache, int64_t* bytes);

/* ---- head-parallel partitioner (no reference symbol) -------------------- */
/* Weight of every (batch, kv-group) unit = active block pairs of its heads. */
int s2_plan_unit_weights(const s2_plan* plan, int batch, int64_t* weights);
/* LPT: units sorted by weight descending (ties by id), each to the least
 * loaded rank (ties to the lowest rank).  owner: num_units ints; load:
 * num_ranks int64 (may be NULL).  Deterministic. */
int s2_partition_lpt(int num_units, const int64_t* weights, int num_ranks, int* owner,
                     int64_t* load);

/* ---- FLOP / byte accounting (analysis.cpp:29-55) ------------------------ */
/* 4 * head_dim * block_size^2 per active pair, summed over heads and batch. */
int s2_plan_fwd_flops(const s2_plan* plan, int batch, int head_dim, double* active_flops,
                      double* dense_causal_flops);

/* ---- reference test inputs ---------------------------------------------- */
/* AttentionTensors::random (attention.cpp:135-144): mt19937_64(seed), U[-1,1]
 * floats from std::uniform_real_distribution<float>, q then k then v, each
 * num_heads * seq_len * head_dim values [H, N, d].  Host buffers; the same
 * stream as the reference for the same seed (libstdc++). */
int s2_random_tensors(int num_heads, int seq_len, int head_dim, uint64_t seed, float* q, float* k,
                      float* v);

/* ---- device memory helpers (so FFI callers need no CUDA runtime) --------- */
int s2_device_count(int* count);
int s2_device_malloc(void** ptr, size_t bytes);
int s2_device_free(void* ptr);
int s2_memcpy_h2d(void* dst, const void* src, size_t bytes, s2_stream_t stream);
int s2_memcpy_d2h(void* dst, const void* src, size_t bytes, s2_stream_t stream);
int s2_stream_synchronize(s2_stream_t stream);

/* ---- per-kernel device timing ------------------------------------------- */
/* When enabled, every kernel launch records a CUDA event pair on its own
 * stream.  collect() synchronizes those events, returns per-kernel-name
 * totals (names: max_kernels x 32 chars) and clears the records. */
int s2_profile_enable(int enable);
int s2_profile_collect(int max_kernels, char* names, double* total_ms, int* launches,
                       int* num_kernels);

/* ---- serialization (reference serialize.hpp / serialize.cpp) -----------
 * JSON documents are UTF-8 text.  to_json outputs are the reference's
 * canonical encoding (object keys sorted, compact separators), so
 * s2_pattern_hash equals shardattn::config_hash for the same config. */

/* to_json(PatternConfig) (serialize.cpp:30-47).  buf may be NULL (size
 * query); *len = bytes excluding the terminating NUL. */
int s2_pattern_to_json(const s2_pattern_config* cfg, char* buf, size_t cap, size_t* len);
/* pattern_config_from_json (serialize.cpp:75-95): defaults num_kv_heads =
 * num_heads, local_blocks = 1, local_stride = 1, offset_scheme
 * "head_mod_stride"; validates (pattern.cpp:36-79).  Segment offsets are
 * written to offsets_buf (offsets_cap ints) and cfg's offset pointers point
 * into it. */
int s2_pattern_from_json(const char* text, s2_pattern_config* cfg, int* offsets_buf,
                         int offsets_cap);
/* config_hash (serialize.cpp:148-156): FNV-1a 64 over the canonical document. */
int s2_pattern_hash(const s2_pattern_config* cfg, uint64_t* hash);

/* to_json(CsrMask) / csr_from_json (serialize.cpp:68-73,108-116); from_json
 * validates (csr.cpp:11-33).  Pass NULL arrays to query num_blocks / nnz. */
int s2_csr_to_json(int head_index, int num_blocks, const int* row_ptr, const int* col_idx,
                   char* buf, size_t cap, size_t* len);
int s2_csr_from_json(const char* text, int* head_index, int* num_blocks, int* row_ptr,
                     int row_cap, int* col_idx, int64_t col_cap, int64_t* nnz);

/* POD mirror of shardattn::LayerSchedule (pattern.hpp:98-104). */
typedef struct s2_layer_schedule {
    int num_layers;
    int num_dense;
    const int* dense_layer_ids; /* host pointer, ascending */
    s2_pattern_config sparse_pattern;
} s2_layer_schedule;
/* LayerSchedule::validate (pattern.cpp:118-125). */
int s2_schedule_validate(const s2_layer_schedule* schedule);
/* to_json(LayerSchedule) / layer_schedule_from_json (serialize.cpp:49-53,97-106);
 * from_json inherits default_pattern when "sparse_pattern" is absent. */
int s2_schedule_to_json(const s2_layer_schedule* schedule, char* buf, size_t cap, size_t* len);
int s2_schedule_from_json(const char* text, const s2_pattern_config* default_pattern,
                          s2_layer_schedule* schedule, int* dense_buf, int dense_cap,
                          int* offsets_buf, int offsets_cap);

/* CliConfigFile / load_config_file (serialize.hpp:31-41, serialize.cpp:123-146):
 * a pattern (top level or under "pattern"), an optional "schedule" and
 * optional "report" {out, format}.  Failures -> S2_ERR_CONFIG with
 * "config '<path>': <reason>" (file missing: "cannot open config file"). */
typedef struct s2_config_file {
    s2_pattern_config pattern;
    int has_schedule;
    s2_layer_schedule schedule; /* sparse_pattern == pattern unless given */
    char out[512];
    char format[64];
} s2_config_file;
int s2_config_file_load(const char* path, s2_config_file* file, int* dense_buf, int dense_cap,
                        int* offsets_buf, int offsets_cap);

/* ---- analysis (reference analysis.hpp / analysis.cpp) ------------------ */
/* equivalent_context_length, analytic_flops_reduction, speedup_upper_bound
 * (analysis.cpp:13-27); same argument checks. */
int s2_equivalent_context_length(double seq_len, double local_window, double stride, double* out);
int s2_analytic_flops_reduction(double seq_len, double local_window, double stride, double* out);
int s2_speedup_upper_bound(int num_heads, double seq_len, double local_window, double* out);
/* exact_flops (analysis.cpp:33-55): nnz_per_head may be NULL. */
typedef struct s2_flops_report {
    double dense_flops, sparse_flops, reduction_factor, equivalent_context;
} s2_flops_report;
int s2_exact_flops(const s2_pattern_config* cfg, int head_dim, s2_flops_report* report,
                   int64_t* nnz_per_head);
/* simulate_decode_cache for one head (analysis.cpp:57-104), computed from
 * the CSC in O(B + total_tokens): evict_after[B], occupancy[total_tokens]
 * (retained tokens per decode step), dead_blocks[total_tokens]; any output
 * array may be NULL. */
int s2_simulate_decode_cache(const s2_pattern_config* cfg, int total_tokens, int head,
                             int* evict_after, int64_t* occupancy, int* dead_blocks,
                             int64_t* peak_tokens, double* mean_tokens);
/* kv_reduction (analysis.cpp:106-121): percent of KV cache saved vs dense,
 * averaged over heads and layers (dense layers keep everything). */
int s2_kv_reduction(const s2_layer_schedule* schedule, double* percent);

/* ---- hybrid layer stacks (reference LayerSchedule / build_layer_masks) ----
 * One plan per distinct layer type of a schedule: the sparse pattern for S2
 * layers and make_dense_config of the same shape (== dense_causal_mask,
 * pattern.cpp:168-181,233-236) for the dense layer ids; every layer of a
 * 24-layer model then runs through the same kernels with its own layout. */
typedef struct s2_layers s2_layers;
int s2_layers_create(const s2_layer_schedule* schedule, s2_layers** layers);
void s2_layers_destroy(s2_layers* layers);
/* Borrowed plan of `layer` (valid until s2_layers_destroy); *is_dense set when
 * it is one of the dense layer ids. */
int s2_layers_plan(s2_layers* layers, int layer, s2_plan** plan, int* is_dense);
/* s2_attn_fwd / s2_attn_bwd with the layer's plan. */
int s2_layers_fwd(s2_layers* layers, int layer, const s2_attn_args* args, s2_stream_t stream);
int s2_layers_bwd(s2_layers* layers, int layer, const s2_attn_bwd_args* args, void* workspace,
                  size_t workspace_bytes, s2_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* S2ATTN_H_ */
