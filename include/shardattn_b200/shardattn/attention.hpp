// Drop-in replacement header for /root/reference/proj/include/shardattn/attention.hpp
// (attention.hpp:17-66).  Host tensors in and out exactly as the reference;
// the work runs on the B200 behind include/s2attn.h:
//   streaming_sharded_attention / dsplit_attention -> fp32 sm_100a kernel
//   naive_masked_attention / dense_masked_attention -> the same kernel after
//     the reference's mask validation (dense: finiteness + causal masks)
// Extensions in the house style (the reference has neither):
//   streaming_sharded_attention_backward -> fp32 sm_100a backward kernels
//   sharded_decode -> compacted KV cache + split-KV decode kernel
#pragma once

#include <cstdint>
#include <vector>

#include "shardattn/csr.hpp"
#include "shardattn/pattern.hpp"

namespace shardattn {

struct AttentionTensors {
    int num_heads = 0;
    int seq_len = 0;
    int head_dim = 0;
    double scale = 0.0;

    std::vector<float> q, k, v;
    std::vector<float> out;
    std::vector<double> lse;

    static AttentionTensors zeros(int num_heads, int seq_len, int head_dim);
    static AttentionTensors random(int num_heads, int seq_len, int head_dim, std::uint64_t seed);

    std::size_t idx(int head, int token, int component) const {
        return (static_cast<std::size_t>(head) * seq_len + token) * head_dim + component;
    }
    std::size_t row_index(int head, int token) const {
        return static_cast<std::size_t>(head) * seq_len + token;
    }
};

void naive_masked_attention(AttentionTensors& t, const std::vector<HeadBlockMask>& masks,
                            int block_size);
void dense_masked_attention(AttentionTensors& t, const std::vector<HeadBlockMask>& masks,
                            int block_size);
void streaming_sharded_attention(AttentionTensors& t, const std::vector<CsrMask>& csr,
                                 int block_size);
void dsplit_attention(AttentionTensors& t, const std::vector<CsrMask>& csr, int block_size,
                      int num_splits);

/// Gradients of sum(dout * out) w.r.t. q, k, v for the forward above, in fp32
/// like the forward (tolerance 1e-4 against an fp64 restatement); head_dim <= 128
/// (larger throws std::invalid_argument).  Shapes as q/k/v.
struct AttentionGrads {
    std::vector<float> dq, dk, dv;
};
void streaming_sharded_attention_backward(const AttentionTensors& t,
                                          const std::vector<CsrMask>& csr, int block_size,
                                          const std::vector<float>& dout, AttentionGrads& grads);

/// Decode of one token position: row `position` of every head, computed the
/// way a generation step would -- the keys/values of tokens 0..position are
/// compacted into a per-head cache that keeps only the blocks some row at or
/// after `position` can still attend (analysis.cpp:57-104's retained set), and
/// one query row per head attends the blocks of its mask row (reference.cpp:28-50
/// for a single row), tokens <= position.  Equals row `position` of
/// streaming_sharded_attention within bf16 tolerance (inputs rounded to bf16).
/// Resizes out / lse like the forward (zeros / -inf) and fills only that row.
/// Throws std::invalid_argument on the forward's conditions and on a position
/// outside [0, seq_len).
void sharded_decode(AttentionTensors& t, const std::vector<CsrMask>& csr, int block_size,
                    int position);

}  // namespace shardattn
