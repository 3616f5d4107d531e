// Score masking shared by the S2 forward kernels (fwd_sm100.cu, fwd_pair2.cu).
// A tile-list mask word covers one 64-key chunk for a 128-row query tile: 8 row
// groups x 4 column groups of 16 tokens (bit 4*rg + g).  Unset groups are -inf;
// inside the diagonal chunk, keys after the query row are -inf as well (in-block
// causality, /root/reference/proj/src/attention.cpp:46).
#pragma once
#include <math.h>
#include <stdint.h>

namespace s2dev {

__device__ __forceinline__ void apply_mask(float* s, int chunk, uint32_t mask, int rg, int q_pos,
                                           int qtile_row0) {
    const uint32_t bits = (mask >> (rg * 4)) & 0xFu;
    const int key0 = chunk * 64;
    const bool diag = key0 + 63 > qtile_row0;
    if (bits == 0xFu && !diag) return;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const bool on = (bits >> g) & 1u;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (!on || (diag && key0 + g * 16 + j > q_pos)) s[g * 16 + j] = -INFINITY;
        }
    }
}

// The same rule for 32 of the chunk's 64 columns: piece `half` (columns
// [32 half, 32 half + 32), groups 2 half and 2 half + 1).
__device__ __forceinline__ void apply_mask32(float* s, int chunk, uint32_t mask, int rg, int q_pos, int qtile_row0,
                                             int half) {
    const uint32_t bits = (mask >> (rg * 4 + 2 * half)) & 0x3u;
    const int key0 = chunk * 64 + 32 * half;
    const bool diag = chunk * 64 + 63 > qtile_row0;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const bool on = (bits >> g) & 1u;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (!on || (diag && key0 + g * 16 + j > q_pos)) s[g * 16 + j] = -INFINITY;
        }
    }
}

}  // namespace s2dev
