// Shared device-side types of the S2 kernels (mirrors csrc/plan.hpp).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace s2dev {

// One forward / dQ work item: a 128-row query tile of one (batch, head).
struct FwdItem {
    int32_t bh;         // data index of the query head (batch*H + h, or packed unit index)
    int32_t head;       // layout head (selects the chunk list)
    int32_t qtile;      // query rows qtile*128 .. +127
    int32_t chunk_cnt;  // number of 64-key chunks
    int64_t chunk_off;  // offset into the chunk array
};

// One dK/dV work item: a pair of 64-key chunks of one (batch, kv head).
struct BwdItem {
    int32_t kvbh;    // data index of the kv head
    int32_t c0, c1;  // chunks (c1 = -1 when single)
    int32_t count;   // q tiles visited
    int64_t offset;  // into the BwdEntry array
    int32_t nsteps;  // (query head, q tile, active 64-row half) steps = hpg * active halves
    int32_t nsteps128;  // (query head, q tile) steps of the 128-row kernel = hpg * active tiles
};
struct BwdEntry {
    int32_t qtile;
    uint32_t mask0, mask1;
};

// Split-KV decode launch parameters (kernels/decode.cu, capi_decode.cpp).
struct DecodeParams {
    const __nv_bfloat16* q;     // [B, H, D]
    const int64_t* row_ptr;     // [Hkv][NB+1] offsets into slot_idx (rows of the mask)
    const int* slot_idx;        // slots of each row's key blocks, ascending key block
    int NB;                     // blocks of the layout
    int bt;                     // current decode row
    int last_tokens;            // valid tokens of block bt (the row's last entry)
    int splits;
    int blocks_per_split;
    int H, Hkv, D, hpg;
    float scale_log2;
    float* o_part;    // [B, H, splits, D]
    float* lse_part;  // [B, H, splits] (log2 domain)
};

}  // namespace s2dev

#include <cstdlib>
#include <cuda_runtime.h>

namespace s2dev {
// Launch with programmatic stream serialization (PDL) unless S2_PDL=0: the
// kernels call griddepcontrol.launch_dependents / .wait, so the next kernel's
// CTAs are scheduled as this one's exit and do their setup during its tail.
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("S2_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <typename Kern, typename... Args>
inline cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // namespace s2dev
