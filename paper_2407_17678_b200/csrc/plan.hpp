// s2_plan: host layout (CSR per head, tile lists) + lazily uploaded device
// copies, keyed per (seq_len, batch, unit set) for the work-item arrays.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels/common.cuh"
#include "layout.hpp"

namespace s2 {

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    int device = -1;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (ptr) {
            int cur = -1;
            cudaGetDevice(&cur);
            if (device >= 0 && device != cur) cudaSetDevice(device);
            cudaFree(ptr);
            if (device >= 0 && device != cur && cur >= 0) cudaSetDevice(cur);
        }
    }
    template <class T>
    T* as() const { return static_cast<T*>(ptr); }
};

// Upload host bytes to a fresh device buffer (synchronous; layout-time only).
cudaError_t upload(DevBuf& buf, const void* host, size_t bytes);

struct WorkItems {
    DevBuf fwd;       // s2dev::FwdItem[] (per 128-row q tile; dQ kernel)
    int num_fwd = 0;
    DevBuf pair;      // PairItem[] (per q-tile pair; forward kernel)
    int num_pair = 0;
    DevBuf bwd;       // s2dev::BwdItem[]
    int num_bwd = 0;
    bool bwd_dropped = false;  // key tiles nobody attends (user CSR without diagonal): dK/dV = 0
    DevBuf pair2;     // PairItem[] regrouped for the CTA-pair forward (fwd_pair2.cu)
    int num_pair2 = 0;
    int clusters = 0;  // CTA pairs of the pair2 forward's persistent grid (0: not built)
    DevBuf fwd_sched, pair_sched, bwd_sched, pair2_sched;  // int[grid + 1] per-CTA (per-cluster) item ranges
    int grid = 0;      // backward kernels (dQ: fwd_sched, dK/dV: bwd_sched): SMs minus the reserve
    int grid_fwd = 0;  // forward (pair_sched): every SM
    DevBuf simt_bh;   // int[num_bh] data index
    DevBuf simt_head; // int[num_bh] layout head
    int num_bh = 0;
};

struct Lists {
    bool tiled = false;  // block_size % 16 == 0 -> tcgen05 lists exist
    FwdList fwd;
    PairList pairs;
    BwdList bwd;
    DevBuf d_chunks;   // int2
    DevBuf d_steps;    // PairStep
    DevBuf d_entries;  // s2dev::BwdEntry
    bool uploaded = false;
    std::map<std::string, std::unique_ptr<WorkItems>> items;
};

}  // namespace s2

struct s2_plan {
    int num_heads = 0, num_kv_heads = 0, seq_len = 0, block_size = 0, num_blocks = 0;
    bool has_pattern = false;
    s2::Pattern pattern;
    std::vector<s2::Csr> csr;  // per head
    std::vector<int64_t> col_off;
    // device CSR (SIMT path)
    s2::DevBuf d_row_ptr, d_col_idx, d_col_off;
    bool csr_uploaded = false;
    // device CSC (SIMT backward): key block -> query blocks, per head
    s2::DevBuf d_col_ptr, d_row_idx, d_row_off;
    bool csc_uploaded = false;
    std::mutex mu;
    int device = -1;  // CUDA device of the first call that built device-side state
    std::map<int, std::unique_ptr<s2::Lists>> lists;  // keyed by seq_len
};
