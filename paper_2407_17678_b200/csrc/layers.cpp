// C ABI: hybrid dense / S2 layer stacks (reference LayerSchedule,
// pattern.hpp:98-104; build_layer_masks, pattern.cpp:168-181).  A stack owns
// two plans (sparse pattern, dense-causal of the same shape) and maps each
// layer id to one of them, so a 24-layer hybrid model (cfg3: dense {0, 1})
// runs every layer through the same tcgen05 kernels.
#include <cstring>
#include <set>

#include "capi_internal.hpp"

struct s2_layers {
    int num_layers = 0;
    std::set<int> dense;
    s2_plan* sparse = nullptr;
    s2_plan* dense_plan = nullptr;
    ~s2_layers() {
        s2_plan_destroy(sparse);
        s2_plan_destroy(dense_plan);
    }
};

using namespace s2;

extern "C" {

int s2_layers_create(const s2_layer_schedule* schedule, s2_layers** out) {
    if (int rc = s2_schedule_validate(schedule)) return rc;
    if (!out) return fail(S2_ERR_INVALID_ARGUMENT, "output pointer is null");
    auto* L = new s2_layers();
    L->num_layers = schedule->num_layers;
    L->dense.insert(schedule->dense_layer_ids, schedule->dense_layer_ids + schedule->num_dense);
    int rc = s2_plan_create(&schedule->sparse_pattern, &L->sparse);
    if (rc == S2_OK && !L->dense.empty()) {
        const s2_pattern_config& sp = schedule->sparse_pattern;
        s2_pattern_config dc;  // make_dense_config(seq_len, block_size, num_heads) + the kv heads
        rc = s2_make_single_stride_config(sp.seq_len, sp.block_size, sp.num_heads, 1, 1, 1, &dc);
        if (rc == S2_OK) {
            dc.num_kv_heads = sp.num_kv_heads;
            rc = s2_plan_create(&dc, &L->dense_plan);
        }
    }
    if (rc != S2_OK) {
        delete L;
        return rc;
    }
    *out = L;
    return S2_OK;
}

void s2_layers_destroy(s2_layers* layers) { delete layers; }

int s2_layers_plan(s2_layers* L, int layer, s2_plan** plan, int* is_dense) {
    if (!L || !plan) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (layer < 0 || layer >= L->num_layers) return fail(S2_ERR_INVALID_ARGUMENT, "layer outside [0, num_layers)");
    const bool d = L->dense.count(layer) != 0;
    *plan = d ? L->dense_plan : L->sparse;
    if (is_dense) *is_dense = d ? 1 : 0;
    return S2_OK;
}

int s2_layers_fwd(s2_layers* L, int layer, const s2_attn_args* args, s2_stream_t stream) {
    s2_plan* p = nullptr;
    if (int rc = s2_layers_plan(L, layer, &p, nullptr)) return rc;
    return s2_attn_fwd(p, args, stream);
}

int s2_layers_bwd(s2_layers* L, int layer, const s2_attn_bwd_args* args, void* workspace,
                  size_t workspace_bytes, s2_stream_t stream) {
    s2_plan* p = nullptr;
    if (int rc = s2_layers_plan(L, layer, &p, nullptr)) return rc;
    return s2_attn_bwd(p, args, workspace, workspace_bytes, stream);
}

}  // extern "C"
