// C ABI: backward (dQ over the CSR tile list, dK/dV over the transposed list).
#include "capi_internal.hpp"

using namespace s2;

extern "C" {
int s2_attn_bwd_workspace_size(const s2_plan* p, const s2_attn_bwd_args* a, size_t* bytes) {
    if (!bytes) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (int rc = check_args(p, a ? &a->fwd : nullptr)) return rc;
    *bytes = 0;
    return S2_OK;
}
int s2_attn_bwd(s2_plan*, const s2_attn_bwd_args*, void*, size_t, s2_stream_t) {
    return fail(S2_ERR_UNSUPPORTED, "backward not built yet");
}
}
