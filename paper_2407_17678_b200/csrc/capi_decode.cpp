// C ABI: compacted KV cache + sparse decode.
#include "capi_internal.hpp"

using namespace s2;

extern "C" {
int s2_kvcache_create(s2_plan*, int, int, int, s2_kvcache**) {
    return fail(S2_ERR_UNSUPPORTED, "decode not built yet");
}
void s2_kvcache_destroy(s2_kvcache*) {}
int s2_kvcache_length(const s2_kvcache*, int*) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_kvcache_bytes(const s2_kvcache*, int64_t*, int64_t*) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_kvcache_retained_tokens(const s2_kvcache*, int, int64_t*) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_kvcache_prefill(s2_kvcache*, const void*, const void*, int, s2_stream_t) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_kvcache_append(s2_kvcache*, const void*, const void*, s2_stream_t) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_attn_decode_workspace_size(const s2_kvcache*, size_t*) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_attn_decode(s2_kvcache*, const void*, void*, float*, double, void*, size_t, s2_stream_t) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
int s2_attn_decode_bytes(const s2_kvcache*, int64_t*) { return fail(S2_ERR_UNSUPPORTED, "decode not built yet"); }
}
