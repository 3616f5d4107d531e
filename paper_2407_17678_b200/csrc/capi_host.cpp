// C ABI: one layer's forward + backward on HOST buffers (the reference API's
// data path: AttentionTensors live in host memory, attention.hpp:17-37),
// pipelined over chunks of (batch, kv-group) units.  Heads are independent
// (test_attention.cpp:217-240), so chunk c's H2D copy, chunk c-1's forward +
// backward and chunk c-2's D2H copy run concurrently on three streams: the
// PCIe transfers overlap each other (full duplex) and the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "capi_internal.hpp"

using namespace s2;

namespace {

struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev;
    int device = -1;
};

// Streams/events of the calling thread's current device (created once).
Pipe* pipe_for_device(int need_events) {
    static thread_local std::vector<Pipe> pipes;
    int dev = 0;
    cudaGetDevice(&dev);
    for (Pipe& p : pipes)
        if (p.device == dev) {
            while (static_cast<int>(p.ev.size()) < need_events) {
                cudaEvent_t e;
                if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
                p.ev.push_back(e);
            }
            return &p;
        }
    Pipe p;
    p.device = dev;
    if (cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    pipes.push_back(p);
    return pipe_for_device(need_events);
}

struct Layout {
    size_t q, kv, lse;  // bytes per unit
    size_t off[9];      // q k v dout out lse dq dk dv
    size_t total;
};

Layout layout(const s2_plan* p, const s2_attn_args& f) {
    const int hpg = p->num_heads / p->num_kv_heads;
    const size_t units = static_cast<size_t>(f.batch) * p->num_kv_heads;
    Layout L{};
    const size_t es = f.dtype == S2_DTYPE_F32 ? 4 : 2;  // element bytes
    L.q = static_cast<size_t>(hpg) * f.seq_len * f.head_dim * es;
    L.kv = static_cast<size_t>(f.seq_len) * f.head_dim * es;
    L.lse = static_cast<size_t>(hpg) * f.seq_len * 4;
    const size_t per[9] = {L.q, L.kv, L.kv, L.q, L.q, L.lse, L.q, L.kv, L.kv};
    size_t o = 0;
    for (int i = 0; i < 9; ++i) {
        L.off[i] = o;
        o += (per[i] * units + 255) / 256 * 256;
    }
    L.total = o;
    return L;
}

int check_host(const s2_plan* p, const s2_attn_bwd_args* a, int num_chunks) {
    if (!p || !a) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (a->fwd.unit_ids) return fail(S2_ERR_INVALID_ARGUMENT, "the host path runs every unit (unit_ids must be NULL)");
    if (num_chunks < 1) return fail(S2_ERR_INVALID_ARGUMENT, "num_chunks must be positive");
    if (int rc = check_args(p, &a->fwd)) return rc;
    if (!a->dout || !a->dq || !a->dk || !a->dv)
        return fail(S2_ERR_INVALID_ARGUMENT, "dout/dq/dk/dv must be non-null host pointers");
    // the shapes s2_attn_bwd takes: bf16 tcgen05 ones, and any fp32 / bf16 with
    // head_dim <= 128 on the FFMA kernels
    if (!use_tcgen05(p, &a->fwd) && a->fwd.head_dim > 128)
        return fail(S2_ERR_UNSUPPORTED, "the host path needs head_dim <= 128 (the backward's limit)");
    return S2_OK;
}

size_t bwd_ws(const s2_plan* p, const s2_attn_args& f, int units_max) {
    const int hpg = p->num_heads / p->num_kv_heads;
    const size_t npad = (static_cast<size_t>(f.seq_len) + 127) / 128 * 128;
    return 2 * static_cast<size_t>(units_max) * hpg * npad * sizeof(float);
}

}  // namespace

extern "C" {

int s2_attn_fwd_bwd_host_workspace_size(const s2_plan* p, const s2_attn_bwd_args* a, int num_chunks,
                                        size_t* bytes) {
    if (!bytes) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (int rc = check_host(p, a, num_chunks)) return rc;
    const int units = a->fwd.batch * p->num_kv_heads;
    const int per = (units + num_chunks - 1) / num_chunks;
    *bytes = layout(p, a->fwd).total + bwd_ws(p, a->fwd, per);
    return S2_OK;
}

int s2_attn_fwd_bwd_host(s2_plan* p, const s2_attn_bwd_args* a, int num_chunks, void* workspace,
                         size_t workspace_bytes, s2_stream_t stream) {
    if (int rc = check_host(p, a, num_chunks)) return rc;
    size_t need = 0;
    s2_attn_fwd_bwd_host_workspace_size(p, a, num_chunks, &need);
    if (!workspace || workspace_bytes < need)
        return fail(S2_ERR_INVALID_ARGUMENT, "workspace too small (s2_attn_fwd_bwd_host_workspace_size)");
    const s2_attn_args& f = a->fwd;
    const int units = f.batch * p->num_kv_heads;
    num_chunks = std::min(num_chunks, units);
    const int per = (units + num_chunks - 1) / num_chunks;
    Pipe* pp = pipe_for_device(3 * num_chunks);
    if (!pp) return fail(S2_ERR_CUDA, "creating the copy streams");
    const cudaStream_t comp = reinterpret_cast<cudaStream_t>(stream);
    const Layout L = layout(p, f);
    char* ws = static_cast<char*>(workspace);
    char* dev[9];
    for (int i = 0; i < 9; ++i) dev[i] = ws + L.off[i];
    void* bws = ws + L.total;
    const size_t bws_bytes = workspace_bytes - L.total;
    const char* hin[4] = {static_cast<const char*>(f.q), static_cast<const char*>(f.k),
                          static_cast<const char*>(f.v), static_cast<const char*>(a->dout)};
    char* hout[5] = {static_cast<char*>(f.out), reinterpret_cast<char*>(f.lse), static_cast<char*>(a->dq),
                     static_cast<char*>(a->dk), static_cast<char*>(a->dv)};
    const size_t in_unit[4] = {L.q, L.kv, L.kv, L.q};
    const size_t out_unit[5] = {L.q, L.lse, L.q, L.kv, L.kv};
    const int in_idx[4] = {0, 1, 2, 3}, out_idx[5] = {4, 5, 6, 7, 8};
    std::vector<int> ids(units);
    for (int u = 0; u < units; ++u) ids[u] = u;
    cudaError_t e = cudaSuccess;
    // the copies must not start before earlier work on the caller's stream
    cudaEvent_t* ev = pp->ev.data();
    if ((e = cudaEventRecord(ev[0], comp)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(pp->h2d, ev[0], 0)) != cudaSuccess)
        return cuda_fail(e, "host pipeline");
    for (int c = 0; c < num_chunks; ++c) {
        const int u0 = c * per, u1 = std::min(units, u0 + per), n = u1 - u0;
        if (n <= 0) break;
        cudaEvent_t ev_in = ev[3 * c], ev_done = ev[3 * c + 1];
        for (int i = 0; i < 4; ++i)
            if ((e = cudaMemcpyAsync(dev[in_idx[i]] + u0 * in_unit[i], hin[i] + u0 * in_unit[i], n * in_unit[i],
                                     cudaMemcpyHostToDevice, pp->h2d)) != cudaSuccess)
                return cuda_fail(e, "host pipeline H2D");
        if ((e = cudaEventRecord(ev_in, pp->h2d)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(comp, ev_in, 0)) != cudaSuccess)
            return cuda_fail(e, "host pipeline");
        s2_attn_bwd_args b = *a;
        b.fwd.num_units = n;
        b.fwd.unit_ids = ids.data() + u0;
        b.fwd.q = dev[0] + u0 * L.q;
        b.fwd.k = dev[1] + u0 * L.kv;
        b.fwd.v = dev[2] + u0 * L.kv;
        b.dout = dev[3] + u0 * L.q;
        b.fwd.out = dev[4] + u0 * L.q;
        b.fwd.lse = reinterpret_cast<float*>(dev[5] + u0 * L.lse);
        b.dq = dev[6] + u0 * L.q;
        b.dk = dev[7] + u0 * L.kv;
        b.dv = dev[8] + u0 * L.kv;
        if (int rc = s2_attn_fwd(p, &b.fwd, stream)) return rc;
        if (int rc = s2_attn_bwd(p, &b, bws, bws_bytes, stream)) return rc;
        if ((e = cudaEventRecord(ev_done, comp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(pp->d2h, ev_done, 0)) != cudaSuccess)
            return cuda_fail(e, "host pipeline");
        for (int i = 0; i < 5; ++i)
            if ((e = cudaMemcpyAsync(hout[i] + u0 * out_unit[i], dev[out_idx[i]] + u0 * out_unit[i],
                                     n * out_unit[i], cudaMemcpyDeviceToHost, pp->d2h)) != cudaSuccess)
                return cuda_fail(e, "host pipeline D2H");
    }
    // the caller's stream covers the whole pipeline
    cudaEvent_t ev_end = ev[2];
    if ((e = cudaEventRecord(ev_end, pp->d2h)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(comp, ev_end, 0)) != cudaSuccess)
        return cuda_fail(e, "host pipeline");
    return S2_OK;
}

}  // extern "C"
