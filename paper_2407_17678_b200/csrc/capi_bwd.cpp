// C ABI: backward (dQ over the CSR tile list, dK/dV over the transposed list).
#include <cmath>
#include <cstdlib>

#include "capi_internal.hpp"
#include "tma_host.hpp"

cudaError_t s2_launch_bwd_prep(const __nv_bfloat16* out, const __nv_bfloat16* dout,
                               const float* lse, float* delta, float* lse2, int num_bh, int N,
                               int Npad, int D, cudaStream_t stream);
cudaError_t s2_launch_bwd_sm100(int which, int D, const CUtensorMap& q, const CUtensorMap& dout,
                                const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o0,
                                const CUtensorMap& o1, const void* items, const int* sched, int grid,
                                const void* entries, const float* lse2, const float* delta,
                                int N, int Npad, int hpg, float scale, cudaStream_t stream,
                                void* g0, void* g1, const void* fused_o = nullptr,
                                const void* fused_dout = nullptr, const float* fused_lse = nullptr,
                                float* fused_delta = nullptr, float* fused_lse2 = nullptr);

cudaError_t s2_launch_bwd_simt(bool bf16, const void* q, const void* k, const void* v, const void* out,
                               const float* lse, const void* dout, void* dq, void* dk, void* dv,
                               const int* bh_list, const int* head_of, int num_bh, const int* row_ptr,
                               const int* col_idx, const int64_t* col_off, const int* col_ptr,
                               const int* row_idx, const int64_t* row_off, float* delta, int N, int Npad,
                               int D, int S, int B, int hpg, float scale, cudaStream_t stream);

using namespace s2;

namespace {
int num_q_heads(const s2_plan* p, const s2_attn_args* a) {
    const int hpg = p->num_heads / p->num_kv_heads;
    return (a->unit_ids ? a->num_units : a->batch * p->num_kv_heads) * hpg;
}
size_t ws_bytes(const s2_plan* p, const s2_attn_args* a) {
    const size_t npad = (static_cast<size_t>(a->seq_len) + 127) / 128 * 128;
    return 2 * static_cast<size_t>(num_q_heads(p, a)) * npad * sizeof(float);
}
int check_bwd(const s2_plan* p, const s2_attn_bwd_args* a) {
    if (!a) return fail(S2_ERR_INVALID_ARGUMENT, "args is null");
    if (int rc = check_args(p, &a->fwd)) return rc;
    if (!a->dout || !a->dq || !a->dk || !a->dv)
        return fail(S2_ERR_INVALID_ARGUMENT, "dout/dq/dk/dv must be non-null device pointers");
    // shapes the tcgen05 kernels do not tile (fp32, other head_dim / block_size)
    // run the fp32-FFMA tile kernels, which stage up to 128 columns
    if (!use_tcgen05(p, &a->fwd) && a->fwd.head_dim > 128)
        return fail(S2_ERR_UNSUPPORTED,
                    "backward needs head_dim <= 128 (bf16 tcgen05: head_dim in {64,128}, block_size % 16 == 0)");
    return S2_OK;
}
}  // namespace

extern "C" {
int s2_attn_bwd_workspace_size(const s2_plan* p, const s2_attn_bwd_args* a, size_t* bytes) {
    if (!bytes) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    if (int rc = check_bwd(p, a)) return rc;
    *bytes = ws_bytes(p, &a->fwd);
    return S2_OK;
}

int s2_attn_bwd(s2_plan* p, const s2_attn_bwd_args* a, void* workspace, size_t workspace_bytes,
                s2_stream_t stream) {
    if (int rc = check_bwd(p, a)) return rc;
    const s2_attn_args& f = a->fwd;
    if (workspace_bytes < ws_bytes(p, &f) || !workspace)
        return fail(S2_ERR_INVALID_ARGUMENT, "workspace too small (s2_attn_bwd_workspace_size)");
    std::lock_guard<std::mutex> lk(p->mu);
    int rc = S2_OK;
    Lists* L = get_lists(p, f.seq_len, &rc);
    if (!L) return rc;
    WorkItems* w = get_items(p, L, f.batch, f.num_units, f.unit_ids, &rc);
    if (!w) return rc;
    const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int hpg = p->num_heads / p->num_kv_heads;
    const int nqbh = num_q_heads(p, &f);
    const int nkv = nqbh / hpg;
    const int N = f.seq_len, D = f.head_dim;
    const int Npad = (N + 127) / 128 * 128;
    const double scale = resolve_scale(f.scale, D);
    float* delta = static_cast<float*>(workspace);
    float* lse2 = delta + static_cast<size_t>(nqbh) * Npad;
    cudaError_t e = cudaSuccess;
    if (!use_tcgen05(p, &f)) {
        if ((rc = ensure_csr_uploaded(p)) || (rc = ensure_csc_uploaded(p))) return rc;
        ProfScope prof("bwd_simt", st);
        e = s2_launch_bwd_simt(f.dtype == S2_DTYPE_BF16, f.q, f.k, f.v, f.out, f.lse, a->dout, a->dq, a->dk,
                               a->dv, w->simt_bh.as<int>(), w->simt_head.as<int>(), w->num_bh,
                               p->d_row_ptr.as<int>(), p->d_col_idx.as<int>(), p->d_col_off.as<int64_t>(),
                               p->d_col_ptr.as<int>(), p->d_row_idx.as<int>(), p->d_row_off.as<int64_t>(), delta,
                               N, Npad, D, p->block_size, p->num_blocks, hpg, float(scale), st);
        if (e != cudaSuccess) return cuda_fail(e, "s2_attn_bwd launch");
        return S2_OK;
    }
    // S2_PREP_FUSED=1 fuses the prep (Delta = rowsum(dO o O), lse2) into the dQ
    // kernel, which then runs first and leaves both in the workspace for dK/dV.  Off
    // by default: the per-item row loads of O and dO stall the elementwise warps at
    // item starts (cfg3: dQ 0.83 -> 1.06 ms against the 0.10 ms prep it saves).
    const char* dkv_env = std::getenv("S2_DKV_V2");
    const bool dkv_v1 = !(dkv_env && dkv_env[0] == '1');
    const char* dq_env = std::getenv("S2_DQ_V2");
    const bool dq_v1 = !(dq_env && dq_env[0] == '1');
    const char* fz_env = std::getenv("S2_PREP_FUSED");
    const bool fused = dq_v1 && fz_env && fz_env[0] == '1';
    if (!fused) {
        ProfScope prof("bwd_prep", st);
        e = s2_launch_bwd_prep(static_cast<const __nv_bfloat16*>(f.out),
                               static_cast<const __nv_bfloat16*>(a->dout), f.lse, delta, lse2,
                               nqbh, N, Npad, D, st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "s2_attn_bwd prep launch");
    try {
        using s2host::make_map_bf16_3d;
        using s2host::make_map_bf16_kmajor;
        // streamed operands: whole-row 4-D boxes (Q/dO halves for dK/dV, Q/dO tiles
        // and K/V chunks for dQ); the dK/dV kernel's K/V pair tiles and the 128-key
        // dQ kernel's K/V stages are two chunks per D/64 slice: 3-D boxes
        const CUtensorMap q64 = make_map_bf16_kmajor(f.q, D, N, nqbh, 64);
        const CUtensorMap do64 = make_map_bf16_kmajor(a->dout, D, N, nqbh, 64);
        const CUtensorMap q128 = make_map_bf16_kmajor(f.q, D, N, nqbh, 128);
        const CUtensorMap do128 = make_map_bf16_kmajor(a->dout, D, N, nqbh, 128);
        const CUtensorMap mk = make_map_bf16_3d(f.k, D, N, nkv, 64, 64);
        const CUtensorMap mv = make_map_bf16_3d(f.v, D, N, nkv, 64, 64);
        const CUtensorMap mk4 = make_map_bf16_kmajor(f.k, D, N, nkv, 64);
        const CUtensorMap mv4 = make_map_bf16_kmajor(f.v, D, N, nkv, 64);
        // key chunks no query attends are never visited (no tile covers them, or a
        // tile has no steps): their dK / dV are 0
        if (w->bwd_dropped || L->bwd.uncovered) {
            const size_t bytes = static_cast<size_t>(nkv) * N * D * 2;
            if ((e = cudaMemsetAsync(a->dk, 0, bytes, st)) != cudaSuccess ||
                (e = cudaMemsetAsync(a->dv, 0, bytes, st)) != cudaSuccess)
                return cuda_fail(e, "s2_attn_bwd memset");
        }
        const CUtensorMap mdk = make_map_bf16_3d(a->dk, D, N, nkv, 64, 64);
        const CUtensorMap mdv = make_map_bf16_3d(a->dv, D, N, nkv, 64, 64);
        const CUtensorMap mdq = make_map_bf16_3d(a->dq, D, N, nqbh, 64, 128);
        auto run_dq = [&]() {
            ProfScope prof("bwd_dq_sm100", st);
            // S2_DQ_V2=1: the experimental 128-key-step dQ kernel (s2_bwd_dq2_kernel;
            // slower at cfg3: its two-chunk K/V stages need 8 KB TMA boxes)
            return s2_launch_bwd_sm100(dq_v1 ? 1 : 2, D, q128, do128, dq_v1 ? mk4 : mk, dq_v1 ? mv4 : mv, mdq, mdq,
                                       w->fwd.ptr, w->fwd_sched.as<int>(), w->grid, L->d_chunks.ptr, lse2, delta, N,
                                       Npad, hpg, float(scale), st, nullptr, nullptr, fused ? f.out : nullptr,
                                       a->dout, f.lse, delta, lse2);
        };
        auto run_dkv = [&]() {
            ProfScope prof("bwd_dkv_sm100", st);
            // S2_DKV_V2=1: the experimental 128-row-step dK/dV kernel (s2_bwd_dkv2_kernel;
            // slower at cfg3)
            if (dkv_v1)
                return s2_launch_bwd_sm100(0, D, q64, do64, mk, mv, mdk, mdv, w->bwd.ptr, w->bwd_sched.as<int>(),
                                           w->grid, L->d_entries.ptr, lse2, delta, N, Npad, hpg, float(scale), st,
                                           nullptr, nullptr);
            return s2_launch_bwd_sm100(3, D, q128, do128, mk, mv, mdk, mdv, w->bwd.ptr, w->bwd_sched.as<int>(),
                                       w->grid, L->d_entries.ptr, lse2, delta, N, Npad, hpg, float(scale), st,
                                       a->dk, a->dv);
        };
        if (fused) {
            e = run_dq();
            if (e == cudaSuccess) e = run_dkv();
        } else {
            e = run_dkv();
            if (e == cudaSuccess) e = run_dq();
        }
    } catch (const std::exception& ex) {
        return fail(S2_ERR_CUDA, ex.what());
    }
    if (e != cudaSuccess) return cuda_fail(e, "s2_attn_bwd launch");
    return S2_OK;
}
}
