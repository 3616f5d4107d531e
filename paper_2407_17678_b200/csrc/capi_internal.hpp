// Helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/s2attn.h"
#include "plan.hpp"

namespace s2 {
extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int check_args(const s2_plan* p, const s2_attn_args* a);
int num_sms();
int persistent_grid();  // num_sms() minus s2_set_sm_reserve
bool use_tcgen05(const s2_plan* p, const s2_attn_args* a);
// The softmax scale of s2_attn_args: +0.0 selects 1/sqrt(head_dim); S2_SCALE_ZERO
// (-0.0) is a literal zero scale (the reference's default-constructed
// AttentionTensors, attention.hpp:23: uniform weights over the admitted keys).
// It is evaluated as 1e-30: every admitted logit then rounds to exactly 0 in
// fp32 (exp2 of it is 1.0f) while masked logits stay -inf (0 * -inf would be NaN).
inline double resolve_scale(double scale, int head_dim) {
    if (scale != 0.0) return scale;
    return std::signbit(scale) ? 1e-30 : 1.0 / std::sqrt(static_cast<double>(head_dim));
}
// A plan's device-side caches (CSR, tile lists, work items) live on the device of
// their first use; a call on another device fails instead of handing it foreign
// pointers.
int check_device(const s2_plan* p);
int ensure_csr_uploaded(s2_plan* p);
int ensure_csc_uploaded(s2_plan* p);
Lists* get_lists(s2_plan* p, int seq_len, int* status);
WorkItems* get_items(s2_plan* p, Lists* L, int batch, int num_units, const int* unit_ids,
                     int* status);
// RAII: records a CUDA event pair around a launch when profiling is enabled.
class ProfScope {
public:
    ProfScope(const char* name, cudaStream_t st);
    ~ProfScope();

private:
    const char* name_;
    cudaStream_t st_;
    void* a_ = nullptr;
    void* b_ = nullptr;
    bool active_ = false;
};
}  // namespace s2
