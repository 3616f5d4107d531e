// Helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

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
int ensure_csr_uploaded(s2_plan* p);
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
