// Per-kernel CUDA-event timing for bench.py (s2_profile_* in s2attn.h).
#include <cuda_runtime.h>

#include <random>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.hpp"

namespace s2 {
namespace {
struct Rec {
    std::string name;
    cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

ProfScope::ProfScope(const char* name, cudaStream_t st) : name_(name), st_(st) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_on) return;
    a_ = take();
    b_ = take();
    cudaEventRecord(static_cast<cudaEvent_t>(a_), st_);
    active_ = true;
}

ProfScope::~ProfScope() {
    if (!active_) return;
    cudaEventRecord(static_cast<cudaEvent_t>(b_), st_);
    std::lock_guard<std::mutex> lk(g_mu);
    g_recs.push_back({name_, static_cast<cudaEvent_t>(a_), static_cast<cudaEvent_t>(b_)});
}
}  // namespace s2

using namespace s2;

extern "C" {
int s2_profile_enable(int enable) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_on = enable != 0;
    for (auto& r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    return S2_OK;
}

int s2_profile_collect(int max_kernels, char* names, double* total_ms, int* launches,
                       int* num_kernels) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<double, int>> acc;
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& x = acc[r.name];
        x.first += ms;
        x.second += 1;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    int n = 0;
    for (auto& kv : acc) {
        if (n >= max_kernels) break;
        if (names) {
            std::memset(names + 32 * n, 0, 32);
            std::strncpy(names + 32 * n, kv.first.c_str(), 31);
        }
        if (total_ms) total_ms[n] = kv.second.first;
        if (launches) launches[n] = kv.second.second;
        ++n;
    }
    if (num_kernels) *num_kernels = n;
    return S2_OK;
}
}

extern "C" {
int s2_random_tensors(int num_heads, int seq_len, int head_dim, uint64_t seed, float* q, float* k,
                      float* v) {
    if (num_heads < 1 || seq_len < 1 || head_dim < 1)
        return fail(S2_ERR_INVALID_ARGUMENT, "tensor dimensions must be positive");
    if (!q || !k || !v) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(num_heads) * seq_len * head_dim;
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<float> u(-1.0f, 1.0f);
    for (float* dst : {q, k, v})
        for (size_t i = 0; i < n; ++i) dst[i] = u(gen);
    return S2_OK;
}

int s2_device_count(int* count) {
    if (!count) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *count = n;
    return S2_OK;
}
int s2_device_malloc(void** ptr, size_t bytes) {
    if (!ptr) return fail(S2_ERR_INVALID_ARGUMENT, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(S2_ERR_NO_DEVICE, "no CUDA device: the S2 kernels need a B200");
    cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 16);
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "cudaMalloc");
}
int s2_device_free(void* ptr) {
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "cudaFree");
}
int s2_memcpy_h2d(void* dst, const void* src, size_t bytes, s2_stream_t stream) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice,
                                    reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "cudaMemcpyAsync H2D");
}
int s2_memcpy_d2h(void* dst, const void* src, size_t bytes, s2_stream_t stream) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost,
                                    reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "cudaMemcpyAsync D2H");
}
int s2_stream_synchronize(s2_stream_t stream) {
    cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? S2_OK : cuda_fail(e, "cudaStreamSynchronize");
}
}
