// Small helpers shared by the runtime translation units.
#pragma once

#include <chrono>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "../capi/status.hpp"

namespace mlt::detail {

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// 2 MiB-aligned THP host buffer, optionally page-locked (runtime.cpp).
uint8_t* host_alloc(size_t bytes, bool pin, double* pin_seconds);
void host_free(void* p, bool pinned);

}  // namespace mlt::detail
