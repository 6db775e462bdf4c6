#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "bd_attn.h"

namespace bd {

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);

// Count of kernels this library has enqueued (bd_launch_count).
void note_launches(int n);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace bd
