#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "bd_attn.h"

namespace bd {

int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);

// Count of kernels this library has enqueued (bd_launch_count).
void note_launches(int n);

// Kernel attributes belong to the CUDA context of a device: set
// MaxDynamicSharedMemorySize of `func` once per (function, current device)
// (thread-safe; the return code of the attribute call is checked).
int ensure_smem_attr(const void* func, int bytes, const char* what);
// Multiprocessor count of the current device (cached per device).
int current_sm_count(int* n_sm);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace bd
