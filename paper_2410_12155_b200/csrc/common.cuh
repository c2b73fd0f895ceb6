// Shared helpers of the libvpfv CUDA sources (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vpfv.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libvpfv is written for sm_100a (B200) only"
#endif

namespace vpfv {

constexpr int NG = 3;  // ghost width (grid.py:17)

__device__ __forceinline__ double ldg(const double *p) { return __ldg(p); }

int set_error(int code, const char *msg);
int check_launch(const char *what);

}  // namespace vpfv
