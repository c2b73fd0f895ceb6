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

// Programmatic dependent launch (the 1D chains; the 2D field chain moment
// finish -> charge -> FFT passes -> tables -> 2D-2V stage kernel): a kernel
// launched with launch_pdl may start while its predecessor in the stream
// drains; it runs its independent prologue, then pdl_wait() before touching
// anything the predecessor wrote.  pdl_trigger() lets the successor start
// launching -- only in kernels whose successors wait first (the field chain
// links): measured, a stage kernel that triggered let the ordinary moment
// launch after it read a half-written f, so no stage kernel triggers.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // VPFV_PDL != 0

// Peer halo push (x-slab ranks over NVLink): after every thread of the CTA
// has made its stores (peer ones included) visible system-wide, count the
// CTA; the last one bumps both neighbours' signal words (csrc/peer.cu).
// P: a stage parameter block with done / sig_lo / sig_hi.
// nthreads > 0: only the first nthreads threads take part (named barrier 1),
// for warp-specialised kernels whose producer warps make no peer stores
template <class StageParams>
__device__ __forceinline__ void peer_done_signal(const StageParams &P, int nthreads = 0) {
    if (!P.done) return;
    __threadfence_system();
    if (nthreads > 0)
        asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
    else
        __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(P.done, 1u);
        if (prev == gridDim.x - 1) {
            *P.done = 0u;  // ready for the next launch (ordered by the kernel boundary)
            __threadfence_system();
            if (P.sig_lo) atomicAdd_system(P.sig_lo, 1ull);
            if (P.sig_hi) atomicAdd_system(P.sig_hi, 1ull);
        }
    }
}

template <typename... Args>
cudaError_t launch_pdl(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace vpfv
