// Signalling for the x-slab halo push over NVLink peer memory.
//
// In the peer mode of DistributedSimulation (parallel.py) each rank's stage
// kernel stores its 3 boundary x planes straight into the x neighbours'
// dest buffers (their ghost planes) as it computes them -- the halo exchange
// of the reference cluster (runner.py:394-437, Exchanger partition.py:679-724)
// fused into the producing kernel, no separate copy or NCCL call.  The last
// CTA of that kernel bumps a 64-bit signal word on each neighbour
// (vpfv_stage_2d2v_fused_peer); before its next stage reads those ghost
// planes a rank runs vpfv_peer_wait, one thread spinning on its own signal
// words with system-scope acquire loads.  The words only grow; each rank
// keeps how many signals it has consumed in device memory, so the same wait
// is valid in every replay of a captured step.  Ordering argument (DESIGN.md
// "Multi-GPU"): a rank starts stage k only after both neighbours finished
// stage k-1, so a push never lands in a buffer a neighbour is still reading.
#include <cuda.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace vpfv {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void peer_signal_kernel(unsigned long long *sig_lo, unsigned long long *sig_hi) {
    __threadfence_system();
    if (sig_lo) atomicAdd_system(sig_lo, 1ull);
    if (sig_hi) atomicAdd_system(sig_hi, 1ull);
}

// sig[0]: signals from the low x neighbour, sig[1]: from the high one
__global__ void peer_wait_kernel(const unsigned long long *sig, unsigned long long *consumed, unsigned need_lo,
                                 unsigned need_hi, unsigned long long timeout_ns, int *timed_out) {
    const unsigned need[2] = {need_lo, need_hi};
    const unsigned long long t0 = now_ns();
    for (int k = 0; k < 2; ++k) {
        if (!need[k]) continue;
        const unsigned long long target = consumed[k] + need[k];
        while (ld_acquire_sys(sig + k) < target) {
            if (now_ns() - t0 > timeout_ns) {  // a lost neighbour must not hang the device
                atomicExch(timed_out, 1);
                return;
            }
            __nanosleep(200);
        }
        consumed[k] = target;
    }
    __threadfence();
}

// The per-step divergence verdict of every rank, exchanged over peer
// memory inside the step (the reference rolls the whole cluster back when any
// box went non-finite, runner.py:453-464).  Each rank stamps its word
// (step << 1 | bad) into its slot of every rank's flag array, then waits
// until all slots of its own array carry this step's stamp and ORs the bad
// bits into *out.  The step counter lives on the device, so a captured step
// replays correctly; ranks advance it in lockstep (one exchange per step).
__global__ void flag_exchange_kernel(const long long *nonfinite, int nspecies, unsigned long long *const *slots,
                                     int world, const unsigned long long *mine, unsigned long long *stamp,
                                     unsigned long long *out, unsigned long long timeout_ns, int *timed_out) {
    __shared__ unsigned long long word;
    const int t = threadIdx.x;
    if (t == 0) {
        bool bad = false;
        for (int s = 0; s < nspecies; ++s) bad |= nonfinite[s] != -1LL;
        const unsigned long long st = *stamp + 1;
        *stamp = st;
        word = (st << 1) | (bad ? 1ull : 0ull);
    }
    __syncthreads();
    const unsigned long long w = word, st = w >> 1;
    if (t < world) {
        __threadfence_system();
        atomicExch_system(slots[t], w);
    }
    unsigned long long any = 0;
    if (t < world) {
        const unsigned long long t0 = now_ns();
        unsigned long long v;
        while (((v = ld_acquire_sys(mine + t)) >> 1) < st) {
            if (now_ns() - t0 > timeout_ns) {
                atomicExch(timed_out, 1);
                v = 1;  // a lost rank counts as diverged
                break;
            }
            __nanosleep(100);
        }
        any = v & 1ull;
    }
    any = __any_sync(0xffffffffu, any != 0) ? 1ull : 0ull;
    if (t == 0) *out = any;
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_flag_exchange(const long long *nonfinite, int nspecies, unsigned long long *const *slots,
                                  int world, const unsigned long long *mine, unsigned long long *stamp,
                                  unsigned long long *out, double timeout_s, int *timed_out, void *stream) {
    if (world < 1 || world > 32 || nspecies < 1 || !nonfinite || !slots || !mine || !stamp || !out || !timed_out)
        return set_error(VPFV_EARG, "flag_exchange: bad arguments");
    flag_exchange_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(nonfinite, nspecies, slots, world, mine, stamp, out,
                                                            (unsigned long long)(timeout_s * 1e9), timed_out);
    return check_launch("flag_exchange");
}

extern "C" int vpfv_peer_signal(unsigned long long *sig_lo, unsigned long long *sig_hi, void *stream) {
    peer_signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sig_lo, sig_hi);
    return check_launch("peer_signal");
}

extern "C" int vpfv_peer_wait(const unsigned long long *sig, unsigned long long *consumed, int need_lo, int need_hi,
                              double timeout_s, int *timed_out, void *stream) {
    if (!sig || !consumed || !timed_out || need_lo < 0 || need_hi < 0)
        return set_error(VPFV_EARG, "peer_wait: bad arguments");
    peer_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(sig, consumed, (unsigned)need_lo, (unsigned)need_hi,
                                                       (unsigned long long)(timeout_s * 1e9), timed_out);
    return check_launch("peer_wait");
}

// ---------------------------------------------------------------------------
// CUDA IPC of state buffers between the rank processes.  A handle names a
// whole allocation (a torch caching-allocator block), so the export also
// returns the buffer's offset in it; the open maps the allocation into the
// calling device's context with peer access enabled (stores and system
// atomics then travel over NVLink), once per allocation and process.

typedef CUresult (*AddressRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

static AddressRangeFn address_range() {
    static AddressRangeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddressRangeFn>(p);
    }
    return fn;
}

extern "C" int vpfv_ipc_export(const void *ptr, unsigned char *handle_out, long long *offset_out) {
    AddressRangeFn fn = address_range();
    if (!fn) return set_error(VPFV_ECUDA, "ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return set_error(VPFV_ECUDA, "ipc_export: not device memory");
    static std::mutex mu;
    static std::map<CUdeviceptr, cudaIpcMemHandle_t> handles;  // one handle per allocation
    std::lock_guard<std::mutex> lock(mu);
    auto it = handles.find(base);
    if (it == handles.end()) {
        cudaIpcMemHandle_t h;
        cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
        if (e != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(e));
        it = handles.emplace(base, h).first;
    }
    memcpy(handle_out, &it->second, sizeof(cudaIpcMemHandle_t));
    *offset_out = (long long)((CUdeviceptr)ptr - base);
    return VPFV_OK;
}

extern "C" int vpfv_ipc_open(const unsigned char *handle, long long offset, void **ptr_out) {
    static std::mutex mu;
    static std::map<std::string, void *> opened;
    std::lock_guard<std::mutex> lock(mu);
    const std::string key(reinterpret_cast<const char *>(handle), sizeof(cudaIpcMemHandle_t));
    auto it = opened.find(key);
    void *base = nullptr;
    if (it != opened.end()) {
        base = it->second;
    } else {
        cudaIpcMemHandle_t h;
        memcpy(&h, handle, sizeof(h));
        cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(e));
        opened[key] = base;
    }
    *ptr_out = static_cast<char *>(base) + offset;
    return VPFV_OK;
}

extern "C" int vpfv_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }
