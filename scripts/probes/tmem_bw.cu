// TMEM <-> register throughput probe (sm_100a): could the stage kernel's x
// windows live in tensor memory instead of registers?
//
// Each CTA allocates 512 TMEM columns; every warp repeatedly loads (and
// optionally stores back) NCOL 32-bit columns of its lane quarter with
// tcgen05.ld/st .32x32b, waiting on each batch.  Prints bytes per clock per
// SM for loads alone, load+store round trips, and stores alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cuda_runtime.h>

#define LD32(r, addr)                                                                                           \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),       \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
                   "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),             \
                   "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),             \
                   "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])              \
                 : "r"(addr))
#define ST32(addr, r)                                                                                          \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
                 "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"            \
                 ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),  \
                 "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),          \
                 "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),         \
                 "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),         \
                 "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                                               \
                 : "memory")

template <int MODE>  // 0: load only, 1: load + store back, 2: store only
__global__ void probe(unsigned *out, long long *cyc, int iters, int ncolbatches) {
    __shared__ unsigned taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = taddr_s;
    // warp w: lanes 32*(w%4).., its own column range (warps sharing a lane quarter split the 512 columns)
    const int nw = blockDim.x >> 5, per_quarter = nw / 4 > 0 ? nw / 4 : 1;
    const int colspan = 512 / per_quarter;
    const unsigned mine = base + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)((warp >> 2) * colspan);
    unsigned r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 32 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        for (int b = 0; b < ncolbatches; ++b) {
            const unsigned a = mine + (unsigned)(b * 32);
            if (MODE != 2) {
                LD32(r, a);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            if (MODE != 0) {
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] += 1u;
                ST32(a, r);
            }
        }
        if (MODE != 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    unsigned acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

template <int MODE>
void run(int warps, int ncolbatches) {
    unsigned *o;
    long long *c;
    cudaMalloc(&o, 148 * 1024 * 4);
    cudaMalloc(&c, 148 * 8);
    const int iters = 2000;
    probe<MODE><<<148, 32 * warps>>>(o, c, iters, ncolbatches);
    probe<MODE><<<148, 32 * warps>>>(o, c, iters, ncolbatches);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * ncolbatches * warps * 32 * 32 * 4 * (MODE == 1 ? 2 : 1);
    printf("mode=%s warps=%2d batches/iter=%d: %.1f B/clk/SM (%s)\n",
           MODE == 0 ? "ld   " : (MODE == 1 ? "ld+st" : "st   "), warps, ncolbatches, bytes / (double)h,
           cudaGetErrorString(e));
    cudaFree(o);
    cudaFree(c);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>(w, 4);
        run<1>(w, 4);
        run<2>(w, 4);
    }
    return 0;
}
