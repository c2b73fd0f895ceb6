// DFMA latency / throughput probe (k independent dependent chains per thread).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_lat dfma_lat.cu && ./dfma_lat
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void chain(double *out, long long *cyc, int iters, double a, double b) {
    double x[K];
    for (int k = 0; k < K; ++k) x[k] = threadIdx.x + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < K; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K>
void run(int warps) {
    double *o; long long *c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8 * 148);
    int iters = 4096;
    chain<K><<<148, 32 * warps>>>(o, c, iters, 0.999, 0.001);
    chain<K><<<148, 32 * warps>>>(o, c, iters, 0.999, 0.001);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / (iters * K);
    printf("K=%2d warps/SM=%2d: %.2f cyc per DFMA per warp-chain step; SM DFMA rate = %.1f lanes/clk\n", K, warps,
           (double)h / iters, 32.0 * warps * K * iters / h);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<1>(1); run<2>(1); run<4>(1); run<8>(1);
    run<1>(4); run<2>(4); run<4>(4); run<8>(4);
    run<1>(8); run<2>(8); run<4>(8); run<8>(8);
    run<1>(16); run<4>(16); run<8>(16);
    return 0;
}
