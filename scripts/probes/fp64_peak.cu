// FP64 throughput peak of the whole GPU (the roofline denominator of the
// fp64-issue-bound stage kernels; MEASURED_PEAKS.json has no fp64 figure).
//
// Every thread runs K independent DFMA chains (K = 8 hides the ~8.4-cycle
// DFMA latency at any occupancy, scripts/probes/dfma_lat.cu), grid = 148 SMs
// x 4 CTAs of 256 threads, timed with CUDA events, best of 10.  Prints one
// JSON line: DFMA/s, FP64 TFLOP/s (2 flops per DFMA) and the SM clock the
// driver reported during the run.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu -lnvidia-ml
#include <cstdio>
#include <cuda_runtime.h>
#include <nvml.h>

template <int K>
__global__ void __launch_bounds__(256) dfma_chains(double *out, int iters, double a, double b) {
    double x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += x[k];
    if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains alive
}

int main() {
    int dev = 0, sms = 0;
    cudaSetDevice(dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *o;
    cudaMalloc(&o, 1 << 20);
    const int K = 8, iters = 1 << 16, threads = 256, blocks = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    nvmlInit();
    nvmlDevice_t h;
    nvmlDeviceGetHandleByIndex(dev, &h);
    float best = 1e30f;
    unsigned clk_sum = 0, clk_n = 0;
    for (int r = 0; r < 12; ++r) {
        cudaEventRecord(e0);
        dfma_chains<K><<<blocks, threads>>>(o, iters, 0.9999999, 1e-7);
        cudaEventRecord(e1);
        unsigned c = 0;
        if (r >= 2 && nvmlDeviceGetClockInfo(h, NVML_CLOCK_SM, &c) == NVML_SUCCESS) {
            clk_sum += c;
            ++clk_n;
        }
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2 && ms < best) best = ms;
    }
    unsigned cmax = 0;
    nvmlDeviceGetMaxClockInfo(h, NVML_CLOCK_SM, &cmax);
    const double dfma = (double)blocks * threads * K * (double)iters;
    const double rate = dfma / (best * 1e-3);
    printf("{\"fp64_dfma_per_s\": %.6e, \"fp64_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, "
           "\"sm_mhz_sampled\": %.0f, \"sm_max_mhz\": %u, \"lanes_per_clk_per_sm\": %.2f, "
           "\"how\": \"%d CTAs x %d threads x %d independent DFMA chains x %d iterations, best of 10, CUDA events\"}\n",
           rate, 2.0 * rate / 1e12, best, sms, clk_n ? (double)clk_sum / clk_n : 0.0, cmax,
           clk_n ? rate / (sms * 1e6 * ((double)clk_sum / clk_n)) : 0.0, blocks, threads, K, iters);
    return 0;
}
