// On-device velocity moments for the diagnostics rows.
//
// Per physical cell, the momentum and kinetic-energy sums over velocity space
// with the midpoint-to-average lift of higher_moments
// (/root/reference/pkg/src/vpfv/fields.py:131-161):
//     <v_d f>   = v_c f + (h_d^2 / 12) df/dv_d
//     <v_d^2 f> = (v_c^2 + h_d^2 / 12) f + (h_d^2 / 6) v_c df/dv_d
// with df/dv_d the centred difference (f[+1] - f[-1]) / (2 h_d), which reaches
// into the (frozen) velocity ghosts.  out[p][2k] = sum_v <v_k f>,
// out[p][2k+1] = sum_v <v_k^2 f> for velocity dim k; the host applies the
// velocity volume and the 1/2 in the reference's order.  The mass uses the
// fold-tree moment (vpfv_moment with vol = 1), finished on the host.
#include "common.cuh"

namespace vpfv {

struct Moments2 {
    const double *vc[2];
    double h[2];
};

template <int V>
__global__ void __launch_bounds__(256) higher_moments_kernel(const double *__restrict__ f, long long xstride,
                                                             long long ystride, int n0, int n1, long long s0,
                                                             Moments2 M, double *__restrict__ out) {
    // physical cell (x, y) = (blockIdx.y, blockIdx.x): its padded velocity
    // block starts at f + x*xstride + y*ystride (f already points at the
    // first interior physical cell); velocity dims (n0[, n1]) with padded row
    // stride s0 (the last dim has stride 1)
    const long long base = (long long)blockIdx.y * xstride + (long long)blockIdx.x * ystride;
    const long long pcell = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    const int nv = V == 1 ? n0 : n0 * n1;
    double acc[2 * V];
#pragma unroll
    for (int k = 0; k < 2 * V; ++k) acc[k] = 0.0;
    for (int c = threadIdx.x; c < nv; c += blockDim.x) {
        const int i0 = V == 1 ? c : c / n1, i1 = V == 1 ? 0 : c % n1;
        const long long at = V == 1 ? base + (i0 + NG) : base + (long long)(i0 + NG) * s0 + (i1 + NG);
        const double fv = f[at];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const long long st = (V == 2 && k == 0) ? s0 : 1;
            const double vc = __ldg(M.vc[k] + (k == 0 ? i0 : i1));
            const double h = M.h[k];
            const double h2 = h * h;
            const double dfd = (f[at + st] - f[at - st]) / (2.0 * h);
            acc[2 * k] += vc * fv + (h2 / 12.0) * dfd;
            acc[2 * k + 1] += (vc * vc + h2 / 12.0) * fv + (h2 / 6.0) * vc * dfd;
        }
    }
    __shared__ double red[2 * V][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 2 * V; ++k) {
        double x = acc[k];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) red[k][warp] = x;
    }
    __syncthreads();
    if (threadIdx.x < 2 * V) {
        double x = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x += red[threadIdx.x][w];
        out[pcell * 2 * V + threadIdx.x] = x;
    }
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_higher_moments(const double *f, int d, int v, const int *N, const double *vc0,
                                   const double *vc1, double h0, double h1, double *out, void *stream) {
    if (d < 1 || d > 2 || v < 1 || v > 2 || v < d) return set_error(VPFV_EDIM, "higher_moments: unsupported d+v");
    long long P[4];
    for (int k = 0; k < d + v; ++k) P[k] = N[k] + 2 * NG;
    long long vblock = 1;  // padded velocity block of one physical cell
    for (int k = d; k < d + v; ++k) vblock *= P[k];
    const long long ystride = d == 2 ? vblock : 0, xstride = d == 2 ? P[1] * vblock : vblock;
    const double *f0 = f + (long long)NG * xstride + (long long)NG * ystride;  // first interior physical cell
    const dim3 grid(d == 2 ? N[1] : 1, N[0]);
    Moments2 M{{vc0, vc1}, {h0, h1}};
    cudaStream_t s = (cudaStream_t)stream;
    if (v == 1)
        higher_moments_kernel<1><<<grid, 256, 0, s>>>(f0, xstride, ystride, N[d], 1, 1, M, out);
    else
        higher_moments_kernel<2><<<grid, 256, 0, s>>>(f0, xstride, ystride, N[d], N[d + 1], P[d + 1], M, out);
    return check_launch("higher_moments");
}

// ---------------------------------------------------------------------------
// Richardson error of a refinement (diagnostics.py:163-180): the fine field
// aggregated exactly onto the coarse cells (arithmetic mean of the 2^D
// children) and the L1 difference, summed per CTA (the host adds the partial
// sums in order and divides by the coarse cell count).

struct Dims4 {
    int n[4];       // coarse interior extents (1 for unused dims)
    long long sa[4], sb[4];  // padded strides of the coarse / fine arrays
    int D;
};

__global__ void __launch_bounds__(256) richardson_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                                         Dims4 g, long long total, double *__restrict__ part) {
    double acc = 0.0;
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (long long)gridDim.x * blockDim.x) {
        long long r = c, oa = 0, ob = 0;
        int idx[4];
        for (int k = g.D - 1; k >= 0; --k) {
            idx[k] = (int)(r % g.n[k]);
            r /= g.n[k];
        }
        for (int k = 0; k < g.D; ++k) {
            oa += (idx[k] + NG) * g.sa[k];
            ob += (2 * idx[k] + NG) * g.sb[k];
        }
        double s = 0.0;
        const int nch = 1 << g.D;
        for (int m = 0; m < nch; ++m) {
            long long o = ob;
            for (int k = 0; k < g.D; ++k)
                if (m & (1 << (g.D - 1 - k))) o += g.sb[k];
            s += b[o];
        }
        acc += fabs(a[oa] - s / (double)nch);
    }
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x += red[w];
        part[blockIdx.x] = x;
    }
}

extern "C" int vpfv_richardson_partials(const double *coarse, const double *fine, int D, const int *N,
                                        double *partials, int nblocks, void *stream) {
    if (D < 1 || D > 4 || nblocks < 1) return set_error(VPFV_EARG, "richardson: bad arguments");
    Dims4 g{};
    g.D = D;
    long long total = 1, sa = 1, sb = 1;
    for (int k = D - 1; k >= 0; --k) {
        g.n[k] = N[k];
        g.sa[k] = sa;
        g.sb[k] = sb;
        sa *= N[k] + 2 * NG;
        sb *= 2 * N[k] + 2 * NG;
        total *= N[k];
    }
    richardson_kernel<<<nblocks, 256, 0, (cudaStream_t)stream>>>(coarse, fine, g, total, partials);
    return check_launch("richardson");
}
