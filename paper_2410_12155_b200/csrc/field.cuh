// Block-level pieces of the per-stage field chain shared by the separate
// kernels (aux.cu) and the fused 1D field kernel (poisson.cu), so both give
// bitwise the same charge density and tables.
#pragma once
#include "common.cuh"

namespace vpfv {

struct Charges {
    double q[8];
};

// moment from partials: per physical cell, fold over the vy chunks of every
// vx row (chunk sums are exact subtrees), then over vx -- the adjacent-pair
// tree of the reference's fold (fields.py:96-128).
__device__ __forceinline__ double fold_small(double *x, int n) {  // single thread, in place
    while (n > 1) {
        int m = n >> 1;
        for (int t = 0; t < m; ++t) x[t] = __dadd_rn(x[2 * t], x[2 * t + 1]);
        if (n & 1) {
            x[m] = x[n - 1];
            n = m + 1;
        } else {
            n = m;
        }
    }
    return x[0];
}

// fold_small of C = 2^k contiguous values in registers (128-bit loads):
// the same adjacent-pair tree
template <int C>
__device__ __forceinline__ double fold_pow2(const double *__restrict__ src) {
    double x[C];
    if (C == 1) {
        x[0] = src[0];
    } else {
#pragma unroll
        for (int t = 0; t < C; t += 2) {
            const double2 d = *reinterpret_cast<const double2 *>(src + t);
            x[t] = d.x;
            x[t + 1] = d.y;
        }
    }
#pragma unroll
    for (int w = 1; w < C; w <<= 1)
#pragma unroll
        for (int t = 0; t < C; t += 2 * w) x[t] = __dadd_rn(x[t], x[t + w]);
    return x[0];
}

// fold_small of one row of c (<= 16) chunks; src 16-byte aligned when c is even
__device__ __forceinline__ double fold_row(const double *__restrict__ src, int c) {
    switch (c) {
        case 1: return fold_pow2<1>(src);
        case 2: return fold_pow2<2>(src);
        case 4: return fold_pow2<4>(src);
        case 8: return fold_pow2<8>(src);
        case 16: return fold_pow2<16>(src);
        default: {
            double tmp[16];
            for (int t = 0; t < c; ++t) tmp[t] = src[t];
            return fold_small(tmp, c);
        }
    }
}

// one warp folds one physical cell's partials [nvx][nlt] (nlt <= 16) through
// two smem buffers of nvx doubles; the sum is valid in every lane
__device__ __forceinline__ double moment_cell_warp(const double *__restrict__ src, int nvx, int nlt, double *bufA,
                                                   double *bufB) {
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < nvx; k += 32) {
        double tmp[16];
        for (int t = 0; t < nlt; ++t) tmp[t] = src[(size_t)k * nlt + t];
        bufA[k] = fold_small(tmp, nlt);
    }
    __syncwarp();
    int len = nvx;
    double *a = bufA, *b = bufB;
    while (len > 1) {
        const int m = len >> 1;
        for (int t = lane; t < m; t += 32) b[t] = __dadd_rn(a[2 * t], a[2 * t + 1]);
        if ((len & 1) && lane == 0) b[m] = a[len - 1];
        __syncwarp();
        len = m + (len & 1);
        double *tmp = a;
        a = b;
        b = tmp;
    }
    const double r = a[0];
    __syncwarp();  // the buffers may be reused by the caller's next cell
    return r;
}

// Sum of one value per thread over the CTA by the adjacent-pair tree over
// thread indices (level w adds thread t+w into t for t % 2w == 0, t+w < nt):
// levels 1..16 by shuffles inside each warp, the rest over the warp sums by
// warp 0 -- bitwise the smem tree.  blockDim.x a multiple of 32; red: 32
// doubles of smem.  The result is valid in every thread.
__device__ __forceinline__ double block_tree_sum(double x, double *red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int w = 1; w < 32; w <<= 1) {
        const double y = __shfl_down_sync(0xffffffffu, x, w);
        if ((lane & (2 * w - 1)) == 0) x = __dadd_rn(x, y);
    }
    if (lane == 0) red[warp] = x;
    __syncthreads();
    if (warp == 0) {
        x = lane < nw ? red[lane] : 0.0;
#pragma unroll
        for (int w = 1; w < 32; w <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, x, w);
            if ((lane & (2 * w - 1)) == 0 && lane + w < nw) x = __dadd_rn(x, y);
        }
        if (lane == 0) red[0] = x;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();  // red may be reused
    return r;
}

// rho = sum_s q_s n_s - mean(rho) over nphys cells by one CTA: fixed-order
// per-thread partials, then the adjacent-pair tree over the threads
// (charge_density, fields.py:164-169).  red: 32 doubles of smem.
__device__ __forceinline__ void charge_block(const double *__restrict__ n, const Charges &q, int ns, int nphys,
                                             double *__restrict__ rho, double *red) {
    const int tid = threadIdx.x, nt = blockDim.x;
    double acc = 0.0;
    for (int p = tid; p < nphys; p += nt) {
        double r = __dmul_rn(q.q[0], n[p]);
        for (int s = 1; s < ns; ++s) r = __dadd_rn(r, __dmul_rn(q.q[s], n[(long long)s * nphys + p]));
        rho[p] = r;
        acc = __dadd_rn(acc, r);
    }
    const double mean = __ddiv_rn(block_tree_sum(acc, red), (double)nphys);
    for (int p = tid; p < nphys; p += nt) rho[p] = __dsub_rn(rho[p], mean);
}

// 1D line tables of row i (the dispatcher's arithmetic, _kernels.py:330-349;
// correction_coeffs c1, fvm.py:168-201): e = qm k^2 E + g,
// c1 = t1 + qm k^2 (E[i+1] - E[i-1]) / den1 (periodic).
__device__ __forceinline__ void table1d_row(const double *__restrict__ E, int i, int n, double qmk2, double g,
                                            double t1, double den1, double &e, double &c1) {
    const double dE = __dsub_rn(E[i + 1 < n ? i + 1 : 0], E[i > 0 ? i - 1 : n - 1]);
    e = __dadd_rn(__dmul_rn(qmk2, E[i]), g);
    c1 = __dadd_rn(t1, __ddiv_rn(__dmul_rn(qmk2, dE), den1));
}

}  // namespace vpfv
