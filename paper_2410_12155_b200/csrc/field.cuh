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

// rho = sum_s q_s n_s - mean(rho) over nphys cells by one CTA: fixed-order
// per-thread partials, then an adjacent-pair tree over the threads
// (charge_density, fields.py:164-169).  part: blockDim.x doubles of smem.
__device__ __forceinline__ void charge_block(const double *__restrict__ n, const Charges &q, int ns, int nphys,
                                             double *__restrict__ rho, double *part) {
    const int tid = threadIdx.x, nt = blockDim.x;
    double acc = 0.0;
    for (int p = tid; p < nphys; p += nt) {
        double r = __dmul_rn(q.q[0], n[p]);
        for (int s = 1; s < ns; ++s) r = __dadd_rn(r, __dmul_rn(q.q[s], n[(long long)s * nphys + p]));
        rho[p] = r;
        acc = __dadd_rn(acc, r);
    }
    part[tid] = acc;
    __syncthreads();
    for (int w = 1; w < nt; w <<= 1) {
        if ((tid % (2 * w)) == 0 && tid + w < nt) part[tid] = __dadd_rn(part[tid], part[tid + w]);
        __syncthreads();
    }
    const double mean = __ddiv_rn(part[0], (double)nphys);
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
