// Zeroth velocity moment with the reference's deterministic fold tree.
//
// n[p] = fold_tree(f[p, velocity block]) * prod(h_v)   (fields.py:28-47, 86-111)
//
// The tree folds the fastest velocity axis first (adjacent pairs, odd tail
// carried), then the next axis.  For a power-of-two row the first five tree
// levels are exactly a warp shuffle-down reduction with ASCENDING offsets
// 1,2,4,8,16 when lane l holds element 32c+l (lane 0 ends with the subtree of
// chunk c); the chunk sums then finish the tree the same way.  Any other row
// length runs the literal round-by-round fold in shared memory.  Either way
// the result is bitwise the reference's (floating-point addition is
// commutative, and the association is the tree's).
#include "common.cuh"

namespace vpfv {

__device__ __forceinline__ bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// tree over 32 lanes (lane l holds element l); result valid in lane 0
__device__ __forceinline__ double warp_tree(double x, int width) {
    for (int off = 1; off < width; off <<= 1) {
        double y = __shfl_down_sync(0xffffffffu, x, off);
        x = __dadd_rn(x, y);
    }
    return x;
}

// Fold n values (global or shared, stride 1) with one warp.  pow2 && n >= 32
// uses shuffles; otherwise ping-pong buffers bufA/bufB (n doubles each).
__device__ double warp_fold(const double *x, int n, double *bufA, double *bufB, int lane) {
    if (is_pow2(n) && n >= 32) {
        const int nch = n >> 5;
        double chunk_sum = 0.0;
        // chunk sums, one per chunk, collected into lanes 0..nch-1 (nch <= 32)
        // or folded sequentially in tree order when nch > 32.
        if (nch <= 32) {
            double mine = 0.0;
            for (int c = 0; c < nch; ++c) {
                double s = warp_tree(x[c * 32 + lane], 32);
                s = __shfl_sync(0xffffffffu, s, 0);
                if (lane == c) mine = s;
            }
            chunk_sum = warp_tree(mine, nch);
            return __shfl_sync(0xffffffffu, chunk_sum, 0);
        }
        // very long rows: chunk sums to smem, then ping-pong (nch is pow2)
        for (int c = 0; c < nch; ++c) {
            double s = warp_tree(x[c * 32 + lane], 32);
            if (lane == 0) bufA[c] = s;
        }
        __syncwarp();
        n = nch;
        x = bufA;
    } else {
        for (int t = lane; t < n; t += 32) bufA[t] = x[t];
        __syncwarp();
        x = bufA;
    }
    double *src = bufA, *dst = bufB;
    while (n > 1) {
        int m = n >> 1;
        for (int t = lane; t < m; t += 32) dst[t] = __dadd_rn(src[2 * t], src[2 * t + 1]);
        if ((n & 1) && lane == 0) dst[m] = src[n - 1];
        __syncwarp();
        n = m + (n & 1);
        double *tmp = src;
        src = dst;
        dst = tmp;
    }
    return src[0];
}

// one CTA per physical cell; warps take outer-velocity rows
__global__ void moment_kernel(const double *__restrict__ f, double *__restrict__ n, int nphys,
                              int ny /* 2nd physical extent or 1 */, long long Pvel,
                              long long s_row, int nv1, int nv2, long long off_v, double vol,
                              int d, long long Py_pad, int nbuf) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    double *rows = sm;                        // nv1
    double *buf = sm + ((nv1 + 1) & ~1);      // per warp 2*nv2
    double *bufA = buf + (size_t)warp * 2 * nbuf, *bufB = bufA + nbuf;
    for (int p = blockIdx.x; p < nphys; p += gridDim.x) {
        long long base;
        if (d == 1) {
            base = (long long)(p + NG) * Pvel;
        } else {
            int ix = p / ny, iy = p - ix * ny;
            base = ((long long)(ix + NG) * Py_pad + (iy + NG)) * Pvel;
        }
        for (int a = warp; a < nv1; a += nwarps) {
            const double *row = f + base + off_v + (long long)a * s_row + NG;
            double s = warp_fold(row, nv2, bufA, bufB, lane);
            if (lane == 0) rows[a] = s;
            __syncwarp();
        }
        __syncthreads();
        if (warp == 0) {
            double tot = (nv1 == 1) ? rows[0] : warp_fold(rows, nv1, bufA, bufB, lane);
            if (lane == 0) n[p] = __dmul_rn(tot, vol);
        }
        __syncthreads();
    }
}

struct Dims4 {
    int n[4];
};

// Fused-moment partials straight from f (the layout the tiled stage kernels'
// epilogues write: the first four fold-tree levels over every aligned 16-wide
// vy chunk of every interior velocity row).  Used when f was edited in place
// on one rank of a peer-mode run, so every rank keeps the same density path.
__global__ void chunk_partials_kernel(const double *__restrict__ f, double *__restrict__ part, int ndim, Dims4 N,
                                      long long nrows, int nch) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= nrows * nch) return;
    const int c = (int)(t % nch);
    long long r = t / nch, off = 0;
    // padded offset of interior row r (dims 0 .. ndim-2), vy handled below
    long long st[4];
    st[ndim - 1] = 1;
    for (int k = ndim - 2; k >= 0; --k) st[k] = st[k + 1] * (N.n[k + 1] + 2 * NG);
    for (int k = ndim - 2; k >= 0; --k) {
        const long long i = r % N.n[k];
        r /= N.n[k];
        off += (i + NG) * st[k];
    }
    const double *x = f + off + NG + 16 * c;
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = x[i];
#pragma unroll
    for (int w = 1; w < 16; w <<= 1)
#pragma unroll
        for (int i = 0; i < 16; i += 2 * w) a[i] = __dadd_rn(a[i], a[i + w]);
    part[t] = a[0];
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_moment(const double *f, double *n, int d, int v, const int *N, double vol,
                           void *stream) {
    if (d < 1 || d > 2 || v < d || d + v > 4) return set_error(VPFV_EDIM, "unsupported (d, v)");
    int nphys = 1;
    for (int k = 0; k < d; ++k) nphys *= N[k];
    const int nv1 = (v == 2) ? N[d] : 1, nv2 = N[d + v - 1];
    long long Pvel = 1;
    for (int k = d; k < d + v; ++k) Pvel *= (N[k] + 2 * NG);
    const long long s_row = (v == 2) ? (N[d + 1] + 2 * NG) : 0;
    const long long off_v = (v == 2) ? (long long)NG * s_row : 0;
    const int ny = (d == 2) ? N[1] : 1;
    const long long Py_pad = (d == 2) ? (N[1] + 2 * NG) : 1;
    int warps = nv1 < 8 ? nv1 : 8;
    const int nbuf = nv1 > nv2 ? nv1 : nv2;
    size_t smem = sizeof(double) * ((size_t)((nv1 + 1) & ~1) + (size_t)warps * 2 * nbuf);
    if (smem > 200 * 1024) return set_error(VPFV_EARG, "velocity extent too large for moment");
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(moment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    int grid = nphys < 65535 ? nphys : 65535;
    moment_kernel<<<grid, warps * 32, smem, (cudaStream_t)stream>>>(
        f, n, nphys, ny, Pvel, s_row, nv1, nv2, off_v, vol, d, Py_pad, nbuf);
    return check_launch("moment");
}

// ---------------------------------------------------------------------------
// schedule="position-major": the reference's compiled per-cell sequential sum
// (fields.py:50-83, _seq_moment_{2,3,4}d): s = 0; s += f[v] over the velocity
// interior in C order; n = s * vol.  One warp per physical cell: the lanes load
// 32 consecutive values of a velocity row (coalesced) and every lane adds them
// in index order from shuffles, so the association is the reference's.
namespace vpfv {
__global__ void moment_seq_kernel(const double *__restrict__ f, double *__restrict__ n, int nphys, int ny,
                                  long long Pvel, long long s_row, int nv1, int nv2, long long off_v, double vol,
                                  int d, long long Py_pad) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nphys) return;
    long long base;
    if (d == 1) {
        base = (long long)(warp + NG) * Pvel;
    } else {
        const int ix = warp / ny, iy = warp - ix * ny;
        base = ((long long)(ix + NG) * Py_pad + (iy + NG)) * Pvel;
    }
    double s = 0.0;
    for (int a = 0; a < nv1; ++a) {
        const double *row = f + base + off_v + (long long)a * s_row + NG;
        for (int c = 0; c < nv2; c += 32) {
            const int m = min(32, nv2 - c);
            const double x = lane < m ? row[c + lane] : 0.0;
            for (int j = 0; j < m; ++j) s = __dadd_rn(s, __shfl_sync(0xffffffffu, x, j));
        }
    }
    if (lane == 0) n[warp] = __dmul_rn(s, vol);
}
}  // namespace vpfv

extern "C" int vpfv_moment_seq(const double *f, double *n, int d, int v, const int *N, double vol,
                               void *stream) {
    if (d < 1 || d > 2 || v < d || d + v > 4) return set_error(VPFV_EDIM, "unsupported (d, v)");
    int nphys = 1;
    for (int k = 0; k < d; ++k) nphys *= N[k];
    const int nv1 = (v == 2) ? N[d] : 1, nv2 = N[d + v - 1];
    long long Pvel = 1;
    for (int k = d; k < d + v; ++k) Pvel *= (N[k] + 2 * NG);
    const long long s_row = (v == 2) ? (N[d + 1] + 2 * NG) : 0;
    const long long off_v = (v == 2) ? (long long)NG * s_row : 0;
    const int ny = (d == 2) ? N[1] : 1;
    const long long Py_pad = (d == 2) ? (N[1] + 2 * NG) : 1;
    const int threads = 256, grid = (nphys * 32 + threads - 1) / threads;
    moment_seq_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(f, n, nphys, ny, Pvel, s_row, nv1, nv2, off_v,
                                                                   vol, d, Py_pad);
    return check_launch("moment_seq");
}

extern "C" int vpfv_moment_chunk_partials(const double *f, double *part, int ndim, const int *N, void *stream) {
    if (ndim < 2 || ndim > 4 || N[ndim - 1] % 16) return set_error(VPFV_EARG, "chunk_partials: vy extent must be a multiple of 16");
    Dims4 D{};
    long long rows = 1;
    for (int k = 0; k < ndim; ++k) D.n[k] = N[k];
    for (int k = 0; k < ndim - 1; ++k) rows *= N[k];
    const int nch = N[ndim - 1] / 16;
    const long long n = rows * nch;
    chunk_partials_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(f, part, ndim, D, rows, nch);
    return check_launch("moment_chunk_partials");
}
