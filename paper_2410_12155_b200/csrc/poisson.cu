// Spectral periodic Poisson solve and field reconstruction (fields.py:172-213).
//
//   rho_hat = FFT(rho);  phi_hat = rho_hat / |k|^2 (k != 0), phi_hat_0 = 0
//   E_hat_d = -i kd_d phi_hat   (kd: Nyquist entry zeroed for even N)
//   E_d = Re IFFT(E_hat_d)
//
// Hand-written fp64 transforms in shared memory: radix-2 decimation-in-time
// for power-of-two lines, a direct O(N^2) DFT with exact (k*n mod N) twiddle
// indices otherwise.  Twiddles exp(-2 pi i m/N) and the wavenumber tables are
// built on the host with numpy (bitwise the reference's k arrays).
// 1D: one CTA does the whole solve.  2D: row pass -> column pass (with the
// spectral multiply and both inverse column transforms) -> inverse row pass.
#include "common.cuh"
#include "field.cuh"

namespace vpfv {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// In-place transform of n complex values held in smem `a` by the whole CTA.
// pow2: `a` must already be in bit-reversed order.  Otherwise `tmp` holds the
// natural-order input and the DFT result is written to `a`.
__device__ void line_transform(double2 *a, double2 *tmp, int n, const double2 *__restrict__ tw,
                               bool inverse, bool pow2) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (pow2) {
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1, step = n / len;
            for (int j = tid; j < (n >> 1); j += nt) {
                const int grp = j / half, pos = j - grp * half;
                const int i1 = grp * len + pos, i2 = i1 + half;
                double2 w = tw[pos * step];
                if (inverse) w.y = -w.y;
                double2 t = cmul(w, a[i2]);
                double2 x = a[i1];
                a[i1] = make_double2(x.x + t.x, x.y + t.y);
                a[i2] = make_double2(x.x - t.x, x.y - t.y);
            }
            __syncthreads();
        }
    } else {
        for (int k = tid; k < n; k += nt) {
            double2 acc = make_double2(0.0, 0.0);
            long long idx = 0;
            for (int m = 0; m < n; ++m) {
                double2 w = tw[idx];
                if (inverse) w.y = -w.y;
                double2 t = cmul(w, tmp[m]);
                acc.x += t.x;
                acc.y += t.y;
                idx += k;
                if (idx >= n) idx -= n;
            }
            a[k] = acc;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int bitrev(int x, int logn) { return (int)(__brev((unsigned)x) >> (32 - logn)); }

// store natural-order value v for position m into the transform input
__device__ __forceinline__ void put(double2 *a, double2 *tmp, int m, double2 v, bool pow2, int logn) {
    if (pow2) a[bitrev(m, logn)] = v;
    else tmp[m] = v;
}

// ---------------------------------------------------------------------------
// 1D: single CTA

// the 1D solve by one CTA; sm2 holds 3 n double2
__device__ void poisson1d_block(const double *__restrict__ rho, double *__restrict__ Ex, double *__restrict__ phi,
                                int n, const double2 *__restrict__ tw, const double *__restrict__ k2,
                                const double *__restrict__ kd, int pow2, int logn, double2 *sm2) {
    double2 *a = sm2, *tmp = sm2 + n, *ph = sm2 + 2 * n;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int m = tid; m < n; m += nt) put(a, tmp, m, make_double2(rho[m], 0.0), pow2, logn);
    __syncthreads();
    line_transform(a, tmp, n, tw, false, pow2);
    // phi_hat and E_hat (E_hat = -i kd phi_hat = (kd*ph.y, -kd*ph.x))
    for (int k = tid; k < n; k += nt) {
        double2 p = make_double2(0.0, 0.0);
        if (k > 0) p = make_double2(a[k].x / k2[k], a[k].y / k2[k]);
        ph[k] = p;
    }
    __syncthreads();
    for (int pass = (phi ? 0 : 1); pass < 2; ++pass) {
        for (int k = tid; k < n; k += nt) {
            double2 v = ph[k];
            if (pass == 1) v = make_double2(kd[k] * v.y, -(kd[k] * v.x));
            put(a, tmp, k, v, pow2, logn);
        }
        __syncthreads();
        line_transform(a, tmp, n, tw, true, pow2);
        const double inv = 1.0 / (double)n;
        double *out = pass == 0 ? phi : Ex;
        for (int m = tid; m < n; m += nt) out[m] = a[m].x * inv;
        __syncthreads();
    }
}

__global__ void poisson1d_kernel(const double *__restrict__ rho, double *__restrict__ Ex,
                                 double *__restrict__ phi, int n, const double2 *__restrict__ tw,
                                 const double *__restrict__ k2, const double *__restrict__ kd,
                                 int pow2, int logn) {
    extern __shared__ double2 sm2[];
    poisson1d_block(rho, Ex, phi, n, tw, k2, kd, pow2, logn, sm2);
}

// The whole 1D field chain of a stage in one CTA (the per-stage
// "moments -> charge -> Poisson -> tables" of Simulation._stage,
// runner.py:183-191): rho from the species densities, the spectral solve,
// then every species' line tables (plain e/c1 or the packed rows of the
// tiled 1D-2V kernel) -- bitwise the separate charge / Poisson / tables
// kernels, whose block-level code it shares (field.cuh).
struct Tables1D {
    int ns;
    const double *part[8];  // moment partials [Nx][rows][chunks] of each species, or none (n given)
    int rows[8], chunks[8];
    double vol[8];
    double *e[8], *c1[8], *packed[8];
    double qmk2[8], g[8], t1[8], den1[8];
    int corrections[8];
};

__global__ void field1d_kernel(double *__restrict__ n, Charges q, int ns, int nx, double *__restrict__ rho,
                               double *__restrict__ Ex, const double2 *__restrict__ tw,
                               const double *__restrict__ k2, const double *__restrict__ kd, int pow2, int logn,
                               Tables1D T) {
    extern __shared__ double2 sm2[];
    if (T.part[0]) {  // n_s from the last stage's fused moment partials (vpfv_moment_partials)
        const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int s = 0; s < T.ns; ++s) {
            if (T.rows[s] == 1) {  // 1D-1V: one thread per cell folds its chunks
                for (int p = threadIdx.x; p < nx; p += blockDim.x) {
                    double tmp[16];
                    for (int t = 0; t < T.chunks[s]; ++t) tmp[t] = T.part[s][(size_t)p * T.chunks[s] + t];
                    n[(size_t)s * nx + p] = __dmul_rn(fold_small(tmp, T.chunks[s]), T.vol[s]);
                }
                continue;
            }
            double *bufA = reinterpret_cast<double *>(sm2) + (size_t)warp * 2 * T.rows[s];
            for (int p = warp; p < nx; p += nw) {
                const double x = moment_cell_warp(T.part[s] + (size_t)p * T.rows[s] * T.chunks[s], T.rows[s],
                                                  T.chunks[s], bufA, bufA + T.rows[s]);
                if ((threadIdx.x & 31) == 0) n[(size_t)s * nx + p] = __dmul_rn(x, T.vol[s]);
            }
        }
        __syncthreads();
    }
    double *part = reinterpret_cast<double *>(sm2 + 3 * nx);
    charge_block(n, q, ns, nx, rho, part);
    __syncthreads();
    poisson1d_block(rho, Ex, nullptr, nx, tw, k2, kd, pow2, logn, sm2);
    for (int s = 0; s < T.ns; ++s) {
        if (T.packed[s]) {
            for (int r = threadIdx.x; r < nx + 2; r += blockDim.x) {  // rows shifted by one, periodic ghosts
                const int i = r == 0 ? nx - 1 : (r == nx + 1 ? 0 : r - 1);
                double *o = T.packed[s] + (size_t)r * 8;
                double e, c1;
                table1d_row(Ex, i, nx, T.qmk2[s], T.g[s], T.t1[s], T.den1[s], e, c1);
                o[0] = e;
                o[1] = T.corrections[s] ? c1 : 0.0;
                for (int k = 2; k < 8; ++k) o[k] = 0.0;
            }
        } else {
            for (int i = threadIdx.x; i < nx; i += blockDim.x) {
                double e, c1;
                table1d_row(Ex, i, nx, T.qmk2[s], T.g[s], T.t1[s], T.den1[s], e, c1);
                T.e[s][i] = e;
                T.c1[s][i] = T.corrections[s] ? c1 : 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 2D: three passes over lines

// forward row transforms: C[i, :] = FFT_y(rho[i, :])
__global__ void rows_fwd_kernel(const double *__restrict__ rho, double2 *__restrict__ C, int nx,
                                int ny, const double2 *__restrict__ twy, int pow2, int logn) {
    extern __shared__ double2 sm2[];
    double2 *a = sm2, *tmp = sm2 + ny;
    const int i = blockIdx.x;
    for (int m = threadIdx.x; m < ny; m += blockDim.x)
        put(a, tmp, m, make_double2(rho[(long long)i * ny + m], 0.0), pow2, logn);
    __syncthreads();
    line_transform(a, tmp, ny, twy, false, pow2);
    for (int m = threadIdx.x; m < ny; m += blockDim.x) C[(long long)i * ny + m] = a[m];
}

// column pass: FFT_x, spectral multiply, inverse FFT_x for each requested
// output; D[o][:, j] (o = 0: Ex, 1: Ey, 2: phi) scaled by 1/nx.
__global__ void cols_kernel(const double2 *__restrict__ C, double2 *__restrict__ D, int nx, int ny,
                            const double2 *__restrict__ twx, const double *__restrict__ kx,
                            const double *__restrict__ ky, const double *__restrict__ kxd,
                            const double *__restrict__ kyd, int nout, int pow2, int logn) {
    extern __shared__ double2 sm2[];
    double2 *a = sm2, *tmp = sm2 + nx, *ph = sm2 + 2 * nx;
    const int j = blockIdx.x;
    const long long plane = (long long)nx * ny;
    for (int m = threadIdx.x; m < nx; m += blockDim.x)
        put(a, tmp, m, C[(long long)m * ny + j], pow2, logn);
    __syncthreads();
    line_transform(a, tmp, nx, twx, false, pow2);
    const double kyj = ky[j];
    for (int m = threadIdx.x; m < nx; m += blockDim.x) {
        const double kk = kx[m] * kx[m] + kyj * kyj;
        ph[m] = kk > 0.0 ? make_double2(a[m].x / kk, a[m].y / kk) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double inv = 1.0 / (double)nx;
    for (int o = 0; o < nout; ++o) {
        for (int m = threadIdx.x; m < nx; m += blockDim.x) {
            double2 v = ph[m];
            if (o < 2) {
                const double kd = (o == 0) ? kxd[m] : kyd[j];
                v = make_double2(kd * v.y, -(kd * v.x));
            }
            put(a, tmp, m, v, pow2, logn);
        }
        __syncthreads();
        line_transform(a, tmp, nx, twx, true, pow2);
        for (int m = threadIdx.x; m < nx; m += blockDim.x)
            D[o * plane + (long long)m * ny + j] = make_double2(a[m].x * inv, a[m].y * inv);
        __syncthreads();
    }
}

// inverse row transforms: out_o[i, :] = Re IFFT_y(D[o][i, :])
__global__ void rows_inv_kernel(const double2 *__restrict__ D, double *__restrict__ Ex,
                                double *__restrict__ Ey, double *__restrict__ phi, int nx, int ny,
                                const double2 *__restrict__ twy, int nout, int pow2, int logn) {
    extern __shared__ double2 sm2[];
    double2 *a = sm2, *tmp = sm2 + ny;
    const int i = blockIdx.x;
    const long long plane = (long long)nx * ny;
    const double inv = 1.0 / (double)ny;
    for (int o = 0; o < nout; ++o) {
        for (int m = threadIdx.x; m < ny; m += blockDim.x)
            put(a, tmp, m, D[o * plane + (long long)i * ny + m], pow2, logn);
        __syncthreads();
        line_transform(a, tmp, ny, twy, true, pow2);
        double *out = o == 0 ? Ex : (o == 1 ? Ey : phi);
        for (int m = threadIdx.x; m < ny; m += blockDim.x) out[(long long)i * ny + m] = a[m].x * inv;
        __syncthreads();
    }
}

static int ilog2_if_pow2(int n) {
    if (n <= 0 || (n & (n - 1))) return -1;
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}

static void allow_smem(const void *fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_poisson_1d(const double *rho, double *Ex, double *phi, int N, const double *tw,
                               const double *k2, const double *kd, void *stream) {
    if (N < 2) return set_error(VPFV_EARG, "poisson_1d: N < 2");
    const int logn = ilog2_if_pow2(N);
    size_t smem = sizeof(double2) * 3 * (size_t)N;
    if (smem > 200 * 1024) return set_error(VPFV_EARG, "poisson_1d: N too large for one CTA");
    static bool once = false;
    if (!once) {
        allow_smem((const void *)poisson1d_kernel);
        once = true;
    }
    poisson1d_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(
        rho, Ex, phi, N, (const double2 *)tw, k2, kd, logn >= 0, logn < 0 ? 0 : logn);
    return check_launch("poisson_1d");
}

extern "C" int vpfv_field_1d(const double *const *partials, const int *rows, const int *chunks, const double *vols,
                             double *n, const double *q_host, int nspecies, int Nx, double *rho, double *Ex,
                             const double *tw, const double *k2, const double *kd, double *const *e,
                             double *const *c1, double *const *packed, const double *qmk2, const double *g,
                             const double *t1, const double *den1, const int *corrections, void *stream) {
    if (nspecies < 1 || nspecies > 8) return set_error(VPFV_EARG, "field_1d: 1..8 species");
    if (Nx < 2) return set_error(VPFV_EARG, "field_1d: Nx < 2");
    const int logn = ilog2_if_pow2(Nx);
    size_t smem = sizeof(double2) * 3 * (size_t)Nx + sizeof(double) * 1024;
    for (int s = 0; partials && s < nspecies; ++s) {
        if (!partials[s] || rows[s] < 1 || chunks[s] < 1 || chunks[s] > 16)
            return set_error(VPFV_EARG, "field_1d: bad moment partials");
        const size_t fin = sizeof(double) * 32 * 2 * (size_t)rows[s];
        if (fin > smem) smem = fin;
    }
    if (smem > 200 * 1024) return set_error(VPFV_EARG, "field_1d: Nx too large for one CTA");
    static bool once = false;
    if (!once) {
        allow_smem((const void *)field1d_kernel);
        once = true;
    }
    Charges q;
    Tables1D T{};
    T.ns = nspecies;
    for (int s = 0; s < 8; ++s) q.q[s] = s < nspecies ? q_host[s] : 0.0;
    for (int s = 0; s < nspecies; ++s) {
        T.part[s] = partials ? partials[s] : nullptr;
        T.rows[s] = partials ? rows[s] : 0;
        T.chunks[s] = partials ? chunks[s] : 0;
        T.vol[s] = partials ? vols[s] : 0.0;
        T.e[s] = e ? e[s] : nullptr;
        T.c1[s] = c1 ? c1[s] : nullptr;
        T.packed[s] = packed ? packed[s] : nullptr;
        T.qmk2[s] = qmk2[s];
        T.g[s] = g[s];
        T.t1[s] = t1[s];
        T.den1[s] = den1[s];
        T.corrections[s] = corrections[s];
        if (!T.packed[s] && !(T.e[s] && T.c1[s])) return set_error(VPFV_EARG, "field_1d: no table outputs");
    }
    field1d_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(n, q, nspecies, Nx, rho, Ex, (const double2 *)tw, k2,
                                                           kd, logn >= 0, logn < 0 ? 0 : logn, T);
    return check_launch("field_1d");
}

extern "C" int vpfv_poisson_2d(const double *rho, double *Ex, double *Ey, double *phi, int Nx,
                               int Ny, const double *twx, const double *twy, const double *kx,
                               const double *ky, const double *kxd, const double *kyd,
                               double *scratch, void *stream) {
    if (Nx < 2 || Ny < 2) return set_error(VPFV_EARG, "poisson_2d: extents < 2");
    const int lx = ilog2_if_pow2(Nx), ly = ilog2_if_pow2(Ny);
    size_t smx = sizeof(double2) * 3 * (size_t)Nx, smy = sizeof(double2) * 2 * (size_t)Ny;
    if (smx > 200 * 1024 || smy > 200 * 1024) return set_error(VPFV_EARG, "poisson_2d: too large");
    static bool once = false;
    if (!once) {
        allow_smem((const void *)rows_fwd_kernel);
        allow_smem((const void *)cols_kernel);
        allow_smem((const void *)rows_inv_kernel);
        once = true;
    }
    cudaStream_t s = (cudaStream_t)stream;
    double2 *C = (double2 *)scratch;
    double2 *D = C + (size_t)Nx * Ny;  // up to 3 planes follow... reuse C's plane for phi
    const int nout = phi ? 3 : 2;
    // D needs nout planes; scratch holds 1 + 3 planes when phi is requested
    rows_fwd_kernel<<<Nx, 256, smy, s>>>(rho, C, Nx, Ny, (const double2 *)twy, ly >= 0, ly < 0 ? 0 : ly);
    cols_kernel<<<Ny, 256, smx, s>>>(C, D, Nx, Ny, (const double2 *)twx, kx, ky, kxd, kyd, nout,
                                     lx >= 0, lx < 0 ? 0 : lx);
    rows_inv_kernel<<<Nx, 256, smy, s>>>(D, Ex, Ey, phi, Nx, Ny, (const double2 *)twy, nout,
                                         ly >= 0, ly < 0 ? 0 : ly);
    return check_launch("poisson_2d");
}
