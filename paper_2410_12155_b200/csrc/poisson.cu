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

#ifdef VPFV_FIELD_PROBE
__device__ unsigned long long g_field_probe[16];
#define FIELD_STAMP(k)                                                                  \
    do {                                                                                \
        if (threadIdx.x == 0) {                                                         \
            unsigned long long t_;                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                      \
            g_field_probe[k] = t_;                                                      \
        }                                                                               \
    } while (0)
#else
#define FIELD_STAMP(k) \
    do {               \
    } while (0)
#endif

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
        // two radix-2 stages (len, 2 len) per pass: one thread carries the 4
        // points they couple through both -- the same butterflies and
        // twiddles as stage-by-stage, with half the barriers
        const int logn = 31 - __clz(n);
        int lg = 1;  // log2 of the current stage length
        for (; lg + 1 <= logn; lg += 2) {
            const int lh = lg - 1, half = 1 << lh;  // stage len = 2 half; next stage len = 4 half
            for (int j = tid; j < (n >> 2); j += nt) {
                const int grp = j >> lh, pos = j & (half - 1);
                const int i0 = (grp << (lh + 2)) + pos;
                double2 w1 = tw[pos << (logn - lg)];               // w_len^pos
                double2 w2 = tw[pos << (logn - lg - 1)];           // w_{2len}^pos
                double2 w3 = tw[(pos + half) << (logn - lg - 1)];  // w_{2len}^{pos+half}
                if (inverse) {
                    w1.y = -w1.y;
                    w2.y = -w2.y;
                    w3.y = -w3.y;
                }
                double2 x0 = a[i0], x1 = a[i0 + half], x2 = a[i0 + 2 * half], x3 = a[i0 + 3 * half];
                double2 t = cmul(w1, x1);
                double2 y0 = make_double2(x0.x + t.x, x0.y + t.y), y1 = make_double2(x0.x - t.x, x0.y - t.y);
                t = cmul(w1, x3);
                double2 y2 = make_double2(x2.x + t.x, x2.y + t.y), y3 = make_double2(x2.x - t.x, x2.y - t.y);
                t = cmul(w2, y2);
                a[i0] = make_double2(y0.x + t.x, y0.y + t.y);
                a[i0 + 2 * half] = make_double2(y0.x - t.x, y0.y - t.y);
                t = cmul(w3, y3);
                a[i0 + half] = make_double2(y1.x + t.x, y1.y + t.y);
                a[i0 + 3 * half] = make_double2(y1.x - t.x, y1.y - t.y);
            }
            __syncthreads();
        }
        if (lg == logn) {  // odd log2 n: the last radix-2 stage
            const int lh = lg - 1, half = 1 << lh;
            for (int j = tid; j < (n >> 1); j += nt) {
                const int grp = j >> lh, pos = j & (half - 1);
                const int i1 = (grp << lg) + pos, i2 = i1 + half;
                double2 w = tw[pos << (logn - lg)];
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

// Shared-memory layout of the 1D solve (double2 units): a[n], tmp[n], ph[n],
// then the staged spectral tables tw[n] (double2) and k2[n], kd[n] (double).
// Staging them once replaces an L1/L2 round trip per butterfly stage.
__host__ __device__ inline size_t poisson1d_smem(int n, bool staged) {
    return sizeof(double2) * 3 * (size_t)n + (staged ? (sizeof(double2) + 2 * sizeof(double)) * (size_t)n : 0);
}

struct Spectral1D {
    const double2 *tw;
    const double *k2, *kd;
};

__device__ __forceinline__ Spectral1D stage_spectral(const double2 *__restrict__ tw, const double *__restrict__ k2,
                                                     const double *__restrict__ kd, int n, double2 *sm2) {
    double2 *tws = sm2 + 3 * n;
    double *k2s = reinterpret_cast<double *>(tws + n), *kds = k2s + n;
    for (int m = threadIdx.x; m < n; m += blockDim.x) {
        tws[m] = tw[m];
        k2s[m] = k2[m];
        kds[m] = kd[m];
    }
    return Spectral1D{tws, k2s, kds};  // visible after the caller's next __syncthreads
}

// the 1D solve by one CTA on a[] already holding the (bit-reversed for pow2)
// transform input: Ex (and phi) to global, and Ex also to Es (smem) if given
__device__ void poisson1d_body(double *__restrict__ Ex, double *Es, double *__restrict__ phi, int n,
                               Spectral1D sp, int pow2, double2 *sm2, int logn) {
    double2 *a = sm2, *tmp = sm2 + n, *ph = sm2 + 2 * n;
    const int tid = threadIdx.x, nt = blockDim.x;
    FIELD_STAMP(3);
    line_transform(a, tmp, n, sp.tw, false, pow2);
    FIELD_STAMP(4);
    // phi_hat and E_hat (E_hat = -i kd phi_hat = (kd*ph.y, -kd*ph.x))
    for (int k = tid; k < n; k += nt) {
        double2 p = make_double2(0.0, 0.0);
        if (k > 0) p = make_double2(a[k].x / sp.k2[k], a[k].y / sp.k2[k]);
        ph[k] = p;
    }
    __syncthreads();
    for (int pass = (phi ? 0 : 1); pass < 2; ++pass) {
        for (int k = tid; k < n; k += nt) {
            double2 v = ph[k];
            if (pass == 1) v = make_double2(sp.kd[k] * v.y, -(sp.kd[k] * v.x));
            put(a, tmp, k, v, pow2, logn);
        }
        __syncthreads();
        FIELD_STAMP(5);
        line_transform(a, tmp, n, sp.tw, true, pow2);
        FIELD_STAMP(6);
        const double inv = 1.0 / (double)n;
        for (int m = tid; m < n; m += nt) {
            const double v = a[m].x * inv;
            if (pass == 0) {
                phi[m] = v;
            } else {
                Ex[m] = v;
                if (Es) Es[m] = v;
            }
        }
        __syncthreads();
    }
}

__global__ void poisson1d_kernel(const double *__restrict__ rho, double *__restrict__ Ex,
                                 double *__restrict__ phi, int n, const double2 *__restrict__ tw,
                                 const double *__restrict__ k2, const double *__restrict__ kd,
                                 int pow2, int logn, int staged) {
    extern __shared__ double2 sm2[];
    const Spectral1D sp = staged ? stage_spectral(tw, k2, kd, n, sm2) : Spectral1D{tw, k2, kd};
    for (int m = threadIdx.x; m < n; m += blockDim.x) put(sm2, sm2 + n, m, make_double2(rho[m], 0.0), pow2, logn);
    __syncthreads();
    poisson1d_body(Ex, nullptr, phi, n, sp, pow2, sm2, logn);
}

// The whole 1D field chain of a stage in one CTA (the per-stage
// "moments -> charge -> Poisson -> tables" of Simulation._stage,
// runner.py:183-191): n_s from the fused moment partials, rho, the spectral
// solve, then every species' line tables (plain e/c1 or the packed rows of
// the tiled 1D-2V kernel) -- bitwise the separate moment-finish / charge /
// Poisson / tables kernels (same per-cell arithmetic and reduction trees,
// field.cuh), with n and rho kept in registers and Ex in shared memory
// between the phases.  Nx <= FIELD1D_MAX_CELLS_PER_THREAD * 1024.
constexpr int FIELD1D_CPT = 2;

struct Tables1D {
    int ns;
    const double *part[8];  // moment partials [Nx][rows][chunks] of each species, or none (n given)
    int rows[8], chunks[8];
    double vol[8];
    double *e[8], *c1[8], *packed[8];
    double qmk2[8], g[8], t1[8], den1[8];
    int corrections[8];
};

__global__ void __launch_bounds__(1024) field1d_kernel(double *__restrict__ n, Charges q, int ns, int nx,
                                                       double *__restrict__ rho, double *__restrict__ Ex,
                                                       const double2 *__restrict__ tw, const double *__restrict__ k2,
                                                       const double *__restrict__ kd, int pow2, int logn,
                                                       Tables1D T) {
    extern __shared__ double2 sm2[];
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    FIELD_STAMP(0);
    double rl[FIELD1D_CPT];  // rho of this thread's cells p = tid + j*nt
    bool own_n = T.part[0] != nullptr;
    for (int s = 0; own_n && s < T.ns; ++s) own_n = T.rows[s] == 1;
    if (T.part[0] && !own_n) {  // 1D-2V partials: a warp per cell (vpfv_moment_partials), n via global
        const int warp = tid >> 5, nw = nt >> 5;
        double *buf = reinterpret_cast<double *>(sm2);  // a/tmp/ph are free until the transform
        for (int s = 0; s < T.ns; ++s) {
            double *bufA = buf + (size_t)warp * 2 * T.rows[s];
            for (int p = warp; p < nx; p += nw) {
                const double x = moment_cell_warp(T.part[s] + (size_t)p * T.rows[s] * T.chunks[s], T.rows[s],
                                                  T.chunks[s], bufA, bufA + T.rows[s]);
                if ((tid & 31) == 0) n[(size_t)s * nx + p] = __dmul_rn(x, T.vol[s]);
            }
        }
        __syncthreads();
    }
    const Spectral1D sp = stage_spectral(tw, k2, kd, nx, sm2);  // after the finish: its buffers overlap
    // rho = sum_s q_s n_s per cell and its fixed-order per-thread sum (charge_block)
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < FIELD1D_CPT; ++j) {
        const int p = tid + j * nt;
        rl[j] = 0.0;
        if (p >= nx) continue;
        double r = 0.0;
        for (int s = 0; s < T.ns; ++s) {
            double ns_p;
            if (own_n) {  // 1D-1V partials: this thread folds its cell's chunks
                ns_p = __dmul_rn(fold_row(T.part[s] + (size_t)p * T.chunks[s], T.chunks[s]), T.vol[s]);
                n[(size_t)s * nx + p] = ns_p;
            } else {
                ns_p = n[(size_t)s * nx + p];
            }
            r = s == 0 ? __dmul_rn(q.q[0], ns_p) : __dadd_rn(r, __dmul_rn(q.q[s], ns_p));
        }
        rl[j] = r;
        acc = __dadd_rn(acc, r);
    }
    FIELD_STAMP(1);
    const double mean = __ddiv_rn(block_tree_sum(acc, red), (double)nx);
    FIELD_STAMP(2);
#pragma unroll
    for (int j = 0; j < FIELD1D_CPT; ++j) {
        const int p = tid + j * nt;
        if (p >= nx) continue;
        const double r = __dsub_rn(rl[j], mean);
        rho[p] = r;
        put(sm2, sm2 + nx, p, make_double2(r, 0.0), pow2, logn);
    }
    __syncthreads();
    // E staged for the tables in ph's region (free once the last put is done)
    double *Eb = reinterpret_cast<double *>(sm2 + 2 * nx);
    poisson1d_body(Ex, Eb, nullptr, nx, sp, pow2, sm2, logn);
    FIELD_STAMP(7);
    for (int s = 0; s < T.ns; ++s) {
        if (T.packed[s]) {
            for (int r = tid; r < nx + 2; r += nt) {  // rows shifted by one, periodic ghosts
                const int i = r == 0 ? nx - 1 : (r == nx + 1 ? 0 : r - 1);
                double2 *o = reinterpret_cast<double2 *>(T.packed[s] + (size_t)r * 8);
                double e, c1;
                table1d_row(Eb, i, nx, T.qmk2[s], T.g[s], T.t1[s], T.den1[s], e, c1);
                o[0] = make_double2(e, T.corrections[s] ? c1 : 0.0);
                o[1] = o[2] = o[3] = make_double2(0.0, 0.0);
            }
        } else {
            for (int i = tid; i < nx; i += nt) {
                double e, c1;
                table1d_row(Eb, i, nx, T.qmk2[s], T.g[s], T.t1[s], T.den1[s], e, c1);
                T.e[s][i] = e;
                T.c1[s][i] = T.corrections[s] ? c1 : 0.0;
            }
        }
    }
    __syncthreads();
    FIELD_STAMP(8);
}

// The same field chain spread over the GPU: the 1D solve is the real
// circulant map E = K (*) rho with K = IFFT(-i kd / k^2) (the spectral
// solve's Green's function, built once on the host with numpy), so instead
// of one CTA walking an FFT while the other SMs idle, each of ~148 CTAs
// rebuilds rho (all Nx cells: from the 1D-1V partials or from n), takes its
// mean, and computes E on its own few cells plus one neighbour each side
// (a warp per cell, lanes striding the sum, shuffle reduction), then those
// cells' table rows.  K2 = K repeated twice, so K2[m - j + Nx] needs no
// modular index.  Rounding differs from the FFT path by O(eps sqrt(Nx)).
__global__ void __launch_bounds__(256) field1d_conv_kernel(double *__restrict__ n, Charges q, int ns, int nx,
                                                           double *__restrict__ rho, double *__restrict__ Ex,
                                                           const double *__restrict__ K2, int per_cta, Tables1D T,
                                                           int trigger) {
    extern __shared__ double sm1[];
    __shared__ double red[32];
    double *rs = sm1, *Es = sm1 + nx;  // rho (all cells), E on this CTA's cells c0-1 .. c0+M
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const bool lead = blockIdx.x == 0;
    if (trigger) pdl_trigger();  // the (programmatic) stage kernel after this may start launching
    pdl_wait();                  // the partials / n of the previous stage
    double acc = 0.0;
    for (int p = tid; p < nx; p += nt) {
        double r = 0.0;
        for (int s = 0; s < T.ns; ++s) {
            double ns_p;
            if (T.part[0]) {
                ns_p = __dmul_rn(fold_row(T.part[s] + (size_t)p * T.chunks[s], T.chunks[s]), T.vol[s]);
                if (lead) n[(size_t)s * nx + p] = ns_p;
            } else {
                ns_p = n[(size_t)s * nx + p];
            }
            r = s == 0 ? __dmul_rn(q.q[0], ns_p) : __dadd_rn(r, __dmul_rn(q.q[s], ns_p));
        }
        rs[p] = r;
        acc = __dadd_rn(acc, r);
    }
    const double mean = __ddiv_rn(block_tree_sum(acc, red), (double)nx);  // its barriers publish rs
    for (int p = tid; p < nx; p += nt) {
        const double r = __dsub_rn(rs[p], mean);
        rs[p] = r;
        if (lead) rho[p] = r;
    }
    __syncthreads();
    const int c0 = blockIdx.x * per_cta, M = min(per_cta, nx - c0);
    for (int o = warp; o < M + 2; o += nw) {
        int m = c0 - 1 + o;
        m += m < 0 ? nx : 0;
        m -= m >= nx ? nx : 0;
        const double *k = K2 + m + nx;  // k[-j] = K[(m - j) mod nx]
        double e = 0.0;
        for (int j = lane; j < nx; j += 32) e = fma(k[-j], rs[j], e);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
        if (lane == 0) Es[o] = e;
    }
    __syncthreads();
    for (int o = tid; o < M; o += nt) Ex[c0 + o] = Es[o + 1];
    for (int s = 0; s < T.ns; ++s) {
        for (int o = tid; o < M; o += nt) {  // table1d_row's arithmetic on the staged E
            const int i = c0 + o;
            const double e = __dadd_rn(__dmul_rn(T.qmk2[s], Es[o + 1]), T.g[s]);
            double c1 = __dadd_rn(T.t1[s], __ddiv_rn(__dmul_rn(T.qmk2[s], __dsub_rn(Es[o + 2], Es[o])), T.den1[s]));
            c1 = T.corrections[s] ? c1 : 0.0;
            if (T.packed[s]) {  // rows shifted by one; the periodic ghost rows 0 and nx+1
                const double2 row = make_double2(e, c1), z = make_double2(0.0, 0.0);
                for (int r : {i + 1, i == nx - 1 ? 0 : -1, i == 0 ? nx + 1 : -1}) {
                    if (r < 0) continue;
                    double2 *out = reinterpret_cast<double2 *>(T.packed[s] + (size_t)r * 8);
                    out[0] = row;
                    out[1] = out[2] = out[3] = z;
                }
            } else {
                T.e[s][i] = e;
                T.c1[s][i] = c1;
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
    pdl_trigger();  // the column pass waits before reading C
    pdl_wait();     // rho
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
    pdl_trigger();  // the inverse row pass waits before reading D
    pdl_wait();     // C of the forward row pass
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
    pdl_trigger();  // the tables kernel waits before reading E
    pdl_wait();     // D of the column pass
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
    const bool staged = poisson1d_smem(N, true) <= 200 * 1024;
    const size_t smem = poisson1d_smem(N, staged);
    if (smem > 200 * 1024) return set_error(VPFV_EARG, "poisson_1d: N too large for one CTA");
    static bool once = false;
    if (!once) {
        allow_smem((const void *)poisson1d_kernel);
        once = true;
    }
    poisson1d_kernel<<<1, 1024, smem, (cudaStream_t)stream>>>(
        rho, Ex, phi, N, (const double2 *)tw, k2, kd, logn >= 0, logn < 0 ? 0 : logn, staged ? 1 : 0);
    return check_launch("poisson_1d");
}

#ifdef VPFV_FIELD_PROBE
extern "C" int vpfv_field_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_field_probe, sizeof(g_field_probe)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int vpfv_field_1d_max_cells(void) { return FIELD1D_CPT * 1024; }

extern "C" int vpfv_field_1d(const double *const *partials, const int *rows, const int *chunks, const double *vols,
                             double *n, const double *q_host, int nspecies, int Nx, double *rho, double *Ex,
                             const double *tw, const double *k2, const double *kd, double *const *e,
                             double *const *c1, double *const *packed, const double *qmk2, const double *g,
                             const double *t1, const double *den1, const int *corrections, void *stream) {
    if (nspecies < 1 || nspecies > 8) return set_error(VPFV_EARG, "field_1d: 1..8 species");
    if (Nx < 2 || Nx > FIELD1D_CPT * 1024) return set_error(VPFV_EARG, "field_1d: Nx outside [2, 2048]");
    const int logn = ilog2_if_pow2(Nx);
    size_t smem = poisson1d_smem(Nx, true);
    for (int s = 0; partials && s < nspecies; ++s) {
        if (!partials[s] || rows[s] < 1 || chunks[s] < 1 || chunks[s] > 16)
            return set_error(VPFV_EARG, "field_1d: bad moment partials");
        if (sizeof(double) * 32 * 2 * (size_t)rows[s] > smem) smem = sizeof(double) * 32 * 2 * (size_t)rows[s];
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

extern "C" int vpfv_field_1d_conv(const double *const *partials, const int *chunks, const double *vols, double *n,
                                  const double *q_host, int nspecies, int Nx, double *rho, double *Ex,
                                  const double *green2, double *const *e, double *const *c1, double *const *packed,
                                  const double *qmk2, const double *g, const double *t1, const double *den1,
                                  const int *corrections, void *stream) {
    if (nspecies < 1 || nspecies > 8) return set_error(VPFV_EARG, "field_1d_conv: 1..8 species");
    if (Nx < 2 || Nx > 16384) return set_error(VPFV_EARG, "field_1d_conv: Nx outside [2, 16384]");
    Charges q;
    Tables1D T{};
    T.ns = nspecies;
    for (int s = 0; s < 8; ++s) q.q[s] = s < nspecies ? q_host[s] : 0.0;
    for (int s = 0; s < nspecies; ++s) {
        if (partials && (!partials[s] || chunks[s] < 1 || chunks[s] > 16))
            return set_error(VPFV_EARG, "field_1d_conv: bad moment partials (one row, <= 16 chunks)");
        T.part[s] = partials ? partials[s] : nullptr;
        T.rows[s] = 1;
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
        if (!T.packed[s] && !(T.e[s] && T.c1[s])) return set_error(VPFV_EARG, "field_1d_conv: no table outputs");
    }
    const int per = (Nx + 147) / 148;
    const int grid = (Nx + per - 1) / per;
    const size_t smem = sizeof(double) * ((size_t)Nx + per + 2);
    static bool once = false;
    if (!once) {
        allow_smem((const void *)field1d_conv_kernel);
        once = true;
    }
    // From 1D-1V partials of one species the caller's next launch is that
    // species' stage kernel, a programmatic dependent: launch programmatically
    // and let it start early.  Otherwise (a moment kernel before, 1D-2V or
    // several species after) an ordinary launch that does not trigger.
    const int trigger = partials && nspecies == 1 ? 1 : 0;
    if (partials) {
        const cudaError_t rc = launch_pdl(field1d_conv_kernel, dim3(grid), dim3(256), smem, (cudaStream_t)stream, n,
                                          q, nspecies, Nx, rho, Ex, green2, per, T, trigger);
        if (rc != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(rc));
    } else {
        field1d_conv_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(n, q, nspecies, Nx, rho, Ex, green2, per, T,
                                                                      0);
    }
    return check_launch("field_1d_conv");
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
    // programmatic links: each launches while its predecessor drains and
    // waits (griddepcontrol.wait) before its first read
    const int py = ly >= 0, lgy = ly < 0 ? 0 : ly, px = lx >= 0, lgx = lx < 0 ? 0 : lx;
    launch_pdl(rows_fwd_kernel, dim3(Nx), dim3(256), smy, s, rho, C, Nx, Ny, (const double2 *)twy, py, lgy);
    launch_pdl(cols_kernel, dim3(Ny), dim3(256), smx, s, (const double2 *)C, D, Nx, Ny, (const double2 *)twx, kx, ky,
               kxd, kyd, nout, px, lgx);
    launch_pdl(rows_inv_kernel, dim3(Nx), dim3(256), smy, s, (const double2 *)D, Ex, Ey, phi, Nx, Ny,
               (const double2 *)twy, nout, py, lgy);
    return check_launch("poisson_2d");
}
