// Fused VP-FV stage kernels for sm_100a (B200).
//
// One pass over the interior computes
//     dest = ca*A + cb*B + cd*dest + cL * RHS(src)
// where RHS is the upwinded 6-point face difference along every phase-space
// dim plus the closed-form diagonal transverse corrections -- the operator of
// /root/reference/pkg/src/vpfv/_kernels.py:92-317 (numba) and
// fvm.py:240-263 (numpy).
//
// Two arithmetic policies share the index logic:
//  * EXACT: the numba kernels' per-cell operation order with round-to-nearest
//    intrinsics (no FMA contraction, IEEE division) -> bitwise equal to the
//    reference kernels (which compile to scalar x86 without FMA).
//  * fast: integer-weight stencil sums with FMA and host-folded reciprocals
//    (-1/(60 h)); agrees with the reference to a few ulps per stage.
//
// Layout: the reference padded C-order storage (velocity dims fastest).
// Periodic dims flagged in `wrap` are read by modular indexing into the
// interior, so the single-GPU driver never refreshes physical ghosts; frozen
// velocity ghosts are read from storage (written once at set-up).
//
// Thread mapping (generic kernel): blockIdx.y enumerates physical cells
// (x or (x,y)), a 1-D block sweeps the velocity plane with the fastest dim
// across lanes -> fully coalesced rows of the padded array.
#include "common.cuh"

namespace vpfv {

// ---------------------------------------------------------------------------
// per-dimension addressing

struct Axis {
    long long st;  // element stride of this dim in the padded array
    int idx;       // interior index of the cell along this dim
    int n;         // interior extent
    bool wrap;     // periodic, read by modular index
    __device__ __forceinline__ long long off(int o) const {
        if (!wrap) return (long long)o * st;
        int t = idx + o;
        t += (t < 0) ? n : 0;
        t -= (t >= n) ? n : 0;
        return (long long)(t - idx) * st;
    }
};

// exact face difference (numba order, _kernels.py:66-89)
__device__ __forceinline__ double fd_exact(const double *__restrict__ s, long long c, const Axis &a,
                                           bool pos) {
    double t;
    if (pos) {
        t = __dmul_rn(-2.0, ldg(s + c + a.off(-3)));
        t = __dadd_rn(t, __dmul_rn(15.0, ldg(s + c + a.off(-2))));
        t = __dsub_rn(t, __dmul_rn(60.0, ldg(s + c + a.off(-1))));
        t = __dadd_rn(t, __dmul_rn(20.0, ldg(s + c)));
        t = __dadd_rn(t, __dmul_rn(30.0, ldg(s + c + a.off(1))));
        t = __dsub_rn(t, __dmul_rn(3.0, ldg(s + c + a.off(2))));
    } else {
        t = __dmul_rn(3.0, ldg(s + c + a.off(-2)));
        t = __dsub_rn(t, __dmul_rn(30.0, ldg(s + c + a.off(-1))));
        t = __dsub_rn(t, __dmul_rn(20.0, ldg(s + c)));
        t = __dadd_rn(t, __dmul_rn(60.0, ldg(s + c + a.off(1))));
        t = __dsub_rn(t, __dmul_rn(15.0, ldg(s + c + a.off(2))));
        t = __dadd_rn(t, __dmul_rn(2.0, ldg(s + c + a.off(3))));
    }
    return __ddiv_rn(t, 60.0);
}

// fast integer-weight sum W (face difference = W / 60)
__device__ __forceinline__ double fd_sum(const double *__restrict__ s, long long c, const Axis &a,
                                         bool pos) {
    double t;
    if (pos) {
        t = -2.0 * ldg(s + c + a.off(-3));
        t = fma(15.0, ldg(s + c + a.off(-2)), t);
        t = fma(-60.0, ldg(s + c + a.off(-1)), t);
        t = fma(20.0, ldg(s + c), t);
        t = fma(30.0, ldg(s + c + a.off(1)), t);
        t = fma(-3.0, ldg(s + c + a.off(2)), t);
    } else {
        t = 3.0 * ldg(s + c + a.off(-2));
        t = fma(-30.0, ldg(s + c + a.off(-1)), t);
        t = fma(-20.0, ldg(s + c), t);
        t = fma(60.0, ldg(s + c + a.off(1)), t);
        t = fma(-15.0, ldg(s + c + a.off(2)), t);
        t = fma(2.0, ldg(s + c + a.off(3)), t);
    }
    return t;
}

// s[+a,-b] + s[-a,+b] - s[+a,+b] - s[-a,-b]   (kernel order)
template <bool EXACT>
__device__ __forceinline__ double diag(const double *__restrict__ s, long long c, const Axis &a,
                                       const Axis &b) {
    double p = ldg(s + c + a.off(1) + b.off(-1));
    double q = ldg(s + c + a.off(-1) + b.off(1));
    double r = ldg(s + c + a.off(1) + b.off(1));
    double u = ldg(s + c + a.off(-1) + b.off(-1));
    if (EXACT) return __dsub_rn(__dsub_rn(__dadd_rn(p, q), r), u);
    return ((p + q) - r) - u;
}

// rhs accumulation of one flux dim
template <bool EXACT>
__device__ __forceinline__ double flux_first(const double *s, long long c, const Axis &ax, double a,
                                             double h, double mh) {
    bool pos = a > 0.0;
    if (EXACT) return __ddiv_rn(__dmul_rn(-a, fd_exact(s, c, ax, pos)), h);
    return (a * mh) * fd_sum(s, c, ax, pos);
}
template <bool EXACT>
__device__ __forceinline__ double flux_next(double rhs, const double *s, long long c, const Axis &ax,
                                            double a, double h, double mh) {
    bool pos = a > 0.0;
    if (EXACT) return __dsub_rn(rhs, __ddiv_rn(__dmul_rn(a, fd_exact(s, c, ax, pos)), h));
    return fma(a * mh, fd_sum(s, c, ax, pos), rhs);
}
template <bool EXACT>
__device__ __forceinline__ double corr_add(double rhs, double cf, double dg) {
    return EXACT ? __dadd_rn(rhs, __dmul_rn(cf, dg)) : fma(cf, dg, rhs);
}
template <bool EXACT>
__device__ __forceinline__ double corr_sub(double rhs, double cf, double dg) {
    return EXACT ? __dsub_rn(rhs, __dmul_rn(cf, dg)) : fma(-cf, dg, rhs);
}

struct Update {
    double *dest;
    const double *A, *B;
    double ca, cb, cd, cL;
    const double *dt_dev;
    double cL_div;
    bool a_is_src, b_is_src;
    unsigned long long *nonfinite;
};

template <bool EXACT>
__device__ __forceinline__ double finish(const Update &u, const double *src, long long c, double rhs,
                                         unsigned long long flat) {
    double cL = u.dt_dev ? __ddiv_rn(*u.dt_dev, u.cL_div) : u.cL;
    double s0 = 0.0;
    if (u.a_is_src || u.b_is_src) s0 = ldg(src + c);
    double out;
    if (EXACT) {
        double a = u.a_is_src ? s0 : ldg(u.A + c);
        double b = u.b_is_src ? s0 : ldg(u.B + c);
        double d = u.dest[c];
        out = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(u.ca, a), __dmul_rn(u.cb, b)),
                                  __dmul_rn(u.cd, d)),
                        __dmul_rn(cL, rhs));
    } else {
        out = cL * rhs;
        if (u.cd != 0.0) out = fma(u.cd, u.dest[c], out);
        if (u.cb != 0.0) out = fma(u.cb, u.b_is_src ? s0 : ldg(u.B + c), out);
        if (u.ca != 0.0) out = fma(u.ca, u.a_is_src ? s0 : ldg(u.A + c), out);
    }
    u.dest[c] = out;
    if (u.nonfinite && !isfinite(out)) atomicMin(u.nonfinite, flat);
    return out;
}

// ---------------------------------------------------------------------------
// 1D-1V  (_kernels.py:92-114)

struct T11 {
    const double *ax, *avx, *c1;
    double hx, hv, mhx, mhv;
};

// partials (fast path, Nv % 128 == 0, 128-thread blocks): the fold-tree
// subtree sum of the new dest over each aligned 128-wide v chunk
// (fields.py:28-47: shuffle levels 1-5, then the 4 warp sums pairwise),
// partials[i][0][chunk] -- finished by vpfv_moment_partials(nvx = 1).
template <bool EXACT>
__global__ void __launch_bounds__(256) stage_1d1v_kernel(Update u, const double *__restrict__ src,
                                                         T11 t, int Nx, int Nv, unsigned wrap,
                                                         double *__restrict__ partials) {
    const int i = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Nv) return;
    const long long P1 = Nv + 2 * NG;
    const long long c = (long long)(i + NG) * P1 + (j + NG);
    Axis X{P1, i, Nx, (wrap & 2u) != 0}, V{1, j, Nv, (wrap & 4u) != 0};
    double a_x = ldg(t.ax + j);  // velocity centres: not written by the predecessor
    pdl_wait();                  // tables and src of the preceding launches
    double a_v = ldg(t.avx + i), c1 = ldg(t.c1 + i);
    double rhs = flux_first<EXACT>(src, c, X, a_x, t.hx, t.mhx);
    rhs = flux_next<EXACT>(rhs, src, c, V, a_v, t.hv, t.mhv);
    rhs = corr_add<EXACT>(rhs, c1, diag<EXACT>(src, c, X, V));
    double out = finish<EXACT>(u, src, c, rhs, (unsigned long long)i * Nv + j);
    if (!EXACT && partials) {
        __shared__ double wsum[4];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) out = __dadd_rn(out, __shfl_xor_sync(0xffffffffu, out, off));
        if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = out;
        __syncthreads();
        if (threadIdx.x == 0)
            partials[(long long)i * gridDim.x + blockIdx.x] =
                __dadd_rn(__dadd_rn(wsum[0], wsum[1]), __dadd_rn(wsum[2], wsum[3]));
    }
}

// ---------------------------------------------------------------------------
// 1D-2V  (_kernels.py:153-197)

struct T12 {
    const double *vxc, *vyc, *evx, *avy, *c1;
    double c2;
    double hx, hvx, hvy, mhx, mhvx, mhvy;
};

template <bool EXACT>
__global__ void __launch_bounds__(256) stage_1d2v_kernel(Update u, const double *__restrict__ src,
                                                         T12 t, int Nx, int Nvx, int Nvy,
                                                         unsigned wrap) {
    const int i = blockIdx.y;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Nvx * Nvy) return;
    const int j = q / Nvy, k = q - j * Nvy;
    const long long P2 = Nvy + 2 * NG, P1 = (long long)(Nvx + 2 * NG) * P2;
    const long long c = (long long)(i + NG) * P1 + (long long)(j + NG) * P2 + (k + NG);
    Axis X{P1, i, Nx, (wrap & 2u) != 0}, VX{P2, j, Nvx, (wrap & 4u) != 0},
        VY{1, k, Nvy, (wrap & 8u) != 0};
    double a_x = ldg(t.vxc + j), a_vy = ldg(t.avy + j);
    const double cB = ldg(t.vyc + Nvy);  // trailing slot carries cB (_kernels.py:166)
    double a_vx = EXACT ? __dadd_rn(ldg(t.evx + i), __dmul_rn(cB, ldg(t.vyc + k)))
                        : fma(cB, ldg(t.vyc + k), ldg(t.evx + i));
    double rhs = flux_first<EXACT>(src, c, X, a_x, t.hx, t.mhx);
    rhs = flux_next<EXACT>(rhs, src, c, VX, a_vx, t.hvx, t.mhvx);
    rhs = flux_next<EXACT>(rhs, src, c, VY, a_vy, t.hvy, t.mhvy);
    rhs = corr_add<EXACT>(rhs, ldg(t.c1 + i), diag<EXACT>(src, c, X, VX));
    rhs = corr_sub<EXACT>(rhs, t.c2, diag<EXACT>(src, c, VX, VY));
    finish<EXACT>(u, src, c, rhs, (unsigned long long)i * Nvx * Nvy + q);
}

// ---------------------------------------------------------------------------
// 2D-2V  (_kernels.py:254-317)

struct T22 {
    const double *vxc, *vyc, *evx, *evy, *c1, *c3, *c4, *c5;
    double cB, c2;
    double hx, hy, hvx, hvy, mhx, mhy, mhvx, mhvy;
};

template <bool EXACT>
__global__ void __launch_bounds__(256) stage_2d2v_kernel(Update u, const double *__restrict__ src,
                                                         T22 t, int Nx, int Ny, int Nvx, int Nvy,
                                                         unsigned wrap) {
    const int p = blockIdx.y;  // physical cell i*Ny + j
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Nvx * Nvy) return;
    const int i = p / Ny, j = p - i * Ny;
    const int k = q / Nvy, l = q - k * Nvy;
    const long long P3 = Nvy + 2 * NG, P2 = (long long)(Nvx + 2 * NG) * P3,
                    P1 = (long long)(Ny + 2 * NG) * P2;
    const long long c = (long long)(i + NG) * P1 + (long long)(j + NG) * P2 +
                        (long long)(k + NG) * P3 + (l + NG);
    Axis X{P1, i, Nx, (wrap & 2u) != 0}, Y{P2, j, Ny, (wrap & 4u) != 0},
        VX{P3, k, Nvx, (wrap & 8u) != 0}, VY{1, l, Nvy, (wrap & 16u) != 0};
    const double vx = ldg(t.vxc + k), vy = ldg(t.vyc + l);
    const double ex = ldg(t.evx + p), ey = ldg(t.evy + p);
    double a_vy, a_vx;
    if (EXACT) {
        a_vy = __dsub_rn(ey, __dmul_rn(t.cB, vx));
        a_vx = __dadd_rn(ex, __dmul_rn(t.cB, vy));
    } else {
        a_vy = fma(-t.cB, vx, ey);
        a_vx = fma(t.cB, vy, ex);
    }
    double rhs = flux_first<EXACT>(src, c, X, vx, t.hx, t.mhx);
    rhs = flux_next<EXACT>(rhs, src, c, Y, vy, t.hy, t.mhy);
    rhs = flux_next<EXACT>(rhs, src, c, VX, a_vx, t.hvx, t.mhvx);
    rhs = flux_next<EXACT>(rhs, src, c, VY, a_vy, t.hvy, t.mhvy);
    rhs = corr_add<EXACT>(rhs, ldg(t.c1 + p), diag<EXACT>(src, c, X, VX));
    rhs = corr_add<EXACT>(rhs, ldg(t.c4 + p), diag<EXACT>(src, c, Y, VY));
    rhs = corr_sub<EXACT>(rhs, t.c2, diag<EXACT>(src, c, VX, VY));
    rhs = corr_sub<EXACT>(rhs, ldg(t.c3 + p), diag<EXACT>(src, c, Y, VX));
    rhs = corr_sub<EXACT>(rhs, ldg(t.c5 + p), diag<EXACT>(src, c, X, VY));
    finish<EXACT>(u, src, c, rhs, (unsigned long long)p * Nvx * Nvy + q);
}

// ---------------------------------------------------------------------------
// launchers

static Update make_update(double *dest, const double *A, const double *B, const double *src,
                          double ca, double cb, double cd, double cL, const double *dt_dev,
                          double cL_div, unsigned long long *nonfinite) {
    Update u;
    u.dest = dest;
    u.A = A;
    u.B = B;
    u.ca = ca;
    u.cb = cb;
    u.cd = cd;
    u.cL = cL;
    u.dt_dev = dt_dev;
    u.cL_div = cL_div;
    u.a_is_src = (A == src);
    u.b_is_src = (B == src);
    u.nonfinite = nonfinite;
    return u;
}

struct Stage22;
bool tma_2d2v_eligible(int Nx, int Ny, int Nvx, int Nvy, unsigned flags);
bool march_1d1v_eligible(int Nx, int Nv, unsigned flags);
int launch_1d1v_march(double *dest, const double *A, const double *B, const double *src, double ca, double cb,
                      double cd, double cL, const double *ax, const double *avx, const double *c1, double hx,
                      double hv, int Nx, int Nv, unsigned flags, const double *dt_dev, double cL_div,
                      unsigned long long *nonfinite, double *partials, cudaStream_t stream);

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_stage_1d1v(double *dest, const double *A, const double *B, const double *src,
                               double ca, double cb, double cd, double cL, const double *ax,
                               const double *avx, const double *c1, double hx, double hv, int Nx,
                               int Nv, unsigned flags, const double *dt_dev, double cL_div,
                               unsigned long long *nonfinite, void *stream) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (Nx < 1 || Nv < 1) return set_error(VPFV_EARG, "bad extents");
    if (march_1d1v_eligible(Nx, Nv, flags))
        return launch_1d1v_march(dest, A, B, src, ca, cb, cd, cL, ax, avx, c1, hx, hv, Nx, Nv, flags, dt_dev, cL_div,
                                 nonfinite, nullptr, (cudaStream_t)stream);
    Update u = make_update(dest, A, B, src, ca, cb, cd, cL, dt_dev, cL_div, nonfinite);
    T11 t{ax, avx, c1, hx, hv, -1.0 / (60.0 * hx), -1.0 / (60.0 * hv)};
    dim3 block(128), grid((Nv + 127) / 128, Nx);
    cudaStream_t s = (cudaStream_t)stream;
    double *none = nullptr;
    cudaError_t e = (flags & VPFV_EXACT)
                        ? launch_pdl(stage_1d1v_kernel<true>, grid, block, 0, s, u, src, t, Nx, Nv, flags, none)
                        : launch_pdl(stage_1d1v_kernel<false>, grid, block, 0, s, u, src, t, Nx, Nv, flags, none);
    if (e != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(e));
    return check_launch("stage_1d1v");
}

extern "C" int vpfv_stage_1d1v_fused(double *dest, const double *A, const double *B, const double *src,
                                     double ca, double cb, double cd, double cL, const double *ax,
                                     const double *avx, const double *c1, double hx, double hv, int Nx,
                                     int Nv, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, double *moment_partials, void *stream) {
    if (!moment_partials)
        return vpfv_stage_1d1v(dest, A, B, src, ca, cb, cd, cL, ax, avx, c1, hx, hv, Nx, Nv, flags, dt_dev, cL_div,
                               nonfinite, stream);
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if ((flags & VPFV_EXACT) || Nv % 128 || Nx < 1)
        return set_error(VPFV_EARG, "1D-1V moment partials need the fast path and Nv % 128 == 0");
    if (march_1d1v_eligible(Nx, Nv, flags))
        return launch_1d1v_march(dest, A, B, src, ca, cb, cd, cL, ax, avx, c1, hx, hv, Nx, Nv, flags, dt_dev, cL_div,
                                 nonfinite, moment_partials, (cudaStream_t)stream);
    Update u = make_update(dest, A, B, src, ca, cb, cd, cL, dt_dev, cL_div, nonfinite);
    T11 t{ax, avx, c1, hx, hv, -1.0 / (60.0 * hx), -1.0 / (60.0 * hv)};
    dim3 block(128), grid(Nv / 128, Nx);
    cudaError_t e = launch_pdl(stage_1d1v_kernel<false>, grid, block, 0, (cudaStream_t)stream, u, src, t, Nx, Nv, flags,
                               moment_partials);
    if (e != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(e));
    return check_launch("stage_1d1v_fused");
}

extern "C" int vpfv_stage_1d2v(double *dest, const double *A, const double *B, const double *src,
                               double ca, double cb, double cd, double cL, const double *vxc,
                               const double *vyc, const double *evx, const double *avy,
                               const double *c1, double c2, double hx, double hvx, double hvy,
                               int Nx, int Nvx, int Nvy, unsigned flags, const double *dt_dev,
                               double cL_div, unsigned long long *nonfinite, void *stream) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (Nx < 1 || Nvx < 1 || Nvy < 1) return set_error(VPFV_EARG, "bad extents");
    Update u = make_update(dest, A, B, src, ca, cb, cd, cL, dt_dev, cL_div, nonfinite);
    T12 t{vxc, vyc, evx, avy, c1, c2, hx, hvx, hvy,
          -1.0 / (60.0 * hx), -1.0 / (60.0 * hvx), -1.0 / (60.0 * hvy)};
    int nq = Nvx * Nvy;
    dim3 block(256), grid((nq + 255) / 256, Nx);
    cudaStream_t s = (cudaStream_t)stream;
    if (flags & VPFV_EXACT)
        stage_1d2v_kernel<true><<<grid, block, 0, s>>>(u, src, t, Nx, Nvx, Nvy, flags);
    else
        stage_1d2v_kernel<false><<<grid, block, 0, s>>>(u, src, t, Nx, Nvx, Nvy, flags);
    return check_launch("stage_1d2v");
}

extern "C" int vpfv_stage_2d2v_fused(double *dest, const double *A, const double *B,
                                     const double *src, double ca, double cb, double cd, double cL,
                                     const double *vxc, const double *vyc, const double *evx,
                                     const double *evy, double cB, const double *c1, double c2,
                                     const double *c3, const double *c4, const double *c5, double hx,
                                     double hy, double hvx, double hvy, int Nx, int Ny, int Nvx,
                                     int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, const double *packed_tables,
                                     double *moment_partials, int xsegments, void *stream);

extern "C" int vpfv_stage_2d2v(double *dest, const double *A, const double *B, const double *src,
                               double ca, double cb, double cd, double cL, const double *vxc,
                               const double *vyc, const double *evx, const double *evy, double cB,
                               const double *c1, double c2, const double *c3, const double *c4,
                               const double *c5, double hx, double hy, double hvx, double hvy,
                               int Nx, int Ny, int Nvx, int Nvy, unsigned flags,
                               const double *dt_dev, double cL_div,
                               unsigned long long *nonfinite, void *stream) {
    return vpfv_stage_2d2v_fused(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2, c3,
                                 c4, c5, hx, hy, hvx, hvy, Nx, Ny, Nvx, Nvy, flags, dt_dev, cL_div,
                                 nonfinite, nullptr, nullptr, 0, stream);
}

extern "C" int vpfv_stage_2d2v_generic(double *dest, const double *A, const double *B,
                                       const double *src, double ca, double cb, double cd, double cL,
                                       const double *vxc, const double *vyc, const double *evx,
                                       const double *evy, double cB, const double *c1, double c2,
                                       const double *c3, const double *c4, const double *c5,
                                       double hx, double hy, double hvx, double hvy, int Nx, int Ny,
                                       int Nvx, int Nvy, unsigned flags, const double *dt_dev,
                                       double cL_div, unsigned long long *nonfinite, void *stream) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (Nx < 1 || Ny < 1 || Nvx < 1 || Nvy < 1) return set_error(VPFV_EARG, "bad extents");
    if ((long long)Nx * Ny > 65535) return set_error(VPFV_EARG, "Nx*Ny > 65535 unsupported");
    Update u = make_update(dest, A, B, src, ca, cb, cd, cL, dt_dev, cL_div, nonfinite);
    T22 t{vxc, vyc, evx, evy, c1, c3, c4, c5, cB, c2, hx, hy, hvx, hvy,
          -1.0 / (60.0 * hx), -1.0 / (60.0 * hy), -1.0 / (60.0 * hvx), -1.0 / (60.0 * hvy)};
    int nq = Nvx * Nvy;
    dim3 block(256), grid((nq + 255) / 256, Nx * Ny);
    cudaStream_t s = (cudaStream_t)stream;
    if (flags & VPFV_EXACT)
        stage_2d2v_kernel<true><<<grid, block, 0, s>>>(u, src, t, Nx, Ny, Nvx, Nvy, flags);
    else
        stage_2d2v_kernel<false><<<grid, block, 0, s>>>(u, src, t, Nx, Ny, Nvx, Nvy, flags);
    return check_launch("stage_2d2v");
}
