/* Plain-C restatement of the reference fused stage kernels and fold-tree
 * moment -- TEST / CPU-BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Restates /root/reference/pkg/src/vpfv/_kernels.py:92-317 (stage_1d1v,
 * stage_1d2v, stage_2d2v) and fields.py:28-47 (fold tree).  The reference
 * kernels are numba-compiled with fastmath=False (no FMA, true division,
 * SURVEY.md 8c); this file is compiled with -ffp-contract=off and no
 * fast-math, evaluates every cell in the same operation order, and is
 * therefore bitwise equal to them.  The outermost loop is split across
 * OpenMP threads (the reference itself is serial, _kernels.py:15-16); cells
 * are independent so threading cannot change any result.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NG 3

static inline double fdp(const double *s, long i, long st) {
    return (-2.0 * s[i - 3 * st] + 15.0 * s[i - 2 * st] - 60.0 * s[i - st]
            + 20.0 * s[i] + 30.0 * s[i + st] - 3.0 * s[i + 2 * st]) / 60.0;
}
static inline double fdn(const double *s, long i, long st) {
    return (3.0 * s[i - 2 * st] - 30.0 * s[i - st] - 20.0 * s[i]
            + 60.0 * s[i + st] - 15.0 * s[i + 2 * st] + 2.0 * s[i + 3 * st]) / 60.0;
}
/* s[+a,-b] + s[-a,+b] - s[+a,+b] - s[-a,-b] */
static inline double dg(const double *s, long i, long sa, long sb) {
    return s[i + sa - sb] + s[i - sa + sb] - s[i + sa + sb] - s[i - sa - sb];
}

/* _kernels.py:92-114 */
void oracle_stage_1d1v(double *dest, const double *A, const double *B, const double *src,
                       double ca, double cb, double cd, double cL,
                       const double *ax, const double *avx, const double *c1,
                       double hx, double hv, int Nx, int Nv) {
    const long P1 = Nv + 2 * NG;
#pragma omp parallel for schedule(static)
    for (int i = NG; i < Nx + NG; ++i) {
        double a_v = avx[i - NG], c1i = c1[i - NG];
        for (int j = NG; j < Nv + NG; ++j) {
            long c = (long)i * P1 + j;
            double a_x = ax[j - NG], rhs;
            if (a_x > 0.0) rhs = -a_x * fdp(src, c, P1) / hx;
            else rhs = -a_x * fdn(src, c, P1) / hx;
            if (a_v > 0.0) rhs -= a_v * fdp(src, c, 1) / hv;
            else rhs -= a_v * fdn(src, c, 1) / hv;
            rhs += c1i * dg(src, c, P1, 1);
            dest[c] = ca * A[c] + cb * B[c] + cd * dest[c] + cL * rhs;
        }
    }
}

/* _kernels.py:153-197 (vyc has Nvy+1 entries, the last is cB) */
void oracle_stage_1d2v(double *dest, const double *A, const double *B, const double *src,
                       double ca, double cb, double cd, double cL,
                       const double *vxc, const double *vyc, const double *evx,
                       const double *avy, const double *c1, double c2,
                       double hx, double hvx, double hvy, int Nx, int Nvx, int Nvy) {
    const long P2 = Nvy + 2 * NG, P1 = (long)(Nvx + 2 * NG) * P2;
    const double cB = vyc[Nvy];
#pragma omp parallel for schedule(static)
    for (int i = NG; i < Nx + NG; ++i) {
        double e_i = evx[i - NG], c1i = c1[i - NG];
        for (int j = NG; j < Nvx + NG; ++j) {
            double a_x = vxc[j - NG], a_vy = avy[j - NG];
            for (int k = NG; k < Nvy + NG; ++k) {
                long c = (long)i * P1 + (long)j * P2 + k;
                double rhs;
                if (a_x > 0.0) rhs = -a_x * fdp(src, c, P1) / hx;
                else rhs = -a_x * fdn(src, c, P1) / hx;
                double a_vx = e_i + cB * vyc[k - NG];
                if (a_vx > 0.0) rhs -= a_vx * fdp(src, c, P2) / hvx;
                else rhs -= a_vx * fdn(src, c, P2) / hvx;
                if (a_vy > 0.0) rhs -= a_vy * fdp(src, c, 1) / hvy;
                else rhs -= a_vy * fdn(src, c, 1) / hvy;
                rhs += c1i * dg(src, c, P1, P2);
                rhs -= c2 * dg(src, c, P2, 1);
                dest[c] = ca * A[c] + cb * B[c] + cd * dest[c] + cL * rhs;
            }
        }
    }
}

/* _kernels.py:254-317 */
void oracle_stage_2d2v(double *dest, const double *A, const double *B, const double *src,
                       double ca, double cb, double cd, double cL,
                       const double *vxc, const double *vyc, const double *evx,
                       const double *evy, double cB, const double *c1, double c2,
                       const double *c3, const double *c4, const double *c5,
                       double hx, double hy, double hvx, double hvy,
                       int Nx, int Ny, int Nvx, int Nvy) {
    const long P3 = Nvy + 2 * NG, P2 = (long)(Nvx + 2 * NG) * P3, P1 = (long)(Ny + 2 * NG) * P2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int i = NG; i < Nx + NG; ++i) {
        for (int j = NG; j < Ny + NG; ++j) {
            long e = (long)(i - NG) * Ny + (j - NG);
            double e_x = evx[e], e_y = evy[e], c1ij = c1[e], c3ij = c3[e], c4ij = c4[e], c5ij = c5[e];
            for (int k = NG; k < Nvx + NG; ++k) {
                double a_x = vxc[k - NG];
                double a_vy = e_y - cB * vxc[k - NG];
                for (int l = NG; l < Nvy + NG; ++l) {
                    long c = (long)i * P1 + (long)j * P2 + (long)k * P3 + l;
                    double a_y = vyc[l - NG];
                    double a_vx = e_x + cB * vyc[l - NG];
                    double rhs;
                    if (a_x > 0.0) rhs = -a_x * fdp(src, c, P1) / hx;
                    else rhs = -a_x * fdn(src, c, P1) / hx;
                    if (a_y > 0.0) rhs -= a_y * fdp(src, c, P2) / hy;
                    else rhs -= a_y * fdn(src, c, P2) / hy;
                    if (a_vx > 0.0) rhs -= a_vx * fdp(src, c, P3) / hvx;
                    else rhs -= a_vx * fdn(src, c, P3) / hvx;
                    if (a_vy > 0.0) rhs -= a_vy * fdp(src, c, 1) / hvy;
                    else rhs -= a_vy * fdn(src, c, 1) / hvy;
                    rhs += c1ij * dg(src, c, P1, P3);
                    rhs += c4ij * dg(src, c, P2, 1);
                    rhs -= c2 * dg(src, c, P3, 1);
                    rhs -= c3ij * dg(src, c, P2, P3);
                    rhs -= c5ij * dg(src, c, P1, 1);
                    dest[c] = ca * A[c] + cb * B[c] + cd * dest[c] + cL * rhs;
                }
            }
        }
    }
}

/* fields.py:28-39: adjacent-pair rounds with the odd tail carried, in place
 * on a scratch vector of length n. */
static double fold_vec(double *x, int n) {
    while (n > 1) {
        int m = n / 2;
        for (int t = 0; t < m; ++t) x[t] = x[2 * t] + x[2 * t + 1];
        if (n % 2) { x[m] = x[n - 1]; n = m + 1; } else n = m;
    }
    return x[0];
}

/* zeroth moment fold tree over the velocity dims (fields.py:42-47, 86-111):
 * fastest velocity axis first.  nphys = product of physical extents,
 * nv1 (outer velocity, 1 if v==1), nv2 (inner velocity); strides in the
 * padded array are passed so 1D/2D physical layouts share the code:
 *   value(p, a, b) = data[base(p) + (a+NG)*s_a + (b+NG)]
 * base(p) enumerates the physical interior cells in C order. */
void oracle_moment(const double *data, double *out, int d, const int *Npad, const int *N,
                   int v, double vol) {
    long nphys = 1;
    for (int k = 0; k < d; ++k) nphys *= N[k];
    int nv1 = (v == 2) ? N[d] : 1, nv2 = N[d + v - 1];
    long s_b = 1, s_a = (v == 2) ? Npad[d + 1] : 0;
    long vel_block = 1;
    for (int k = d; k < d + v; ++k) vel_block *= Npad[k];
#pragma omp parallel
    {
        double *row = malloc(sizeof(double) * (size_t)(nv2 > nv1 ? nv2 : nv1));
        double *outer = malloc(sizeof(double) * (size_t)nv1);
#pragma omp for schedule(static)
        for (long p = 0; p < nphys; ++p) {
            long base;
            if (d == 1) base = (p + NG) * vel_block;
            else {
                long ix = p / N[1], iy = p % N[1];
                base = ((ix + NG) * Npad[1] + (iy + NG)) * vel_block;
            }
            long voff = (v == 2) ? (long)NG * s_a : 0;
            for (int a = 0; a < nv1; ++a) {
                const double *r = data + base + voff + (long)a * s_a + NG * s_b;
                memcpy(row, r, sizeof(double) * (size_t)nv2);
                outer[a] = fold_vec(row, nv2);
            }
            double s = (v == 2) ? fold_vec(outer, nv1) : outer[0];
            out[p] = s * vol;
        }
        free(row);
        free(outer);
    }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
