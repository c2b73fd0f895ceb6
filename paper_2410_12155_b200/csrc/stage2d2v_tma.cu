// 2D-2V fused stage, x-marching with TMA-staged halo tiles (sm_100a, fast path).
//
// Same operator as stage_2d2v (/root/reference/pkg/src/vpfv/_kernels.py:254-317)
// with the fast arithmetic policy.  Organisation:
//
//  * A CTA owns a (y, vx, vy) = (BJ, BK, BL) block of columns and marches
//    along x (the slowest dim) over planes p = i0-3 .. i1+2.
//  * Every plane's (BJ+6, BK+6, BL+8) halo tile (the vy box starts at the
//    16 B-aligned padded column l0 -- TMA requires an aligned inner start) is copied global -> shared by
//    the Tensor Memory Accelerator (cp.async.bulk.tensor.4d, one core box plus
//    two 3-row y-halo boxes so periodic y wraps cost nothing), NSTAGE deep,
//    completion tracked by mbarrier transaction counts.
//  * Each thread keeps, per column, 7 register accumulators for the cells
//    p-3..p+3 currently "in flight" along x.  When plane p lands, it adds
//      - its x-stencil contribution (a_x/(60 h_x) * w_o * s(p)) to cells p-o,
//      - the in-plane part T(p): y/vx/vy fluxes + (y,vy),(vx,vy),(y,vx)
//        corrections, all read from shared memory with immediate offsets,
//      - the x-coupled corrections through D(p) = s[k-1]-s[k+1] and
//        G(p) = s[l-1]-s[l+1]:  c1(q)(D(q+1)-D(q-1)) - c5(q)(G(q+1)-G(q-1)),
//    then finalises cell p-3 with the RK4 stage combination and streams it
//    to HBM (coalesced 256 B warp rows).
//  * Optionally the epilogue also emits the velocity-moment partials of the
//    new dest: a warp-shuffle fold-tree subtree over each aligned 32-wide vy
//    chunk (bitwise the reference fold tree's first five levels), finished by
//    vpfv_moment_from_partials.  This saves the separate moment pass over f.
//
// Requirements (checked by the launcher, else the generic kernel runs):
// Ny % BJ == 0, Nvx % BK == 0, Nvy % BL == 0, even Nvy (16 B TMA strides),
// periodic-or-halo x/y, stored (frozen) velocity ghosts.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "tma.cuh"

namespace vpfv {



struct Stage22 {
    double *dest;
    double cL;
    const double *dt_dev;
    double cL_div;
    int nops;          // RK operands staged by TMA (A, B, dest as needed)
    double opc[3];     // their coefficients
    unsigned long long *nonfinite;
    const double *vxc, *vyc, *evx, *evy, *c1, *c3, *c4, *c5;
    double cB, c2, mhx, mhy, mhvx, mhvy;
    int Nx, Ny, Nvx, Nvy;
    int wrap_x, wrap_y;
    int i0, i1;        // x range of cells this launch updates (interior indices)
    int nseg, seglen;  // x segments per column block
    int sj, sk;        // super-tile of column blocks (block order)
    double *partials;  // moment partials [Nx][Ny][Nvx][Nvy/BL] or nullptr
};

template <int BJ, int BK, int BL, int NSTAGE>
struct Tile {
    static constexpr int J = BJ + 6, K = BK + 6, L = BL + 8;
    static constexpr int KL = K * L;
    static constexpr int ELEMS = J * K * L;              // src halo tile
    static constexpr int OL = BL + 2;                     // operand row (16 B aligned start)
    static constexpr int OELEMS = BJ * BK * OL;           // one RK operand core tile
    static constexpr int TELEMS = 3 * BJ * 8;              // packed E tables, planes p-1..p+1
    static constexpr int STAGE_ELEMS = ELEMS + 3 * OELEMS + TELEMS;
    static constexpr int TAB_BYTES = TELEMS * 8;
    static constexpr int HALO_BYTES = ELEMS * 8, OP_BYTES = OELEMS * 8;
    static constexpr int SMEM = NSTAGE * STAGE_ELEMS * 8 + 64;
    static constexpr int NSTAGE_ = NSTAGE, BJ_ = BJ, BK_ = BK, BL_ = BL;
    static_assert((ELEMS * 8) % 128 == 0 && (OELEMS * 8) % 128 == 0, "TMA destinations must stay 128 B aligned");
};

struct Maps {
    CUtensorMap core, halo, op[3], tab;
};

// upwinded 6-point weighted sum (face difference * 60) along an in-tile
// direction of stride ST, evaluated as three independent pairs (ILP); the
// sign test is warp-uniform in practice.
template <int ST>
__device__ __forceinline__ double wsum(const double *c, bool pos) {
    if (pos) {
        const double t1 = fma(15.0, c[-2 * ST], -2.0 * c[-3 * ST]);
        const double t2 = fma(20.0, c[0], -60.0 * c[-ST]);
        const double t3 = fma(-3.0, c[2 * ST], 30.0 * c[ST]);
        return (t1 + t2) + t3;
    }
    const double t1 = fma(-30.0, c[-ST], 3.0 * c[-2 * ST]);
    const double t2 = fma(60.0, c[ST], -20.0 * c[0]);
    const double t3 = fma(2.0, c[3 * ST], -15.0 * c[2 * ST]);
    return (t1 + t2) + t3;
}

template <int SA, int SB>
__device__ __forceinline__ double dsum(const double *c) {  // s[+a,-b]+s[-a,+b]-s[+a,+b]-s[-a,-b]
    return (c[SA - SB] + c[-SA + SB]) - (c[SA + SB] + c[-SA - SB]);
}

__device__ __forceinline__ double warp_tree_sum(double x) {
    for (int off = 1; off < 32; off <<= 1) x = __dadd_rn(x, __shfl_down_sync(0xffffffffu, x, off));
    return x;
}

// Plane n: the src halo tile of plane p = p_first + n, and the RK operand core
// tiles of cell-plane q = p - 3 when q is updated by this CTA.  The copies of
// one plane are split into parts (0: expect_tx + tables, 1-3: halo/core/halo,
// 4+o: operand o) so that a different warp issues each part and no warp
// carries the whole producer cost (the per-plane barrier waits for the
// slowest warp).  complete_tx may land before the expect_tx: the mbarrier
// transaction count is allowed to go transiently negative, and the phase
// cannot complete before part 0 arrives.
template <class TL>
__device__ __forceinline__ void issue_part(int w, double *stages, uint64_t *bars, const Maps *M, int n,
                                           int p_first, int i0, int i1, const Stage22 &P, int l0, int k0,
                                           int j0, int cy_lo, int cy_core, int cy_hi) {
    const int s = n % TL::NSTAGE_;
    double *dst = stages + s * TL::STAGE_ELEMS;
    const int p = p_first + n;  // in [-3, Nx + 3)
    int px = p;
    if (P.wrap_x) px = px < 0 ? px + P.Nx : (px >= P.Nx ? px - P.Nx : px);
    const int q = p - 3;
    const bool ops = (q >= i0 && q < i1);
    const int cx = px + NG;
    switch (w) {
        case 0:
            tma::mbar_expect_tx(&bars[s], TL::HALO_BYTES + TL::TAB_BYTES + (ops ? P.nops * TL::OP_BYTES : 0));
            // packed tables rows px..px+2 = planes p-1, p, p+1 (row = x + 1)
            tma::load3d(dst + TL::ELEMS + 3 * TL::OELEMS, &M->tab, &bars[s], 0, j0, px);
            break;
        case 1: tma::load4d(dst, &M->halo, &bars[s], l0, k0, cy_lo, cx); break;
        case 2: tma::load4d(dst + 3 * TL::KL, &M->core, &bars[s], l0, k0, cy_core, cx); break;
        case 3: tma::load4d(dst + (3 + TL::BJ_) * TL::KL, &M->halo, &bars[s], l0, k0, cy_hi, cx); break;
        default: {
            const int o = w - 4;
            if (ops && o < P.nops)
                tma::load4d(dst + TL::ELEMS + o * TL::OELEMS, &M->op[o], &bars[s], l0 + 2, k0 + NG, j0 + NG,
                            q + NG);
        }
    }
}

template <int BJ, int BK, int BL, int NSTAGE, int CK, int MINB>
__global__ void __launch_bounds__(BJ * (BK / CK) * BL, MINB)
    stage2d2v_tma_kernel(const __grid_constant__ Maps maps, const Stage22 P) {
    using TL = Tile<BJ, BK, BL, NSTAGE>;
    constexpr int L = TL::L, KL = TL::KL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + NSTAGE * TL::STAGE_ELEMS * 8);

    const int tid = threadIdx.x;
    // column block; x segment outermost so the CTAs resident at once cover
    // neighbouring column blocks of the same x range (halo reuse in L2)
    const int nlt = P.Nvy / BL, nkt = P.Nvx / BK, njt = P.Ny / BJ;
    const int ncols = nlt * nkt * njt;
    int b = blockIdx.x % ncols;
    const int seg = blockIdx.x / ncols;
    // L2-friendly order: all vy tiles of a (y, vx) column block are adjacent,
    // and column blocks are visited in (sj x sk) super-tiles, so a wave of
    // resident CTAs covers a compact (y, vx) region whose halos it shares
    const int lt = b % nlt;
    b /= nlt;
    const int sj = min(P.sj, njt), sk = min(P.sk, nkt);
    const int nsk = (nkt + sk - 1) / sk;
    const int st = b / (sj * sk), wi = b % (sj * sk);
    const int st_j = st / nsk, st_k = st % nsk;
    const int rows_j = min(sj, njt - st_j * sj), cols_k = min(sk, nkt - st_k * sk);
    const int jt = st_j * sj + (wi / cols_k) % rows_j;
    const int kt = st_k * sk + wi % cols_k;
    const int j0 = jt * BJ, k0 = kt * BK, l0 = lt * BL;
    const int i0 = P.i0 + seg * P.seglen;
    const int i1 = min(P.i1, i0 + P.seglen);
    if (i0 >= i1) return;

    // thread -> CK consecutive vx cells (a, kb .. kb+CK-1) at vy lane `lane`
    // of its BL-wide row group (BL = 32: one warp per row, 16: two rows)
    const int lane = tid % BL, colid = tid / BL;
    const int a = colid / (BK / CK);
    const int kb = (colid % (BK / CK)) * CK;
    const int jj = j0 + a;
    const int kfirst = k0 + kb;
    const int ll = l0 + lane;

    int yl = j0 - 3, yh = j0 + BJ;
    if (P.wrap_y) {
        if (yl < 0) yl += P.Ny;
        if (yh >= P.Ny) yh -= P.Ny;
    }
    const int cy_lo = yl + NG, cy_core = j0 + NG, cy_hi = yh + NG;

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) tma::mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int p_first = i0 - 3, p_last = i1 + 2;
    const int nplanes = p_last - p_first + 1;
    const Maps *M = &maps;
    if (tid == 0) {
        for (int n = 0; n < NSTAGE - 1 && n < nplanes; ++n)
            for (int w = 0; w < 7; ++w)
                issue_part<TL>(w, stages, bars, M, n, p_first, i0, i1, P, l0, k0, j0, cy_lo, cy_core, cy_hi);
    }
    const int warp = tid >> 5;
    const bool issuer = (tid & 31) == 0 && warp < 4 + P.nops;

    double ax_s[CK], bvx[CK];
    bool xpos[CK];
#pragma unroll
    for (int i = 0; i < CK; ++i) {
        const double v = __ldg(P.vxc + kfirst + i);
        ax_s[i] = v * P.mhx;
        xpos[i] = v > 0.0;
        bvx[i] = -P.cB * v;
    }
    const double vy = __ldg(P.vyc + ll);
    const double ay_s = vy * P.mhy;
    const bool ypos = vy > 0.0;
    const double cBvy = P.cB * vy;
    const double cL = P.dt_dev ? __ddiv_rn(*P.dt_dev, P.cL_div) : P.cL;
    const double mc2 = -P.c2, mhvx = P.mhvx, mhvy = P.mhvy;
    const int nops = P.nops;
    const double oc0 = P.opc[0], oc1 = P.opc[1], oc2 = P.opc[2];

    const int off = ((a + 3) * TL::K + (kb + 3)) * L + (lane + 3);   // first cell in the halo tile
    const int ooff = TL::ELEMS + (a * BK + kb) * TL::OL + lane + 1;  // first cell in operand tile 0

    const long long P3 = P.Nvy + 2 * NG, P2 = (long long)(P.Nvx + 2 * NG) * P3,
                    P1 = (long long)(P.Ny + 2 * NG) * P2;
    long long gq = (long long)(p_first - 3 + NG) * P1 + (long long)(jj + NG) * P2 +
                   (long long)(kfirst + NG) * P3 + (ll + NG);  // cell q = p - 3

    double acc[CK][7];
#pragma unroll
    for (int i = 0; i < CK; ++i)
#pragma unroll
        for (int m = 0; m < 7; ++m) acc[i][m] = 0.0;

    int stage_s = 0;
    unsigned stage_par = 0;
    // Accumulator ring: cell c = p_first + m lives in slot m % 7; the plane
    // loop is unrolled by 7 so every slot index is a compile-time constant.
    for (int blk = 0; blk < nplanes; blk += 7) {
#pragma unroll
        for (int r = 0; r < 7; ++r) {
            const int n = blk + r;
            if (n >= nplanes) break;
            const int p = p_first + n;
            if (issuer && n + NSTAGE - 1 < nplanes)
                issue_part<TL>(warp, stages, bars, M, n + NSTAGE - 1, p_first, i0, i1, P, l0, k0, j0, cy_lo,
                               cy_core, cy_hi);
            // no range tests: contributions of halo planes land in accumulator
            // slots of cells outside [i0, i1), which are never finalised
            const int s = stage_s;
            tma::mbar_wait(&bars[s], stage_par);
            if (++stage_s == NSTAGE) {
                stage_s = 0;
                stage_par ^= 1u;
            }
            const double *stage = stages + s * TL::STAGE_ELEMS;
            const double *c0 = stage + off;
            const double *tb = stage + TL::ELEMS + 3 * TL::OELEMS + a * 8;  // row p-1, this j
            const double evx = tb[BJ * 8 + 0], evy = tb[BJ * 8 + 1];
            const double c3 = tb[BJ * 8 + 3], c4 = tb[BJ * 8 + 4];
            const double c1m = tb[2], c5m = tb[5];
            const double c1p = tb[2 * BJ * 8 + 2], c5p = tb[2 * BJ * 8 + 5];

            const double avx = evx + cBvy;
            const double avx_s = avx * mhvx;
            const bool vxpos = avx > 0.0;
            // register reuse along vx: the (j, l) column k = kb-3 .. kb+CK+2 and
            // the j+-1 columns k = kb-1 .. kb+CK (y stencil + (y,vx) diagonal)
            double col[CK + 6], cyp[CK + 2], cym[CK + 2];
#pragma unroll
            for (int m = 0; m < CK + 6; ++m) col[m] = c0[(m - 3) * L];
#pragma unroll
            for (int m = 0; m < CK + 2; ++m) {
                cyp[m] = c0[KL + (m - 1) * L];
                cym[m] = c0[-KL + (m - 1) * L];
            }
#pragma unroll
            for (int i = 0; i < CK; ++i) {
                const double *c = c0 + i * L;
                // x-stencil contribution of s(p) to cells p - o: slot (r - o) mod 7
                const double t = ax_s[i] * col[i + 3];
#ifdef VPFV_EXP_SKIP_X
                if (P.Nx < 0) {
#else
                if (xpos[i]) {
#endif
                    acc[i][(r + 10) % 7] = fma(-2.0, t, acc[i][(r + 10) % 7]);
                    acc[i][(r + 9) % 7] = fma(15.0, t, acc[i][(r + 9) % 7]);
                    acc[i][(r + 8) % 7] = fma(-60.0, t, acc[i][(r + 8) % 7]);
                    acc[i][r] = fma(20.0, t, acc[i][r]);
                    acc[i][(r + 6) % 7] = fma(30.0, t, acc[i][(r + 6) % 7]);
                    acc[i][(r + 5) % 7] = fma(-3.0, t, acc[i][(r + 5) % 7]);
                } else {
                    acc[i][(r + 9) % 7] = fma(3.0, t, acc[i][(r + 9) % 7]);
                    acc[i][(r + 8) % 7] = fma(-30.0, t, acc[i][(r + 8) % 7]);
                    acc[i][r] = fma(-20.0, t, acc[i][r]);
                    acc[i][(r + 6) % 7] = fma(60.0, t, acc[i][(r + 6) % 7]);
                    acc[i][(r + 5) % 7] = fma(-15.0, t, acc[i][(r + 5) % 7]);
                    acc[i][(r + 4) % 7] = fma(2.0, t, acc[i][(r + 4) % 7]);
                }
                // x-coupled corrections: D(p) = s[k-1]-s[k+1], G(p) = s[l-1]-s[l+1]
#ifndef VPFV_EXP_SKIP_DG
                const double D = col[i + 2] - col[i + 4];
                const double G = c[-1] - c[1];
                acc[i][(r + 6) % 7] = fma(c1m, D, fma(-c5m, G, acc[i][(r + 6) % 7]));
                acc[i][(r + 1) % 7] = fma(-c1p, D, fma(c5p, G, acc[i][(r + 1) % 7]));
#endif
#ifdef VPFV_EXP_SKIP_T
                if (P.Nx < 0)
#endif
                {
                    const double avy = evy + bvx[i];
                    double wy, wvx;
                    if (ypos) {
                        wy = (fma(15.0, c[-2 * KL], -2.0 * c[-3 * KL]) + fma(20.0, col[i + 3], -60.0 * cym[i + 1])) +
                             fma(-3.0, c[2 * KL], 30.0 * cyp[i + 1]);
                    } else {
                        wy = (fma(-30.0, cym[i + 1], 3.0 * c[-2 * KL]) + fma(60.0, cyp[i + 1], -20.0 * col[i + 3])) +
                             fma(2.0, c[3 * KL], -15.0 * c[2 * KL]);
                    }
                    if (vxpos) {
                        wvx = (fma(15.0, col[i + 1], -2.0 * col[i]) + fma(20.0, col[i + 3], -60.0 * col[i + 2])) +
                              fma(-3.0, col[i + 5], 30.0 * col[i + 4]);
                    } else {
                        wvx = (fma(-30.0, col[i + 2], 3.0 * col[i + 1]) + fma(60.0, col[i + 4], -20.0 * col[i + 3])) +
                              fma(2.0, col[i + 6], -15.0 * col[i + 5]);
                    }
                    const double Ty = ay_s * wy;
                    const double Tvx = avx_s * wvx;
                    const double Tvy = (avy * mhvy) * wsum<1>(c, avy > 0.0);
                    const double dyvx = (cyp[i] + cym[i + 2]) - (cyp[i + 2] + cym[i]);
                    const double Tc = fma(c4, dsum<KL, 1>(c), fma(mc2, dsum<L, 1>(c), -c3 * dyvx));
                    acc[i][r] += (Ty + Tvx) + (Tvy + Tc);
                }
            }
            // finalise cells q = p - 3 (slot (r + 4) % 7) from the staged RK operands
            const int q = p - 3;
            if (q >= i0 && q < i1) {
                const double *op = stage + ooff;
                double out[CK];
#pragma unroll
                for (int i = 0; i < CK; ++i) {
                    double rk = oc0 * op[i * TL::OL];
                    if (nops > 1) rk = fma(oc1, op[TL::OELEMS + i * TL::OL], rk);
                    if (nops > 2) rk = fma(oc2, op[2 * TL::OELEMS + i * TL::OL], rk);
                    out[i] = fma(cL, acc[i][(r + 4) % 7], rk);
                    P.dest[gq + i * P3] = out[i];
                }
                if (P.nonfinite) {
#pragma unroll
                    for (int i = 0; i < CK; ++i)
                        if (!isfinite(out[i]))
                            atomicMin(P.nonfinite,
                                      (((unsigned long long)q * P.Ny + jj) * P.Nvx + kfirst + i) * P.Nvy + ll);
                }
#ifdef VPFV_EXP_SKIP_PARTIALS
                if (P.partials && P.Nx < 0) {
#else
                if (P.partials) {
#endif
                    // fold-tree subtrees of two rows at once: lanes pair up
                    // (even lane keeps row i, odd lane row i+1), then the usual
                    // ascending shuffle levels on one register
                    const long long pb = ((long long)q * P.Ny + jj) * P.Nvx + kfirst;
                    const bool odd = lane & 1;
#pragma unroll
                    for (int i = 0; i < CK; i += 2) {
                        const double keep = odd ? out[i + 1] : out[i];
                        const double send = odd ? out[i] : out[i + 1];
                        double v = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1, BL));
#pragma unroll
                        for (int off = 2; off < BL; off <<= 1)
                            v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off, BL));
                        if (lane < 2) P.partials[(pb + i + lane) * nlt + lt] = v;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < CK; ++i) acc[i][(r + 4) % 7] = 0.0;
            gq += P1;
            __syncthreads();  // stage s is free for the next refill
        }
    }
}

// ---------------------------------------------------------------------------
// moment from partials: per physical cell, fold over the vy chunks of every
// vx row (chunk sums are exact 32-wide subtrees), then over vx, times vol.

__device__ double fold_small(double *x, int n) {  // single thread, in place
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

__global__ void moment_partials_kernel(const double *__restrict__ part, double *__restrict__ n,
                                       int nphys, int nvx, int nlt, double vol) {
    extern __shared__ double sm[];  // per warp: two buffers of nvx
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int p = blockIdx.x * wpb + warp;
    if (p >= nphys) return;
    double *bufA = sm + (size_t)warp * 2 * nvx, *bufB = bufA + nvx;
    const double *src = part + (size_t)p * nvx * nlt;
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
    if (lane == 0) n[p] = __dmul_rn(a[0], vol);
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launch

// Tile configurations: (BJ, BL, NSTAGE, CK) with BK = 8.  Chosen at run time
// (VPFV_TCFG overrides; default 0).
constexpr int TBK = 8;
struct TCfg {
    int bj, bl, ns, ck;
};
static const TCfg kCfgs[] = {{4, 32, 3, 2}, {8, 16, 3, 2}, {4, 32, 2, 2}, {4, 16, 2, 2}, {2, 32, 2, 2}};

static int tile_cfg() {
    static int c = -1;
    if (c < 0) {
        const char *e = getenv("VPFV_TCFG");
        c = e ? atoi(e) : 0;
        if (c < 0 || c > 4) c = 0;
    }
    return c;
}

int tma_2d2v_chunk() { return kCfgs[tile_cfg()].bl; }

bool tma_2d2v_eligible(int Nx, int Ny, int Nvx, int Nvy, unsigned flags) {
    const TCfg &c = kCfgs[tile_cfg()];
    if (flags & VPFV_EXACT) return false;
    if (flags & (VPFV_WRAP(2) | VPFV_WRAP(3))) return false;  // velocity ghosts must be stored
    if (Ny % c.bj || Nvx % TBK || Nvy % c.bl || (Nvy & 1)) return false;
    if (Nx < 1 || Ny < 3 + c.bj) return false;
    return tma_available();
}

int tma_2d2v_columns(int Ny, int Nvx, int Nvy) {
    const TCfg &c = kCfgs[tile_cfg()];
    return (Ny / c.bj) * (Nvx / TBK) * (Nvy / c.bl);
}

template <int BJ, int BL, int NS, int CK, int MINB = 1>
static int launch_cfg(const Maps &maps, const Stage22 &P, cudaStream_t s) {
    using TL = Tile<BJ, TBK, BL, NS>;
    auto kern = stage2d2v_tma_kernel<BJ, TBK, BL, NS, CK, MINB>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, TL::SMEM);
        attr = true;
    }
    const int nblocks = (P.Ny / BJ) * (P.Nvx / TBK) * (P.Nvy / BL) * P.nseg;
    kern<<<nblocks, BJ * (TBK / CK) * BL, TL::SMEM, s>>>(maps, P);
    return check_launch("stage_2d2v_tma");
}

// ops: up to three (coefficient, array) RK operands, already de-duplicated
int launch_tma_2d2v(const double *src, const double *const ops[3], const double *tab, Stage22 P,
                    unsigned flags, int nseg, cudaStream_t s) {
    const TCfg &c = kCfgs[tile_cfg()];
    const int Npad[4] = {P.Nx + 6, P.Ny + 6, P.Nvx + 6, P.Nvy + 6};
    const int box_core[4] = {c.bl + 8, TBK + 6, c.bj, 1};
    const int box_halo[4] = {c.bl + 8, TBK + 6, 3, 1};
    const int box_op[4] = {c.bl + 2, TBK, c.bj, 1};
    Maps maps;
    // 4D fp64 padded arrays, innermost (vy) first
    const unsigned long long dims[4] = {(unsigned long long)Npad[3], (unsigned long long)Npad[2],
                                        (unsigned long long)Npad[1], (unsigned long long)Npad[0]};
    const unsigned long long strides[3] = {dims[0] * 8, dims[0] * dims[1] * 8, dims[0] * dims[1] * dims[2] * 8};
    auto box4 = [](const int *b) {
        struct B {
            unsigned v[4];
        } r{{(unsigned)b[0], (unsigned)b[1], (unsigned)b[2], (unsigned)b[3]}};
        return r;
    };
    const auto bc = box4(box_core), bh = box4(box_halo), bo = box4(box_op);
    if (!tma_map(src, 4, dims, strides, bc.v, &maps.core) || !tma_map(src, 4, dims, strides, bh.v, &maps.halo))
        return set_error(VPFV_ECUDA, "cuTensorMapEncodeTiled failed");
    for (int o = 0; o < P.nops; ++o)
        if (!tma_map(ops[o], 4, dims, strides, bo.v, &maps.op[o]))
            return set_error(VPFV_ECUDA, "cuTensorMapEncodeTiled failed");
    for (int o = P.nops; o < 3; ++o) maps.op[o] = maps.core;
    // packed tables [(Nx+2)][Ny][8]
    const unsigned long long tdims[3] = {8, (unsigned long long)P.Ny, (unsigned long long)P.Nx + 2};
    const unsigned long long tstr[2] = {64, (unsigned long long)P.Ny * 64};
    const unsigned tbox[3] = {8, (unsigned)c.bj, 3};
    if (!tma_map(tab, 3, tdims, tstr, tbox, &maps.tab)) return set_error(VPFV_ECUDA, "table map failed");
    P.wrap_x = (flags & VPFV_WRAP(0)) != 0;
    P.wrap_y = (flags & VPFV_WRAP(1)) != 0;
    P.i0 = 0;
    P.i1 = P.Nx;
    P.nseg = nseg < 1 ? 1 : nseg;
    P.seglen = (P.Nx + P.nseg - 1) / P.nseg;
    static int sjk[2] = {-1, -1};
    if (sjk[0] < 0) {
        const char *e = getenv("VPFV_SUPER");
        sjk[0] = 8;
        sjk[1] = 4;
        if (e) sscanf(e, "%d,%d", &sjk[0], &sjk[1]);
    }
    P.sj = sjk[0] > 0 ? sjk[0] : 1;
    P.sk = sjk[1] > 0 ? sjk[1] : 1;
    switch (tile_cfg()) {
        case 1: return launch_cfg<8, 16, 3, 2>(maps, P, s);
        case 2: return launch_cfg<4, 32, 2, 2>(maps, P, s);
        case 3: return launch_cfg<4, 16, 2, 2, 2>(maps, P, s);
        case 4: return launch_cfg<2, 32, 2, 2, 2>(maps, P, s);
        default: return launch_cfg<4, 32, 3, 2>(maps, P, s);
    }
}

int launch_moment_from_partials(const double *part, double *n, int nphys, int nvx, int nlt, double vol,
                                cudaStream_t s) {
    if (nlt > 16) return set_error(VPFV_EARG, "moment partials: at most 16 vy chunks");
    const int wpb = 4;
    size_t smem = sizeof(double) * (size_t)wpb * 2 * nvx;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(moment_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    moment_partials_kernel<<<(nphys + wpb - 1) / wpb, 32 * wpb, smem, s>>>(part, n, nphys, nvx, nlt, vol);
    return check_launch("moment_from_partials");
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_stage_2d2v_generic(double *, const double *, const double *, const double *, double,
                                       double, double, double, const double *, const double *,
                                       const double *, const double *, double, const double *, double,
                                       const double *, const double *, const double *, double, double,
                                       double, double, int, int, int, int, unsigned, const double *,
                                       double, unsigned long long *, void *);

extern "C" int vpfv_stage_2d2v_fused(double *dest, const double *A, const double *B,
                                     const double *src, double ca, double cb, double cd, double cL,
                                     const double *vxc, const double *vyc, const double *evx,
                                     const double *evy, double cB, const double *c1, double c2,
                                     const double *c3, const double *c4, const double *c5, double hx,
                                     double hy, double hvx, double hvy, int Nx, int Ny, int Nvx,
                                     int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, const double *packed_tables,
                                     double *moment_partials, int xsegments, void *stream) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (!packed_tables || !tma_2d2v_eligible(Nx, Ny, Nvx, Nvy, flags)) {
        if (moment_partials) return set_error(VPFV_EARG, "fused moment needs the tiled 2D-2V path");
        return vpfv_stage_2d2v_generic(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2,
                                       c3, c4, c5, hx, hy, hvx, hvy, Nx, Ny, Nvx, Nvy, flags, dt_dev,
                                       cL_div, nonfinite, stream);
    }
    Stage22 P{};
    P.dest = dest;
    P.cL = cL;
    P.dt_dev = dt_dev;
    P.cL_div = cL_div;
    // RK operands: ca*A + cb*B + cd*dest, merging B into A when they alias
    const double *ops[3] = {nullptr, nullptr, nullptr};
    int nops = 0;
    if (ca != 0.0 || (cb != 0.0 && B == A)) {
        ops[nops] = A;
        P.opc[nops++] = (B == A) ? ca + cb : ca;
    }
    if (cb != 0.0 && B != A) {
        ops[nops] = B;
        P.opc[nops++] = cb;
    }
    if (cd != 0.0) {
        ops[nops] = dest;
        P.opc[nops++] = cd;
    }
    if (nops == 0) {  // pure RHS: one zero-weighted operand keeps the code path uniform
        ops[nops] = src;
        P.opc[nops++] = 0.0;
    }
    P.nops = nops;
    P.nonfinite = nonfinite;
    P.vxc = vxc;
    P.vyc = vyc;
    P.evx = evx;
    P.evy = evy;
    P.c1 = c1;
    P.c3 = c3;
    P.c4 = c4;
    P.c5 = c5;
    P.cB = cB;
    P.c2 = c2;
    P.mhx = -1.0 / (60.0 * hx);
    P.mhy = -1.0 / (60.0 * hy);
    P.mhvx = -1.0 / (60.0 * hvx);
    P.mhvy = -1.0 / (60.0 * hvy);
    P.Nx = Nx;
    P.Ny = Ny;
    P.Nvx = Nvx;
    P.Nvy = Nvy;
    P.partials = moment_partials;
    int nseg = xsegments;
    static int env_seg = -1;
    if (env_seg < 0) {
        const char *e = getenv("VPFV_XSEG");
        env_seg = e ? atoi(e) : 0;
    }
    if (nseg <= 0 && env_seg > 0) nseg = env_seg;
    if (nseg <= 0) {  // at least ~4 waves of one CTA per SM, segments >= 8 planes
        const int cols = tma_2d2v_columns(Ny, Nvx, Nvy);
        nseg = (4 * 148 + cols - 1) / cols;
        if (nseg > Nx / 8) nseg = Nx / 8;
        if (nseg < 1) nseg = 1;
    }
    return launch_tma_2d2v(src, ops, packed_tables, P, flags, nseg, (cudaStream_t)stream);
}

extern "C" int vpfv_moment_partials(const double *partials, double *n, int nphys, int Nvx, int nchunks,
                                    double vol, void *stream) {
    return launch_moment_from_partials(partials, n, nphys, Nvx, nchunks, vol, (cudaStream_t)stream);
}

extern "C" int vpfv_stage_2d2v_tiled_ok(int Nx, int Ny, int Nvx, int Nvy, unsigned flags) {
    return tma_2d2v_eligible(Nx, Ny, Nvx, Nvy, flags) && Nvy / tma_2d2v_chunk() <= 16 ? 1 : 0;
}

extern "C" int vpfv_stage_2d2v_partials_chunk(void) { return tma_2d2v_chunk(); }
