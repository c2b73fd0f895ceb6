// 1D-2V fused stage, x-marching with TMA-staged (vx, vy) halo tiles (fast path).
//
// Operator of stage_1d2v (/root/reference/pkg/src/vpfv/_kernels.py:153-197):
//   rhs = -a_x D_x f - a_vx D_vx f - a_vy D_vy f + c1 diag(x,vx) - c2 diag(vx,vy)
// with a_x = vxc[j], a_vx = evx[i] + cB vyc[k], a_vy = avy[j].  Same
// organisation as the 2D-2V kernel (stage2d2v_tma.cu): a CTA owns a (vx, vy)
// = (BK, BL) column block and marches x; per plane one TMA box brings the
// (BK+6) x (BL+8) halo tile, up to three RK-operand core boxes and the packed
// (evx, c1) table rows of planes p-1..p+1; each thread keeps 7 register
// accumulators per cell (plane loop unrolled x7) and CK consecutive vx cells
// share one vx column of registers; the x-coupled (x,vx) correction uses
// D(p) = s[k-1] - s[k+1]; the optional epilogue emits fold-tree moment
// partials per 32-wide vy chunk.
#include "common.cuh"
#include "tma.cuh"

namespace vpfv {

struct Stage12 {
    double *dest;
    double cL;
    const double *dt_dev;
    double cL_div;
    int nops;
    double opc[3];
    unsigned long long *nonfinite;
    const double *vxc, *vyc, *avy;
    double cB, c2, mhx, mhvx, mhvy;
    int Nx, Nvx, Nvy;
    int wrap_x;
    int i0, i1, nseg, seglen;
    double *partials;  // [Nx][Nvx][Nvy/BL] or nullptr
};

struct Maps12 {
    CUtensorMap halo, op[3], tab;
};

template <int BK, int BL, int NSTAGE>
struct Tile12 {
    static constexpr int K = BK + 6, L = BL + 8;
    static constexpr int ELEMS = K * L;
    static constexpr int OL = BL + 2;
    static constexpr int OELEMS = BK * OL;
    static constexpr int TELEMS = 32;  // 3 table rows of 8, padded to 256 B
    static constexpr int STAGE_ELEMS = ELEMS + 3 * OELEMS + TELEMS;
    static constexpr int SMEM = NSTAGE * STAGE_ELEMS * 8 + 64;
    static_assert((ELEMS * 8) % 128 == 0 && (OELEMS * 8) % 128 == 0, "TMA destinations must stay 128 B aligned");
};

// Copies of plane n split into parts issued by different warps (see
// issue_part in stage2d2v_tma.cu): 0 = expect_tx + tables, 1 = halo, 2+o =
// RK operand o.
template <class TL>
__device__ __forceinline__ void issue12(int w, double *stages, uint64_t *bars, const Maps12 *M, int n,
                                        int p_first, int i0, int i1, const Stage12 &P, int l0, int k0,
                                        int nstage) {
    const int s = n % nstage;
    double *dst = stages + s * TL::STAGE_ELEMS;
    const int p = p_first + n;  // in [-3, Nx + 3)
    int px = p;
    if (P.wrap_x) px = px < 0 ? px + P.Nx : (px >= P.Nx ? px - P.Nx : px);
    const int q = p - 3;
    const bool ops = (q >= i0 && q < i1);
    if (w == 0) {
        tma::mbar_expect_tx(&bars[s], (TL::ELEMS + 24 + (ops ? P.nops * TL::OELEMS : 0)) * 8);
        tma::load2d(dst + TL::ELEMS + 3 * TL::OELEMS, &M->tab, &bars[s], 0, px);
    } else if (w == 1) {
        tma::load3d(dst, &M->halo, &bars[s], l0, k0, px + NG);
    } else if (ops && w - 2 < P.nops) {
        const int o = w - 2;
        tma::load3d(dst + TL::ELEMS + o * TL::OELEMS, &M->op[o], &bars[s], l0 + 2, k0 + NG, q + NG);
    }
}

template <int BK, int BL, int NSTAGE, int CK>
__global__ void __launch_bounds__((BK / CK) * BL, 1)
    stage1d2v_tma_kernel(const __grid_constant__ Maps12 maps, const Stage12 P) {
    using TL = Tile12<BK, BL, NSTAGE>;
    constexpr int L = TL::L;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + NSTAGE * TL::STAGE_ELEMS * 8);

    const int tid = threadIdx.x;
    const int nlt = P.Nvy / BL, nkt = P.Nvx / BK;
    const int ncols = nlt * nkt;
    const int b = blockIdx.x % ncols, seg = blockIdx.x / ncols;
    const int lt = b % nlt, kt = b / nlt;
    const int k0 = kt * BK, l0 = lt * BL;
    const int i0 = P.i0 + seg * P.seglen;
    const int i1 = min(P.i1, i0 + P.seglen);
    if (i0 >= i1) return;

    const int lane = tid % BL, colid = tid / BL;
    const int kb = colid * CK;
    const int kfirst = k0 + kb;
    const int ll = l0 + lane;

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) tma::mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int p_first = i0 - 3, nplanes = i1 - i0 + 6;
    const Maps12 *M = &maps;
    if (tid == 0)
        for (int n = 0; n < NSTAGE - 1 && n < nplanes; ++n)
            for (int w = 0; w < 5; ++w) issue12<TL>(w, stages, bars, M, n, p_first, i0, i1, P, l0, k0, NSTAGE);
    const int warp = tid >> 5;
    const bool issuer = (tid & 31) == 0 && warp < 2 + P.nops;

    double ax_s[CK], avy_s[CK];
    bool xpos[CK], vypos[CK];
#pragma unroll
    for (int i = 0; i < CK; ++i) {
        const double v = __ldg(P.vxc + kfirst + i);
        ax_s[i] = v * P.mhx;
        xpos[i] = v > 0.0;
        const double ay = __ldg(P.avy + kfirst + i);
        avy_s[i] = ay * P.mhvy;
        vypos[i] = ay > 0.0;
    }
    const double cBvy = __ldg(P.vyc + P.Nvy) * __ldg(P.vyc + ll);  // cB rides in vyc[Nvy] (_kernels.py:166)
    const double cL = P.dt_dev ? __ddiv_rn(*P.dt_dev, P.cL_div) : P.cL;
    const double mc2 = -P.c2, mhvx = P.mhvx;
    const int nops = P.nops;
    const double oc0 = P.opc[0], oc1 = P.opc[1], oc2 = P.opc[2];
    const int off = (kb + 3) * L + lane + 3;
    const int ooff = TL::ELEMS + kb * TL::OL + lane + 1;
    const long long P2 = P.Nvy + 2 * NG, P1 = (long long)(P.Nvx + 2 * NG) * P2;
    long long gq = (long long)(p_first - 3 + NG) * P1 + (long long)(kfirst + NG) * P2 + (ll + NG);

    double acc[CK][7];
#pragma unroll
    for (int i = 0; i < CK; ++i)
#pragma unroll
        for (int m = 0; m < 7; ++m) acc[i][m] = 0.0;
    int stage_s = 0;
    unsigned stage_par = 0;

    for (int blk = 0; blk < nplanes; blk += 7) {
#pragma unroll
        for (int r = 0; r < 7; ++r) {
            const int n = blk + r;
            if (n >= nplanes) break;
            const int p = p_first + n;
            if (issuer && n + NSTAGE - 1 < nplanes)
                issue12<TL>(warp, stages, bars, M, n + NSTAGE - 1, p_first, i0, i1, P, l0, k0, NSTAGE);
            const int s = stage_s;
            tma::mbar_wait(&bars[s], stage_par);
            if (++stage_s == NSTAGE) {
                stage_s = 0;
                stage_par ^= 1u;
            }
            const double *stage = stages + s * TL::STAGE_ELEMS;
            const double *c0 = stage + off;
            const double *tb = stage + TL::ELEMS + 3 * TL::OELEMS;  // rows p-1, p, p+1: (evx, c1)
            const double evx = tb[8], c1m = tb[1], c1p = tb[17];
            const double avx = evx + cBvy;
            const double avx_s = avx * mhvx;
            const bool vxpos = avx > 0.0;
            double col[CK + 6];
#pragma unroll
            for (int m = 0; m < CK + 6; ++m) col[m] = c0[(m - 3) * L];
#pragma unroll
            for (int i = 0; i < CK; ++i) {
                const double *c = c0 + i * L;
                const double t = ax_s[i] * col[i + 3];
                if (xpos[i]) {
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
                const double D = col[i + 2] - col[i + 4];
                acc[i][(r + 6) % 7] = fma(c1m, D, acc[i][(r + 6) % 7]);
                acc[i][(r + 1) % 7] = fma(-c1p, D, acc[i][(r + 1) % 7]);
                double wvx, wvy;
                if (vxpos)
                    wvx = (fma(15.0, col[i + 1], -2.0 * col[i]) + fma(20.0, col[i + 3], -60.0 * col[i + 2])) +
                          fma(-3.0, col[i + 5], 30.0 * col[i + 4]);
                else
                    wvx = (fma(-30.0, col[i + 2], 3.0 * col[i + 1]) + fma(60.0, col[i + 4], -20.0 * col[i + 3])) +
                          fma(2.0, col[i + 6], -15.0 * col[i + 5]);
                if (vypos[i])
                    wvy = (fma(15.0, c[-2], -2.0 * c[-3]) + fma(20.0, c[0], -60.0 * c[-1])) + fma(-3.0, c[2], 30.0 * c[1]);
                else
                    wvy = (fma(-30.0, c[-1], 3.0 * c[-2]) + fma(60.0, c[1], -20.0 * c[0])) + fma(2.0, c[3], -15.0 * c[2]);
                const double dvv = (c[L - 1] + c[-L + 1]) - (c[L + 1] + c[-L - 1]);
                acc[i][r] = fma(avx_s, wvx, fma(avy_s[i], wvy, fma(mc2, dvv, acc[i][r])));
            }
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
                    P.dest[gq + i * P2] = out[i];
                }
                if (P.nonfinite) {
#pragma unroll
                    for (int i = 0; i < CK; ++i)
                        if (!isfinite(out[i]))
                            atomicMin(P.nonfinite, ((unsigned long long)q * P.Nvx + kfirst + i) * P.Nvy + ll);
                }
                if (P.partials) {
                    const long long pb = (long long)q * P.Nvx + kfirst;
                    const bool odd = lane & 1;
#pragma unroll
                    for (int i = 0; i < CK; i += 2) {
                        const double keep = odd ? out[i + 1] : out[i];
                        const double send = odd ? out[i] : out[i + 1];
                        double v = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1, BL));
#pragma unroll
                        for (int o = 2; o < BL; o <<= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o, BL));
                        if (lane < 2) P.partials[(pb + i + lane) * nlt + lt] = v;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < CK; ++i) acc[i][(r + 4) % 7] = 0.0;
            gq += P1;
            __syncthreads();
        }
    }
}

constexpr int T12K = 32, T12L = 32, T12NS = 3, T12CK = 2;
using Tile12Cfg = Tile12<T12K, T12L, T12NS>;

bool tma_1d2v_eligible(int Nx, int Nvx, int Nvy, unsigned flags) {
    if (flags & VPFV_EXACT) return false;
    if (flags & (VPFV_WRAP(1) | VPFV_WRAP(2))) return false;
    if (Nvx % T12K || Nvy % T12L || Nx < 1 || Nvy / T12L > 16) return false;
    return tma_available();
}

}  // namespace vpfv

using namespace vpfv;

extern "C" int vpfv_stage_1d2v(double *, const double *, const double *, const double *, double, double,
                               double, double, const double *, const double *, const double *,
                               const double *, const double *, double, double, double, double, int, int,
                               int, unsigned, const double *, double, unsigned long long *, void *);

extern "C" int vpfv_stage_1d2v_tiled_ok(int Nx, int Nvx, int Nvy, unsigned flags) {
    return tma_1d2v_eligible(Nx, Nvx, Nvy, flags) ? 1 : 0;
}

extern "C" int vpfv_tables_1d_packed(const double *Ex, double *packed, int Nx, double qmk2, double g,
                                     double t1, double den1, void *stream);

extern "C" int vpfv_stage_1d2v_fused(double *dest, const double *A, const double *B, const double *src,
                                     double ca, double cb, double cd, double cL, const double *vxc,
                                     const double *vyc, const double *evx, const double *avy,
                                     const double *c1, double c2, double hx, double hvx, double hvy, int Nx,
                                     int Nvx, int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, const double *packed_tables,
                                     double *moment_partials, int xsegments, void *stream) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (!packed_tables || !tma_1d2v_eligible(Nx, Nvx, Nvy, flags)) {
        if (moment_partials) return set_error(VPFV_EARG, "fused moment needs the tiled 1D-2V path");
        return vpfv_stage_1d2v(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, avy, c1, c2, hx, hvx, hvy, Nx,
                               Nvx, Nvy, flags, dt_dev, cL_div, nonfinite, stream);
    }
    Stage12 P{};
    P.dest = dest;
    P.cL = cL;
    P.dt_dev = dt_dev;
    P.cL_div = cL_div;
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
    if (nops == 0) {
        ops[nops] = src;
        P.opc[nops++] = 0.0;
    }
    P.nops = nops;
    P.nonfinite = nonfinite;
    P.vxc = vxc;
    P.vyc = vyc;
    P.avy = avy;
    P.c2 = c2;
    P.mhx = -1.0 / (60.0 * hx);
    P.mhvx = -1.0 / (60.0 * hvx);
    P.mhvy = -1.0 / (60.0 * hvy);
    P.Nx = Nx;
    P.Nvx = Nvx;
    P.Nvy = Nvy;
    P.wrap_x = (flags & VPFV_WRAP(0)) != 0;
    P.partials = moment_partials;
    P.i0 = 0;
    P.i1 = Nx;
    const int cols = (Nvx / T12K) * (Nvy / T12L);
    int nseg = xsegments;
    if (nseg <= 0) {
        nseg = (4 * 148 + cols - 1) / cols;
        if (nseg > Nx / 8) nseg = Nx / 8;
        if (nseg < 1) nseg = 1;
    }
    P.nseg = nseg;
    P.seglen = (Nx + nseg - 1) / nseg;
    Maps12 maps;
    const unsigned long long dims[3] = {(unsigned long long)Nvy + 6, (unsigned long long)Nvx + 6,
                                        (unsigned long long)Nx + 6};
    const unsigned long long strides[2] = {dims[0] * 8, dims[0] * dims[1] * 8};
    const unsigned bh[3] = {T12L + 8, T12K + 6, 1}, bo[3] = {T12L + 2, T12K, 1};
    if (!tma_map(src, 3, dims, strides, bh, &maps.halo)) return set_error(VPFV_ECUDA, "tensor map failed");
    for (int o = 0; o < nops; ++o)
        if (!tma_map(ops[o], 3, dims, strides, bo, &maps.op[o])) return set_error(VPFV_ECUDA, "tensor map failed");
    for (int o = nops; o < 3; ++o) maps.op[o] = maps.halo;
    const unsigned long long tdims[2] = {8, (unsigned long long)Nx + 2};
    const unsigned long long tstr[1] = {64};
    const unsigned tbox[2] = {8, 3};
    if (!tma_map(packed_tables, 2, tdims, tstr, tbox, &maps.tab)) return set_error(VPFV_ECUDA, "table map failed");
    auto kern = stage1d2v_tma_kernel<T12K, T12L, T12NS, T12CK>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tile12Cfg::SMEM);
        attr = true;
    }
    const int nblocks = cols * nseg;
    kern<<<nblocks, (T12K / T12CK) * T12L, Tile12Cfg::SMEM, (cudaStream_t)stream>>>(maps, P);
    return check_launch("stage_1d2v_tma");
}
