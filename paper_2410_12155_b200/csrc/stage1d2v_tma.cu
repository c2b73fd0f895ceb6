// 1D-2V fused stage: x-marching, TMA-staged (vx, vy) halo tiles, 8-cell
// (default) or 4-cell register blocks (sm_100a, fast arithmetic path).
//
// Operator of stage_1d2v (/root/reference/pkg/src/vpfv/_kernels.py:153-197):
//   rhs = -a_x D_x f - a_vx D_vx f - a_vy D_vy f + c1 diag(x,vx) - c2 diag(vx,vy)
//   dest = ca A + cb B + cd dest + cL rhs                 (interior cells only)
// with a_x = vxc[j], a_vx = evx[i] + cB vyc[k], a_vy = avy[j].
//
// The 2D-2V kernel's design (stage2d2v_tma.cu) with no y direction:
//  * a CTA (64 threads, 4 per SM; round 1: 128 threads, 3 per SM) owns a
//    (vx, vy) = (32, 16) column block
//    and marches x; each thread keeps, per cell, a sliding window of 6 fp64
//    accumulators (cells p-3..p+2) and scatters s(p) into it -- the x
//    direction costs no shared-memory traffic;
//  * per plane one (38, 24) halo tile, the packed (evx, c1) rows of planes
//    p-1..p+1 and the RK operand tiles of cell plane p-3 arrive by TMA, 3
//    (8-cell) or 4 (4-cell) stages deep on mbarrier transaction counts (a
//    1D-2V plane is too short a step to hide an operand load issued one
//    plane ahead);
//  * a thread owns 8 (or 4) consecutive vx cells at one vy lane: 70 (38)
//    shared loads per plane, 8.75 (9.5) per cell, and the per-plane
//    overhead (ring wait, barrier, epilogue branches, partials) over twice
//    the cells; diag(vx,vy) = G(vx+1) - G(vx-1) with
//    G = s[vy-1] - s[vy+1], and the x-coupled correction uses
//    D = s[vx-1] - s[vx+1];
//  * RK operands aliasing src are folded into the accumulator (cfold/cL s);
//  * epilogue: coalesced stores, a per-thread non-finite sum, and optionally
//    the fold-tree moment partials over aligned 16-wide vy chunks.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace vpfv {

struct Stage12 {
    double *dest;
    const double *src;
    double cL;
    const double *dt_dev;
    double cL_div;
    int nops;
    double opc[2];
    int fold;
    double cfold;
    unsigned long long *nonfinite;
    const double *vxc, *vyc, *avy;
    double c2, mhx, mhvx, mhvy;
    int Nx, Nvx, Nvy;
    int wrap_x;
    int i0, i1, nseg, seglen;
    double *partials;  // [Nx][Nvx][Nvy/16] or nullptr
    // peer halo push (vpfv_stage_1d2v_fused_peer; as Stage22 in stage2d2v_tma.cu)
    double *peer_lo, *peer_hi;
    unsigned long long *sig_lo, *sig_hi;
    unsigned *done;
};

namespace r12 {
constexpr int BL = 16, OPS_MAX = 2;
// BB: consecutive vx cells per thread (4, or 8: half the per-plane overhead
// per cell at half the warps); NS: stage ring depth
template <int BK_, int MINB_, int BB_ = 4, int NS_ = 4>
struct Geo {
    static constexpr int BK = BK_, MINB = MINB_, BB = BB_, NS = NS_;
    static constexpr int THREADS = (BK / BB) * BL;
    static constexpr int TK = BK + 6, TW = BL + 8;  // halo tile (vy box starts 16 B aligned)
    static constexpr int HALO = TK * TW;
    static constexpr int TAB = 32;                  // 3 table rows of 8, padded to 256 B
    static constexpr int OPW = BL + 2, OPE = BK * OPW;
    // a stage: plane p's halo tile, its table rows, and the RK operand tiles
    // of the cell plane p-3 that the iteration of plane p finalises
    static constexpr int STAGE = HALO + TAB + OPS_MAX * OPE;
    static constexpr int BAR_OFF = NS * STAGE * 8;
    static constexpr int SMEM = BAR_OFF + 64;
    static_assert((STAGE * 8) % 128 == 0 && (HALO * 8) % 128 == 0 && (OPE * 8) % 128 == 0,
                  "TMA destinations must stay 128 B aligned");
};
}  // namespace r12

struct Maps12 {
    CUtensorMap halo, op[r12::OPS_MAX], tab;
};

__device__ __forceinline__ double w12pos(double m3, double m2, double m1, double z, double p1, double p2) {
    return fma(-3.0, p2, fma(30.0, p1, fma(20.0, z, fma(-60.0, m1, fma(15.0, m2, -2.0 * m3)))));
}
__device__ __forceinline__ double w12neg(double m2, double m1, double z, double p1, double p2, double p3) {
    return fma(2.0, p3, fma(-15.0, p2, fma(60.0, p1, fma(-20.0, z, fma(-30.0, m1, 3.0 * m2)))));
}

// x scatter of s(p) into a cell's window (w[j] = cell p-3+j before plane p),
// extraction of cell p-3, slide (see scatter_cell in stage2d2v_tma.cu)
template <int SIGN>
__device__ __forceinline__ void scatter12(double (&w)[6], double ti, double &fin) {
    // in-order renaming (slot j's FMA reads slot j+1) and an exact add for
    // the a_x > 0 finished cell, as in the 2D-2V kernel's scatter_cell
    if (SIGN > 0) {
        fin = __dadd_rn(w[0], 0.0);
        w[0] = fma(-3.0, ti, w[1]);
        w[1] = fma(30.0, ti, w[2]);
        w[2] = fma(20.0, ti, w[3]);
        w[3] = fma(-60.0, ti, w[4]);
        w[4] = fma(15.0, ti, w[5]);
        w[5] = -2.0 * ti;
    } else {
        fin = fma(2.0, ti, w[0]);
        w[0] = fma(-15.0, ti, w[1]);
        w[1] = fma(60.0, ti, w[2]);
        w[2] = fma(-20.0, ti, w[3]);
        w[3] = fma(-30.0, ti, w[4]);
        w[4] = 3.0 * ti;
        w[5] = 0.0;
    }
}

// PEER: the x-halo push of vpfv_stage_1d2v_fused_peer, compiled only into the
// instantiation that needs it (the ordinary launches carry no extra code)
template <class GEO, bool PEER>
__global__ void __launch_bounds__(GEO::THREADS, GEO::MINB)
    stage1d2v_rb_kernel(const __grid_constant__ Maps12 maps, const Stage12 P) {
    using namespace r12;
    constexpr int BK = GEO::BK, TW = GEO::TW, HALO = GEO::HALO, TAB = GEO::TAB, STAGE = GEO::STAGE, OPW = GEO::OPW,
                  OPE = GEO::OPE, BAR_OFF = GEO::BAR_OFF, BB = GEO::BB, NS = GEO::NS;
    static_assert(BB % 4 == 0 && BB <= 8, "4 or 8 cells per thread");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + BAR_OFF);  // NS stage barriers
    const unsigned sbase = tma::smem_addr(smem_raw);

    const int tid = threadIdx.x;
    const int nlt = P.Nvy / BL, nkt = P.Nvx / BK;
    const int ncols = nlt * nkt;
    const int blk = blockIdx.x % ncols, seg = blockIdx.x / ncols;
    const int lt = blk % nlt, kt = blk / nlt;
    const int k0 = kt * BK, l0 = lt * BL;
    const int i0 = P.i0 + seg * P.seglen;
    const int i1 = min(P.i1, i0 + P.seglen);
    if (i0 >= i1) {
        if (PEER) peer_done_signal(P);
        return;
    }

    // thread -> cells (vx0 + b, vy), b < BB; half-warps are 16-lane vy rows
    const int lane = tid & 31, warp = tid >> 5;
    const int tl = lane & 15;
    const int tk = (warp << 1) | (lane >> 4);
    const int vx0 = k0 + BB * tk, vy = l0 + tl;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) tma::mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int p_first = i0 - 3, nplanes = i1 - i0 + 6;
    const Maps12 *M = &maps;
    const int nops = P.nops;
    auto issue_plane = [&](int n) {  // plane n (+ operands of cell plane n-3) into stage n % NS
        const int s = n % NS;
        const unsigned dst = sbase + s * STAGE * 8, bar = sbase + BAR_OFF + s * 8;
        int px = p_first + n;
        if (P.wrap_x) px = px < 0 ? px + P.Nx : (px >= P.Nx ? px - P.Nx : px);
        const int q = p_first + n - 3;
        const int nop = (q >= i0 && q < i1) ? nops : 0;
        tma::mbar_expect_tx_s(bar, (HALO + 24 + nop * OPE) * 8);
        tma::load3d_s(dst, &M->halo, bar, l0, k0, px + NG);
        tma::load2d_s(dst + HALO * 8, &M->tab, bar, 0, px);
        for (int o = 0; o < nop; ++o)
            tma::load3d_s(dst + (HALO + TAB + o * OPE) * 8, &M->op[o], bar, l0 + 2, k0 + NG, q + NG);
    };
    if (tid == 0)
        for (int n = 0; n < NS - 1 && n < nplanes; ++n) issue_plane(n);

    double ax_s[BB], avy_s[BB];
    bool xpos[BB], ypos[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
        const double v = __ldg(P.vxc + vx0 + b);
        ax_s[b] = v * P.mhx;
        xpos[b] = v > 0.0;
        const double ay = __ldg(P.avy + vx0 + b);
        avy_s[b] = ay * P.mhvy;
        ypos[b] = ay > 0.0;
    }
    bool ypos_all = true, yneg_all = true;
#pragma unroll
    for (int b = 0; b < BB; ++b) {
        ypos_all = ypos_all && ypos[b];
        yneg_all = yneg_all && !ypos[b];
    }
    const double cBvy = __ldg(P.vyc + P.Nvy) * __ldg(P.vyc + vy);  // cB rides in vyc[Nvy] (_kernels.py:166)
    const double cL = P.dt_dev ? __ddiv_rn(*P.dt_dev, P.cL_div) : P.cL;
    const bool fold = P.fold && cL != 0.0;
    const double kfold = fold ? P.cfold / cL : 0.0;
    const bool fold_fb = P.fold && !fold;
    const double mc2 = -P.c2, mhvx = P.mhvx;
    const double oc0 = P.opc[0], oc1 = P.opc[1];
    const int off = (BB * tk + 3) * TW + tl + 3;
    const int ooff = BB * tk * OPW + tl + 1;
    const long long P2 = P.Nvy + 2 * NG, P1 = (long long)(P.Nvx + 2 * NG) * P2;
    long long gq = (long long)(p_first - 3 + NG) * P1 + (long long)(vx0 + NG) * P2 + (vy + NG);
    // moment partials of row vx0 + tl for the first iteration's cell plane (lanes tl < BB store),
    // advanced one plane per iteration
    const long long pstep = (long long)P.Nvx * nlt;
    double *ppart = P.partials + (long long)(p_first - 3) * pstep + (long long)(vx0 + (tl % BB)) * nlt + lt;

    double acc[BB][6];
#pragma unroll
    for (int i = 0; i < BB; ++i)
#pragma unroll
        for (int m = 0; m < 6; ++m) acc[i][m] = 0.0;

    for (int n = 0; n < nplanes; ++n) {
        const int p = p_first + n, q = p - 3;
        const bool inner = p >= i0 && p < i1;
        const bool fin_q = q >= i0 && q < i1;
        if (tid == 0 && n + NS - 1 < nplanes) issue_plane(n + NS - 1);
        const int nq = n / NS, stage_s = n - nq * NS;
        tma::mbar_wait_s(sbase + BAR_OFF + stage_s * 8, nq & 1);
        const double *stage = stages + stage_s * STAGE;
        const double *c = stage + off;
        const double *tb = stage + HALO;  // table rows p-1, p, p+1: (evx, c1)
        const double evx = tb[8], c1m = tb[1], c1p = tb[17];

        // the vx line at the thread's vy: offsets -3 .. BB+2 (the cells' own
        // values included); then the vy lines in groups of four cells.  Per
        // cell the arithmetic and its order are those of the 4-cell layout,
        // so every BB gives bitwise the same stage.
        double r0[BB + 6];
        r0[0] = c[-3 * TW];
        r0[1] = c[-2 * TW];
        r0[2] = c[-TW];
#pragma unroll
        for (int b = 0; b < BB; ++b) r0[b + 3] = c[b * TW];
        r0[BB + 3] = c[BB * TW];
        r0[BB + 4] = c[(BB + 1) * TW];
        r0[BB + 5] = c[(BB + 2) * TW];
        double s0[BB], G[BB];
#pragma unroll
        for (int b = 0; b < BB; ++b) s0[b] = r0[b + 3];
        // x-coupled correction c1 diag(x,vx): D(p) = s[vx-1] - s[vx+1] feeds cells p-1 and p+1
#pragma unroll
        for (int b = 0; b < BB; ++b) {
            const double D = r0[b + 2] - r0[b + 4];
            acc[b][2] = fma(c1m, D, acc[b][2]);
            acc[b][4] = fma(-c1p, D, acc[b][4]);
        }
        const double avx = evx + cBvy;  // independent of vx
        const double avx_s = avx * mhvx;
        if (inner) {
            if (avx > 0.0) {
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    acc[b][3] = fma(avx_s, w12pos(r0[b], r0[b + 1], r0[b + 2], r0[b + 3], r0[b + 4], r0[b + 5]), acc[b][3]);
            } else {
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    acc[b][3] = fma(avx_s, w12neg(r0[b + 1], r0[b + 2], r0[b + 3], r0[b + 4], r0[b + 5], r0[b + 6]),
                                    acc[b][3]);
            }
        }
#pragma unroll
        for (int h = 0; h < BB; h += 4) {
            if (BB > 4) asm volatile("" ::: "memory");  // one group of four vy lines at a time (registers)
            double v[4][7];
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
#pragma unroll
                for (int d = 0; d < 7; ++d) v[bb][d] = d == 3 ? s0[h + bb] : c[(h + bb) * TW + d - 3];
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) G[h + bb] = v[bb][2] - v[bb][4];
            if (inner) {
                if (ypos_all) {
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb)
                        acc[h + bb][3] = fma(avy_s[h + bb], w12pos(v[bb][0], v[bb][1], v[bb][2], v[bb][3], v[bb][4],
                                                                    v[bb][5]), acc[h + bb][3]);
                } else if (yneg_all) {
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb)
                        acc[h + bb][3] = fma(avy_s[h + bb], w12neg(v[bb][1], v[bb][2], v[bb][3], v[bb][4], v[bb][5],
                                                                    v[bb][6]), acc[h + bb][3]);
                } else {
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        const double w = ypos[h + bb] ? w12pos(v[bb][0], v[bb][1], v[bb][2], v[bb][3], v[bb][4], v[bb][5])
                                                      : w12neg(v[bb][1], v[bb][2], v[bb][3], v[bb][4], v[bb][5], v[bb][6]);
                        acc[h + bb][3] = fma(avy_s[h + bb], w, acc[h + bb][3]);
                    }
                }
            }
        }
        if (inner) {
            // -c2 diag(vx,vy) = -c2 (G(vx+1) - G(vx-1)); fold of the src operand
            const double gm = c[-TW - 1] - c[-TW + 1], gp = c[BB * TW - 1] - c[BB * TW + 1];
            double gr[BB + 2];
            gr[0] = gm;
            gr[BB + 1] = gp;
#pragma unroll
            for (int b = 0; b < BB; ++b) gr[b + 1] = G[b];
#pragma unroll
            for (int b = 0; b < BB; ++b) acc[b][3] = fma(kfold, s0[b], fma(mc2, gr[b + 2] - gr[b], acc[b][3]));
        }

        // x stencil scatter, extract cell q, slide
        double fin[BB];
        if (xpos[0] && xpos[BB - 1]) {
#pragma unroll
            for (int b = 0; b < BB; ++b) scatter12<1>(acc[b], ax_s[b] * s0[b], fin[b]);
        } else if (!xpos[0] && !xpos[BB - 1]) {
#pragma unroll
            for (int b = 0; b < BB; ++b) scatter12<-1>(acc[b], ax_s[b] * s0[b], fin[b]);
        } else {
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                if (xpos[b])
                    scatter12<1>(acc[b], ax_s[b] * s0[b], fin[b]);
                else
                    scatter12<-1>(acc[b], ax_s[b] * s0[b], fin[b]);
            }
        }

        if (fin_q) {
            const double *op = stage + HALO + TAB + ooff;
            double out[BB];
            if (nops == 0) {
#pragma unroll
                for (int b = 0; b < BB; ++b) out[b] = cL * fin[b];
            } else if (nops == 1) {
#pragma unroll
                for (int b = 0; b < BB; ++b) out[b] = fma(cL, fin[b], oc0 * op[b * OPW]);
            } else {
#pragma unroll
                for (int b = 0; b < BB; ++b) out[b] = fma(cL, fin[b], fma(oc1, op[OPE + b * OPW], oc0 * op[b * OPW]));
            }
            if (fold_fb) {
#pragma unroll
                for (int b = 0; b < BB; ++b) out[b] = fma(P.cfold, P.src[gq + b * P2], out[b]);
            }
            double *dq = P.dest + gq;
#pragma unroll
            for (int b = 0; b < BB; ++b) __stcs(dq + b * P2, out[b]);
            if (PEER && P.peer_lo && q < NG) {  // my plane q -> the low neighbour's ghost plane Nx + q
                double *pq = P.peer_lo + gq + (long long)P.Nx * P1;
#pragma unroll
                for (int b = 0; b < BB; ++b) pq[b * P2] = out[b];
            }
            if (PEER && P.peer_hi && q >= P.Nx - NG) {  // my plane q -> the high neighbour's ghost plane q - Nx
                double *pq = P.peer_hi + gq - (long long)P.Nx * P1;
#pragma unroll
                for (int b = 0; b < BB; ++b) pq[b * P2] = out[b];
            }
            if (P.nonfinite) {
                double sum = (out[0] + out[1]) + (out[2] + out[3]);
#pragma unroll
                for (int b = 4; b < BB; b += 4) sum += (out[b] + out[b + 1]) + (out[b + 2] + out[b + 3]);
                if (!isfinite(sum)) {
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        if (!isfinite(out[b]))
                            atomicMin(P.nonfinite, ((unsigned long long)q * P.Nvx + vx0 + b) * P.Nvy + vy);
                }
            }
            if (P.partials) {
                // reference fold tree (fields.py:28-47) over each aligned
                // 16-wide vy chunk: transpose-reduce the BB rows over the lanes
                // (after level k, lane bit k-1 selects the row half)
                double w1;
                if (BB == 8) {
                    const bool o1 = tl & 1, o2 = tl & 2, o4 = tl & 4;
                    double w4[4], w2[2];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const double keep = o1 ? out[(2 * m + 1) % BB] : out[(2 * m) % BB];
                        const double send = o1 ? out[(2 * m) % BB] : out[(2 * m + 1) % BB];
                        w4[m] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
                    }
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const double keep = o2 ? w4[2 * m + 1] : w4[2 * m];
                        const double send = o2 ? w4[2 * m] : w4[2 * m + 1];
                        w2[m] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
                    }
                    const double keep = o4 ? w2[1] : w2[0];
                    const double send = o4 ? w2[0] : w2[1];
                    w1 = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 4));
                    w1 = __dadd_rn(w1, __shfl_xor_sync(0xffffffffu, w1, 8));
                } else {
                    const bool o1 = tl & 1, o2 = tl & 2;
                    double w2[2];
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const double keep = o1 ? out[2 * m + 1] : out[2 * m];
                        const double send = o1 ? out[2 * m] : out[2 * m + 1];
                        w2[m] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 1));
                    }
                    const double keep = o2 ? w2[1] : w2[0];
                    const double send = o2 ? w2[0] : w2[1];
                    w1 = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 2));
                    w1 = __dadd_rn(w1, __shfl_xor_sync(0xffffffffu, w1, 4));
                    w1 = __dadd_rn(w1, __shfl_xor_sync(0xffffffffu, w1, 8));
                }
                if (tl < BB) *ppart = w1;  // lane tl: row tl
            }
        }
        gq += P1;
        ppart += pstep;
        __syncthreads();  // the stage and the operand tiles are free for the next refill
    }
    if (PEER) peer_done_signal(P);
}

// Geometry (VPFV_R12_CFG): 4 = (32, 16) tiles with 8 cells per thread (64
// threads, <=256 registers), 4 CTAs per SM, 3-deep ring (default: -5 % at
// 256^3 against 1); 1 = the same tiles with 4 cells per thread (128
// threads, <=168 registers) at 3 CTAs per SM and a 4-deep ring (round 1's
// default); 0 = that at 2 CTAs per SM; 2 = (64, 16) tiles at 1 CTA per SM;
// 3 = 8 cells per thread at 3 CTAs per SM (+18 %: too few warps).
static int geo12_cfg() {
#ifndef VPFV_R12_CFG_DEFAULT
#define VPFV_R12_CFG_DEFAULT 4
#endif
    static int c = -1;
    if (c < 0) {
        const char *e = getenv("VPFV_R12_CFG");
        c = e ? atoi(e) : VPFV_R12_CFG_DEFAULT;
        if (c < 0 || c > 4) c = VPFV_R12_CFG_DEFAULT;
    }
    return c;
}

bool tma_1d2v_eligible(int Nx, int Nvx, int Nvy, unsigned flags) {
    if (flags & VPFV_EXACT) return false;
    if (flags & (VPFV_WRAP(1) | VPFV_WRAP(2))) return false;
    if (Nvx % 32 || Nvy % r12::BL || Nx < 1 || Nvy / r12::BL > 16) return false;
    return tma_available();
}

template <class GEO>
static int launch12(const double *src, const double *const ops[r12::OPS_MAX], const double *tab, Stage12 P,
                    int xsegments, cudaStream_t s) {
    using namespace r12;
    const int cols = (P.Nvx / GEO::BK) * (P.Nvy / BL);
    int nseg = xsegments;
    if (nseg <= 0) {  // ~6 waves at 2 CTAs per SM, segments >= 8 planes
        nseg = (6 * 148 + cols - 1) / cols;
        if (nseg > P.Nx / 8) nseg = P.Nx / 8;
        if (nseg < 1) nseg = 1;
    }
    P.nseg = nseg;
    P.seglen = (P.i1 - P.i0 + nseg - 1) / nseg;
    Maps12 maps;
    const unsigned long long dims[3] = {(unsigned long long)P.Nvy + 6, (unsigned long long)P.Nvx + 6,
                                        (unsigned long long)P.Nx + 6};
    const unsigned long long strides[2] = {dims[0] * 8, dims[0] * dims[1] * 8};
    const unsigned bh[3] = {GEO::TW, GEO::TK, 1}, bo[3] = {GEO::OPW, GEO::BK, 1};
    if (!tma_map(src, 3, dims, strides, bh, &maps.halo)) return set_error(VPFV_ECUDA, "tensor map failed");
    for (int o = 0; o < OPS_MAX; ++o) {
        if (o < P.nops) {
            if (!tma_map(ops[o], 3, dims, strides, bo, &maps.op[o])) return set_error(VPFV_ECUDA, "tensor map failed");
        } else {
            maps.op[o] = maps.halo;
        }
    }
    const unsigned long long tdims[2] = {8, (unsigned long long)P.Nx + 2};
    const unsigned long long tstr[1] = {64};
    const unsigned tbox[2] = {8, 3};
    if (!tma_map(tab, 2, tdims, tstr, tbox, &maps.tab)) return set_error(VPFV_ECUDA, "table map failed");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(stage1d2v_rb_kernel<GEO, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEO::SMEM);
        cudaFuncSetAttribute(stage1d2v_rb_kernel<GEO, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEO::SMEM);
        attr = true;
    }
    if (P.done)
        stage1d2v_rb_kernel<GEO, true><<<cols * nseg, GEO::THREADS, GEO::SMEM, s>>>(maps, P);
    else
        stage1d2v_rb_kernel<GEO, false><<<cols * nseg, GEO::THREADS, GEO::SMEM, s>>>(maps, P);
    return check_launch("stage_1d2v_tma");
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

extern "C" int vpfv_stage_1d2v_partials_chunk(void) { return r12::BL; }

namespace {
struct Operands12 {  // ca A + cb B + cd dest grouped by array; the src part is folded
    const double *ptr[3];
    double coef[3];
    int n = 0, fold = 0;
    double cfold = 0.0;
    void add(const double *p, double c, const double *src) {
        if (c == 0.0) return;
        if (p == src) {
            cfold += c;
            fold = 1;
            return;
        }
        for (int i = 0; i < n; ++i)
            if (ptr[i] == p) {
                coef[i] += c;
                return;
            }
        ptr[n] = p;
        coef[n++] = c;
    }
};
}  // namespace

static int stage_1d2v_fused_impl(double *dest, const double *A, const double *B, const double *src, double ca,
                                 double cb, double cd, double cL, const double *vxc, const double *vyc,
                                 const double *evx, const double *avy, const double *c1, double c2, double hx,
                                 double hvx, double hvy, int Nx, int Nvx, int Nvy, unsigned flags,
                                 const double *dt_dev, double cL_div, unsigned long long *nonfinite,
                                 const double *packed_tables, double *moment_partials, int xsegments, void *stream,
                                 const Stage12 *peer) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    Operands12 ops;
    ops.add(A, ca, src);
    ops.add(B, cb, src);
    ops.add(dest, cd, src);
    if (!packed_tables || !tma_1d2v_eligible(Nx, Nvx, Nvy, flags) || ops.n > r12::OPS_MAX) {
        if (moment_partials) return set_error(VPFV_EARG, "fused moment needs the tiled 1D-2V path");
        if (peer) return set_error(VPFV_EARG, "peer halo push needs the tiled 1D-2V path");
        return vpfv_stage_1d2v(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, avy, c1, c2, hx, hvx, hvy, Nx,
                               Nvx, Nvy, flags, dt_dev, cL_div, nonfinite, stream);
    }
    Stage12 P{};
    P.dest = dest;
    P.src = src;
    P.cL = cL;
    P.dt_dev = dt_dev;
    P.cL_div = cL_div;
    P.nops = ops.n;
    for (int o = 0; o < ops.n; ++o) P.opc[o] = ops.coef[o];
    P.fold = ops.fold;
    P.cfold = ops.cfold;
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
    if (peer) {
        P.peer_lo = peer->peer_lo;
        P.peer_hi = peer->peer_hi;
        P.sig_lo = peer->sig_lo;
        P.sig_hi = peer->sig_hi;
        P.done = peer->done;
    }
    const double *opp[r12::OPS_MAX] = {ops.n > 0 ? ops.ptr[0] : nullptr, ops.n > 1 ? ops.ptr[1] : nullptr};
    cudaStream_t st = (cudaStream_t)stream;
    const int cfg = geo12_cfg();
    if (cfg == 2 && Nvx % 64 == 0) return launch12<r12::Geo<64, 1>>(src, opp, packed_tables, P, xsegments, st);
    if (cfg == 1) return launch12<r12::Geo<32, 3>>(src, opp, packed_tables, P, xsegments, st);
    if (cfg == 3) return launch12<r12::Geo<32, 3, 8, 4>>(src, opp, packed_tables, P, xsegments, st);
    if (cfg == 4) return launch12<r12::Geo<32, 4, 8, 3>>(src, opp, packed_tables, P, xsegments, st);
    return launch12<r12::Geo<32, 2>>(src, opp, packed_tables, P, xsegments, st);
}

extern "C" int vpfv_stage_1d2v_fused(double *dest, const double *A, const double *B, const double *src,
                                     double ca, double cb, double cd, double cL, const double *vxc,
                                     const double *vyc, const double *evx, const double *avy,
                                     const double *c1, double c2, double hx, double hvx, double hvy, int Nx,
                                     int Nvx, int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, const double *packed_tables,
                                     double *moment_partials, int xsegments, void *stream) {
    return stage_1d2v_fused_impl(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, avy, c1, c2, hx, hvx, hvy, Nx, Nvx,
                                 Nvy, flags, dt_dev, cL_div, nonfinite, packed_tables, moment_partials, xsegments,
                                 stream, nullptr);
}

extern "C" int vpfv_stage_1d2v_fused_peer(double *dest, const double *A, const double *B, const double *src,
                                          double ca, double cb, double cd, double cL, const double *vxc,
                                          const double *vyc, const double *evx, const double *avy,
                                          const double *c1, double c2, double hx, double hvx, double hvy, int Nx,
                                          int Nvx, int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                          unsigned long long *nonfinite, const double *packed_tables,
                                          double *moment_partials, double *peer_lo, double *peer_hi,
                                          unsigned long long *sig_lo, unsigned long long *sig_hi, unsigned *done,
                                          void *stream) {
    if (!packed_tables || !tma_1d2v_eligible(Nx, Nvx, Nvy, flags))
        return set_error(VPFV_EARG, "peer halo push needs the tiled 1D-2V path");
    if (Nx < NG || !done) return set_error(VPFV_EARG, "peer halo push: Nx >= 3 and a done counter");
    Stage12 peer{};
    peer.peer_lo = peer_lo;
    peer.peer_hi = peer_hi;
    peer.sig_lo = sig_lo;
    peer.sig_hi = sig_hi;
    peer.done = done;
    return stage_1d2v_fused_impl(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, avy, c1, c2, hx, hvx, hvy, Nx, Nvx,
                                 Nvy, flags, dt_dev, cL_div, nonfinite, packed_tables, moment_partials, 0, stream,
                                 &peer);
}
