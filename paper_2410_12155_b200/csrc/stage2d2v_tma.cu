// 2D-2V fused stage: x-marching, TMA-staged halo tiles, 2x4 register blocks
// (sm_100a, fast arithmetic path).
//
// Same operator as stage_2d2v (/root/reference/pkg/src/vpfv/_kernels.py:254-317):
//   rhs = -a_x D_x f - a_y D_y f - a_vx D_vx f - a_vy D_vy f
//         + c1 diag(x,vx) + c4 diag(y,vy) - c2 diag(vx,vy) - c3 diag(y,vx) - c5 diag(x,vy)
//   dest = ca A + cb B + cd dest + cL rhs            (interior cells only)
//
// Why this shape.  The stencil has radius 3 along four axes plus the
// (+-1, +-1) diagonals of five axis pairs; it is fp64 and HBM-bound in
// principle, but every cell's ~31-point footprint has to reach the FP64
// pipes through the SM's 128 B/clk shared-memory/L1 datapath.  The design
// therefore minimises datapath bytes per cell:
//
//  * A CTA (256 threads, one per SM) owns a (y, vx, vy) = (8, 16, 16)
//    column block and marches along x (the slowest dim) over planes
//    p = i0-3 .. i1+2.  The x direction costs no shared-memory traffic: each
//    thread keeps, per cell, a sliding window of 6 register accumulators for
//    the cells p-3..p+2 in flight along x and scatters s(p) into them.
//  * Each plane's (14, 22, 24) halo tile is copied global -> shared by TMA
//    (cp.async.bulk.tensor.4d: a core box plus two 3-row y-halo boxes, so
//    periodic y wraps are free), 3 stages deep, completion tracked by
//    mbarrier transaction counts.  On x-halo planes only the core box moves.
//  * Each thread owns a 2 (y) x 4 (vx) block of cells at one vy lane; the
//    block's footprint is 120 shared loads per plane, 15 per cell (one cell
//    per thread would need 31).  The diagonal corrections are rebuilt from
//    per-row differences D = s[vx-1]-s[vx+1] and G = s[vy-1]-s[vy+1] that the
//    x-coupled corrections need anyway:  diag(vx,vy) = G(vx+1)-G(vx-1),
//    diag(y,vy) = G(y+1)-G(y-1), diag(y,vx) = D(y+1)-D(y-1).
//  * RK operands that alias src are folded into the accumulator when their
//    plane is resident (cfold/cL * s(q)), so stage 1 reads only src; other
//    operands are TMA-staged one plane ahead of their use.
//  * The epilogue writes dest (coalesced 128 B half-warp rows) and, when
//    asked, the velocity-moment partials of the new dest: the exact first
//    four levels of the reference fold tree over each aligned 16-wide vy
//    chunk (transpose-reduce over the 16 vy lanes), finished by
//    vpfv_moment_partials.  This replaces a separate moment pass over f.
//  * Round 2 (default, 1 CTA/SM geometry): warp-specialised.  A fourth
//    warpgroup gives up its registers (setmaxnreg 24; the 8 compute warps
//    take 240) and two of its lanes issue every TMA load -- halo planes and
//    RK operand tiles -- each blocked in mbarrier.try_wait on the empty
//    barrier its stream refills; compute warps wait on full barriers and
//    arrive on empty ones, with no CTA barrier in the plane loop.  The
//    headline 128-wide velocity shape (and config 5's 64-wide one) runs an
//    instantiation with compile-time padded strides.
//
// Requirements (checked by the launcher, else the generic kernel runs):
// Ny % 8 == 0, Nvx % 16 == 0, Nvy % 16 == 0, periodic-or-halo x/y, stored
// (frozen) velocity ghosts, at most two RK operands besides src.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "tma.cuh"
#include "field.cuh"

namespace vpfv {

struct Stage22 {
    double *dest;
    const double *src;
    double cL;
    const double *dt_dev;
    double cL_div;
    int nops;          // RK operands staged by TMA (those that do not alias src)
    double opc[2];     // their coefficients
    int fold;          // src is an RK operand too: its coefficient is folded
    double cfold;
    unsigned long long *nonfinite;
    const double *vxc, *vyc;
    double cB, c2, mhx, mhy, mhvx, mhvy;
    int Nx, Ny, Nvx, Nvy;
    int wrap_x, wrap_y;
    int i0, i1;        // x range of cells this launch updates (interior indices)
    int nseg, seglen;  // x segments per column block
    int sj, sk;        // super-tile of column blocks (block order)
    double *partials;  // moment partials [Nx][Ny][Nvx][Nvy/16] or nullptr
    // peer halo push (x-slab ranks over NVLink, vpfv_stage_2d2v_fused_peer):
    // planes 0..2 also go to the low x neighbour's dest (its high ghost
    // planes), planes Nx-3..Nx-1 to the high neighbour's low ghost planes;
    // the last CTA to finish bumps the neighbours' signal words
    double *peer_lo, *peer_hi;
    unsigned long long *sig_lo, *sig_hi;
    unsigned *done;
};


namespace rb {
constexpr int BJ = 8, BL = 16, OPS_MAX = 2;
// packed table entry (vpfv_tables_2d_packed): evx, evy, c3, c4, c1, c5, 0, 0
enum { T_EVX = 0, T_EVY = 1, T_C3 = 2, T_C4 = 3, T_C1 = 4, T_C5 = 5 };
// Tile geometry: (BJ, BK, BL) column block, NS-deep stage ring, MINB CTAs
// per SM; one thread per 2 (y) x BB (vx) cells at one vy lane.
template <int BK_, int NS_, int MINB_, int NOPB_ = 1, int BB_ = 4>
struct Geo {
    static constexpr int BK = BK_, NS = NS_, MINB = MINB_, BB = BB_, NOPB = NOPB_;  // NOPB: operand buffers
    static constexpr int THREADS = (BJ / 2) * (BK / BB) * BL;
    static constexpr int TJ = BJ + 6, TK = BK + 6, TW = BL + 8;  // halo tile (vy box starts 16 B aligned)
    static constexpr int KL = TK * TW, HALO = TJ * KL;
    static constexpr int TAB = 3 * BJ * 8;  // packed tables of planes p-1, p, p+1
    static constexpr int STAGE = HALO + TAB;
    static constexpr int OPW = BL + 2;      // RK operand row (16 B aligned start)
    static constexpr int OPE = BJ * BK * OPW;
    static constexpr int HALO_BYTES = HALO * 8, CORE_BYTES = BJ * KL * 8, TAB_BYTES = TAB * 8, OP_BYTES = OPE * 8;
    // barriers: NS stage-full, NOPB operand-full, then (warp-specialised) NS
    // stage-empty and NOPB operand-empty
    static constexpr int BAR_OFF = NS * STAGE * 8 + NOPB * OPS_MAX * OPE * 8;
    static constexpr int SMEM = BAR_OFF + 64;
    static_assert(2 * (NS + NOPB) <= 8, "barrier block");
    static_assert((STAGE * 8) % 128 == 0 && (HALO * 8) % 128 == 0 && (OPE * 8) % 128 == 0,
                  "TMA destinations must stay 128 B aligned");
    static_assert(SMEM * MINB <= 228 * 1024 - MINB * 1024, "shared memory budget");
};
using GeoWide = Geo<16, 3, 1>;   // (8, 16, 16) tiles, 1 CTA of 8 warps per SM
using GeoPair = Geo<8, 2, 2>;    // (8, 8, 16) tiles, 2 CTAs of 4 warps per SM (desynchronised)
// stages with RK operands, warp-specialised: a 2-deep halo ring and double-
// buffered operand tiles, so compute warps are not coupled through one buffer
using GeoWideOp = Geo<16, 2, 1, 2>;
}  // namespace rb

#define RB_GEOMETRY(G)                                                                                          \
    constexpr int BK = G::BK, NS = G::NS, BB = G::BB, TK = G::TK, TW = G::TW, KL = G::KL, HALO = G::HALO,     \
                  STAGE = G::STAGE, OPW = G::OPW, OPE = G::OPE, HALO_BYTES = G::HALO_BYTES,                    \
                  CORE_BYTES = G::CORE_BYTES, TAB_BYTES = G::TAB_BYTES, OP_BYTES = G::OP_BYTES,                \
                  BAR_OFF = G::BAR_OFF, NOPB = G::NOPB;                                                          \
    (void)NOPB, (void)BK, (void)NS, (void)BB, (void)TK, (void)TW, (void)KL, (void)HALO, (void)STAGE, (void)OPW, (void)OPE, \
        (void)HALO_BYTES, (void)CORE_BYTES, (void)TAB_BYTES, (void)OP_BYTES, (void)BAR_OFF

struct Maps {
    CUtensorMap core, halo, op[rb::OPS_MAX], tab;
};

// upwinded 6-point face-difference sums (x 60); offsets -3..2 for a > 0 and
// -2..3 for a <= 0 (_kernels.py:28-30, ties to the negative branch)
__device__ __forceinline__ double wpos(double m3, double m2, double m1, double z, double p1, double p2) {
    return fma(-3.0, p2, fma(30.0, p1, fma(20.0, z, fma(-60.0, m1, fma(15.0, m2, -2.0 * m3)))));
}
__device__ __forceinline__ double wneg(double m2, double m1, double z, double p1, double p2, double p3) {
    return fma(2.0, p3, fma(-15.0, p2, fma(60.0, p1, fma(-20.0, z, fma(-30.0, m1, 3.0 * m2)))));
}

#ifdef VPFV_NO_SCHED_FENCE
#define SCHED_FENCE()
#else
#define SCHED_FENCE() asm volatile("" ::: "memory")  // limit load hoisting (register pressure)
#endif

// x stencil scatter of s(p) into one cell's accumulator window, extraction
// of the finished cell p-3 and the window slide.  Before plane p, w[j] holds
// cell p-3+j; a cell's slot is initialised by its first contribution --
// x-stencil offset -3 (a_x > 0) or -2 (a_x <= 0) -- so no slot is zeroed.
template <int SIGN>  // +1: a_x > 0, -1: a_x <= 0
__device__ __forceinline__ void scatter_cell(double (&w)[6], double ti, double &fin) {
    // The slide as in-order renaming: slot j's FMA reads slot j+1, so each
    // result can take the register its slot had, and the finished cell comes
    // out of an instruction (w0 + 0: exact, and unlike 0*t + w0 it cannot pick
    // up a non-finite value from this plane) instead of pinning w[0]'s
    // register past the slide.  Measured 235 -> 95 register moves in the
    // kernel, -5 % per RK4 step with the hoisted y-arm branch (bitwise).
    if (SIGN > 0) {
        fin = __dadd_rn(w[0], 0.0);
        w[0] = fma(-3.0, ti, w[1]);
        w[1] = fma(30.0, ti, w[2]);
        w[2] = fma(20.0, ti, w[3]);
        w[3] = fma(-60.0, ti, w[4]);
        w[4] = fma(15.0, ti, w[5]);
        w[5] = -2.0 * ti;  // cell p+3 enters
    } else {
        fin = fma(2.0, ti, w[0]);
        w[0] = fma(-15.0, ti, w[1]);
        w[1] = fma(60.0, ti, w[2]);
        w[2] = fma(-20.0, ti, w[3]);
        w[3] = fma(-30.0, ti, w[4]);
        w[4] = 3.0 * ti;  // cell p+2 enters (its slot was freed last plane)
        w[5] = 0.0;
    }
}

// The sign of a_x is per vx; a thread's BB vx cells share it unless the zero
// crossing falls inside them (one uniform branch, no predication).
template <int BB>
__device__ __forceinline__ void window_apply(double (&acc)[2 * BB][6], const double (&s0)[2 * BB],
                                             const double (&ax_s)[BB], const bool (&xpos)[BB],
                                             double (&fin)[2 * BB]) {
    if (xpos[0] && xpos[BB - 1]) {
#pragma unroll
        for (int i = 0; i < 2 * BB; ++i) scatter_cell<1>(acc[i], ax_s[i % BB] * s0[i], fin[i]);
    } else if (!xpos[0] && !xpos[BB - 1]) {
#pragma unroll
        for (int i = 0; i < 2 * BB; ++i) scatter_cell<-1>(acc[i], ax_s[i % BB] * s0[i], fin[i]);
    } else {
#pragma unroll
        for (int i = 0; i < 2 * BB; ++i) {
            if (xpos[i % BB])
                scatter_cell<1>(acc[i], ax_s[i % BB] * s0[i], fin[i]);
            else
                scatter_cell<-1>(acc[i], ax_s[i % BB] * s0[i], fin[i]);
        }
    }
}

// One plane's copies are split into parts issued by different warps so that
// no warp carries the whole producer cost: 0 = expect_tx + tables, 1-3 =
// y-low halo / core / y-high halo.  complete_tx may land before expect_tx
// (the transaction count may go transiently negative; the phase cannot
// complete before part 0 arrives).  On x-halo planes only the core moves.
template <class GEO>
__device__ __forceinline__ void issue_plane_part(int w, unsigned sbase, const Maps *M, int n, int p_first,
                                                 const Stage22 &P, int i0, int i1, int l0, int k0, int j0, int cy_lo,
                                                 int cy_core, int cy_hi) {
    using namespace rb;
    RB_GEOMETRY(GEO);
    const int s = n % NS;
    const unsigned dst = sbase + s * STAGE * 8, bar = sbase + BAR_OFF + s * 8;
    const int p = p_first + n;  // in [i0-3, i1+3)
    int px = p;
    if (P.wrap_x) px = px < 0 ? px + P.Nx : (px >= P.Nx ? px - P.Nx : px);
    const bool inner = p >= i0 && p < i1;
    const int cx = px + NG;
    switch (w) {
        case 0:
            tma::mbar_expect_tx_s(bar, (inner ? HALO_BYTES : CORE_BYTES) + TAB_BYTES);
            // packed table rows px..px+2 = planes p-1, p, p+1 (row = x + 1)
            tma::load3d_s(dst + HALO * 8, &M->tab, bar, 0, j0, px);
            break;
        case 1:
            if (inner) tma::load4d_s(dst, &M->halo, bar, l0, k0, cy_lo, cx);
            break;
        case 2: tma::load4d_s(dst + 3 * KL * 8, &M->core, bar, l0, k0, cy_core, cx); break;
        case 3:
            if (inner) tma::load4d_s(dst + (3 + BJ) * KL * 8, &M->halo, bar, l0, k0, cy_hi, cx);
            break;
        default: break;
    }
}

// PEER: the x-halo push of vpfv_stage_2d2v_fused_peer, compiled only into the
// instantiation that needs it (the ordinary launches carry no extra code)
// WS: warp-specialised variant -- a fourth warpgroup (warps 8-11, 24
// registers; one lane works) issues every TMA load, driven by full/empty
// mbarriers, and the compute warps (240 registers) never meet at a CTA
// barrier inside the plane loop (VPFV_RB_WS=1).
// NV > 0: an instantiation for Nvx == Nvy == NV, so the padded strides are
// compile-time and the epilogue's eight stores take one base address plus
// immediate offsets (VPFV_RB_NV; the launcher picks it when the extents match)
template <class GEO, bool PEER, bool WS = false, int NV = 0>
__global__ void __launch_bounds__(GEO::THREADS + (WS ? 128 : 0), GEO::MINB)
    stage2d2v_rb_kernel(const __grid_constant__ Maps maps, const Stage22 P) {
    using namespace rb;
    RB_GEOMETRY(GEO);
    static_assert(WS || NOPB == 1, "double-buffered operands need the producer warpgroup");
    pdl_wait();  // programmatic dependent of the tables kernel: nothing global before this
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *stages = reinterpret_cast<double *>(smem_raw);
    const double *opbuf = stages + NS * STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + BAR_OFF);  // NS stage barriers + 1 operand barrier
    const unsigned sbase = tma::smem_addr(smem_raw);
    const unsigned opbar = sbase + BAR_OFF + NS * 8, opdst = sbase + NS * STAGE * 8;

    const int tid = threadIdx.x;
    // column block; x segment outermost so the CTAs resident at once cover
    // neighbouring column blocks of the same x range (halo reuse in L2)
    const int nlt = P.Nvy / BL, nkt = P.Nvx / BK, njt = P.Ny / BJ;
    const int ncols = nlt * nkt * njt;
    int blk = blockIdx.x % ncols;
    const int seg = blockIdx.x / ncols;
    // all vy tiles of a (y, vx) column block are adjacent, and column blocks
    // are visited in (sj x sk) super-tiles
    const int lt = blk % nlt;
    blk /= nlt;
    const int sj = min(P.sj, njt), sk = min(P.sk, nkt);
    const int nsk = (nkt + sk - 1) / sk;
    const int st = blk / (sj * sk), wi = blk % (sj * sk);
    const int st_j = st / nsk, st_k = st % nsk;
    const int rows_j = min(sj, njt - st_j * sj), cols_k = min(sk, nkt - st_k * sk);
    const int jt = st_j * sj + (wi / cols_k) % rows_j;
    const int kt = st_k * sk + wi % cols_k;
    const int j0 = jt * BJ, k0 = kt * BK, l0 = lt * BL;
    const int i0 = P.i0 + seg * P.seglen;
    const int i1 = min(P.i1, i0 + P.seglen);
    if (i0 >= i1) {
        if (PEER) peer_done_signal(P);
        return;
    }

    // thread -> cells (y0 + a, vx0 + b, vy), a < 2, b < BB
    const int lane = tid & 31, warp = tid >> 5;
    const int tl = lane & 15;
    const int rg = (warp << 1) | (lane >> 4);
    constexpr int NC = 2 * BB;  // cells per thread
    const int tj = rg / (BK / BB), tk = rg % (BK / BB);
    const int y0 = j0 + 2 * tj, vx0 = k0 + BB * tk, vy = l0 + tl;

    int yl = j0 - 3, yh = j0 + BJ;
    if (P.wrap_y) {
        if (yl < 0) yl += P.Ny;
        if (yh >= P.Ny) yh -= P.Ny;
    }
    const int cy_lo = yl + NG, cy_core = j0 + NG, cy_hi = yh + NG;

    if (tid == 0) {
        for (int s = 0; s < NS + NOPB; ++s) tma::mbar_init(&bars[s], 1);
        if (WS)  // empty barriers: every compute thread arrives once per plane / per operand tile
            for (int s = NS + NOPB; s < 2 * (NS + NOPB); ++s) tma::mbar_init(&bars[s], GEO::THREADS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int p_first = i0 - 3, p_last = i1 + 2;
    const int nplanes = p_last - p_first + 1;
    const Maps *M = &maps;
    // operand buffer k: full barrier opbar + 8k, empty barrier opempty + 8k, tiles at opdst + k * OPB
    const unsigned emptybar = sbase + BAR_OFF + (NS + NOPB) * 8, opempty = sbase + BAR_OFF + (2 * NS + NOPB) * 8;
    constexpr int OPB = OPS_MAX * OPE * 8;
    if (WS) {
        if (warp >= GEO::THREADS / 32) {  // the producer warpgroup
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
            // two producer lanes, each blocked in mbarrier.try_wait (suspended, not
            // spinning) on its own stream: warp 8 issues halo planes as soon as
            // their ring slot's empty barrier completes, warp 9 operand tiles as
            // soon as the operand buffer's does
            if (tid == GEO::THREADS) {
                for (int nh = 0; nh < nplanes; ++nh) {
#ifndef VPFV_WS_HINT_NS
#define VPFV_WS_HINT_NS 1000000
#endif
                    if (nh >= NS) tma::mbar_wait_sleep_s(emptybar + (nh % NS) * 8, (nh / NS - 1) & 1, VPFV_WS_HINT_NS);
                    for (int w = 0; w < 4; ++w)
                        issue_plane_part<GEO>(w, sbase, M, nh, p_first, P, i0, i1, l0, k0, j0, cy_lo, cy_core, cy_hi);
                }
            } else if (tid == GEO::THREADS + 32 && P.nops) {
                for (int no = 0; no < i1 - i0; ++no) {
                    const int kb = no % NOPB;
                    if (no >= NOPB) tma::mbar_wait_sleep_s(opempty + kb * 8, (no / NOPB - 1) & 1, VPFV_WS_HINT_NS);
                    const int q = i0 + no;
                    tma::mbar_expect_tx_s(opbar + kb * 8, P.nops * OP_BYTES);
                    for (int o = 0; o < P.nops; ++o)
                        tma::load4d_s(opdst + kb * OPB + o * OPE * 8, &M->op[o], opbar + kb * 8, l0 + 2, k0 + NG,
                                      j0 + NG, q + NG);
                }
            }
            return;  // no peer stores here: the compute threads count the CTA (named barrier)
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
    } else if (tid == 0) {
        for (int n = 0; n < NS - 1 && n < nplanes; ++n)
            for (int w = 0; w < 4; ++w)
                issue_plane_part<GEO>(w, sbase, M, n, p_first, P, i0, i1, l0, k0, j0, cy_lo, cy_core, cy_hi);
    }

    // per-thread constants
    double ax_s[BB], bvx[BB];
    bool xpos[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
        const double v = __ldg(P.vxc + vx0 + b);
        ax_s[b] = v * P.mhx;
        xpos[b] = v > 0.0;
        bvx[b] = -P.cB * v;
    }
    const double vyv = __ldg(P.vyc + vy);
    const double ay_s = vyv * P.mhy;
    const bool ypos = vyv > 0.0;
    const double cBvy = P.cB * vyv;
    double bvx_min = bvx[0], bvx_max = bvx[0];
#pragma unroll
    for (int b = 1; b < BB; ++b) {
        bvx_min = fmin(bvx_min, bvx[b]);
        bvx_max = fmax(bvx_max, bvx[b]);
    }
    const double cL = P.dt_dev ? __ddiv_rn(*P.dt_dev, P.cL_div) : P.cL;
    const bool fold = P.fold && cL != 0.0;        // else the src operand is read at finalisation
    const double kfold = fold ? P.cfold / cL : 0.0;
    const bool fold_fb = P.fold && !fold;
    const double mc2 = -P.c2, mhvx = P.mhvx, mhvy = P.mhvy;
    const int nops = P.nops;
    const double oc0 = P.opc[0], oc1 = P.opc[1];

    const int off = ((2 * tj + 3) * TK + (BB * tk + 3)) * TW + (tl + 3);  // cell (a=0, b=0) in the halo tile
    const int ooff = ((2 * tj) * BK + BB * tk) * OPW + tl + 1;          // cell (0, 0) in an operand tile
    const int toff = (2 * tj) * 8;                                      // table entry of row y0, plane p-1

    const long long P3 = NV > 0 ? NV + 2 * NG : P.Nvy + 2 * NG,
                    P2 = (long long)(NV > 0 ? NV + 2 * NG : P.Nvx + 2 * NG) * P3,
                    P1 = (long long)(P.Ny + 2 * NG) * P2;
    // padded index of cell (q = p - 3, y0, vx0, vy) for the first plane
    long long gq = (long long)(p_first - 3 + NG) * P1 + (long long)(y0 + NG) * P2 +
                   (long long)(vx0 + NG) * P3 + (vy + NG);

    // moment partials of row (y0 + tl/BB, vx0 + tl%BB) for the cell plane of the
    // first iteration (lanes tl >= NC never store), advanced one plane per iteration
    const long long pstep = (long long)P.Ny * P.Nvx * nlt;
    double *ppart = P.partials + (long long)(p_first - 3) * pstep +
                    ((long long)(y0 + (tl % NC) / BB) * P.Nvx + vx0 + (tl % NC) % BB) * nlt + lt;

    double acc[NC][6];
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
        for (int m = 0; m < 6; ++m) acc[i][m] = 0.0;

    for (int n = 0; n < nplanes; ++n) {
        const int p = p_first + n, q = p - 3;
        const bool inner = p >= i0 && p < i1;
        const bool fin_q = q >= i0 && q < i1;
        // producers: plane n+NS-1 into the stage freed at the end of plane n-1,
        // and this plane's RK operand tiles (cell plane q) into the operand buffer
        // (plane parts from lane 0 of warps 0-3; operand o from lane 0 of warp
        // 4+o, or from lane 16 of warp o when the CTA has only 4 warps)
        constexpr int NWARPS = GEO::THREADS / 32;
        if (!WS && lane == 0 && warp < 4 && n + NS - 1 < nplanes)
            issue_plane_part<GEO>(warp, sbase, M, n + NS - 1, p_first, P, i0, i1, l0, k0, j0, cy_lo, cy_core, cy_hi);
        if (!WS) {
            const int o = NWARPS >= 4 + OPS_MAX ? warp - 4 : warp;
            const bool op_lane = NWARPS >= 4 + OPS_MAX ? lane == 0 : lane == 16;
            if (op_lane && o >= 0 && o < nops && fin_q) {
                if (o == 0) tma::mbar_expect_tx_s(opbar, nops * OP_BYTES);
#ifdef VPFV_OP_EVICT_FIRST  // RK operands are read once: keep them from displacing src halos in L2
                tma::load4d_s_hint(opdst + o * OPE * 8, &M->op[o], opbar, l0 + 2, k0 + NG, j0 + NG, q + NG,
                                   tma::policy_evict_first());
#else
                tma::load4d_s(opdst + o * OPE * 8, &M->op[o], opbar, l0 + 2, k0 + NG, j0 + NG, q + NG);
#endif
            }
        }
        // stage and parity from the plane number (loop-carried counters get spilled)
        const int nq3 = n / NS, stage_s = n - nq3 * NS;
        tma::mbar_wait_s(sbase + BAR_OFF + stage_s * 8, nq3 & 1);
        const double *stage = stages + stage_s * STAGE;
        const double *c = stage + off;
        const double *tb = stage + HALO + toff;
        double evx[2], evy[2], c3[2], c4[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const double *e1 = tb + (BJ + a) * 8;
            evx[a] = e1[T_EVX];
            evy[a] = e1[T_EVY];
            c3[a] = e1[T_C3];
            c4[a] = e1[T_C4];
        }

        // acc[i][2], acc[i][3], acc[i][4] hold cells p-1, p, p+1: every
        // contribution goes straight into its slot.  The y-corner terms are
        // linear in the per-row differences G = s[vy-1]-s[vy+1] and
        // D = s[vx-1]-s[vx+1]:  c4 diag(y,vy) = c4 (G(y+1) - G(y-1)),
        // -c3 diag(y,vx) = -c3 (D(y+1) - D(y-1)); each row's G and D are
        // consumed as soon as they exist (rows -1 and 2 are the y arms).
        double s0[NC];

        // ---- own rows (a = 0, 1): vy lines, vx lines, D and G -------------
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            SCHED_FENCE();  // one row at a time
            const double *ca = c + a * KL;
            double v[BB][7];
#pragma unroll
            for (int b = 0; b < BB; ++b)
#pragma unroll
                for (int d = 0; d < 7; ++d) v[b][d] = ca[b * TW + d - 3];
            double r0[BB + 6];  // vy-offset-0 values at vx offsets -3 .. BB+2
            r0[0] = ca[-3 * TW];
            r0[1] = ca[-2 * TW];
            r0[2] = ca[-TW];
            r0[BB + 3] = ca[BB * TW];
            r0[BB + 4] = ca[(BB + 1) * TW];
            r0[BB + 5] = ca[(BB + 2) * TW];
            double G[BB], D[BB];
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                r0[b + 3] = v[b][3];
                s0[a * BB + b] = v[b][3];
                G[b] = v[b][2] - v[b][4];
            }
#pragma unroll
            for (int b = 0; b < BB; ++b) D[b] = r0[b + 2] - r0[b + 4];
            // x-coupled corrections: cell p-1 gets c1(p-1) D(p) - c5(p-1) G(p),
            // cell p+1 gets -c1(p+1) D(p) + c5(p+1) G(p)
            const double *e0 = tb + a * 8, *e2 = e0 + 2 * BJ * 8;
            const double c1m = e0[T_C1], c5m = e0[T_C5], c1p = e2[T_C1], c5p = e2[T_C5];
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                const int i = a * BB + b;
                acc[i][2] = fma(c1m, D[b], fma(-c5m, G[b], acc[i][2]));
                acc[i][4] = fma(-c1p, D[b], fma(c5p, G[b], acc[i][4]));
            }
            if (inner) {
                // y corners of the other own row: G(0) and D(0) feed cell row 1
                // with the minus sign, G(1) and D(1) feed row 0 with the plus sign
                const int o = (1 - a) * BB;
                const double sg = a ? 1.0 : -1.0;
#pragma unroll
                for (int b = 0; b < BB; ++b)
                    acc[o + b][3] = fma(sg * c4[1 - a], G[b], fma(-sg * c3[1 - a], D[b], acc[o + b][3]));
                const double gm = ca[-TW - 1] - ca[-TW + 1];         // G at vx offset -1
                const double gp = ca[BB * TW - 1] - ca[BB * TW + 1];  // G at vx offset BB
                const double avx = evx[a] + cBvy;                    // a_vx is independent of vx
                const double avx_s = avx * mhvx;
                if (avx > 0.0) {
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        acc[a * BB + b][3] = fma(avx_s, wpos(r0[b], r0[b + 1], r0[b + 2], r0[b + 3], r0[b + 4], r0[b + 5]),
                                                acc[a * BB + b][3]);
                } else {
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        acc[a * BB + b][3] = fma(avx_s, wneg(r0[b + 1], r0[b + 2], r0[b + 3], r0[b + 4], r0[b + 5], r0[b + 6]),
                                                acc[a * BB + b][3]);
                }
                // a_vy = evy - cB vx: one branch for the row when the four
                // signs agree (always when cB == 0; fl(e + x) is monotone in x)
                if (evy[a] + bvx_min > 0.0) {
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        acc[a * BB + b][3] = fma((evy[a] + bvx[b]) * mhvy,
                                                wpos(v[b][0], v[b][1], v[b][2], v[b][3], v[b][4], v[b][5]), acc[a * BB + b][3]);
                } else if (evy[a] + bvx_max <= 0.0) {
#pragma unroll
                    for (int b = 0; b < BB; ++b)
                        acc[a * BB + b][3] = fma((evy[a] + bvx[b]) * mhvy,
                                                wneg(v[b][1], v[b][2], v[b][3], v[b][4], v[b][5], v[b][6]), acc[a * BB + b][3]);
                } else {
#pragma unroll
                    for (int b = 0; b < BB; ++b) {
                        const double avy = evy[a] + bvx[b];
                        const double w = avy > 0.0 ? wpos(v[b][0], v[b][1], v[b][2], v[b][3], v[b][4], v[b][5])
                                                   : wneg(v[b][1], v[b][2], v[b][3], v[b][4], v[b][5], v[b][6]);
                        acc[a * BB + b][3] = fma(avy * mhvy, w, acc[a * BB + b][3]);
                    }
                }
                // diag(vx,vy) = G(vx+1) - G(vx-1)
                double gr[BB + 2];
                gr[0] = gm;
                gr[BB + 1] = gp;
#pragma unroll
                for (int b = 0; b < BB; ++b) gr[b + 1] = G[b];
#pragma unroll
                for (int b = 0; b < BB; ++b) acc[a * BB + b][3] = fma(mc2, gr[b + 2] - gr[b], acc[a * BB + b][3]);
            }
        }

        // ---- y arms: y stencil, the arm rows' y corners, folded src operand --
        // (ypos is per thread: one branch around the loop, not one per b)
        auto yarms = [&](auto ypos_tag) {
            constexpr bool YP = decltype(ypos_tag)::value;
            const double *rm = c - KL, *rp = c + 2 * KL;  // rows a = -1 and a = 2
            // the arm rows at the thread's vy, vx offsets -1 .. BB, loaded once:
            // qm/qp and the D differences of all BB cells come from them
            // (12 loads instead of 24 per plane)
            double am[BB + 2], ap[BB + 2];
#pragma unroll
            for (int b = 0; b < BB + 2; ++b) {
                am[b] = rm[(b - 1) * TW];
                ap[b] = rp[(b - 1) * TW];
            }
#pragma unroll
            for (int b = 0; b < BB; ++b) {
                SCHED_FENCE();
                const double qm = am[b + 1], qp = ap[b + 1];
                const double Dkm = am[b] - am[b + 2];
                const double Dkp = ap[b] - ap[b + 2];
                const double Gm = rm[b * TW - 1] - rm[b * TW + 1];
                const double Gp = rp[b * TW - 1] - rp[b * TW + 1];
                const double z0 = s0[b], z1 = s0[BB + b];
                double w0, w1;
                if (YP) {
                    const double ym3 = c[-3 * KL + b * TW], ym2 = c[-2 * KL + b * TW], y3 = c[3 * KL + b * TW];
                    w0 = wpos(ym3, ym2, qm, z0, z1, qp);
                    w1 = wpos(ym2, qm, z0, z1, qp, y3);
                } else {
                    const double ym2 = c[-2 * KL + b * TW], y3 = c[3 * KL + b * TW], y4 = c[4 * KL + b * TW];
                    w0 = wneg(ym2, qm, z0, z1, qp, y3);
                    w1 = wneg(qm, z0, z1, qp, y3, y4);
                }
                double t0 = fma(ay_s, w0, acc[b][3]), t1 = fma(ay_s, w1, acc[BB + b][3]);
                t0 = fma(-c4[0], Gm, fma(c3[0], Dkm, t0));  // row -1 feeds row 0 with the minus sign
                t1 = fma(c4[1], Gp, fma(-c3[1], Dkp, t1));  // row 2 feeds row 1 with the plus sign
                acc[b][3] = fma(kfold, z0, t0);
                acc[BB + b][3] = fma(kfold, z1, t1);
            }
        };
        if (inner) {
            if (ypos)
                yarms(std::true_type{});
            else
                yarms(std::false_type{});
        }

        // ---- x stencil scatter, extract cell q, slide the window -------------
        double fin[NC];
        window_apply<BB>(acc, s0, ax_s, xpos, fin);

        // ---- finalise cells q: RK combination, store, non-finite, moment ----
        if (fin_q) {
            const int kb = (q - i0) % NOPB;  // operand buffer of this plane
            if (nops) tma::mbar_wait_s(opbar + kb * 8, ((q - i0) / NOPB) & 1);  // its ((q-i0)/NOPB)-th fill
            const double *op = opbuf + kb * (OPB / 8) + ooff;
            double out[NC];
            if (nops == 0) {
#pragma unroll
                for (int i = 0; i < NC; ++i) out[i] = cL * fin[i];
            } else if (nops == 1) {
#pragma unroll
                for (int i = 0; i < NC; ++i) out[i] = fma(cL, fin[i], oc0 * op[(i / BB) * BK * OPW + (i % BB) * OPW]);
            } else {
#pragma unroll
                for (int i = 0; i < NC; ++i) {
                    const int oi = (i / BB) * BK * OPW + (i % BB) * OPW;
                    out[i] = fma(cL, fin[i], fma(oc1, op[OPE + oi], oc0 * op[oi]));
                }
            }
            if (WS && nops) tma::mbar_arrive_s(opempty + kb * 8);  // this thread is done with the operand tiles
            double *dq = P.dest + gq;
            if (fold_fb) {  // cL == 0: the src operand could not be folded
#pragma unroll
                for (int i = 0; i < NC; ++i)
                    out[i] = fma(P.cfold, P.src[gq + (i / BB) * P2 + (i % BB) * P3], out[i]);
            }
#pragma unroll
            for (int i = 0; i < NC; ++i)  // default L2 policy (evict-first measured 0.3-0.5 % slower)
                dq[(i / BB) * P2 + (i % BB) * P3] = out[i];
            if (PEER && P.peer_lo && q < NG) {  // my plane q -> the low neighbour's ghost plane Nx + q
                double *pq = P.peer_lo + gq + (long long)P.Nx * P1;
#pragma unroll
                for (int i = 0; i < NC; ++i) pq[(i / BB) * P2 + (i % BB) * P3] = out[i];
            }
            if (PEER && P.peer_hi && q >= P.Nx - NG) {  // my plane q -> the high neighbour's ghost plane q - Nx
                double *pq = P.peer_hi + gq - (long long)P.Nx * P1;
#pragma unroll
                for (int i = 0; i < NC; ++i) pq[(i / BB) * P2 + (i % BB) * P3] = out[i];
            }
            bool bad = false;
            if (P.partials) {
                // reference fold tree over each aligned 16-wide vy chunk
                // (fields.py:28-47): transpose-reduce the NC rows over the 16
                // vy lanes; after level k lane bit k-1 selects the row half
                double w1;
                if (NC == 8) {
                    const bool o1 = tl & 1, o2 = tl & 2, o4 = tl & 4;
                    double w4[4], w2[2];
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        const double keep = o1 ? out[2 * m + 1] : out[2 * m];
                        const double send = o1 ? out[2 * m] : out[2 * m + 1];
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
                } else {  // NC == 4
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
                if (tl < NC) __stcs(ppart, w1);  // lane tl holds row tl = BB a + b
                bad = !isfinite(w1);  // every output of the half-warp reached some lane's row sum
            }
            if (P.nonfinite) {
                // the partials' row sums cover every output (inf/nan propagate;
                // a finite overflow only sends the warp to the exact scan);
                // without partials, one sum per thread
                if (!P.partials) {
                    double sum = out[0];
#pragma unroll
                    for (int i = 1; i < NC; ++i) sum += out[i];
                    bad = !isfinite(sum);
                }
                if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
                    for (int i = 0; i < NC; ++i)
                        if (!isfinite(out[i]))
                            atomicMin(P.nonfinite,
                                      (((unsigned long long)q * P.Ny + y0 + (i / BB)) * P.Nvx + vx0 + (i % BB)) * P.Nvy + vy);
                }
            }
        }
        gq += P1;
        ppart += pstep;
        if (WS)
            tma::mbar_arrive_s(emptybar + stage_s * 8);  // this thread is done with the stage
        else
            __syncthreads();  // the stage and the operand tiles are free for the next refill
    }
    if (PEER) peer_done_signal(P, WS ? GEO::THREADS : 0);
}

// ---------------------------------------------------------------------------
// moment from partials: per physical cell, fold over the vy chunks of every
// vx row (chunk sums are exact subtrees), then over vx, times vol.

__global__ void moment_partials_kernel(const double *__restrict__ part, double *__restrict__ n,
                                       int nphys, int nvx, int nlt, double vol) {
    extern __shared__ double sm[];  // per warp: two buffers of nvx
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int p = blockIdx.x * wpb + warp;
    if (p >= nphys) return;
    double *bufA = sm + (size_t)warp * 2 * nvx;
    const double x = moment_cell_warp(part + (size_t)p * nvx * nlt, nvx, nlt, bufA, bufA + nvx);
    if ((threadIdx.x & 31) == 0) n[p] = __dmul_rn(x, vol);
}

// Fast path for power-of-two Nvx (32..256) and chunk counts (1..16): one warp
// per physical cell, lane L holds the Nvx/32 consecutive vx rows
// [L*R, L*R+R) (all their chunks, 128-bit loads), folds each row's chunks and
// then its rows in registers -- the reference tree's first levels -- and the
// remaining levels with ascending xor shuffles (adjacent pairs first).
template <int R, int NLT>
__global__ void __launch_bounds__(256) moment_partials_vec_kernel(const double *__restrict__ part,
                                                                  double *__restrict__ n, int nphys, double vol) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nphys) return;
    const double *src = part + ((size_t)warp * 32 + lane) * (R * NLT);
    double rows[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {  // one vx row: its NLT chunks, folded in registers
        double x[NLT];
        if (NLT % 2 == 0) {
#pragma unroll
            for (int t = 0; t < NLT; t += 2) {
                const double2 d = __ldcs(reinterpret_cast<const double2 *>(src + r * NLT + t));
                x[t] = d.x;
                x[t + 1] = d.y;
            }
        } else {
            x[0] = __ldcs(src + r * NLT);
        }
#pragma unroll
        for (int w = 1; w < NLT; w <<= 1)
#pragma unroll
            for (int t = 0; t < NLT; t += 2 * w) x[t] = __dadd_rn(x[t], x[t + w]);
        rows[r] = x[0];
    }
#pragma unroll
    for (int w = 1; w < R; w <<= 1)  // the lane's rows, adjacent pairs level by level
#pragma unroll
        for (int t = 0; t < R; t += 2 * w) rows[t] = __dadd_rn(rows[t], rows[t + w]);
    double v = rows[0];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) n[warp] = __dmul_rn(v, vol);
}

// One CTA per physical cell, one thread per vx row (Nvx a power of two,
// 32..1024): the row's chunks folded in registers, rows 1-5 levels of the
// tree by xor shuffles, the warp sums' levels by warp 0 -- the same
// adjacent-pair tree as the kernels above, with Nvx threads' loads in flight
// per cell instead of 32 (a 256-cell 1D-2V grid is 256 warps otherwise).
template <int NLT>
__global__ void __launch_bounds__(1024) moment_partials_row_kernel(const double *__restrict__ part,
                                                                   double *__restrict__ n, double vol) {
    __shared__ double wsum[32];
    pdl_trigger();  // the 2D field chain after this is programmatic (every link waits first)
    pdl_wait();     // the stage kernel's partials
    const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    double v = fold_pow2<NLT>(part + ((size_t)p * blockDim.x + t) * NLT);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? wsum[lane] : 0.0;
        for (int off = 1; off < nw; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) n[p] = __dmul_rn(v, vol);
    }
}

// moment_partials_row_kernel that also stores n into every rank's density
// buffer (peer-mapped) and, from its last CTA, bumps every other rank's
// density signal word: the all-gather of the x-slab densities fused into
// the finish (DistributedSimulation halo="peer").
struct DensityPush {
    double *dst[8];               // this slab's rows in each rank's n (own included)
    unsigned long long *sig[8];   // the other ranks' density words
    int ndst, nsig;
    unsigned *done;
};

template <int NLT>
__global__ void __launch_bounds__(1024) moment_partials_push_kernel(const double *__restrict__ part, double vol,
                                                                    const DensityPush D) {
    __shared__ double wsum[32];
    const int p = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    double v = fold_pow2<NLT>(part + ((size_t)p * blockDim.x + t) * NLT);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? wsum[lane] : 0.0;
        for (int off = 1; off < nw; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
        v = __dmul_rn(__shfl_sync(0xffffffffu, v, 0), vol);  // lanes >= nw summed zeros
        if (lane < D.ndst) D.dst[lane][p] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (t == 0) {
        const unsigned prev = atomicAdd(D.done, 1u);
        if (prev == gridDim.x - 1) {
            *D.done = 0u;
            __threadfence_system();
            for (int k = 0; k < D.nsig; ++k) atomicAdd_system(D.sig[k], 1ull);
        }
    }
}

template <int R>
static bool launch_vec_r(const double *part, double *n, int nphys, int nlt, double vol, cudaStream_t s) {
    const int grid = (nphys + 7) / 8;
    switch (nlt) {
        case 1: moment_partials_vec_kernel<R, 1><<<grid, 256, 0, s>>>(part, n, nphys, vol); return true;
        case 2: moment_partials_vec_kernel<R, 2><<<grid, 256, 0, s>>>(part, n, nphys, vol); return true;
        case 4: moment_partials_vec_kernel<R, 4><<<grid, 256, 0, s>>>(part, n, nphys, vol); return true;
        case 8: moment_partials_vec_kernel<R, 8><<<grid, 256, 0, s>>>(part, n, nphys, vol); return true;
        case 16: moment_partials_vec_kernel<R, 16><<<grid, 256, 0, s>>>(part, n, nphys, vol); return true;
        default: return false;
    }
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launch

static int tile_cfg(int Nvx, int Nvy) {
    // 0: (8,16,16) tiles x 1 CTA/SM (default: measured best at 128^4 and, with
    // the species of a 64^4 run launched concurrently, at 64^4); 1: (8,8,16)
    // tiles x 2 CTAs/SM (VPFV_RB_CFG=1, or when Nvx is not a multiple of 16)
    static int env = -2;
    if (env == -2) {
        const char *e = getenv("VPFV_RB_CFG");
        env = e ? atoi(e) : -1;
    }
    if (env == 0 || env == 1) return env;
    return Nvx % 16 ? 1 : 0;
}

static int tile_bk(int Nvx, int Nvy) { return tile_cfg(Nvx, Nvy) == 1 ? rb::GeoPair::BK : rb::GeoWide::BK; }

bool tma_2d2v_eligible(int Nx, int Ny, int Nvx, int Nvy, unsigned flags) {
    if (flags & VPFV_EXACT) return false;
    if (flags & (VPFV_WRAP(2) | VPFV_WRAP(3))) return false;  // velocity ghosts must be stored
    if (Ny % rb::BJ || Nvx % tile_bk(Nvx, Nvy) || Nvy % rb::BL) return false;
    if (Nx < 1 || Ny < rb::BJ) return false;
    return tma_available();
}

int tma_2d2v_columns(int Ny, int Nvx, int Nvy) {
    return (Ny / rb::BJ) * (Nvx / tile_bk(Nvx, Nvy)) * (Nvy / rb::BL);
}

static bool rb_ws_enabled() {  // VPFV_RB_WS: the warp-specialised 2D-2V kernel (default on)
    static int ws = -1;
    if (ws < 0) {
        const char *e = getenv("VPFV_RB_WS");
#ifndef VPFV_RB_WS_DEFAULT
#define VPFV_RB_WS_DEFAULT 1
#endif
        ws = e ? atoi(e) != 0 : VPFV_RB_WS_DEFAULT;
    }
    return ws != 0;
}

template <class GEO>
static int launch_geo(const double *src, const double *const ops[rb::OPS_MAX], const double *tab, Stage22 P,
                      unsigned flags, int nseg, cudaStream_t s) {
    using namespace rb;
    const unsigned long long dims[4] = {(unsigned long long)P.Nvy + 6, (unsigned long long)P.Nvx + 6,
                                        (unsigned long long)P.Ny + 6, (unsigned long long)P.Nx + 6};
    const unsigned long long strides[3] = {dims[0] * 8, dims[0] * dims[1] * 8, dims[0] * dims[1] * dims[2] * 8};
    const unsigned box_core[4] = {GEO::TW, GEO::TK, BJ, 1}, box_halo[4] = {GEO::TW, GEO::TK, 3, 1},
                   box_op[4] = {GEO::OPW, GEO::BK, BJ, 1};
    Maps maps;
    if (!tma_map(src, 4, dims, strides, box_core, &maps.core) || !tma_map(src, 4, dims, strides, box_halo, &maps.halo))
        return set_error(VPFV_ECUDA, "cuTensorMapEncodeTiled failed");
    for (int o = 0; o < OPS_MAX; ++o) {
        if (o < P.nops) {
            if (!tma_map(ops[o], 4, dims, strides, box_op, &maps.op[o]))
                return set_error(VPFV_ECUDA, "cuTensorMapEncodeTiled failed");
        } else {
            maps.op[o] = maps.core;
        }
    }
    // packed tables [(Nx+2)][Ny][8]
    const unsigned long long tdims[3] = {8, (unsigned long long)P.Ny, (unsigned long long)P.Nx + 2};
    const unsigned long long tstr[2] = {64, (unsigned long long)P.Ny * 64};
    const unsigned tbox[3] = {8, (unsigned)BJ, 3};
    if (!tma_map(tab, 3, tdims, tstr, tbox, &maps.tab)) return set_error(VPFV_ECUDA, "table map failed");
    P.wrap_x = (flags & VPFV_WRAP(0)) != 0;
    P.wrap_y = (flags & VPFV_WRAP(1)) != 0;
    P.nseg = nseg < 1 ? 1 : nseg;
    P.seglen = (P.i1 - P.i0 + P.nseg - 1) / P.nseg;  // the caller set the x range [i0, i1)
    static int sjk[2] = {-1, -1};
    if (sjk[0] < 0) {
        const char *e = getenv("VPFV_SUPER");
        sjk[0] = 4;
        sjk[1] = 8;
        if (e) sscanf(e, "%d,%d", &sjk[0], &sjk[1]);
    }
    P.sj = sjk[0] > 0 ? sjk[0] : 1;
    P.sk = sjk[1] > 0 ? sjk[1] : 1;
    static bool attr = false;
    if (!attr) {
        if constexpr (GEO::NOPB == 1) {
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GEO::SMEM);
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GEO::SMEM);
        }
        if constexpr (GEO::MINB == 1 && GEO::THREADS == 256) {
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GEO::SMEM);
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GEO::SMEM);
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, false, true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GEO::SMEM);
            cudaFuncSetAttribute(stage2d2v_rb_kernel<GEO, false, true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GEO::SMEM);
        }
        attr = true;
    }
    const bool ws = rb_ws_enabled();
    const int nblocks = (P.Ny / BJ) * (P.Nvx / GEO::BK) * (P.Nvy / BL) * P.nseg;
    bool launched = false;
    if constexpr (GEO::MINB == 1 && GEO::THREADS == 256) {  // one CTA per SM: the register pool setmaxnreg redistributes
        if (ws) {
#ifndef VPFV_RB_NV_DEFAULT
#define VPFV_RB_NV_DEFAULT 1
#endif
            static int nv = -1;
            if (nv < 0) {
                const char *e = getenv("VPFV_RB_NV");
                nv = e ? atoi(e) != 0 : VPFV_RB_NV_DEFAULT;
            }
            if (P.done)
                launch_pdl(stage2d2v_rb_kernel<GEO, true, true>, dim3(nblocks), dim3(GEO::THREADS + 128), GEO::SMEM, s, maps, P);
            else if (nv && P.Nvx == 128 && P.Nvy == 128)
                launch_pdl(stage2d2v_rb_kernel<GEO, false, true, 128>, dim3(nblocks), dim3(GEO::THREADS + 128), GEO::SMEM, s, maps, P);
            else if (nv && P.Nvx == 64 && P.Nvy == 64)  // config 5's 2 x 64^4
                launch_pdl(stage2d2v_rb_kernel<GEO, false, true, 64>, dim3(nblocks), dim3(GEO::THREADS + 128), GEO::SMEM, s, maps, P);
            else
                launch_pdl(stage2d2v_rb_kernel<GEO, false, true>, dim3(nblocks), dim3(GEO::THREADS + 128), GEO::SMEM, s, maps, P);
            launched = true;
        }
    }
    if constexpr (GEO::NOPB != 1) {
        if (!launched) return set_error(VPFV_EARG, "double-buffered operand geometry needs the warp-specialised kernel");
    } else if (!launched) {
        if (P.done)
            launch_pdl(stage2d2v_rb_kernel<GEO, true>, dim3(nblocks), dim3(GEO::THREADS), GEO::SMEM, s, maps, P);
        else
            launch_pdl(stage2d2v_rb_kernel<GEO, false>, dim3(nblocks), dim3(GEO::THREADS), GEO::SMEM, s, maps, P);
    }
    return check_launch("stage_2d2v_tma");
}

static int launch_rb(const double *src, const double *const ops[rb::OPS_MAX], const double *tab, Stage22 P,
                     unsigned flags, int nseg, cudaStream_t s) {
    if (tile_cfg(P.Nvx, P.Nvy) == 1) return launch_geo<rb::GeoPair>(src, ops, tab, P, flags, nseg, s);
    static int opdb = -1;
    if (opdb < 0) {
        const char *e = getenv("VPFV_RB_OPDB");
#ifndef VPFV_RB_OPDB_DEFAULT
#define VPFV_RB_OPDB_DEFAULT 0  // measured: stages 2-4 +2 % (the 2-deep halo ring costs more than the decoupling gains)
#endif
        opdb = e ? atoi(e) != 0 : VPFV_RB_OPDB_DEFAULT;
    }
    if (opdb && P.nops > 0 && rb_ws_enabled()) return launch_geo<rb::GeoWideOp>(src, ops, tab, P, flags, nseg, s);
    return launch_geo<rb::GeoWide>(src, ops, tab, P, flags, nseg, s);
}

int launch_moment_from_partials(const double *part, double *n, int nphys, int nvx, int nlt, double vol,
                                cudaStream_t s) {
    if (nlt > 16) return set_error(VPFV_EARG, "moment partials: at most 16 vy chunks");
    if (nvx >= 32 && nvx <= 1024 && (nvx & (nvx - 1)) == 0 && (nlt & (nlt - 1)) == 0) {
        switch (nlt) {
            case 1: launch_pdl(moment_partials_row_kernel<1>, dim3(nphys), dim3(nvx), 0, s, part, n, vol); break;
            case 2: launch_pdl(moment_partials_row_kernel<2>, dim3(nphys), dim3(nvx), 0, s, part, n, vol); break;
            case 4: launch_pdl(moment_partials_row_kernel<4>, dim3(nphys), dim3(nvx), 0, s, part, n, vol); break;
            case 8: launch_pdl(moment_partials_row_kernel<8>, dim3(nphys), dim3(nvx), 0, s, part, n, vol); break;
            default: launch_pdl(moment_partials_row_kernel<16>, dim3(nphys), dim3(nvx), 0, s, part, n, vol); break;
        }
        return check_launch("moment_from_partials");
    }
    bool done = false;
    switch (nvx) {
        case 32: done = launch_vec_r<1>(part, n, nphys, nlt, vol, s); break;
        case 64: done = launch_vec_r<2>(part, n, nphys, nlt, vol, s); break;
        case 128: done = launch_vec_r<4>(part, n, nphys, nlt, vol, s); break;
        case 256: done = launch_vec_r<8>(part, n, nphys, nlt, vol, s); break;
        default: break;
    }
    if (done) return check_launch("moment_from_partials");
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

namespace {
// RK operands ca A + cb B + cd dest grouped by array: the src-aliased part
// is folded into the accumulator, the others are staged by TMA.
struct Operands {
    const double *ptr[3];
    double coef[3];
    int n = 0;
    double cfold = 0.0;
    int fold = 0;
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

static int stage_2d2v_fused_impl(double *dest, const double *A, const double *B, const double *src, double ca,
                                 double cb, double cd, double cL, const double *vxc, const double *vyc,
                                 const double *evx, const double *evy, double cB, const double *c1, double c2,
                                 const double *c3, const double *c4, const double *c5, double hx, double hy,
                                 double hvx, double hvy, int Nx, int Ny, int Nvx, int Nvy, int x_begin, int x_end,
                                 unsigned flags, const double *dt_dev, double cL_div, unsigned long long *nonfinite,
                                 const double *packed_tables, double *moment_partials, int xsegments,
                                 void *stream, const Stage22 *peer = nullptr) {
    if (dest == src) return set_error(VPFV_EALIAS, "dest must not alias src");
    if (x_begin < 0 || x_end > Nx || x_begin > x_end) return set_error(VPFV_EARG, "bad x range");
    if (x_begin == x_end) return VPFV_OK;
    const bool full = x_begin == 0 && x_end == Nx;
    Operands ops;
    ops.add(A, ca, src);
    ops.add(B, cb, src);
    ops.add(dest, cd, src);
    if (!packed_tables || !tma_2d2v_eligible(Nx, Ny, Nvx, Nvy, flags) || ops.n > rb::OPS_MAX) {
        if (moment_partials) return set_error(VPFV_EARG, "fused moment needs the tiled 2D-2V path");
        if (peer) return set_error(VPFV_EARG, "peer halo push needs the tiled 2D-2V path");
        if (!full) return set_error(VPFV_EARG, "x sub-ranges need the tiled 2D-2V path");
        return vpfv_stage_2d2v_generic(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2,
                                       c3, c4, c5, hx, hy, hvx, hvy, Nx, Ny, Nvx, Nvy, flags, dt_dev,
                                       cL_div, nonfinite, stream);
    }
    Stage22 P{};
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
    P.i0 = x_begin;
    P.i1 = x_end;
    P.partials = moment_partials;
    if (peer) {
        P.peer_lo = peer->peer_lo;
        P.peer_hi = peer->peer_hi;
        P.sig_lo = peer->sig_lo;
        P.sig_hi = peer->sig_hi;
        P.done = peer->done;
    }
    int nseg = xsegments;
    static int env_seg = -1;
    if (env_seg < 0) {
        const char *e = getenv("VPFV_XSEG");
        env_seg = e ? atoi(e) : 0;
    }
    if (env_seg > 0) nseg = env_seg;  // VPFV_XSEG overrides the caller (A/B experiments)
    if (nseg <= 0) {  // ~1.5 waves of one CTA per SM, segments >= 8 planes (each adds 6 x-halo planes)
        const int cols = tma_2d2v_columns(Ny, Nvx, Nvy);
        nseg = (3 * 148 / 2 + cols - 1) / cols;
        if (nseg > (x_end - x_begin) / 8) nseg = (x_end - x_begin) / 8;
        if (nseg < 1) nseg = 1;
    }
    const double *opp[rb::OPS_MAX] = {ops.n > 0 ? ops.ptr[0] : nullptr, ops.n > 1 ? ops.ptr[1] : nullptr};
    return launch_rb(src, opp, packed_tables, P, flags, nseg, (cudaStream_t)stream);
}

extern "C" int vpfv_stage_2d2v_fused(double *dest, const double *A, const double *B,
                                     const double *src, double ca, double cb, double cd, double cL,
                                     const double *vxc, const double *vyc, const double *evx,
                                     const double *evy, double cB, const double *c1, double c2,
                                     const double *c3, const double *c4, const double *c5, double hx,
                                     double hy, double hvx, double hvy, int Nx, int Ny, int Nvx,
                                     int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                                     unsigned long long *nonfinite, const double *packed_tables,
                                     double *moment_partials, int xsegments, void *stream) {
    return stage_2d2v_fused_impl(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2, c3, c4, c5, hx,
                                 hy, hvx, hvy, Nx, Ny, Nvx, Nvy, 0, Nx, flags, dt_dev, cL_div, nonfinite,
                                 packed_tables, moment_partials, xsegments, stream);
}

extern "C" int vpfv_stage_2d2v_fused_range(double *dest, const double *A, const double *B,
                                           const double *src, double ca, double cb, double cd, double cL,
                                           const double *vxc, const double *vyc, const double *evx,
                                           const double *evy, double cB, const double *c1, double c2,
                                           const double *c3, const double *c4, const double *c5, double hx,
                                           double hy, double hvx, double hvy, int Nx, int Ny, int Nvx,
                                           int Nvy, int x_begin, int x_end, unsigned flags,
                                           const double *dt_dev, double cL_div,
                                           unsigned long long *nonfinite, const double *packed_tables,
                                           double *moment_partials, void *stream) {
    return stage_2d2v_fused_impl(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2, c3, c4, c5, hx,
                                 hy, hvx, hvy, Nx, Ny, Nvx, Nvy, x_begin, x_end, flags, dt_dev, cL_div, nonfinite,
                                 packed_tables, moment_partials, 0, stream);
}

extern "C" int vpfv_stage_2d2v_fused_peer(double *dest, const double *A, const double *B, const double *src,
                                          double ca, double cb, double cd, double cL, const double *vxc,
                                          const double *vyc, const double *evx, const double *evy, double cB,
                                          const double *c1, double c2, const double *c3, const double *c4,
                                          const double *c5, double hx, double hy, double hvx, double hvy, int Nx,
                                          int Ny, int Nvx, int Nvy, unsigned flags, const double *dt_dev,
                                          double cL_div, unsigned long long *nonfinite,
                                          const double *packed_tables, double *moment_partials, double *peer_lo,
                                          double *peer_hi, unsigned long long *sig_lo, unsigned long long *sig_hi,
                                          unsigned *done, void *stream) {
    if (!packed_tables || !tma_2d2v_eligible(Nx, Ny, Nvx, Nvy, flags))
        return set_error(VPFV_EARG, "peer halo push needs the tiled 2D-2V path");
    if (Nx < NG || !done) return set_error(VPFV_EARG, "peer halo push: Nx >= 3 and a done counter");
    Stage22 peer{};
    peer.peer_lo = peer_lo;
    peer.peer_hi = peer_hi;
    peer.sig_lo = sig_lo;
    peer.sig_hi = sig_hi;
    peer.done = done;
    return stage_2d2v_fused_impl(dest, A, B, src, ca, cb, cd, cL, vxc, vyc, evx, evy, cB, c1, c2, c3, c4, c5, hx,
                                 hy, hvx, hvy, Nx, Ny, Nvx, Nvy, 0, Nx, flags, dt_dev, cL_div, nonfinite,
                                 packed_tables, moment_partials, 0, stream, &peer);
}

extern "C" int vpfv_moment_partials_push(const double *partials, int nphys, int Nvx, int nchunks, double vol,
                                         double *const *dst, int ndst, unsigned long long *const *sig, int nsig,
                                         unsigned *done, void *stream) {
    if (ndst < 1 || ndst > 8 || nsig < 0 || nsig > 8 || !done)
        return set_error(VPFV_EARG, "moment_partials_push: 1..8 destinations, 0..8 signals, a done counter");
    if (Nvx < 32 || Nvx > 1024 || (Nvx & (Nvx - 1)) || nchunks < 1 || nchunks > 16 || (nchunks & (nchunks - 1)))
        return set_error(VPFV_EARG, "moment_partials_push: Nvx a power of two in [32, 1024], chunks in {1..16}");
    DensityPush D{};
    for (int k = 0; k < ndst; ++k) D.dst[k] = dst[k];
    for (int k = 0; k < nsig; ++k) D.sig[k] = sig[k];
    D.ndst = ndst;
    D.nsig = nsig;
    D.done = done;
    cudaStream_t s = (cudaStream_t)stream;
    switch (nchunks) {
        case 1: moment_partials_push_kernel<1><<<nphys, Nvx, 0, s>>>(partials, vol, D); break;
        case 2: moment_partials_push_kernel<2><<<nphys, Nvx, 0, s>>>(partials, vol, D); break;
        case 4: moment_partials_push_kernel<4><<<nphys, Nvx, 0, s>>>(partials, vol, D); break;
        case 8: moment_partials_push_kernel<8><<<nphys, Nvx, 0, s>>>(partials, vol, D); break;
        default: moment_partials_push_kernel<16><<<nphys, Nvx, 0, s>>>(partials, vol, D); break;
    }
    return check_launch("moment_partials_push");
}

extern "C" int vpfv_moment_partials(const double *partials, double *n, int nphys, int Nvx, int nchunks,
                                    double vol, void *stream) {
    return launch_moment_from_partials(partials, n, nphys, Nvx, nchunks, vol, (cudaStream_t)stream);
}

extern "C" int vpfv_stage_2d2v_tiled_ok(int Nx, int Ny, int Nvx, int Nvy, unsigned flags) {
    return tma_2d2v_eligible(Nx, Ny, Nvx, Nvy, flags) && Nvy / rb::BL <= 16 ? 1 : 0;
}

extern "C" int vpfv_stage_2d2v_partials_chunk(void) { return rb::BL; }
