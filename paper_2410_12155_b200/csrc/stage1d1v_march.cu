// 1D-1V fused stage, x-marching with bulk-copied rows (sm_100a, fast path).
//
// Operator of stage_1d1v (/root/reference/pkg/src/vpfv/_kernels.py:92-114):
//   rhs = -a_x D_x f - a_v D_v f + c1[i] diag(x, v),  a_x = ax[j], a_v = avx[i]
//   dest = ca A + cb B + cd dest + cL rhs                 (interior cells only)
//
// The generic kernel (stage.cu) gives every cell its own thread and ~20
// cached global loads with modular index arithmetic; at 1024^2 that is
// issue-bound at a fifth of the L2 bandwidth.  Here a CTA (128 threads) owns
// a 128-wide v column block and marches bx rows of x:
//  * each x row of src (the 134-double v segment with its 3-cell halos, one
//    contiguous 16-byte-aligned run of the padded array) and the rows of the
//    RK operands that do not alias src arrive by cp.async.bulk, two rows per
//    mbarrier, 8 row pairs deep, 4 pairs ahead of the x window;
//  * a thread computes two rows per step; a producer warp refills ring
//    slots as the compute warps release them (full/empty mbarriers);
//  * a thread's x stencil is its own column of the ring, the v stencil and
//    the diagonal corner terms the neighbouring columns: no index math per
//    load, one barrier per row;
//  * per-cell arithmetic is the generic fast kernel's expression for
//    expression (fd sums, FMA order, RK combination), so both paths agree
//    bitwise; the optional fold-tree moment partials are the same
//    128-wide-chunk sums (partials[i][0][chunk]).
// Requirements (else the generic kernel runs): fast path, Nv % 128 == 0,
// stored (non-periodic) v ghosts.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "tma.cuh"

namespace vpfv {

namespace m11 {
constexpr int W = 128;    // v cells per CTA (one column per thread)
constexpr int RS = W + 6;  // src row: interior j0-3 .. j0+130 (134 doubles = 1072 B)
constexpr int OS = W + 2;  // operand row: interior j0-1 .. j0+128 (130 doubles, 16-byte aligned start)
constexpr int NP = 8;      // ring of row pairs (16 rows)
constexpr int PFP = 4;     // pairs in flight ahead of the window's leading pair
constexpr int BX_MAX = 64;
static_assert(PFP + 4 <= NP, "the refilled pair must be older than the x window");
}  // namespace m11

struct March11 {
    double *dest;
    const double *src;
    const double *ops[3];  // RK operands staged by the ring (those not aliasing src): A, B, dest
    int opA, opB, opD;     // their ring index, or -1 (A/B aliasing src, dest with cd == 0)
    int nops;
    double ca, cb, cd, cL;
    const double *dt_dev;
    double cL_div;
    unsigned long long *nonfinite;
    const double *ax, *avx, *c1;
    double mhx, mhv;
    int Nx, Nv, bx;
    int wrap_x;
    double *partials;  // [Nx][Nv/128] or nullptr
};

// fd_sum of stage.cu on a 7-value window v[0..6] = s[-3..+3]
__device__ __forceinline__ double fd7(bool pos, double v0, double v1, double v2, double v3, double v4, double v5,
                                      double v6) {
    double t;
    if (pos) {
        t = -2.0 * v0;
        t = fma(15.0, v1, t);
        t = fma(-60.0, v2, t);
        t = fma(20.0, v3, t);
        t = fma(30.0, v4, t);
        t = fma(-3.0, v5, t);
    } else {
        t = 3.0 * v1;
        t = fma(-30.0, v2, t);
        t = fma(-20.0, v3, t);
        t = fma(60.0, v4, t);
        t = fma(-15.0, v5, t);
        t = fma(2.0, v6, t);
    }
    return t;
}

// 128-wide chunk sum of one row: shuffle levels, then the 4 warp sums pairwise
__device__ __forceinline__ double warp_fold(double v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// OPS: which RK terms are present (bit 0: ca A, 1: cb B, 2: cd dest) -- the
// combination's tests are resolved at compile time.  Warps 0-3 compute (one
// v column per thread), warp 4 is the producer: it refills a ring slot as
// soon as the four compute warps have released it (empty barrier), so no
// CTA-wide barrier sits on the compute path.
template <int OPS>
__global__ void __launch_bounds__(160, 1) stage_1d1v_march_kernel(const March11 P) {
    using namespace m11;
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t full[NP], empty[NP];
    __shared__ double tabs[2][BX_MAX];
    __shared__ double wsum[2][2][4];  // [pair parity][row of the pair][warp]
    double *ring = sm;                // NP x 2 x RS
    double *opr = sm + NP * 2 * RS;   // nops x NP x 2 x OS
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = blockIdx.x * W, j = j0 + tid;
    const int i0 = blockIdx.y * P.bx, i1 = min(i0 + P.bx, P.Nx);
    const int Nx = P.Nx;
    const long long P1 = P.Nv + 2 * NG;
    const int rfirst = i0 - 3, rlast = i1 + 2;  // rows read; row r is ring row R = r - rfirst, pair R >> 1
    const unsigned full_s = tma::smem_addr(full), empty_s = tma::smem_addr(empty);

    if (tid == 0) {
        for (int q = 0; q < NP; ++q) {
            tma::mbar_init(&full[q], 1);
            tma::mbar_init(&empty[q], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();  // the tables (field kernel) and src / operands of the preceding launches
    for (int k = tid; k < i1 - i0; k += blockDim.x) {
        tabs[0][k] = __ldg(P.avx + i0 + k);
        tabs[1][k] = __ldg(P.c1 + i0 + k);
    }
    __syncthreads();

    if (warp == 4) {  // producer: pair q = ring rows 2q, 2q+1 (src segments + operand rows of interior rows)
        if (lane != 0) return;
        const unsigned ring_s = tma::smem_addr(ring), opr_s = tma::smem_addr(opr);
        const unsigned src_bytes = RS * 8, op_bytes = OS * 8;
        const int nops = P.nops;
        const int npairs = (rlast - rfirst + 2) / 2;
        for (int q = 0; q < npairs; ++q) {
            const int slot = q & (NP - 1);
            if (q >= NP) tma::mbar_wait_s(empty_s + slot * 8, ((q / NP) - 1) & 1);
            const int r0 = rfirst + 2 * q;
            const int nr = r0 + 1 <= rlast ? 2 : 1;
            int nint = 0;
            for (int k = 0; k < nr; ++k) nint += (r0 + k >= i0 && r0 + k < i1) ? 1 : 0;
            const unsigned bar = full_s + slot * 8;
            tma::mbar_expect_tx_s(bar, nr * src_bytes + nint * nops * op_bytes);
            for (int k = 0; k < nr; ++k) {
                const int r = r0 + k;
                int rr = r;
                if (P.wrap_x) rr = r < 0 ? r + Nx : (r >= Nx ? r - Nx : r);
                tma::bulk_g2s(ring_s + (slot * 2 + k) * RS * 8, P.src + (long long)(rr + NG) * P1 + j0, src_bytes,
                              bar);
                if (r >= i0 && r < i1)
                    for (int o = 0; o < nops; ++o)
                        tma::bulk_g2s(opr_s + ((o * NP + slot) * 2 + k) * OS * 8,
                                      P.ops[o] + (long long)(r + NG) * P1 + NG + j0 - 1, op_bytes, bar);
            }
        }
        return;
    }

    auto wait_pair = [&](int q) { tma::mbar_wait_s(full_s + (q & (NP - 1)) * 8, (q / NP) & 1); };
    const double a_x = __ldg(P.ax + j);
    const double kx = a_x * P.mhx, mhv = P.mhv;
    const bool posx = a_x > 0.0;
    const double cL = P.dt_dev ? __ddiv_rn(*P.dt_dev, P.cL_div) : P.cL;
    const double ca = P.ca, cb = P.cb, cd = P.cd;
    (void)ca, (void)cb, (void)cd;
    const int opA = P.opA, opB = P.opB, opD = P.opD;
    const int Nv = P.Nv;
    double *const dest = P.dest;
    double *const partials = P.partials;
    for (int q = 0; q < 3; ++q) wait_pair(q);
    unsigned long long first_bad = ~0ull;  // smallest non-finite flat index seen by this thread

    // RK combination of finish<false> (stage.cu) for the cell in ring row R
    auto combine = [&](double rhs, double s0, int R) {
        const double *o = opr + ((R >> 1) & (NP - 1)) * 2 * OS + (R & 1) * OS + tid + 1;
        double out = cL * rhs;
        if (OPS & 4) out = fma(cd, o[opD * NP * 2 * OS], out);
        if (OPS & 2) out = fma(cb, opB < 0 ? s0 : o[opB * NP * 2 * OS], out);
        if (OPS & 1) out = fma(ca, opA < 0 ? s0 : o[opA * NP * 2 * OS], out);
        return out;
    };

    for (int t = 0, i = i0; i < i1; ++t, i += 2) {  // rows i, i+1 = ring rows 2t+3, 2t+4
        wait_pair(t + 3);
        const double *p0 = ring + ((t + 0) & (NP - 1)) * 2 * RS, *p1 = ring + ((t + 1) & (NP - 1)) * 2 * RS;
        const double *p2 = ring + ((t + 2) & (NP - 1)) * 2 * RS, *p3 = ring + ((t + 3) & (NP - 1)) * 2 * RS;
        // ring rows 2t .. 2t+7 = x rows i-3 .. i+4 (row i+4 is stale when i+1 == i1: unused)
        const double *y2 = p1, *y3 = p1 + RS, *y4 = p2, *y5 = p2 + RS;
        const int c = tid + 3;
        const double x0 = p0[c], x1 = p0[RS + c], x2 = y2[c], x3 = y3[c], x4 = y4[c], x5 = y5[c], x6 = p3[c],
                     x7 = p3[RS + c];
        const bool two = i + 1 < i1;
        const int k0 = i - i0, k1 = two ? k0 + 1 : k0;
        const double av0 = tabs[0][k0], c10 = tabs[1][k0], av1 = tabs[0][k1], c11 = tabs[1][k1];
        // both rows' chains side by side (row i: v row y3, diagonal rows y2/y4;
        // row i+1: v row y4, diagonal rows y3/y5)
        double rhs0 = kx * fd7(posx, x0, x1, x2, x3, x4, x5, x6);
        double rhs1 = kx * fd7(posx, x1, x2, x3, x4, x5, x6, x7);
        rhs0 = fma(av0 * mhv,
                   fd7(av0 > 0.0, y3[tid], y3[tid + 1], y3[tid + 2], x3, y3[tid + 4], y3[tid + 5], y3[tid + 6]), rhs0);
        rhs1 = fma(av1 * mhv,
                   fd7(av1 > 0.0, y4[tid], y4[tid + 1], y4[tid + 2], x4, y4[tid + 4], y4[tid + 5], y4[tid + 6]), rhs1);
        rhs0 = fma(c10, ((y4[tid + 2] + y2[tid + 4]) - y4[tid + 4]) - y2[tid + 2], rhs0);
        rhs1 = fma(c11, ((y5[tid + 2] + y3[tid + 4]) - y5[tid + 4]) - y3[tid + 2], rhs1);
        const double out0 = combine(rhs0, x3, 2 * t + 3);
        const double out1 = two ? combine(rhs1, x4, 2 * t + 4) : 0.0;
        __syncwarp();
        if (lane == 0) tma::mbar_arrive_s(empty_s + (t & (NP - 1)) * 8);  // pair t is no longer read
        dest[(long long)(i + NG) * P1 + NG + j] = out0;
        if (!isfinite(out0)) first_bad = min(first_bad, (unsigned long long)i * Nv + j);
        if (two) {
            dest[(long long)(i + 1 + NG) * P1 + NG + j] = out1;
            if (!isfinite(out1)) first_bad = min(first_bad, (unsigned long long)(i + 1) * Nv + j);
        }
        if (partials) {
            const double v0 = warp_fold(out0), v1 = warp_fold(out1);
            if (lane == 0) {
                wsum[t & 1][0][warp] = v0;
                wsum[t & 1][1][warp] = v1;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the compute warps' sums of this pair
            if (tid == 0) {
                const double *w0 = wsum[t & 1][0], *w1 = wsum[t & 1][1];
                const long long o = (long long)i * gridDim.x + blockIdx.x;
                partials[o] = __dadd_rn(__dadd_rn(w0[0], w0[1]), __dadd_rn(w0[2], w0[3]));
                if (two) partials[o + gridDim.x] = __dadd_rn(__dadd_rn(w1[0], w1[1]), __dadd_rn(w1[2], w1[3]));
            }
        }
    }
    if (P.nonfinite && first_bad != ~0ull) atomicMin(P.nonfinite, first_bad);
}

// host: eligibility and launch (called by vpfv_stage_1d1v[_fused], stage.cu)
bool march_1d1v_eligible(int Nx, int Nv, unsigned flags) {
    if (flags & VPFV_EXACT) return false;
    if (flags & VPFV_WRAP(1)) return false;  // v ghosts must be stored
    if (Nv % m11::W || Nx < 1) return false;
    const char *e = getenv("VPFV_1D1V_MARCH");  // 0: generic kernel, 1: always march (tests, A/B)
    const int env = e ? atoi(e) : -1;
    if (env == 0) return false;
    if (env == 1) return true;
    return (long long)Nx * Nv >= (1 << 18);  // small grids are latency-bound: the generic kernel's 1 row per CTA wins
}

int launch_1d1v_march(double *dest, const double *A, const double *B, const double *src, double ca, double cb,
                      double cd, double cL, const double *ax, const double *avx, const double *c1, double hx,
                      double hv, int Nx, int Nv, unsigned flags, const double *dt_dev, double cL_div,
                      unsigned long long *nonfinite, double *partials, cudaStream_t stream) {
    using namespace m11;
    March11 P{};
    P.dest = dest;
    P.src = src;
    P.nops = 0;
    P.opA = P.opB = P.opD = -1;
    if (ca != 0.0 && A != src) {
        P.opA = P.nops;
        P.ops[P.nops++] = A;
    }
    if (cb != 0.0 && B != src) {
        if (B == A && P.opA >= 0) {
            P.opB = P.opA;
        } else {
            P.opB = P.nops;
            P.ops[P.nops++] = B;
        }
    }
    if (cd != 0.0) {
        P.opD = P.nops;
        P.ops[P.nops++] = dest;
    }
    P.ca = ca;
    P.cb = cb;
    P.cd = cd;
    P.cL = cL;
    P.dt_dev = dt_dev;
    P.cL_div = cL_div;
    P.nonfinite = nonfinite;
    P.ax = ax;
    P.avx = avx;
    P.c1 = c1;
    P.mhx = -1.0 / (60.0 * hx);
    P.mhv = -1.0 / (60.0 * hv);
    P.Nx = Nx;
    P.Nv = Nv;
    P.wrap_x = (flags & VPFV_WRAP(0)) ? 1 : 0;
    P.partials = partials;
    // about `cps` CTAs per SM over the whole grid
    const char *e = getenv("VPFV_1D1V_CPS");
    const int cps = e ? atoi(e) : 4;
    const int nvb = Nv / W;
    int nxb = (148 * cps + nvb - 1) / nvb;
    int bx = (Nx + nxb - 1) / nxb;
    bx = bx < 4 ? 4 : (bx > BX_MAX ? BX_MAX : bx);
    bx += bx & 1;  // whole row pairs
    P.bx = bx;
    const size_t smem = sizeof(double) * 2 * ((size_t)NP * RS + (size_t)P.nops * NP * OS);
    const int ops = (ca != 0.0 ? 1 : 0) | (cb != 0.0 ? 2 : 0) | (cd != 0.0 ? 4 : 0);
    static const void *fns[8] = {
        (const void *)stage_1d1v_march_kernel<0>, (const void *)stage_1d1v_march_kernel<1>,
        (const void *)stage_1d1v_march_kernel<2>, (const void *)stage_1d1v_march_kernel<3>,
        (const void *)stage_1d1v_march_kernel<4>, (const void *)stage_1d1v_march_kernel<5>,
        (const void *)stage_1d1v_march_kernel<6>, (const void *)stage_1d1v_march_kernel<7>};
    static bool attr = false;
    if (!attr) {
        for (int k = 0; k < 8; ++k) cudaFuncSetAttribute(fns[k], cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    dim3 grid(nvb, (Nx + bx - 1) / bx);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    void *args[] = {(void *)&P};
    const cudaError_t rc = cudaLaunchKernelExC(&cfg, fns[ops], args);
    if (rc != cudaSuccess) return set_error(VPFV_ECUDA, cudaGetErrorString(rc));
    return check_launch("stage_1d1v_march");
}

}  // namespace vpfv
