/* vpfv.h -- C ABI of the B200-native VP-FV stage library (libvpfv.so, sm_100a).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `vpfv` (/root/reference/pkg/src/vpfv).  Every entry point takes plain
 * device pointers, sizes and a cudaStream_t (passed as void*), never
 * allocates, never synchronises, and is safe to capture in a CUDA graph.
 * All return an int status (VPFV_OK on success).
 *
 * Arrays named like the reference's are the reference's arrays: padded
 * float64 C-order storage `(N_0+6, ..., N_{D-1}+6)` with velocity dims
 * fastest (grid.py:3-8, :62-64), per-line tables as built by the reference
 * dispatcher `fused_stage` (_kernels.py:330-365).
 */
#ifndef VPFV_H
#define VPFV_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -- mapped to the reference's exceptions by the
 * Python host layer: EALIAS/EDIM/EARG -> ValueError (_kernels.py:328-329,
 * :366-367), ENONFINITE -> FloatingPointError (_kernels.py:368-373). */
#define VPFV_OK          0
#define VPFV_EALIAS      1
#define VPFV_EDIM        2
#define VPFV_ENONFINITE  3
#define VPFV_ECUDA       4
#define VPFV_EARG        5
#define VPFV_ENCCL       6

/* stage flags */
#define VPFV_EXACT       0x1   /* evaluate in the reference kernels' exact
                                  operation order (no FMA, IEEE division):
                                  bitwise equal to the numba kernels */
#define VPFV_WRAP_SHIFT  1     /* bit (1+k): dim k is periodic and is read by
                                  modular indexing into the interior instead
                                  of from its ghost storage */
#define VPFV_WRAP(k)     (1u << (VPFV_WRAP_SHIFT + (k)))

/* "no non-finite value seen" value of the non-finite index word */
#define VPFV_FINITE      0xFFFFFFFFFFFFFFFFull

/* ---------------------------------------------------------------------- */
/* Fused stage: dest = ca*A + cb*B + cd*dest + cL*RHS(src) on the interior.
 *
 * Replaces `stage_1d1v(dest, A, B, src, ca, cb, cd, cL, ax, avx, c1, hx, hv)`
 * (/root/reference/pkg/src/vpfv/_kernels.py:92-114), `stage_1d2v(...)`
 * (:153-197) and `stage_2d2v(...)` (:254-317), plus the non-finite scan of
 * `fused_stage` (:368-373), which is folded into the epilogue: if
 * `nonfinite` is non-NULL the C-order interior flat index of the first
 * non-finite output is atomically min-ed into it (initialise to
 * VPFV_FINITE).  `cL` is used as given unless `dt_dev` is non-NULL, in
 * which case cL = (*dt_dev) / cL_div is read on the device (lets one CUDA
 * graph serve every time step).  dest == src -> VPFV_EALIAS.
 */
int vpfv_stage_1d1v(double *dest, const double *A, const double *B, const double *src,
                    double ca, double cb, double cd, double cL,
                    const double *ax, const double *avx, const double *c1,
                    double hx, double hv, int Nx, int Nv,
                    unsigned flags, const double *dt_dev, double cL_div,
                    unsigned long long *nonfinite, void *stream);

/* 1D-1V stage with the fused velocity-moment epilogue (fast path, Nv % 128
 * == 0): as vpfv_stage_1d1v, and moment_partials[x][0][c] receives the
 * fold-tree subtree sum of the new dest over the aligned 128-wide v chunk c
 * (finish with vpfv_moment_partials(nphys = Nx, Nvx = 1, nchunks = Nv/128)).
 * moment_partials == NULL is vpfv_stage_1d1v. */
int vpfv_stage_1d1v_fused(double *dest, const double *A, const double *B, const double *src,
                          double ca, double cb, double cd, double cL, const double *ax,
                          const double *avx, const double *c1, double hx, double hv, int Nx, int Nv,
                          unsigned flags, const double *dt_dev, double cL_div,
                          unsigned long long *nonfinite, double *moment_partials, void *stream);

int vpfv_stage_1d2v(double *dest, const double *A, const double *B, const double *src,
                    double ca, double cb, double cd, double cL,
                    const double *vxc, const double *vyc /* Nvy+1, last = cB */,
                    const double *evx, const double *avy, const double *c1, double c2,
                    double hx, double hvx, double hvy, int Nx, int Nvx, int Nvy,
                    unsigned flags, const double *dt_dev, double cL_div,
                    unsigned long long *nonfinite, void *stream);

int vpfv_stage_2d2v(double *dest, const double *A, const double *B, const double *src,
                    double ca, double cb, double cd, double cL,
                    const double *vxc, const double *vyc, const double *evx,
                    const double *evy, double cB, const double *c1, double c2,
                    const double *c3, const double *c4, const double *c5,
                    double hx, double hy, double hvx, double hvy,
                    int Nx, int Ny, int Nvx, int Nvy,
                    unsigned flags, const double *dt_dev, double cL_div,
                    unsigned long long *nonfinite, void *stream);

/* 2D-2V stage with the fused velocity-moment epilogue: as vpfv_stage_2d2v,
 * and when moment_partials is non-NULL the kernel also writes, for every new
 * dest cell row (x, y, vx) and every aligned vy chunk c (width
 * vpfv_stage_2d2v_partials_chunk(), 16), the fold-tree subtree sum
 * moment_partials[((x*Ny + y)*Nvx + vx)*(Nvy/chunk) + c]
 * (finish with vpfv_moment_partials).  Runs the TMA-tiled x-marching kernel
 * (requires the fast path, stored velocity ghosts, Ny%8 == Nvx%16 == Nvy%16
 * == 0 and at most two RK operands besides src); otherwise falls back to the generic kernel (and rejects a non-NULL
 * moment_partials with VPFV_EARG).  The tiled path reads the E tables from
 * packed_tables (vpfv_tables_2d_packed); with packed_tables NULL the generic
 * kernel runs.  xsegments <= 0 picks a split of the x march automatically.
 * vpfv_stage_2d2v == this with packed_tables and moment_partials NULL. */
int vpfv_stage_2d2v_fused(double *dest, const double *A, const double *B, const double *src,
                          double ca, double cb, double cd, double cL,
                          const double *vxc, const double *vyc, const double *evx,
                          const double *evy, double cB, const double *c1, double c2,
                          const double *c3, const double *c4, const double *c5,
                          double hx, double hy, double hvx, double hvy,
                          int Nx, int Ny, int Nvx, int Nvy,
                          unsigned flags, const double *dt_dev, double cL_div,
                          unsigned long long *nonfinite, const double *packed_tables,
                          double *moment_partials, int xsegments, void *stream);

/* 1D-2V with the tiled x-marching kernel and optional fused moment partials
 * [Nx][Nvx][Nvy/16] (finish with vpfv_moment_partials(nphys = Nx)); tiled
 * when packed_tables (vpfv_tables_1d_packed) is given, the fast path is
 * requested, velocity ghosts are stored, Nvx % 32 == Nvy % 16 == 0 and at
 * most two RK operands differ from src; otherwise the generic kernel (and
 * moment_partials must be NULL). */
int vpfv_stage_1d2v_fused(double *dest, const double *A, const double *B, const double *src,
                          double ca, double cb, double cd, double cL,
                          const double *vxc, const double *vyc, const double *evx,
                          const double *avy, const double *c1, double c2,
                          double hx, double hvx, double hvy, int Nx, int Nvx, int Nvy,
                          unsigned flags, const double *dt_dev, double cL_div,
                          unsigned long long *nonfinite, const double *packed_tables,
                          double *moment_partials, int xsegments, void *stream);
int vpfv_stage_1d2v_tiled_ok(int Nx, int Nvx, int Nvy, unsigned flags);

/* Width of the vy chunks of the 1D-2V moment partials (16): partials hold
 * [Nx][Nvx][Nvy/chunk] fold-tree subtree sums. */
int vpfv_stage_1d2v_partials_chunk(void);

/* vpfv_stage_2d2v_fused (full x range) that also pushes its x halo to the
 * slab neighbours over peer memory: planes 0..2 of dest are stored into
 * peer_lo (the low x neighbour's dest, same padded shape) at its ghost planes
 * Nx..Nx+2, planes Nx-3..Nx-1 into peer_hi at ghost planes 0..2; the last CTA
 * then adds 1 to *sig_lo (the low neighbour's "from high" word) and *sig_hi
 * (the high neighbour's "from low" word).  done: a zeroed device counter per
 * concurrently running launch.  Replaces the per-stage halo exchange of the
 * reference cluster (runner.py:394-437, partition.py:679-724). */
int vpfv_stage_2d2v_fused_peer(double *dest, const double *A, const double *B, const double *src,
                               double ca, double cb, double cd, double cL, const double *vxc,
                               const double *vyc, const double *evx, const double *evy, double cB,
                               const double *c1, double c2, const double *c3, const double *c4,
                               const double *c5, double hx, double hy, double hvx, double hvy, int Nx,
                               int Ny, int Nvx, int Nvy, unsigned flags, const double *dt_dev,
                               double cL_div, unsigned long long *nonfinite,
                               const double *packed_tables, double *moment_partials, double *peer_lo,
                               double *peer_hi, unsigned long long *sig_lo, unsigned long long *sig_hi,
                               unsigned *done, void *stream);

/* vpfv_moment_partials (vol applied) whose results also go to every rank's
 * density buffer: dst[k] = this slab's first cell in rank k's n (peer-mapped,
 * own included); the last CTA then adds 1 to each sig[k] (the other ranks'
 * density words).  The all-gather of the x-slab densities of the reference
 * cluster's _global_density (runner.py:341-384) fused into the finish.
 * Nvx a power of two in [32, 1024]; <= 8 ranks. */
int vpfv_moment_partials_push(const double *partials, int nphys, int Nvx, int nchunks, double vol,
                              double *const *dst, int ndst, unsigned long long *const *sig, int nsig,
                              unsigned *done, void *stream);

/* vpfv_stage_1d2v_fused (full x range) with the same peer halo push as
 * vpfv_stage_2d2v_fused_peer (planes 0..2 / Nx-3..Nx-1 stored into the x
 * neighbours' ghost planes, the last CTA signalling sig_lo / sig_hi). */
int vpfv_stage_1d2v_fused_peer(double *dest, const double *A, const double *B, const double *src,
                               double ca, double cb, double cd, double cL, const double *vxc,
                               const double *vyc, const double *evx, const double *avy,
                               const double *c1, double c2, double hx, double hvx, double hvy, int Nx,
                               int Nvx, int Nvy, unsigned flags, const double *dt_dev, double cL_div,
                               unsigned long long *nonfinite, const double *packed_tables,
                               double *moment_partials, double *peer_lo, double *peer_hi,
                               unsigned long long *sig_lo, unsigned long long *sig_hi, unsigned *done,
                               void *stream);

/* Signal both neighbours once (after an initial halo exchange by other means).
 * With vpfv_peer_wait: the completion half of the reference cluster's halo
 * exchange (Exchanger, /root/reference/pkg/src/vpfv/partition.py:679-724). */
int vpfv_peer_signal(unsigned long long *sig_lo, unsigned long long *sig_hi, void *stream);

/* The step's divergence verdict across ranks over peer memory (the
 * reference rolls the whole cluster back when any box is non-finite,
 * runner.py:453-464): this rank's word (step << 1 | any nonfinite[s] != -1)
 * is stored into *slots[r] (its slot in rank r's flag array, peer-mapped;
 * `slots` is a device array of world such pointers) for every r; then it waits until every word of its own array `mine`
 * (world words) carries the step's stamp and writes the OR of their bad bits
 * to *out (device word; copy it to pinned memory to read it on the host).
 * `stamp` is this rank's device step counter.  Timeout -> *timed_out = 1 and
 * the rank counts as diverged.  No host synchronisation; graph-capturable. */
int vpfv_flag_exchange(const long long *nonfinite, int nspecies, unsigned long long *const *slots,
                       int world, const unsigned long long *mine, unsigned long long *stamp,
                       unsigned long long *out, double timeout_s, int *timed_out, void *stream);

/* Wait (one device thread, system-scope acquire) until sig[0] / sig[1] (this
 * rank's words, written by its low / high neighbour) exceed consumed[k] by
 * need_lo / need_hi, then advance consumed.  After timeout_s seconds it sets
 * *timed_out = 1 and returns instead of hanging the device. */
int vpfv_peer_wait(const unsigned long long *sig, unsigned long long *consumed, int need_lo, int need_hi,
                   double timeout_s, int *timed_out, void *stream);

/* CUDA IPC of a device buffer between rank processes (no reference
 * counterpart: the reference cluster shares one address space,
 * runner.py:259-496): export writes the
 * handle of the allocation holding ptr (vpfv_ipc_handle_size() bytes) and
 * ptr's offset in it; open maps it into the calling device's context with
 * peer access (once per allocation and process) and returns the buffer. */
int vpfv_ipc_handle_size(void);
int vpfv_ipc_export(const void *ptr, unsigned char *handle_out, long long *offset_out);
int vpfv_ipc_open(const unsigned char *handle, long long offset, void **ptr_out);

/* vpfv_stage_2d2v_fused restricted to the interior x cells [x_begin, x_end)
 * (tiled path only; VPFV_EARG otherwise).  Planes x_begin-3 .. x_end+2 are
 * read, so a slab whose x ghosts are still in flight can update its x
 * interior [3, Nx-3) while they arrive, then [0, 3) and [Nx-3, Nx): the
 * overlapped halo exchange of paper_2410_12155_b200.parallel.  Replaces the
 * per-box stage of SimulatedCluster._stage (runner.py:394-437). */
int vpfv_stage_2d2v_fused_range(double *dest, const double *A, const double *B, const double *src,
                                double ca, double cb, double cd, double cL,
                                const double *vxc, const double *vyc, const double *evx,
                                const double *evy, double cB, const double *c1, double c2,
                                const double *c3, const double *c4, const double *c5,
                                double hx, double hy, double hvx, double hvy,
                                int Nx, int Ny, int Nvx, int Nvy, int x_begin, int x_end,
                                unsigned flags, const double *dt_dev, double cL_div,
                                unsigned long long *nonfinite, const double *packed_tables,
                                double *moment_partials, void *stream);

/* 1 when vpfv_stage_2d2v_fused would take the tiled path (and so accepts
 * moment_partials) for these extents and flags, else 0. */
int vpfv_stage_2d2v_tiled_ok(int Nx, int Ny, int Nvx, int Nvy, unsigned flags);

/* Width of the vy chunks the fused-moment partials are summed over (the
 * tiled kernel's vy tile, 16): partials hold Nvy/chunk values per row. */
int vpfv_stage_2d2v_partials_chunk(void);

/* The untiled one-thread-per-cell 2D-2V kernel (exact or fast), always. */
int vpfv_stage_2d2v_generic(double *dest, const double *A, const double *B, const double *src,
                            double ca, double cb, double cd, double cL,
                            const double *vxc, const double *vyc, const double *evx,
                            const double *evy, double cB, const double *c1, double c2,
                            const double *c3, const double *c4, const double *c5,
                            double hx, double hy, double hvx, double hvy,
                            int Nx, int Ny, int Nvx, int Nvy,
                            unsigned flags, const double *dt_dev, double cL_div,
                            unsigned long long *nonfinite, void *stream);

/* Finish the fused moment: n[p] = fold(fold over chunks per vx row, then
 * over vx) * vol -- bitwise the reference fold tree when Nvy % 32 == 0. */
int vpfv_moment_partials(const double *partials, double *n, int nphys, int Nvx, int nchunks,
                         double vol, void *stream);

/* ---------------------------------------------------------------------- */
/* Velocity moment.  n[p] = fold_tree(f[p, :]) * vol over the velocity dims,
 * fastest axis first, adjacent pairs with the odd tail carried -- bitwise
 * the reference `zeroth_moment(f, "velocity-major")` (fields.py:28-47,
 * 86-111).  N holds the d+v interior extents. */
int vpfv_moment(const double *f, double *n, int d, int v, const int *N, double vol,
                void *stream);

/* Velocity moment with schedule="position-major": the per-cell sequential
 * sum s += f over the velocity interior in C order, then n = s * vol --
 * bitwise the reference's compiled _seq_moment_{2,3,4}d (fields.py:50-83,
 * :100-106). */
int vpfv_moment_seq(const double *f, double *n, int d, int v, const int *N, double vol,
                    void *stream);

/* Momentum / kinetic-energy velocity sums per physical cell with the
 * midpoint-to-average lift of higher_moments (fields.py:131-161):
 * out[p][2k] = sum_v (v_c f + h_k^2/12 df/dv_k),
 * out[p][2k+1] = sum_v ((v_c^2 + h_k^2/12) f + h_k^2/6 v_c df/dv_k) for each
 * velocity dim k (centres vc0 / vc1, widths h0 / h1); p runs over the physical
 * grid in C order.  Needs the velocity ghosts (frozen values) in f.  Used by
 * the device diagnostics rows (conserved_quantities, diagnostics.py:85-122). */
int vpfv_higher_moments(const double *f, int d, int v, const int *N, const double *vc0,
                        const double *vc1, double h0, double h1, double *out, void *stream);

/* Richardson error of a refinement (richardson_error, diagnostics.py:163-180)
 * on padded device arrays: coarse interior N[0..D-1], fine interior 2N; each
 * of nblocks CTAs writes the sum of |coarse - mean of its 2^D fine children|
 * over its share of the coarse cells to partials[block]; the error is the
 * in-order sum of the partials divided by prod(N).  Feeds the convergence
 * ladders of paper_2410_12155_b200.convergence (cli.py:144-181). */
int vpfv_richardson_partials(const double *coarse, const double *fine, int D, const int *N,
                             double *partials, int nblocks, void *stream);

/* rho = sum_s q[s] * n[s*nphys + p], then rho -= mean(rho)
 * (fields.py:164-169; the mean is a fixed-order tree sum / nphys). */
int vpfv_charge_density(const double *n, const double *q_host, int nspecies, int nphys,
                        double *rho, void *stream);

/* x[i] = x[i] * a, i < n (one rounding, __dmul_rn): the velocity volume
 * applied to fold-tree sums gathered across velocity partitions, so that
 * n = fold * vol exactly as the single-box moment (fields.py:99-111). */
int vpfv_scale(double *x, double a, long long n, void *stream);

/* The whole 1D field chain of a stage in one CTA: when partials != NULL,
 * n[s] = vols[s] * fold(partials[s]) (as vpfv_moment_partials, partials[s]
 * [Nx][rows[s]][chunks[s]], chunks <= 16), else n is given; then
 * rho = sum_s q_s n_s - mean (n: [nspecies][Nx]), the spectral solve for Ex (as vpfv_poisson_1d), then
 * each species' line tables from Ex -- plain e[s]/c1[s] (vpfv_tables_1d) or
 * packed[s] rows (vpfv_tables_1d_packed) when packed[s] != NULL, with c1 = 0
 * when corrections[s] == 0.  Bitwise the separate charge / Poisson / tables
 * calls (shared block-level code); replaces three launches per stage of
 * Simulation._stage (runner.py:183-191) for d = 1.  Nx <= vpfv_field_1d_max_cells(). */
int vpfv_field_1d_max_cells(void);

/* The same chain over ~148 CTAs: Ex = K (*) rho with green2 = the spectral
 * solve's (fields.py:172-213) Green's function K = IFFT(-i kd / k^2) stored
 * twice (2 Nx doubles), each
 * CTA rebuilding rho and computing E and the tables on its own cells.
 * partials (1D-1V: one row of chunks[s] <= 16 per cell) or n given.  Agrees
 * with the FFT path to O(eps sqrt(Nx)); Nx <= 16384. */
int vpfv_field_1d_conv(const double *const *partials, const int *chunks, const double *vols, double *n,
                       const double *q_host, int nspecies, int Nx, double *rho, double *Ex,
                       const double *green2, double *const *e, double *const *c1, double *const *packed,
                       const double *qmk2, const double *g, const double *t1, const double *den1,
                       const int *corrections, void *stream);
int vpfv_field_1d(const double *const *partials, const int *rows, const int *chunks, const double *vols,
                  double *n, const double *q_host, int nspecies, int Nx, double *rho, double *Ex,
                  const double *tw, const double *k2, const double *kd, double *const *e,
                  double *const *c1, double *const *packed, const double *qmk2, const double *g,
                  const double *t1, const double *den1, const int *corrections, void *stream);

/* ---------------------------------------------------------------------- */
/* Spectral Poisson solve (fields.py:172-213), hand-written fp64 FFT.
 * Host-precomputed tables (numpy, bitwise the reference's k arrays):
 *   tw*  : exp(-2 pi i m / N) for m < N, interleaved (re, im)
 *   k2   : |k|^2 per mode (1D: N; 2D: kx/ky passed separately)
 *   kd   : derivative wavenumber with the even-N Nyquist entry zeroed
 * scratch: >= 4*Nx*Ny complex values (2D), unused in 1D.  phi may be NULL. */
int vpfv_poisson_1d(const double *rho, double *Ex, double *phi, int N,
                    const double *tw, const double *k2, const double *kd, void *stream);
int vpfv_poisson_2d(const double *rho, double *Ex, double *Ey, double *phi, int Nx, int Ny,
                    const double *twx, const double *twy, const double *kx, const double *ky,
                    const double *kxd, const double *kyd, double *scratch, void *stream);

/* ---------------------------------------------------------------------- */
/* Per-stage line tables from E, in the reference dispatcher's arithmetic
 * (_kernels.py:330-365, fvm.py:168-201):
 *   e[i]  = qmk2*E[i] + g                          (avx / evx)
 *   c1[i] = t1 + (qmk2*(E[i+1]-E[i-1])) / den1      (periodic differences)
 * 2D adds evy, c3, c4, c5 with nqmk2 = (-qm)*kappa2. */
int vpfv_tables_1d(const double *Ex, double *e, double *c1, int Nx,
                   double qmk2, double g, double t1, double den1, void *stream);
int vpfv_tables_2d(const double *Ex, const double *Ey, double *evx, double *evy,
                   double *c1, double *c3, double *c4, double *c5, int Nx, int Ny,
                   double qmk2, double nqmk2, double gx, double gy,
                   double t1, double t4, double denx, double deny, void *stream);

/* 1D tables packed for the tiled 1D-2V kernel: packed[(Nx+2)][8] =
 * (evx, c1, 0, ...) with periodic ghost rows 0 (= x Nx-1) and Nx+1 (= x 0). */
int vpfv_tables_1d_packed(const double *Ex, double *packed, int Nx, double qmk2, double g,
                          double t1, double den1, void *stream);

/* The same 2D tables packed for the tiled kernel: packed[(Nx+2)][Ny][8] =
 * (evx, evy, c3, c4, c1, c5, 0, 0) with x rows shifted by one and periodic
 * ghost rows 0 (= x Nx-1) and Nx+1 (= x 0). */
int vpfv_tables_2d_packed(const double *Ex, const double *Ey, double *packed, int Nx, int Ny,
                          double qmk2, double nqmk2, double gx, double gy,
                          double t1, double t4, double denx, double deny, void *stream);

/* ---------------------------------------------------------------------- */
/* Ghost fill of the periodic dims named in dims_mask (bit k = dim k), whole
 * columns, ascending dims -- the periodic half of fill_local_ghosts
 * (grid.py:263-277).  Frozen velocity slabs are written once at set-up. */
int vpfv_wrap_fill(double *f, int ndim, const int *N, unsigned dims_mask, void *stream);

/* ---------------------------------------------------------------------- */
/* Strided box copy between padded arrays (halo pack/unpack, scatter/gather):
 * copies the box `ext` (D extents) from src at origin so[] (strides ss[])
 * to dst at origin do[] (strides ds[]).  Strides/origins in elements. */
int vpfv_box_copy(double *dst, const long long *ds, const int *dorig,
                  const double *src, const long long *ss, const int *sorig,
                  int ndim, const int *ext, void *stream);

/* ---------------------------------------------------------------------- */
/* The tiled stage kernels' fused-moment partials computed from f itself:
 * part[row][c] = the first four fold-tree levels (fields.py:28-47) over the
 * aligned 16-wide vy chunk c of every interior velocity row of the padded
 * array f (ndim 2..4, N interior extents, N[ndim-1] % 16 == 0). */
int vpfv_moment_chunk_partials(const double *f, double *part, int ndim, const int *N, void *stream);

/* ---------------------------------------------------------------------- */
/* Separable initial condition on the padded box (nphys padded physical
 * cells x nv1 x nv2 padded velocity cells, velocity fastest):
 * out = sum_{t < nterms} (P_t[p] * V1_t[k]) * V2_t[l], each product and the
 * sum rounded once in that order -- numpy's broadcast of the reference
 * set-ups (problems.py:210-507), so bitwise the host builder.  nv2 == 1:
 * one velocity dim, V2 unused.  Replaces the host product + upload of
 * make_problem for production-size grids. */
int vpfv_init_separable(double *out, long long nphys, int nv1, int nv2,
                        const double *P0, const double *V10, const double *V20,
                        const double *P1, const double *V11, const double *V21,
                        int nterms, void *stream);

/* ---------------------------------------------------------------------- */
/* NCCL mode of the x-slab layer for non-torch hosts (csrc/comm.cu), the
 * reference cluster's exchange (Exchanger, partition.py:679-724) and field
 * gather (runner.py:336-392) over an NCCL communicator (opaque pointer).
 * vpfv_comm_unique_id fills vpfv_comm_id_size() bytes on one rank; every
 * rank passes them to vpfv_comm_init.  vpfv_halo_exchange_x: the 3 first /
 * last interior x planes of the padded array f (extents N) to the x
 * neighbours' high / low ghost planes, ranks forming a periodic ring.
 * vpfv_density_allgather: count doubles per rank into n (rank order).
 * vpfv_flag_allreduce: in-place max of one int64 (the divergence verdict).
 * Stream-ordered, graph-capturable; VPFV_ENCCL on NCCL errors. */
int vpfv_comm_id_size(void);
int vpfv_comm_unique_id(unsigned char *id_out);
int vpfv_comm_init(void **comm_out, int world, int rank, const unsigned char *id, int device);
int vpfv_comm_destroy(void *comm);
int vpfv_halo_exchange_x(void *comm, double *f, int ndim, const int *N, void *stream);
int vpfv_density_allgather(void *comm, const double *n_local, double *n, long long count, void *stream);
int vpfv_flag_allreduce(void *comm, long long *flag, void *stream);

/* ---------------------------------------------------------------------- */
int vpfv_version(void);
/* 0 if device `dev` is an sm_100 part this library was built for. */
int vpfv_check_device(int dev);
const char *vpfv_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* VPFV_H */
