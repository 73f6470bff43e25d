/*
 * vpb200 — C ABI of the B200-native SLDG / cubic-spline Vlasov hot path.
 *
 * Every pointer argument is a DEVICE pointer (CUDA global memory) unless the
 * comment says otherwise; `stream` is a cudaStream_t passed as void*.  Entry
 * points return VPB_OK (0) or a nonzero status; vpb_last_error() gives the
 * message of the calling thread's most recent failure.  No C++ exceptions
 * cross this boundary and the library keeps no ownership of caller buffers
 * (it caches only small per-size constant tables: the spline factors).
 *
 * Field layout for the *_axis entry points ("canonical"): f[v2][v1][x2][x1],
 * row-major, x1 fastest; each axis holds cells*(order) dofs with the dG
 * nodes innermost (reference: pkg/src/slvp/field.py:67-76, 246-251).
 * dims[4] = dofs per axis in GRID order (x1, x2, v1, v2).  A 1x1v grid is
 * dims = {nx, 1, nv, 1}.
 *
 * Reference interfaces replaced (all paths under /root/reference/pkg/src/slvp):
 *   vpb_dg_sweep_contig      <- kernels.dg_sweep_contig      kernels.py:63-66, _kernels.pyx:202-225
 *   vpb_dg_sweep_strided     <- kernels.dg_sweep_strided     kernels.py:69-72, _kernels.pyx:228-279
 *   vpb_spline_sweep_contig  <- kernels.spline_sweep_contig  kernels.py:55-56, _kernels.pyx:126-149
 *   vpb_spline_sweep_strided <- kernels.spline_sweep_strided kernels.py:59-60, _kernels.pyx:152-199
 *   vpb_dg_tables            <- dg.projection_pairs          dg.py:99-152
 *   vpb_dg_sweep_axis        <- field._sweep + DGAdvection   field.py:166-202, dg.py:178-209
 *   vpb_spline_sweep_axis    <- field._sweep + SplineAdvection field.py:166-202, spline.py:91-110
 *   vpb_density              <- poisson.compute_density      poisson.py:85-95
 *   vpb_field_solve          <- poisson.solve_poisson        poisson.py:123-196
 *   vpb_diagnostics          <- driver.diagnostics + poisson.electric_energy
 *                                                           driver.py:279-316, poisson.py:199-217
 *   vpb_electric_energy      <- poisson.electric_energy      poisson.py:199-217
 *   vpb_fill_separable       <- driver.initialize (broadcast product) driver.py:182-198
 *   vpb_halo_*               <- (new) x-axis halo pack/unpack for sharded fields
 * The reference's `threads` / `block` arguments are CPU scheduling knobs and
 * have no GPU meaning; they are dropped.
 */
#ifndef VPB200_H
#define VPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VPB_OK = 0,
  VPB_ERR_INVALID = 1,     /* bad argument (same cases the reference rejects with ValueError) */
  VPB_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
  VPB_ERR_UNSUPPORTED = 3  /* valid but not implemented (e.g. order > 9) */
};

const char* vpb_version(void);
const char* vpb_strerror(int code);
const char* vpb_last_error(void);
/* Kernels launched by this library since load (process-wide, all threads).
 * Instrumentation for bench.py's gpu_launches; no reference counterpart. */
unsigned long long vpb_launch_count(void);

/* ------------------------------------------------------------------------
 * Reference plugin API: the four line-kernel entry points.
 * ---------------------------------------------------------------------- */

/* lines/out: [nlines][n] C-contiguous, n = ncells*nloc.  idx[r] selects the
 * table row (a,b: [ntable][nloc][nloc], q, alpha: [ntable]).  out is a
 * separate buffer (the reference returns a new array). */
int vpb_dg_sweep_contig(const double* lines, double* out, int64_t nlines, int64_t n,
                        const int64_t* idx, const double* a, const double* b,
                        const int64_t* q, const double* alpha, int64_t ntable,
                        int32_t ncells, int32_t nloc, void* stream);

/* view: 4-D strided array (element strides), last axis = the line; lines are
 * enumerated in C order over shape[0..2].  Updated IN PLACE. */
int vpb_dg_sweep_strided(double* view, const int64_t shape[4], const int64_t strides[4],
                         const int64_t* idx, const double* a, const double* b,
                         const int64_t* q, const double* alpha, int64_t ntable,
                         int32_t ncells, int32_t nloc, void* stream);

/* Cubic-spline advection: out_i = spline(line)(x_i - table[idx[r]]). */
int vpb_spline_sweep_contig(const double* lines, double* out, int64_t nlines, int64_t n,
                            const int64_t* idx, const double* table, int64_t ntable,
                            double h, void* stream);
int vpb_spline_sweep_strided(double* view, const int64_t shape[4], const int64_t strides[4],
                             const int64_t* idx, const double* table, int64_t ntable,
                             double h, void* stream);

/* ------------------------------------------------------------------------
 * Device-resident hot path (canonical layout).
 * ---------------------------------------------------------------------- */

/* projection_pairs: shift[t] = values[t]*scale; s = shift/h; q = floor(s);
 * alpha = s - q (carry alpha>=1 -> q+1, alpha=0); a,b = [ntable][order][order]. */
int vpb_dg_tables(const double* values, int64_t ntable, double scale, double h, int32_t order,
                  double* a, double* b, int64_t* q, double* alpha, void* stream);

/* One dG sweep along `axis` (0=x1, 1=x2, 2=v1, 3=v2) from src to dst
 * (distinct buffers).  Table row per line: x1 -> iv1, x2 -> iv2,
 * v1/v2 -> ix2*dims[0]+ix1 (the device E layout).  *flag |= 1 if any output
 * is non-finite (flag may be NULL). */
int vpb_dg_sweep_axis(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                      int32_t order, const double* a, const double* b, const int64_t* q,
                      const double* alpha, int32_t* flag, void* stream);

/* Both space sweeps of a Strang half step, x1 then x2, in ONE pass over f
 * (driver.py:220-228 _advect_space): per (iv2, iv1) plane the x1 tables use
 * row iv1 and the x2 tables row iv2.  Bitwise equal to vpb_dg_sweep_axis(0)
 * followed by vpb_dg_sweep_axis(1); half the HBM traffic.  flag1/flag2 get
 * the non-finite reports of the x1 and x2 results.  Needs a 2x2v field with
 * dims[0]*order even. */
int vpb_dg_sweep_xplane(const double* src, double* dst, const int64_t dims[4], int32_t order,
                        const double* a1, const double* b1, const int64_t* q1,
                        const double* alpha1, const double* a2, const double* b2,
                        const int64_t* q2, const double* alpha2, int32_t* flag1,
                        int32_t* flag2, void* stream);

/* Both velocity sweeps of a Strang step, v1 then v2, in ONE pass over f
 * (driver.py:231-242 _advect_velocity): the tables of both are indexed by the
 * x position ix2*dims[0]+ix1.  Bitwise equal to vpb_dg_sweep_axis(2) then
 * vpb_dg_sweep_axis(3); half the HBM traffic. */
int vpb_dg_sweep_vplane(const double* src, double* dst, const int64_t dims[4], int32_t order,
                        const double* a1, const double* b1, const int64_t* q1,
                        const double* alpha1, const double* a2, const double* b2,
                        const int64_t* q2, const double* alpha2, int32_t* flag1,
                        int32_t* flag2, void* stream);

/* vpb_dg_sweep_xplane plus the density of its OUTPUT, collapsed to cell
 * centres (poisson.py:85-95 then :129-139): rc_out[c2][c1] (C2 x C1) and
 * stats[0] = weighted density mean / volume (poisson.py:143-160).  Each CTA
 * accumulates its own planes into `work` (vpb_dg_xplane_density_work_len
 * doubles); a fixed-order pass sums the CTA partials.  Feed rc_out to
 * vpb_field_solve with a geometry whose r1, r2 = C1, C2 and g = DFT.
 * wv1, wv2: DEVICE velocity weights.  mid_host: HOST, the `order` Lagrange
 * weights at the cell centre; wcell1_host / wcell2_host: HOST, the `order`
 * space quadrature weights of one x1 / x2 cell (uniform grid). */
int64_t vpb_dg_xplane_density_work_len(const int64_t dims[4], int32_t order);
int vpb_dg_sweep_xplane_density(const double* src, double* dst, const int64_t dims[4],
                                int32_t order, const double* a1, const double* b1,
                                const int64_t* q1, const double* alpha1, const double* a2,
                                const double* b2, const int64_t* q2, const double* alpha2,
                                int32_t* flag1, int32_t* flag2, const double* wv1,
                                const double* wv2, const double* mid_host,
                                const double* wcell1_host, const double* wcell2_host,
                                double volume, double* work, double* rc_out, double* stats,
                                void* stream);

/* vpb_dg_sweep_xplane_density plus the diagnostics moments of the OUTPUT
 * (driver.py:279-316: mass, l1, l2^2, kinetic -> diag_out[0..3]); v1sq /
 * v2sq: DEVICE squared velocity nodes.  With the field solve of rc_out and
 * vpb_electric_energy this is a whole DiagnosticsRecord of the post-step
 * state without re-reading f.  Same work buffer as the density variant. */
int vpb_dg_sweep_xplane_moments(const double* src, double* dst, const int64_t dims[4],
                                int32_t order, const double* a1, const double* b1,
                                const int64_t* q1, const double* alpha1, const double* a2,
                                const double* b2, const int64_t* q2, const double* alpha2,
                                int32_t* flag1, int32_t* flag2, const double* wv1,
                                const double* wv2, const double* mid_host,
                                const double* wcell1_host, const double* wcell2_host,
                                const double* v1sq, const double* v2sq, double volume,
                                double* work, double* rc_out, double* stats, double* diag_out,
                                void* stream);

/* Two consecutive x half steps in one HBM pass: the closing x1(τ/2) x2(τ/2)
 * of a Strang step followed by the opening x1(τ/2) x2(τ/2) of the next one
 * (driver.py:245-265 applied twice; run loop driver.py:371-377), with the
 * same tables for both.  Bitwise equal to four separate sweeps.  flag1a /
 * flag2a: x1 / x2 of the first half step, flag1b / flag2b: of the second. */
int vpb_dg_sweep_xplane2(const double* src, double* dst, const int64_t dims[4], int32_t order,
                         const double* a1, const double* b1, const int64_t* q1,
                         const double* alpha1, const double* a2, const double* b2,
                         const int64_t* q2, const double* alpha2, int32_t* flag1a,
                         int32_t* flag2a, int32_t* flag1b, int32_t* flag2b, void* stream);

/* vpb_dg_sweep_xplane2 with the density epilogue of
 * vpb_dg_sweep_xplane_density on its output (the density the next step's
 * field solve needs). */
int64_t vpb_dg_xplane2_density_work_len(const int64_t dims[4], int32_t order);
int vpb_dg_sweep_xplane2_density(const double* src, double* dst, const int64_t dims[4],
                                 int32_t order, const double* a1, const double* b1,
                                 const int64_t* q1, const double* alpha1, const double* a2,
                                 const double* b2, const int64_t* q2, const double* alpha2,
                                 int32_t* flag1a, int32_t* flag2a, int32_t* flag1b,
                                 int32_t* flag2b, const double* wv1, const double* wv2,
                                 const double* mid_host, const double* wcell1_host,
                                 const double* wcell2_host, double volume, double* work,
                                 double* rc_out, double* stats, void* stream);

/* Composed tables for two same-table sweeps along one axis: out[t] =
 * {A A, A B + B A, B B} (row-major p x p each, fused multiply-adds), i.e.
 * _kernels.pyx:113-123 applied twice as one three-cell stencil
 * out[c] = AA u[c-2q-2] + (AB+BA) u[c-2q-1] + BB u[c-2q].  a, b: DEVICE
 * [n][p][p] from vpb_dg_tables; out: DEVICE [n][3][p][p]. */
int vpb_dg_compose_tables(const double* a, const double* b, int64_t n, int32_t order,
                          double* out, void* stream);

/* The merged x half steps of vpb_dg_sweep_xplane2 (closing x1 x2 of a Strang
 * step + opening x1 x2 of the next, driver.py:245-265 / 371-377) with
 * composed stencils: x1 x2 x1 x2 = (x1 x1)(x2 x2) applied as one three-cell
 * stencil per axis (k1 / k2 from vpb_dg_compose_tables; q / alpha from
 * vpb_dg_tables: alpha == 0 rows stay exact copies from cell c-2q).  Equal
 * to vpb_dg_sweep_xplane2 up to round-off ("fast" arithmetic mode).  flag:
 * any non-finite output (or NULL). */
int vpb_dg_sweep_xcomp(const double* src, double* dst, const int64_t dims[4], int32_t order,
                       const double* k1, const int64_t* q1, const double* alpha1,
                       const double* k2, const int64_t* q2, const double* alpha2, int32_t* flag,
                       void* stream);

/* vpb_dg_sweep_xcomp with the density epilogue of vpb_dg_sweep_xplane_density
 * on its output (work: vpb_dg_xcomp_density_work_len doubles). */
int64_t vpb_dg_xcomp_density_work_len(const int64_t dims[4], int32_t order);
int vpb_dg_sweep_xcomp_density(const double* src, double* dst, const int64_t dims[4],
                               int32_t order, const double* k1, const int64_t* q1,
                               const double* alpha1, const double* k2, const int64_t* q2,
                               const double* alpha2, int32_t* flag, const double* wv1,
                               const double* wv2, const double* mid_host,
                               const double* wcell1_host, const double* wcell2_host,
                               double volume, double* work, double* rc_out, double* stats,
                               void* stream);

/* {0, A, B} per table row: one x sweep as the three-cell stencil of
 * vpb_dg_sweep_xstencil with qmul = 1 (out: DEVICE [n][3][p][p]). */
int vpb_dg_single_tables(const double* a, const double* b, int64_t n, int32_t order, double* out,
                         void* stream);

/* Three-cell x-plane stencil pass on an x1-SHARDED field (one rank's box
 * [v2][v1][x2][x1 local]; x2 whole): output cell c of every x row reads x1
 * cells c-Q-2 .. c-Q with Q = qmul*q, then the same along x2.  qmul = 2 with
 * vpb_dg_compose_tables tables = the merged closing + opening x half steps
 * (vpb_dg_sweep_xcomp); qmul = 1 with vpb_dg_single_tables = one x half step
 * (_advect_space, driver.py:220-228).  x1 cells -wl..-1 and C1..C1+wr-1 come
 * from hl / hr in the vpb_halo_pack layout [plane][x2 row][w*p] (16-byte
 * aligned; p*p*w even, i.e. even widths for odd p), staged into shared
 * memory with the rows; the row is not periodic.  The _density variant adds the epilogue of
 * vpb_dg_sweep_xplane_density for the shard's cells (rc_out: the shard's
 * [C2][C1 local] cell-centre slab; stats[0]: its share of the mean / volume). */
int vpb_dg_sweep_xstencil(const double* src, double* dst, const int64_t dims[4], int32_t order,
                          const double* k1, const int64_t* q1, const double* alpha1,
                          const double* k2, const int64_t* q2, const double* alpha2, int32_t qmul,
                          const double* hl, int32_t wl, const double* hr, int32_t wr,
                          int32_t* flag, void* stream);
int64_t vpb_dg_xstencil_density_work_len(const int64_t dims[4], int32_t order, int32_t wl,
                                         int32_t wr);
int vpb_dg_sweep_xstencil_density(const double* src, double* dst, const int64_t dims[4],
                                  int32_t order, const double* k1, const int64_t* q1,
                                  const double* alpha1, const double* k2, const int64_t* q2,
                                  const double* alpha2, int32_t qmul, const double* hl, int32_t wl,
                                  const double* hr, int32_t wr, int32_t* flag, const double* wv1,
                                  const double* wv2, const double* mid_host,
                                  const double* wcell1_host, const double* wcell2_host,
                                  double volume, double* work, double* rc_out, double* stats,
                                  void* stream);
/* The halo stencil pass (with or without the density epilogue: wv1 may be
 * NULL) on v2 rows [v2_0, v2_0 + v2_rows) of the shard, so the sharded step
 * can overlap the x1 halo exchange of the next block of rows with this
 * block (dist.ShardedSolver.advance).  phase bit 1: first
 * block of the pass (zero `work`), bit 2: last (reduce to rc_out / stats). */
int vpb_dg_sweep_xstencil_rows(const double* src, double* dst, const int64_t dims[4],
                               int32_t order, int64_t v2_0, int64_t v2_rows, const double* k1,
                               const int64_t* q1, const double* alpha1, const double* k2,
                               const int64_t* q2, const double* alpha2, int32_t qmul,
                               const double* hl, int32_t wl, const double* hr, int32_t wr,
                               int32_t* flag, const double* wv1, const double* wv2,
                               const double* mid_host, const double* wcell1_host,
                               const double* wcell2_host, double volume, double* work,
                               double* rc_out, double* stats, int32_t phase, void* stream);

/* The merged x pass with the density epilogue (vpb_dg_sweep_xcomp_density)
 * on v2 rows [v2_0, v2_0 + v2_rows) of a field not sharded in x (a velocity
 * shard); tables indexed by the field's v2 row.  The work buffer
 * (vpb_dg_xcomp_density_work_len of `dims`) accumulates over the calls of
 * one pass: phase bit 1 (first call) zeroes it, bit 2 (last) reduces it to
 * rc_out / stats. */
int vpb_dg_sweep_xcomp_rows(const double* src, double* dst, const int64_t dims[4], int32_t order,
                            int64_t v2_0, int64_t v2_rows, const double* k1, const int64_t* q1,
                            const double* alpha1, const double* k2, const int64_t* q2,
                            const double* alpha2, int32_t* flag, const double* wv1,
                            const double* wv2, const double* mid_host,
                            const double* wcell1_host, const double* wcell2_host, double volume,
                            double* work, double* rc_out, double* stats, int32_t phase,
                            void* stream);

/* The stencil pass on an x1 x x2 sharded field (the 4 x 2 process grid of
 * dist.ShardedSolver): x1 halos hl / hr as for vpb_dg_sweep_xstencil, and the
 * plane is not periodic in x2 either -- source x2 cells -wl2..-1 and
 * C2..C2+wr2-1 come from x2l / x2r, three parts each in the shard's own
 * layouts: [0] the x1 dofs [plane][w2 cells][P rows][n1] (vpb_halo_pack axis
 * 1 of the neighbour), [1] / [2] the left / right x1 halo cells of those rows
 * [plane][w2 cells][P rows][wl*P] / [wr*P] (the corners, taken from the
 * neighbour's x1 halo buffers).  wv1 == NULL: no density epilogue; else as
 * vpb_dg_sweep_xstencil_density (work: vpb_dg_xstencil_density_work_len). */
int vpb_dg_sweep_xstencil2(const double* src, double* dst, const int64_t dims[4], int32_t order,
                           const double* k1, const int64_t* q1, const double* alpha1,
                           const double* k2, const int64_t* q2, const double* alpha2,
                           int32_t qmul, const double* hl, int32_t wl, const double* hr,
                           int32_t wr, int32_t wl2, const double* const x2l[3], int32_t wr2,
                           const double* const x2r[3], int32_t* flag, const double* wv1,
                           const double* wv2, const double* mid_host,
                           const double* wcell1_host, const double* wcell2_host, double volume,
                           double* work, double* rc_out, double* stats, void* stream);

/* Fused v1 v2 pass of one v2 shard of a velocity-sharded field
 * (dist.VShardedSolver): `src` holds src_v2_cells v2 cells -- the shard's
 * dims[3]/order cells starting at cell v2_offset, neighbour halo cells
 * before and after (contiguous rows: v2 is the outermost axis) -- and `dst`
 * the shard's cells.  Replaces _advect_velocity (driver.py:231-242) on the
 * shard; halo_flag is raised if a shift needs a cell beyond the halos. */
int vpb_dg_sweep_vplane_v2halo(const double* src, double* dst, const int64_t dims[4],
                               int32_t order, int32_t src_v2_cells, int32_t v2_offset,
                               const double* a1, const double* b1, const int64_t* q1,
                               const double* alpha1, const double* a2, const double* b2,
                               const int64_t* q2, const double* alpha2, int32_t* flag1,
                               int32_t* flag2, int32_t* halo_flag, void* stream);

/* The same pass with the halo regions read in place from the neighbouring
 * shards' own buffers (peer memory over NVLink, CUDA IPC-mapped; the halo
 * exchange fused into the pass): left halo = cells [l_cell0, l_cell0 + H)
 * of src_l, own cells from cell c_cell0 of src, right halo = cells
 * [r_cell0, r_cell0 + H) of src_r (each buffer src_*_cells v2 cells). */
int vpb_dg_sweep_vplane_v2peer(const double* src_l, int32_t src_l_cells, int32_t l_cell0,
                               const double* src, int32_t src_cells, int32_t c_cell0,
                               const double* src_r, int32_t src_r_cells, int32_t r_cell0,
                               int32_t halo_cells, double* dst, const int64_t dims[4],
                               int32_t order, const double* a1, const double* b1,
                               const int64_t* q1, const double* alpha1, const double* a2,
                               const double* b2, const int64_t* q2, const double* alpha2,
                               int32_t* flag1, int32_t* flag2, int32_t* halo_flag, void* stream);

/* One spline sweep along `axis`; shift of line = values[table row]*scale. */
int vpb_spline_sweep_axis(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                          const double* values, double scale, double h, int32_t* flag,
                          void* stream);

/* Two consecutive spline sweeps along `axis` with the same shifts in one
 * pass (the closing and opening x half steps of consecutive Strang steps,
 * driver.py:245-265 / 371-377): E^2 (6 T^-1)^2 u -- the circulant solve and
 * evaluation of _kernels.pyx:37-93 commute, so the recursive-filter solve
 * runs twice and the evaluation is the 7-tap self-convolution of the weights
 * at offset 2 j0.  Equal to two vpb_spline_sweep_axis calls up to round-off.
 * Needs n % 16 == 0, n >= 32; VPB_ERR_UNSUPPORTED otherwise. */
int vpb_spline_sweep_axis2(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                           const double* values, double scale, double h, int32_t* flag,
                           void* stream);

/* The x1 (contiguous axis) double sweep of vpb_spline_sweep_axis2 with the
 * density of its output as an epilogue (compute_density, poisson.py:85-95,
 * fused into the merged x half steps; the x2 double sweep runs first, the
 * two commute): part[((iv2*(nv1/32) + b)*n2 + ix2)*n1 + ix1] = sum over the
 * 32 v1 rows of block b of out * wv1[iv1], in row order.  vpb_density over
 * dims {n1, n2, nv1/32, nv2} with unit v1 weights and wv2 reduces part to rho.
 * Needs nv1 % 32 == 0, n1 % 8 == 0, n1 >= 64, 16-byte aligned buffers;
 * vpb_spline_density_part_len(dims) doubles of part (0: unsupported). */
int64_t vpb_spline_density_part_len(const int64_t dims[4]);
int vpb_spline_sweep_x1dbl_density(const double* src, double* dst, const int64_t dims[4],
                                   const double* values, double scale, double h, int32_t* flag,
                                   const double* wv1, double* part, void* stream);

/* rho[ix2*n1+ix1] = sum_v f * wv1[iv1] * wv2[iv2].  work: vpb_density_work_len doubles. */
int64_t vpb_density_work_len(const int64_t dims[4]);
int vpb_density(const double* f, const int64_t dims[4], const double* wv1, const double* wv2,
                double* rho, double* work, void* stream);

/* Spectral field solve on small dense transforms (all complex arrays are
 * interleaved re,im, row-major):
 *   rhohat = G1 * R * G2^T        (R[i1][i2] = rho[i2*n1+i1])
 *   E_d    = Re(M1 * (K_d .* rhohat) * M2^T),  d = 0, 1
 * E is written as e[d*n1*n2 + i2*n1 + i1].  stats[0] = weighted density mean
 * (neutrality check, poisson.py:143-160).  *flag |= 1 if E is non-finite. */
typedef struct {
  int64_t n1, n2;       /* dofs along x1, x2 (n2 = 1 for 1x1v) */
  int64_t c1, c2;       /* Fourier sizes (cells for dG, points for spline) */
  int32_t ncomp;        /* field components: 2 for 2x2v, 1 for 1x1v */
  const double* g1;     /* complex [c1][n1] */
  const double* g2;     /* complex [c2][n2] */
  const double* m1;     /* complex [n1][c1] */
  const double* m2;     /* complex [n2][c2] */
  const double* kmul;   /* complex [ncomp][c1][c2] */
  const double* wx1;    /* [n1] quadrature weights */
  const double* wx2;    /* [n2] */
  double volume;        /* spatial measure */
  int64_t r1, r2;       /* input density grid (0: the nodal n1, n2; c1, c2 when the
                           input is already collapsed to cell centres and g = DFT) */
} vpb_field_geom;

int64_t vpb_field_work_len(const vpb_field_geom* geom);
int vpb_field_solve(const double* rho, const vpb_field_geom* geom, double* e, double* stats,
                    double* work, int32_t* flag, void* stream);

/* Diagnostics (driver.py:279-316): out[0..4] = mass, l1, l2^2, kinetic, EE.
 * wx = [n1*n2] product weights wx1[ix1]*wx2[ix2] in device layout; e may be
 * NULL (EE = 0).  work: vpb_diag_work_len doubles. */
int64_t vpb_diag_work_len(const int64_t dims[4]);
int vpb_diagnostics(const double* f, const int64_t dims[4], const double* wx,
                    const double* wv1, const double* wv2, const double* v1sq,
                    const double* v2sq, const double* e, int32_t ncomp, double* out,
                    double* work, void* stream);

/* out[0] = 0.5 * sum_d sum_x e[d*nx + x]^2 * wx[x]  (poisson.py:199-217). */
int vpb_electric_energy(const double* e, int32_t ncomp, int64_t nx, const double* wx,
                        double* out, void* stream);

/* f[iv2][iv1][x] = (g2[iv2]*g1[iv1]) * space[x]  (x = ix2*n1+ix1). */
int vpb_fill_separable(double* f, const int64_t dims[4], const double* g1, const double* g2,
                       const double* space, void* stream);

/* ------------------------------------------------------------------------
 * Sharded fields (multi-GPU layer): the local shard holds cells [c0, c0+cl)
 * of the sharded x axis; halos are cell slabs of the full line geometry.
 * ---------------------------------------------------------------------- */

/* Pack `width` cells of every line along `axis` (0 or 1) starting at local
 * cell `cell0` into a contiguous buffer [lines][width*order] (lines in C
 * order over the transverse axes). */
int vpb_halo_pack(int32_t axis, const double* f, const int64_t dims[4], int32_t order,
                  int64_t cell0, int64_t width, double* buf, void* stream);

/* Strided slab copy (the all-to-all reshard of the multi-GPU spline step):
 * `outer` runs of `run` doubles; run k is read at src + k*src_stride and
 * written at dst + k*dst_stride. */
int vpb_slab_copy(const double* src, int64_t src_stride, double* dst, int64_t dst_stride,
                  int64_t outer, int64_t run, void* stream);

/* dG sweep of a shard along a sharded x axis (axis 0 or 1).  Source cells
 * outside the local range [0, cl) are read from the halo buffers (no
 * periodic wrap inside the shard): `left` holds the wl cells just below the
 * shard, `right` the wr cells just above it, both in the halo layout of
 * vpb_halo_pack.  Requires wl >= max(q+1, 0) and wr >= max(-q, 0) over the
 * table rows used. */
int vpb_dg_sweep_axis_halo(int32_t axis, const double* src, double* dst, const int64_t dims[4],
                           int32_t order, const double* left, int64_t wl, const double* right,
                           int64_t wr, const double* a, const double* b, const int64_t* q,
                           const double* alpha, int32_t* flag, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VPB200_H */
