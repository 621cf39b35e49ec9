/*
 * rubs_b200.h -- C ABI of the B200-native space-variant box-spline filter.
 *
 * The reference (arxiv/paper_1003_2022, package "rubs") is pure Python; its
 * drop-in boundary is the public Python API (pkg/src/rubs/__init__.py:46-53).
 * Each entry point below replaces one reference function; the reference
 * file:line it replaces is given with it.  The Python host layer
 * (paper_1003_2022_b200/) binds these with ctypes and keeps the reference
 * signatures, argument meaning and exceptions.
 *
 * Conventions
 *   - Images are row-major; element (r, c) sits at lattice point
 *     (n1, n2) = (c, r): x = column, y = row (reference zp.py:56-66).
 *   - ld_* are row strides in ELEMENTS (not bytes).
 *   - "Device" entry points take device pointers and enqueue on `stream`
 *     (a cudaStream_t, NULL = legacy default stream); they synchronise the
 *     stream before returning so that the status is final.
 *   - "_host" entry points take host pointers (pageable or pinned), stage
 *     the copies themselves and return when the result is in `out`.
 *   - Outputs are always float64, like the reference (engine.py:285).
 *   - No torch types cross this boundary.
 *
 * Status codes (mapped by the Python layer to the reference's exceptions):
 *   RUBS_OK           0
 *   RUBS_EVALUE       1  -> ValueError      (engine.py:286-289, 210-215)
 *   RUBS_EOVERFLOW    2  -> OverflowError   (engine.py:195-200)
 *   RUBS_EOUTOFGRID   3  -> OutOfGrid       (solver.py:304-307)
 *   RUBS_ECUDA        4  -> RuntimeError    (CUDA error / OOM)
 *   RUBS_EUNSUPPORTED 5  -> RuntimeError    (configuration not handled)
 *   RUBS_EINFEASIBLE  6  -> Infeasible      (solver.py:64-82; N=3 mapping)
 */
#ifndef RUBS_B200_H
#define RUBS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RUBS_OK 0
#define RUBS_EVALUE 1
#define RUBS_EOVERFLOW 2
#define RUBS_EOUTOFGRID 3
#define RUBS_ECUDA 4
#define RUBS_EUNSUPPORTED 5
#define RUBS_EINFEASIBLE 6

#define RUBS_F32 0
#define RUBS_F64 1

/* Library version string and the last error message of this thread. */
const char *rubs_b200_version(void);
const char *rubs_b200_last_error(void);

/* Number of kernel launches issued by this thread since the last reset
 * (bench.py reports it as gpu_launches). */
int64_t rubs_b200_launch_count(void);
void rubs_b200_reset_launch_count(void);

/* Optional device timing of the library's own kernels (CUDA events on the
 * launching stream, read back at the end of each call).  kind: 0 = tile
 * filter kernel, 1 = margin pre-pass, 2 = all kernels.  Totals accumulate
 * until reset.  Used by bench.py for the roofline's per-launch duration. */
void rubs_b200_set_profiling(int enable);
void rubs_b200_kernel_time(int kind, double *total_ms, int64_t *launches);
void rubs_b200_reset_kernel_time(void);

/* Measured fp64 FMA peak of the current device: a DFMA-chain kernel on every
 * SM (8 independent chains per thread, all CTAs resident), timed with CUDA
 * events; *tflops = 2 x DFMA / s.  The roofline denominator of bench.py's
 * "fp64" object.  Returns a status code. */
int rubs_b200_dfma_peak(double *tflops, double *ms);

/*
 * 1 if a four-direction filter call on this thread since the last query met
 * pixels whose OWN minimal region exceeds the float64 precision budget
 * ("needle" kernels: three widths at the 0.05 floor next to one of tens of
 * pixels) -- their results may be accurate to ~1e-8 relative
 * instead of 1e-9.  Not an error (the reference's fast path is at ~1e-6 on
 * such inputs); reading clears it.  No reference counterpart.
 */
int rubs_b200_precision_limited(void);

/*
 * Space-variant filter, per-pixel scale field.
 * Replaces engine.filter_space_variant (pkg/src/rubs/engine.py:265-324).
 *   f        device image, H x W, dtype RUBS_F32 | RUBS_F64, row stride ld_f
 *   field    device (H, W, 4) float64 scale-vectors, row stride ld_field
 *            (in pixels, i.e. the (r, c, k) element is at
 *            field[(r * ld_field + c) * 4 + k]);
 *            or, when field_is_uniform != 0, a HOST pointer to 4 doubles
 *            (the reference's (4,) broadcast, engine.py:208-209)
 *   iterations  >= 1 (engine.py:288-289, 292-323)
 *   out      device H x W float64, row stride ld_out
 * Entries below SCALE_FLOOR = 0.05 are clamped (engine.py:58, 292);
 * non-finite entries give RUBS_EVALUE (engine.py:214-215).
 */
int rubs_b200_filter(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                     const double *field, int field_is_uniform, int64_t ld_field,
                     int iterations, double *out, int64_t ld_out, void *stream);

/* Same, host buffers (timed by bench.py as the end-to-end call). */
int rubs_b200_filter_host(const void *f, int f_dtype, int64_t H, int64_t W,
                          const double *field, int field_is_uniform, int iterations,
                          double *out);

/*
 * Device-resident scale lookup table (the reference's ScaleLut,
 * solver.py:232-247).  Built on the host by build_lut (solver.py:250-281)
 * and uploaded once.
 */
typedef struct rubs_lut rubs_lut;
int rubs_b200_lut_create(const double *rho_grid, const double *phi_grid,
                         const double *entries /* n_rho*n_phi*4 */, int n_rho, int n_phi,
                         rubs_lut **out);
void rubs_b200_lut_destroy(rubs_lut *lut);

/*
 * Vectorised LUT lookup on the device.
 * Replaces solver.lookup_many (pkg/src/rubs/solver.py:289-335).
 *   size, elong, orient   device arrays of n values, dtype p_dtype
 *   out                   device n x 4 float64
 */
int rubs_b200_lookup(const rubs_lut *lut, const void *size, const void *elong,
                     const void *orient, int p_dtype, int64_t n, double *out, void *stream);

/*
 * Fused mapping + filter: per-pixel (size, elongation, orientation) ->
 * scale-vector through the LUT (solver.py:289-335), then the space-variant
 * filter (engine.py:265-324).  Equivalent to
 *   filter_space_variant(f, lookup_many(lut, size, elong, orient), iterations)
 * without materialising the (H, W, 4) field.
 *   size/elong/orient   device H x W arrays, dtype p_dtype, row stride ld_p
 */
int rubs_b200_filter_params(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                            const void *size, const void *elong, const void *orient,
                            int p_dtype, int64_t ld_p, const rubs_lut *lut, int iterations,
                            double *out, int64_t ld_out, void *stream);

/* Same, host buffers. */
int rubs_b200_filter_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                 const void *size, const void *elong, const void *orient,
                                 int p_dtype, const rubs_lut *lut, int iterations,
                                 double *out);

/*
 * A batch of n same-shape images through the fused path, host buffers
 * (BASELINE config 4: the per-image reference call engine.py:265, repeated).
 * Image i's inputs go up while image i-1 is filtered and image i-2's result
 * comes back (two device slots, copy and compute streams overlapped), so a
 * batch runs at the larger of the PCIe and the compute time per image.
 * Errors are reported for the first failing image (its index in *failed,
 * -1 if none); pinned host buffers let the copies run asynchronously.
 *   f[i]                       host H x W image i (f_dtype)
 *   size[i]/elong[i]/orient[i] host H x W parameter planes (p_dtype)
 *   out[i]                     host H x W float64 result
 */
int rubs_b200_filter_params_batch_host(int n, const void *const *f, int f_dtype, int64_t H,
                                       int64_t W, const void *const *size,
                                       const void *const *elong, const void *const *orient,
                                       int p_dtype, const rubs_lut *lut, int iterations,
                                       double *const *out, int *failed);

/*
 * Row bands (multi-GPU sharding of one large image): one pass
 * over output rows [out_row0, out_row0 + out_rows) of an H_total x W image.
 *   f          device rows [f_row0, f_row0 + f_rows) of the image (the band
 *              plus the halo rows received from the neighbouring ranks)
 *   field / size, elong, orient
 *              device rows [*_row0, ...) of the per-pixel arrays, covering
 *              at least the output rows
 * Rows of the image outside [f_row0, f_row0 + f_rows) read as zero, so the
 * halo must cover the read margins of the output rows (the whole-image
 * result is then reproduced exactly).  iterations = 1.
 */
int rubs_b200_filter_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows, int64_t W,
                          int64_t ld_f, int64_t H_total, const double *field, int64_t field_row0,
                          int64_t ld_field, int64_t out_row0, int64_t out_rows, double *out,
                          int64_t ld_out, void *stream);
int rubs_b200_filter_params_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows,
                                 int64_t W, int64_t ld_f, int64_t H_total, const void *size,
                                 const void *elong, const void *orient, int p_dtype,
                                 int64_t p_row0, int64_t ld_p, const rubs_lut *lut,
                                 int64_t out_row0, int64_t out_rows, double *out, int64_t ld_out,
                                 void *stream);

/*
 * Read margins (left, right, below, above) of the floored, pass-scaled
 * scale-vectors over rows [row0, row0 + rows) -- the reference's
 * _read_margins (pkg/src/rubs/engine.py:247-262), exact arithmetic.  Row
 * bands use them to size the halo exchanged between ranks.  Arrays hold
 * global rows from row0 on; H_total is the full image height.
 */
int rubs_b200_read_margins(const double *field, int field_is_uniform, int64_t rows, int64_t W,
                           int64_t ld_field, int64_t H_total, int64_t row0, int iterations,
                           int *out4, void *stream);
int rubs_b200_read_margins_params(const void *size, const void *elong, const void *orient,
                                  int p_dtype, int64_t rows, int64_t W, int64_t ld_p,
                                  int64_t H_total, int64_t row0, const rubs_lut *lut,
                                  int iterations, int *out4, void *stream);

/*
 * Global pre-integration with the reference's canvas semantics.
 * Replaces engine.preintegrate (pkg/src/rubs/engine.py:145-201).
 * rubs_b200_preintegrate_shape returns the canvas geometry for the given
 * image placement and requested lattice ranges (engine.py:169-177):
 *   rows, cols   plane shape;  c_lo, r_lo  lattice of plane[0, 0]
 * rubs_b200_preintegrate then fills `plane` (device, rows x cols float64,
 * row stride ld_plane) and applies the 2^53 guard (RUBS_EOVERFLOW).
 */
int rubs_b200_preintegrate_shape(int64_t h, int64_t w, int64_t col0, int64_t row0,
                                 int64_t need_c0, int64_t need_c1, int64_t need_r0,
                                 int64_t need_r1, int64_t *rows, int64_t *cols,
                                 int64_t *c_lo, int64_t *r_lo);
int rubs_b200_preintegrate(const void *f, int f_dtype, int64_t h, int64_t w, int64_t ld_f,
                           int64_t col0, int64_t row0, int64_t need_c0, int64_t need_c1,
                           int64_t need_r0, int64_t need_r1, double *plane, int64_t ld_plane,
                           void *stream);

/*
 * Seven-tap ZP interpolation of a pre-integrated plane at n points.
 * Replaces zp.interpolate (pkg/src/rubs/zp.py:186-228); reads outside the
 * plane clamp to its edge like the reference.
 */
int rubs_b200_interpolate(const double *plane, int64_t rows, int64_t cols, int64_t ld_plane,
                          int64_t col0, int64_t row0, const double *x1, const double *x2,
                          int64_t n, double *out, void *stream);

/*
 * The reference's own caller of the hot path: structure-tensor driven
 * adaptive smoothing (pkg/src/rubs/tensor.py), on the device.
 *
 * rubs_b200_structure_tensor replaces tensor.structure_tensor
 * (tensor.py:52-75): j = (H, W, 3) float64 (J11, J12, J22), central
 * differences on the reflect-padded image, averaged with the isotropic
 * filter of width max(window_sigma sqrt(6), 0.05) (0 disables it).
 *
 * rubs_b200_anisotropy replaces tensor.anisotropy_from_tensor
 * (tensor.py:90-171): size / elong / orient float64 (H, W), isotropic
 * (H, W) bytes (may be NULL); size_range = {min, max} or NULL for the
 * default (0.5, 3 noise_sigma^2 + 0.5).  RUBS_EVALUE for a bad
 * bound_fraction or size_range, as the reference raises ValueError.
 *
 * rubs_b200_adaptive_smooth replaces tensor.adaptive_smooth
 * (tensor.py:174-224): the above, the LUT mapping and filter of f and of
 * a flat image (iterations passes), and the per-pixel gain correction.
 * All pointers are device pointers; work is queued on `stream`.
 */
int rubs_b200_structure_tensor(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                               double window_sigma, double *j, void *stream);
int rubs_b200_anisotropy(const double *j, int64_t H, int64_t W, double noise_sigma,
                         const double *size_range, double bound_fraction, double iso_gain,
                         double *size, double *elong, double *orient, unsigned char *isotropic,
                         void *stream);
int rubs_b200_adaptive_smooth(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                              double noise_sigma, double window_sigma, int iterations,
                              const rubs_lut *lut, double bound_fraction,
                              const double *size_range, double iso_gain, double *out,
                              int64_t ld_out, void *stream);

/*
 * Three-direction (N=3) radially-uniform box spline: directions at 0, 60
 * and 120 degrees (the reference's direction_vectors(3), geometry.py:76-81;
 * covariance sum a_k^2/12 u_k u_k^T, covariance_general, geometry.py:102-106),
 * BASELINE.json config 3.  The reference has no N=3 filter (SURVEY.md §0
 * fact 6); these entry points extend engine.filter_space_variant
 * (engine.py:265-324) with its semantics -- zero padding, floor 0.05 before
 * the 1/sqrt(m) scaling, iterated passes on canvases extended by the global
 * support with the field edge-clamped -- to the N=3 kernel, computed
 * exactly (no interpolation of the image).
 *   field    device (H, W, 3) float64, element (r, c, k) at
 *            field[(r * ld_field + c) * 3 + k]; or, when field_is_uniform,
 *            a HOST pointer to 3 doubles
 */
int rubs_b200_filter3(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                      const double *field, int field_is_uniform, int64_t ld_field,
                      int iterations, double *out, int64_t ld_out, void *stream);
int rubs_b200_filter3_host(const void *f, int f_dtype, int64_t H, int64_t W,
                           const double *field, int field_is_uniform, int iterations,
                           double *out);

/*
 * Fused N=3 mapping + filter: per-pixel (size, elongation, orientation) ->
 * covariance (covariance_from_params, geometry.py:153-172) -> the unique
 * N=3 scales matching it (closed form; RUBS_EINFEASIBLE beyond the N=3
 * elongation bound, min 3 at 30/90/150 degrees) -> filter.
 */
int rubs_b200_filter3_params(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                             const void *size, const void *elong, const void *orient,
                             int p_dtype, int64_t ld_p, int iterations, double *out,
                             int64_t ld_out, void *stream);
int rubs_b200_filter3_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                  const void *size, const void *elong, const void *orient,
                                  int p_dtype, int iterations, double *out);

/*
 * N=3 row bands (multi-GPU sharding of config 3's single image, as the N=4
 * rubs_b200_filter_params_rows): output rows [out_row0, out_row0 +
 * out_rows) from image rows [f_row0, f_row0 + f_rows) (rows outside read as
 * zero, so the halo must cover the band's reach) and parameter rows from
 * p_row0 on.  rubs_b200_read_margins3_params gives the reach of a band's
 * parameter rows: out2 = {columns, rows} = max over its pixels of
 * ceil(a1/2 + (a2 + a3)/4) + 1 and ceil((a2 + a3) sqrt3 / 4) + 1.
 */
int rubs_b200_read_margins3_params(const void *size, const void *elong, const void *orient,
                                   int p_dtype, int64_t rows, int64_t W, int64_t ld_p,
                                   int *out2, void *stream);
int rubs_b200_filter3_params_rows(const void *f, int f_dtype, int64_t f_row0, int64_t f_rows,
                                  int64_t W, int64_t ld_f, int64_t H_total, const void *size,
                                  const void *elong, const void *orient, int p_dtype,
                                  int64_t p_row0, int64_t ld_p, int64_t out_row0,
                                  int64_t out_rows, double *out, int64_t ld_out, void *stream);

/*
 * N=3 lattice mode: the paper's O(1) algorithm for the off-grid directions
 * (285, 662: "one needs to interpolate the image for
 * implementing the associated running-sums").  The image is moved once onto
 * the triangular lattice of spacing `spacing` (in [0.125, 1], pixels) that
 * contains the three directions, by the adjoint of linear interpolation;
 * the exact N=3 kernel is then applied to that resampled image in O(1) per
 * pixel (exact int128 running sums along the lattice directions, an
 * 8-vertex finite difference, linear interpolation on the lattice
 * triangles).  Against the exact filter above this differs by the
 * resampling error only; arguments and errors as
 * rubs_b200_filter3 / _params, plus RUBS_EVALUE for non-finite image
 * entries (integer running sums carry no NaN).
 */
int rubs_b200_filter3_lattice(const void *f, int f_dtype, int64_t H, int64_t W, int64_t ld_f,
                              const double *field, int field_is_uniform, int64_t ld_field,
                              int iterations, double spacing, double *out, int64_t ld_out,
                              void *stream);
int rubs_b200_filter3_lattice_params(const void *f, int f_dtype, int64_t H, int64_t W,
                                     int64_t ld_f, const void *size, const void *elong,
                                     const void *orient, int p_dtype, int64_t ld_p,
                                     int iterations, double spacing, double *out,
                                     int64_t ld_out, void *stream);
/* Row-band entry of the lattice mode (one pass, fused mapping): output rows
 * [out_row0, out_row0 + out_rows) of an H_total-row image whose rows
 * [f_row0, f_row0 + f_rows) are given (rows outside count as zero, so the
 * caller supplies the band's halo: its kernels' vertical reach + 1); the
 * parameter arrays hold global rows from p_row0 on.  Mirrors
 * rubs_b200_filter3_params_rows.  Bands reproduce the whole-image call up to
 * the blocks' quantisation exponents (~1e-17 relative), not bit for bit. */
int rubs_b200_filter3_lattice_params_rows(const void *f, int f_dtype, int64_t f_row0,
                                          int64_t f_rows, int64_t W, int64_t ld_f,
                                          int64_t H_total, const void *size, const void *elong,
                                          const void *orient, int p_dtype, int64_t p_row0,
                                          int64_t ld_p, int64_t out_row0, int64_t out_rows,
                                          double spacing, double *out, int64_t ld_out,
                                          void *stream);
int rubs_b200_filter3_lattice_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                   const double *field, int field_is_uniform, int iterations,
                                   double spacing, double *out);
int rubs_b200_filter3_lattice_params_host(const void *f, int f_dtype, int64_t H, int64_t W,
                                          const void *size, const void *elong,
                                          const void *orient, int p_dtype, int iterations,
                                          double spacing, double *out);

/* The N=3 mapping alone: device arrays of n parameters -> device n x 3. */
int rubs_b200_scales3(const void *size, const void *elong, const void *orient, int p_dtype,
                      int64_t n, double *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RUBS_B200_H */
