/*
 * bccb_b200.h — C ABI of the B200-native BCCB Gram operator and its fused
 * ISTA / FISTA / ADMM iterations.
 *
 * This is the drop-in boundary under the reference package `bccblasso`
 * (/root/reference/pkg/src/bccblasso).  Every entry point names the reference
 * interface it replaces.  Plain C types only: device buffers are passed as raw
 * device pointers (void*), CUDA streams as void* (cudaStream_t), sizes as int.
 *
 * Layouts (all row-major, batch outermost):
 *   grid vector x      [batch][L2][L1]   flat index l = l1 + l2*L1 per snapshot
 *                                        (reference: bccb.py:10-11, 120-125)
 *   spectral box       [batch][K1][K2]   fft2(x)[k2][k1] for k1 < K1, k2 < K2
 *   complex64  = interleaved float  (re, im)
 *   complex128 = interleaved double (re, im)
 *
 * Errors: every function returns a bccb_status; the matching message is
 * available from bccb_last_error() (thread-local).  The Python shim maps the
 * codes to the reference exception classes (pkg/src/bccblasso/errors.py:4-65).
 */
#ifndef BCCB_B200_H
#define BCCB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BCCB_OK = 0,
  BCCB_ERR_INVALID = 1,     /* InvalidArgumentError   (errors.py:8)  */
  BCCB_ERR_DIVERGENCE = 2,  /* DivergenceError        (errors.py:48) */
  BCCB_ERR_SINGULAR = 3,    /* SingularOperatorError  (errors.py:28) */
  BCCB_ERR_CUDA = 4,        /* CUDA runtime failure                  */
  BCCB_ERR_UNSUPPORTED = 5  /* size outside the GPU engine's range   */
} bccb_status;

typedef struct bccb_plan_s* bccb_plan_t;

/* Message of the last failing call on this thread ("" if none). */
const char* bccb_last_error(void);

/* Library version string. */
const char* bccb_version(void);

/* ---------------------------------------------------------------- plans */

/* Operator from its eigenvalue box.
 * Replaces BccbOperator(l1, l2, eigenvalues) (bccb.py:50-74) and the eigen step
 * of bccb_from_first_column (bccb.py:93-105).
 *   box_t   : host complex128 [K1][K2]: eig_t[k2][k1] = eigenvalues[k1][k2] on the box
 *   lam_out : the (constant) eigenvalue outside the box (ignored when the box is full)
 * K1 <= L1, K2 <= L2.  Pass K1 = L1, K2 = L2 for a general operator. */
int bccb_plan_create(int l1, int l2, int k1, int k2, const double* box_t, double lam_out_re,
                     double lam_out_im, int device, bccb_plan_t* out);

/* Gram of a sparse planar array on the uniform L1 x L2 grid.
 * Replaces gram_operator(geometry, l1, l2) (bccb.py:108-110) -> gram_first_column
 * (bccb.py:77-90) -> bccb_from_first_column (93-105): the eigenvalues are built
 * directly as L1*L2 * (aliased occupancy count), no first column, no zgemm.
 *   occupancy : host uint8 [m1_count][m2_count] (ArrayGeometry.occupancy, arrays.py:20-48)
 * Also stores the occupied coordinates (scan order m2 outer, m1 inner; arrays.py:55-62)
 * for bccb_adjoint. */
int bccb_plan_create_gram(int l1, int l2, int m1_count, int m2_count, const uint8_t* occupancy,
                          int device, bccb_plan_t* out);

int bccb_plan_destroy(bccb_plan_t plan);

/* Band of the plan: *k1, *k2 (spectral box size); *m = occupied elements (0 if not a Gram plan). */
int bccb_plan_info(bccb_plan_t plan, int* l1, int* l2, int* k1, int* k2, int* m);

/* Copy the eigenvalue box back (host complex128 [K1][K2]) and the outside value. */
int bccb_plan_eigen_box(bccb_plan_t plan, double* box_t, double* lam_out_re, double* lam_out_im);

/* Device workspace (bytes) needed by the operator / solver calls for `batch` snapshots. */
size_t bccb_workspace_bytes(bccb_plan_t plan, int batch);

/* ---------------------------------------------------------------- operator */

/* y = G x for a batch (complex64 in/out, device).  Replaces bccb_matvec (bccb.py:113-125). */
int bccb_matvec(bccb_plan_t plan, int batch, const void* x, void* y, void* workspace,
                void* stream);

/* Same in complex128 end to end (complex128 band FFTs): drop-in precision for float64 callers. */
int bccb_matvec_z(bccb_plan_t plan, int batch, const void* x, void* y, void* workspace,
                  void* stream);

/* out_box = fft2(x) restricted to the box (complex64 [batch][K1][K2]).
 * Replaces the spectrum computation np.fft.fft2 of bccb.py:104/123 for a band. */
int bccb_spectrum_box(bccb_plan_t plan, int batch, const void* x, void* out_box, void* workspace,
                      void* stream);

/* out = alpha * x + scale * ifft2_unnormalised(box)  (box: complex64 [batch][K1][K2]; x may be
 * NULL when alpha == 0; out may be NULL).  maxabs (device float [batch], may be NULL) receives
 * max |out| per snapshot (it must be zeroed by the caller).  Used for A^H y and for the
 * out-of-band residual of a user-supplied right-hand side. */
int bccb_synthesize(bccb_plan_t plan, int batch, const void* box, float scale, const void* x,
                    float alpha, void* out, float* maxabs, void* workspace, void* stream);

/* complex128 counterparts of bccb_spectrum_box / bccb_synthesize (x, out_box, box, out:
 * device complex128), on the float64 band engine: the eigenvalue transform of
 * bccb_from_first_column (bccb.py:93-105: fft2 of the first column) and its inverse
 * bccb_first_column (bccb.py:151-153) at float64 accuracy. */
int bccb_spectrum_box_z(bccb_plan_t plan, int batch, const void* x, void* out_box, void* workspace,
                        void* stream);
int bccb_synthesize_z(bccb_plan_t plan, int batch, const void* box, double scale, void* out,
                      void* workspace, void* stream);

/* A^H y for a batch of snapshots (Gram plans only).
 * Replaces apply_adjoint (dictionary.py:129-136) on the grid f = -1/2 + l/L
 * (dictionary.py:41-45) plus the per-snapshot max|b| of the tau rule
 * (experiments.py:232, cli.py:241-244):
 *   y        : device complex64 [batch][M] in occupancy scan order
 *   bhat_box : device complex64 [batch][K1][K2] <- fft2(b) on the box (= L * signed scatter of y)
 *   b        : device complex64 [batch][L2][L1] <- b (may be NULL)
 *   maxabs   : device float [batch] <- max|b| (may be NULL) */
int bccb_adjoint(bccb_plan_t plan, int batch, const void* y, void* bhat_box, void* b,
                 float* maxabs, void* workspace, void* stream);

/* ---------------------------------------------------------------- solvers */

/* ISTA (d == NULL) / FISTA (d != NULL): iterations first_iteration .. first_iteration+iterations-1
 * run fused and in place (first_iteration > 0 continues a run: the momentum sequence and the
 * divergence record carry on; first_bad is reset only when first_iteration == 0).
 * Replaces the loops of ista_solve (solvers.py:252-291) and fista_solve (solvers.py:311-355).
 *   mu       : step size (SolverConfig.step_size_mu)
 *   tau      : device double [batch], per-snapshot sparsity weight (kappa = mu * tau)
 *   bhat_box : device complex64 [batch][K1][K2] = fft2(b) on the box
 *   extra    : device complex64 [batch][L2][L1] out-of-band part of b (NULL if none)
 *   c        : device complex128 [batch][L2][L1] iterate (in: initial_c, out: estimate)
 *   d        : device complex64  [batch][L2][L1] momentum state c_t - c_{t-1} (in: zeros)
 *   first_bad: device int [batch] <- first iteration with a non-finite iterate (INT_MAX if none)
 * The momentum coefficients follow _next_alpha (solvers.py:294-296) from alpha = 1. */
int bccb_fista_run(bccb_plan_t plan, int batch, int first_iteration, int iterations, double mu,
                   const double* tau,
                   const void* bhat_box, const void* extra, void* c, void* d, int* first_bad,
                   void* workspace, void* stream);

/* bccb_fista_run from iteration 0 with the objective trace of solvers.py:233-242,
 * f(c_{t+1}) - ||y||^2 = -2 Re<b, c> + Re<c, G c> + tau ||c||_1, accumulated on the device for
 * every iteration inside the same pass kernels (record_objective=True without a host round
 * trip; replaces the trace lines solvers.py:272-280 and 340-343).  The quadratic part is taken
 * on the spectral box by Parseval; tau ||c||_1 is summed by the rows pass.
 *   trace : device double [batch][iterations] <- the objective minus ||y||^2 (caller adds it)
 * Returns BCCB_ERR_UNSUPPORTED (the caller falls back to per-iteration reductions) unless the
 * plan is a Gram-type operator (zero spectrum outside the box), b lies on the box (no extra)
 * and the grid has a specialised rows pass. */
int bccb_fista_run_traced(bccb_plan_t plan, int batch, int iterations, double mu, const double* tau,
                          const void* bhat_box, void* c, void* d, int* first_bad, double* trace,
                          void* workspace, void* stream);

/* ADMM: iterations first_iteration .. first_iteration+iterations-1, fused and in place.
 * Replaces admm_solve (solvers.py:385-448): precompute P = (G + rho I)^-1, q = P b
 * (403-415) folded into the spectral box; loop c = q + rho P(z - v), z = S_{rho tau}(c + v),
 * v = v + (c - z) (426-436).
 *   z        : device complex128 [batch][L2][L1] (in: initial z; out: final z = the estimate)
 *   v        : device complex128 [batch][L2][L1] scaled dual (in: zeros; out: final)
 *   c_last   : device complex128 [batch][L2][L1] <- c of the last iteration (may be NULL)
 * Runs on the complex128 band engine: v grows like t*|q| when z stays 0 (config 3, SURVEY
 * finding 7) and the band correction cancels it, so complex64 would lose ~log2(t) bits.
 * Returns BCCB_ERR_SINGULAR if G + rho I is numerically singular (bccb.py:133-148). */
int bccb_admm_run(bccb_plan_t plan, int batch, int first_iteration, int iterations, double rho,
                  const double* tau,
                  const void* bhat_box, const void* extra, void* z, void* v, void* c_last,
                  int* first_bad, void* workspace, void* stream);

/* ---------------------------------------------------------------- peaks */

/* Workspace (bytes) for bccb_topk. */
size_t bccb_topk_workspace_bytes(int batch, long long length, int k);

/* Per-snapshot top-k of |values| in extract_support order (solvers.py:494-499: stable
 * argsort of -|c|, ties to the lower index).  values: device [batch][length], complex64
 * (is_double = 0) or complex128 (is_double = 1).  k <= 64.
 *   idx : device int32 [batch][k] flat grid indices l = l1 + l2*L1
 *   mag : device float [batch][k] |values| at those indices (may be NULL) */
int bccb_topk(int batch, long long length, const void* values, int is_double, int k, int* idx,
              float* mag, void* workspace, void* stream);

/* ---------------------------------------------------------------- accounting */

/* Total kernel launches issued by the library in this process (bench: gpu_launches). */
long long bccb_launch_count(void);

/* Bracket every launch of this thread with CUDA events on its stream until
 * bccb_profile_end, which synchronises and returns the summed device time and launch
 * count per kernel kind: [0] rows pass (band IFFT + solver epilogue + band FFT),
 * [1] column pass (band FFT * spectrum + band IFFT), [2] other (setup, scatter). */
int bccb_profile_begin(void);
int bccb_profile_end(double* ms_by_kind, long long* launches_by_kind);

/* Number of streams a large batch is split over (1..8; 0 restores the default: env
 * BCCB_SUBSTREAMS, else 3; fewer when a part would have < 2048 lines).  The parts are
 * independent snapshots, so results are bitwise identical either way. */
int bccb_set_substreams(int n);

/* Sub-batch stream count a solver call on `plan` with this batch would use now (bench:
 * how many launches of a pass run concurrently). */
int bccb_substreams_for(bccb_plan_t plan, int batch);

/* Kernel path: 0 = automatic (small-grid persistent solver, shape-specialised and fused
 * kernels, generic fallback), 1 = generic runtime-shape kernels only.  Results agree to
 * floating-point rounding (the paths evaluate the soft threshold with different float64
 * sequences); used to cross-check the specialised kernels. */
int bccb_set_path(int path);

#ifdef __cplusplus
}
#endif

#endif /* BCCB_B200_H */
