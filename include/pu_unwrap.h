/*
 * pu_unwrap.h — C ABI of the B200-native L1 phase unwrapper (libpu_unwrap.so).
 *
 * Drop-in boundary for the hot path `phaseirls.unwrap` (reference
 * pkg/src/phaseirls/irls.py:132-224).  The reference is pure Python; its
 * only compiled seam is the numba kernel module rebound by
 * `kernels.select_backend` (kernels.py:170-187).  Each entry point below
 * replaces one reference function on that path (cited per function); the
 * Python host (paper_2401_09961_b200/) mirrors irls.py / pcg.py above it.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller.
 *  - A "plane" is an N x M grid stored row-major with row pitch
 *    pu_pitch(h) elements (dtype of the handle: float or double); pitch
 *    padding must be zero-initialised by the caller.  A "system vector"
 *    (reference SystemVector, operators.py:39-101) is 3 consecutive planes
 *    [u | vv | vh]; vv's last row and vh's last column are zero pads.
 *    Arc-shaped inputs (gv, gh, cv, ch, wv, wh, dv, dh) are planes with the
 *    same pads.
 *  - Scalar results are written as fp64 to caller-provided device memory.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  No entry
 *    point synchronises unless documented.
 *  - Return value: PU_OK or an error code; pu_last_error() describes it.
 *    No C++ exception crosses the ABI.
 */
#ifndef PU_UNWRAP_H
#define PU_UNWRAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PU_ABI_VERSION 1

enum pu_dtype { PU_F32 = 0, PU_F64 = 1 };

enum pu_status {
  PU_OK = 0,
  PU_ERR_ARG = 1,          /* invalid argument (reference raises ValueError) */
  PU_ERR_CUDA = 2,         /* CUDA runtime error */
  PU_ERR_UNSUPPORTED = 3,  /* grid size outside the shared-memory FFT limits */
  PU_ERR_NOMEM = 4,
  PU_ERR_BREAKDOWN = 5     /* NumericalBreakdown (pcg.py:24-29): a non-finite PCG value (pu_unwrap) */
};

/* Device-side PCG control block (caller allocates pu_pcg_ctrl_bytes()).
 * Mirrors pcg_solve's scalars and outcome (pcg.py:24-38, 47-116). */
typedef struct pu_pcg_ctrl {
  double rho, alpha, beta, thr, bnorm, pap, rn, mean_ru, rho_s;
  int32_t done;        /* loop finished */
  int32_t converged;   /* PcgOutcome.converged */
  int32_t breakdown;   /* -1, or NumericalBreakdown.iteration */
  int32_t bkind;       /* 0 initial residual, 1 p'Ap, 2 ||r||, 3 r.z */
  int32_t iterations;  /* PcgOutcome.iterations = len(residual_norms) - 1 */
  int32_t max_iters;
  int32_t pad_[2];
} pu_pcg_ctrl;

typedef struct pu_handle pu_handle;

int pu_abi_version(void);
const char* pu_last_error(void);
int pu_pcg_ctrl_bytes(void);
/* Number of kernels this library has launched in the process so far. */
int64_t pu_launch_count(void);

/* Plan an N x M grid (FFT tables, launch shapes, reduction scratch).
 * tau/delta: ModelParams (objective.py:30-41). */
int pu_create(pu_handle** out, int n, int m, int dtype, double tau, double delta);
int pu_destroy(pu_handle* h);
int64_t pu_pitch(const pu_handle* h);
int64_t pu_plane_elems(const pu_handle* h);
/* Describe the launch plan (for logs): writes a NUL-terminated string. */
int pu_describe(const pu_handle* h, char* buf, int cap);

/* Layout helpers: compact fp64 (rows x cols, pitch lds) <-> plane. */
int pu_pack(pu_handle* h, const double* src, int64_t lds, int rows, int cols, void* dst, void* stream);
int pu_unpack(pu_handle* h, const void* src, int rows, int cols, double* dst, void* stream);
/* plane -> compact (rows x cols) array in the handle's dtype (for half-size D2H in fp32 mode). */
int pu_unpack_native(pu_handle* h, const void* src, int rows, int cols, void* dst, void* stream);
int pu_fill(pu_handle* h, void* dst, int nplanes, double value, void* stream);
int pu_copy(pu_handle* h, const void* src, void* dst, int nplanes, void* stream);

/* phase.py:140-149 wrapped_gradients (+ wrap_to_principal phase.py:118-137,
 * kernels.diff_rows/diff_cols kernels.py:87-103).  x: fp64 N x M, pitch ldx.
 * Bit-identical to the reference in fp64. lo must be 0 or -pi. */
int pu_wrapped_gradients(pu_handle* h, const double* x, int64_t ldx, void* gv, void* gh, double lo,
                         void* stream);

/* pu_wrapped_gradients + the input check of phase.py:100-115 from the same
 * loads (whole grids): check[0] = number of non-finite x, check[1] = number
 * of finite x outside [0, 2pi) (device fp64).  The caller raises the
 * reference's ValueError when either is non-zero (the Python host reads them
 * with the first scalar snapshot, so no extra synchronisation). */
int pu_wrapped_gradients_checked(pu_handle* h, const double* x, int64_t ldx, void* gv, void* gh, double lo,
                                 double* check, void* stream);

/* irls.py:167 initial state x = (0, -gv, -gh). */
int pu_init_state(pu_handle* h, const void* gv, const void* gh, void* x, void* stream);

/* operators.py:156-162 build_rhs. b: system vector. */
int pu_build_rhs(pu_handle* h, const void* gv, const void* gh, void* b, void* stream);

/* operators.py:138-153 apply_system (= kernels.apply_system_blocks,
 * kernels.py:125-145). y = A(d) x. */
int pu_apply_system(pu_handle* h, const void* x, const void* dv, const void* dh, void* y, void* stream);

/* operators.py:70-75 SystemVector.dot over nplanes planes (1 or 3). */
int pu_dot(pu_handle* h, const void* a, const void* b, int nplanes, double* out, void* stream);

/* preconditioner.py:86-100 sylvester_solve on one plane (u block): z = the
 * Neumann-Poisson pseudo-inverse of tau * r via DCT-II/III.  spec: one plane
 * of scratch.  r and z may alias. */
int pu_sylvester_solve(pu_handle* h, const void* r, void* z, void* spec, void* stream);

/* preconditioner.py:103-115 apply_preconditioner (block diagonal D^+). */
int pu_apply_preconditioner(pu_handle* h, const void* r, const void* dv, const void* dh, void* z, void* spec,
                            void* stream);

/* objective.py:92-100 update_weights + irls.py:191 (d = c^2 / w) and the
 * H_delta pair of irls.py:176-177: out[0] = H(x, w_prev) (if wpv != NULL),
 * out[1] = H(x, w).  cv/ch may both be NULL (uniform unit weights). */
int pu_weights_hpair(pu_handle* h, const void* x, const void* cv, const void* ch, const void* gv,
                     const void* gh, const void* wpv, const void* wph, void* wv, void* wh, void* dv, void* dh,
                     double* out, void* stream);

/* objective.py:77-89 eval_h_delta. out[0] = H_delta(x, w). */
int pu_eval_h_delta(pu_handle* h, const void* x, const void* wv, const void* wh, const void* gv,
                    const void* gh, const void* cv, const void* ch, double* out, void* stream);

/* objective.py:63-66 eval_f. out[0] = F, out[1] = weighted L1 part. */
int pu_eval_f(pu_handle* h, const void* x, const void* gv, const void* gh, const void* cv, const void* ch,
              double* out, void* stream);

/* objective.py:118-125 candidate_step with stepsize 1/lipschitz. */
int pu_candidate_step(pu_handle* h, const void* x, const void* wv, const void* wh, const void* gv,
                      const void* gh, const void* cv, const void* ch, double lipschitz, void* out, void* stream);

/* irls.py:202-205: out[0] = H(xa, w), out[1] = H(xb, w),
 * out[2] = mean(u) of the accepted state, out[3] = 1.0 if xa is accepted. */
int pu_hpair_states(pu_handle* h, const void* xa, const void* xb, const void* wv, const void* wh,
                    const void* gv, const void* gh, const void* cv, const void* ch, double* out, void* stream);

/* irls.py:206-215: dst = (sel[1] ? xa : xb) with u -= sel[0];
 * out[0] = H(dst, w).  dst must not alias xa or xb. */
int pu_accept_center(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst,
                     const void* wv, const void* wh, const void* gv, const void* gh, const void* cv,
                     const void* ch, double* out, void* stream);

/* One IRLS inner step, irls.py:191-205: the explicit gradient candidate of
 * `state` (objective.py:118-125) -> cand, the PCG solve warm-started from
 * `state` and run IN PLACE on it (it becomes the proposal; the candidate and
 * the start-up residual share one pass over the state), then
 * out[0] = H(proposal, w), out[1] = H(cand, w), out[2] = mean u of the
 * accepted one, out[3] = 1.0 if the proposal is accepted.  cv/ch may both be
 * NULL for uniform unit weights.  PCG scratch and ctrl as in pu_pcg_solve.
 * b may be NULL: b = build_rhs(gv, gh) (pu_build_rhs) is then formed inside
 * the start-up kernel from the gradient loads the candidate step makes
 * anyway (bit-identical; the three b planes are never read). */
int pu_irls_step(pu_handle* h, void* state, const void* b, const void* gv, const void* gh, const void* cv,
                 const void* ch, const void* wv, const void* wh, const void* dv, const void* dh, double lipschitz,
                 int max_iters, double rel_tol, void* cand, void* r, void* p0, void* p1, void* spec, void* ctrl,
                 double* res_norms, double* out, void* stream);

/* pu_irls_step in two halves, so the host can run the first speculatively
 * while it reads the previous iteration's scalars and applies the budget
 * rule (irls.py:178-189): pu_irls_begin = candidate step + PCG start-up +
 * z0 = M r0 (needs no budget; leaves the state untouched), pu_irls_iterate =
 * the budget's iterations (in place on `state`) + the H pair.  Same
 * arguments and outputs as pu_irls_step; each half is replayed as a graph. */
int pu_irls_begin(pu_handle* h, void* state, const void* b, const void* gv, const void* gh, const void* cv,
                  const void* ch, const void* wv, const void* wh, const void* dv, const void* dh, double lipschitz,
                  double rel_tol, void* cand, void* r, void* p0, void* p1, void* spec, void* ctrl, double* res_norms,
                  void* stream);
int pu_irls_iterate(pu_handle* h, void* state, const void* gv, const void* gh, const void* cv, const void* ch,
                    const void* wv, const void* wh, const void* dv, const void* dh, int max_iters, void* cand, void* r,
                    void* p0, void* p1, void* spec, void* ctrl, double* res_norms, double* out, void* stream);

/* CUDA-graph replay of pu_irls_step (default on): each (budget, pointers,
 * scalars) combination is captured once and relaunched as one graph when the
 * stream is not the legacy default stream and the budget is <= 64. */
int pu_set_graphs(pu_handle* h, int on);

/* irls.py:206-215 fused with the next iteration's irls.py:173-177:
 * dst = (sel[1] ? xa : xb) with u -= sel[0]; w_next, d from dst;
 * out[0] = H(dst, w_k), out[1] = H(dst, w_next).  dst must not alias xa/xb. */
int pu_accept_weights(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst, const void* gv,
                      const void* gh, const void* cv, const void* ch, const void* wkv, const void* wkh, void* wnv,
                      void* wnh, void* dv, void* dh, double* out, void* stream);

/* pu_accept_weights of iteration k (irls.py:203-215, 173-177) fused with the
 * budget-free start of iteration k + 1 (irls.py:191-202: objective.py:118-125
 * candidate, pcg.py:59-75 start-up; the kernel of pu_irls_begin, b = NULL):
 * besides dst, w_next, d and out[0..1] it writes r = b - A dst
 * (b = build_rhs(gv, gh)) and cand = dst - (1/L) grad H(dst, w_next) from the
 * same registers, one pass over the accepted state instead of two.  The
 * start-up sums are held in the handle; ctrl is not touched until
 * pu_irls_begin_z0 finalises them.  Band handles: xa and xb need their ghost
 * rows (u both ways, v from above); the sums go to the band totals (the H
 * pair to the S_ACC row, the start-up sums to S_START's) for the all-reduce
 * and pu_finalize, as after pu_accept_weights and pu_pcg_begin.
 * Every value agrees with pu_accept_weights + pu_irls_begin (fp32 bitwise,
 * fp64 to the last bits of the FMA contraction). */
int pu_accept_weights_start(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst,
                            const void* gv, const void* gh, const void* cv, const void* ch, const void* wkv,
                            const void* wkh, void* wnv, void* wnh, void* dv, void* dh, double* out, double lipschitz,
                            void* r, void* cand, void* stream);
/* The rest of pu_irls_begin after pu_accept_weights_start: finalise the held
 * start-up sums into ctrl/res_norms (pcg.py:59-75) and z0 = M r0, rho0,
 * p0 = z0 (pcg.py:77-79).  Replayed as a CUDA graph.  PU_ERR_ARG unless a
 * pu_accept_weights_start on the same handle precedes it. */
int pu_irls_begin_z0(pu_handle* h, const void* dv, const void* dh, double rel_tol, void* r, void* p0, void* p1,
                     void* spec, void* ctrl, double* res_norms, void* stream);

/* pcg.py:47-116 pcg_solve with apply_system and apply_preconditioner fused
 * in (5 kernels per iteration).  x = x0 on entry (x may alias x0: solve in
 * place); otherwise x0 is not modified.  z is unused (kept for ABI stability).
 * r, z, p0, p1: system-vector scratch; spec: one plane.  ctrl: device
 * pu_pcg_ctrl; res_norms: device fp64 [max_iters + 1].  Enqueues without
 * synchronising when max_iters <= 64; longer budgets poll ctrl->done
 * every 64 iterations. */
int pu_pcg_solve(pu_handle* h, const void* b, const void* x0, void* x, const void* dv, const void* dh,
                 void* r, void* z, void* p0, void* p1, void* spec, int max_iters, double rel_tol,
                 void* ctrl, double* res_norms, void* stream);

/* Harness metrics on the device (whole-grid handles), against compact or
 * pitched fp64 device grids (row pitch ldx / ldr elements):
 *  pu_shift_error    phase.py:152-175: out[0] alpha = mean(x_u - u),
 *                    out[1] max |err|, out[2] rmse, out[3] congruent fraction
 *                    (|err / 2pi - rint| <= 1e-3), err = x_u - (u + alpha);
 *  pu_kmap_mismatch  SURVEY §8(d): mean(rint((u - x)/2pi) != rint((u_ref - x)/2pi));
 *  pu_congruent_round phase.py:178-184: out (compact N x M fp64) =
 *                    x + 2pi rint((u - x)/2pi).
 * u is the u plane of a system vector (handle dtype). */
int pu_shift_error(pu_handle* h, const void* u, const double* xu, int64_t ldx, double* out, void* stream);
int pu_kmap_mismatch(pu_handle* h, const void* u, const double* uref, int64_t ldr, const double* x, int64_t ldx,
                     double* out, void* stream);
int pu_congruent_round(pu_handle* h, const void* u, const double* x, int64_t ldx, double* out, void* stream);

/* Per-launch CUDA-event timing on the launching stream (off by default).
 * pu_timing_read synchronises on the recorded events and returns the number
 * of records (kind, iteration, milliseconds) written, up to cap; kinds:
 * 0 pcg_start, 1 K1 (p, Ap, p'Ap), 2 K2a (x, r, z_s, norms), 3 K3 (column
 * DCT pair), 4 K4 (row DCT-III), 5 reprojection update, 6 weights,
 * 7 candidate, 8 H pair, 9 accept, 10 K2b (row DCT-II of r_u).
 * Iteration -1 = PCG setup / outer kernel. */
int pu_timing_enable(pu_handle* h, int on);
int pu_timing_read(pu_handle* h, int* kinds, int* its, float* ms, int cap);

/* ------------------------------------------------------------------------
 * Row-sharded grids (BASELINE config C4: one image across the GPUs of a box;
 * SURVEY.md §8(e)).  The reference has no distributed mode; these entry
 * points split its pcg_solve iteration (pcg.py:81-108) at the points where a
 * sharded run exchanges data, so the host (paper_2401_09961_b200/band.py)
 * can put the collectives between them:
 *   - halo: every plane of a band handle has ghost rows -1 and `rows`
 *     (plane = (rows + 2) * pitch elements; pass pointers to row 0), which
 *     mirror the neighbouring bands' edge rows;
 *   - all-reduce: in band mode every reduction leaves its band totals in the
 *     `totals` buffer (row `site`, PU_MAX_SUMS doubles) instead of
 *     finalising; after summing them over ranks, pu_finalize runs the
 *     finalisers of the listed sites;
 *   - all-to-all: the row DCT-II writes the spectrum in the packed layout
 *     chunk q = columns [q mb, (q+1) mb) x rows, row pitch mb; after the
 *     transpose each rank runs the column transform on its N x cols block
 *     (pitch mb); the reverse transpose returns the same packed layout to the
 *     row DCT-III.
 * The same calls on a whole-grid handle reproduce pu_pcg_solve.
 * ------------------------------------------------------------------------ */
typedef struct pu_band {
  int32_t n_glob;      /* N of the whole grid */
  int32_t row0, rows;  /* this rank's rows [row0, row0 + rows) */
  int32_t nq;          /* ranks = column chunks of the transpose */
  int32_t mb;          /* columns per chunk: multiple of 8, nq * mb >= M */
  int32_t col0, cols;  /* this rank's column block: col0 = rank * mb, cols = min(mb, M - col0) >= 1 */
} pu_band;

enum pu_site { PU_SITE_WH = 1, PU_SITE_HPAIR = 3, PU_SITE_ACC = 4, PU_SITE_START = 6, PU_SITE_K1 = 7,
               PU_SITE_K2 = 8, PU_SITE_K3 = 9, PU_SITE_UPD = 10, PU_SITE_MET = 12, PU_NSITES = 13 };
#define PU_MAX_SUMS_ABI 12

int pu_create_band(pu_handle** out, int m, const pu_band* band, int dtype, double tau, double delta);
/* Device fp64 [PU_NSITES * PU_MAX_SUMS_ABI] that receives band totals; NULL
 * restores single-grid finalisation. */
int pu_set_band_totals(pu_handle* h, double* totals);
/* Fused transpose, push model (every cross-GPU access is a store): the
 * device tables (nq uint64 each) hold every rank's column block (N x mb,
 * pitch mb) and every rank's back buffer (packed rows, as spec_in) -- on this
 * GPU, or a peer's mapped with pu_ipc_open over NVLink.  The row DCT-II
 * stores each chunk straight into its owner's column block (spec_out is
 * ignored), the column transform stores each output row into the owner's
 * back buffer, and the row DCT-III reads its own back buffer (spec_in).  The
 * caller orders the kernels across ranks (the all-reduces between them do).
 * NULL, NULL: the packed all-to-all layout. */
int pu_set_band_peers(pu_handle* h, const uint64_t* col_blocks, const uint64_t* back_buffers);
/* CUDA IPC for the peer tables: a 64-byte handle of a pu_dev_alloc block,
 * opened in another process on a peer GPU. */
int pu_ipc_handle(const void* dev_ptr, void* handle);
int pu_ipc_open(const void* handle, void** dev_ptr);
int pu_ipc_close(void* dev_ptr);
int pu_dev_alloc(int64_t bytes, void** dev_ptr);
int pu_dev_free(void* dev_ptr);
/* Run the finalisers of the sites in `mask` (bit = pu_site) on `totals` (the
 * all-reduced buffer), in PCG order, skipping PCG sites once ctrl->done.
 * mode: 1 = PCG set-up (z0, rho0), 2 = iteration `it`.  out: the scalar
 * block of the outer-iteration sites (WH, HPAIR, ACC). */
int pu_finalize(pu_handle* h, unsigned mask, int mode, int it, void* ctrl, double* res_norms, double* out,
                double rel_tol, int max_iters, void* stream);
/* The budget of a PCG loop whose set-up was finalised with a placeholder
 * max_iters (the speculative start-up of row bands): ctrl->max_iters =
 * max_iters, enqueued on `stream`. */
int pu_set_max_iters(pu_handle* h, void* ctrl, int max_iters, void* stream);
/* pcg.py:59-75 (+ the candidate step objective.py:118-125 when cand != NULL,
 * as in pu_irls_step).  x may alias x0.  b may be NULL when cand != NULL
 * (b = build_rhs(gv, gh) formed in the kernel, as in pu_irls_step). */
int pu_pcg_begin(pu_handle* h, const void* b, const void* x0, void* x, const void* dv, const void* dh, void* r,
                 void* ctrl, double* res_norms, int max_iters, double rel_tol, const void* gv, const void* gh,
                 const void* cv, const void* ch, const void* wv, const void* wh, double lipschitz, void* cand,
                 void* stream);
/* K2a + K2b: it < 0 = set-up (row DCT-II of r0 only; rho_s of r0 came with
 * pu_pcg_begin); else x += alpha p, r -= alpha A p
 * (submean: after pu_pcg_update_sum, r_u -= mean instead), ||r||, rho_s;
 * then the row DCT-II of r_u into spec_out (packed in band mode). */
int pu_pcg_residual_rows(pu_handle* h, const void* p, const void* dv, const void* dh, void* x, void* r, void* ctrl,
                         double* res_norms, void* spec_out, int it, int submean, void* stream);
/* pcg.py:90-93 on every 50th iteration: update and sum(r_u). */
int pu_pcg_update_sum(pu_handle* h, const void* p, const void* dv, const void* dh, void* x, void* r, void* ctrl,
                      int it, void* stream);
/* K3: column DCT-II, spectral division, rho_u, column DCT-III, in place
 * (it < 0: set-up). */
int pu_pcg_columns(pu_handle* h, void* spec, void* ctrl, int it, void* stream);
/* K4: pnew_u = beta pold_u + row DCT-III(spec_in) (first: no axpy). */
int pu_pcg_rows_inv(pu_handle* h, const void* spec_in, void* pnew, const void* pold, int first, void* ctrl, int it,
                    void* stream);
/* K1: slack blocks of the new direction (+ the ghost row in band mode), A p,
 * p'Ap. */
int pu_pcg_direction(pu_handle* h, const void* r, const void* pold, void* pnew, const void* dv, const void* dh,
                     void* ctrl, int it, void* stream);

/* ------------------------------------------------------------------------
 * The whole unwrap behind one call, for hosts that bind C (cgo, JNI,
 * N-API, ctypes) instead of running the Python mirror of irls.py:
 * reference `unwrap(x, c, model, params, gradient_lo) -> UnwrapResult`
 * (irls.py:132-224, re-exported at __init__.py:4).  Host arrays in and out;
 * the IRLS outer loop (weights, H pair, CG-budget rule irls.py:111-129,
 * warm-started PCG, safeguard, centring, trace) runs in C++ over the entry
 * points above, on its own handle and stream, so concurrent calls are safe
 * (SPEC.md:391, 453-454).
 * ------------------------------------------------------------------------ */
typedef struct pu_irls_params {   /* irls.py:43-64 IrlsParams (same defaults) */
  int32_t max_iter_cg_start;      /* 5 */
  int32_t max_outer_iters;        /* 100 */
  int32_t max_cg_iters_cap;       /* 10000 */
  int32_t pad_;
  double rel_improvement_tol;     /* 1e-3 */
  double cg_growth_factor;        /* 1.7 */
  double cg_rel_tol;              /* 1e-10 */
} pu_irls_params;

typedef struct pu_iteration_record {  /* irls.py:67-75 IterationRecord */
  int32_t k, m_cg, cg_iters;
  int32_t has_delta_rel;              /* 0: delta_rel is None (k = 0) */
  double delta_rel, h_delta;
  int32_t sufficient_decrease, fallback_used;
} pu_iteration_record;

/* Fill *p with the IrlsParams defaults. */
void pu_irls_params_default(pu_irls_params* p);

/* Unwrap a wrapped phase grid.
 *  x          host fp64, n x m row-major, every value finite and in [0, 2pi)
 *             (phase.py:100-115);
 *  cv, ch     host fp64 arc weights, (n-1) x m and n x (m-1), finite, >= 0,
 *             not all zero (phase.py:54-73); both NULL = uniform unit weights;
 *  tau, delta ModelParams (objective.py:30-41); params NULL = defaults;
 *  gradient_lo 0 or -pi (phase.py:140-149);  dtype PU_F64 (the reference's
 *             precision) or PU_F32;  device: CUDA ordinal;
 *  u, vv, vh  host fp64 outputs, n x m, (n-1) x m, n x (m-1), mean(u) = 0;
 *  trace      up to trace_cap records; *trace_len = records written (the
 *             full count is returned even when it exceeds trace_cap).
 * Returns PU_OK; PU_ERR_ARG for what the reference rejects with ValueError
 * (checked before any device work); PU_ERR_BREAKDOWN with
 * *breakdown_iteration = NumericalBreakdown.iteration; PU_ERR_UNSUPPORTED /
 * PU_ERR_CUDA / PU_ERR_NOMEM otherwise.  pu_last_error() has the message. */
int pu_unwrap(const double* x, int n, int m, const double* cv, const double* ch, double tau, double delta,
              const pu_irls_params* params, double gradient_lo, int dtype, int device, double* u, double* vv,
              double* vh, pu_iteration_record* trace, int trace_cap, int* trace_len, int* breakdown_iteration);

/* ------------------------------------------------------------------------
 * GPU synthetic scenes (reference synth.py:43-109):
 * the per-pixel work of the reference's scene recipes, for large benchmark
 * inputs.  Parameters (bump centres/widths/peaks, fault seam) are drawn on
 * the host from the reference's Philox stream (synth_gpu.py).  Plateau,
 * fault mask and wrapping are exact; bumps agree with the host generator to
 * ~1e-15 (device exp); the phase noise is a device Philox-4x32 / Box-Muller
 * stream (statistically equivalent, not numpy's realisation).  Device fp64
 * arrays, row pitch ld.
 * ------------------------------------------------------------------------ */
/* out = sum_b params[4b+3] exp(-((i - params[4b])^2 + (j - params[4b+1])^2) / (2 params[4b+2]^2)) */
int pu_synth_bumps(double* out, int rows, int cols, int64_t ld, const double* params, int count, void* stream);
/* out += lin[i] * amplitude * (j >= seam[i])  (plateau-discontinuity, tapered fault) */
int pu_synth_fault(double* out, int rows, int cols, int64_t ld, const int64_t* seam, const double* lin,
                   double amplitude, void* stream);
/* x = wrap_to_principal(x + sigma * N(0,1), 0) (sigma = 0: wrap only) */
int pu_synth_wrap_noise(double* x, int rows, int cols, int64_t ld, double sigma, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PU_UNWRAP_H */
