// Device kernels of the B200 phase unwrapper (sm_100a).
//
// Reference correspondence (paths relative to phaseirls/):
//   k_grad            phase.py:118-149 + kernels.py:87-103   wrapped gradients
//   k_rhs             operators.py:156-162                   right-hand side b
//   k_apply_system    operators.py:138-153, kernels.py:125-145  3-block map A
//   k_dot             operators.py:70-75                     SystemVector.dot
//   k_weights_hpair   objective.py:92-100 + :77-89, irls.py:173-191
//   k_hpair_states    objective.py:77-89 (x2), irls.py:202-205
//   k_candidate       objective.py:108-125
//   k_accept          irls.py:206-215 (select, centre, H of the accepted)
//   k_eval_f          objective.py:63-66
//   k_pcg_*           pcg.py:47-116 with preconditioner.py:86-115 fused in
#pragma once

#include "pu_common.cuh"
#include "pu_fft.cuh"
#include "pu_fin.cuh"

namespace pu {

// ---------------------------------------------------------------------------
// correctly rounded helpers (no FMA contraction) where the reference's
// rounding sequence is mirrored
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

#define PU_TWO_PI 6.283185307179586

// Element loop over the valid N x M cells: thread-strided columns, block-strided rows.
#define PU_FOR_CELLS(g, i, j)                                                        \
  for (int i = blockIdx.x; i < (g).n; i += gridDim.x)                                 \
    for (int j = threadIdx.x; j < (g).m; j += blockDim.x)

// ---------------------------------------------------------------------------
// Stencil sources and the fused 3-block system map at one cell.
// ---------------------------------------------------------------------------
template <typename T>
struct PlainSrc {
  const T* u; const T* v; const T* h;
  __device__ __forceinline__ T U(long long o) const { return u[o]; }
  __device__ __forceinline__ T V(long long o) const { return v[o]; }
  __device__ __forceinline__ T H(long long o) const { return h[o]; }
};

// p_new = beta * p_old + z   (pcg.py:107-108: p.scale(beta); p.add(z)), or z at it = 0
template <typename T>
struct PUpdSrc {
  const T* z; const T* p; long long plane; T beta; bool first;
  __device__ __forceinline__ T at(long long o) const {
    const T zz = z[o];
    return first ? zz : add_rn(mul_rn(beta, p[o]), zz);
  }
  __device__ __forceinline__ T U(long long o) const { return at(o); }
  __device__ __forceinline__ T V(long long o) const { return at(o + plane); }
  __device__ __forceinline__ T H(long long o) const { return at(o + 2 * plane); }
};

// y = A x at cell (i, j); also returns x at the cell.  Pad entries of x are
// zero by the layout invariant, so the vv/vh pads read as 0.
template <typename T, typename Src>
__device__ __forceinline__ void sys_at(const Grid& g, const Src& s, const T* __restrict__ dv,
                                       const T* __restrict__ dh, int i, int j, T& xu, T& xv, T& xh,
                                       T& au, T& av, T& ah) {
  const long long o = (long long)i * g.ld + j;
  const T inv = (T)g.inv_tau;
  xu = s.U(o);
  xv = s.V(o);
  xh = s.H(o);
  T su = 0, rv = 0, rvm = 0, ut = 0, rh = 0, rhm = 0;
  const bool hasv = dn_ok(g, i), hash = j < g.m - 1;
  if (hasv) { su = s.U(o + g.ld) - xu; rv = su - xv; }
  if (up_ok(g, i)) { rvm = (xu - s.U(o - g.ld)) - s.V(o - g.ld); }
  if (hash) { ut = s.U(o + 1) - xu; rh = ut - xh; }
  if (j > 0) { rhm = (xu - s.U(o - 1)) - s.H(o - 1); }
  au = inv * ((rvm - rv) + (rhm - rh));
  av = hasv ? dv[o] * xv + inv * (xv - su) : (T)0;
  ah = hash ? dh[o] * xh + inv * (xh - ut) : (T)0;
}

// ---------------------------------------------------------------------------
// Input stage
// ---------------------------------------------------------------------------
__device__ __forceinline__ double wrap_lo(double a, double lo) {
  // phase.py:130-134 without FMA contraction so results are bit-identical
  const double k = floor(__ddiv_rn(__dsub_rn(a, lo), PU_TWO_PI));
  double y = __dsub_rn(a, __dmul_rn(PU_TWO_PI, k));
  const double hi = __dadd_rn(lo, PU_TWO_PI);
  if (y >= hi) y = __dsub_rn(y, PU_TWO_PI);
  if (y < lo) y = __dadd_rn(y, PU_TWO_PI);
  return y;
}

template <typename T>
__global__ void k_grad(Grid g, const double* __restrict__ x, long long ldx, T* gv, T* gh, double lo) {
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    const double xij = x[(long long)i * ldx + j];
    gv[o] = dn_ok(g, i) ? (T)wrap_lo(__dsub_rn(x[(long long)(i + 1) * ldx + j], xij), lo) : (T)0;
    gh[o] = (j < g.m - 1) ? (T)wrap_lo(__dsub_rn(x[(long long)i * ldx + j + 1], xij), lo) : (T)0;
  }
}

// k_grad + the input check of phase.py:100-115 from the same loads:
// out[0] = number of non-finite x, out[1] = number of finite x outside
// [0, 2 pi).  The host raises ValueError on the first scalar read.
template <typename T>
__global__ void k_grad_check(Grid g, const double* __restrict__ x, long long ldx, T* gv, T* gh, double lo,
                             RedScratch rs, int site, double* out) {
  double acc[2] = {0.0, 0.0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    const double xij = x[(long long)i * ldx + j];
    if (!isfinite(xij)) acc[0] += 1.0;
    else if (xij < 0.0 || xij >= PU_TWO_PI) acc[1] += 1.0;
    gv[o] = dn_ok(g, i) ? (T)wrap_lo(__dsub_rn(x[(long long)(i + 1) * ldx + j], xij), lo) : (T)0;
    gh[o] = (j < g.m - 1) ? (T)wrap_lo(__dsub_rn(x[(long long)i * ldx + j + 1], xij), lo) : (T)0;
  }
  double tot[2];
  if (grid_reduce<2>(acc, rs, site, tot) && threadIdx.x == 0) {
    out[0] = tot[0];
    out[1] = tot[1];
  }
}

// irls.py:167 — initial state (u, vv, vh) = (0, -gv, -gh)
template <typename T>
__global__ void k_init_state(Grid g, const T* __restrict__ gv, const T* __restrict__ gh, T* x) {
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    x[o] = (T)0;
    x[o + g.plane] = dn_ok(g, i) ? -gv[o] : (T)0;
    x[o + 2 * g.plane] = (j < g.m - 1) ? -gh[o] : (T)0;
  }
}

template <typename T>
__global__ void k_rhs(Grid g, const T* __restrict__ gv, const T* __restrict__ gh, T* b) {
  const T inv = (T)g.inv_tau;
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    const T gvo = dn_ok(g, i) ? gv[o] : (T)0, gvm = up_ok(g, i) ? gv[o - g.ld] : (T)0;
    const T gho = (j < g.m - 1) ? gh[o] : (T)0, ghm = (j > 0) ? gh[o - 1] : (T)0;
    b[o] = inv * ((gvm - gvo) + (ghm - gho));
    b[o + g.plane] = -inv * gvo;
    b[o + 2 * g.plane] = -inv * gho;
  }
}

// compact fp64 (rows x cols, pitch lds) <-> padded plane; the region of the
// plane outside rows x cols but inside n x m is zeroed.
template <typename T>
__global__ void k_pack(Grid g, const double* __restrict__ src, long long lds, int rows, int cols, T* dst) {
  PU_FOR_CELLS(g, i, j) {
    dst[(long long)i * g.ld + j] = (i < rows && j < cols) ? (T)src[(long long)i * lds + j] : (T)0;
  }
}

template <typename T, typename D>
__global__ void k_unpack(Grid g, const T* __restrict__ src, int rows, int cols, D* dst) {
  for (int i = blockIdx.x; i < rows; i += gridDim.x)
    for (int j = threadIdx.x; j < cols; j += blockDim.x)
      dst[(long long)i * cols + j] = (D)src[(long long)i * g.ld + j];
}

template <typename T>
__global__ void k_fill(Grid g, T* dst, int nplanes, T val) {
  for (int pl = 0; pl < nplanes; ++pl)
    PU_FOR_CELLS(g, i, j) dst[pl * g.plane + (long long)i * g.ld + j] = val;
}

template <typename T>
__global__ void k_copy(Grid g, const T* __restrict__ src, T* dst, int nplanes) {
  for (int pl = 0; pl < nplanes; ++pl)
    PU_FOR_CELLS(g, i, j) {
      const long long o = pl * g.plane + (long long)i * g.ld + j;
      dst[o] = src[o];
    }
}

// ---------------------------------------------------------------------------
// System map, dot products
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_apply_system(Grid g, const T* __restrict__ x, const T* __restrict__ dv,
                               const T* __restrict__ dh, T* y) {
  PlainSrc<T> s{x, x + g.plane, x + 2 * g.plane};
  PU_FOR_CELLS(g, i, j) {
    T xu, xv, xh, au, av, ah;
    sys_at<T>(g, s, dv, dh, i, j, xu, xv, xh, au, av, ah);
    const long long o = (long long)i * g.ld + j;
    y[o] = au;
    y[o + g.plane] = av;
    y[o + 2 * g.plane] = ah;
  }
}

template <typename T>
__global__ void k_dot(Grid g, const T* __restrict__ a, const T* __restrict__ b, int nplanes,
                      RedScratch rs, int site, double* out) {
  double acc[1] = {0.0};
  for (int pl = 0; pl < nplanes; ++pl)
    PU_FOR_CELLS(g, i, j) {
      const long long o = pl * g.plane + (long long)i * g.ld + j;
      acc[0] += (double)a[o] * (double)b[o];
    }
  double tot[1];
  if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0) out[0] = tot[0];
}

// ---------------------------------------------------------------------------
// Objective pieces.  The slack term of H_delta for one arc is
//   0.5 * (((c v)^2 + delta^2) / w + w)        (objective.py:86-88)
// and the penalty squares (S u - g - v)^2 enter as sum / (2 tau) (:52-55).
// All per-cell terms are formed in fp64 from the stored values.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double slack_term(double c, double v, double w, double d2) {
  const double cv = c * v;
  return (cv * cv + d2) / w + w;
}

// penalty residuals at (i, j) for state (u, vv, vh) with gradients (gv, gh)
template <typename T>
__device__ __forceinline__ void pen_at(const Grid& g, const T* u, const T* vv, const T* vh, const T* gv,
                                       const T* gh, int i, int j, double ushift, double& rv, double& rh) {
  const long long o = (long long)i * g.ld + j;
  rv = 0.0; rh = 0.0;
  const double uo = (double)u[o] - ushift;
  if (dn_ok(g, i)) rv = (((double)u[o + g.ld] - ushift) - uo) - (double)gv[o] - (double)vv[o];
  if (j < g.m - 1) rh = (((double)u[o + 1] - ushift) - uo) - (double)gh[o] - (double)vh[o];
}

// Weight refresh w = sqrt((c v)^2 + delta^2), d = c^2 / w (irls.py:173, 191)
// plus H_delta(state, w_prev) and H_delta(state, w) (irls.py:176-177).
// out[0] = H(x, w_prev) (when wp != nullptr), out[1] = H(x, w).
template <typename T>
__global__ void k_weights_hpair(Grid g, const T* __restrict__ x, const T* __restrict__ cv,
                                const T* __restrict__ ch, const T* __restrict__ gv, const T* __restrict__ gh,
                                const T* __restrict__ wpv, const T* __restrict__ wph, T* wv, T* wh, T* dv,
                                T* dh, RedScratch rs, int site, double* out) {
  const double d2 = g.delta * g.delta;
  const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
  // acc: [old_v, old_h, new_v, new_h, pen_v, pen_h]
  double acc[6] = {0, 0, 0, 0, 0, 0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    if (dn_ok(g, i)) {
      const T c = cv[o], v = vv[o];
      const T cvt = c * v;
      const T w = sqrt(cvt * cvt + (T)d2);
      wv[o] = w;
      dv[o] = c * c / w;
      acc[2] += slack_term((double)c, (double)v, (double)w, d2);
      if (wpv) acc[0] += slack_term((double)c, (double)v, (double)wpv[o], d2);
    } else {
      wv[o] = (T)1; dv[o] = (T)0;
    }
    if (j < g.m - 1) {
      const T c = ch[o], v = vh[o];
      const T cvt = c * v;
      const T w = sqrt(cvt * cvt + (T)d2);
      wh[o] = w;
      dh[o] = c * c / w;
      acc[3] += slack_term((double)c, (double)v, (double)w, d2);
      if (wph) acc[1] += slack_term((double)c, (double)v, (double)wph[o], d2);
    } else {
      wh[o] = (T)1; dh[o] = (T)0;
    }
    double rv, rh;
    pen_at<T>(g, u, vv, vh, gv, gh, i, j, 0.0, rv, rh);
    acc[4] += rv * rv;
    acc[5] += rh * rh;
  }
  double tot[6];
  if (grid_reduce<6>(acc, rs, site, tot) && threadIdx.x == 0) {
    const double pen = (tot[4] + tot[5]) / (2.0 * g.tau);
    out[0] = (0.5 * tot[0] + 0.5 * tot[1]) + pen;
    out[1] = (0.5 * tot[2] + 0.5 * tot[3]) + pen;
  }
}

// H_delta of an arbitrary state with given weights (objective.py:77-89).
template <typename T>
__global__ void k_eval_h(Grid g, const T* __restrict__ x, const T* __restrict__ wv, const T* __restrict__ wh,
                         const T* __restrict__ gv, const T* __restrict__ gh, const T* __restrict__ cv,
                         const T* __restrict__ ch, RedScratch rs, int site, double* out) {
  const double d2 = g.delta * g.delta;
  const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
  double acc[4] = {0, 0, 0, 0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    if (dn_ok(g, i)) acc[0] += slack_term((double)cv[o], (double)vv[o], (double)wv[o], d2);
    if (j < g.m - 1) acc[1] += slack_term((double)ch[o], (double)vh[o], (double)wh[o], d2);
    double rv, rh;
    pen_at<T>(g, u, vv, vh, gv, gh, i, j, 0.0, rv, rh);
    acc[2] += rv * rv;
    acc[3] += rh * rh;
  }
  double tot[4];
  if (grid_reduce<4>(acc, rs, site, tot) && threadIdx.x == 0)
    out[0] = (0.5 * tot[0] + 0.5 * tot[1]) + (tot[2] + tot[3]) / (2.0 * g.tau);
}

// H_delta(proposal, w) and H_delta(cand, w) plus both u sums (irls.py:202-208).
// out[0] = H(a), out[1] = H(b), out[2] = mean u of the accepted one,
// out[3] = 1.0 if a is accepted (sufficient decrease) else 0.0.
template <typename T>
__global__ void k_hpair_states(Grid g, const T* __restrict__ xa, const T* __restrict__ xb,
                               const T* __restrict__ wv, const T* __restrict__ wh, const T* __restrict__ gv,
                               const T* __restrict__ gh, const T* __restrict__ cv, const T* __restrict__ ch,
                               RedScratch rs, int site, double* out) {
  const double d2 = g.delta * g.delta;
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const T* x = s ? xb : xa;
      const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
      if (dn_ok(g, i)) acc[5 * s + 0] += slack_term((double)cv[o], (double)vv[o], (double)wv[o], d2);
      if (j < g.m - 1) acc[5 * s + 1] += slack_term((double)ch[o], (double)vh[o], (double)wh[o], d2);
      double rv, rh;
      pen_at<T>(g, u, vv, vh, gv, gh, i, j, 0.0, rv, rh);
      acc[5 * s + 2] += rv * rv;
      acc[5 * s + 3] += rh * rh;
      acc[5 * s + 4] += (double)u[o];
    }
  }
  double tot[10];
  if (grid_reduce<10>(acc, rs, site, tot) && threadIdx.x == 0) {
    const double ha = (0.5 * tot[0] + 0.5 * tot[1]) + (tot[2] + tot[3]) / (2.0 * g.tau);
    const double hb = (0.5 * tot[5] + 0.5 * tot[6]) + (tot[7] + tot[8]) / (2.0 * g.tau);
    const bool take_a = ha <= hb;
    out[0] = ha;
    out[1] = hb;
    out[2] = (take_a ? tot[4] : tot[9]) / ((double)g.n_glob * (double)g.m);
    out[3] = take_a ? 1.0 : 0.0;
  }
}

// Explicit gradient step cand = x - (1/L) grad H(x, w) (objective.py:108-125).
template <typename T>
__global__ void k_candidate(Grid g, const T* __restrict__ x, const T* __restrict__ wv, const T* __restrict__ wh,
                            const T* __restrict__ gv, const T* __restrict__ gh, const T* __restrict__ cv,
                            const T* __restrict__ ch, T neg_inv_lip, T* out) {
  const T inv = (T)g.inv_tau;
  const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    const bool hasv = dn_ok(g, i), hash = j < g.m - 1;
    const T uo = u[o];
    T rv = 0, rvm = 0, rh = 0, rhm = 0;
    if (hasv) rv = ((u[o + g.ld] - uo) - gv[o]) - vv[o];
    if (up_ok(g, i)) rvm = ((uo - u[o - g.ld]) - gv[o - g.ld]) - vv[o - g.ld];
    if (hash) rh = ((u[o + 1] - uo) - gh[o]) - vh[o];
    if (j > 0) rhm = ((uo - u[o - 1]) - gh[o - 1]) - vh[o - 1];
    const T gu = inv * ((rvm - rv) + (rhm - rh));
    out[o] = add_rn(uo, mul_rn(neg_inv_lip, gu));
    if (hasv) {
      const T c = cv[o], v = vv[o];
      const T gvv = c * c / wv[o] * v - inv * rv;
      out[o + g.plane] = add_rn(v, mul_rn(neg_inv_lip, gvv));
    } else {
      out[o + g.plane] = (T)0;
    }
    if (hash) {
      const T c = ch[o], v = vh[o];
      const T gvh = c * c / wh[o] * v - inv * rh;
      out[o + 2 * g.plane] = add_rn(v, mul_rn(neg_inv_lip, gvh));
    } else {
      out[o + 2 * g.plane] = (T)0;
    }
  }
}

// accepted = (flag ? a : b); accepted.u -= mean; out[0] = H(accepted, w)
// (irls.py:206-215).  `sel` points at k_hpair_states' out[2..3].
template <typename T>
__global__ void k_accept(Grid g, const T* __restrict__ xa, const T* __restrict__ xb, const double* sel,
                         T* dst, const T* __restrict__ wv, const T* __restrict__ wh, const T* __restrict__ gv,
                         const T* __restrict__ gh, const T* __restrict__ cv, const T* __restrict__ ch,
                         RedScratch rs, int site, double* out) {
  const double mean = sel[0];
  const T* x = sel[1] != 0.0 ? xa : xb;
  const T tmean = (T)mean;
  const double d2 = g.delta * g.delta;
  const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
  double acc[4] = {0, 0, 0, 0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    const T uo = u[o] - tmean;
    double rv = 0.0, rh = 0.0;
    if (dn_ok(g, i)) {
      const T un = u[o + g.ld] - tmean;
      rv = ((double)un - (double)uo) - (double)gv[o] - (double)vv[o];
      acc[0] += slack_term((double)cv[o], (double)vv[o], (double)wv[o], d2);
    }
    if (j < g.m - 1) {
      const T un = u[o + 1] - tmean;
      rh = ((double)un - (double)uo) - (double)gh[o] - (double)vh[o];
      acc[1] += slack_term((double)ch[o], (double)vh[o], (double)wh[o], d2);
    }
    acc[2] += rv * rv;
    acc[3] += rh * rh;
    dst[o] = uo;  // dst never aliases xa / xb (neighbour reads above)
    dst[o + g.plane] = vv[o];
    dst[o + 2 * g.plane] = vh[o];
  }
  double tot[4];
  if (grid_reduce<4>(acc, rs, site, tot) && threadIdx.x == 0)
    out[0] = (0.5 * tot[0] + 0.5 * tot[1]) + (tot[2] + tot[3]) / (2.0 * g.tau);
}

// ---------------------------------------------------------------------------
// Harness metrics on the device (phase.py:152-184; SURVEY §8(d) parity
// metrics), against fp64 grids with row pitch ldx, so large results need no
// device-to-host copy.
// ---------------------------------------------------------------------------
// shift_error pass 1: alpha = mean(x_u - u); clears the max slot
template <typename T>
__global__ void k_shift_alpha(Grid g, const T* __restrict__ u, const double* __restrict__ xu, long long ldx,
                              RedScratch rs, int site, double* out) {
  double acc[1] = {0.0};
  PU_FOR_CELLS(g, i, j) acc[0] += xu[(long long)i * ldx + j] - (double)u[(long long)i * g.ld + j];
  double tot[1];
  if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0) {
    out[0] = tot[0] / ((double)g.n * (double)g.m);
    out[1] = 0.0;
  }
}

// shift_error pass 2: err = x_u - (u + alpha); out[1] = max |err|, out[2] =
// rmse, out[3] = fraction of cells within 1e-3 cycles of a multiple of 2 pi
template <typename T>
__global__ void k_shift_stats(Grid g, const T* __restrict__ u, const double* __restrict__ xu, long long ldx,
                              RedScratch rs, int site, double* out) {
  const double alpha = out[0];
  double acc[2] = {0.0, 0.0};
  double mx = 0.0;
  PU_FOR_CELLS(g, i, j) {
    const double err = xu[(long long)i * ldx + j] - ((double)u[(long long)i * g.ld + j] + alpha);
    const double cyc = err / PU_TWO_PI;
    acc[0] += err * err;
    acc[1] += fabs(cyc - rint(cyc)) <= 1e-3 ? 1.0 : 0.0;
    mx = fmax(mx, fabs(err));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  // non-negative doubles order like their bit patterns: an integer max is exact
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(mx));
  double tot[2];
  if (grid_reduce<2>(acc, rs, site, tot) && threadIdx.x == 0) {
    const double cells = (double)g.n * (double)g.m;
    out[2] = sqrt(tot[0] / cells);
    out[3] = tot[1] / cells;
  }
}

// K-map mismatch fraction: mean(rint((u - x)/2pi) != rint((u_ref - x)/2pi))
template <typename T>
__global__ void k_kmap(Grid g, const T* __restrict__ u, const double* __restrict__ uref, long long ldr,
                       const double* __restrict__ x, long long ldx, RedScratch rs, int site, double* out) {
  double acc[1] = {0.0};
  PU_FOR_CELLS(g, i, j) {
    const double xi = x[(long long)i * ldx + j];
    const double ka = rint(((double)u[(long long)i * g.ld + j] - xi) / PU_TWO_PI);
    const double kb = rint((uref[(long long)i * ldr + j] - xi) / PU_TWO_PI);
    acc[0] += ka != kb ? 1.0 : 0.0;
  }
  double tot[1];
  if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0) out[0] = tot[0] / ((double)g.n * (double)g.m);
}

// congruent_round: out = x + 2pi rint((u - x)/2pi), compact fp64 (pitch m)
template <typename T>
__global__ void k_congruent(Grid g, const T* __restrict__ u, const double* __restrict__ x, long long ldx,
                            double* __restrict__ out) {
  PU_FOR_CELLS(g, i, j) {
    const double xi = x[(long long)i * ldx + j];
    out[(long long)i * g.m + j] = xi + PU_TWO_PI * rint(((double)u[(long long)i * g.ld + j] - xi) / PU_TWO_PI);
  }
}

// F = sum |c v| + penalties (objective.py:63-66); out[1] = l1 part.
template <typename T>
__global__ void k_eval_f(Grid g, const T* __restrict__ x, const T* __restrict__ gv, const T* __restrict__ gh,
                         const T* __restrict__ cv, const T* __restrict__ ch, RedScratch rs, int site, double* out) {
  const T* u = x; const T* vv = x + g.plane; const T* vh = x + 2 * g.plane;
  double acc[4] = {0, 0, 0, 0};
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    if (dn_ok(g, i)) acc[0] += fabs((double)cv[o] * (double)vv[o]);
    if (j < g.m - 1) acc[1] += fabs((double)ch[o] * (double)vh[o]);
    double rv, rh;
    pen_at<T>(g, u, vv, vh, gv, gh, i, j, 0.0, rv, rh);
    acc[2] += rv * rv;
    acc[3] += rh * rh;
  }
  double tot[4];
  if (grid_reduce<4>(acc, rs, site, tot) && threadIdx.x == 0) {
    out[1] = tot[0] + tot[1];
    out[0] = out[1] + (tot[2] + tot[3]) / (2.0 * g.tau);
  }
}

}  // namespace pu
