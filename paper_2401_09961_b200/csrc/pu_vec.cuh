// Vectorised element-wise PCG kernels (sm_100a).
//
// Each thread owns a chunk of 4 consecutive cells of one row and moves every
// plane as one 16-byte (fp32) or two 16-byte (fp64) accesses, so a warp keeps
// ~20 independent loads in flight instead of one scalar chain per cell.  Pitch
// padding (j >= m) is read as zero and written back as zero.
//
//   k_pcg_p_v     K1: slack p_s <- beta p_s + r_s / (d + 1/tau) (p_u came from
//                 K4); p'Ap as the quadratic form of A; alpha (pcg.py:82-89)
//   k_pcg_r_v     K2a: x += alpha p; r -= alpha A p; optional mean re-projection;
//                 ||r||; rho_s = <r_s, r_s / (d + 1/tau)> (pcg.py:90-104,
//                 preconditioner.py:115); the row DCT of r_u runs next (K2b)
//   k_pcg_start_v x = x0, r = b - A x0, ||b||, ||r0||, rho_s of r0 (pcg.py:59-79),
//                 optionally fused with the candidate step (objective.py:118-125)
#pragma once

#include "pu_kernels.cuh"
#include "pu_q4.cuh"
#include "pu_fft.cuh"

// resident CTAs per SM the element-wise kernels are compiled for: the fp32
// budget in fp32; 2 (128 registers) in fp64, where the fp32 budgets spill
#define PU_MINB(T, N) (sizeof(T) == 4 ? (N) : 2)
// fp64 once-per-outer-iteration kernels (H pair, acceptance, start-up): 2
// CTAs/SM (128 registers, ~150-200 B of spills) by default; PU_OUTER64_MINB=1
// builds them at 1 CTA/SM without spills (A/B, the way k_accept_start_v
// won: 0.70 vs 0.865 ms)
#ifndef PU_OUTER64_MINB
#define PU_OUTER64_MINB 2
#endif
#define PU_MINB_OUTER(T, N) (sizeof(T) == 4 ? (N) : PU_OUTER64_MINB)
#ifndef PU_F64_RSQRT_W
#define PU_F64_RSQRT_W 1
#endif

namespace pu {

// chunk loop: chunk q covers cells (i, 4c .. 4c+3), c < cpr = ceil(m / 4)
#define PU_FOR_CHUNKS(g, i, j0)                                                            \
  for (long long q_ = (long long)blockIdx.x * blockDim.x + threadIdx.x,                   \
                 cpr_ = ((g).m + 3) / 4, nq_ = (long long)(g).n * cpr_;                  \
       q_ < nq_; q_ += (long long)gridDim.x * blockDim.x)                                   \
    for (int i = (int)(q_ / cpr_), j0 = (int)(q_ - (long long)i * cpr_) * 4, once_ = 1; once_; once_ = 0)

// A x at the 4 cells of a chunk given the chunk's x (centre, above, below,
// left/right neighbours).  ok[k]: cell exists (j < m).
template <typename T>
struct Stencil4 {
  Q4<T> u, v, h;      // x at (i, j0..j0+3)
  Q4<T> ua, va;       // x_u, x_v at (i-1, .) (zero if i == 0)
  Q4<T> ub;           // x_u at (i+1, .)      (zero if i == n-1)
  T ul, ur, hl;       // x_u at (i, j0-1), (i, j0+4); x_h at (i, j0-1)
};

template <typename T>
__device__ __forceinline__ void apply4(const Grid& g, int i, int j0, const Stencil4<T>& s, const Q4<T>& dv,
                                       const Q4<T>& dh, Q4<T>& au, Q4<T>& av, Q4<T>& ah) {
  const T inv = (T)g.inv_tau;
  const bool hasv = dn_ok(g, i), hasa = up_ok(g, i);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    const T xu = s.u.a[k];
    const T left = (k == 0) ? s.ul : s.u.a[k - 1];
    const T right = (k == 3) ? s.ur : s.u.a[k + 1];
    const T hleft = (k == 0) ? s.hl : s.h.a[k - 1];
    T su = 0, rv = 0, rvm = 0, ut = 0, rh = 0, rhm = 0;
    const bool hash = j < g.m - 1;
    if (hasv) { su = s.ub.a[k] - xu; rv = su - s.v.a[k]; }
    if (hasa) { rvm = (xu - s.ua.a[k]) - s.va.a[k]; }
    if (hash) { ut = right - xu; rh = ut - s.h.a[k]; }
    if (j > 0) { rhm = (xu - left) - hleft; }
    const bool ok = j < g.m;
    au.a[k] = ok ? inv * ((rvm - rv) + (rhm - rh)) : (T)0;
    av.a[k] = (ok && hasv) ? dv.a[k] * s.v.a[k] + inv * (s.v.a[k] - su) : (T)0;
    ah.a[k] = (ok && hash) ? dh.a[k] * s.h.a[k] + inv * (s.h.a[k] - ut) : (T)0;
  }
}

// slack block of the preconditioner, z = r / (d + 1/tau) (preconditioner.py:115):
// fast division in fp32 mode (K1 and K2a use the same expression, so rho and
// p stay consistent), IEEE division in fp64 mode (parity with the reference)
__device__ __forceinline__ float slack_div(float a, float b) { return a * rcp_approx(b); }
__device__ __forceinline__ double slack_div(double a, double b) { return a / b; }
// K1's slack preconditioner and the H-pair slack terms in fp64: reciprocal
// seed + two Newton steps (<= 1 ulp) instead of the IEEE division.  Measured
// (profiles/r02_ab_f64div.txt): K1 214 -> 186.5 us (the kernel then streams
// at the HBM peak); in K2a the same change was 3% slower, so K2a keeps the
// IEEE division for rho_s (the two z_s differ by at most 1 ulp).
__device__ __forceinline__ float slack_div_p(float a, float b) { return slack_div(a, b); }
__device__ __forceinline__ double slack_div_p(double a, double b) { return a * rcp_nr(b); }

// scalar neighbour load that tolerates the grid edge
template <typename T>
__device__ __forceinline__ T ldg_or0(const T* p, bool ok) { return ok ? __ldg(p) : (T)0; }

// slack block of the new search direction at 4 cells of row i (plane offset
// po, diagonal d), masked to valid arcs: beta p_old + r / (d + 1/tau)
template <typename T>
__device__ __forceinline__ Q4<T> pslack4(const Grid& g, const T* __restrict__ r, const T* __restrict__ pold,
                                         const T* __restrict__ d, long long o, long long po, int i, int j0,
                                         bool vert, T beta, bool first) {
  const T inv = (T)g.inv_tau;
  const Q4<T> rr = ldg4(r + o + po), dd = ldg4(d + o);
  Q4<T> out;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    const bool ok = vert ? (dn_ok(g, i) && j < g.m) : (j < g.m - 1);
    out.a[k] = ok ? slack_div_p(rr.a[k], dd.a[k] + inv) : (T)0;
  }
  if (!first) {
    const Q4<T> pp = ldg4(pold + o + po);
#pragma unroll
    for (int k = 0; k < 4; ++k) out.a[k] = add_rn(mul_rn(beta, pp.a[k]), out.a[k]);
  }
  return out;
}

// Band mode, before K1: the vv slack of the new direction in the ghost row -1
// (the band above owns it; recomputed here from the mirrored r_vv, p_vv, dv
// rows with K1's arithmetic, so K2a's stencil sees the same value)
template <typename T>
__global__ void k_ghost_pslack(Grid g, const T* __restrict__ r, const T* __restrict__ pold, T* __restrict__ pnew,
                               const T* __restrict__ dv, const PcgCtrl* ctrl, int it) {
  if (ctrl->done || !g.top) return;
  const T beta = (T)ctrl->beta;
  for (int j0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x); j0 < g.m; j0 += 4 * gridDim.x * blockDim.x) {
    const long long o = -g.ld + j0;
    st4(pnew + o + g.plane, pslack4<T>(g, r, pold, dv, o, g.plane, -1, j0, true, beta, it == 0));
  }
}

// ---------------------------------------------------------------------------
// K1.  The u block of the new search direction, p_u = beta p_u_old + z_u, was
// already written by the row DCT-III kernel (K4) of the previous iteration;
// here the slack blocks follow: z_s = r_s / (d + 1/tau) (never stored) and
// p_s = beta p_s_old + z_s (z_s at it = 0).  Then p'Ap of the new p from the
// forward differences only (pcg.py:82-89, 102-108).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void pcg_p_body(const Grid& g, const T* __restrict__ r, const T* __restrict__ pold,
                                           T* __restrict__ pnew, const T* __restrict__ dv, const T* __restrict__ dh,
                                           PcgCtrl* ctrl, const RedScratch& rs, int site, int it) {
  pdl_enter(g);
  if (ctrl->done) return;
  const bool first = it == 0;
  const T beta = (T)ctrl->beta;
  const T inv = (T)g.inv_tau;
  const long long P = g.plane, ld = g.ld;
  auto ps4 = [&](long long o, long long po, const T* d, int i, int j0, bool vert) -> Q4<T> {
    return pslack4<T>(g, r, pold, d, o, po, i, j0, vert, beta, first);
  };
  // p'Ap as the quadratic form of A (operators.py:138-153): with
  // rv = S p_u - p_vv and rh = p_u T - p_vh,
  //   p'Ap = (||rv||^2 + ||rh||^2) / tau + sum dv p_vv^2 + sum dh p_vh^2,
  // an identity of the reference's p.dot(apply_a(p)) that needs only the
  // forward differences (row below, next column) and no recomputed neighbours
  double acc[1] = {0.0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> u = ldg4(pnew + o);
    const bool hasv = dn_ok(g, i);
    const Q4<T> ub = hasv ? ldg4(pnew + o + ld) : zero4<T>();
    const T ur = ldg_or0(pnew + o + 4, j0 + 4 < g.m);
    const Q4<T> v = ps4(o, P, dv, i, j0, true);
    const Q4<T> h = ps4(o, 2 * P, dh, i, j0, false);
    const Q4<T> d1 = ldg4(dv + o), d2 = ldg4(dh + o);
    st4(pnew + o + P, v);
    st4(pnew + o + 2 * P, h);
    T part = (T)0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const T right = (k == 3) ? ur : u.a[k + 1];
      const T rv = (hasv && j < g.m) ? (ub.a[k] - u.a[k]) - v.a[k] : (T)0;
      const T rh = (j < g.m - 1) ? (right - u.a[k]) - h.a[k] : (T)0;
      part += inv * (rv * rv + rh * rh) + d1.a[k] * v.a[k] * v.a[k] + d2.a[k] * h.a[k] * h.a[k];
    }
    acc[0] += (double)part;
  }
  pdl_trigger(g);
  double tot[1];
  if (red_final<1>(acc, rs, site, tot) && threadIdx.x == 0) fin_k1(ctrl, tot, it);
}

template <typename T>
__global__ void __launch_bounds__(256, PU_MINB(T, 4)) k_pcg_p_v(Grid g, const T* __restrict__ r, const T* __restrict__ pold,
                                                    T* __restrict__ pnew, const T* __restrict__ dv,
                                                    const T* __restrict__ dh, PcgCtrl* ctrl, RedScratch rs, int site,
                                                    int it) {
  pcg_p_body<T>(g, r, pold, pnew, dv, dh, ctrl, rs, site, it);
}

// ---------------------------------------------------------------------------
// K2a: residual update + slack preconditioner + norms.
// UPDATE: x += alpha p, r -= alpha A p.  SUBMEAN: r_u -= ctrl->mean_ru.
// MODE_ITER finaliser: ||r|| exits (pcg.py:94-100); MODE_INIT: rho_s only.
// ---------------------------------------------------------------------------
template <typename T, bool UPDATE, bool SUBMEAN, int MODE>
__device__ __forceinline__ void pcg_r_body(const Grid& g, const T* __restrict__ p, const T* __restrict__ dv,
                                           const T* __restrict__ dh, T* __restrict__ x, T* __restrict__ r,
                                           PcgCtrl* ctrl, double* res_norms, const RedScratch& rs, int site, int it) {
  pdl_enter(g);
  if (ctrl->done) return;
  const long long P = g.plane, ld = g.ld;
  const T alpha = (T)ctrl->alpha, nalpha = (T)(-ctrl->alpha);
  const T mean = (T)ctrl->mean_ru;
  const T inv = (T)g.inv_tau;
  double acc[2] = {0.0, 0.0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    Q4<T> ru, rv, rh;
    const Q4<T> d1 = ldg4(dv + o), d2 = ldg4(dh + o);
    if (UPDATE) {
      Stencil4<T> s;
      s.u = ldg4(p + o);
      s.v = ldg4(p + o + P);
      s.h = ldg4(p + o + 2 * P);
      s.ua = up_ok(g, i) ? ldg4(p + o - ld) : zero4<T>();
      s.va = up_ok(g, i) ? ldg4(p + o - ld + P) : zero4<T>();
      s.ub = dn_ok(g, i) ? ldg4(p + o + ld) : zero4<T>();
      s.ul = ldg_or0(p + o - 1, j0 > 0);
      s.hl = ldg_or0(p + o - 1 + 2 * P, j0 > 0);
      s.ur = ldg_or0(p + o + 4, j0 + 4 < g.m);
      Q4<T> au, av, ah;
      apply4<T>(g, i, j0, s, d1, d2, au, av, ah);
      Q4<T> xu = ldx4(x + o), xv = ldx4(x + o + P), xh = ldx4(x + o + 2 * P);
      ru = ldx4(r + o); rv = ldx4(r + o + P); rh = ldx4(r + o + 2 * P);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // pcg.py:90-91
        xu.a[k] = add_rn(xu.a[k], mul_rn(alpha, s.u.a[k]));
        xv.a[k] = add_rn(xv.a[k], mul_rn(alpha, s.v.a[k]));
        xh.a[k] = add_rn(xh.a[k], mul_rn(alpha, s.h.a[k]));
        ru.a[k] = add_rn(ru.a[k], mul_rn(nalpha, au.a[k]));
        rv.a[k] = add_rn(rv.a[k], mul_rn(nalpha, av.a[k]));
        rh.a[k] = add_rn(rh.a[k], mul_rn(nalpha, ah.a[k]));
      }
      st4(x + o, xu); st4(x + o + P, xv); st4(x + o + 2 * P, xh);
      st4(r + o + P, rv); st4(r + o + 2 * P, rh);
      if (!SUBMEAN) st4(r + o, ru);
    } else {
      ru = ldx4(r + o); rv = ldx4(r + o + P); rh = ldx4(r + o + 2 * P);
    }
    if (SUBMEAN) {  // pcg.py:92-93
#pragma unroll
      for (int k = 0; k < 4; ++k) ru.a[k] = (j0 + k < g.m) ? ru.a[k] - mean : (T)0;
      st4(r + o, ru);
    }
    T prr = (T)0, prz = (T)0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // z_s = r_s / (d + 1/tau) (preconditioner.py:115), recomputed by K1
      const int j = j0 + k;
      const T zv = (dn_ok(g, i) && j < g.m) ? slack_div(rv.a[k], d1.a[k] + inv) : (T)0;
      const T zh = (j < g.m - 1) ? slack_div(rh.a[k], d2.a[k] + inv) : (T)0;
      prr += ru.a[k] * ru.a[k] + rv.a[k] * rv.a[k] + rh.a[k] * rh.a[k];
      prz += rv.a[k] * zv + rh.a[k] * zh;
    }
    acc[0] += (double)prr;  // chunk partials in T, grid sums in fp64
    acc[1] += (double)prz;
  }
  pdl_trigger(g);
  double tot[2];
  if (red_final<2>(acc, rs, site, tot) && threadIdx.x == 0) fin_k2(g, ctrl, res_norms, tot, it, MODE);
}

template <typename T, bool UPDATE, bool SUBMEAN, int MODE>
__global__ void __launch_bounds__(256, PU_MINB(T, 3)) k_pcg_r_v(Grid g, const T* __restrict__ p, const T* __restrict__ dv,
                                                 const T* __restrict__ dh, T* __restrict__ x, T* __restrict__ r,
                                                 PcgCtrl* ctrl, double* res_norms, RedScratch rs, int site, int it) {
  pcg_r_body<T, UPDATE, SUBMEAN, MODE>(g, p, dv, dh, x, r, ctrl, res_norms, rs, site, it);
}

// update + sum(r_u) for the every-50 re-projection (the mean is subtracted by
// k_pcg_r_v<false, true, ...> next)
template <typename T>
__device__ __forceinline__ void pcg_upd_sum_body(const Grid& g, const T* __restrict__ p, const T* __restrict__ dv,
                                                 const T* __restrict__ dh, T* __restrict__ x, T* __restrict__ r,
                                                 PcgCtrl* ctrl, const RedScratch& rs, int site) {
  pdl_enter(g);
  if (ctrl->done) return;
  const long long P = g.plane, ld = g.ld;
  const T alpha = (T)ctrl->alpha, nalpha = (T)(-ctrl->alpha);
  double acc[1] = {0.0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> d1 = ldg4(dv + o), d2 = ldg4(dh + o);
    Stencil4<T> s;
    s.u = ldg4(p + o);
    s.v = ldg4(p + o + P);
    s.h = ldg4(p + o + 2 * P);
    s.ua = up_ok(g, i) ? ldg4(p + o - ld) : zero4<T>();
    s.va = up_ok(g, i) ? ldg4(p + o - ld + P) : zero4<T>();
    s.ub = dn_ok(g, i) ? ldg4(p + o + ld) : zero4<T>();
    s.ul = ldg_or0(p + o - 1, j0 > 0);
    s.hl = ldg_or0(p + o - 1 + 2 * P, j0 > 0);
    s.ur = ldg_or0(p + o + 4, j0 + 4 < g.m);
    Q4<T> au, av, ah;
    apply4<T>(g, i, j0, s, d1, d2, au, av, ah);
    Q4<T> xu = ldx4(x + o), xv = ldx4(x + o + P), xh = ldx4(x + o + 2 * P);
    Q4<T> ru = ldx4(r + o), rv = ldx4(r + o + P), rh = ldx4(r + o + 2 * P);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xu.a[k] = add_rn(xu.a[k], mul_rn(alpha, s.u.a[k]));
      xv.a[k] = add_rn(xv.a[k], mul_rn(alpha, s.v.a[k]));
      xh.a[k] = add_rn(xh.a[k], mul_rn(alpha, s.h.a[k]));
      ru.a[k] = add_rn(ru.a[k], mul_rn(nalpha, au.a[k]));
      rv.a[k] = add_rn(rv.a[k], mul_rn(nalpha, av.a[k]));
      rh.a[k] = add_rn(rh.a[k], mul_rn(nalpha, ah.a[k]));
      acc[0] += (double)ru.a[k];
    }
    st4(x + o, xu); st4(x + o + P, xv); st4(x + o + 2 * P, xh);
    st4(r + o, ru); st4(r + o + P, rv); st4(r + o + 2 * P, rh);
  }
  double tot[1];
  if (red_final<1>(acc, rs, site, tot) && threadIdx.x == 0) fin_upd(g, ctrl, tot);
}

template <typename T>
__global__ void __launch_bounds__(256) k_pcg_upd_sum_v(Grid g, const T* __restrict__ p, const T* __restrict__ dv,
                                                       const T* __restrict__ dh, T* __restrict__ x,
                                                       T* __restrict__ r, PcgCtrl* ctrl, RedScratch rs, int site) {
  pcg_upd_sum_body<T>(g, p, dv, dh, x, r, ctrl, rs, site);
}

// setup: x = x0 (skipped when x aliases x0), r = b - A x0, ||b||, ||r0||
// (pcg.py:59-75).  CAND: also the explicit gradient step of the same state,
// cand = x0 - (1/L) grad H(x0, w) (objective.py:108-125), from the same loads.
// cv/ch == nullptr means uniform unit arc weights.  RHSG (b == nullptr at the
// C ABI): b = build_rhs(gv, gh) (operators.py:156-162) is formed in registers
// from the candidate step's gradient loads with k_rhs's arithmetic (bit-
// identical), so the three b planes are never read (18 -> 15 planes moved).
template <typename T>
struct CandArgs {
  const T* gv; const T* gh; const T* cv; const T* ch; const T* wv; const T* wh; T neg_inv_lip; T* out;
};

template <typename T, bool CAND, bool RHSG = false>
__global__ void __launch_bounds__(256, PU_MINB_OUTER(T, 2)) k_pcg_start_v(Grid g, const T* __restrict__ b, const T* x0, T* x,
                                                        T* __restrict__ r, const T* __restrict__ dv,
                                                        const T* __restrict__ dh, PcgCtrl* ctrl, double* res_norms,
                                                        double rel_tol, int max_iters, RedScratch rs, int site,
                                                        CandArgs<T> ca) {
  const long long P = g.plane, ld = g.ld;
  const bool copy = x != x0;
  const T inv = (T)g.inv_tau;
  double acc[3] = {0.0, 0.0, 0.0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> d1 = ldg4(dv + o), d2 = ldg4(dh + o);
    Stencil4<T> s;
    s.u = ldg4(x0 + o);
    s.v = ldg4(x0 + o + P);
    s.h = ldg4(x0 + o + 2 * P);
    s.ua = up_ok(g, i) ? ldg4(x0 + o - ld) : zero4<T>();
    s.va = up_ok(g, i) ? ldg4(x0 + o - ld + P) : zero4<T>();
    s.ub = dn_ok(g, i) ? ldg4(x0 + o + ld) : zero4<T>();
    s.ul = ldg_or0(x0 + o - 1, j0 > 0);
    s.hl = ldg_or0(x0 + o - 1 + 2 * P, j0 > 0);
    s.ur = ldg_or0(x0 + o + 4, j0 + 4 < g.m);
    Q4<T> bu, bv, bh;
    if constexpr (!RHSG) { bu = ldg4(b + o); bv = ldg4(b + o + P); bh = ldg4(b + o + 2 * P); }
    // candidate-step operands: in fp32 issued with the start-up loads, so the
    // chunk waits for memory once instead of twice (fp64 would spill)
    Q4<T> g1, g2, ga, w1, w2, c1, c2;
    T gl = (T)0;
    auto load_cand = [&]() {
      g1 = ldg4(ca.gv + o); g2 = ldg4(ca.gh + o);
      ga = up_ok(g, i) ? ldg4(ca.gv + o - ld) : zero4<T>();
      gl = ldg_or0(ca.gh + o - 1, j0 > 0);
      if constexpr (sizeof(T) == 4) {  // fp64 uses the diagonal d instead
        w1 = ldg4(ca.wv + o); w2 = ldg4(ca.wh + o);
        if (ca.cv) { c1 = ldg4(ca.cv + o); c2 = ldg4(ca.ch + o); }
      }
    };
    constexpr bool EARLY = sizeof(T) == 4 || RHSG;
    if constexpr (CAND && EARLY) load_cand();
    if constexpr (RHSG) {  // k_rhs (pu_kernels.cuh) per cell, from the loaded gradients
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + k;
        const bool ok = j < g.m;
        const T gvo = (ok && dn_ok(g, i)) ? g1.a[k] : (T)0, gvm = ok ? ga.a[k] : (T)0;
        const T gho = (j < g.m - 1) ? g2.a[k] : (T)0;
        const T ghm = (ok && j > 0) ? ((k == 0) ? gl : g2.a[k - 1]) : (T)0;
        bu.a[k] = ok ? inv * ((gvm - gvo) + (ghm - gho)) : (T)0;
        bv.a[k] = ok ? -inv * gvo : (T)0;
        bh.a[k] = ok ? -inv * gho : (T)0;
      }
    }
    Q4<T> au, av, ah;
    apply4<T>(g, i, j0, s, d1, d2, au, av, ah);
    Q4<T> ru, rv, rh;
    T pb = (T)0, pr = (T)0, prz = (T)0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      ru.a[k] = add_rn(bu.a[k], -au.a[k]);
      rv.a[k] = add_rn(bv.a[k], -av.a[k]);
      rh.a[k] = add_rn(bh.a[k], -ah.a[k]);
      pb += bu.a[k] * bu.a[k] + bv.a[k] * bv.a[k] + bh.a[k] * bh.a[k];
      pr += ru.a[k] * ru.a[k] + rv.a[k] * rv.a[k] + rh.a[k] * rh.a[k];
      // rho_s of r0 (pcg.py:77-79, slack part of preconditioner.py:115), as K2a forms it
      const T zv = (dn_ok(g, i) && j < g.m) ? slack_div(rv.a[k], d1.a[k] + inv) : (T)0;
      const T zh = (j < g.m - 1) ? slack_div(rh.a[k], d2.a[k] + inv) : (T)0;
      prz += rv.a[k] * zv + rh.a[k] * zh;
    }
    acc[0] += (double)pb;  // chunk partials in T, grid sums in fp64
    acc[1] += (double)pr;
    acc[2] += (double)prz;
    if (copy) { st4(x + o, s.u); st4(x + o + P, s.v); st4(x + o + 2 * P, s.h); }
    st4(r + o, ru); st4(r + o + P, rv); st4(r + o + 2 * P, rh);
    if constexpr (CAND) {
      if constexpr (!EARLY) load_cand();
      const bool hasb = dn_ok(g, i), hasa = up_ok(g, i);
      Q4<T> ou, ov, oh;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + k;
        const bool ok = j < g.m, hash = j < g.m - 1;
        const T uo = s.u.a[k];
        const T left = (k == 0) ? s.ul : s.u.a[k - 1];
        const T right = (k == 3) ? s.ur : s.u.a[k + 1];
        const T hleft = (k == 0) ? s.hl : s.h.a[k - 1];
        const T gleft = (k == 0) ? gl : g2.a[k - 1];
        T rvv = 0, rvm = 0, rhh = 0, rhm = 0;
        if (hasb) rvv = ((s.ub.a[k] - uo) - g1.a[k]) - s.v.a[k];
        if (hasa) rvm = ((uo - s.ua.a[k]) - ga.a[k]) - s.va.a[k];
        if (hash) rhh = ((right - uo) - g2.a[k]) - s.h.a[k];
        if (j > 0) rhm = ((uo - left) - gleft) - hleft;
        const T gu = inv * ((rvm - rvv) + (rhm - rhh));
        // c^2 / w: in fp64 the diagonal d itself (diag_w formed it from the
        // same weights), so the candidate needs no c or w loads
        T qv, qh;
        if constexpr (sizeof(T) == 8) {
          qv = d1.a[k];
          qh = d2.a[k];
        } else {
          const T cv2 = ca.cv ? c1.a[k] * c1.a[k] : (T)1, ch2 = ca.cv ? c2.a[k] * c2.a[k] : (T)1;
          qv = slack_div(cv2, w1.a[k]);
          qh = slack_div(ch2, w2.a[k]);
        }
        const T gvv = qv * s.v.a[k] - inv * rvv;
        const T gvh = qh * s.h.a[k] - inv * rhh;
        ou.a[k] = ok ? add_rn(uo, mul_rn(ca.neg_inv_lip, gu)) : (T)0;
        ov.a[k] = (ok && hasb) ? add_rn(s.v.a[k], mul_rn(ca.neg_inv_lip, gvv)) : (T)0;
        oh.a[k] = hash ? add_rn(s.h.a[k], mul_rn(ca.neg_inv_lip, gvh)) : (T)0;
      }
      st4(ca.out + o, ou); st4(ca.out + o + P, ov); st4(ca.out + o + 2 * P, oh);
    }
  }
  double tot[3];
  if (red_final<3>(acc, rs, site, tot) && threadIdx.x == 0) fin_start(ctrl, res_norms, tot, rel_tol, max_iters);
}

}  // namespace pu

namespace pu {

// ---------------------------------------------------------------------------
// Vectorised outer-iteration kernels (irls.py:172-215).  Same per-cell
// arithmetic as the scalar kernels in pu_kernels.cuh; slack terms are formed
// in the storage precision T and accumulated in fp64.
// ---------------------------------------------------------------------------

// forward-difference penalty residuals of a 4-cell chunk, squared and summed
// in the storage precision T (fp32 partials of 4 terms in fp32 mode; the
// grid-wide sums are fp64):  rv = (u[i+1] - u[i]) - gv - vv,
// rh = (u[j+1] - u[j]) - gh - vh
template <typename T>
__device__ __forceinline__ void pen4(const Grid& g, int i, int j0, const Q4<T>& u, const Q4<T>& ub, T ur,
                                     const Q4<T>& vv, const Q4<T>& vh, const Q4<T>& gv, const Q4<T>& gh, double& sv,
                                     double& sh) {
  T pv = (T)0, ph = (T)0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    if (dn_ok(g, i) && j < g.m) {
      const T rv = ((ub.a[k] - u.a[k]) - gv.a[k]) - vv.a[k];
      pv += rv * rv;
    }
    if (j < g.m - 1) {
      const T right = (k == 3) ? ur : u.a[k + 1];
      const T rh = ((right - u.a[k]) - gh.a[k]) - vh.a[k];
      ph += rh * rh;
    }
  }
  sv += (double)pv;
  sh += (double)ph;
}

// slack term of H_delta for one arc: ((c v)^2 + delta^2) / w + w
template <typename T>
__device__ __forceinline__ T slack4(T c, T v, T w, T d2) {
  const T cv = c * v;
  return slack_div_p(cv * cv + d2, w) + w;
}
// slack4 with 1/w given (fp64: slack_div_p is a * rcp_nr(w), so this is the
// same arithmetic; fp32 divides as slack4)
__device__ __forceinline__ float slack4r(float c, float v, float w, float, float d2) { return slack4(c, v, w, d2); }
__device__ __forceinline__ double slack4r(double c, double v, double w, double rw, double d2) {
  const double cv = c * v;
  return (cv * cv + d2) * rw + w;
}
// d = c^2 / w of a new weight, and 1/w for slack4r: fp64 one reciprocal +
// Newton (rcp_nr) for both; fp32 the IEEE quotient (rw unused)
__device__ __forceinline__ float diag_w(float c, float w, float& rw) { rw = w; return c * c / w; }
__device__ __forceinline__ double diag_w(double c, double w, double& rw) { rw = rcp_nr(w); return c * c * rw; }

// w = sqrt((c v)^2 + delta^2), d = c^2 / w; H(x, w_prev), H(x, w)
template <typename T>
__global__ void __launch_bounds__(256, PU_MINB_OUTER(T, 3)) k_weights_hpair_v(Grid g, const T* __restrict__ x, const T* __restrict__ cv,
                                                         const T* __restrict__ ch, const T* __restrict__ gv,
                                                         const T* __restrict__ gh, const T* __restrict__ wpv,
                                                         const T* __restrict__ wph, T* __restrict__ wv,
                                                         T* __restrict__ wh, T* __restrict__ dv, T* __restrict__ dh,
                                                         RedScratch rs, int site, double* out) {
  const long long P = g.plane, ld = g.ld;
  const T d2 = (T)(g.delta * g.delta);
  const bool hasprev = wpv != nullptr;
  double acc[6] = {0, 0, 0, 0, 0, 0};  // old_v, old_h, new_v, new_h, pen_v, pen_h
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> u = ldg4(x + o), vv = ldg4(x + o + P), vh = ldg4(x + o + 2 * P);
    const Q4<T> ub = dn_ok(g, i) ? ldg4(x + o + ld) : zero4<T>();
    const T ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
    const Q4<T> g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    Q4<T> c1 = ones4<T>(), c2 = ones4<T>();
    if (cv) { c1 = ldg4(cv + o); c2 = ldg4(ch + o); }
    Q4<T> p1 = zero4<T>(), p2 = zero4<T>();
    if (hasprev) { p1 = ldg4(wpv + o); p2 = ldg4(wph + o); }
    Q4<T> w1, w2, e1, e2;
    T part[4] = {(T)0, (T)0, (T)0, (T)0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool okv = dn_ok(g, i) && j < g.m, okh = j < g.m - 1;
      const T a = c1.a[k] * vv.a[k], b = c2.a[k] * vh.a[k];
      const T wa = sqrt(a * a + d2), wb = sqrt(b * b + d2);
      w1.a[k] = okv ? wa : (T)1;
      w2.a[k] = okh ? wb : (T)1;
      T ra, rb;
      const T da = diag_w(c1.a[k], wa, ra), db = diag_w(c2.a[k], wb, rb);
      e1.a[k] = okv ? da : (T)0;
      e2.a[k] = okh ? db : (T)0;
      if (okv) {
        part[2] += slack4r(c1.a[k], vv.a[k], wa, ra, d2);
        if (hasprev) part[0] += slack4(c1.a[k], vv.a[k], p1.a[k], d2);
      }
      if (okh) {
        part[3] += slack4r(c2.a[k], vh.a[k], wb, rb, d2);
        if (hasprev) part[1] += slack4(c2.a[k], vh.a[k], p2.a[k], d2);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += (double)part[q];
    st4(wv + o, w1); st4(wh + o, w2); st4(dv + o, e1); st4(dh + o, e2);
    pen4<T>(g, i, j0, u, ub, ur, vv, vh, g1, g2, acc[4], acc[5]);
  }
  double tot[6];
  if (red_final<6>(acc, rs, site, tot) && threadIdx.x == 0) fin_hpair6(g, tot, out);
}

// H(xa, w), H(xb, w), mean u of the accepted one, acceptance flag
template <typename T>
__global__ void __launch_bounds__(256, PU_MINB_OUTER(T, 2)) k_hpair_states_v(Grid g, const T* __restrict__ xa, const T* __restrict__ xb,
                                                        const T* __restrict__ wv, const T* __restrict__ wh,
                                                        const T* __restrict__ gv, const T* __restrict__ gh,
                                                        const T* __restrict__ cv, const T* __restrict__ ch,
                                                        RedScratch rs, int site, double* out) {
  const long long P = g.plane, ld = g.ld;
  const T d2 = (T)(g.delta * g.delta);
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    Q4<T> c1 = ones4<T>(), c2 = ones4<T>();
    if (cv) { c1 = ldg4(cv + o); c2 = ldg4(ch + o); }
    const Q4<T> w1 = ldg4(wv + o), w2 = ldg4(wh + o);
    Q4<T> r1 = w1, r2 = w2;  // 1/w, shared by both states (fp64)
    if constexpr (sizeof(T) == 8) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { r1.a[k] = rcp_nr(w1.a[k]); r2.a[k] = rcp_nr(w2.a[k]); }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const T* x = s ? xb : xa;
      const Q4<T> u = ldg4(x + o), vv = ldg4(x + o + P), vh = ldg4(x + o + 2 * P);
      const Q4<T> ub = dn_ok(g, i) ? ldg4(x + o + ld) : zero4<T>();
      const T ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
      T pv = (T)0, ph = (T)0, pu = (T)0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + k;
        if (dn_ok(g, i) && j < g.m) pv += slack4r(c1.a[k], vv.a[k], w1.a[k], r1.a[k], d2);
        if (j < g.m - 1) ph += slack4r(c2.a[k], vh.a[k], w2.a[k], r2.a[k], d2);
        if (j < g.m) pu += u.a[k];
      }
      acc[5 * s + 0] += (double)pv;
      acc[5 * s + 1] += (double)ph;
      acc[5 * s + 4] += (double)pu;
      pen4<T>(g, i, j0, u, ub, ur, vv, vh, g1, g2, acc[5 * s + 2], acc[5 * s + 3]);
    }
  }
  double tot[10];
  if (red_final<10>(acc, rs, site, tot) && threadIdx.x == 0) fin_hpair_states(g, tot, out);
}

// cand = x - (1/L) grad H(x, w)   (objective.py:108-125)
template <typename T>
__global__ void __launch_bounds__(256, PU_MINB(T, 3)) k_candidate_v(Grid g, const T* __restrict__ x, const T* __restrict__ wv,
                                                     const T* __restrict__ wh, const T* __restrict__ gv,
                                                     const T* __restrict__ gh, const T* __restrict__ cv,
                                                     const T* __restrict__ ch, T neg_inv_lip, T* __restrict__ out) {
  const long long P = g.plane, ld = g.ld;
  const T inv = (T)g.inv_tau;
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const Q4<T> u = ldg4(x + o), vv = ldg4(x + o + P), vh = ldg4(x + o + 2 * P);
    const Q4<T> g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    const bool hasb = dn_ok(g, i), hasa = up_ok(g, i);
    const Q4<T> ub = hasb ? ldg4(x + o + ld) : zero4<T>();
    const Q4<T> ua = hasa ? ldg4(x + o - ld) : zero4<T>();
    const Q4<T> va = hasa ? ldg4(x + o - ld + P) : zero4<T>();
    const Q4<T> ga = hasa ? ldg4(gv + o - ld) : zero4<T>();
    const T ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
    const T ul = ldg_or0(x + o - 1, j0 > 0);
    const T hl = ldg_or0(x + o - 1 + 2 * P, j0 > 0);
    const T gl = ldg_or0(gh + o - 1, j0 > 0);
    const Q4<T> c1 = ldg4(cv + o), c2 = ldg4(ch + o), w1 = ldg4(wv + o), w2 = ldg4(wh + o);
    Q4<T> ou, ov, oh;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool ok = j < g.m, hash = j < g.m - 1;
      const T uo = u.a[k];
      const T left = (k == 0) ? ul : u.a[k - 1];
      const T right = (k == 3) ? ur : u.a[k + 1];
      const T hleft = (k == 0) ? hl : vh.a[k - 1];
      const T gleft = (k == 0) ? gl : g2.a[k - 1];
      T rv = 0, rvm = 0, rh = 0, rhm = 0;
      if (hasb) rv = ((ub.a[k] - uo) - g1.a[k]) - vv.a[k];
      if (hasa) rvm = ((uo - ua.a[k]) - ga.a[k]) - va.a[k];
      if (hash) rh = ((right - uo) - g2.a[k]) - vh.a[k];
      if (j > 0) rhm = ((uo - left) - gleft) - hleft;
      const T gu = inv * ((rvm - rv) + (rhm - rh));
      ou.a[k] = ok ? add_rn(uo, mul_rn(neg_inv_lip, gu)) : (T)0;
      const T gvv = c1.a[k] * c1.a[k] / w1.a[k] * vv.a[k] - inv * rv;
      const T gvh = c2.a[k] * c2.a[k] / w2.a[k] * vh.a[k] - inv * rh;
      ov.a[k] = (ok && hasb) ? add_rn(vv.a[k], mul_rn(neg_inv_lip, gvv)) : (T)0;
      oh.a[k] = hash ? add_rn(vh.a[k], mul_rn(neg_inv_lip, gvh)) : (T)0;
    }
    st4(out + o, ou); st4(out + o + P, ov); st4(out + o + 2 * P, oh);
  }
}

// dst = (sel[1] ? xa : xb) with u -= sel[0]; H(dst, w)   (irls.py:206-215)
template <typename T>
__global__ void __launch_bounds__(256, PU_MINB(T, 3)) k_accept_v(Grid g, const T* __restrict__ xa, const T* __restrict__ xb,
                                                  const double* sel, T* __restrict__ dst, const T* __restrict__ wv,
                                                  const T* __restrict__ wh, const T* __restrict__ gv,
                                                  const T* __restrict__ gh, const T* __restrict__ cv,
                                                  const T* __restrict__ ch, RedScratch rs, int site, double* out) {
  const long long P = g.plane, ld = g.ld;
  const T* x = sel[1] != 0.0 ? xa : xb;
  const T mean = (T)sel[0];
  const T d2 = (T)(g.delta * g.delta);
  double acc[4] = {0, 0, 0, 0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    Q4<T> u = ldg4(x + o);
    const Q4<T> vv = ldg4(x + o + P), vh = ldg4(x + o + 2 * P);
    Q4<T> ub = dn_ok(g, i) ? ldg4(x + o + ld) : zero4<T>();
    T ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
    const Q4<T> c1 = ldg4(cv + o), c2 = ldg4(ch + o), g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    const Q4<T> w1 = ldg4(wv + o), w2 = ldg4(wh + o);
    T pv = (T)0, ph = (T)0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      u.a[k] = (j < g.m) ? u.a[k] - mean : (T)0;
      ub.a[k] = ub.a[k] - mean;
      if (dn_ok(g, i) && j < g.m) pv += slack4(c1.a[k], vv.a[k], w1.a[k], d2);
      if (j < g.m - 1) ph += slack4(c2.a[k], vh.a[k], w2.a[k], d2);
    }
    acc[0] += (double)pv;
    acc[1] += (double)ph;
    ur = ur - mean;
    pen4<T>(g, i, j0, u, ub, ur, vv, vh, g1, g2, acc[2], acc[3]);
    st4(dst + o, u); st4(dst + o + P, vv); st4(dst + o + 2 * P, vh);
  }
  double tot[4];
  if (grid_reduce<4>(acc, rs, site, tot) && threadIdx.x == 0)
    out[0] = (0.5 * tot[0] + 0.5 * tot[1]) + (tot[2] + tot[3]) / (2.0 * g.tau);
}

// Acceptance and centring of iteration k fused with the weight refresh of
// iteration k + 1 (irls.py:206-215 then 173-177): dst = (sel[1] ? xa : xb)
// with u -= sel[0]; w_next = sqrt((c v)^2 + delta^2), d = c^2 / w_next;
// out[0] = H(dst, w_k) (the trace value and the next h_old), out[1] =
// H(dst, w_next) (the next h_new).  cv/ch == nullptr: unit weights.
template <typename T>
__global__ void __launch_bounds__(256, PU_MINB_OUTER(T, 2)) k_accept_weights_v(Grid g, const T* __restrict__ xa,
                                                             const T* __restrict__ xb, const double* sel,
                                                             T* __restrict__ dst, const T* __restrict__ gv,
                                                             const T* __restrict__ gh, const T* __restrict__ cv,
                                                             const T* __restrict__ ch, const T* __restrict__ wkv,
                                                             const T* __restrict__ wkh, T* __restrict__ wnv,
                                                             T* __restrict__ wnh, T* __restrict__ dv, T* __restrict__ dh,
                                                             RedScratch rs, int site, double* out) {
  const long long P = g.plane, ld = g.ld;
  const T* x = sel[1] != 0.0 ? xa : xb;
  const T mean = (T)sel[0];
  const T d2 = (T)(g.delta * g.delta);
  double acc[6] = {0, 0, 0, 0, 0, 0};  // old_v, old_h, new_v, new_h, pen_v, pen_h
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    Q4<T> u = ldg4(x + o);
    const Q4<T> vv = ldg4(x + o + P), vh = ldg4(x + o + 2 * P);
    Q4<T> ub = dn_ok(g, i) ? ldg4(x + o + ld) : zero4<T>();
    T ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
    const Q4<T> g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    Q4<T> c1 = ones4<T>(), c2 = ones4<T>();
    if (cv) { c1 = ldg4(cv + o); c2 = ldg4(ch + o); }
    const Q4<T> p1 = ldg4(wkv + o), p2 = ldg4(wkh + o);
    Q4<T> w1, w2, e1, e2;
    T part[4] = {(T)0, (T)0, (T)0, (T)0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool okv = dn_ok(g, i) && j < g.m, okh = j < g.m - 1;
      u.a[k] = (j < g.m) ? u.a[k] - mean : (T)0;
      ub.a[k] = ub.a[k] - mean;
      const T a = c1.a[k] * vv.a[k], bb = c2.a[k] * vh.a[k];
      const T wa = sqrt(a * a + d2), wb = sqrt(bb * bb + d2);
      w1.a[k] = okv ? wa : (T)1;
      w2.a[k] = okh ? wb : (T)1;
      T ra, rb;
      const T da = diag_w(c1.a[k], wa, ra), db = diag_w(c2.a[k], wb, rb);
      e1.a[k] = okv ? da : (T)0;
      e2.a[k] = okh ? db : (T)0;
      if (okv) {
        part[0] += slack4(c1.a[k], vv.a[k], p1.a[k], d2);
        part[2] += slack4r(c1.a[k], vv.a[k], wa, ra, d2);
      }
      if (okh) {
        part[1] += slack4(c2.a[k], vh.a[k], p2.a[k], d2);
        part[3] += slack4r(c2.a[k], vh.a[k], wb, rb, d2);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += (double)part[q];
    ur = ur - mean;
    pen4<T>(g, i, j0, u, ub, ur, vv, vh, g1, g2, acc[4], acc[5]);
    st4(dst + o, u); st4(dst + o + P, vv); st4(dst + o + 2 * P, vh);
    st4(wnv + o, w1); st4(wnh + o, w2); st4(dv + o, e1); st4(dh + o, e2);
  }
  double tot[6];
  if (red_final<6>(acc, rs, site, tot) && threadIdx.x == 0) fin_hpair6(g, tot, out);
}


// k_accept_weights_v of iteration k fused with the budget-free start of
// iteration k + 1 (k_pcg_start_v<T, true, true> on the accepted state):
// dst = (sel[1] ? xa : xb) with u -= sel[0]; w_next, d; H(dst, w_k),
// H(dst, w_next) -> out[0..1] (fin_hpair6); then from the same registers
// r = b - A dst with b = build_rhs(gv, gh), cand = dst - (1/L) grad H(dst,
// w_next), and the start-up sums ||b||^2, ||r0||^2, rho_s(r0) -> held[0..2]
// (fin_start runs later, in pu_irls_begin_z0, so the PCG control block is
// untouched until the host has snapshot iteration k).  One pass over the
// accepted state instead of two: 20 planes moved instead of 14 + 15.  Same
// per-cell arithmetic and per-thread accumulation order as the two kernels
// (same grid), so every value and sum is bit-identical to them.
// (fp32: 2 CTAs/SM, 104 B of spills, 0.268 ms at C3; 1 CTA/SM at 196
// registers without spills: 0.333 ms.  fp64: 2 CTAs/SM spill, 0.865 ms vs
// 0.80 for the two kernels; 1 CTA/SM, 0.70 ms, is the fp64 build.  Its FMA
// contraction differs from the two-kernel build in the last bits, so fp64
// results agree with the unfused path to ~1e-15, not bitwise.)
// Row bands: the neighbour rows of xa and xb are the ghost rows (exchanged
// before the launch); the sums go to the band totals (S_ACC and S_START rows)
// for the cross-rank all-reduce, finalised by k_finalize.
template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 2 : 1) k_accept_start_v(
    Grid g, const T* __restrict__ xa, const T* __restrict__ xb, const double* sel, T* __restrict__ dst,
    const T* __restrict__ gv, const T* __restrict__ gh, const T* __restrict__ cv, const T* __restrict__ ch,
    const T* __restrict__ wkv, const T* __restrict__ wkh, T* __restrict__ wnv, T* __restrict__ wnh,
    T* __restrict__ dv, T* __restrict__ dh, RedScratch rs, int site, double* out, T* __restrict__ r,
    T neg_inv_lip, T* __restrict__ cand, double* held) {
  const long long P = g.plane, ld = g.ld;
  const T* x = sel[1] != 0.0 ? xa : xb;
  const T mean = (T)sel[0];
  const T d2 = (T)(g.delta * g.delta);
  const T inv = (T)g.inv_tau;
  // old_v, old_h, new_v, new_h, pen_v, pen_h | ||b||^2, ||r0||^2, rho_s
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  PU_FOR_CHUNKS(g, i, j0) {
    const long long o = (long long)i * ld + j0;
    const bool hasb = dn_ok(g, i), hasa = up_ok(g, i);
    Stencil4<T> s;  // the accepted state, centred (as k_pcg_start_v reads dst)
    s.u = ldg4(x + o);
    s.v = ldg4(x + o + P);
    s.h = ldg4(x + o + 2 * P);
    s.ua = hasa ? ldg4(x + o - ld) : zero4<T>();
    s.va = hasa ? ldg4(x + o - ld + P) : zero4<T>();
    s.ub = hasb ? ldg4(x + o + ld) : zero4<T>();
    s.ul = ldg_or0(x + o - 1, j0 > 0);
    s.hl = ldg_or0(x + o - 1 + 2 * P, j0 > 0);
    s.ur = ldg_or0(x + o + 4, j0 + 4 < g.m);
    const Q4<T> g1 = ldg4(gv + o), g2 = ldg4(gh + o);
    const Q4<T> ga = hasa ? ldg4(gv + o - ld) : zero4<T>();
    const T gl = ldg_or0(gh + o - 1, j0 > 0);
    Q4<T> c1 = ones4<T>(), c2 = ones4<T>();
    if (cv) { c1 = ldg4(cv + o); c2 = ldg4(ch + o); }
    const Q4<T> p1 = ldg4(wkv + o), p2 = ldg4(wkh + o);
    // centring (irls.py:210): cells past the last column stay zero, as stored
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = j0 + k < g.m;
      s.u.a[k] = ok ? s.u.a[k] - mean : (T)0;
      s.ua.a[k] = (ok && hasa) ? s.ua.a[k] - mean : (T)0;
      s.ub.a[k] = (ok && hasb) ? s.ub.a[k] - mean : (T)0;
    }
    if (j0 > 0) s.ul = s.ul - mean;
    if (j0 + 4 < g.m) s.ur = s.ur - mean;
    // weights of k + 1 and the H pair (k_accept_weights_v)
    Q4<T> w1, w2, e1, e2;
    T part[4] = {(T)0, (T)0, (T)0, (T)0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool okv = hasb && j < g.m, okh = j < g.m - 1;
      const T a = c1.a[k] * s.v.a[k], bb = c2.a[k] * s.h.a[k];
#if PU_F64_RSQRT_W
      // fp64: w = x rsqrt(x) and 1/w = rsqrt(x) from one reciprocal square
      // root (profiles/r02_ab_rsqrt.txt: 504 -> 490 us; PU_F64_RSQRT_W=0 for
      // the sqrt + reciprocal form)
      T wa, wb, ra, rb, da, db;
      if constexpr (sizeof(T) == 8) {
        const T xa = a * a + d2, xb = bb * bb + d2;
        ra = rsqrt(xa); rb = rsqrt(xb);
        wa = xa * ra; wb = xb * rb;
        da = c1.a[k] * c1.a[k] * ra; db = c2.a[k] * c2.a[k] * rb;
      } else {
        wa = sqrt(a * a + d2); wb = sqrt(bb * bb + d2);
        da = diag_w(c1.a[k], wa, ra); db = diag_w(c2.a[k], wb, rb);
      }
#else
      const T wa = sqrt(a * a + d2), wb = sqrt(bb * bb + d2);
      // fp64: one reciprocal of each new weight serves d = c^2 / w and the
      // H(dst, w_next) slack term (reciprocal + Newton, as K1; diag_w)
      T ra, rb;
      const T da = diag_w(c1.a[k], wa, ra), db = diag_w(c2.a[k], wb, rb);
#endif
      w1.a[k] = okv ? wa : (T)1;
      w2.a[k] = okh ? wb : (T)1;
      e1.a[k] = okv ? da : (T)0;
      e2.a[k] = okh ? db : (T)0;
      if (okv) {
        part[0] += slack4(c1.a[k], s.v.a[k], p1.a[k], d2);
        part[2] += slack4r(c1.a[k], s.v.a[k], wa, ra, d2);
      }
      if (okh) {
        part[1] += slack4(c2.a[k], s.h.a[k], p2.a[k], d2);
        part[3] += slack4r(c2.a[k], s.h.a[k], wb, rb, d2);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] += (double)part[q];
    pen4<T>(g, i, j0, s.u, s.ub, s.ur, s.v, s.h, g1, g2, acc[4], acc[5]);
    st4(dst + o, s.u); st4(dst + o + P, s.v); st4(dst + o + 2 * P, s.h);
    st4(wnv + o, w1); st4(wnh + o, w2); st4(dv + o, e1); st4(dh + o, e2);
    // start-up of k + 1 (k_pcg_start_v<T, true, true>)
    Q4<T> au, av, ah;
    apply4<T>(g, i, j0, s, e1, e2, au, av, ah);
    T pb = (T)0, pr = (T)0, prz = (T)0;
    Q4<T> ru, rv, rh;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool ok = j < g.m;
      const T gvo = (ok && hasb) ? g1.a[k] : (T)0, gvm = ok ? ga.a[k] : (T)0;
      const T gho = (j < g.m - 1) ? g2.a[k] : (T)0;
      const T ghm = (ok && j > 0) ? ((k == 0) ? gl : g2.a[k - 1]) : (T)0;
      const T bu = ok ? inv * ((gvm - gvo) + (ghm - gho)) : (T)0;
      const T bv = ok ? -inv * gvo : (T)0;
      const T bh = ok ? -inv * gho : (T)0;
      ru.a[k] = add_rn(bu, -au.a[k]);
      rv.a[k] = add_rn(bv, -av.a[k]);
      rh.a[k] = add_rn(bh, -ah.a[k]);
      pb += bu * bu + bv * bv + bh * bh;
      pr += ru.a[k] * ru.a[k] + rv.a[k] * rv.a[k] + rh.a[k] * rh.a[k];
      const T zv = (hasb && j < g.m) ? slack_div_p(rv.a[k], e1.a[k] + inv) : (T)0;
      const T zh = (j < g.m - 1) ? slack_div_p(rh.a[k], e2.a[k] + inv) : (T)0;
      prz += rv.a[k] * zv + rh.a[k] * zh;
    }
    acc[6] += (double)pb;
    acc[7] += (double)pr;
    acc[8] += (double)prz;
    st4(r + o, ru); st4(r + o + P, rv); st4(r + o + 2 * P, rh);
    Q4<T> ou, ov, oh;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = j0 + k;
      const bool ok = j < g.m, hash = j < g.m - 1;
      const T uo = s.u.a[k];
      const T left = (k == 0) ? s.ul : s.u.a[k - 1];
      const T right = (k == 3) ? s.ur : s.u.a[k + 1];
      const T hleft = (k == 0) ? s.hl : s.h.a[k - 1];
      const T gleft = (k == 0) ? gl : g2.a[k - 1];
      T rvv = 0, rvm = 0, rhh = 0, rhm = 0;
      if (hasb) rvv = ((s.ub.a[k] - uo) - g1.a[k]) - s.v.a[k];
      if (hasa) rvm = ((uo - s.ua.a[k]) - ga.a[k]) - s.va.a[k];
      if (hash) rhh = ((right - uo) - g2.a[k]) - s.h.a[k];
      if (j > 0) rhm = ((uo - left) - gleft) - hleft;
      const T gu = inv * ((rvm - rvv) + (rhm - rhh));
      // c^2 / w_next: in fp64 exactly the diagonal d just formed (e1, e2: the
      // same IEEE division) wherever ov / oh use it; fp32 divides as k_pcg_start_v
      T qv, qh;
      if constexpr (sizeof(T) == 8) {
        qv = e1.a[k];
        qh = e2.a[k];
      } else {
        const T cv2 = cv ? c1.a[k] * c1.a[k] : (T)1, ch2 = cv ? c2.a[k] * c2.a[k] : (T)1;
        qv = slack_div(cv2, w1.a[k]);
        qh = slack_div(ch2, w2.a[k]);
      }
      const T gvv = qv * s.v.a[k] - inv * rvv;
      const T gvh = qh * s.h.a[k] - inv * rhh;
      ou.a[k] = ok ? add_rn(uo, mul_rn(neg_inv_lip, gu)) : (T)0;
      ov.a[k] = (ok && hasb) ? add_rn(s.v.a[k], mul_rn(neg_inv_lip, gvv)) : (T)0;
      oh.a[k] = hash ? add_rn(s.h.a[k], mul_rn(neg_inv_lip, gvh)) : (T)0;
    }
    st4(cand + o, ou); st4(cand + o + P, ov); st4(cand + o + 2 * P, oh);
  }
  double tot[9];
  if (grid_reduce<9>(acc, rs, site, tot) && threadIdx.x == 0) {
    if (rs.dist) {  // band mode: the H-pair sums to `site`'s row, the start-up sums to S_START's
#pragma unroll
      for (int q = 0; q < 6; ++q) rs.dist[site * PU_MAX_SUMS + q] = tot[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) rs.dist[S_START * PU_MAX_SUMS + q] = tot[6 + q];
      return;
    }
    fin_hpair6(g, tot, out);
    held[0] = tot[6]; held[1] = tot[7]; held[2] = tot[8];
  }
}

// pu_irls_begin_z0: fin_start from the start-up sums held by k_accept_start_v
static __global__ void k_fin_start_held(PcgCtrl* ctrl, double* res_norms, const double* held, double rel_tol,
                                 int max_iters) {
  if (threadIdx.x == 0 && blockIdx.x == 0) fin_start(ctrl, res_norms, held, rel_tol, max_iters);
}

}  // namespace pu
