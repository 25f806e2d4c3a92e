// DCT preconditioner passes and the fused PCG iteration (sm_100a).
//
// One PCG iteration of pcg.py:81-108 is four kernels:
//   K1 k_pcg_p     p <- beta p + z (z at it = 0); A p recomputed on the fly; p'Ap;
//                  last block: alpha = rho / p'Ap, curvature exits (pcg.py:82-89)
//   K2 k_rows_fwd  x += alpha p; r -= alpha A p (A p recomputed from p);
//                  ||r||^2; slack preconditioner z_s = r_s / (d + 1/tau); rho_s;
//                  row DCT-II of r_u -> spectral plane T;  last block: ||r|| exits
//   K3 k_cols_spec column DCT-II, x tau/(lam_i + lam_j) with (0,0) -> 0,
//                  rho_u = <r_hat, z_hat> (Parseval), column DCT-III;
//                  last block: beta = (rho_s + rho_u) / rho
//   K4 k_rows_inv  row DCT-III of T -> z_u
// The standalone preconditioner (preconditioner.py:86-115) is K2..K4 with the
// plain policies.  Every PCG kernel returns immediately once ctrl->done is set.
#pragma once

#include "pu_kernels.cuh"

namespace pu {

enum { MODE_API = 0, MODE_INIT = 1, MODE_ITER = 2 };

// ---------------------------------------------------------------------------
// K1: p update + A p + p'Ap
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_pcg_p(Grid g, const T* __restrict__ z, const T* __restrict__ pold, T* pnew,
                        const T* __restrict__ dv, const T* __restrict__ dh, PcgCtrl* ctrl, RedScratch rs,
                        int site, int it) {
  if (ctrl->done) return;
  PUpdSrc<T> s{z, pold, g.plane, (T)ctrl->beta, it == 0};
  double acc[1] = {0.0};
  PU_FOR_CELLS(g, i, j) {
    T xu, xv, xh, au, av, ah;
    sys_at<T>(g, s, dv, dh, i, j, xu, xv, xh, au, av, ah);
    const long long o = (long long)i * g.ld + j;
    pnew[o] = xu;
    pnew[o + g.plane] = xv;
    pnew[o + 2 * g.plane] = xh;
    acc[0] += (double)xu * (double)au + (double)xv * (double)av + (double)xh * (double)ah;
  }
  double tot[1];
  if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0) {
    const double pap = tot[0];
    ctrl->pap = pap;
    if (!isfinite(pap)) {
      ctrl->breakdown = it; ctrl->bkind = 1; ctrl->done = 1;
    } else if (pap <= PU_TINY_CURVATURE) {
      ctrl->converged = ctrl->rn <= ctrl->thr; ctrl->done = 1;
    } else {
      ctrl->alpha = ctrl->rho / pap;
    }
  }
}

// Setup: x = x0, r = b - A x0, ||b||, ||r0|| and the early exits (pcg.py:59-75).
template <typename T>
__global__ void k_pcg_start(Grid g, const T* __restrict__ b, const T* __restrict__ x0, T* x, T* r,
                            const T* __restrict__ dv, const T* __restrict__ dh, PcgCtrl* ctrl,
                            double* res_norms, double rel_tol, int max_iters, RedScratch rs, int site) {
  PlainSrc<T> s{x0, x0 + g.plane, x0 + 2 * g.plane};
  double acc[2] = {0.0, 0.0};
  PU_FOR_CELLS(g, i, j) {
    T xu, xv, xh, au, av, ah;
    sys_at<T>(g, s, dv, dh, i, j, xu, xv, xh, au, av, ah);
    const long long o = (long long)i * g.ld + j;
    const T bu = b[o], bv = b[o + g.plane], bh = b[o + 2 * g.plane];
    x[o] = xu; x[o + g.plane] = xv; x[o + 2 * g.plane] = xh;
    const T ru = add_rn(bu, -au), rv = add_rn(bv, -av), rh = add_rn(bh, -ah);
    r[o] = ru; r[o + g.plane] = rv; r[o + 2 * g.plane] = rh;
    acc[0] += (double)bu * bu + (double)bv * bv + (double)bh * bh;
    acc[1] += (double)ru * ru + (double)rv * rv + (double)rh * rh;
  }
  double tot[2];
  if (grid_reduce<2>(acc, rs, site, tot) && threadIdx.x == 0) {
    const double bn = sqrt(tot[0]);
    const double rn = sqrt(tot[1]);
    ctrl->bnorm = bn;
    ctrl->thr = rel_tol * bn;
    ctrl->rn = rn;
    ctrl->max_iters = max_iters;
    ctrl->breakdown = -1; ctrl->bkind = -1; ctrl->converged = 0; ctrl->done = 0;
    ctrl->iterations = 0; ctrl->alpha = 0; ctrl->beta = 0; ctrl->rho = 0; ctrl->pap = 0;
    res_norms[0] = rn;
    if (!isfinite(rn)) {
      ctrl->breakdown = 0; ctrl->bkind = 0; ctrl->done = 1;
    } else if (rn <= ctrl->thr || max_iters == 0) {
      ctrl->converged = rn <= ctrl->thr; ctrl->done = 1;
    }
  }
}

// Every REPROJECT_EVERY-th iteration (pcg.py:92-93): update x, r and sum r_u
// so that K2 can subtract the mean before forming ||r||.
template <typename T>
__global__ void k_pcg_update_sum(Grid g, const T* __restrict__ p, const T* __restrict__ dv,
                                 const T* __restrict__ dh, T* x, T* r, PcgCtrl* ctrl, RedScratch rs, int site) {
  if (ctrl->done) return;
  const T alpha = (T)ctrl->alpha, nalpha = (T)(-ctrl->alpha);
  PlainSrc<T> s{p, p + g.plane, p + 2 * g.plane};
  double acc[1] = {0.0};
  PU_FOR_CELLS(g, i, j) {
    T pu_, pv_, ph_, au, av, ah;
    sys_at<T>(g, s, dv, dh, i, j, pu_, pv_, ph_, au, av, ah);
    const long long o = (long long)i * g.ld + j;
    x[o] = add_rn(x[o], mul_rn(alpha, pu_));
    x[o + g.plane] = add_rn(x[o + g.plane], mul_rn(alpha, pv_));
    x[o + 2 * g.plane] = add_rn(x[o + 2 * g.plane], mul_rn(alpha, ph_));
    const T ru = add_rn(r[o], mul_rn(nalpha, au));
    r[o] = ru;
    r[o + g.plane] = add_rn(r[o + g.plane], mul_rn(nalpha, av));
    r[o + 2 * g.plane] = add_rn(r[o + 2 * g.plane], mul_rn(nalpha, ah));
    acc[0] += (double)ru;
  }
  double tot[1];
  if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0)
    ctrl->mean_ru = tot[0] / ((double)g.n * (double)g.m);
}

// ---------------------------------------------------------------------------
// Row-pass element policies for k_rows_fwd (value of r_u at (i, j) to be
// transformed; side effects and partial sums for the PCG variants).
// ---------------------------------------------------------------------------
template <typename T>
struct RowsPlain {
  static constexpr int NS = 1;
  static constexpr bool REDUCE = false;
  const T* src;
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ T elem(const Grid& g, int i, int j, double (&acc)[NS]) const {
    return src[(long long)i * g.ld + j];
  }
  __device__ __forceinline__ void finish(const Grid&, double (&)[NS]) const {}
};

template <typename T, bool UPDATE, bool SUBMEAN, int MODE>
struct RowsPcg {
  static constexpr int NS = 2;  // ||r||^2, rho_s
  static constexpr bool REDUCE = true;
  const T* p; T* x; T* r; T* z; const T* dv; const T* dh; PcgCtrl* ctrl; double* res_norms; int it;
  __device__ __forceinline__ bool skip() const { return ctrl->done != 0; }
  __device__ __forceinline__ T elem(const Grid& g, int i, int j, double (&acc)[NS]) const {
    const long long o = (long long)i * g.ld + j;
    T ru, rv, rh;
    if (UPDATE) {
      const T alpha = (T)ctrl->alpha, nalpha = (T)(-ctrl->alpha);
      PlainSrc<T> s{p, p + g.plane, p + 2 * g.plane};
      T pu_, pv_, ph_, au, av, ah;
      sys_at<T>(g, s, dv, dh, i, j, pu_, pv_, ph_, au, av, ah);
      x[o] = add_rn(x[o], mul_rn(alpha, pu_));
      x[o + g.plane] = add_rn(x[o + g.plane], mul_rn(alpha, pv_));
      x[o + 2 * g.plane] = add_rn(x[o + 2 * g.plane], mul_rn(alpha, ph_));
      ru = add_rn(r[o], mul_rn(nalpha, au));
      rv = add_rn(r[o + g.plane], mul_rn(nalpha, av));
      rh = add_rn(r[o + 2 * g.plane], mul_rn(nalpha, ah));
      r[o + g.plane] = rv;
      r[o + 2 * g.plane] = rh;
      if (!SUBMEAN) r[o] = ru;
    } else {
      ru = r[o]; rv = r[o + g.plane]; rh = r[o + 2 * g.plane];
    }
    if (SUBMEAN) {
      ru = ru - (T)ctrl->mean_ru;
      r[o] = ru;
    }
    acc[0] += (double)ru * ru + (double)rv * rv + (double)rh * rh;
    const T inv = (T)g.inv_tau;
    const T zv = (i < g.n - 1) ? rv / (dv[o] + inv) : (T)0;
    const T zh = (j < g.m - 1) ? rh / (dh[o] + inv) : (T)0;
    z[o + g.plane] = zv;
    z[o + 2 * g.plane] = zh;
    acc[1] += (double)rv * zv + (double)rh * zh;
    return ru;
  }
  __device__ __forceinline__ void finish(const Grid&, double (&tot)[NS]) const {
    ctrl->rho_s = tot[1];
    if (MODE == MODE_ITER) {
      const double rn = sqrt(tot[0]);
      ctrl->rn = rn;
      if (!isfinite(rn)) {
        ctrl->breakdown = it + 1; ctrl->bkind = 2; ctrl->done = 1;
        return;
      }
      res_norms[it + 1] = rn;
      ctrl->iterations = it + 1;
      if (rn <= ctrl->thr) { ctrl->converged = 1; ctrl->done = 1; }
    }
  }
};

// ---------------------------------------------------------------------------
// K2 family: element phase over `rows_per_cta` rows, then a row DCT-II of the
// staged values.  Two rows share one complex FFT (real + imaginary part).
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LS, class Pol>
__global__ void __launch_bounds__(fft_max_threads(LS, EMAX), fft_min_blocks(LS, EMAX)) k_rows_fwd(Grid g, FftPlan<T> pl, int rows_per_cta, T* out, Pol pol, RedScratch rs, int site) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  if (pol.skip()) return;
  const int n = g.m;
  const int i0 = blockIdx.x * rows_per_cta;
  const int nrows = min(rows_per_cta, g.n - i0);
  const int nseq = (nrows + 1) >> 1;
  double acc[Pol::NS];
#pragma unroll
  for (int s = 0; s < Pol::NS; ++s) acc[s] = 0.0;
  for (int rr = 0; rr < 2 * nseq; ++rr) {
    cplx<T>* sb = buf + (rr >> 1) * pl.ldseq;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const T val = (rr < nrows) ? pol.elem(g, i0 + rr, j, acc) : (T)0;
      T* slot = reinterpret_cast<T*>(sb + spad(mperm(j, n)));
      slot[rr & 1] = val;
    }
  }
  __syncthreads();
  fft_n<T, EMAX, LS>(buf, nseq, pl);
  const int half = n / 2 + 1;
  for (int e = threadIdx.x; e < nseq * half; e += blockDim.x) {
    const int s = e / half, k = e - s * half;
    const int nk = (n - k) % n;
    const cplx<T>* sb = buf + s * pl.ldseq;
    const PairOut<T> q = dct2_post<T>(sb[spad(k)], sb[spad(nk)], k, nk, pl);
    const long long oa = (long long)(i0 + 2 * s) * g.ld, ob = oa + g.ld;
    const bool hasb = 2 * s + 1 < nrows;
    out[oa + k] = q.a_k;
    if (hasb) out[ob + k] = q.b_k;
    if (nk != k) {
      out[oa + nk] = q.a_nk;
      if (hasb) out[ob + nk] = q.b_nk;
    }
  }
  if constexpr (Pol::REDUCE) {
    double tot[Pol::NS];
    if (grid_reduce<Pol::NS>(acc, rs, site, tot) && threadIdx.x == 0) pol.finish(g, tot);
  }
}

// ---------------------------------------------------------------------------
// K4 / API: row DCT-III (orthonormal inverse) of `in` into `out`.
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LS>
__global__ void __launch_bounds__(fft_max_threads(LS, EMAX), fft_min_blocks(LS, EMAX)) k_rows_inv(Grid g, FftPlan<T> pl, int rows_per_cta, const T* __restrict__ in, T* out,
                           const PcgCtrl* ctrl) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  if (ctrl && ctrl->done) return;
  const int n = g.m;
  const int i0 = blockIdx.x * rows_per_cta;
  const int nrows = min(rows_per_cta, g.n - i0);
  const int nseq = (nrows + 1) >> 1;
  const int half = n / 2 + 1;
  for (int e = threadIdx.x; e < nseq * half; e += blockDim.x) {
    const int s = e / half, k = e - s * half;
    const int nk = (n - k) % n;
    const long long oa = (long long)(i0 + 2 * s) * g.ld, ob = oa + g.ld;
    const bool hasb = 2 * s + 1 < nrows;
    const T ak = in[oa + k], ank = in[oa + nk];
    const T bk = hasb ? in[ob + k] : (T)0, bnk = hasb ? in[ob + nk] : (T)0;
    cplx<T> ck, cnk;
    dct3_pre<T>(ak, ank, bk, bnk, k, nk, pl, ck, cnk);
    cplx<T>* sb = buf + s * pl.ldseq;
    sb[spad(k)] = ck;
    if (nk != k) sb[spad(nk)] = cnk;
  }
  __syncthreads();
  fft_n<T, EMAX, LS>(buf, nseq, pl);
  const T invn = (T)(1.0 / (double)n);
  for (int rr = 0; rr < nrows; ++rr) {
    const cplx<T>* sb = buf + (rr >> 1) * pl.ldseq;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const cplx<T> v = sb[spad(mperm(j, n))];
      out[(long long)(i0 + rr) * g.ld + j] = ((rr & 1) ? -v.y : v.x) * invn;
    }
  }
}

// ---------------------------------------------------------------------------
// K3 / API: column DCT-II, spectral division, column DCT-III, in place on a
// panel of `cols_per_cta` columns; reduces rho_u = <r_hat, z_hat>.
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LS, int MODE>
__global__ void __launch_bounds__(fft_max_threads(LS, EMAX), fft_min_blocks(LS, EMAX)) k_cols_spec(Grid g, FftPlan<T> pl, const double* __restrict__ lam_cols, int cols_per_cta, T* data,
                            PcgCtrl* ctrl, RedScratch rs, int site, int it) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  if (MODE != MODE_API && ctrl->done) return;
  const int n = g.n;
  const int W = cols_per_cta;
  const int j0 = blockIdx.x * W;
  const int ncols = min(W, g.m - j0);
  const int nseq = (ncols + 1) >> 1;
  for (int e = threadIdx.x; e < n * 2 * nseq; e += blockDim.x) {
    const int i = e / (2 * nseq), c = e - i * (2 * nseq);
    const T val = (c < ncols) ? data[(long long)i * g.ld + j0 + c] : (T)0;
    T* slot = reinterpret_cast<T*>(buf + (c >> 1) * pl.ldseq + spad(mperm(i, n)));
    slot[c & 1] = val;
  }
  __syncthreads();
  fft_n<T, EMAX, LS>(buf, nseq, pl);
  double acc[1] = {0.0};
  const int half = n / 2 + 1;
  const double tau = g.tau;
  for (int e = threadIdx.x; e < nseq * half; e += blockDim.x) {
    const int s = e / half, k = e - s * half;
    const int nk = (n - k) % n;
    cplx<T>* sb = buf + s * pl.ldseq;
    const PairOut<T> q = dct2_post<T>(sb[spad(k)], sb[spad(nk)], k, nk, pl);
    const int ja = j0 + 2 * s, jb = ja + 1;
    const bool hasb = jb < g.m;
    const double lk = __ldg(pl.lam + k), lnk = __ldg(pl.lam + nk);
    const double la = __ldg(lam_cols + ja), lb = hasb ? __ldg(lam_cols + jb) : 0.0;
    // preconditioner.py:96-99: z = tau * r / (lam_s + lam_t), (0,0) -> 0
    auto sdiv = [&](T v, double den) -> T { return den == 0.0 ? (T)0 : (T)(tau * (double)v / den); };
    const T zak = sdiv(q.a_k, lk + la), zbk = hasb ? sdiv(q.b_k, lk + lb) : (T)0;
    T zank = 0, zbnk = 0;
    acc[0] += (double)q.a_k * zak + (hasb ? (double)q.b_k * zbk : 0.0);
    if (nk != k) {
      zank = sdiv(q.a_nk, lnk + la);
      zbnk = hasb ? sdiv(q.b_nk, lnk + lb) : (T)0;
      acc[0] += (double)q.a_nk * zank + (hasb ? (double)q.b_nk * zbnk : 0.0);
    } else {
      zank = zak; zbnk = zbk;
    }
    cplx<T> ck, cnk;
    dct3_pre<T>(zak, zank, zbk, zbnk, k, nk, pl, ck, cnk);
    sb[spad(k)] = ck;
    if (nk != k) sb[spad(nk)] = cnk;
  }
  __syncthreads();
  fft_n<T, EMAX, LS>(buf, nseq, pl);
  const T invn = (T)(1.0 / (double)n);
  for (int e = threadIdx.x; e < n * 2 * nseq; e += blockDim.x) {
    const int i = e / (2 * nseq), c = e - i * (2 * nseq);
    if (c < ncols) {
      const cplx<T> v = buf[(c >> 1) * pl.ldseq + spad(mperm(i, n))];
      data[(long long)i * g.ld + j0 + c] = ((c & 1) ? -v.y : v.x) * invn;
    }
  }
  if (MODE != MODE_API) {
    double tot[1];
    if (grid_reduce<1>(acc, rs, site, tot) && threadIdx.x == 0) {
      const double rho_next = ctrl->rho_s + tot[0];
      if (MODE == MODE_INIT) {
        ctrl->rho = rho_next;
      } else {
        if (!isfinite(rho_next)) {
          ctrl->breakdown = it + 1; ctrl->bkind = 3; ctrl->done = 1;
        } else {
          ctrl->beta = rho_next / ctrl->rho;
          ctrl->rho = rho_next;
        }
      }
    }
  }
}

// slack part of the standalone preconditioner: z_s = r_s / (d + 1/tau)
template <typename T>
__global__ void k_precond_slack(Grid g, const T* __restrict__ r, const T* __restrict__ dv, const T* __restrict__ dh,
                                T* z) {
  const T inv = (T)g.inv_tau;
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    z[o + g.plane] = (i < g.n - 1) ? r[o + g.plane] / (dv[o] + inv) : (T)0;
    z[o + 2 * g.plane] = (j < g.m - 1) ? r[o + 2 * g.plane] / (dh[o] + inv) : (T)0;
  }
}

}  // namespace pu
