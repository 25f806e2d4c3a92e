// Finalisers of the grid-wide reductions (one thread), shared by the fused
// kernels (single GPU: run by the last block of the reduction) and by
// k_finalize (row-sharded grids: run after the band totals have been summed
// across ranks, see pu_create_band in pu_api.cu).
//
// Sites (RedScratch tickets and, in band mode, rows of the totals buffer):
#pragma once

#include "pu_common.cuh"

namespace pu {

enum Site { S_DOT = 0, S_WH, S_EVH, S_HPAIR, S_ACC, S_EVF, S_START, S_K1, S_K2, S_K3, S_UPD, S_K2B, S_MET, S_NSITES };
// ticket of the input check (whole grids only: no band totals row)
enum { S_CHK = S_NSITES };
enum { MODE_API = 0, MODE_INIT = 1, MODE_ITER = 2 };

#define PU_TINY_CURVATURE 1e-300

// Band mode: store the band totals for the cross-rank all-reduce and skip the
// finaliser; otherwise true in the one block whose thread 0 finalises.
template <int NS>
__device__ __forceinline__ bool red_final(double (&v)[NS], RedScratch rs, int site, double (&tot)[NS]) {
  if (!grid_reduce<NS>(v, rs, site, tot)) return false;
  if (rs.dist) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) rs.dist[site * PU_MAX_SUMS + s] = tot[s];
    }
    return false;
  }
  return true;
}

// pcg.py:59-79: ||b||, ||r0||, threshold, initial exits; rho_s of z0 = M r0
__device__ __forceinline__ void fin_start(PcgCtrl* ctrl, double* res_norms, const double* tot, double rel_tol,
                                          int max_iters) {
  ctrl->rho_s = tot[2];
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

// pcg.py:82-89: p'Ap -> alpha, curvature exits
__device__ __forceinline__ void fin_k1(PcgCtrl* ctrl, const double* tot, int it) {
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

// pcg.py:94-100 (+ rho_s of preconditioner.py:115): ||r|| exits.
// On the last iteration of the budget the reference still forms z = M r and
// rho (pcg.py:101-108) only to check rho for a NumericalBreakdown; z and p are
// then discarded.  When rho_s is finite and ||r||^2 is below the bound for
// which rho_u = <r_hat, tau r_hat / lambda> and every transform intermediate
// provably stay finite in T (g.tail_rn2_max, set by the host), that check
// cannot fire, so the loop ends here and the transforms of the tail are
// skipped.  Otherwise they run and K3 performs the check.
__device__ __forceinline__ void fin_k2(const Grid& g, PcgCtrl* ctrl, double* res_norms, const double* tot, int it,
                                       int mode) {
  ctrl->rho_s = tot[1];
  if (mode == MODE_ITER) {
    const double rn = sqrt(tot[0]);
    ctrl->rn = rn;
    if (!isfinite(rn)) {
      ctrl->breakdown = it + 1; ctrl->bkind = 2; ctrl->done = 1;
    } else {
      res_norms[it + 1] = rn;
      ctrl->iterations = it + 1;
      if (rn <= ctrl->thr) {
        ctrl->converged = 1; ctrl->done = 1;
      } else if (it + 1 == ctrl->max_iters && isfinite(tot[1]) && tot[0] <= g.tail_rn2_max) {
        ctrl->done = 1;  // budget exhausted, rho provably finite: nothing left to compute
      }
    }
  }
}

// pcg.py:101-106: rho = r.z (slack + spectral parts), beta
__device__ __forceinline__ void fin_k3(PcgCtrl* ctrl, const double* tot, int it, int mode) {
  const double rho_next = ctrl->rho_s + tot[0];
  if (mode == MODE_INIT) {
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

// pcg.py:92-93 (project_out_constant): mean of r_u
__device__ __forceinline__ void fin_upd(const Grid& g, PcgCtrl* ctrl, const double* tot) {
  ctrl->mean_ru = tot[0] / ((double)g.n_glob * (double)g.m);
}

// objective.py:77-89 twice: H(x, w_prev), H(x, w) from the 6 slack/penalty sums
__device__ __forceinline__ void fin_hpair6(const Grid& g, const double* tot, double* out) {
  const double pen = (tot[4] + tot[5]) / (2.0 * g.tau);
  out[0] = (0.5 * tot[0] + 0.5 * tot[1]) + pen;
  out[1] = (0.5 * tot[2] + 0.5 * tot[3]) + pen;
}

// irls.py:202-210: H(proposal), H(cand), mean u of the accepted one, flag
__device__ __forceinline__ void fin_hpair_states(const Grid& g, const double* tot, double* out) {
  const double ha = (0.5 * tot[0] + 0.5 * tot[1]) + (tot[2] + tot[3]) / (2.0 * g.tau);
  const double hb = (0.5 * tot[5] + 0.5 * tot[6]) + (tot[7] + tot[8]) / (2.0 * g.tau);
  const bool take_a = ha <= hb;
  out[0] = ha;
  out[1] = hb;
  out[2] = (take_a ? tot[4] : tot[9]) / ((double)g.n_glob * (double)g.m);
  out[3] = take_a ? 1.0 : 0.0;
}

// Band mode: finalisers of the sites in `mask` (bit = site), in PCG order,
// on the all-reduced totals.  One thread.
struct FinArgs {
  PcgCtrl* ctrl;
  double* res_norms;
  double* out;
  double rel_tol;
  int max_iters;
  int it;
  int mode;
};

static __global__ void k_finalize(Grid g, const double* __restrict__ tot, unsigned mask, FinArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  auto T_ = [&](int site) { return tot + site * PU_MAX_SUMS; };
  if (mask & (1u << S_START)) fin_start(a.ctrl, a.res_norms, T_(S_START), a.rel_tol, a.max_iters);
  if (mask & (1u << S_WH)) fin_hpair6(g, T_(S_WH), a.out);
  if (mask & (1u << S_HPAIR)) fin_hpair_states(g, T_(S_HPAIR), a.out);
  if (mask & (1u << S_ACC)) fin_hpair6(g, T_(S_ACC), a.out);
  // PCG sites: skipped once the loop has ended, as the fused kernels are
  if (a.ctrl && (mask & ((1u << S_K1) | (1u << S_K2) | (1u << S_K3) | (1u << S_UPD)))) {
    if (a.ctrl->done) return;
    if (mask & (1u << S_K1)) fin_k1(a.ctrl, T_(S_K1), a.it);
    if (a.ctrl->done) return;
    if (mask & (1u << S_UPD)) fin_upd(g, a.ctrl, T_(S_UPD));
    if (mask & (1u << S_K2)) fin_k2(g, a.ctrl, a.res_norms, T_(S_K2), a.it, a.mode);
    if (a.ctrl->done) return;
    if (mask & (1u << S_K3)) fin_k3(a.ctrl, T_(S_K3), a.it, a.mode);
  }
}

}  // namespace pu
