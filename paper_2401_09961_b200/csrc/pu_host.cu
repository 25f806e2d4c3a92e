// pu_unwrap: the whole reference `unwrap` (irls.py:132-224) behind one C
// call, for hosts that bind C instead of running the Python mirror of the
// outer loop.  Everything here goes through the public entry points of
// include/pu_unwrap.h (the same launch sequence as paper_2401_09961_b200/
// irls.py: pu_irls_begin + pu_irls_iterate + pu_accept_weights per outer
// iteration), so results are bit-identical to the Python host's.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "pu_unwrap.h"

namespace pu {
int fail_ext(int code, const char* msg);  // pu_api.cu: the thread's pu_last_error slot
}

namespace {

const double kTwoPi = 6.283185307179586;

int bad(const std::string& msg) { return pu::fail_ext(PU_ERR_ARG, msg.c_str()); }

int cuda_fail(cudaError_t e, const char* what) {
  return pu::fail_ext(e == cudaErrorMemoryAllocation ? PU_ERR_NOMEM : PU_ERR_CUDA,
                      (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

// Scalar slots of the device block (the Python Workspace uses the same order).
enum { S_HOLD = 0, S_HNEW, S_HPROP, S_HCAND, S_MEAN, S_TAKE, S_HACC, S_HNEXT, NSCAL = 16 };

// Argument checks of the reference, before any device work.
int validate(const double* x, int n, int m, const double* cv, const double* ch, double tau, double delta,
             const pu_irls_params& p, double lo, int dtype, double* u, double* vv, double* vh) {
  if (!x) return bad("x must not be NULL");
  if (n < 1 || m < 1) return bad("phase grid must be 2-D and non-empty");  // phase.py:104-106
  const size_t cells = (size_t)n * (size_t)m;
  for (size_t i = 0; i < cells; ++i) {
    if (!std::isfinite(x[i])) return bad("phase grid contains non-finite values");  // phase.py:108-110
    if (x[i] < 0.0 || x[i] >= kTwoPi) return bad("wrapped phase values must lie in [0, 2*pi)");  // phase.py:111-114
  }
  if ((cv == nullptr) != (ch == nullptr)) return bad("cv and ch must both be given or both NULL");
  if (cv) {  // phase.py:61-73
    const size_t nv = (size_t)(n - 1) * m, nh = (size_t)n * (m - 1);
    bool any = false;
    for (size_t i = 0; i < nv + nh; ++i) {
      const double c = i < nv ? cv[i] : ch[i - nv];
      if (!std::isfinite(c)) return bad("weights must be finite");
      if (c < 0.0) return bad("weights must be nonnegative");
      any = any || c > 0.0;
    }
    if (nv + nh > 0 && !any) return bad("at least one weight must be positive");
  }
  if (!(tau > 0) || !std::isfinite(tau)) return bad("tau must be positive and finite");      // objective.py:37-39
  if (!(delta > 0) || !std::isfinite(delta)) return bad("delta must be positive and finite");  // objective.py:40-41
  if (p.max_iter_cg_start < 1) return bad("max_iter_cg_start must be >= 1");  // irls.py:52-64
  if (!(p.rel_improvement_tol > 0)) return bad("rel_improvement_tol must be positive");
  if (!(p.cg_growth_factor > 1)) return bad("cg_growth_factor must exceed 1");
  if (p.max_outer_iters < 1) return bad("max_outer_iters must be >= 1");
  if (p.max_cg_iters_cap < p.max_iter_cg_start) return bad("max_cg_iters_cap must be >= max_iter_cg_start");
  if (!(p.cg_rel_tol >= 0)) return bad("cg_rel_tol must be >= 0");
  if (!(lo == 0.0 || lo == -3.141592653589793)) return bad("lo must be 0 or -pi");
  if (dtype != PU_F32 && dtype != PU_F64) return bad("dtype must be PU_F32 or PU_F64");
  if (!u || (n > 1 && !vv) || (m > 1 && !vh)) return bad("output arrays must not be NULL");
  return PU_OK;
}

// Owned device state of one call; released on every exit path.
struct Run {
  pu_handle* h = nullptr;
  cudaStream_t st = nullptr;
  std::vector<void*> dev;
  void* pin = nullptr;
  ~Run() {
    if (st) cudaStreamSynchronize(st);
    for (void* p : dev) cudaFree(p);
    if (pin) cudaFreeHost(pin);
    if (st) cudaStreamDestroy(st);
    if (h) pu_destroy(h);
  }
  cudaError_t alloc(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) {
      dev.push_back(*p);
      e = cudaMemsetAsync(*p, 0, bytes, st);  // pitch padding and pads must be zero
    }
    return e;
  }
};

#define PU_CK(call, what)                                   \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);      \
  } while (0)
#define PU_OK_OR(call)              \
  do {                              \
    const int rc_ = (call);         \
    if (rc_ != PU_OK) return rc_;   \
  } while (0)

}  // namespace

extern "C" void pu_irls_params_default(pu_irls_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->max_iter_cg_start = 5;
  p->max_outer_iters = 100;
  p->max_cg_iters_cap = 10000;
  p->rel_improvement_tol = 1e-3;
  p->cg_growth_factor = 1.7;
  p->cg_rel_tol = 1e-10;
}

extern "C" int pu_unwrap(const double* x, int n, int m, const double* cv, const double* ch, double tau, double delta,
                         const pu_irls_params* params, double gradient_lo, int dtype, int device, double* u, double* vv,
                         double* vh, pu_iteration_record* trace, int trace_cap, int* trace_len,
                         int* breakdown_iteration) {
  pu_irls_params p;
  if (params) p = *params;
  else pu_irls_params_default(&p);
  if (trace_len) *trace_len = 0;
  if (breakdown_iteration) *breakdown_iteration = -1;
  PU_OK_OR(validate(x, n, m, cv, ch, tau, delta, p, gradient_lo, dtype, u, vv, vh));

  PU_CK(cudaSetDevice(device), "cudaSetDevice");
  Run R;
  // graphs of pu_irls_begin / pu_irls_iterate need a non-legacy stream
  PU_CK(cudaStreamCreateWithFlags(&R.st, cudaStreamNonBlocking), "cudaStreamCreate");
  PU_OK_OR(pu_create(&R.h, n, m, dtype, tau, delta));
  const size_t esz = dtype == PU_F32 ? 4 : 8;
  const size_t plane = (size_t)pu_plane_elems(R.h) * esz;
  const size_t ctrl_bytes = (size_t)pu_pcg_ctrl_bytes();
  char* base = nullptr;
  // planes: state x2, cand, rhs, grad, w x2, d, r, p0, p1, spec, weights
  const bool uniform = cv == nullptr;
  const int nplanes = 3 + 3 + 3 + 3 + 3 + 2 + 2 + 2 + 2 + 3 + 3 + 3 + 1 + (uniform ? 0 : 2);
  PU_CK(R.alloc(reinterpret_cast<void**>(&base), plane * nplanes), "cudaMalloc planes");
  char* at = base;
  auto take = [&](int k) { char* q = at; at += plane * k; return q; };
  void* S[2] = {take(3), take(3)};
  // the candidate of iteration k lives in Cs[k & 1]: the fused acceptance of
  // k reads it while writing the candidate of k + 1
  void* Cs[2] = {take(3), take(3)};
  void* rhs = take(3);
  char* G = take(2);
  char* W[2] = {take(2), take(2)};
  char* D = take(2);
  void* r = take(3);
  void* p0 = take(3);
  void* p1 = take(3);
  void* spec = take(1);
  char* C = uniform ? nullptr : take(2);
  void *gv = G, *gh = G + plane, *dv = D, *dh = D + plane;
  const void* cvp = uniform ? nullptr : C;
  const void* chp = uniform ? nullptr : C + plane;
  // fp64 scalar block followed by the PCG control record; residual norms
  double* blk = nullptr;
  double* norms = nullptr;
  PU_CK(R.alloc(reinterpret_cast<void**>(&blk), NSCAL * 8 + ctrl_bytes), "cudaMalloc scalars");
  PU_CK(R.alloc(reinterpret_cast<void**>(&norms), sizeof(double) * ((size_t)p.max_cg_iters_cap + 65)),
        "cudaMalloc norms");
  void* ctrl = reinterpret_cast<char*>(blk) + NSCAL * 8;
  PU_CK(cudaMallocHost(&R.pin, NSCAL * 8 + ctrl_bytes), "cudaMallocHost");
  const double* hs = static_cast<const double*>(R.pin);
  const pu_pcg_ctrl* hc = reinterpret_cast<const pu_pcg_ctrl*>(static_cast<char*>(R.pin) + NSCAL * 8);

  // inputs: x (compact fp64), arc weights packed into planes
  double* xd = nullptr;
  PU_CK(R.alloc(reinterpret_cast<void**>(&xd), sizeof(double) * (size_t)n * m), "cudaMalloc x");
  PU_CK(cudaMemcpyAsync(xd, x, sizeof(double) * (size_t)n * m, cudaMemcpyHostToDevice, R.st), "upload x");
  double cmax = 1.0;
  if (!uniform) {
    const size_t nv = (size_t)(n - 1) * m, nh = (size_t)n * (m - 1);
    double* cd = nullptr;
    PU_CK(R.alloc(reinterpret_cast<void**>(&cd), sizeof(double) * (nv + nh + 1)), "cudaMalloc weights");
    PU_CK(cudaMemcpyAsync(cd, cv, sizeof(double) * nv, cudaMemcpyHostToDevice, R.st), "upload cv");
    PU_CK(cudaMemcpyAsync(cd + nv, ch, sizeof(double) * nh, cudaMemcpyHostToDevice, R.st), "upload ch");
    if (nv) PU_OK_OR(pu_pack(R.h, cd, m, n - 1, m, C, R.st));
    if (nh) PU_OK_OR(pu_pack(R.h, cd + nv, m - 1, n, m - 1, C + plane, R.st));
    cmax = 0.0;  // WeightField.max_weight (phase.py:79-86)
    for (size_t i = 0; i < nv; ++i) cmax = std::max(cmax, cv[i]);
    for (size_t i = 0; i < nh; ++i) cmax = std::max(cmax, ch[i]);
  }
  const double lip = 12.0 / tau + cmax * cmax / delta;  // objective.py:103-105

  // irls.py:160-177: gradients, rhs, x_0 = (0, -gv, -gh), w_0, d_0, H(x_0, w_0)
  PU_OK_OR(pu_wrapped_gradients(R.h, xd, m, gv, gh, gradient_lo, R.st));
  // fp32: b = build_rhs(gv, gh) is formed inside the start-up kernel (b = NULL)
  const void* b = nullptr;
  if (dtype == PU_F64) {
    PU_OK_OR(pu_build_rhs(R.h, gv, gh, rhs, R.st));
    b = rhs;
  }
  PU_OK_OR(pu_init_state(R.h, gv, gh, S[0], R.st));
  PU_OK_OR(pu_weights_hpair(R.h, S[0], cvp, chp, gv, gh, nullptr, nullptr, W[0], W[0] + plane, dv, dh, blk + S_HOLD,
                            R.st));

  int count = 0;
  auto record = [&](int k, int m_cg, bool has_delta, double delta_rel) -> int {
    if (hc->breakdown >= 0) {  // pcg.py:24-29 -> NumericalBreakdown(iteration)
      if (breakdown_iteration) *breakdown_iteration = hc->breakdown;
      static const char* what[4] = {"initial residual is not finite", "curvature p'Ap is not finite",
                                    "residual norm is not finite", "preconditioned product is not finite"};
      const int kind = hc->bkind;
      return pu::fail_ext(PU_ERR_BREAKDOWN, (std::string("iteration ") + std::to_string(hc->breakdown) + ": " +
                                             (kind >= 0 && kind < 4 ? what[kind] : "non-finite value")).c_str());
    }
    if (trace && count < trace_cap) {
      pu_iteration_record& t = trace[count];
      std::memset(&t, 0, sizeof(t));
      t.k = k;
      t.m_cg = m_cg;
      t.has_delta_rel = has_delta ? 1 : 0;
      t.delta_rel = has_delta ? delta_rel : 0.0;
      t.h_delta = hs[S_HACC];
      t.cg_iters = hc->iterations;
      t.sufficient_decrease = hs[S_TAKE] != 0.0;
      t.fallback_used = hs[S_TAKE] == 0.0;
    }
    ++count;
    return PU_OK;
  };

  // irls.py:172-222, as the Python host runs it (irls._LoopJob): iteration k
  // is finished, its scalars are snapshot asynchronously, and the
  // budget-free first half of k + 1 (pu_irls_begin: candidate step, PCG
  // start-up, z0) is enqueued before the host waits for the snapshot.  From
  // 2048^2 cells the acceptance of k also runs the start-up of k + 1 in the
  // same pass (pu_accept_weights_start; then pu_irls_begin_z0).
  const bool fused = (long long)n * m >= 2048LL * 2048LL;  // irls._fuse_start on a single unwrap
  cudaEvent_t snap = nullptr;
  PU_CK(cudaEventCreateWithFlags(&snap, cudaEventDisableTiming), "cudaEventCreate");
  struct EvGuard { cudaEvent_t e; ~EvGuard() { if (e) cudaEventDestroy(e); } } evg{snap};
  int cur = 0;
  bool prestarted = false;
  auto begin = [&](int k) -> int {
    char* w = W[k & 1];
    if (prestarted) {
      prestarted = false;
      return pu_irls_begin_z0(R.h, dv, dh, p.cg_rel_tol, r, p0, p1, spec, ctrl, norms, R.st);
    }
    return pu_irls_begin(R.h, S[cur], b, gv, gh, cvp, chp, w, w + plane, dv, dh, lip, p.cg_rel_tol, Cs[k & 1], r, p0,
                         p1, spec, ctrl, norms, R.st);
  };
  auto finish = [&](int k, int m_cg) -> int {
    char* w = W[k & 1];
    char* wn = W[(k + 1) & 1];
    PU_OK_OR(pu_irls_iterate(R.h, S[cur], gv, gh, cvp, chp, w, w + plane, dv, dh, m_cg, Cs[k & 1], r, p0, p1, spec,
                             ctrl, norms, blk + S_HPROP, R.st));
    if (fused && k + 1 < p.max_outer_iters) {
      PU_OK_OR(pu_accept_weights_start(R.h, S[cur], Cs[k & 1], blk + S_MEAN, S[1 - cur], gv, gh, cvp, chp, w,
                                       w + plane, wn, wn + plane, dv, dh, blk + S_HACC, lip, r, Cs[(k + 1) & 1],
                                       R.st));
      prestarted = true;
    } else {
      PU_OK_OR(pu_accept_weights(R.h, S[cur], Cs[k & 1], blk + S_MEAN, S[1 - cur], gv, gh, cvp, chp, w, w + plane,
                                 wn, wn + plane, dv, dh, blk + S_HACC, R.st));
    }
    cur = 1 - cur;
    return PU_OK;
  };
  auto enqueue = [&](int k, int m_cg) -> int {
    if (k == 0) PU_OK_OR(begin(0));
    PU_OK_OR(finish(k, m_cg));
    PU_CK(cudaMemcpyAsync(R.pin, blk, NSCAL * 8 + ctrl_bytes, cudaMemcpyDeviceToHost, R.st), "snapshot");
    PU_CK(cudaEventRecord(snap, R.st), "cudaEventRecord");
    if (k + 1 < p.max_outer_iters) PU_OK_OR(begin(k + 1));  // speculative: needs no budget
    return PU_OK;
  };
  std::vector<int> hist{p.max_iter_cg_start};
  PU_OK_OR(enqueue(0, hist[0]));
  int pend_k = 0, pend_m = hist[0];
  bool pend_has = false;
  double pend_delta = 0.0;
  for (int k = 1;; ++k) {
    PU_CK(cudaEventSynchronize(snap), "cudaEventSynchronize");
    PU_OK_OR(record(pend_k, pend_m, pend_has, pend_delta));
    if (k >= p.max_outer_iters) break;
    // H(state_k, w_{k-1}) is the accepted value of k-1; H(state_k, w_k) its refresh
    const double h_old = hs[S_HACC], h_new = hs[S_HNEXT];
    double delta_rel = 0.0;
    if (h_old != 0.0) {
      if (!(h_old > 0)) return bad("reference objective value must be positive");  // irls.py:111-115
      delta_rel = (h_old - h_new) / h_old;
    }
    const int m_prev = hist[k - 1];
    const int m_prev2 = k >= 2 ? hist[k - 2] : m_prev;
    int m_cg;
    // irls.py:118-129: keep while improving, stop after a fruitless grow, else grow
    if (delta_rel > p.rel_improvement_tol) {
      m_cg = m_prev;
    } else if (m_prev != m_prev2 || m_prev >= p.max_cg_iters_cap) {
      break;
    } else {
      m_cg = (int)std::min<double>(std::ceil(p.cg_growth_factor * m_prev), (double)p.max_cg_iters_cap);
    }
    hist.push_back(m_cg);
    PU_OK_OR(enqueue(k, m_cg));
    pend_k = k;
    pend_m = m_cg;
    pend_has = true;
    pend_delta = delta_rel;
  }
  if (trace_len) *trace_len = count;

  // results: planes -> compact fp64 on the device -> host (irls.py:224)
  double* out = nullptr;
  const size_t cells = (size_t)n * m;
  PU_CK(R.alloc(reinterpret_cast<void**>(&out), sizeof(double) * cells), "cudaMalloc result");
  const char* fin = static_cast<const char*>(S[cur]);
  struct Part { const char* src; int rows, cols; double* dst; } parts[3] = {
      {fin, n, m, u}, {fin + plane, n - 1, m, vv}, {fin + 2 * plane, n, m - 1, vh}};
  for (const Part& q : parts) {
    if (q.rows < 1 || q.cols < 1) continue;
    PU_OK_OR(pu_unpack(R.h, q.src, q.rows, q.cols, out, R.st));
    PU_CK(cudaMemcpyAsync(q.dst, out, sizeof(double) * (size_t)q.rows * q.cols, cudaMemcpyDeviceToHost, R.st),
          "download result");
    PU_CK(cudaStreamSynchronize(R.st), "cudaStreamSynchronize");
  }
  return PU_OK;
}
