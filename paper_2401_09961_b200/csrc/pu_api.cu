// Host side of libpu_unwrap.so: FFT/DCT plans, launch shapes, the PCG
// enqueue loop and the extern "C" entry points declared in include/pu_unwrap.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "pu_dct_launch.cuh"
#include "pu_split.cuh"
#include "pu_vec.cuh"

namespace pu {

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// the same error slot for the other translation units (pu_host.cu)
int fail_ext(int code, const char* msg) { return fail(code, msg); }

#define PU_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(PU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// process-wide count of kernels launched through this library (bench.py reports it)
static std::atomic<long long> g_launches{0};

#define PU_LAUNCH_CHECK()                                                                   \
  do {                                                                                      \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                     \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess) return fail(PU_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define PU_DCT(call)                                       \
  do {                                                     \
    g_launches.fetch_add(1, std::memory_order_relaxed);    \
    PU_CUDA(call);                                         \
  } while (0)

#define PU_RC(call)                 \
  do {                              \
    const int rc_ = (call);         \
    if (rc_ != PU_OK) return rc_;   \
  } while (0)


typedef long double ld_t;
static const ld_t kPi = 3.141592653589793238462643383279502884L;

// ---------------------------------------------------------------------------
// Plans
// ---------------------------------------------------------------------------
static void host_fft_pow2(std::vector<std::complex<ld_t>>& a) {
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const ld_t ang = -2.0L * kPi * (ld_t)k / (ld_t)len;
        const std::complex<ld_t> w(cosl(ang), sinl(ang));
        const std::complex<ld_t> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

static bool factor_smooth(int n, int emax, std::vector<int>& rad) {
  rad.clear();
  int r = n;
  int p2 = 0;
  while (r % 2 == 0) { r /= 2; ++p2; }
  const int big = emax >= 16 ? 4 : 3;  // log2 of the largest power-of-two radix
  while (p2 >= big) { rad.push_back(1 << big); p2 -= big; }
  if (p2 > 0) rad.push_back(1 << p2);
  for (int p : {3, 5, 7}) while (r % p == 0) { rad.push_back(p); r /= p; }
  return r == 1;
}

template <typename T>
struct HostPlan {
  FftPlan<T> dev{};
  std::vector<void*> allocs;
  int seq_capacity = 0;  // min over stages of R * floor(EMAX/R)
  int emax = 0;

  int build(int n) {
    emax = emax_of<T>();
    std::memset(&dev, 0, sizeof(dev));
    dev.n = n;
    std::vector<int> rad;
    int L = n;
    bool blue = !factor_smooth(n, emax, rad);
    if (blue) {
      L = 1;
      while (L < 2 * n - 1) L <<= 1;
      factor_smooth(L, emax, rad);
    }
    if ((int)rad.size() > PU_FFT_MAX_STAGES) return fail(PU_ERR_UNSUPPORTED, "too many FFT stages");
    dev.L = L;
    dev.bluestein = blue ? 1 : 0;
    dev.nst = (int)rad.size();
    seq_capacity = emax;
    std::sort(rad.begin(), rad.end());  // the radix with Q > 1 runs first, twiddle-free
    for (size_t s = 0; s < rad.size(); ++s) {
      dev.rad[s] = rad[s];
      seq_capacity = std::min(seq_capacity, rad[s] * (emax / rad[s]));
    }
    dev.cap = seq_capacity;
    dev.ldseq = ldseq_for(L);  // spad(L-1) + 1 (+ pad), kept even for 16-byte alignment
    using C = cplx<T>;
    std::vector<C> tw(L), dct2w(n), dct3w(n), chirp(n), filt(L);
    std::vector<T> lam(n);
    for (int k = 0; k < L; ++k) {
      const ld_t a = -2.0L * kPi * (ld_t)k / (ld_t)L;
      tw[k].x = (T)cosl(a); tw[k].y = (T)sinl(a);
    }
    for (int k = 0; k < n; ++k) {
      const ld_t a = kPi * (ld_t)k / (2.0L * (ld_t)n);
      const ld_t sk = sqrtl((k == 0 ? 1.0L : 2.0L) / (ld_t)n);
      dct2w[k].x = (T)(sk * cosl(a)); dct2w[k].y = (T)(sk * sinl(a));
      dct3w[k].x = (T)(cosl(a) / (sk * n)); dct3w[k].y = (T)(sinl(a) / (sk * n));
      const ld_t sh = sinl(a);
      lam[k] = (T)(4.0L * sh * sh);  // 2 - 2 cos(pi k / n), cancellation-free
    }
    lam[0] = (T)0;
    // twiddle blocks of the compile-time plan (fft_stages_s): stage s >= 1 with
    // stride NS and radix R stores W_{NS R}^k for k < NS
    std::vector<C> stw;
    if (!blue && (L & (L - 1)) == 0 && L >= 512) {
      const int big = emax >= 16 ? 16 : 8;
      int rem = L;
      while (rem > 1 && rem % big == 0) rem /= big;
      int ns = rem == 1 ? big : rem;  // first (twiddle-free) radix
      while (ns < L) {
        const int R = big;
        for (int k = 0; k < ns; ++k) {
          const ld_t a = -2.0L * kPi * (ld_t)k / (ld_t)(ns * R);
          C c; c.x = (T)cosl(a); c.y = (T)sinl(a);
          stw.push_back(c);
        }
        ns *= R;
      }
    }
    if (blue) {
      std::vector<std::complex<ld_t>> h(L, std::complex<ld_t>(0, 0));
      for (int k = 0; k < n; ++k) {
        const long long q = ((long long)k * k) % (2LL * n);
        const ld_t a = -kPi * (ld_t)q / (ld_t)n;
        chirp[k].x = (T)cosl(a); chirp[k].y = (T)sinl(a);
        const std::complex<ld_t> b(cosl(-a), sinl(-a));  // conj(chirp)
        h[k] = b;
        if (k > 0) h[L - k] = b;
      }
      host_fft_pow2(h);
      for (int k = 0; k < L; ++k) {
        filt[k].x = (T)(h[k].real() / (ld_t)L);
        filt[k].y = (T)(h[k].imag() / (ld_t)L);
      }
    }
    int rc;
    if ((rc = upload(tw, &dev.tw)) || (rc = upload(dct2w, &dev.dct2w)) || (rc = upload(dct3w, &dev.dct3w)) ||
        (rc = upload(lam, &dev.lam)) || (rc = upload(stw, &dev.stw)))
      return rc;
    if (blue && ((rc = upload(chirp, &dev.chirp)) || (rc = upload(filt, &dev.filt)))) return rc;
    return PU_OK;
  }

  template <typename V, typename P>
  int upload(const std::vector<V>& v, const P** dst) {
    void* p = nullptr;
    PU_CUDA(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(V)));
    allocs.push_back(p);
    PU_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
    *dst = reinterpret_cast<const P*>(p);
    return PU_OK;
  }

  void release() {
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
  }

  // threads for `nseq` sequences: at least one whole sequence per stage,
  // at most the instantiation's launch bound (larger groups run sequentially)
  int max_threads() const {
    const bool stat = !dev.bluestein && (dev.L & (dev.L - 1)) == 0 && dev.L >= 512 &&
                      dev.L <= (sizeof(T) == 4 ? 16384 : 8192);
    return fft_max_threads(stat ? dev.L : 0, emax, sizeof(T));
  }
  int threads_for(int nseq) const {
    const long long need = ((long long)nseq * dev.L + seq_capacity - 1) / seq_capacity;
    long long t = ((need + 31) / 32) * 32;
    t = std::min<long long>(t, max_threads());
    const long long one = ((dev.L + seq_capacity - 1) / seq_capacity + 31) / 32 * 32;
    return (int)std::max<long long>(std::max<long long>(t, one), 64);
  }
  size_t smem_for(int nseq) const { return (size_t)nseq * dev.ldseq * sizeof(cplx<T>); }
};

template <typename T>
struct DctOps {
  cudaError_t (*set_attrs)(size_t, size_t);
  decltype(&DctLaunch<T, 0>::rows_pipe) rows_pipe;
  decltype(&DctLaunch<T, 0>::rows_pipe_blocks_per_sm) rows_pipe_bps;
  decltype(&DctLaunch<T, 0>::cols) cols;
  decltype(&DctLaunch<T, 0>::cols_blocks_per_sm) cols_bps;
  int ls;
};

template <typename T, int LS>
static DctOps<T> make_ops() {
  using D = DctLaunch<T, LS>;
  return DctOps<T>{&D::set_attrs, &D::rows_pipe, &D::rows_pipe_blocks_per_sm,
                   &D::cols, &D::cols_blocks_per_sm, LS};
}

template <typename T>
static DctOps<T> ops_for(int L) {  // L = internal length of a non-Bluestein plan, else 0
  switch (L) {
    case 512: return make_ops<T, 512>();
    case 1024: return make_ops<T, 1024>();
    case 2048: return make_ops<T, 2048>();
    case 4096: return make_ops<T, 4096>();
    case 8192: return make_ops<T, 8192>();
    default: break;
  }
  if constexpr (sizeof(T) == 4) {
    if (L == 16384) return make_ops<T, 16384>();
  }
  return make_ops<T, 0>();
}

// Optional per-launch CUDA-event timing (bench.py's roofline numbers are
// taken from these, on the launching stream).
struct Timer {
  bool on = false;
  struct Rec { int kind, it; cudaEvent_t a, b; bool pooled; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  std::vector<Rec>* sink = nullptr;  // set while a CUDA graph is being captured
  cudaEvent_t get() {
    cudaEvent_t e = nullptr;
    if (sink == nullptr && !pool.empty()) { e = pool.back(); pool.pop_back(); }
    else cudaEventCreate(&e);
    return e;
  }
  // during stream capture a plain cudaEventRecord only orders streams; the
  // External flag makes it a real event-record node of the graph
  void record(cudaEvent_t e, cudaStream_t st) {
    if (sink) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
  cudaEvent_t begin(cudaStream_t st) {
    if (!on) return nullptr;
    cudaEvent_t a = get();
    record(a, st);
    return a;
  }
  void end(cudaStream_t st, cudaEvent_t a, int kind, int it) {
    if (!on || !a) return;
    cudaEvent_t b = get();
    record(b, st);
    // events recorded during capture become graph nodes owned by the graph cache
    (sink ? *sink : recs).push_back(Rec{kind, it, a, b, sink == nullptr});
  }
  int read(int* kinds, int* its, float* ms, int cap) {
    int n = 0;
    for (auto& r : recs) {
      float t = 0.f;
      cudaEventSynchronize(r.b);
      cudaEventElapsedTime(&t, r.a, r.b);
      if (n < cap) { kinds[n] = r.kind; its[n] = r.it; ms[n] = t; }
      ++n;
      if (r.pooled) {
        pool.push_back(r.a);
        pool.push_back(r.b);
      }
    }
    recs.clear();
    return std::min(n, cap);
  }
  ~Timer() {
    for (auto& r : recs)
      if (r.pooled) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Captured CUDA graphs of whole IRLS inner steps (candidate + PCG budget +
// H pair), keyed by budget, pointers and scalars.  A PCG budget is hundreds
// of small launches; one graph launch removes the per-kernel host cost that
// dominates grids of 1024^2 and below.
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  std::vector<Timer::Rec> timed;  // event pairs captured inside the graph
  long long kernels = 0;          // kernels per replay (for pu_launch_count)
};

struct GraphCache {
  std::map<std::vector<unsigned long long>, GraphEntry> m;
  void clear() {
    for (auto& kv : m) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      for (auto& r : kv.second.timed) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    }
    m.clear();
  }
  ~GraphCache() { clear(); }
};

enum TimeKind { TK_START = 0, TK_K1, TK_K2, TK_K3, TK_K4, TK_UPD, TK_WEIGHTS, TK_CAND, TK_HPAIR, TK_ACCEPT, TK_K2B };

static const size_t kSmemLimit = 227 * 1024 - 4096;  // leave room for static reduction scratch

// ---------------------------------------------------------------------------
// Handle
// ---------------------------------------------------------------------------
struct HandleBase {
  virtual ~HandleBase() {}
};

template <typename T>
struct Impl : HandleBase {
  Grid g{};
  HostPlan<T> prow, pcol;  // row transforms (length m), column transforms (length n)
  // lengths 2 LHS (fp64 16384, fp32 32768): a 2-CTA cluster per sequence
  // (pu_split.cuh); prow_h / pcol_h hold the LHS-point static plans
  static constexpr int LHS = sizeof(T) == 4 ? 16384 : 8192;
  bool row_split = false, col_split = false;
  HostPlan<T> prow_h, pcol_h;
  // programmatic dependent launch of the PCG-iteration kernels (PU_PDL=1/2;
  // g.pdl / gc.pdl carry the mode into the kernels); pdl_now is set while
  // pcg_iterate enqueues
  int pdl_mode = 0;
  bool pdl_now = false;
  int cols_per_cta = 2, col_threads = 64;
  int col_nfull = 1 << 30, col_nhalf = 0;  // balanced column grid: full panels, then half panels
  size_t col_smem = 0;
  int ew_grid = 1, ew_threads = 32;
  int pipe_grid = 1, pipe_threads = 64;
  bool col_is_static = false;
  size_t pipe_smem = 0;
  RedScratch rs{};
  int* pinned_done = nullptr;
  double* held = nullptr;  // start-up sums of k_accept_start_v, finalised by pu_irls_begin_z0
  bool held_pending = false;  // host-side: an accept_start was enqueued and not yet finalised
  DctOps<T> rops{}, cops{};  // transform kernels for the row / column internal lengths
  Timer tm;
  GraphCache graphs;
  bool use_graphs = true;
  bool band = false;   // row band of a sharded grid (init with pu_band)
  Grid gc{};           // grid of the column transform (band: the column block, else g)
  Pack pk{};           // packed transpose layout of the band's spectrum (nq = 0: plain)
  int col0 = 0;        // first global column of the band's column block
  Push push{};         // peer mode: K3 sends its output rows to their owners' buffers

  ~Impl() override {
    prow.release();
    pcol.release();
    prow_h.release();
    pcol_h.release();
    if (rs.partials) cudaFree(rs.partials);
    if (rs.ticket) cudaFree(rs.ticket);
    if (pinned_done) cudaFreeHost(pinned_done);
    if (held) cudaFree(held);
  }

  // b == nullptr: the whole N x M grid.  Otherwise one row band of a
  // row-sharded grid (pu_create_band): planes carry ghost rows -1 and n, the
  // column transform runs on the band's column block of the transposed
  // spectrum, and reductions leave band totals for the cross-rank all-reduce.
  int init(int n, int m, double tau, double delta, const pu_band* b = nullptr) {
    const int n_glob = b ? b->n_glob : n;
    if (b) n = b->rows;
    band = b != nullptr;
    g.n = n; g.m = m;
    g.ld = ((long long)m + 7) / 8 * 8;
    g.plane = (long long)(n + (band ? 2 : 0)) * g.ld;
    g.tau = tau; g.inv_tau = 1.0 / tau; g.delta = delta;
    g.n_glob = n_glob;
    g.top = band && b->row0 > 0;
    g.bot = band && b->row0 + b->rows < n_glob;
    {
      // bound of fin_k2: rho_u <= tau ||r||^2 / lambda_min (orthonormal DCT) and
      // the unnormalised transforms grow values by at most N M; keep 16x margin
      auto lam1 = [](int len) { const double s = std::sin(3.141592653589793 / (2.0 * len)); return 4.0 * s * s; };
      double lam_min = INFINITY;
      if (n_glob > 1) lam_min = std::min(lam_min, lam1(n_glob));
      if (m > 1) lam_min = std::min(lam_min, lam1(m));
      const double tmax = sizeof(T) == 4 ? 3.4028234663852886e38 : 1.7976931348623157e308;
      const double grow = 16.0 * (double)n_glob * (double)m * (std::isfinite(lam_min) ? tau / lam_min + 1.0 : 1.0);
      g.tail_rn2_max = tmax / grow;
    }
    if (!band) {
      const char* e = std::getenv("PU_PDL");
      pdl_mode = e ? std::atoi(e) : 0;
      if (pdl_mode < 0 || pdl_mode > 2) pdl_mode = 0;
    }
    g.pdl = pdl_mode;
    gc = g;
    if (band) {
      gc.n = n_glob; gc.m = b->cols; gc.ld = b->mb; gc.plane = (long long)n_glob * b->mb;
      gc.top = gc.bot = 0;
      pk = Pack{b->nq, b->mb, (long long)n * b->mb, nullptr, (long long)b->row0, FastDiv((unsigned)b->mb)};
      col0 = b->col0;
    }
    int rc;
    if ((rc = prow.build(m)) || (rc = pcol.build(n_glob))) return rc;
    // (Bluestein plans: internal length L = 2 LHS, i.e. non-smooth n in (LHS/2, LHS])
    row_split = prow.dev.L == 2 * LHS && std::getenv("PU_NO_SPLIT") == nullptr;
    col_split = pcol.dev.L == 2 * LHS && std::getenv("PU_NO_SPLIT") == nullptr;
    if (row_split && (rc = prow_h.build(LHS))) return rc;
    if (col_split && (rc = pcol_h.build(LHS))) return rc;
    // row kernels (k_rows_pipe): one row pair per CTA, whole sequence in one group
    if (!row_split && pipe_bytes(2) > kSmemLimit) prow.dev.stage1 = 1;
    if (!row_split &&
        (prow.threads_for(1) > prow.max_threads() || pipe_bytes(prow.dev.stage1 ? 1 : 2) > kSmemLimit))
      return fail(PU_ERR_UNSUPPORTED, "row length " + std::to_string(m) + " exceeds the shared-memory FFT limit");
    // column kernels (k_cols_spec): panel of W = 2 cc columns
    // 2 sequences (W = 4 columns) per CTA, all in one thread group (<= 512
    // threads) so two CTAs stay resident per SM; the spectral plane is
    // L2-resident between K2b and K4, so 16-byte (fp32) row segments cost L2,
    // not HBM, efficiency
    // static plans use PU_PANEL_COLS (2 packed sequences) in one thread group;
    // runtime plans (odd sizes, Bluestein) fall back to 1 sequence if needed
    const int scc = static_panel_cols(pcol.dev.L, EM, sizeof(T)) / 2;  // sequences per CTA of a static plan
    const bool col_static = !pcol.dev.bluestein && (pcol.dev.L & (pcol.dev.L - 1)) == 0 && pcol.dev.L >= 512 &&
                            pcol.dev.L <= (sizeof(T) == 4 ? 16384 : 8192) && pcol.seq_capacity == EM &&
                            (long long)scc * pcol.dev.L <= 1024LL * pcol.seq_capacity &&
                            pcol.smem_for(scc) <= kSmemLimit;
    int cc = col_static ? scc : PU_PANEL_COLS / 2;
    if (!col_static && pcol.smem_for(cc) > kSmemLimit) cc = 1;
    if (col_split) cc = 1;  // one column pair per cluster
    if (!col_split && (pcol.threads_for(cc) > pcol.max_threads() || pcol.smem_for(cc) > kSmemLimit))
      return fail(PU_ERR_UNSUPPORTED, "column length " + std::to_string(n_glob) + " exceeds the shared-memory FFT limit");
    col_is_static = col_static;
    cols_per_cta = 2 * cc;
    col_threads = pcol.threads_for(cc);
    col_smem = pcol.smem_for(cc);
    // element-wise kernels: block-strided rows, thread-strided columns
    ew_threads = std::min(256, std::max(32, (m + 31) / 32 * 32));
    ew_grid = std::min(n, 148 * 8);
    // (a balanced column grid has at most twice the panels)
    rs.stride = std::max(148 * 8, 2 * ((std::max(m, gc.m) + cols_per_cta - 1) / cols_per_cta)) + 1;
    PU_CUDA(cudaMalloc(&rs.partials, sizeof(double) * PU_MAX_SUMS * rs.stride));
    PU_CUDA(cudaMalloc(&rs.ticket, sizeof(unsigned int) * 32));
    PU_CUDA(cudaMemset(rs.ticket, 0, sizeof(unsigned int) * 32));
    PU_CUDA(cudaMallocHost(&pinned_done, sizeof(int)));
    PU_CUDA(cudaMalloc(&held, sizeof(double) * PU_MAX_SUMS));
    return set_smem_attrs();
  }

  static constexpr int EM = emax_of<T>();

  // dynamic shared memory of the row kernels with `staged` rows of staging
  size_t pipe_bytes(int staged) const {
    const size_t row = std::max<size_t>(stage_row_bytes(prow.dev.n, sizeof(T)),
                                        (size_t)pk.nq * pk.mb * sizeof(T));  // packed band input
    return 128 + staged * row + (size_t)prow.dev.ldseq * 2 * sizeof(T);
  }

  int set_smem_attrs() {
    rops = ops_for<T>(prow.dev.bluestein ? 0 : prow.dev.L);
    cops = ops_for<T>(col_is_static ? pcol.dev.L : 0);
    // the attribute is per kernel (process-wide): always raise it to the cap so
    // that handles of different sizes sharing an instantiation never shrink it
    PU_CUDA(rops.set_attrs(kSmemLimit, kSmemLimit));
    PU_CUDA(cops.set_attrs(kSmemLimit, kSmemLimit));
    if (row_split || col_split) PU_CUDA((SplitLaunch<T, LHS>::set_attrs()));
    if (!col_split) {
      // k_cols_spec is one CTA per SM (shared memory); when the panels leave a
      // partial last wave, turn it into half panels spread over every SM
      // (4096 fp32: 444 panels of 8 columns + 136 of 4 instead of 3.46 waves)
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int per_sm = cops.cols_bps(col_threads, col_smem);
      const int slots = sms * std::max(1, per_sm);
      const int npan = (gc.m + cols_per_cta - 1) / cols_per_cta;
      const int nfull = npan / slots * slots;
      const int nhalf = (gc.m - nfull * cols_per_cta + cols_per_cta / 2 - 1) / (cols_per_cta / 2);
      const bool balance = col_is_static && col_fused_rt(pcol.dev.L, EM) && cols_per_cta >= 8 &&
                           std::getenv("PU_COL_NOBALANCE") == nullptr;
      if (balance && nfull > 0 && npan % slots != 0 && nhalf <= slots) {
        col_nfull = nfull;
        col_nhalf = nhalf;
      } else if (balance && 2 * npan <= sms) {
        // small grids (fewer panels than half the SMs: 512² and 1024²): half
        // panels throughout, twice the CTAs for the same columns
        col_nfull = 0;
        col_nhalf = (gc.m + cols_per_cta / 2 - 1) / (cols_per_cta / 2);
      }
    }
    // persistent pipelined row kernels: one row pair per iteration
    pipe_threads = prow.threads_for(1);
    pipe_smem = pipe_bytes(prow.dev.stage1 ? 1 : 2);
    if (!row_split && pipe_smem > kSmemLimit)
      return fail(PU_ERR_UNSUPPORTED, "row length " + std::to_string(g.m) + " exceeds the row pipeline staging");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int bps = rops.rows_pipe_bps(pipe_threads, pipe_smem);
    pipe_grid = std::max(1, (g.n + 1) / 2);  // one row pair per CTA
    (void)bps;
    return PU_OK;
  }

  // row transform (K2b forward / K4 inverse) and column pass (K3 / API) of
  // the handle's plans: one-CTA kernels, or the 2-CTA cluster split
  cudaError_t rows(bool inv, cudaStream_t st, const T* in, T* out, const PcgCtrl* ctrl, const T* pold, int first,
                   Pack p) {
    if (row_split)
      return SplitLaunch<T, LHS>::rows(inv, (g.n + 1) / 2, st, g, prow.dev, prow_h.dev, in, out, ctrl, pold, first,
                                       p);
    return rops.rows_pipe(inv, pl_(st), g, prow.dev, in, out, ctrl, pold, first, p);
  }
  cudaError_t cols(int mode, cudaStream_t st, T* data, PcgCtrl* ctrl, int it, Push ps) {
    if (col_split)
      return SplitLaunch<T, LHS>::cols(mode, (gc.m + 1) / 2, st, gc, pcol.dev, pcol_h.dev, prow.dev.lam + col0, data,
                                       ctrl, rs, S_K3, it, ps);
    return cops.cols(mode, cl(st), gc, pcol.dev, prow.dev.lam + col0, cols_per_cta, data, ctrl, rs, S_K3, it, ps,
                     col_nfull);
  }

  XLaunch cl(cudaStream_t st) const { return XLaunch{col_grid(), col_threads, col_smem, st, pdl_now}; }
  XLaunch pl_(cudaStream_t st) const { return XLaunch{pipe_grid, pipe_threads, pipe_smem, st, pdl_now}; }

  int col_grid() const { return col_nhalf ? col_nfull + col_nhalf : (gc.m + cols_per_cta - 1) / cols_per_cta; }

  // ---- preconditioner passes ----
  int sylvester(const T* r, T* z, T* spec, cudaStream_t st) {
    PU_DCT(rows(false, st, r, spec, nullptr, nullptr, 0, Pack{}));
    PU_DCT(cols(MODE_API, st, spec, nullptr, 0, Push{}));
    PU_DCT(rows(true, st, spec, z, nullptr, nullptr, 0, Pack{}));
    return PU_OK;
  }

  int vec_grid() const {
    const long long chunks = (long long)g.n * ((g.m + 3) / 4);
    return (int)std::max<long long>(1, std::min<long long>((chunks + 255) / 256, 148 * 8));
  }

  // One fused PCG solve (pcg.py:47-116); 5 kernels per iteration:
  // K1 p/Ap/p'Ap, K2a residual update + slack precond + norms, K2b row DCT-II,
  // K3 column DCT pair + spectral division + rho, K4 row DCT-III.
  int pcg(const T* b, const T* x0, T* x, const T* dv, const T* dh, T* r, T* z, T* p0, T* p1, T* spec,
          int max_iters, double rel_tol, PcgCtrl* ctrl, double* norms, cudaStream_t st,
          const CandArgs<T>* cand = nullptr) {
    PU_RC(pcg_setup(b, x0, x, dv, dh, r, p0, p1, spec, max_iters, rel_tol, ctrl, norms, st, cand));
    return pcg_iterate(x, dv, dh, r, p0, p1, spec, max_iters, ctrl, norms, st);
  }

  // pcg.py:59-79: start-up (+ the candidate step) and z0 = M r0, p0 = z0
  int pcg_setup(const T* b, const T* x0, T* x, const T* dv, const T* dh, T* r, T* p0, T* p1, T* spec,
                int max_iters, double rel_tol, PcgCtrl* ctrl, double* norms, cudaStream_t st,
                const CandArgs<T>* cand, bool prestarted = false) {
    const int vg = vec_grid();
    cudaEvent_t e = tm.begin(st);
    if (prestarted) {  // r and cand came from k_accept_start_v; its sums wait in `held`
      k_fin_start_held<<<1, 32, 0, st>>>(ctrl, norms, held, rel_tol, max_iters);
    } else if (cand && !b) {  // b = build_rhs(gv, gh) formed in the kernel
      k_pcg_start_v<T, true, true><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs,
                                                        S_START, *cand);
    } else if (cand) {
      k_pcg_start_v<T, true><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs, S_START,
                                                  *cand);
    } else {
      k_pcg_start_v<T, false><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs,
                                                   S_START, CandArgs<T>{});
    }
    PU_LAUNCH_CHECK();
    tm.end(st, e, TK_START, -1);
    // z = M r, rho = r.z (pcg.py:77-79); rho_s came with the start-up sums
    e = tm.begin(st);
    PU_DCT(rows(false, st, r, spec, ctrl, nullptr, 0, Pack{}));
    tm.end(st, e, TK_K2B, -1);
    e = tm.begin(st);
    PU_DCT(cols(MODE_INIT, st, spec, ctrl, -1, Push{}));
    tm.end(st, e, TK_K3, -1);
    // p of iteration k lives in pbuf[k & 1]; K4 writes its u block (p = z at k = 0)
    T* pbuf[2] = {p0, p1};
    e = tm.begin(st);
    PU_DCT(rows(true, st, spec, pbuf[0], ctrl, pbuf[1], 1, Pack{}));
    tm.end(st, e, TK_K4, -1);
    return PU_OK;
  }

  // pcg.py:81-108: the iterations of one budget
  int pcg_iterate(T* x, const T* dv, const T* dh, T* r, T* p0, T* p1, T* spec, int max_iters, PcgCtrl* ctrl,
                  double* norms, cudaStream_t st) {
    const int vg = vec_grid();
    // PDL only without per-launch timing events (an event between two
    // kernels breaks the programmatic edge)
    const bool pdl = pdl_mode > 0 && !tm.on;
    struct PdlScope { bool& f; PdlScope(bool& f_, bool v) : f(f_) { f = v; } ~PdlScope() { f = false; } } scope(pdl_now, pdl);
    cudaEvent_t e;
    T* pbuf[2] = {p0, p1};
    const int chunk = 64;
    for (int it = 0; it < max_iters; ++it) {
      if (it > 0 && it % chunk == 0) {
        PU_CUDA(cudaMemcpyAsync(pinned_done, &ctrl->done, sizeof(int), cudaMemcpyDeviceToHost, st));
        PU_CUDA(cudaStreamSynchronize(st));
        if (*pinned_done) break;
      }
      T* pn = pbuf[it & 1];
      const T* po = pbuf[(it + 1) & 1];
      e = tm.begin(st);
      PU_DCT(launch_k(k_pcg_p_v<T>, vg, 256, 0, st, pdl, g, r, po, pn, dv, dh, ctrl, rs, (int)S_K1, it));
      tm.end(st, e, TK_K1, it);
      if ((it + 1) % 50 == 0) {
        e = tm.begin(st);
        k_pcg_upd_sum_v<T><<<vg, 256, 0, st>>>(g, pn, dv, dh, x, r, ctrl, rs, S_UPD);
        PU_LAUNCH_CHECK();
        tm.end(st, e, TK_UPD, it);
        e = tm.begin(st);
        k_pcg_r_v<T, false, true, MODE_ITER><<<vg, 256, 0, st>>>(g, pn, dv, dh, x, r, ctrl, norms, rs, S_K2, it);
        PU_LAUNCH_CHECK();
        tm.end(st, e, TK_K2, it);
      } else {
        e = tm.begin(st);
        PU_DCT(launch_k(k_pcg_r_v<T, true, false, MODE_ITER>, vg, 256, 0, st, pdl, g, (const T*)pn, dv, dh, x, r,
                        ctrl, norms, rs, (int)S_K2, it));
        tm.end(st, e, TK_K2, it);
      }
      e = tm.begin(st);
      PU_DCT(rows(false, st, r, spec, ctrl, nullptr, 0, Pack{}));
      tm.end(st, e, TK_K2B, it);
      e = tm.begin(st);
      PU_DCT(cols(MODE_ITER, st, spec, ctrl, it, Push{}));
      tm.end(st, e, TK_K3, it);
      e = tm.begin(st);  // u block of p for iteration it + 1: beta p_u + z_u
      PU_DCT(rows(true, st, spec, pbuf[(it + 1) & 1], ctrl, pn, 0, Pack{}));
      tm.end(st, e, TK_K4, it);
    }
    return PU_OK;
  }

  // ---- the same iteration as separate launches, for row-sharded grids (the
  // host all-reduces the band totals and calls finalize() between them; see
  // paper_2401_09961_b200/band.py).  On a whole grid they reproduce pcg(). ----
  int pcg_begin(const T* b, const T* x0, T* x, const T* dv, const T* dh, T* r, PcgCtrl* ctrl, double* norms,
                double rel_tol, int max_iters, const CandArgs<T>* cand, cudaStream_t st) {
    const int vg = vec_grid();
    cudaEvent_t e = tm.begin(st);
    if (cand && !b)  // b = build_rhs(gv, gh) formed in the kernel
      k_pcg_start_v<T, true, true><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs,
                                                        S_START, *cand);
    else if (cand)
      k_pcg_start_v<T, true><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs, S_START,
                                                  *cand);
    else
      k_pcg_start_v<T, false><<<vg, 256, 0, st>>>(g, b, x0, x, r, dv, dh, ctrl, norms, rel_tol, max_iters, rs,
                                                   S_START, CandArgs<T>{});
    PU_LAUNCH_CHECK();
    tm.end(st, e, TK_START, -1);
    return PU_OK;
  }

  // K2a (it < 0: initial rho_s only; submean: the every-50 re-projection
  // after pcg_update_sum) then K2b, the row DCT-II of r_u into spec_out
  // (packed for the transpose in band mode)
  int pcg_residual_rows(const T* p, const T* dv, const T* dh, T* x, T* r, PcgCtrl* ctrl, double* norms, T* spec_out,
                        int it, int submean, cudaStream_t st) {
    const int vg = vec_grid();
    cudaEvent_t e = tm.begin(st);
    if (it < 0) {  // set-up: rho_s of r0 came with pu_pcg_begin; only the row transform
      PU_DCT(rows(false, st, r, spec_out, ctrl, nullptr, 0, pk));
      tm.end(st, e, TK_K2B, it);
      return PU_OK;
    }
    if (submean)
      k_pcg_r_v<T, false, true, MODE_ITER><<<vg, 256, 0, st>>>(g, p, dv, dh, x, r, ctrl, norms, rs, S_K2, it);
    else
      k_pcg_r_v<T, true, false, MODE_ITER><<<vg, 256, 0, st>>>(g, p, dv, dh, x, r, ctrl, norms, rs, S_K2, it);
    PU_LAUNCH_CHECK();
    tm.end(st, e, TK_K2, it);
    e = tm.begin(st);
    PU_DCT(rows(false, st, r, spec_out, ctrl, nullptr, 0, pk));
    tm.end(st, e, TK_K2B, it);
    return PU_OK;
  }

  int pcg_update_sum(const T* p, const T* dv, const T* dh, T* x, T* r, PcgCtrl* ctrl, int it, cudaStream_t st) {
    cudaEvent_t e = tm.begin(st);
    k_pcg_upd_sum_v<T><<<vec_grid(), 256, 0, st>>>(g, p, dv, dh, x, r, ctrl, rs, S_UPD);
    PU_LAUNCH_CHECK();
    tm.end(st, e, TK_UPD, it);
    return PU_OK;
  }

  // K3 on the (column block of the) spectrum, in place
  int pcg_columns(T* spec, PcgCtrl* ctrl, int it, cudaStream_t st) {
    cudaEvent_t e = tm.begin(st);
    PU_DCT(cols(it < 0 ? MODE_INIT : MODE_ITER, st, spec, ctrl, it, push));
    tm.end(st, e, TK_K3, it);
    return PU_OK;
  }

  // K4: u block of the next direction, pnew_u = beta pold_u + DCT-III rows (first: no axpy)
  int pcg_rows_inv(const T* spec_in, T* pnew, const T* pold, int first, PcgCtrl* ctrl, int it, cudaStream_t st) {
    cudaEvent_t e = tm.begin(st);
    // the packed rows come from the local buffer (pushed there by K3 in peer
    // mode), this rank's own chunk from its column block (K3 left it in place)
    Pack local = pk;
    if (local.peers) local.own_q = col0 / pk.mb;
    PU_DCT(rows(true, st, spec_in, pnew, ctrl, pold, first, local));
    tm.end(st, e, TK_K4, it);
    return PU_OK;
  }

  // K1 (band mode: after the ghost-row slack of the new direction)
  int pcg_direction(const T* r, const T* pold, T* pnew, const T* dv, const T* dh, PcgCtrl* ctrl, int it,
                    cudaStream_t st) {
    cudaEvent_t e = tm.begin(st);
    if (g.top) {
      const int thr = 256, blocks = std::max(1, std::min(148, (g.m / 4 + thr - 1) / thr));
      k_ghost_pslack<T><<<blocks, thr, 0, st>>>(g, r, pold, pnew, dv, ctrl, it);
      PU_LAUNCH_CHECK();
    }
    k_pcg_p_v<T><<<vec_grid(), 256, 0, st>>>(g, r, pold, pnew, dv, dh, ctrl, rs, S_K1, it);
    PU_LAUNCH_CHECK();
    tm.end(st, e, TK_K1, it);
    return PU_OK;
  }
};

}  // namespace pu

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace pu;

struct pu_handle {
  int dtype;
  Impl<float>* f = nullptr;
  Impl<double>* d = nullptr;
};

#define PU_DISPATCH(h, ...)                            \
  do {                                                 \
    if (!(h)) return fail(PU_ERR_ARG, "null handle");  \
    if ((h)->dtype == PU_F32) {                        \
      using T = float;                                 \
      auto& I = *(h)->f;                               \
      __VA_ARGS__                                      \
    } else {                                           \
      using T = double;                                \
      auto& I = *(h)->d;                               \
      __VA_ARGS__                                      \
    }                                                  \
  } while (0)

#define ST(s) reinterpret_cast<cudaStream_t>(s)
#define CP(p) reinterpret_cast<const T*>(p)
#define MP(p) reinterpret_cast<T*>(p)

extern "C" {

int pu_abi_version(void) { return PU_ABI_VERSION; }
int64_t pu_launch_count(void) { return g_launches.load(); }
const char* pu_last_error(void) { return g_last_error.c_str(); }
int pu_pcg_ctrl_bytes(void) { return (int)sizeof(pu_pcg_ctrl); }

int pu_create(pu_handle** out, int n, int m, int dtype, double tau, double delta) {
  if (!out) return fail(PU_ERR_ARG, "null output");
  *out = nullptr;
  if (n < 1 || m < 1) return fail(PU_ERR_ARG, "grid dimensions must be >= 1");
  if (!(tau > 0) || !std::isfinite(tau)) return fail(PU_ERR_ARG, "tau must be positive and finite");
  if (!(delta > 0) || !std::isfinite(delta)) return fail(PU_ERR_ARG, "delta must be positive and finite");
  if (dtype != PU_F32 && dtype != PU_F64) return fail(PU_ERR_ARG, "dtype must be PU_F32 or PU_F64");
  pu_handle* h = new pu_handle();
  h->dtype = dtype;
  int rc;
  if (dtype == PU_F32) {
    h->f = new Impl<float>();
    rc = h->f->init(n, m, tau, delta);
  } else {
    h->d = new Impl<double>();
    rc = h->d->init(n, m, tau, delta);
  }
  if (rc != PU_OK) {
    std::string keep = g_last_error;
    delete h->f;
    delete h->d;
    delete h;
    g_last_error = keep;
    return rc;
  }
  *out = h;
  return PU_OK;
}

int pu_destroy(pu_handle* h) {
  if (!h) return PU_OK;
  delete h->f;
  delete h->d;
  delete h;
  return PU_OK;
}

int64_t pu_pitch(const pu_handle* h) { return h ? (h->dtype == PU_F32 ? h->f->g.ld : h->d->g.ld) : -1; }
int64_t pu_plane_elems(const pu_handle* h) { return h ? (h->dtype == PU_F32 ? h->f->g.plane : h->d->g.plane) : -1; }

int pu_describe(const pu_handle* h, char* buf, int cap) {
  if (!h || !buf || cap < 1) return fail(PU_ERR_ARG, "bad arguments");
  auto fmt = [&](auto& I) {
    std::snprintf(buf, cap,
                  "{\"n\":%d,\"m\":%d,\"ld\":%lld,\"dtype\":\"%s\",\"row_fft\":{\"n\":%d,\"L\":%d,\"bluestein\":%d,"
                  "\"stages\":%d,\"split\":%d},\"col_fft\":{\"n\":%d,\"L\":%d,\"bluestein\":%d,\"stages\":%d,"
                  "\"split\":%d},"
                  "\"row_pipe_grid\":%d,\"row_threads\":%d,\"row_smem\":%zu,\"cols_per_cta\":%d,"
                  "\"col_grid\":%d,\"col_half_panels\":%d,\"col_threads\":%d,\"col_smem\":%zu,\"ew_grid\":%d,"
                  "\"ew_threads\":%d}",
                  I.g.n, I.g.m, I.g.ld, h->dtype == PU_F32 ? "f32" : "f64", I.prow.dev.n, I.prow.dev.L,
                  I.prow.dev.bluestein, I.prow.dev.nst, (int)I.row_split, I.pcol.dev.n, I.pcol.dev.L,
                  I.pcol.dev.bluestein, I.pcol.dev.nst, (int)I.col_split, I.pipe_grid, I.pipe_threads, I.pipe_smem, I.cols_per_cta, I.col_grid(), I.col_nhalf, I.col_threads,
                  I.col_smem, I.ew_grid, I.ew_threads);
  };
  if (h->dtype == PU_F32) fmt(*h->f); else fmt(*h->d);
  return PU_OK;
}

int pu_pack(pu_handle* h, const double* src, int64_t lds, int rows, int cols, void* dst, void* stream) {
  PU_DISPATCH(h, {
    k_pack<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, src, lds, rows, cols, MP(dst));
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_unpack(pu_handle* h, const void* src, int rows, int cols, double* dst, void* stream) {
  PU_DISPATCH(h, {
    if (rows > 0 && cols > 0) {
      k_unpack<T, double><<<std::min(rows, 148 * 8), I.ew_threads, 0, ST(stream)>>>(I.g, CP(src), rows, cols, dst);
      PU_LAUNCH_CHECK();
    }
  });
  return PU_OK;
}

int pu_unpack_native(pu_handle* h, const void* src, int rows, int cols, void* dst, void* stream) {
  PU_DISPATCH(h, {
    if (rows > 0 && cols > 0) {
      k_unpack<T, T><<<std::min(rows, 148 * 8), I.ew_threads, 0, ST(stream)>>>(I.g, CP(src), rows, cols, MP(dst));
      PU_LAUNCH_CHECK();
    }
  });
  return PU_OK;
}

int pu_fill(pu_handle* h, void* dst, int nplanes, double value, void* stream) {
  PU_DISPATCH(h, {
    k_fill<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, MP(dst), nplanes, (T)value);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_copy(pu_handle* h, const void* src, void* dst, int nplanes, void* stream) {
  PU_DISPATCH(h, {
    k_copy<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(src), MP(dst), nplanes);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_wrapped_gradients(pu_handle* h, const double* x, int64_t ldx, void* gv, void* gh, double lo, void* stream) {
  if (!(lo == 0.0 || lo == -3.141592653589793)) return fail(PU_ERR_ARG, "lo must be 0 or -pi");
  PU_DISPATCH(h, {
    k_grad<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, x, ldx, MP(gv), MP(gh), lo);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_wrapped_gradients_checked(pu_handle* h, const double* x, int64_t ldx, void* gv, void* gh, double lo,
                                 double* check, void* stream) {
  if (!(lo == 0.0 || lo == -3.141592653589793)) return fail(PU_ERR_ARG, "lo must be 0 or -pi");
  if (!check) return fail(PU_ERR_ARG, "check must not be NULL");
  PU_DISPATCH(h, {
    if (I.band) return fail(PU_ERR_ARG, "pu_wrapped_gradients_checked runs on whole grids");
    k_grad_check<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, x, ldx, MP(gv), MP(gh), lo, I.rs, S_CHK,
                                                               check);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_init_state(pu_handle* h, const void* gv, const void* gh, void* x, void* stream) {
  PU_DISPATCH(h, {
    k_init_state<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(gv), CP(gh), MP(x));
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_build_rhs(pu_handle* h, const void* gv, const void* gh, void* b, void* stream) {
  PU_DISPATCH(h, {
    k_rhs<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(gv), CP(gh), MP(b));
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_apply_system(pu_handle* h, const void* x, const void* dv, const void* dh, void* y, void* stream) {
  PU_DISPATCH(h, {
    k_apply_system<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(x), CP(dv), CP(dh), MP(y));
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_dot(pu_handle* h, const void* a, const void* b, int nplanes, double* out, void* stream) {
  if (nplanes < 1 || nplanes > 3) return fail(PU_ERR_ARG, "nplanes must be 1..3");
  PU_DISPATCH(h, {
    k_dot<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(a), CP(b), nplanes, I.rs, S_DOT, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_sylvester_solve(pu_handle* h, const void* r, void* z, void* spec, void* stream) {
  PU_DISPATCH(h, { return I.sylvester(CP(r), MP(z), MP(spec), ST(stream)); });
}

int pu_apply_preconditioner(pu_handle* h, const void* r, const void* dv, const void* dh, void* z, void* spec,
                            void* stream) {
  PU_DISPATCH(h, {
    k_precond_slack<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(r), CP(dv), CP(dh), MP(z));
    PU_LAUNCH_CHECK();
    return I.sylvester(CP(r), MP(z), MP(spec), ST(stream));
  });
}

int pu_weights_hpair(pu_handle* h, const void* x, const void* cv, const void* ch, const void* gv, const void* gh,
                     const void* wpv, const void* wph, void* wv, void* wh, void* dv, void* dh, double* out,
                     void* stream) {
  PU_DISPATCH(h, {
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_weights_hpair_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(I.g, CP(x), CP(cv), CP(ch), CP(gv), CP(gh),
                                                                  CP(wpv), CP(wph), MP(wv), MP(wh), MP(dv), MP(dh),
                                                                  I.rs, S_WH, out);
    PU_LAUNCH_CHECK();
    I.tm.end(ST(stream), te_, TK_WEIGHTS, -1);
  });
  return PU_OK;
}

int pu_eval_h_delta(pu_handle* h, const void* x, const void* wv, const void* wh, const void* gv, const void* gh,
                    const void* cv, const void* ch, double* out, void* stream) {
  PU_DISPATCH(h, {
    k_eval_h<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(x), CP(wv), CP(wh), CP(gv), CP(gh), CP(cv),
                                                           CP(ch), I.rs, S_EVH, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_eval_f(pu_handle* h, const void* x, const void* gv, const void* gh, const void* cv, const void* ch,
              double* out, void* stream) {
  PU_DISPATCH(h, {
    k_eval_f<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(x), CP(gv), CP(gh), CP(cv), CP(ch), I.rs,
                                                           S_EVF, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_shift_error(pu_handle* h, const void* u, const double* xu, int64_t ldx, double* out, void* stream) {
  PU_DISPATCH(h, {
    if (I.band) return fail(PU_ERR_ARG, "metrics need a whole-grid handle");
    k_shift_alpha<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(u), xu, ldx, I.rs, S_MET, out);
    PU_LAUNCH_CHECK();
    k_shift_stats<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(u), xu, ldx, I.rs, S_MET, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_kmap_mismatch(pu_handle* h, const void* u, const double* uref, int64_t ldr, const double* x, int64_t ldx,
                     double* out, void* stream) {
  PU_DISPATCH(h, {
    if (I.band) return fail(PU_ERR_ARG, "metrics need a whole-grid handle");
    k_kmap<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(u), uref, ldr, x, ldx, I.rs, S_MET, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_congruent_round(pu_handle* h, const void* u, const double* x, int64_t ldx, double* out, void* stream) {
  PU_DISPATCH(h, {
    k_congruent<T><<<I.ew_grid, I.ew_threads, 0, ST(stream)>>>(I.g, CP(u), x, ldx, out);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_candidate_step(pu_handle* h, const void* x, const void* wv, const void* wh, const void* gv, const void* gh,
                      const void* cv, const void* ch, double lipschitz, void* out, void* stream) {
  if (!(lipschitz > 0)) return fail(PU_ERR_ARG, "lipschitz constant must be positive");
  PU_DISPATCH(h, {
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_candidate_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(I.g, CP(x), CP(wv), CP(wh), CP(gv), CP(gh), CP(cv),
                                                              CP(ch), (T)(-1.0 / lipschitz), MP(out));
    PU_LAUNCH_CHECK();
    I.tm.end(ST(stream), te_, TK_CAND, -1);
  });
  return PU_OK;
}

int pu_hpair_states(pu_handle* h, const void* xa, const void* xb, const void* wv, const void* wh, const void* gv,
                    const void* gh, const void* cv, const void* ch, double* out, void* stream) {
  PU_DISPATCH(h, {
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_hpair_states_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(I.g, CP(xa), CP(xb), CP(wv), CP(wh), CP(gv),
                                                                 CP(gh), CP(cv), CP(ch), I.rs, S_HPAIR, out);
    PU_LAUNCH_CHECK();
    I.tm.end(ST(stream), te_, TK_HPAIR, -1);
  });
  return PU_OK;
}

int pu_accept_center(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst, const void* wv,
                     const void* wh, const void* gv, const void* gh, const void* cv, const void* ch, double* out,
                     void* stream) {
  if (dst == xa || dst == xb) return fail(PU_ERR_ARG, "dst must not alias xa or xb");
  PU_DISPATCH(h, {
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_accept_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(I.g, CP(xa), CP(xb), sel, MP(dst), CP(wv), CP(wh),
                                                           CP(gv), CP(gh), CP(cv), CP(ch), I.rs, S_ACC, out);
    PU_LAUNCH_CHECK();
    I.tm.end(ST(stream), te_, TK_ACCEPT, -1);
  });
  return PU_OK;
}

}  // extern "C"

// Replays `body` (which enqueues kernels on st) as a CUDA graph cached under
// `key` when graphs are on and the stream is capturable; else runs it eagerly.
template <typename I_t, typename F>
static int run_graph(I_t& I, std::vector<unsigned long long> key, cudaStream_t st, bool eligible, F&& body) {
  if (!I.use_graphs || st == nullptr || !eligible) return body();
  key.push_back((unsigned long long)I.tm.on);
  key.push_back((unsigned long long)(uintptr_t)st);
  auto found = I.graphs.m.find(key);
  if (found == I.graphs.m.end()) {
    if (I.graphs.m.size() >= 96) I.graphs.clear();
    GraphEntry ent;
    I.tm.sink = &ent.timed;
    PU_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const long long l0 = g_launches.load();
    const int rc = body();
    ent.kernels = g_launches.load() - l0;
    g_launches.fetch_sub(ent.kernels);  // counted per replay below
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    I.tm.sink = nullptr;
    if (rc != PU_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
    PU_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&ent.exec, graph, 0);
    cudaGraphDestroy(graph);
    PU_CUDA(ie);
    found = I.graphs.m.emplace(key, std::move(ent)).first;
  }
  PU_CUDA(cudaGraphLaunch(found->second.exec, st));
  g_launches.fetch_add(found->second.kernels);
  if (I.tm.on)
    for (const auto& rec : found->second.timed) I.tm.recs.push_back(Timer::Rec{rec.kind, rec.it, rec.a, rec.b, false});
  return PU_OK;
}

static unsigned long long dbits(double v) {
  union { double d; unsigned long long u; } x{v};
  return x.u;
}
#define PU_KP(p) ((unsigned long long)(uintptr_t)(p))

// the budget of a loop whose start-up ran with a placeholder (pu_irls_begin)
__global__ void k_set_max_iters(PcgCtrl* ctrl, int max_iters) {
  if (threadIdx.x == 0 && blockIdx.x == 0) ctrl->max_iters = max_iters;
}

extern "C" {

int pu_irls_begin(pu_handle* h, void* state, const void* b, const void* gv, const void* gh, const void* cv,
                  const void* ch, const void* wv, const void* wh, const void* dv, const void* dh, double lipschitz,
                  double rel_tol, void* cand, void* r, void* p0, void* p1, void* spec, void* ctrl, double* res_norms,
                  void* stream) {
  if (rel_tol < 0) return fail(PU_ERR_ARG, "rel_tol must be >= 0");
  if (!(lipschitz > 0)) return fail(PU_ERR_ARG, "lipschitz constant must be positive");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  PU_DISPATCH(h, {
    I.held_pending = false;  // a full start-up supersedes any held accept_start sums
    cudaStream_t st = ST(stream);
    auto body = [&]() -> int {
      const CandArgs<T> ca{CP(gv), CP(gh), CP(cv), CP(ch), CP(wv), CP(wh), (T)(-1.0 / lipschitz), MP(cand)};
      // the budget is not known yet: a placeholder (never 0) until pu_irls_iterate sets it
      return I.pcg_setup(CP(b), CP(state), MP(state), CP(dv), CP(dh), MP(r), MP(p0), MP(p1), MP(spec), 1 << 30,
                         rel_tol, reinterpret_cast<PcgCtrl*>(ctrl), res_norms, st, &ca);
    };
    return run_graph(I, {1ull, dbits(lipschitz), dbits(rel_tol), PU_KP(state), PU_KP(b), PU_KP(gv), PU_KP(gh),
                         PU_KP(cv), PU_KP(ch), PU_KP(wv), PU_KP(wh), PU_KP(dv), PU_KP(dh), PU_KP(cand), PU_KP(r),
                         PU_KP(p0), PU_KP(p1), PU_KP(spec), PU_KP(ctrl), PU_KP(res_norms)},
                     st, true, body);
  });
}

int pu_irls_iterate(pu_handle* h, void* state, const void* gv, const void* gh, const void* cv, const void* ch,
                    const void* wv, const void* wh, const void* dv, const void* dh, int max_iters, void* cand, void* r,
                    void* p0, void* p1, void* spec, void* ctrl, double* res_norms, double* out, void* stream) {
  if (max_iters < 0) return fail(PU_ERR_ARG, "max_iters must be >= 0");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  PU_DISPATCH(h, {
    cudaStream_t st = ST(stream);
    auto body = [&]() -> int {
      PcgCtrl* c = reinterpret_cast<PcgCtrl*>(ctrl);
      k_set_max_iters<<<1, 32, 0, st>>>(c, max_iters);
      PU_LAUNCH_CHECK();
      PU_RC(I.pcg_iterate(MP(state), CP(dv), CP(dh), MP(r), MP(p0), MP(p1), MP(spec), max_iters, c, res_norms, st));
      cudaEvent_t te_ = I.tm.begin(st);
      k_hpair_states_v<T><<<I.vec_grid(), 256, 0, st>>>(I.g, CP(state), CP(cand), CP(wv), CP(wh), CP(gv), CP(gh),
                                                         CP(cv), CP(ch), I.rs, S_HPAIR, out);
      PU_LAUNCH_CHECK();
      I.tm.end(st, te_, TK_HPAIR, -1);
      return PU_OK;
    };
    return run_graph(I, {2ull, (unsigned long long)max_iters, PU_KP(state), PU_KP(gv), PU_KP(gh), PU_KP(cv),
                         PU_KP(ch), PU_KP(wv), PU_KP(wh), PU_KP(dv), PU_KP(dh), PU_KP(cand), PU_KP(r), PU_KP(p0),
                         PU_KP(p1), PU_KP(spec), PU_KP(ctrl), PU_KP(res_norms), PU_KP(out)},
                     st, max_iters <= 64, body);
  });
}

int pu_irls_step(pu_handle* h, void* state, const void* b, const void* gv, const void* gh, const void* cv,
                 const void* ch, const void* wv, const void* wh, const void* dv, const void* dh, double lipschitz,
                 int max_iters, double rel_tol, void* cand, void* r, void* p0, void* p1, void* spec, void* ctrl,
                 double* res_norms, double* out, void* stream) {
  if (max_iters < 0) return fail(PU_ERR_ARG, "max_iters must be >= 0");
  if (rel_tol < 0) return fail(PU_ERR_ARG, "rel_tol must be >= 0");
  if (!(lipschitz > 0)) return fail(PU_ERR_ARG, "lipschitz constant must be positive");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  PU_DISPATCH(h, {
    cudaStream_t st = ST(stream);
    auto body = [&]() -> int {
      const CandArgs<T> ca{CP(gv), CP(gh), CP(cv), CP(ch), CP(wv), CP(wh), (T)(-1.0 / lipschitz), MP(cand)};
      int rc = I.pcg(CP(b), CP(state), MP(state), CP(dv), CP(dh), MP(r), nullptr, MP(p0), MP(p1), MP(spec),
                     max_iters, rel_tol, reinterpret_cast<PcgCtrl*>(ctrl), res_norms, st, &ca);
      if (rc != PU_OK) return rc;
      cudaEvent_t te_ = I.tm.begin(st);
      k_hpair_states_v<T><<<I.vec_grid(), 256, 0, st>>>(I.g, CP(state), CP(cand), CP(wv), CP(wh), CP(gv), CP(gh),
                                                         CP(cv), CP(ch), I.rs, S_HPAIR, out);
      PU_LAUNCH_CHECK();
      I.tm.end(st, te_, TK_HPAIR, -1);
      return PU_OK;
    };
    // graphs need a capturable (non-legacy) stream and a budget that the
    // enqueue loop runs without polling (<= 64 iterations)
    return run_graph(I, {0ull, (unsigned long long)max_iters, dbits(lipschitz), dbits(rel_tol), PU_KP(state),
                         PU_KP(b), PU_KP(gv), PU_KP(gh), PU_KP(cv), PU_KP(ch), PU_KP(wv), PU_KP(wh), PU_KP(dv),
                         PU_KP(dh), PU_KP(cand), PU_KP(r), PU_KP(p0), PU_KP(p1), PU_KP(spec), PU_KP(ctrl),
                         PU_KP(res_norms), PU_KP(out)},
                     st, max_iters <= 64, body);
  });
}

int pu_set_graphs(pu_handle* h, int on) {
  PU_DISPATCH(h, {
    I.use_graphs = on != 0;
    if (!I.use_graphs) I.graphs.clear();
  });
  return PU_OK;
}

int pu_accept_weights(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst, const void* gv,
                      const void* gh, const void* cv, const void* ch, const void* wkv, const void* wkh, void* wnv,
                      void* wnh, void* dv, void* dh, double* out, void* stream) {
  if (dst == xa || dst == xb) return fail(PU_ERR_ARG, "dst must not alias xa or xb");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  PU_DISPATCH(h, {
    I.held_pending = false;  // the plain acceptance leaves no start-up sums behind
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_accept_weights_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(I.g, CP(xa), CP(xb), sel, MP(dst), CP(gv), CP(gh),
                                                               CP(cv), CP(ch), CP(wkv), CP(wkh), MP(wnv), MP(wnh),
                                                               MP(dv), MP(dh), I.rs, S_ACC, out);
    PU_LAUNCH_CHECK();
    I.tm.end(ST(stream), te_, TK_ACCEPT, -1);
  });
  return PU_OK;
}

int pu_accept_weights_start(pu_handle* h, const void* xa, const void* xb, const double* sel, void* dst,
                            const void* gv, const void* gh, const void* cv, const void* ch, const void* wkv,
                            const void* wkh, void* wnv, void* wnh, void* dv, void* dh, double* out, double lipschitz,
                            void* r, void* cand, void* stream) {
  if (dst == xa || dst == xb) return fail(PU_ERR_ARG, "dst must not alias xa or xb");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  if (!(lipschitz > 0)) return fail(PU_ERR_ARG, "lipschitz constant must be positive");
  if (!r || !cand || !gv || !gh) return fail(PU_ERR_ARG, "r, cand, gv and gh are required");
  PU_DISPATCH(h, {
    cudaEvent_t te_ = I.tm.begin(ST(stream));
    k_accept_start_v<T><<<I.vec_grid(), 256, 0, ST(stream)>>>(
        I.g, CP(xa), CP(xb), sel, MP(dst), CP(gv), CP(gh), CP(cv), CP(ch), CP(wkv), CP(wkh), MP(wnv), MP(wnh),
        MP(dv), MP(dh), I.rs, S_ACC, out, MP(r), (T)(-1.0 / lipschitz), MP(cand), I.held);
    PU_LAUNCH_CHECK();
    I.held_pending = !I.band;  // bands: the start-up sums are in the totals (finalised with pu_finalize)
    I.tm.end(ST(stream), te_, TK_ACCEPT, -1);
  });
  return PU_OK;
}

int pu_irls_begin_z0(pu_handle* h, const void* dv, const void* dh, double rel_tol, void* r, void* p0, void* p1,
                     void* spec, void* ctrl, double* res_norms, void* stream) {
  if (rel_tol < 0) return fail(PU_ERR_ARG, "rel_tol must be >= 0");
  PU_DISPATCH(h, {
    if (!I.held_pending) return fail(PU_ERR_ARG, "pu_irls_begin_z0 must follow pu_accept_weights_start");
    I.held_pending = false;
    cudaStream_t st = ST(stream);
    auto body = [&]() -> int {
      return I.pcg_setup(nullptr, nullptr, nullptr, CP(dv), CP(dh), MP(r), MP(p0), MP(p1), MP(spec), 1 << 30,
                         rel_tol, reinterpret_cast<PcgCtrl*>(ctrl), res_norms, st, nullptr, true);
    };
    return run_graph(I, {3ull, dbits(rel_tol), PU_KP(dv), PU_KP(dh), PU_KP(r), PU_KP(p0), PU_KP(p1), PU_KP(spec),
                         PU_KP(ctrl), PU_KP(res_norms)},
                     st, true, body);
  });
}

int pu_timing_enable(pu_handle* h, int on) {
  PU_DISPATCH(h, { I.tm.on = on != 0; });
  return PU_OK;
}

int pu_timing_read(pu_handle* h, int* kinds, int* its, float* ms, int cap) {
  if (!kinds || !its || !ms || cap < 0) return -1;
  PU_DISPATCH(h, { return I.tm.read(kinds, its, ms, cap); });
}

int pu_pcg_solve(pu_handle* h, const void* b, const void* x0, void* x, const void* dv, const void* dh, void* r,
                 void* z, void* p0, void* p1, void* spec, int max_iters, double rel_tol, void* ctrl, double* res_norms,
                 void* stream) {
  if (max_iters < 0) return fail(PU_ERR_ARG, "max_iters must be >= 0");
  if (rel_tol < 0) return fail(PU_ERR_ARG, "rel_tol must be >= 0");
  if (!b) return fail(PU_ERR_ARG, "b must not be NULL");
  PU_DISPATCH(h, {
    return I.pcg(CP(b), CP(x0), MP(x), CP(dv), CP(dh), MP(r), MP(z), MP(p0), MP(p1), MP(spec), max_iters, rel_tol,
                 reinterpret_cast<PcgCtrl*>(ctrl), res_norms, ST(stream));
  });
}

int pu_create_band(pu_handle** out, int m, const pu_band* b, int dtype, double tau, double delta) {
  if (!out || !b) return fail(PU_ERR_ARG, "null argument");
  *out = nullptr;
  if (b->n_glob < 2 || m < 1 || b->rows < 1 || b->row0 < 0 || b->row0 + b->rows > b->n_glob)
    return fail(PU_ERR_ARG, "invalid row band");
  if (b->nq < 1 || b->mb < 8 || b->mb % 8 != 0 || (long long)b->nq * b->mb < m)
    return fail(PU_ERR_ARG, "transpose chunks: mb must be a multiple of 8 with nq * mb >= M");
  if (b->col0 < 0 || b->cols < 1 || b->cols > b->mb || b->col0 + b->cols > m || b->col0 % b->mb != 0)
    return fail(PU_ERR_ARG, "invalid column block");
  if (!(tau > 0) || !std::isfinite(tau)) return fail(PU_ERR_ARG, "tau must be positive and finite");
  if (!(delta > 0) || !std::isfinite(delta)) return fail(PU_ERR_ARG, "delta must be positive and finite");
  if (dtype != PU_F32 && dtype != PU_F64) return fail(PU_ERR_ARG, "dtype must be PU_F32 or PU_F64");
  pu_handle* h = new pu_handle();
  h->dtype = dtype;
  int rc;
  if (dtype == PU_F32) {
    h->f = new Impl<float>();
    rc = h->f->init(b->rows, m, tau, delta, b);
  } else {
    h->d = new Impl<double>();
    rc = h->d->init(b->rows, m, tau, delta, b);
  }
  if (rc != PU_OK) {
    std::string keep = g_last_error;
    delete h->f;
    delete h->d;
    delete h;
    g_last_error = keep;
    return rc;
  }
  *out = h;
  return PU_OK;
}

int pu_set_band_peers(pu_handle* h, const uint64_t* col_blocks, const uint64_t* back_buffers) {
  if ((col_blocks == nullptr) != (back_buffers == nullptr)) return fail(PU_ERR_ARG, "give both tables or neither");
  PU_DISPATCH(h, {
    if (!I.band) return fail(PU_ERR_ARG, "pu_set_band_peers needs a band handle");
    I.pk.peers = reinterpret_cast<const unsigned long long*>(col_blocks);
    const int nq = I.pk.nq;
    I.push = Push{reinterpret_cast<const unsigned long long*>(back_buffers), I.g.n_glob / nq, I.g.n_glob % nq,
                  I.pk.mb, I.col0 / I.pk.mb, FastDiv((unsigned)(I.g.n_glob / nq + 1)),
                  FastDiv((unsigned)(I.g.n_glob / nq))};
  });
  return PU_OK;
}

int pu_ipc_handle(const void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return fail(PU_ERR_ARG, "null argument");
  cudaIpcMemHandle_t hd;
  PU_CUDA(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)));
  std::memcpy(handle, &hd, sizeof(hd));
  return PU_OK;
}

int pu_ipc_open(const void* handle, void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(PU_ERR_ARG, "null argument");
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  PU_CUDA(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  return PU_OK;
}

int pu_ipc_close(void* dev_ptr) {
  PU_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return PU_OK;
}

int pu_dev_alloc(int64_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes < 0) return fail(PU_ERR_ARG, "bad arguments");
  PU_CUDA(cudaMalloc(dev_ptr, (size_t)std::max<int64_t>(bytes, 1)));
  PU_CUDA(cudaMemset(*dev_ptr, 0, (size_t)std::max<int64_t>(bytes, 1)));
  return PU_OK;
}

int pu_dev_free(void* dev_ptr) {
  if (dev_ptr) PU_CUDA(cudaFree(dev_ptr));
  return PU_OK;
}

int pu_set_band_totals(pu_handle* h, double* totals) {
  PU_DISPATCH(h, { I.rs.dist = totals; });
  return PU_OK;
}

int pu_finalize(pu_handle* h, unsigned mask, int mode, int it, void* ctrl, double* res_norms, double* out,
                double rel_tol, int max_iters, void* stream) {
  PU_DISPATCH(h, {
    if (!I.rs.dist) return fail(PU_ERR_ARG, "pu_finalize needs pu_set_band_totals");
    const FinArgs a{reinterpret_cast<PcgCtrl*>(ctrl), res_norms, out, rel_tol, max_iters, it, mode};
    k_finalize<<<1, 32, 0, ST(stream)>>>(I.g, I.rs.dist, mask, a);
    PU_LAUNCH_CHECK();
  });
  return PU_OK;
}

int pu_set_max_iters(pu_handle* h, void* ctrl, int max_iters, void* stream) {
  if (!h) return fail(PU_ERR_ARG, "null handle");
  if (!ctrl || max_iters < 0) return fail(PU_ERR_ARG, "pu_set_max_iters: ctrl required, max_iters >= 0");
  k_set_max_iters<<<1, 32, 0, ST(stream)>>>(reinterpret_cast<PcgCtrl*>(ctrl), max_iters);
  PU_LAUNCH_CHECK();
  return PU_OK;
}

int pu_pcg_begin(pu_handle* h, const void* b, const void* x0, void* x, const void* dv, const void* dh, void* r,
                 void* ctrl, double* res_norms, int max_iters, double rel_tol, const void* gv, const void* gh,
                 const void* cv, const void* ch, const void* wv, const void* wh, double lipschitz, void* cand,
                 void* stream) {
  if (max_iters < 0) return fail(PU_ERR_ARG, "max_iters must be >= 0");
  if (rel_tol < 0) return fail(PU_ERR_ARG, "rel_tol must be >= 0");
  if (cand && !(lipschitz > 0)) return fail(PU_ERR_ARG, "lipschitz constant must be positive");
  if (!b && !(cand && gv && gh)) return fail(PU_ERR_ARG, "b may be NULL only with the candidate step (gv, gh, cand)");
  if ((cv == nullptr) != (ch == nullptr)) return fail(PU_ERR_ARG, "cv and ch must both be given or both NULL");
  PU_DISPATCH(h, {
    const CandArgs<T> ca{CP(gv), CP(gh), CP(cv), CP(ch), CP(wv), CP(wh), (T)(cand ? -1.0 / lipschitz : 0.0),
                         MP(cand)};
    return I.pcg_begin(CP(b), CP(x0), MP(x), CP(dv), CP(dh), MP(r), reinterpret_cast<PcgCtrl*>(ctrl), res_norms,
                       rel_tol, max_iters, cand ? &ca : nullptr, ST(stream));
  });
}

int pu_pcg_residual_rows(pu_handle* h, const void* p, const void* dv, const void* dh, void* x, void* r, void* ctrl,
                         double* res_norms, void* spec_out, int it, int submean, void* stream) {
  PU_DISPATCH(h, {
    return I.pcg_residual_rows(CP(p), CP(dv), CP(dh), MP(x), MP(r), reinterpret_cast<PcgCtrl*>(ctrl), res_norms,
                               MP(spec_out), it, submean, ST(stream));
  });
}

int pu_pcg_update_sum(pu_handle* h, const void* p, const void* dv, const void* dh, void* x, void* r, void* ctrl,
                      int it, void* stream) {
  PU_DISPATCH(h, {
    return I.pcg_update_sum(CP(p), CP(dv), CP(dh), MP(x), MP(r), reinterpret_cast<PcgCtrl*>(ctrl), it, ST(stream));
  });
}

int pu_pcg_columns(pu_handle* h, void* spec, void* ctrl, int it, void* stream) {
  PU_DISPATCH(h, { return I.pcg_columns(MP(spec), reinterpret_cast<PcgCtrl*>(ctrl), it, ST(stream)); });
}

int pu_pcg_rows_inv(pu_handle* h, const void* spec_in, void* pnew, const void* pold, int first, void* ctrl, int it,
                    void* stream) {
  PU_DISPATCH(h, {
    return I.pcg_rows_inv(CP(spec_in), MP(pnew), CP(pold), first, reinterpret_cast<PcgCtrl*>(ctrl), it, ST(stream));
  });
}

int pu_pcg_direction(pu_handle* h, const void* r, const void* pold, void* pnew, const void* dv, const void* dh,
                     void* ctrl, int it, void* stream) {
  PU_DISPATCH(h, {
    return I.pcg_direction(CP(r), CP(pold), MP(pnew), CP(dv), CP(dh), reinterpret_cast<PcgCtrl*>(ctrl), it,
                           ST(stream));
  });
}

}  // extern "C"
