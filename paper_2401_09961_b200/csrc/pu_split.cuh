// Transforms longer than one CTA's shared memory: a 2-CTA cluster per
// packed sequence (sm_100a thread-block clusters + distributed shared memory).
//
// The reference's eigenbasis solve works at any length (preconditioner.py:
// 64-100); here a DCT of length n = 2 LH whose packed complex sequence does
// not fit one CTA (fp64 n = 16384: 256 KiB) is split over the two CTAs of a
// cluster, each holding LH = n/2 complex values in its own shared memory:
//
//   forward (DIF):  CTA q loads v[j] and v[j + LH] (Makhoul order: spatial
//     2j and n-1-2j) and forms y_0 = v[j] + v[j+LH] (q = 0) or
//     y_1 = (v[j] - v[j+LH]) W_n^j (q = 1); its LH-point FFT (the static
//     plan) then yields the bins k = 2k' + q.  Bins k and n - k have the same
//     parity, so the DCT-II post-processing / spectral scaling / DCT-III
//     pre-processing of every pair stays inside one CTA.
//   inverse (DIT):  CTA q holds the pre-twiddled bins of parity q, runs its
//     LH-point FFT (E or O), and after a cluster barrier reads the partner's
//     half through DSMEM: X[t] = E[t] + W_n^t O[t] (q = 0, spatial rows 2t),
//     X[t + LH] = E[t] - W_n^t O[t] (q = 1, spatial rows n-1-2t).
//
// Same arithmetic contract as the one-CTA kernels (pu_pipe.cuh, pu_pcg.cuh):
// DCT-II post / DCT-III pre from pu_fft.cuh, 1/n and the orthonormal scales
// folded into the tables, rho_u by Parseval reduced with the deterministic
// ticket reduction.  Global accesses are direct (no staging): the two CTAs of
// a cluster read interleaved halves of the same rows, so DRAM sees each
// sector once and L2 serves the partner.
#pragma once

#include <cooperative_groups.h>

#include "pu_pipe.cuh"

namespace pu {

namespace cgx = cooperative_groups;

// threads of a split kernel: one static-plan group of LH / EMAX
template <int LH, int EMAX>
__host__ __device__ constexpr int split_threads() { return LH / EMAX; }

// spatial index of Makhoul position p of a length-n sequence (inverse of mperm)
__device__ __forceinline__ int mspatial(int p, int n) { return p < (n + 1) / 2 ? 2 * p : 2 * n - 1 - 2 * p; }

// forward DIF stage from two complex loads; writes y_q into buf (natural order)
template <typename T, int LH, typename Load>
__device__ __forceinline__ void split_dif_load(int q, const FftPlan<T>& pl, cplx<T>* buf, Load load) {
  const int n = 2 * LH;
  for (int j = threadIdx.x; j < LH; j += blockDim.x) {
    const cplx<T> x0 = load(2 * j), x1 = load(n - 1 - 2 * j);
    cplx<T> y;
    if (q == 0) y = cadd<T>(x0, x1);
    else y = cmul<T>(csub<T>(x0, x1), __ldg(pl.tw + j));
    PU_ASSERT(spad(j) < ldseq_for(LH));
    *sm_chk(&buf[spad(j)]) = y;
  }
}

// number of bin pairs (k, n - k) CTA q owns: k = 2e + q <= n/2
template <int LH>
__device__ __forceinline__ int split_pairs(int q) { return q == 0 ? LH / 2 + 1 : LH / 2; }

// inverse DIT combine through DSMEM; store(spatial m, X) for this CTA's outputs
template <typename T, int LH, typename Store>
__device__ __forceinline__ void split_dit_store(int q, const FftPlan<T>& pl, cplx<T>* buf, Store store) {
  cgx::cluster_group cl = cgx::this_cluster();
  cl.sync();  // both halves transformed
  const cplx<T>* other = cl.map_shared_rank(buf, q ^ 1);
  const int n = 2 * LH;
  for (int t = threadIdx.x; t < LH; t += blockDim.x) {
    PU_ASSERT(spad(t) < ldseq_for(LH));
    const cplx<T> mine = *sm_chk(&buf[spad(t)]), theirs = other[spad(t)];
    const cplx<T> e = q == 0 ? mine : theirs;
    const cplx<T> o = cmul<T>(q == 0 ? theirs : mine, __ldg(pl.tw + t));
    const cplx<T> x = q == 0 ? cadd<T>(e, o) : csub<T>(e, o);
    store(q == 0 ? 2 * t : n - 1 - 2 * t, x);
  }
  cl.sync();  // the partner may still be reading this CTA's buffer
}

// Length-n DFT, n = pl.n <= LH (a Bluestein plan: non-smooth n, internal
// length L = 2 LH), split over the cluster the same way: a_p = x_p chirp_p
// is zero past n, so the DIF butterfly is y_0 = a, y_1 = a W_L^j; the filter
// multiplies bins of this CTA's parity; the second FFT's DIT combine is only
// needed for t < n, all in CTA 0.  On return CTA 0 holds Z_k, k < n, at
// spad(k) (CTA 1's buffer is scratch).  REMOTE: val reads CTA 0's buffer, so
// every value is gathered into registers before any CTA writes its buffer.
template <typename T, int EMAX, int LH, typename Val>
__device__ __forceinline__ void split_bluestein(int q, const FftPlan<T>& pl, const FftPlan<T>& ph, cplx<T>* buf,
                                                Val val, bool remote) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int n = pl.n;
  constexpr int PER = EMAX;  // LH / (LH / EMAX threads)
  cplx<T> a[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = threadIdx.x + i * blockDim.x;
    a[i] = j < n ? cmul<T>(val(j), __ldg(pl.chirp + j)) : mk<T>((T)0, (T)0);
  }
  if (remote) cl.sync();  // CTA 0's buffer has been read by both CTAs
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = threadIdx.x + i * blockDim.x;
    if (j < LH) *sm_chk(&buf[spad(j)]) = q == 0 ? a[i] : cmul<T>(a[i], __ldg(pl.tw + j));
  }
  __syncthreads();
  fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
  for (int kk = threadIdx.x; kk < LH; kk += blockDim.x)  // bin k = 2 kk + q
    buf[spad(kk)] = cconj<T>(cmul<T>(buf[spad(kk)], __ldg(pl.filt + 2 * kk + q)));
  __syncthreads();
  fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
  cl.sync();  // E (CTA 0) and O (CTA 1) complete
  if (q == 0) {
    const cplx<T>* other = cl.map_shared_rank(buf, 1);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const cplx<T> x = cadd<T>(buf[spad(t)], cmul<T>(other[spad(t)], __ldg(pl.tw + t)));
      buf[spad(t)] = cmul<T>(cconj<T>(x), __ldg(pl.chirp + t));
    }
  }
  cl.sync();  // CTA 1's buffer is no longer read; CTA 0's results are visible to its threads
}

// ---------------------------------------------------------------------------
// Row transforms (K2b forward, K4 inverse) of one row pair per cluster.
// pl: full-length tables (tw = W_n^k, dct2w, dct3w); ph: the LH static plan.
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LH, bool INV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(split_threads<LH, EMAX>(), 1)
    k_rows_split(Grid g, FftPlan<T> pl, FftPlan<T> ph, const T* __restrict__ in, T* __restrict__ out,
                 const PcgCtrl* ctrl, const T* __restrict__ pold, int first, Pack pk) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  if (ctrl && ctrl->done) return;  // uniform over the cluster
  constexpr int n = 2 * LH;
  const int q = (int)(blockIdx.x & 1);
  const int ia = 2 * (int)(blockIdx.x >> 1);
  const bool hasb = ia + 1 < g.n;
  const long long oa = (long long)ia * g.ld, ob = oa + g.ld;
  const bool pout = !INV && pk.nq > 0, pin = INV && pk.nq > 0;
  auto at = [&](int row, int k) -> T* {  // spectrum element (row ia + row, column k)
    if (!pout) return out + oa + (long long)row * g.ld + k;
    const int c = (int)pk.mbd.div((unsigned)k);
    T* base = pk.peers ? reinterpret_cast<T*>(__ldg(pk.peers + c)) + (pk.row0 + ia + row) * pk.mb
                       : out + c * pk.chunk + (long long)(ia + row) * pk.mb;
    return base + (k - c * pk.mb);
  };
  auto src = [&](int row, int k) -> T {
    if (row == 1 && !hasb) return (T)0;
    if (!pin) return in[oa + (long long)row * g.ld + k];
    const int c = (int)pk.mbd.div((unsigned)k);
    if (pk.peers && c == pk.own_q)  // this rank's own rows: in place in its column block
      return reinterpret_cast<const T*>(__ldg(pk.peers + c))[(pk.row0 + ia + row) * pk.mb + (k - c * pk.mb)];
    return in[c * pk.chunk + (long long)(ia + row) * pk.mb + (k - c * pk.mb)];
  };
  if (pl.bluestein) {  // non-smooth n <= LH: Bluestein over the cluster, CTA 0 finishes
    const int nn = pl.n;
    if constexpr (!INV) {
      split_bluestein<T, EMAX, LH>(q, pl, ph, buf, [&](int p) {
        const int m = mspatial(p, nn);
        return mk<T>(in[oa + m], hasb ? in[ob + m] : (T)0);
      }, false);
      if (q == 0) {
        for (int k = threadIdx.x; k < nn / 2 + 1; k += blockDim.x) {
          const int nk = k == 0 ? 0 : nn - k;
          const PairOut<T> r = dct2_post<T>(buf[spad(k)], buf[spad(nk)], k, nk, pl);
          *at(0, k) = r.a_k;
          if (hasb) *at(1, k) = r.b_k;
          if (nk != k) {
            *at(0, nk) = r.a_nk;
            if (hasb) *at(1, nk) = r.b_nk;
          }
        }
      }
    } else {
      split_bluestein<T, EMAX, LH>(q, pl, ph, buf, [&](int k) {
        const int nk = k == 0 ? 0 : nn - k;
        return dct3_pre_k<T>(src(0, k), src(0, nk), src(1, k), src(1, nk), k, pl);
      }, false);
      if (q == 0) {
        const bool axpy = pold != nullptr && !first;
        const T beta = axpy ? (T)ctrl->beta : (T)0;
        for (int m = threadIdx.x; m < nn; m += blockDim.x) {
          const cplx<T> x = buf[spad(mperm(m, nn))];
          T va = x.x, vb = -x.y;  // 1/n folded into dct3w
          if (axpy) {
            va = add_rn(mul_rn(beta, pold[oa + m]), va);
            if (hasb) vb = add_rn(mul_rn(beta, pold[ob + m]), vb);
          }
          out[oa + m] = va;
          if (hasb) out[ob + m] = vb;
        }
      }
    }
    return;
  }
  if constexpr (!INV) {
    split_dif_load<T, LH>(q, pl, buf, [&](int m) {
      return mk<T>(in[oa + m], hasb ? in[ob + m] : (T)0);
    });
    __syncthreads();
    fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
    for (int e = threadIdx.x; e < split_pairs<LH>(q); e += blockDim.x) {
      const int k = 2 * e + q, nk = k == 0 ? 0 : n - k;
      const int lk = e, lnk = (nk - q) >> 1;
      const PairOut<T> r = dct2_post<T>(buf[spad(lk)], buf[spad(lnk)], k, nk, pl);
      *at(0, k) = r.a_k;
      if (hasb) *at(1, k) = r.b_k;
      if (nk != k) {
        *at(0, nk) = r.a_nk;
        if (hasb) *at(1, nk) = r.b_nk;
      }
    }
  } else {
    for (int e = threadIdx.x; e < split_pairs<LH>(q); e += blockDim.x) {
      const int k = 2 * e + q, nk = k == 0 ? 0 : n - k;
      const int lk = e, lnk = (nk - q) >> 1;
      cplx<T> ck, cnk;
      dct3_pre<T>(src(0, k), src(0, nk), src(1, k), src(1, nk), k, nk, pl, ck, cnk);
      buf[spad(lk)] = ck;
      if (nk != k) buf[spad(lnk)] = cnk;
    }
    __syncthreads();
    fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
    const bool axpy = pold != nullptr && !first;
    const T beta = axpy ? (T)ctrl->beta : (T)0;
    split_dit_store<T, LH>(q, pl, buf, [&](int m, cplx<T> x) {
      T va = x.x, vb = -x.y;  // 1/n folded into dct3w
      if (axpy) {
        va = add_rn(mul_rn(beta, pold[oa + m]), va);
        if (hasb) vb = add_rn(mul_rn(beta, pold[ob + m]), vb);
      }
      out[oa + m] = va;
      if (hasb) out[ob + m] = vb;
    });
  }
}

// ---------------------------------------------------------------------------
// K3 / API on one column pair per cluster: column DCT-II, x tau/(lam_i +
// lam_j) with (0,0) -> 0, rho_u (Parseval), column DCT-III, in place (or
// pushed to the owners' buffers in the peer-transpose band mode).
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LH, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(split_threads<LH, EMAX>(), 1)
    k_cols_split(Grid g, FftPlan<T> pl, FftPlan<T> ph, const T* __restrict__ lam_cols, T* data, PcgCtrl* ctrl,
                 RedScratch rs, int site, int it, Push ps) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  if (MODE != MODE_API && ctrl->done) return;  // uniform over the cluster
  constexpr int n = 2 * LH;
  const int q = (int)(blockIdx.x & 1);
  const int ja = 2 * (int)(blockIdx.x >> 1), jb = ja + 1;
  const bool hasb = jb < g.m;
  if (pl.bluestein) {  // non-smooth n <= LH: Bluestein over the cluster, CTA 0 finishes
    const int nn = pl.n;
    split_bluestein<T, EMAX, LH>(q, pl, ph, buf, [&](int p) {
      const T* row = data + (long long)mspatial(p, nn) * g.ld + ja;
      return hasb ? *reinterpret_cast<const cplx<T>*>(row) : mk<T>(row[0], (T)0);
    }, false);
    T accB = (T)0;
    const T ttau = (T)g.tau;
    const T la = __ldg(lam_cols + ja), lb = hasb ? __ldg(lam_cols + jb) : (T)0;
    auto sdiv = [&](T v, T den) -> T { return den == (T)0 ? (T)0 : fast_div(ttau * v, den); };
    if (q == 0) {
      for (int k = threadIdx.x; k < nn / 2 + 1; k += blockDim.x) {
        const int nk = k == 0 ? 0 : nn - k;
        const PairOut<T> r = dct2_post<T>(buf[spad(k)], buf[spad(nk)], k, nk, pl);
        const T lk_ = __ldg(pl.lam + k), lnk_ = __ldg(pl.lam + nk);
        const T zak = sdiv(r.a_k, lk_ + la), zbk = hasb ? sdiv(r.b_k, lk_ + lb) : (T)0;
        T zank, zbnk;
        accB += r.a_k * zak + r.b_k * zbk;
        if (nk != k) {
          zank = sdiv(r.a_nk, lnk_ + la);
          zbnk = hasb ? sdiv(r.b_nk, lnk_ + lb) : (T)0;
          accB += r.a_nk * zank + r.b_nk * zbnk;
        } else {
          zank = zak; zbnk = zbk;
        }
        cplx<T> ck, cnk;
        dct3_pre<T>(zak, zank, zbk, zbnk, k, nk, pl, ck, cnk);
        buf[spad(k)] = ck;
        if (nk != k) buf[spad(nk)] = cnk;
      }
    }
    cgx::this_cluster().sync();  // the pre-processed spectrum of CTA 0 is visible to CTA 1
    const cplx<T>* src0 = cgx::this_cluster().map_shared_rank(buf, 0);
    split_bluestein<T, EMAX, LH>(q, pl, ph, buf, [&](int j) { return src0[spad(j)]; }, true);
    if (q == 0) {
      for (int m = threadIdx.x; m < nn; m += blockDim.x) {
        const cplx<T> x = buf[spad(mperm(m, nn))];
        T* row = ps.backs ? push_row<T>(ps, m, data, g.ld) : data + (long long)m * g.ld;
        if (hasb) *reinterpret_cast<cplx<T>*>(row + ja) = mk<T>(x.x, -x.y);
        else row[ja] = x.x;
      }
    }
    if (MODE != MODE_API) {
      double acc[1] = {(double)accB};
      double tot[1];
      if (red_final<1>(acc, rs, site, tot) && threadIdx.x == 0) fin_k3(ctrl, tot, it, MODE);
    }
    return;
  }
  split_dif_load<T, LH>(q, pl, buf, [&](int m) {
    const T* row = data + (long long)m * g.ld + ja;
    return hasb ? *reinterpret_cast<const cplx<T>*>(row) : mk<T>(row[0], (T)0);
  });
  __syncthreads();
  fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
  T accT = (T)0;
  const T ttau = (T)g.tau;
  const T la = __ldg(lam_cols + ja), lb = hasb ? __ldg(lam_cols + jb) : (T)0;
  auto sdiv = [&](T v, T den) -> T { return den == (T)0 ? (T)0 : fast_div(ttau * v, den); };
  for (int e = threadIdx.x; e < split_pairs<LH>(q); e += blockDim.x) {
    const int k = 2 * e + q, nk = k == 0 ? 0 : n - k;
    const int lk = e, lnk = (nk - q) >> 1;
    const PairOut<T> r = dct2_post<T>(buf[spad(lk)], buf[spad(lnk)], k, nk, pl);
    const T lk_ = __ldg(pl.lam + k), lnk_ = __ldg(pl.lam + nk);
    const T zak = sdiv(r.a_k, lk_ + la), zbk = hasb ? sdiv(r.b_k, lk_ + lb) : (T)0;
    T zank, zbnk;
    accT += r.a_k * zak + r.b_k * zbk;
    if (nk != k) {
      zank = sdiv(r.a_nk, lnk_ + la);
      zbnk = hasb ? sdiv(r.b_nk, lnk_ + lb) : (T)0;
      accT += r.a_nk * zank + r.b_nk * zbnk;
    } else {
      zank = zak; zbnk = zbk;
    }
    cplx<T> ck, cnk;
    dct3_pre<T>(zak, zank, zbk, zbnk, k, nk, pl, ck, cnk);
    buf[spad(lk)] = ck;
    if (nk != k) buf[spad(lnk)] = cnk;
  }
  __syncthreads();
  fft_stages_s<T, EMAX, LH, 1, 0>(buf, 0, 1, ph.stw);
  split_dit_store<T, LH>(q, pl, buf, [&](int m, cplx<T> x) {
    T* row = ps.backs ? push_row<T>(ps, m, data, g.ld) : data + (long long)m * g.ld;
    if (hasb) *reinterpret_cast<cplx<T>*>(row + ja) = mk<T>(x.x, -x.y);
    else row[ja] = x.x;
  });
  if (MODE != MODE_API) {
    double acc[1] = {(double)accT};
    double tot[1];
    if (red_final<1>(acc, rs, site, tot) && threadIdx.x == 0) fin_k3(ctrl, tot, it, MODE);
  }
}

// Host launch wrappers (instantiated in pu_split_inst.cu for the two
// supported half lengths: double 8192 -> n = 16384, float 16384 -> n = 32768).
template <typename T, int LH>
struct SplitLaunch {
  static constexpr int EM = emax_of<T>();
  static constexpr int threads() { return split_threads<LH, EM>(); }
  static size_t smem() { return (size_t)ldseq_for(LH) * sizeof(cplx<T>); }
  static cudaError_t set_attrs();
  static cudaError_t rows(bool inv, int pairs, cudaStream_t st, const Grid& g, const FftPlan<T>& pl,
                          const FftPlan<T>& ph, const T* in, T* out, const PcgCtrl* ctrl, const T* pold, int first,
                          Pack pk);
  static cudaError_t cols(int mode, int colpairs, cudaStream_t st, const Grid& g, const FftPlan<T>& pl,
                          const FftPlan<T>& ph, const T* lam_cols, T* data, PcgCtrl* ctrl, RedScratch rs, int site,
                          int it, Push ps);
};

#ifdef PU_SPLIT_DEFINE
template <typename T, int LH>
cudaError_t SplitLaunch<T, LH>::set_attrs() {
  cudaError_t e;
  const int s = (int)smem();
#define PU_SATTR(K) \
  if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, s)) != cudaSuccess) return e;
  PU_SATTR((k_rows_split<T, EM, LH, false>));
  PU_SATTR((k_rows_split<T, EM, LH, true>));
  PU_SATTR((k_cols_split<T, EM, LH, MODE_API>));
  PU_SATTR((k_cols_split<T, EM, LH, MODE_INIT>));
  PU_SATTR((k_cols_split<T, EM, LH, MODE_ITER>));
#undef PU_SATTR
  return cudaSuccess;
}

template <typename T, int LH>
cudaError_t SplitLaunch<T, LH>::rows(bool inv, int pairs, cudaStream_t st, const Grid& g, const FftPlan<T>& pl,
                                     const FftPlan<T>& ph, const T* in, T* out, const PcgCtrl* ctrl, const T* pold,
                                     int first, Pack pk) {
  if (inv)
    k_rows_split<T, EM, LH, true><<<2 * pairs, threads(), smem(), st>>>(g, pl, ph, in, out, ctrl, pold, first, pk);
  else
    k_rows_split<T, EM, LH, false><<<2 * pairs, threads(), smem(), st>>>(g, pl, ph, in, out, ctrl, nullptr, 0, pk);
  return cudaGetLastError();
}

template <typename T, int LH>
cudaError_t SplitLaunch<T, LH>::cols(int mode, int colpairs, cudaStream_t st, const Grid& g, const FftPlan<T>& pl,
                                     const FftPlan<T>& ph, const T* lam_cols, T* data, PcgCtrl* ctrl, RedScratch rs,
                                     int site, int it, Push ps) {
  const int grid = 2 * colpairs;
  if (mode == MODE_API)
    k_cols_split<T, EM, LH, MODE_API><<<grid, threads(), smem(), st>>>(g, pl, ph, lam_cols, data, ctrl, rs, site, it, ps);
  else if (mode == MODE_INIT)
    k_cols_split<T, EM, LH, MODE_INIT><<<grid, threads(), smem(), st>>>(g, pl, ph, lam_cols, data, ctrl, rs, site, it, ps);
  else
    k_cols_split<T, EM, LH, MODE_ITER><<<grid, threads(), smem(), st>>>(g, pl, ph, lam_cols, data, ctrl, rs, site, it, ps);
  return cudaGetLastError();
}
#endif  // PU_SPLIT_DEFINE

extern template struct SplitLaunch<double, 8192>;
extern template struct SplitLaunch<float, 16384>;

}  // namespace pu
