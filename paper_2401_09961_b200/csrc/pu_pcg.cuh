// DCT preconditioner passes and the fused PCG iteration (sm_100a).
//
// One PCG iteration of pcg.py:81-108 is five kernels:
//   K1 k_pcg_p_v   slack p_s <- beta p_s + z_s (z at it = 0; p_u came from K4);
//                  p'Ap as a quadratic form; last block: alpha = rho / p'Ap,
//                  curvature exits (pcg.py:82-89)
//   K2a k_pcg_r_v  x += alpha p; r -= alpha A p (A p recomputed from p);
//                  ||r||^2; slack preconditioner z_s = r_s / (d + 1/tau); rho_s;
//                  last block: ||r|| exits            (pu_vec.cuh)
//   K2b k_rows_pipe<false> row DCT-II of r_u -> spectral plane T (pu_pipe.cuh)
//   K3 k_cols_spec column DCT-II, x tau/(lam_i + lam_j) with (0,0) -> 0,
//                  rho_u = <r_hat, z_hat> (Parseval), column DCT-III;
//                  last block: beta = (rho_s + rho_u) / rho
//   K4 k_rows_pipe<true>  row DCT-III of T -> z_u, p_u = beta p_u + z_u (pu_pipe.cuh)
// The standalone preconditioner (preconditioner.py:86-115) is K2..K4 with the
// plain policies.  Every PCG kernel returns immediately once ctrl->done is set.
#pragma once

#include "pu_kernels.cuh"
#include "pu_q4.cuh"

namespace pu {


// ---------------------------------------------------------------------------
// Column-panel staging for K3.  A panel is W = 2 * nseq columns x n rows;
// column pair (2s, 2s+1) is packed as (re, im) of complex sequence s at the
// Makhoul-permuted position.  Full panels move as 16-byte vectors, UNR per
// thread in flight before any shared-memory store (the kernel was latency
// bound on one scalar load per thread otherwise).
// ---------------------------------------------------------------------------
template <typename T> struct V16;
template <> struct V16<float> { using type = float4; static constexpr int N = 4; };
template <> struct V16<double> { using type = double2; static constexpr int N = 2; };

template <typename T>
__device__ __forceinline__ void panel_load(const Grid& g, const FftPlan<T>& pl, const T* __restrict__ data, int j0,
                                           const int W, int ncols, int nseq, cplx<T>* buf, const int n) {
  using V = typename V16<T>::type;
  constexpr int VN = V16<T>::N;
  constexpr int UNR = 4;
  if (ncols == W && W % VN == 0) {
    const int vpr = W / VN;
    const int items = n * vpr;
    for (int base = 0; base < items; base += UNR * blockDim.x) {
      V r[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int e = base + u * blockDim.x + threadIdx.x;
        if (e < items) {
          const int i = e / vpr, v = e - i * vpr;
          PU_ASSERT(i < g.n && j0 + (v + 1) * VN <= g.ld);
          r[u] = __ldg(reinterpret_cast<const V*>(data + (long long)i * g.ld + j0 + v * VN));
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int e = base + u * blockDim.x + threadIdx.x;
        if (e < items) {
          const int i = e / vpr, v = e - i * vpr;
          const int p = spad(mperm(i, n));
          PU_ASSERT(p < pl.ldseq);
          if constexpr (VN == 4) {
            *sm_chk(&buf[(2 * v) * pl.ldseq + p]) = mk<T>(r[u].x, r[u].y);
            *sm_chk(&buf[(2 * v + 1) * pl.ldseq + p]) = mk<T>(r[u].z, r[u].w);
          } else {
            *sm_chk(&buf[v * pl.ldseq + p]) = mk<T>(r[u].x, r[u].y);
          }
        }
      }
    }
  } else {
    for (int e = threadIdx.x; e < n * 2 * nseq; e += blockDim.x) {
      const int i = e / (2 * nseq), c = e - i * (2 * nseq);
      PU_ASSERT(i < g.n && (c >= ncols || j0 + c < g.ld));
      const T val = (c < ncols) ? data[(long long)i * g.ld + j0 + c] : (T)0;
      T* slot = reinterpret_cast<T*>(sm_chk(buf + (c >> 1) * pl.ldseq + spad(mperm(i, n))));
      slot[c & 1] = val;
    }
  }
}

// Row-sharded push mode (band.py, peer transpose): the column transform sends
// each output row straight to the packed input buffer of the rank that owns
// the row (element (local row i_r, column q mb + j) of rank r's band at
// q rows_r mb + i_r mb + j), so every cross-GPU access of the fused
// transpose is a store.  backs == null: write the column block in place.
struct Push {
  const unsigned long long* backs;  // device: every rank's back-buffer address
  int base, extra;                  // row bands: rows_r = base + (r < extra)
  int mb, q;                        // chunk width; this rank's chunk index
  FastDiv bigd, based;              // i / (base + 1), i / base
};

// destination row pointer of global row i: the owner's back buffer, or in
// place (`data`, pitch ld) for this rank's own rows, which K4 reads from its
// column block (Pack::own_q)
template <typename T>
__device__ __forceinline__ T* push_row(const Push& ps, int i, T* data, long long ld) {
  const int big = ps.base + 1, cut = ps.extra * big;
  int r, ir, rows;
  if (i < cut) {
    r = (int)ps.bigd.div((unsigned)i); ir = i - r * big; rows = big;
  } else {
    r = ps.extra + (int)ps.based.div((unsigned)(i - cut)); ir = i - cut - (r - ps.extra) * ps.base; rows = ps.base;
  }
  if (r == ps.q) return data + (long long)i * ld;
  return reinterpret_cast<T*>(__ldg(ps.backs + r)) + (long long)ps.q * rows * ps.mb + (long long)ir * ps.mb;
}

// inverse of panel_load after the DCT-III FFT: column 2s = Re/n, 2s+1 = -Im/n
template <typename T>
__device__ __forceinline__ void panel_store(const Grid& g, const FftPlan<T>& pl, T* data, int j0, int W, int ncols,
                                            int nseq, const cplx<T>* buf, const int n, const Push& ps) {
  using V = typename V16<T>::type;
  constexpr int VN = V16<T>::N;
  if (ncols == W && W % VN == 0) {
    const int vpr = W / VN;
    const int items = n * vpr;
    for (int e = threadIdx.x; e < items; e += blockDim.x) {
      const int i = e / vpr, v = e - i * vpr;
      const int p = spad(mperm(i, n));
      V o;
      if constexpr (VN == 4) {
        const cplx<T> a = buf[(2 * v) * pl.ldseq + p], b = buf[(2 * v + 1) * pl.ldseq + p];
        o.x = a.x; o.y = -a.y; o.z = b.x; o.w = -b.y;  // 1/n folded into dct3w
      } else {
        const cplx<T> a = buf[v * pl.ldseq + p];
        o.x = a.x; o.y = -a.y;
      }
      PU_ASSERT(i < g.n && j0 + (v + 1) * VN <= g.ld && p < pl.ldseq);
      T* row = ps.backs ? push_row<T>(ps, i, data, g.ld) : data + (long long)i * g.ld;
      *reinterpret_cast<V*>(row + j0 + v * VN) = o;
    }
  } else {
    for (int e = threadIdx.x; e < n * 2 * nseq; e += blockDim.x) {
      const int i = e / (2 * nseq), c = e - i * (2 * nseq);
      if (c < ncols) {
        const cplx<T> v = buf[(c >> 1) * pl.ldseq + spad(mperm(i, n))];
        T* row = ps.backs ? push_row<T>(ps, i, data, g.ld) : data + (long long)i * g.ld;
        row[j0 + c] = (c & 1) ? -v.y : v.x;
      }
    }
  }
  (void)nseq;
}

// ---------------------------------------------------------------------------
// Static (power-of-two) column plans: the first forward
// stage reads its butterfly straight from global memory and the last inverse
// stage stores straight to global memory, so the panel never makes the extra
// shared-memory round trip of panel_load / panel_store.  Thread t works on
// sequence t % NSEQ, butterfly t / NSEQ: the NSEQ threads of one butterfly
// index cover one full 2 NSEQ-column row segment (up to 32 bytes).
// Makhoul order: FFT index idx holds row 2 idx (idx < L/2) or
// 2L - 1 - 2 idx (idx >= L/2); butterfly j's inputs / last-stage outputs sit
// at idx = j + r L/R, so rows are 2 j + 2 r L/R (r < R/2) and
// 2L - 1 - 2 j - 2 r L/R.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr bool col_fused_rt(int L, int emax) {
  const int big = emax >= 16 ? 16 : 8, r0 = first_radix_rt(L, emax);
  return (r0 == 2 || r0 == 4 || r0 == 8 || r0 == 16) && emax % r0 == 0 && L >= r0 * big && (L / big) % 16 == 0;
}
template <int L, int EMAX>
__host__ __device__ constexpr bool col_fused_ok() { return col_fused_rt(L, EMAX); }

// first forward stage, Q = EMAX / R butterflies per thread (all loads in flight first)
template <typename T, int EMAX, int L, int NSEQ>
__device__ __forceinline__ void col_first_stage(const Grid& g, const T* __restrict__ data, int j0, cplx<T>* buf) {
  constexpr int R = first_radix<L, EMAX>(), Q = EMAX / R, NB = L / R, LD = ldseq_for(L);
  const long long ld = g.ld, step = 2LL * NB * ld;
  cplx<T> v[Q][R];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = threadIdx.x + q * blockDim.x, s = b % NSEQ, j = b / NSEQ;
    if (b >= NSEQ * NB) break;  // CTAs may be rounded up
    const T* pa = data + (long long)(2 * j) * ld + j0 + 2 * s;
    const T* pb = data + (long long)(2 * L - 1 - 2 * j) * ld + j0 + 2 * s;
    // rows touched: 2 j + 2 r NB (r < R/2) and 2L - 1 - 2 j - 2 r NB (R/2 <= r < R)
    PU_ASSERT(2 * j + 2 * (R / 2 - 1) * NB < g.n && 2 * L - 1 - 2 * j - 2 * (R - 1) * NB >= 0 &&
              2 * L - 1 - 2 * j - R * NB < g.n && j0 + 2 * s + 2 <= ld);
#pragma unroll
    for (int r = 0; r < R / 2; ++r) v[q][r] = __ldg(reinterpret_cast<const cplx<T>*>(pa + r * step));
#pragma unroll
    for (int r = R / 2; r < R; ++r) v[q][r] = __ldg(reinterpret_cast<const cplx<T>*>(pb - r * step));
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = threadIdx.x + q * blockDim.x, s = b % NSEQ, j = b / NSEQ;
    if (b >= NSEQ * NB) break;
    Dft<T, R>::run(v[q]);
    cplx<T>* dst = buf + s * LD + spad(j * R);  // spad(j R + r) = spad(j R) + r for R | 16
#pragma unroll
    for (int r = 0; r < R; ++r) {
      PU_ASSERT(spad(j * R) + r < LD);
      *sm_chk(&dst[r]) = v[q][r];
    }
  }
  __syncthreads();
}

// last inverse stage (NS = L / R, one butterfly per thread): twiddle, DFT,
// store column 2s = Re, 2s + 1 = -Im (as panel_store) of each output row
template <typename T, int EMAX, int L, int NSEQ>
__device__ __forceinline__ void col_last_stage(const Grid& g, T* data, int j0, const cplx<T>* buf,
                                               const cplx<T>* __restrict__ stw, const Push& ps) {
  constexpr int R = EMAX >= 16 ? 16 : 8, NS = L / R, LD = ldseq_for(L);
  constexpr int OFF = stage_off<L, EMAX>(NS);
  const int s = threadIdx.x % NSEQ, j = threadIdx.x / NSEQ;
  if (j < NS) {  // CTAs may be rounded up (no early return: a grid reduction follows)
    const cplx<T>* src = buf + s * LD + spad(j);
    cplx<T> v[R], w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      PU_ASSERT(spad(j) + r * (NS + NS / 16) < LD);
      v[r] = *sm_chk(&src[r * (NS + NS / 16)]);
    }
    w[1] = __ldg(stw + OFF + j);
#pragma unroll
    for (int r = 2; r < R; ++r) w[r] = cmul<T>(w[r / 2], w[r - r / 2]);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul<T>(v[r], w[r]);
    Dft<T, R>::run(v);
    if (ps.backs) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = r < R / 2 ? 2 * j + 2 * r * NS : 2 * L - 1 - 2 * j - 2 * r * NS;
        *reinterpret_cast<cplx<T>*>(push_row<T>(ps, i, data, g.ld) + j0 + 2 * s) = mk<T>(v[r].x, -v[r].y);
      }
    } else {
      const long long ld = g.ld, step = 2LL * NS * ld;
      PU_ASSERT(2 * j + 2 * (R / 2 - 1) * NS < g.n && 2 * L - 1 - 2 * j - R * NS < g.n &&
                2 * L - 1 - 2 * j - 2 * (R - 1) * NS >= 0 && j0 + 2 * s + 2 <= ld);
      T* pa = data + (long long)(2 * j) * ld + j0 + 2 * s;
      T* pb = data + (long long)(2 * L - 1 - 2 * j) * ld + j0 + 2 * s;
#pragma unroll
      for (int r = 0; r < R / 2; ++r) *reinterpret_cast<cplx<T>*>(pa + r * step) = mk<T>(v[r].x, -v[r].y);
#pragma unroll
      for (int r = R / 2; r < R; ++r) *reinterpret_cast<cplx<T>*>(pb - r * step) = mk<T>(v[r].x, -v[r].y);
    }
  }
}

// ---------------------------------------------------------------------------
// K3 / API: column DCT-II, spectral division, column DCT-III, in place on a
// panel of `cols_per_cta` columns; reduces rho_u = <r_hat, z_hat>.
// cols_panel is one panel (index pidx) and returns this thread's share of
// rho_u; k_cols_spec runs one panel per CTA, the persistent small-grid PCG
// kernel (pu_persist.cuh) loops over panels.
// ---------------------------------------------------------------------------
template <typename T, int EMAX, int LS>
__device__ __forceinline__ T cols_panel(const Grid& g, const FftPlan<T>& pl, const T* __restrict__ lam_cols,
                                        int cols_per_cta, T* data, const Push& ps, int nfull, int pidx,
                                        cplx<T>* buf) {
  const int n = LS > 0 ? LS : g.n;  // static plans are only used when n == L
  // static plans: compile-time panel width; runtime plans: 4 or 2 (smem)
  const int W0 = LS > 0 ? static_panel_cols(LS, EMAX, sizeof(T)) : cols_per_cta;
  // balanced grid (static plans): CTAs past `nfull` take half panels, so the
  // last wave is spread over every SM instead of a few full panels
  constexpr bool HALF_OK = LS > 0 && static_panel_cols(LS > 0 ? LS : 4096, EMAX, sizeof(T)) >= 8;  // host: cols_per_cta >= 8
  const bool halfp = HALF_OK && pidx >= nfull;
  const int W = halfp ? W0 / 2 : W0;
  const int j0 = halfp ? nfull * W0 + (pidx - nfull) * W : pidx * W0;
  const int ncols = min(W, g.m - j0);
  const int nseq = (ncols + 1) >> 1;
  constexpr bool FUSE = LS > 0 && col_fused_ok<(LS > 0 ? LS : 4096), EMAX>();
  constexpr int LF = LS > 0 ? LS : 4096;  // (LS == 0: FUSE is false, LF unused)
  const bool fuse = FUSE && ncols == W;
  // K3 group mode (PU_K3_GROUPS): after the CTA-wide first stage, every
  // sequence's stages, post-processing and inverse stages synchronise only
  // its own NB threads (named barriers), the last stage is CTA-wide again
#ifdef PU_K3_GROUPS
  constexpr bool GRP = FUSE && grp_ok<LF, EMAX>();
#else
  constexpr bool GRP = false;
#endif
  constexpr int NBG = LF / EMAX;  // threads per sequence in group mode
  if (fuse) {
    if constexpr (FUSE) {
      constexpr int NSF = static_panel_cols(LF, EMAX, sizeof(T)) / 2;
      if (halfp) {
        if constexpr (NSF >= 4) col_first_stage<T, EMAX, LF, NSF / 2>(g, data, j0, buf);
      } else {
        col_first_stage<T, EMAX, LF, NSF>(g, data, j0, buf);
      }
      fft_stages_range<T, EMAX, LF, first_radix<LF, EMAX>(), 0, LF, GRP>(buf, 0, nseq, pl.stw);
    }
  } else {
    panel_load<T>(g, pl, data, j0, W, ncols, nseq, buf, n);
    __syncthreads();
    fft_n<T, EMAX, LS>(buf, nseq, pl);
  }
  T accT = (T)0;  // per-thread partial of rho_u in T (a few dozen terms), fp64 across threads
  const int half = n / 2 + 1;
  const double tau = g.tau;
  const bool grp = GRP && fuse;
  // group mode: sequence s = threadIdx.x / NBG, its NBG threads stride over k
  const int e0 = grp ? (int)threadIdx.x % NBG + ((int)threadIdx.x / NBG) * half : (int)threadIdx.x;
  const int e1 = grp ? ((int)threadIdx.x / NBG < nseq ? ((int)threadIdx.x / NBG + 1) * half : 0) : nseq * half;
  const int es = grp ? NBG : (int)blockDim.x;
  for (int e = e0; e < e1; e += es) {
    const int s = e / half, k = e - s * half;
    const int nk = k == 0 ? 0 : n - k;
    cplx<T>* sb = buf + s * pl.ldseq;
    PU_ASSERT(spad(k) < pl.ldseq && spad(nk) < pl.ldseq);
    const PairOut<T> q = dct2_post<T>(*sm_chk(&sb[spad(k)]), *sm_chk(&sb[spad(nk)]), k, nk, pl);
    const int ja = j0 + 2 * s, jb = ja + 1;
    const bool hasb = jb < g.m;
    const T lk = __ldg(pl.lam + k), lnk = __ldg(pl.lam + nk);
    const T la = __ldg(lam_cols + ja), lb = hasb ? __ldg(lam_cols + jb) : (T)0;
    // preconditioner.py:96-99: z = tau * r / (lam_s + lam_t), (0,0) -> 0
    const T ttau = (T)tau;
    auto sdiv = [&](T v, T den) -> T { return den == (T)0 ? (T)0 : fast_div(ttau * v, den); };
    const T zak = sdiv(q.a_k, lk + la), zbk = hasb ? sdiv(q.b_k, lk + lb) : (T)0;
    T zank = 0, zbnk = 0;
    accT += q.a_k * zak + q.b_k * zbk;
    if (nk != k) {
      zank = sdiv(q.a_nk, lnk + la);
      zbnk = hasb ? sdiv(q.b_nk, lnk + lb) : (T)0;
      accT += q.a_nk * zank + q.b_nk * zbnk;
    } else {
      zank = zak; zbnk = zbk;
    }
    cplx<T> ck, cnk;
    dct3_pre<T>(zak, zank, zbk, zbnk, k, nk, pl, ck, cnk);
    sb[spad(k)] = ck;
    if (nk != k) sb[spad(nk)] = cnk;
  }
  if (grp) stage_sync<GRP>(NBG, nseq);
  else __syncthreads();
  if (fuse) {
    if constexpr (FUSE) {
      fft_stages_range<T, EMAX, LF, 1, 0, LF / (EMAX >= 16 ? 16 : 8), GRP>(buf, 0, nseq, pl.stw);
      if constexpr (GRP) __syncthreads();  // the last stage reads across sequences
      constexpr int NSF = static_panel_cols(LF, EMAX, sizeof(T)) / 2;
      if (halfp) {
        if constexpr (NSF >= 4) col_last_stage<T, EMAX, LF, NSF / 2>(g, data, j0, buf, pl.stw, ps);
      } else {
        col_last_stage<T, EMAX, LF, NSF>(g, data, j0, buf, pl.stw, ps);
      }
    }
  } else {
    fft_n<T, EMAX, LS>(buf, nseq, pl);
    panel_store<T>(g, pl, data, j0, W, ncols, nseq, buf, n, ps);
  }
  return accT;
}

template <typename T, int EMAX, int LS, int MODE>
__global__ void __launch_bounds__(fft_max_threads(LS, EMAX, sizeof(T)), fft_min_blocks(LS, EMAX)) k_cols_spec(Grid g, FftPlan<T> pl, const T* __restrict__ lam_cols, int cols_per_cta, T* data,
                            PcgCtrl* ctrl, RedScratch rs, int site, int it, Push ps, int nfull) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(smraw);
  pdl_enter(g);
  if (MODE != MODE_API && ctrl->done) return;
  const T accT = cols_panel<T, EMAX, LS>(g, pl, lam_cols, cols_per_cta, data, ps, nfull, (int)blockIdx.x, buf);
  pdl_trigger(g);
  if (MODE != MODE_API) {
    double acc[1] = {(double)accT};
    double tot[1];
    if (red_final<1>(acc, rs, site, tot) && threadIdx.x == 0) fin_k3(ctrl, tot, it, MODE);
  }
}

// slack part of the standalone preconditioner: z_s = r_s / (d + 1/tau)
template <typename T>
__global__ void k_precond_slack(Grid g, const T* __restrict__ r, const T* __restrict__ dv, const T* __restrict__ dh,
                                T* z) {
  const T inv = (T)g.inv_tau;
  PU_FOR_CELLS(g, i, j) {
    const long long o = (long long)i * g.ld + j;
    z[o + g.plane] = dn_ok(g, i) ? r[o + g.plane] / (dv[o] + inv) : (T)0;
    z[o + 2 * g.plane] = (j < g.m - 1) ? r[o + 2 * g.plane] / (dh[o] + inv) : (T)0;
  }
}

}  // namespace pu
