// Shared-memory FFT engine and DCT-II/III building blocks (sm_100a).
//
// The reference applies its Poisson preconditioner with dense eigenbases
// (preconditioner.py:64-100).  Those bases are the orthonormal DCT-II basis
// (SURVEY.md §0 fact 2), so here every 1-D transform is a DCT computed by
// Makhoul's n-point method on a complex FFT that packs two real sequences:
//     v[p(m)] = a[m] + i b[m],  p(m) = m/2 (m even), n-1-(m-1)/2 (m odd)
//     Z = FFT_n(v);  X_a[k] = s_k Re(e^{-i pi k/2n} (Z_k + conj Z_{n-k})/2), ...
// The FFT itself is a Stockham autosort transform on one shared-memory
// buffer: each stage loads its butterflies into registers, barriers, and
// writes them back (radix 16/8/4/2 and 3/5/7).  Lengths with other prime
// factors use Bluestein's chirp-z on an internal power-of-two length L.
#pragma once

#include "pu_common.cuh"

namespace pu {

#define PU_FFT_MAX_STAGES 20
#ifndef PU_PANEL_COLS
#define PU_PANEL_COLS 4  // columns per CTA of the column-transform kernel (2 packed sequences)
#endif

// Complex values per thread of one FFT stage (the largest radix): 16 in fp32;
// in fp64 PU_F64_EMAX (8: radix-8 stages at <= 64 registers; 16: radix-16
// stages, one fewer shared-memory round trip per 4096-point FFT, at <= 128
// registers with half the threads).
#ifndef PU_F64_EMAX
#define PU_F64_EMAX 8
#endif
template <typename T>
__host__ __device__ constexpr int emax_of() { return sizeof(T) == 4 ? 16 : PU_F64_EMAX; }

// Per-instantiation launch bounds.  Transform kernels run every sequence of
// the CTA in one group (no loop over sequence groups: ptxas hoists the
// thread-invariant twiddles/addresses of such loops and spills), so a CTA
// has nseq * L / EMAX threads: up to 1024 at <= 64 registers, or up to 512
// at <= 128 registers for 16 complex doubles per thread.
__host__ __device__ constexpr int fft_max_threads(int LS, int EMAX, int tsize = 4) {
  return (tsize == 8 && EMAX >= 16) ? 512 : 1024;
}
__host__ __device__ constexpr int fft_min_blocks(int LS, int EMAX) { return 1; }

__host__ __device__ constexpr int ldseq_for(int L);
// columns per CTA of a static column plan: 4, 2 or 1 packed sequences, the
// most that fit one thread group and the shared memory (2 columns each)
__host__ __device__ constexpr int static_panel_cols(int L, int emax, int tsize = 4) {
  return (4 * L <= fft_max_threads(L, emax, tsize) * emax && 4LL * ldseq_for(L) * 2 * tsize <= 220 * 1024)
             ? 2 * PU_PANEL_COLS
             : ((2 * L <= fft_max_threads(L, emax, tsize) * emax && 2LL * ldseq_for(L) * 2 * tsize <= 220 * 1024)
                    ? PU_PANEL_COLS
                    : PU_PANEL_COLS / 2);
}
#define PU_FFT_MAX_THREADS 1024  // absolute per-CTA thread cap of the transform kernels

// Plan for one transform length (built on the host, pu_api.cu HostPlan).
template <typename T>
struct FftPlan {
  int n;                  // transform length
  int L;                  // internal FFT length (n, or Bluestein power of two)
  int nst;                // number of Stockham stages
  int bluestein;          // 1 if Bluestein
  int rad[PU_FFT_MAX_STAGES];
  int ldseq;              // shared-memory stride between sequences (padded)
  int cap;                // complex values per thread a stage can hold (min R*floor(EMAX/R))
  const cplx<T>* tw;      // [L]  exp(-2 pi i k / L)                      (runtime plan)
  const cplx<T>* stw;     // per-stage W_{NS R}^k, k < NS, of the static plan (stage >= 1)
  const cplx<T>* chirp;   // [n]  exp(-i pi k^2 / n)                     (Bluestein)
  const cplx<T>* filt;    // [L]  FFT_L(conj chirp, symmetric)/L          (Bluestein)
  const cplx<T>* dct2w;   // [n]  s_k (cos, sin)(pi k / 2n)   DCT-II post, scale folded
  const cplx<T>* dct3w;   // [n]  (cos, sin)(pi k / 2n) / (s_k n)  DCT-III pre, 1/n folded
  const T* lam;           // [n]  2 - 2 cos(pi k / n) = 4 sin^2(pi k / 2n), lam[0] = 0
  int stage1;             // row pipeline stages one row at a time (long rows, pu_pipe.cuh)
};

// Bank-conflict padding: one complex slot every 16.
__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }

// Makhoul permutation p(m).
__device__ __forceinline__ int mperm(int m, int n) { return (m & 1) ? (n - 1 - (m >> 1)) : (m >> 1); }

// ---------------------------------------------------------------------------
// In-register DFTs (forward, e^{-2 pi i jk/R}).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ cplx<T> mul_negi(cplx<T> a) { return mk<T>(a.y, -a.x); }  // a * (-i)

template <typename T, int R>
struct Dft;

template <typename T>
struct Dft<T, 2> {
  __device__ __forceinline__ static void run(cplx<T>* a) {
    cplx<T> t = a[1];
    a[1] = csub<T>(a[0], t);
    a[0] = cadd<T>(a[0], t);
  }
};

template <typename T>
struct Dft<T, 4> {
  __device__ __forceinline__ static void run(cplx<T>* a) {
    cplx<T> s0 = cadd<T>(a[0], a[2]), d0 = csub<T>(a[0], a[2]);
    cplx<T> s1 = cadd<T>(a[1], a[3]), d1 = mul_negi<T>(csub<T>(a[1], a[3]));
    a[0] = cadd<T>(s0, s1);
    a[2] = csub<T>(s0, s1);
    a[1] = cadd<T>(d0, d1);
    a[3] = csub<T>(d0, d1);
  }
};

// cos/sin(2 pi k / 16), k = 0..15
__device__ __forceinline__ double c16(int k) {
  const double t[16] = {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508984,
                        0.0, -0.38268343236508984, -0.70710678118654757, -0.92387953251128674,
                        -1.0, -0.92387953251128674, -0.70710678118654757, -0.38268343236508984,
                        0.0, 0.38268343236508984, 0.70710678118654757, 0.92387953251128674};
  return t[k & 15];
}
__device__ __forceinline__ double s16(int k) { return c16(k + 12); }  // sin(x) = cos(x - pi/2)

// twiddle W_16^k = exp(-2 pi i k/16) applied to a
template <typename T, int K>
__device__ __forceinline__ cplx<T> w16(cplx<T> a) {
  constexpr int k = K & 15;
  if constexpr (k == 0) return a;
  else if constexpr (k == 4) return mul_negi<T>(a);
  else if constexpr (k == 8) return mk<T>(-a.x, -a.y);
  else if constexpr (k == 12) return mk<T>(-a.y, a.x);
  else {
    const T c = (T)c16(k), s = (T)(-s16(k));
    return mk<T>(a.x * c - a.y * s, a.x * s + a.y * c);
  }
}

template <typename T>
struct Dft<T, 8> {
  __device__ __forceinline__ static void run(cplx<T>* a) {
    // radix-2 DIT over two radix-4 halves
    cplx<T> e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
    Dft<T, 4>::run(e);
    Dft<T, 4>::run(o);
    cplx<T> t1 = w16<T, 2>(o[1]), t2 = w16<T, 4>(o[2]), t3 = w16<T, 6>(o[3]);
    a[0] = cadd<T>(e[0], o[0]); a[4] = csub<T>(e[0], o[0]);
    a[1] = cadd<T>(e[1], t1);   a[5] = csub<T>(e[1], t1);
    a[2] = cadd<T>(e[2], t2);   a[6] = csub<T>(e[2], t2);
    a[3] = cadd<T>(e[3], t3);   a[7] = csub<T>(e[3], t3);
  }
};

template <typename T>
struct Dft<T, 16> {
  __device__ __forceinline__ static void run(cplx<T>* a) {
    // 4 x 4: columns (stride 4), twiddle, rows
    cplx<T> c0[4] = {a[0], a[4], a[8], a[12]};
    cplx<T> c1[4] = {a[1], a[5], a[9], a[13]};
    cplx<T> c2[4] = {a[2], a[6], a[10], a[14]};
    cplx<T> c3[4] = {a[3], a[7], a[11], a[15]};
    Dft<T, 4>::run(c0); Dft<T, 4>::run(c1); Dft<T, 4>::run(c2); Dft<T, 4>::run(c3);
    // twiddle c_q[k] *= W16^(q k)
    c1[1] = w16<T, 1>(c1[1]); c1[2] = w16<T, 2>(c1[2]); c1[3] = w16<T, 3>(c1[3]);
    c2[1] = w16<T, 2>(c2[1]); c2[2] = w16<T, 4>(c2[2]); c2[3] = w16<T, 6>(c2[3]);
    c3[1] = w16<T, 3>(c3[1]); c3[2] = w16<T, 6>(c3[2]); c3[3] = w16<T, 9>(c3[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cplx<T> r[4] = {c0[k], c1[k], c2[k], c3[k]};
      Dft<T, 4>::run(r);
      a[k] = r[0]; a[k + 4] = r[1]; a[k + 8] = r[2]; a[k + 12] = r[3];
    }
  }
};

// Odd primes: direct O(R^2) DFT with exact constant tables.
template <typename T, int R>
struct DftOdd {
  __device__ __forceinline__ static double cs(int k) {
    // cos(2 pi k / R) for R in {3,5,7}
    if (R == 3) { const double t[3] = {1.0, -0.5, -0.5}; return t[k % 3]; }
    if (R == 5) { const double t[5] = {1.0, 0.30901699437494745, -0.80901699437494734, -0.80901699437494734, 0.30901699437494745}; return t[k % 5]; }
    const double t[7] = {1.0, 0.62348980185873359, -0.22252093395631434, -0.90096886790241915,
                         -0.90096886790241915, -0.22252093395631434, 0.62348980185873359};
    return t[k % 7];
  }
  __device__ __forceinline__ static double sn(int k) {
    // sin(2 pi k / R)
    if (R == 3) { const double t[3] = {0.0, 0.86602540378443860, -0.86602540378443860}; return t[k % 3]; }
    if (R == 5) { const double t[5] = {0.0, 0.95105651629515353, 0.58778525229247314, -0.58778525229247314, -0.95105651629515353}; return t[k % 5]; }
    const double t[7] = {0.0, 0.78183148246802981, 0.97492791218182362, 0.43388373911755812,
                         -0.43388373911755812, -0.97492791218182362, -0.78183148246802981};
    return t[k % 7];
  }
  __device__ __forceinline__ static void run(cplx<T>* a) {
    cplx<T> out[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      T re = a[0].x, im = a[0].y;
#pragma unroll
      for (int j = 1; j < R; ++j) {
        const T c = (T)cs(j * k), s = (T)(-sn(j * k));
        re += a[j].x * c - a[j].y * s;
        im += a[j].x * s + a[j].y * c;
      }
      out[k] = mk<T>(re, im);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = out[k];
  }
};
template <typename T> struct Dft<T, 3> { __device__ __forceinline__ static void run(cplx<T>* a) { DftOdd<T, 3>::run(a); } };
template <typename T> struct Dft<T, 5> { __device__ __forceinline__ static void run(cplx<T>* a) { DftOdd<T, 5>::run(a); } };
template <typename T> struct Dft<T, 7> { __device__ __forceinline__ static void run(cplx<T>* a) { DftOdd<T, 7>::run(a); } };

// ---------------------------------------------------------------------------
// One Stockham stage over sequences [seq0, seq0 + nseq) of length L held in
// shared memory.  Butterfly j (0 <= j < L/R) of a sequence reads X[j + r L/R],
// applies the twiddles W_{Ns R}^{r (j mod Ns)}, runs a radix-R DFT and writes
// Y[(j / Ns) Ns R + (j mod Ns) + r Ns].  Each thread holds at most EMAX complex
// values (Q = EMAX/R butterflies), so the caller sizes the sequence group so
// that blockDim.x * Q >= nseq * L / R.  FIRST stages (Ns = 1) need no twiddles;
// plans put the radix with Q > 1 first so the others run with Q = 1.
// ---------------------------------------------------------------------------
template <typename T, int R, int EMAX, bool FIRST>
__device__ __forceinline__ void fft_stage(cplx<T>* buf, int L, int seq0, int nseq, int ldseq, int Ns,
                                          const cplx<T>* __restrict__ tw) {
  constexpr int Q = EMAX / R;
  static_assert(Q >= 1, "radix exceeds per-thread capacity");
  const int nb = L / R;
  const int total = nseq * nb;
  cplx<T> v[Q][R];
  int obase[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = threadIdx.x + q * blockDim.x;
    obase[q] = -1;
    if (b < total) {
      const int s = b / nb;
      const int j = b - s * nb;
      const cplx<T>* sb = buf + (seq0 + s) * ldseq;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        PU_ASSERT(spad(j + r * nb) < ldseq);
        v[q][r] = *sm_chk(&sb[spad(j + r * nb)]);
      }
      if constexpr (FIRST) {
        obase[q] = (seq0 + s) * ldseq + j * R;
      } else {
        const int k = j % Ns;
        const int tws = (L / (Ns * R)) * k;
#pragma unroll
        for (int r = 1; r < R; ++r) v[q][r] = cmul<T>(v[q][r], __ldg(tw + r * tws));
        obase[q] = (seq0 + s) * ldseq + (j - k) * R + k;
      }
      Dft<T, R>::run(v[q]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (obase[q] >= 0) {
      // obase already includes the sequence offset; spad acts on the in-sequence index
      const int s0 = (obase[q] / ldseq) * ldseq;
      const int i0 = obase[q] - s0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        PU_ASSERT(spad(i0 + r * (FIRST ? 1 : Ns)) < ldseq);
        *sm_chk(&buf[s0 + spad(i0 + r * (FIRST ? 1 : Ns))]) = v[q][r];
      }
    }
  }
  __syncthreads();
}

template <typename T, int EMAX, bool FIRST>
__device__ __forceinline__ void fft_stage_rt(int R, cplx<T>* buf, int L, int seq0, int nseq, int ldseq, int Ns,
                                             const cplx<T>* tw) {
  switch (R) {
    case 16: if constexpr (EMAX >= 16) fft_stage<T, 16, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 8: fft_stage<T, 8, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 4: fft_stage<T, 4, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 2: fft_stage<T, 2, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 3: fft_stage<T, 3, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 5: fft_stage<T, 5, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    case 7: fft_stage<T, 7, EMAX, FIRST>(buf, L, seq0, nseq, ldseq, Ns, tw); break;
    default: break;
  }
}

// Full forward FFT of length plan.L on nseq sequences (in place, natural
// order), processed in groups of sequences sized to the thread block.
template <typename T, int EMAX>
__device__ __forceinline__ void fft_pow(cplx<T>* buf, int nseq, const FftPlan<T>& pl) {
  const int grp = max(1, (int)(blockDim.x * pl.cap) / pl.L);
  for (int sg = 0; sg < nseq; sg += grp) {
    const int cnt = min(grp, nseq - sg);
    int Ns = 1;
    for (int st = 0; st < pl.nst; ++st) {
      const int R = pl.rad[st];
      if (st == 0) fft_stage_rt<T, EMAX, true>(R, buf, pl.L, sg, cnt, pl.ldseq, 1, pl.tw);
      else fft_stage_rt<T, EMAX, false>(R, buf, pl.L, sg, cnt, pl.ldseq, Ns, pl.tw);
      Ns *= R;
    }
  }
}

// ---------------------------------------------------------------------------
// Compile-time plans for power-of-two internal lengths (the production sizes):
// stage 0 takes the remainder radix (twiddle-free, Q = EMAX/R butterflies per
// thread), every later stage the largest radix (16 for fp32, 8 for fp64) with
// Q = 1.  All strides are constants, so addressing folds into immediates.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ldseq_for(int L) { return (L + (L >> 4) + 2) + ((L + (L >> 4) + 2) & 1); }

__host__ __device__ constexpr int first_radix_rt(int L, int emax) {
  const int big = emax >= 16 ? 16 : 8;
  int rem = L;
  while (rem > 1 && rem % big == 0) rem /= big;
  return rem == 1 ? big : rem;
}
template <int L, int EMAX>
__host__ __device__ constexpr int first_radix() { return first_radix_rt(L, EMAX); }

// GRP: stage barriers per sequence (named barrier 2 + s over the NB threads
// that own sequence s; needs Q == 1 and NB a multiple of 32) instead of
// CTA-wide, so the sequences of a column panel progress independently.
template <bool GRP>
__device__ __forceinline__ void stage_sync(int nb, int nseq) {
  if constexpr (GRP) {
    const int s = threadIdx.x / nb;
    if (s < nseq) asm volatile("bar.sync %0, %1;" ::"r"(2 + s), "r"(nb) : "memory");
  } else {
    __syncthreads();
  }
}

template <typename T, int R, int EMAX, int L, int NS, int OFF, bool GRP = false>
__device__ __forceinline__ void fft_stage_s(cplx<T>* buf, int seq0, int nseq, const cplx<T>* __restrict__ stw) {
  constexpr int Q = EMAX / R;
  constexpr int NB = L / R;
  constexpr int LD = ldseq_for(L);
  static_assert(Q >= 1 && NB * R == L, "bad static stage");
  static_assert(!GRP || (Q == 1 && NB % 32 == 0), "grouped stages need one butterfly per thread");
  const int total = nseq * NB;
  cplx<T> v[Q][R];
  int ob[Q], sbase[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = threadIdx.x + q * blockDim.x;
    ob[q] = -1;
    if (b < total) {
      const int s = b / NB;
      const int j = b - s * NB;
      const int base = (seq0 + s) * LD;
      sbase[q] = base;
      if constexpr (NB % 16 == 0) {
        // spad(j + r NB) = spad(j) + r (NB + NB/16): one base register, immediate offsets
        const cplx<T>* src = buf + base + spad(j);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          PU_ASSERT(spad(j) + r * (NB + NB / 16) < LD);
          v[q][r] = *sm_chk(&src[r * (NB + NB / 16)]);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          PU_ASSERT(spad(j + r * NB) < LD);
          v[q][r] = *sm_chk(&buf[base + spad(j + r * NB)]);
        }
      }
      if constexpr (NS > 1) {
        // twiddles W_{NS R}^{r k}: one table load (w = W^k), powers by a
        // balanced product tree (depth <= log2 R, a few ulp)
        const int k = j % NS;
        cplx<T> w[R];
        // opaque table pointer: keeps the (loop-invariant) twiddle loads and their
        // power tree inside persistent loops instead of hoisted into registers
        unsigned long long tp = reinterpret_cast<unsigned long long>(stw);
        asm volatile("" : "+l"(tp));
        w[1] = __ldg(reinterpret_cast<const cplx<T>*>(tp) + OFF + k);
#pragma unroll
        for (int r = 2; r < R; ++r) w[r] = cmul<T>(w[r / 2], w[r - r / 2]);
#pragma unroll
        for (int r = 1; r < R; ++r) v[q][r] = cmul<T>(v[q][r], w[r]);
        ob[q] = (j - k) * R + k;
      } else {
        ob[q] = j * R;
      }
      Dft<T, R>::run(v[q]);
    }
  }
  stage_sync<GRP>(NB, nseq);
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ob[q] >= 0) {
      const int base = sbase[q];
      const int i0 = ob[q];
      if constexpr (NS % 16 == 0) {
        cplx<T>* dst = buf + base + spad(i0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          PU_ASSERT(spad(i0) + r * (NS + NS / 16) < LD);
          *sm_chk(&dst[r * (NS + NS / 16)]) = v[q][r];
        }
      } else if constexpr (NS == 1 && R == 16) {
        cplx<T>* dst = buf + base + spad(i0);  // i0 = 16 j: spad(16 j + r) = 17 j + r
#pragma unroll
        for (int r = 0; r < R; ++r) {
          PU_ASSERT(spad(i0) + r < LD);
          *sm_chk(&dst[r]) = v[q][r];
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          PU_ASSERT(spad(i0 + r * NS) < LD);
          *sm_chk(&buf[base + spad(i0 + r * NS)]) = v[q][r];
        }
      }
    }
  }
  stage_sync<GRP>(NB, nseq);
}

// Stage s >= 1 of the static plan reads W_{NS R}^k, k < NS, from its block at
// OFF; blocks are laid out in stage order (mirrored by HostPlan::build).
template <typename T, int EMAX, int L, int NS, int OFF>
__device__ __forceinline__ void fft_stages_s(cplx<T>* buf, int seq0, int nseq, const cplx<T>* stw) {
  if constexpr (NS < L) {
    constexpr int R = (NS == 1) ? first_radix<L, EMAX>() : (EMAX >= 16 ? 16 : 8);
    fft_stage_s<T, R, EMAX, L, NS, OFF>(buf, seq0, nseq, stw);
    fft_stages_s<T, EMAX, L, NS * R, (NS == 1 ? OFF : OFF + NS)>(buf, seq0, nseq, stw);
  }
}

// Stages NS in [NS, STOP) of the static plan (the column kernel runs the
// first / last stage itself, straight from / to global memory).
template <typename T, int EMAX, int L, int NS, int OFF, int STOP, bool GRP = false>
__device__ __forceinline__ void fft_stages_range(cplx<T>* buf, int seq0, int nseq, const cplx<T>* stw) {
  if constexpr (NS < STOP) {
    constexpr int R = (NS == 1) ? first_radix<L, EMAX>() : (EMAX >= 16 ? 16 : 8);
    fft_stage_s<T, R, EMAX, L, NS, OFF, GRP>(buf, seq0, nseq, stw);
    fft_stages_range<T, EMAX, L, NS * R, (NS == 1 ? OFF : OFF + NS), STOP, GRP>(buf, seq0, nseq, stw);
  }
}

// every stage of the static plan of L has one butterfly per thread and NB a
// multiple of 32 (grouped barriers possible)
template <int L, int EMAX>
__host__ __device__ constexpr bool grp_ok() {
  return EMAX / first_radix<L, EMAX>() == 1 && (L / first_radix<L, EMAX>()) % 32 == 0 &&
         (L / (EMAX >= 16 ? 16 : 8)) % 32 == 0;
}

// offset of stage NS's twiddle block in pl.stw (mirrors fft_stages_s)
template <int L, int EMAX>
__host__ __device__ constexpr int stage_off(int target) {
  int ns = first_radix<L, EMAX>(), off = 0;
  while (ns < target) { off += ns; ns *= (EMAX >= 16 ? 16 : 8); }
  return off;
}

// Forward FFT of internal length L on all sequences; LS > 0 selects the
// compile-time plan (requires pl.L == LS), LS == 0 the runtime plan.
template <typename T, int EMAX, int LS>
__device__ __forceinline__ void fft_internal(cplx<T>* buf, int nseq, const FftPlan<T>& pl) {
  if constexpr (LS > 0) {
    // the launch guarantees blockDim.x * EMAX >= nseq * LS: one group, no loop
    fft_stages_s<T, EMAX, LS, 1, 0>(buf, 0, nseq, pl.stw);
  } else {
    fft_pow<T, EMAX>(buf, nseq, pl);
  }
}

// Forward DFT of length plan.n (entries [0, n) of each sequence), in place.
// Callers must __syncthreads() before (data staged) — this returns synced.
template <typename T, int EMAX, int LS>
__device__ __forceinline__ void fft_n(cplx<T>* buf, int nseq, const FftPlan<T>& pl) {
  if (!pl.bluestein) {
    fft_internal<T, EMAX, LS>(buf, nseq, pl);
    return;
  }
  const int n = pl.n, L = pl.L;
  // a_m = x_m * chirp_m, zero-padded to L
  for (int e = threadIdx.x; e < nseq * L; e += blockDim.x) {
    const int s = e / L, m = e - s * L;
    cplx<T>* sb = buf + s * pl.ldseq;
    if (m < n) sb[spad(m)] = cmul<T>(sb[spad(m)], __ldg(pl.chirp + m));
    else sb[spad(m)] = mk<T>((T)0, (T)0);
  }
  __syncthreads();
  fft_internal<T, EMAX, LS>(buf, nseq, pl);
  for (int e = threadIdx.x; e < nseq * L; e += blockDim.x) {
    const int s = e / L, k = e - s * L;
    cplx<T>* sb = buf + s * pl.ldseq;
    sb[spad(k)] = cconj<T>(cmul<T>(sb[spad(k)], __ldg(pl.filt + k)));
  }
  __syncthreads();
  fft_internal<T, EMAX, LS>(buf, nseq, pl);
  for (int e = threadIdx.x; e < nseq * n; e += blockDim.x) {
    const int s = e / n, k = e - s * n;
    cplx<T>* sb = buf + s * pl.ldseq;
    sb[spad(k)] = cmul<T>(cconj<T>(sb[spad(k)]), __ldg(pl.chirp + k));
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// DCT-II post-processing for the packed pair (a + i b) at bins k and n-k.
// Given Z = FFT(v), returns the orthonormal DCT-II coefficients.
// ---------------------------------------------------------------------------
template <typename T>
struct PairOut { T a_k, b_k, a_nk, b_nk; };

template <typename T>
__device__ __forceinline__ PairOut<T> dct2_post(cplx<T> zk, cplx<T> znk, int k, int nk, const FftPlan<T>& pl) {
  const T h = (T)0.5;
  const T reA = h * (zk.x + znk.x), imA = h * (zk.y - znk.y);
  const T reB = h * (zk.y + znk.y), imB = -h * (zk.x - znk.x);
  const cplx<T> wk = __ldg(pl.dct2w + k), wn = __ldg(pl.dct2w + nk);  // s_k e^{i theta_k}
  PairOut<T> o;
  o.a_k = wk.x * reA + wk.y * imA;
  o.b_k = wk.x * reB + wk.y * imB;
  o.a_nk = wn.x * reA - wn.y * imA;
  o.b_nk = wn.x * reB - wn.y * imB;
  return o;
}

// DCT-III pre-processing: from orthonormal coefficients (a_k, a_nk, b_k, b_nk)
// build conj(Z'_k), conj(Z'_nk) where Z' = V_a + i V_b and
// V_k = e^{i pi k/2n} (Y_k - i Y_{n-k}) / n, Y = X / s (s_k = s_{n-k} for
// k >= 1; V_0 = Y_0 / n).  A forward FFT of the conjugated data is then
// n * conj(IFFT), so the DCT-III output is (Re, -Im) of it directly.
template <typename T>
__device__ __forceinline__ void dct3_pre(T ak, T ank, T bk, T bnk, int k, int nk, const FftPlan<T>& pl,
                                         cplx<T>& out_k, cplx<T>& out_nk) {
  const cplx<T> wk = __ldg(pl.dct3w + k);
  T vaRe, vaIm, vbRe, vbIm;
  if (k == 0) {
    vaRe = ak * wk.x; vaIm = 0; vbRe = bk * wk.x; vbIm = 0;
  } else {
    vaRe = wk.x * ak + wk.y * ank; vaIm = wk.y * ak - wk.x * ank;
    vbRe = wk.x * bk + wk.y * bnk; vbIm = wk.y * bk - wk.x * bnk;
  }
  out_k = mk<T>(vaRe - vbIm, -(vaIm + vbRe));  // conj(Va + i Vb)
  if (nk != k) {
    const cplx<T> wn = __ldg(pl.dct3w + nk);
    const T uaRe = wn.x * ank + wn.y * ak, uaIm = wn.y * ank - wn.x * ak;
    const T ubRe = wn.x * bnk + wn.y * bk, ubIm = wn.y * bnk - wn.x * bk;
    out_nk = mk<T>(uaRe - ubIm, -(uaIm + ubRe));
  }
}

// conj(Z'_k) alone (the out_k half of dct3_pre, same arithmetic)
template <typename T>
__device__ __forceinline__ cplx<T> dct3_pre_k(T ak, T ank, T bk, T bnk, int k, const FftPlan<T>& pl) {
  const cplx<T> wk = __ldg(pl.dct3w + k);
  T vaRe, vaIm, vbRe, vbIm;
  if (k == 0) {
    vaRe = ak * wk.x; vaIm = 0; vbRe = bk * wk.x; vbIm = 0;
  } else {
    vaRe = wk.x * ak + wk.y * ank; vaIm = wk.y * ak - wk.x * ank;
    vbRe = wk.x * bk + wk.y * bnk; vbIm = wk.y * bk - wk.x * bnk;
  }
  return mk<T>(vaRe - vbIm, -(vaIm + vbRe));
}

// division for the spectral scaling: a * MUFU reciprocal (~1 ulp) in fp32,
// rcp-based in fp64; deterministic, so repeated applications agree bitwise
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_div(float a, float b) { return a * rcp_approx(b); }
// fp64: MUFU reciprocal seed + two Newton steps (<= 1 ulp, no IEEE rounding
// fix-up path: the spectral scaling is ~6% of K3's fp64 stall samples with __drcp_rn)
__device__ __forceinline__ double rcp_nr(double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  double e = fma(-b, y, 1.0);
  y = fma(e, y, y);
  e = fma(-b, y, 1.0);
  return fma(e, y, y);
}
__device__ __forceinline__ double fast_div(double a, double b) { return a * rcp_nr(b); }

// correctly rounded reciprocal
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }

}  // namespace pu
