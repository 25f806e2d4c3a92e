// Pipelined row transforms (K2b: row DCT-II, K4: row DCT-III) on sm_100a.
//
// One CTA per row pair (one packed complex FFT).  The two raw rows are
// fetched by the bulk-copy engine (TMA: cp.async.bulk + mbarrier transaction
// counting) in one shot, without registers or per-thread loads; several CTAs
// per SM overlap their copies with each other's FFTs.  (A persistent variant
// that prefetched the next pair made ptxas hoist every thread-invariant
// twiddle and address out of the loop and spill; one pair per CTA compiles to
// 64 registers.)
#pragma once

#include "pu_pcg.cuh"

namespace pu {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on *m
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
// bulk prefetch of `bytes` (multiple of 16) global bytes into L2 (TMA engine)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "PU_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PU_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}

// Opaque copy of a pointer: stops the compiler from hoisting per-iteration
// shared-memory addresses out of the persistent loop (it did, and spilled).
template <typename P>
__device__ __forceinline__ P* launder_ptr(P* p) {
  unsigned long long v = reinterpret_cast<unsigned long long>(p);
  asm volatile("" : "+l"(v));
  return reinterpret_cast<P*>(v);
}

// bytes of one staged row (multiple of 16 for cp.async.bulk)
__host__ __device__ constexpr unsigned stage_row_bytes(int n, int tsize) {
  return ((unsigned)n * (unsigned)tsize + 15u) & ~15u;
}
// dynamic shared memory of k_rows_pipe (`rows_staged` = 2, or 1 for pl.stage1)
__host__ __device__ constexpr size_t rows_pipe_smem(int n, int tsize, int ldseq, int rows_staged = 2) {
  return 128 + (size_t)rows_staged * stage_row_bytes(n, tsize) + (size_t)ldseq * 2 * tsize;
}

// Forward row transform of a static power-of-two plan (K2b): the first FFT
// stage gathers its butterflies straight from the two staged rows (Makhoul
// order: FFT index idx holds column 2 idx, or 2n - 1 - 2 idx past n/2) into
// registers, so the packing pass disappears and, once every thread holds its
// inputs, the FFT buffer may overwrite the staging: the forward kernel needs
// max(2 rows, FFT buffer) of shared memory instead of their sum (4 instead of
// 3 CTAs per SM at 4096 fp32).
template <int L, int EMAX>
__host__ __device__ constexpr bool rows_fused_ok() {
  constexpr int r0 = first_radix<L, EMAX>();
  return (r0 == 2 || r0 == 4 || r0 == 8 || r0 == 16) && EMAX % r0 == 0;
}
// shared memory of a fused launch from that of the plain one (128 + 2 staged rows + buffer)
__host__ __device__ constexpr size_t rows_fused_smem(size_t plain, int tsize, int ldseq) {
  return 128 + (plain - 128 - (size_t)ldseq * 2 * tsize > (size_t)ldseq * 2 * tsize
                    ? plain - 128 - (size_t)ldseq * 2 * tsize : (size_t)ldseq * 2 * tsize);
}

template <typename T, int EMAX, int L>
__device__ __forceinline__ void rows_first_stage(const T* sa, const T* sb, bool hasb, cplx<T>* buf) {
  constexpr int R = first_radix<L, EMAX>(), Q = EMAX / R, NB = L / R;
  cplx<T> v[Q][R];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = threadIdx.x + q * blockDim.x;
    if (j >= NB) break;  // the launch may round the CTA up (>= 64 threads)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = r < R / 2 ? 2 * (j + r * NB) : 2 * L - 1 - 2 * (j + r * NB);
      v[q][r] = mk<T>(sa[m], hasb ? sb[m] : (T)0);
    }
    Dft<T, R>::run(v[q]);
  }
  __syncthreads();  // every staged value is in registers: buf may overwrite the staging
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (threadIdx.x + q * blockDim.x >= NB) break;
    cplx<T>* dst = buf + spad((threadIdx.x + q * blockDim.x) * R);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[r] = v[q][r];
  }
}

// Inverse row transform (K4), same scheme: the first FFT stage builds its
// inputs with the DCT-III pre-twiddle straight from the staged spectrum rows
// (bins k and n - k), the buffer aliases the staging, and the axpy reads the
// old direction from global memory (no staging left for its prefetch).
template <typename T, int EMAX, int L>
__device__ __forceinline__ void rows_first_stage_inv(const T* sa, const T* sb, bool hasb, cplx<T>* buf,
                                                     const FftPlan<T>& pl) {
  constexpr int R = first_radix<L, EMAX>(), Q = EMAX / R, NB = L / R;
  cplx<T> v[Q][R];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j = threadIdx.x + q * blockDim.x;
    if (j >= NB) break;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = j + r * NB, nk = k == 0 ? 0 : L - k;
      v[q][r] = hasb ? dct3_pre_k<T>(sa[k], sa[nk], sb[k], sb[nk], k, pl)
                     : dct3_pre_k<T>(sa[k], sa[nk], (T)0, (T)0, k, pl);
    }
    Dft<T, R>::run(v[q]);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (threadIdx.x + q * blockDim.x >= NB) break;
    cplx<T>* dst = buf + spad((threadIdx.x + q * blockDim.x) * R);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[r] = v[q][r];
  }
}

// Row-sharded grids (pu_create_band): the spectrum travels between the row
// bands and the column bands of the all-to-all transpose in a packed layout,
// chunk q = columns [q mb, (q + 1) mb) of the band's rows, row pitch mb:
// element (i, k) at (k / mb) * chunk + i * mb + k % mb.  The forward kernel
// writes it, the inverse one reads its rows as nq bulk copies.  nq = 0: plain.
//
// With `peers` set, the transpose is fused into the kernels instead: element
// (band row i, column k) lives in rank q = k / mb's column block (N x mb,
// pitch mb; peers[q] = its address, on this GPU or a peer mapped over NVLink)
// at row row0 + i, so the forward kernel stores straight into the other
// ranks' blocks and the inverse kernel fetches its rows from them.
struct Pack {
  int nq;
  int mb;
  long long chunk;
  const unsigned long long* peers;  // device array of nq block addresses, or null
  long long row0;                   // this band's first global row
  FastDiv mbd;                      // k / mb
  int own_q = -1;                   // inverse (K4) in peer mode: chunk own_q is read in place from peers[own_q]
};

// pl.stage1 (rows too long for two staged rows next to the FFT buffer, e.g.
// 16384 fp32): one staging row; row b is fetched after row a has been packed
// (its half of the packing is linear, so the sum is bitwise the same), and
// K4 reads the old direction straight from global memory.
//
// INV with `pold` != nullptr (PCG K4): out = beta * pold + DCT-III(in), i.e.
// the u block of the next search direction (pcg.py:107-108); `first` gives
// out = DCT-III(in) (p = z at iteration 0).
// debug check: staging rows + FFT buffer inside the CTA's shared memory
template <typename T>
__device__ __forceinline__ bool row_pair_smem_ok(unsigned char* smraw, bool one, bool ffuse, unsigned RB, int ldseq) {
  const size_t need = 128 + (ffuse ? 0 : (one ? 1 : 2) * (size_t)RB) + (size_t)ldseq * sizeof(cplx<T>);
  const size_t need_f = 128 + (size_t)(one ? 1 : 2) * RB;
  sm_chk(smraw + (need > need_f ? need : need_f) - 1);
  return true;
}

// One row pair s of K2b (forward) / K4 (inverse); the mbarrier at smraw is
// initialised by the caller and `ph` is its current phase parity (advanced
// here by the phases this pair consumed).  k_rows_pipe runs one pair per CTA;
// the persistent small-grid PCG kernel (pu_persist.cuh) loops over pairs.
template <typename T, int EMAX, int LS, bool INV>
__device__ __forceinline__ void rows_pair(const Grid& g, const FftPlan<T>& pl, const T* __restrict__ in,
                                          T* __restrict__ out, const PcgCtrl* ctrl, const T* __restrict__ pold,
                                          int first, const Pack& pk, int s, unsigned char* smraw, unsigned& ph) {
  int waits = 0;  // mbarrier phases completed by this row pair
  const int n = LS > 0 ? LS : g.m;  // static plans only when n == L
  const int S = (g.n + 1) >> 1;     // row pairs
  const unsigned RBrow = stage_row_bytes(n, sizeof(T));  // one plain row
  const bool pin = INV && pk.nq > 0, pout = !INV && pk.nq > 0;
  const unsigned RB = pin ? (unsigned)(pk.nq * pk.mb * sizeof(T)) : RBrow;  // one staged input row
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw);
  T* sa = reinterpret_cast<T*>(smraw + 128);
  const bool one = pl.stage1 != 0;
  constexpr bool FFUSE = LS > 0 && rows_fused_ok<(LS > 0 ? LS : 512), EMAX>();
  const bool ffuse = FFUSE && !one;  // launched with rows_fused_smem (DctLaunch::rows_pipe)
  T* sb = one ? sa : reinterpret_cast<T*>(smraw + 128 + RB);
  cplx<T>* buf0 = reinterpret_cast<cplx<T>*>(smraw + 128 + (ffuse ? 0 : (one ? 1 : 2) * RB));
  PU_ASSERT(row_pair_smem_ok<T>(smraw, one, ffuse, RB, pl.ldseq));
  auto fetch = [&](T* dst, int row) {  // one thread; RB bytes
    if (pin) {
      for (int q = 0; q < pk.nq; ++q) {
        const bool direct = pk.peers && (pk.own_q < 0 || q == pk.own_q);
        const T* src = direct ? reinterpret_cast<const T*>(pk.peers[q]) + (pk.row0 + row) * pk.mb
                              : in + q * pk.chunk + (long long)row * pk.mb;
        bulk_g2s(dst + q * pk.mb, src, pk.mb * (unsigned)sizeof(T), mbar);
      }
    } else {
      PU_ASSERT(row < g.n && RB <= g.ld * sizeof(T));
      bulk_g2s(dst, in + (long long)row * g.ld, RB, mbar);
    }
  };
  auto issue = [&](int seq) {  // one thread
    const int ia = 2 * seq;
    const bool hb = ia + 1 < g.n;
    if (one) {
      mbar_expect_tx(mbar, RB);
      fetch(sa, ia);
      return;
    }
    mbar_expect_tx(mbar, hb ? 2 * RB : RB);
    fetch(sa, ia);
    if (hb) fetch(sb, ia + 1);
  };
  // stage1: after the row-a pass, fetch row b into the same staging row
  auto issue_b = [&](int ia) {
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_proxy_async();
      mbar_expect_tx(mbar, RB);
      fetch(sa, ia + 1);
    }
    mbar_wait(mbar, ph ^ 1);
    ++waits;
  };
  if (threadIdx.x == 0 && s < S) {
    fence_proxy_async();  // the staging may have been read by the previous pair (persistent loop)
    issue(s);
    if (INV && ffuse && pold != nullptr && !first) {
      // fused K4 reads the old direction from global memory in its output
      // pass: start pulling its two rows into L2 now, behind the FFT
      bulk_prefetch_l2(pold + (long long)(2 * s) * g.ld, RBrow);
      if (2 * s + 1 < g.n) bulk_prefetch_l2(pold + (long long)(2 * s + 1) * g.ld, RBrow);
    }
  }
  const int half = n / 2 + 1;
  if (s < S) {
    cplx<T>* buf = buf0;
    mbar_wait(mbar, ph);
    ++waits;
    const int ia = 2 * s;
    const bool hasb = ia + 1 < g.n;
    if (one) {
      if constexpr (!INV) {
        for (int j0 = 4 * threadIdx.x; j0 < n; j0 += 4 * blockDim.x) {
          const int je = min(j0 + 4, n);
          for (int j = j0; j < je; ++j) buf[spad(mperm(j, n))] = mk<T>(sa[j], (T)0);
        }
        if (hasb) {
          issue_b(ia);
          for (int j0 = 4 * threadIdx.x; j0 < n; j0 += 4 * blockDim.x) {
            const int je = min(j0 + 4, n);
            for (int j = j0; j < je; ++j) buf[spad(mperm(j, n))].y = sa[j];
          }
        }
      } else {
        for (int k = threadIdx.x; k < half; k += blockDim.x) {
          const int nk = k == 0 ? 0 : n - k;
          cplx<T> ck, cnk;
          dct3_pre<T>(sa[k], sa[nk], (T)0, (T)0, k, nk, pl, ck, cnk);
          buf[spad(k)] = ck;
          if (nk != k) buf[spad(nk)] = cnk;
        }
        if (hasb) {
          issue_b(ia);
          for (int k = threadIdx.x; k < half; k += blockDim.x) {
            const int nk = k == 0 ? 0 : n - k;
            cplx<T> ck, cnk;
            dct3_pre<T>((T)0, (T)0, sa[k], sa[nk], k, nk, pl, ck, cnk);
            buf[spad(k)] = cadd<T>(buf[spad(k)], ck);
            if (nk != k) buf[spad(nk)] = cadd<T>(buf[spad(nk)], cnk);
          }
        }
      }
    } else if constexpr (!INV) {
      if (ffuse) {
        if constexpr (FFUSE) rows_first_stage<T, EMAX, LS>(sa, sb, hasb, buf);
      } else {
      // Makhoul permutation + (a + i b) packing
      for (int j0 = 4 * threadIdx.x; j0 < n; j0 += 4 * blockDim.x) {
        if (j0 + 4 <= n) {
          const Q4<T> a = ld4(sa + j0);
          const Q4<T> b = hasb ? ld4(sb + j0) : zero4<T>();
#pragma unroll
          for (int k = 0; k < 4; ++k) buf[spad(mperm(j0 + k, n))] = mk<T>(a.a[k], b.a[k]);
        } else {
          for (int j = j0; j < n; ++j) buf[spad(mperm(j, n))] = mk<T>(sa[j], hasb ? sb[j] : (T)0);
        }
      }
      }
    } else if (ffuse) {
      if constexpr (FFUSE) rows_first_stage_inv<T, EMAX, LS>(sa, sb, hasb, buf, pl);
    } else {
      for (int k = threadIdx.x; k < half; k += blockDim.x) {
        const int nk = k == 0 ? 0 : n - k;
        cplx<T> ck, cnk;
        dct3_pre<T>(sa[k], sa[nk], hasb ? sb[k] : (T)0, hasb ? sb[nk] : (T)0, k, nk, pl, ck, cnk);
        buf[spad(k)] = ck;
        if (nk != k) buf[spad(nk)] = cnk;
      }
    }
    __syncthreads();
    const bool axpy = INV && pold != nullptr && !first;
    if (axpy && !one && !ffuse && threadIdx.x == 0) {
      // staging is free now: fetch the old search direction rows behind the FFT
      fence_proxy_async();
      mbar_expect_tx(mbar, hasb ? 2 * RBrow : RBrow);
      bulk_g2s(sa, pold + (long long)ia * g.ld, RBrow, mbar);
      if (hasb) bulk_g2s(sb, pold + (long long)(ia + 1) * g.ld, RBrow, mbar);
    }
    if (ffuse) {
      if constexpr (FFUSE) fft_stages_range<T, EMAX, LS, first_radix<LS, EMAX>(), 0, LS>(buf, 0, 1, pl.stw);
    } else {
      fft_n<T, EMAX, LS>(buf, 1, pl);
    }
    const long long oa = (long long)ia * g.ld, ob = oa + g.ld;
    if constexpr (!INV) {
      if (pout) {
        // packed: column k of rows ia, ia + 1 -> chunk k / mb (local buffer,
        // or the owning rank's column block)
        auto at = [&](int k) -> T* {
          const int q = (int)pk.mbd.div((unsigned)k);
          T* base = pk.peers ? reinterpret_cast<T*>(__ldg(pk.peers + q)) + (pk.row0 + ia) * pk.mb
                             : out + q * pk.chunk + (long long)ia * pk.mb;
          return base + (k - q * pk.mb);
        };
        for (int k = threadIdx.x; k < half; k += blockDim.x) {
          const int nk = k == 0 ? 0 : n - k;
          const PairOut<T> q = dct2_post<T>(buf[spad(k)], buf[spad(nk)], k, nk, pl);
          T* ok_ = at(k);
          ok_[0] = q.a_k;
          if (hasb) ok_[pk.mb] = q.b_k;
          if (nk != k) {
            T* onk = at(nk);
            onk[0] = q.a_nk;
            if (hasb) onk[pk.mb] = q.b_nk;
          }
        }
      } else {
        for (int k = threadIdx.x; k < half; k += blockDim.x) {
          const int nk = k == 0 ? 0 : n - k;
          const PairOut<T> q = dct2_post<T>(buf[spad(k)], buf[spad(nk)], k, nk, pl);
          out[oa + k] = q.a_k;
          if (hasb) out[ob + k] = q.b_k;
          if (nk != k) {
            out[oa + nk] = q.a_nk;
            if (hasb) out[ob + nk] = q.b_nk;
          }
        }
      }
    } else {
      const int cpr = (n + 3) >> 2;
      const T beta = axpy ? (T)ctrl->beta : (T)0;
      if (axpy && !one && !ffuse) {
        mbar_wait(mbar, ph ^ 1);
        ++waits;
      }
      for (int e = threadIdx.x; e < 2 * cpr; e += blockDim.x) {
        const int rr = e >= cpr, j0 = (e - rr * cpr) * 4;
        if (rr && !hasb) continue;
        Q4<T> o;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = j0 + k;
          if (j < n) {
            const cplx<T> v = buf[spad(mperm(j, n))];
            o.a[k] = rr ? -v.y : v.x;  // 1/n folded into dct3w
          } else {
            o.a[k] = (T)0;
          }
        }
        const long long oo = (rr ? ob : oa) + j0;
        if (axpy) {
          const Q4<T> pp = (one || ffuse) ? ldg4(pold + oo) : ld4((rr ? sb : sa) + j0);
#pragma unroll
          for (int k = 0; k < 4; ++k) o.a[k] = (j0 + k < n) ? add_rn(mul_rn(beta, pp.a[k]), o.a[k]) : (T)0;
        }
        st4(out + oo, o);
      }
    }
  }
  ph ^= (unsigned)(waits & 1);
}

template <typename T, int EMAX, int LS, bool INV>
__global__ void __launch_bounds__(fft_max_threads(LS, EMAX, sizeof(T)), fft_min_blocks(LS, EMAX))
    k_rows_pipe(Grid g, FftPlan<T> pl, const T* __restrict__ in, T* __restrict__ out, const PcgCtrl* ctrl,
                const T* __restrict__ pold, int first, Pack pk) {
  extern __shared__ __align__(128) unsigned char smraw[];
  pdl_enter(g);
  if (ctrl && ctrl->done) return;
  if (threadIdx.x == 0) {
    mbar_init(reinterpret_cast<uint64_t*>(smraw), 1);
    fence_mbar_init();
  }
  __syncthreads();
  unsigned ph = 0;
  rows_pair<T, EMAX, LS, INV>(g, pl, in, out, ctrl, pold, first, pk, (int)blockIdx.x, smraw, ph);
}

}  // namespace pu
