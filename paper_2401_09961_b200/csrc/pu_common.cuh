// Common device-side definitions for the B200 phase unwrapper.
//
// Memory layout: every grid-shaped array is an N x M
// row-major plane with row pitch `ld` (elements, multiple of 8).  A system
// vector (reference SystemVector, operators.py:39-101) is three consecutive
// planes [u | vv | vh]; vv keeps a zero last row, vh a zero last column, and
// pitch padding is zero, so BLAS-1 reductions may run over whole planes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pu_unwrap.h"
#ifdef PU_DEBUG_CHECKS
#include <cstdio>
#endif

namespace pu {

// ---------------------------------------------------------------------------
// Debug build checks (-DPU_DEBUG_CHECKS, build_ext PU_BUILD_DEFS): device
// asserts on shared-memory addresses (inside the CTA's allocation, read from
// %total_smem_size) and on the global indices of the transform and reduction
// kernels.  compute-sanitizer is closed on the GPU pool of this project, so
// the GPU test suite runs once against this build instead.
// Compiled out of the production library.
// ---------------------------------------------------------------------------
#ifdef PU_DEBUG_CHECKS
// trap (no printf: a printf per inlined site multiplied the compile time)
#define PU_ASSERT(c)     \
  do {                   \
    if (!(c)) __trap();  \
  } while (0)
// a dynamic-shared-memory address [p, p + 1) lies inside this CTA's
// dynamic allocation (base of the extern array .. + %dynamic_smem_size)
template <typename P>
__device__ __forceinline__ P* sm_chk(P* p) {
  extern __shared__ __align__(16) unsigned char pu_dyn_smem_[];
  unsigned dyn;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const unsigned base = (unsigned)__cvta_generic_to_shared(pu_dyn_smem_);
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  if (a < base || a + sizeof(P) > base + dyn) __trap();
  return p;
}
#else
#define PU_ASSERT(c) ((void)0)
template <typename P>
__device__ __forceinline__ P* sm_chk(P* p) { return p; }
#endif

// q = n / d for 0 <= n < 2^31 by a multiply-high and a shift (round-up
// reciprocal, Granlund & Montgomery 1994): the band kernels divide column and
// row indices by runtime block sizes once per element
struct FastDiv {
  unsigned d = 1, mul = 0, shr = 0;
  FastDiv() = default;
  __host__ explicit FastDiv(unsigned divisor) : d(divisor < 1 ? 1 : divisor) {
    if (d == 1) return;
    unsigned l = 0;
    while ((1u << l) < d) ++l;  // ceil(log2 d)
    const unsigned p = 31 + l;
    mul = (unsigned)(((1ull << p) + d - 1) / d);
    shr = p - 32;
  }
  __host__ __device__ __forceinline__ unsigned div(unsigned n) const {
#ifdef __CUDA_ARCH__
    return d == 1 ? n : __umulhi(n, mul) >> shr;
#else
    return d == 1 ? n : (unsigned)(((unsigned long long)n * mul) >> 32) >> shr;
#endif
  }
};

struct Grid {
  int n;            // rows (N)
  int m;            // cols (M)
  long long ld;     // row pitch in elements
  long long plane;  // n * ld
  double tau;
  double inv_tau;
  double delta;
  // row band of a row-sharded grid (pu_create_band): rows [row0, row0 + n) of
  // n_glob; `top`/`bot` = a neighbour band's row is mirrored in the ghost row
  // -1 / n of every plane.  Single-GPU grids: n_glob = n, top = bot = 0.
  int n_glob;
  int top;
  int bot;
  // largest ||r||^2 for which the preconditioned product r.z of the PCG tail
  // is provably finite in T (see fin_k2); set by the host
  double tail_rn2_max;
  // programmatic dependent launch of the PCG-iteration kernels (PU_PDL):
  // 0 off, 1 wait at entry, 2 wait at entry + trigger the next launch before
  // the kernel's tail (reduction / final stores)
  int pdl;
};

// griddepcontrol: no-ops unless the kernel was launched with the
// programmatic-stream-serialization attribute
__device__ __forceinline__ void pdl_enter(const Grid& g) {
  if (g.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger(const Grid& g) {
  if (g.pdl == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// vertical neighbours of row i within the global grid (ghost rows count)
__host__ __device__ __forceinline__ bool dn_ok(const Grid& g, int i) { return i < g.n - 1 || g.bot; }
__host__ __device__ __forceinline__ bool up_ok(const Grid& g, int i) { return i > 0 || g.top; }

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };
template <typename T> using cplx = typename Vec2<T>::type;

template <typename T> __device__ __forceinline__ cplx<T> mk(T x, T y) { cplx<T> c; c.x = x; c.y = y; return c; }
template <typename T> __device__ __forceinline__ cplx<T> cadd(cplx<T> a, cplx<T> b) { return mk<T>(a.x + b.x, a.y + b.y); }
template <typename T> __device__ __forceinline__ cplx<T> csub(cplx<T> a, cplx<T> b) { return mk<T>(a.x - b.x, a.y - b.y); }
template <typename T> __device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename T> __device__ __forceinline__ cplx<T> cconj(cplx<T> a) { return mk<T>(a.x, -a.y); }

// ---------------------------------------------------------------------------
// PCG device control block (one per solve, lives in device memory).
// Mirrors the scalar state of pcg_solve (pcg.py:47-116): every kernel of the
// iteration first reads `done` and returns early once the loop has ended, so
// the host can enqueue a whole budget without synchronising.
// ---------------------------------------------------------------------------
using PcgCtrl = pu_pcg_ctrl;  // layout shared with the C ABI (include/pu_unwrap.h)

// Deterministic two-level reduction: each block writes its partial sums to
// `partials[s * stride + blockIdx.x]`; the last block to arrive (atomic
// ticket) reduces them in a fixed order and runs the finaliser.  The result
// therefore does not depend on block scheduling.
struct RedScratch {
  double* partials;       // [PU_MAX_SUMS][stride]
  unsigned int* ticket;   // one counter per reduction site
  int stride;             // >= max gridDim.x of any reducing kernel
  double* dist;           // band mode: [S_NSITES][PU_MAX_SUMS] band totals (pu_fin.cuh), else null
};

#define PU_MAX_SUMS 12
#define PU_RED_THREADS_MAX 1024

template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS], double* sh /* [NS][32] */) {
  // warp shuffle, then one warp over the per-warp results
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_xor_sync(0xffffffffu, v[s], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) sh[s * 32 + warp] = v[s];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double t = lane < nw ? sh[s * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[s] = t;  // valid in warp 0
    }
  }
  __syncthreads();
}

// Returns true in exactly one warp of one block (warp 0 of the last block to
// finish); there every lane holds `tot[s]` = the grid-wide sums.  Only warp 0
// of each block waits: the other warps leave their warp sums in shared memory,
// signal with a non-blocking bar.arrive on named barrier 1 and exit, so the
// tail of the block costs no CTA-wide barrier (K3 spent ~14% of its stall
// samples in the old two-__syncthreads block sum).  Every order is fixed
// (xor butterflies, warp index, block index), so the result does not depend
// on scheduling.  All warps of the block must call it (no early exits).
template <int NS>
__device__ __forceinline__ bool grid_reduce(double (&v)[NS], RedScratch rs, int site, double (&tot)[NS]) {
  __shared__ double sh[NS * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_xor_sync(0xffffffffu, v[s], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) sh[s * 32 + warp] = v[s];
  }
  if (warp != 0) {
    asm volatile("bar.arrive 1, %0;" ::"r"(nw * 32) : "memory");
    return false;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double t = lane < nw ? sh[s * 32 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[s] = t;
  }
  unsigned int ticket = 0;
  PU_ASSERT((int)blockIdx.x < rs.stride && site >= 0 && site < 32);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) rs.partials[(size_t)s * rs.stride + blockIdx.x] = v[s];
    __threadfence();
    ticket = atomicAdd(rs.ticket + site, 1u);
  }
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != gridDim.x - 1) return false;
  __threadfence();
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double acc = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) acc += ((volatile double*)rs.partials)[(size_t)s * rs.stride + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    tot[s] = acc;
  }
  if (lane == 0) rs.ticket[site] = 0u;  // re-arm for the next launch
  return true;
}

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

}  // namespace pu
