// Host launch wrappers for the transform kernels, one explicit instantiation
// per (dtype, internal FFT length) in its own translation unit
// (pu_dct_inst.cu compiled with -DPU_INST_T / -DPU_INST_LS) so the
// compile-time FFT plans build in parallel.  LS = 0 is the runtime plan used
// for every other length.
#pragma once

#include "pu_pcg.cuh"

namespace pu {

struct XLaunch {
  int grid;
  int threads;
  size_t smem;
  cudaStream_t st;
};

template <typename T, int LS>
struct DctLaunch {
  static constexpr int EM = sizeof(T) == 4 ? 16 : 8;

  static cudaError_t set_attrs(size_t row_smem, size_t col_smem);

  static cudaError_t rows_plain(const XLaunch& c, const Grid& g, const FftPlan<T>& pl, int rpc, const T* src, T* out,
                                const PcgCtrl* ctrl, RedScratch rs, int site);
  static cudaError_t rows_inv(const XLaunch& c, const Grid& g, const FftPlan<T>& pl, int rpc, const T* in, T* out,
                              const PcgCtrl* ctrl);
  static cudaError_t cols(int mode, const XLaunch& c, const Grid& g, const FftPlan<T>& pl, const T* lam_cols,
                          int cpc, T* data, PcgCtrl* ctrl, RedScratch rs, int site, int it);
};

#ifdef PU_DCT_DEFINE
template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::set_attrs(size_t row_smem, size_t col_smem) {
  cudaError_t e;
#define PU_ATTR(K, S) \
  if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(S))) != cudaSuccess) return e;
  PU_ATTR((k_rows_fwd<T, EM, LS, RowsPlain<T>>), row_smem);
  PU_ATTR((k_rows_inv<T, EM, LS>), row_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_API>), col_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_INIT>), col_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_ITER>), col_smem);
#undef PU_ATTR
  return cudaSuccess;
}

template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::rows_plain(const XLaunch& c, const Grid& g, const FftPlan<T>& pl, int rpc,
                                         const T* src, T* out, const PcgCtrl* ctrl, RedScratch rs, int site) {
  RowsPlain<T> pol{src, ctrl};
  k_rows_fwd<T, EM, LS, RowsPlain<T>><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, rpc, out, pol, rs, site);
  return cudaGetLastError();
}

template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::rows_inv(const XLaunch& c, const Grid& g, const FftPlan<T>& pl, int rpc, const T* in,
                                       T* out, const PcgCtrl* ctrl) {
  k_rows_inv<T, EM, LS><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, rpc, in, out, ctrl);
  return cudaGetLastError();
}

template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::cols(int mode, const XLaunch& c, const Grid& g, const FftPlan<T>& pl,
                                   const T* lam_cols, int cpc, T* data, PcgCtrl* ctrl, RedScratch rs, int site,
                                   int it) {
  if (mode == MODE_API)
    k_cols_spec<T, EM, LS, MODE_API><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, lam_cols, cpc, data, ctrl, rs, site, it);
  else if (mode == MODE_INIT)
    k_cols_spec<T, EM, LS, MODE_INIT><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, lam_cols, cpc, data, ctrl, rs, site, it);
  else
    k_cols_spec<T, EM, LS, MODE_ITER><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, lam_cols, cpc, data, ctrl, rs, site, it);
  return cudaGetLastError();
}
#endif  // PU_DCT_DEFINE

// Static internal lengths with their own instantiation (see build_ext.py).
#define PU_STATIC_LS_F32(X) X(float, 512) X(float, 1024) X(float, 2048) X(float, 4096) X(float, 8192) X(float, 16384)
#define PU_STATIC_LS_F64(X) X(double, 512) X(double, 1024) X(double, 2048) X(double, 4096) X(double, 8192)

#define PU_EXTERN_DCT(T, LS) extern template struct DctLaunch<T, LS>;
PU_EXTERN_DCT(float, 0)
PU_EXTERN_DCT(double, 0)
PU_STATIC_LS_F32(PU_EXTERN_DCT)
PU_STATIC_LS_F64(PU_EXTERN_DCT)

}  // namespace pu
