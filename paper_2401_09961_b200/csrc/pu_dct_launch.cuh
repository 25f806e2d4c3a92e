// Host launch wrappers for the transform kernels, one explicit instantiation
// per (dtype, internal FFT length) in its own translation unit
// (pu_dct_inst.cu compiled with -DPU_INST_T / -DPU_INST_LS) so the
// compile-time FFT plans build in parallel.  LS = 0 is the runtime plan used
// for every other length.
#pragma once

#include <utility>

#include "pu_pipe.cuh"

namespace pu {

struct XLaunch {
  int grid;
  int threads;
  size_t smem;
  cudaStream_t st;
  bool pdl = false;  // programmatic dependent launch (Grid::pdl)
};

// <<<grid, block, smem, st>>>, or with the programmatic-stream-serialization
// attribute: the kernel may be scheduled while the previous one in the stream
// drains, and waits for it in griddepcontrol.wait (pdl_enter)
template <typename... P, typename... A>
cudaError_t launch_k(void (*kernel)(P...), int grid, int block, size_t smem, cudaStream_t st, bool pdl, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

template <typename T, int LS>
struct DctLaunch {
  static constexpr int EM = emax_of<T>();

  static cudaError_t set_attrs(size_t row_smem, size_t col_smem);

  // pipelined persistent row transforms (pu_pipe.cuh); grid from occupancy
  static cudaError_t rows_pipe(bool inv, const XLaunch& c, const Grid& g, const FftPlan<T>& pl, const T* in, T* out,
                               const PcgCtrl* ctrl, const T* pold, int first, Pack pk);
  static int rows_pipe_blocks_per_sm(int threads, size_t smem);
  static int cols_blocks_per_sm(int threads, size_t smem);
  // row kernels of a static plan: FFT buffer aliases the staging rows
  static bool rows_fused(const FftPlan<T>& pl);
  static cudaError_t cols(int mode, const XLaunch& c, const Grid& g, const FftPlan<T>& pl, const T* lam_cols,
                          int cpc, T* data, PcgCtrl* ctrl, RedScratch rs, int site, int it, Push ps, int nfull);
};

#ifdef PU_DCT_DEFINE
template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::set_attrs(size_t row_smem, size_t col_smem) {
  cudaError_t e;
#define PU_ATTR(K, S) \
  if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(S))) != cudaSuccess) return e;
  PU_ATTR((k_rows_pipe<T, EM, LS, false>), row_smem);
  PU_ATTR((k_rows_pipe<T, EM, LS, true>), row_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_API>), col_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_INIT>), col_smem);
  PU_ATTR((k_cols_spec<T, EM, LS, MODE_ITER>), col_smem);
#undef PU_ATTR
  return cudaSuccess;
}

template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::rows_pipe(bool inv, const XLaunch& c, const Grid& g, const FftPlan<T>& pl, const T* in,
                                        T* out, const PcgCtrl* ctrl, const T* pold, int first, Pack pk) {
  const size_t smem = rows_fused(pl) ? rows_fused_smem(c.smem, sizeof(T), pl.ldseq) : c.smem;
  const PcgCtrl* cc = ctrl;
  const T* po = inv ? pold : nullptr;
  const int fi = inv ? first : 0;
  if (inv) return launch_k(k_rows_pipe<T, EM, LS, true>, c.grid, c.threads, smem, c.st, c.pdl, g, pl, in, out, cc, po, fi, pk);
  return launch_k(k_rows_pipe<T, EM, LS, false>, c.grid, c.threads, smem, c.st, c.pdl, g, pl, in, out, cc, po, fi, pk);
}

template <typename T, int LS>
int DctLaunch<T, LS>::cols_blocks_per_sm(int threads, size_t smem) {
  int a = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_cols_spec<T, EM, LS, MODE_ITER>, threads, smem);
  return a;
}

template <typename T, int LS>
bool DctLaunch<T, LS>::rows_fused(const FftPlan<T>& pl) {
  if constexpr (LS > 0) return rows_fused_ok<LS, EM>() && !pl.stage1;
  return false;
}

template <typename T, int LS>
int DctLaunch<T, LS>::rows_pipe_blocks_per_sm(int threads, size_t smem) {
  int a = 0, b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_rows_pipe<T, EM, LS, false>, threads, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_rows_pipe<T, EM, LS, true>, threads, smem);
  return std::max(1, std::min(a, b));
}

template <typename T, int LS>
cudaError_t DctLaunch<T, LS>::cols(int mode, const XLaunch& c, const Grid& g, const FftPlan<T>& pl,
                                   const T* lam_cols, int cpc, T* data, PcgCtrl* ctrl, RedScratch rs, int site,
                                   int it, Push ps, int nfull) {
  if (mode == MODE_API)
    k_cols_spec<T, EM, LS, MODE_API><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, lam_cols, cpc, data, ctrl, rs, site, it, ps, nfull);
  else if (mode == MODE_INIT)
    k_cols_spec<T, EM, LS, MODE_INIT><<<c.grid, c.threads, c.smem, c.st>>>(g, pl, lam_cols, cpc, data, ctrl, rs, site, it, ps, nfull);
  else
    return launch_k(k_cols_spec<T, EM, LS, MODE_ITER>, c.grid, c.threads, c.smem, c.st, c.pdl, g, pl, lam_cols, cpc,
                    data, ctrl, rs, site, it, ps, nfull);
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
