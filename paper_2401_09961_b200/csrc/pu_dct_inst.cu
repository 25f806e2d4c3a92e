// One explicit instantiation of the transform kernels; compiled once per
// (PU_INST_T, PU_INST_LS) pair by build_ext.py.
#define PU_DCT_DEFINE
#include "pu_dct_launch.cuh"

#if !defined(PU_INST_T) || !defined(PU_INST_LS)
#error "compile with -DPU_INST_T=float|double -DPU_INST_LS=<internal FFT length or 0>"
#endif

namespace pu {
template struct DctLaunch<PU_INST_T, PU_INST_LS>;
}
