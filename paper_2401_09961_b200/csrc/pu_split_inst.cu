// One explicit instantiation of the cluster-split transforms (pu_split.cuh);
// compiled once per (PU_INST_T, PU_INST_LH) pair by build_ext.py.
#define PU_SPLIT_DEFINE
#include "pu_split.cuh"

#if !defined(PU_INST_T) || !defined(PU_INST_LH)
#error "compile with -DPU_INST_T=float|double -DPU_INST_LH=<half length>"
#endif

namespace pu {
template struct SplitLaunch<PU_INST_T, PU_INST_LH>;
}
