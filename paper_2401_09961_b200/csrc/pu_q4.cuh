// 4-element vector helpers shared by the element-wise and transform kernels.
#pragma once

#include "pu_common.cuh"

// fp64 4-cell chunks as one 32-byte access (LDG/STG.E.ENL2.256 on sm_100)
// instead of two 16-byte ones: half the load/store instructions of the
// element-wise kernels.  Global memory only (shared memory keeps ld4).
#ifndef PU_F64_V256
#define PU_F64_V256 1
#endif

namespace pu {

template <typename T>
struct Q4 {
  T a[4];
};

struct __align__(32) D4x32 {
  double x, y, z, w;
};

__device__ __forceinline__ Q4<float> ld4(const float* p) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  return Q4<float>{{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ Q4<double> ld4(const double* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  return Q4<double>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ Q4<float> ldg4(const float* p) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  return Q4<float>{{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ Q4<double> ldg4(const double* p) {
#if PU_F64_V256
  const D4x32 v = *reinterpret_cast<const D4x32*>(p);
  return Q4<double>{{v.x, v.y, v.z, v.w}};
#else
  const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Q4<double>{{a.x, a.y, b.x, b.y}};
#endif
}
// global loads of planes the kernel also writes (no read-only path)
__device__ __forceinline__ Q4<float> ldx4(const float* p) { return ld4(p); }
__device__ __forceinline__ Q4<double> ldx4(const double* p) { return ld4(p); }
__device__ __forceinline__ void st4(float* p, const Q4<float>& q) {
  *reinterpret_cast<float4*>(p) = make_float4(q.a[0], q.a[1], q.a[2], q.a[3]);
}
__device__ __forceinline__ void st4(double* p, const Q4<double>& q) {
#if PU_F64_V256
  *reinterpret_cast<D4x32*>(p) = D4x32{q.a[0], q.a[1], q.a[2], q.a[3]};
#else
  reinterpret_cast<double2*>(p)[0] = make_double2(q.a[0], q.a[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(q.a[2], q.a[3]);
#endif
}
template <typename T>
__device__ __forceinline__ Q4<T> zero4() {
  return Q4<T>{{(T)0, (T)0, (T)0, (T)0}};
}
template <typename T>
__device__ __forceinline__ Q4<T> ones4() {
  return Q4<T>{{(T)1, (T)1, (T)1, (T)1}};
}

}  // namespace pu
