// GPU synthetic scene generation (reference
// synth.py:43-109), for large benchmark inputs (C4 16384²: ~60 s on the
// host generator).  The scene recipe is the reference's: the bump and seam
// parameters are drawn on the host from the reference's Philox stream
// (paper_2401_09961_b200/synth_gpu.py), the per-pixel work runs here.
//
// What is and is not bit-identical to the host generator:
//  - plateau-discontinuity, the tapered fault mask and wrap_to_principal:
//    exact (integer compares, exact products, the reference's rounding
//    sequence);
//  - gaussian-bumps: sum over bumps in the reference's order of
//    peak * exp(-d2 / (2 w^2)), with CUDA's exp (<= 1 ulp, like the host
//    libm): agrees to ~1e-15 relative, not bitwise;
//  - phase noise: a counter-based Philox-4x32-10 stream with Box-Muller
//    normals on the device, statistically equivalent to numpy's ziggurat
//    normals but a different realisation.
// The parity tests therefore keep the host generator (sha256-pinned to the
// reference); this path is for throughput runs.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace pu {
int fail_ext(int code, const char* msg);
}

namespace {

const double kTwoPi = 6.283185307179586;

// bumps: params[4 b + {0,1,2,3}] = r0, c0, width, peak (synth.py:57-66)
__global__ void k_bumps(double* out, int rows, int cols, long long ld, const double* __restrict__ params, int count) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e - (long long)i * cols);
    const double rr = (double)i, cc = (double)j;
    double acc = 0.0;
    for (int b = 0; b < count; ++b) {
      const double r0 = params[4 * b], c0 = params[4 * b + 1], w = params[4 * b + 2], pk = params[4 * b + 3];
      const double dr = __dsub_rn(rr, r0), dc = __dsub_rn(cc, c0);
      const double d2 = __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dc, dc));
      const double den = __dmul_rn(2.0, __dmul_rn(w, w));
      acc = __dadd_rn(acc, __dmul_rn(pk, exp(__ddiv_rn(-d2, den))));
    }
    out[(long long)i * ld + j] = acc;
  }
}

// out += lin[i] * amplitude * (j >= seam[i])   (synth.py plateau + the tapered fault of SURVEY Appendix B)
__global__ void k_fault(double* out, int rows, int cols, long long ld, const long long* __restrict__ seam,
                        const double* __restrict__ lin, double amplitude) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e - (long long)i * cols);
    const double mask = (long long)j >= seam[i] ? amplitude : 0.0;
    out[(long long)i * ld + j] = __dadd_rn(out[(long long)i * ld + j], __dmul_rn(lin[i], mask));
  }
}

__device__ __forceinline__ double wrap0(double a) {  // phase.py:118-137 with lo = 0
  double y = __dsub_rn(a, __dmul_rn(kTwoPi, floor(__ddiv_rn(a, kTwoPi))));
  if (y >= kTwoPi) y = __dsub_rn(y, kTwoPi);
  if (y < 0.0) y = __dadd_rn(y, kTwoPi);
  return y;
}

// Philox-4x32-10 (Salmon et al. 2011), counter = (pixel pair index, 0), key = seed
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x, p1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((unsigned)(p1 >> 32) ^ c.y ^ k.x, (unsigned)p1, (unsigned)(p0 >> 32) ^ c.w ^ k.y, (unsigned)p0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// x = wrap0(x + sigma * N(0, 1)) (synth.py:101-109 semantics; device normals)
__global__ void k_noise_wrap(double* x, int rows, int cols, long long ld, double sigma, unsigned long long seed) {
  const uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  const long long npix = (long long)rows * cols;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; 2 * q < npix;
       q += (long long)gridDim.x * blockDim.x) {
    const uint4 r = philox(make_uint4((unsigned)q, (unsigned)(q >> 32), 0u, 0u), key);
    // two 53-bit uniforms in (0, 1], Box-Muller
    const double u1 = ((double)(((unsigned long long)r.x << 21) ^ (r.y >> 11)) + 1.0) * 0x1.0p-53;
    const double u2 = ((double)(((unsigned long long)r.z << 21) ^ (r.w >> 11)) + 0.5) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double s, c;
    sincospi(2.0 * u2, &s, &c);
    const double z[2] = {rad * c, rad * s};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long e = 2 * q + h;
      if (e >= npix) break;
      const int i = (int)(e / cols), j = (int)(e - (long long)i * cols);
      double* p = x + (long long)i * ld + j;
      *p = wrap0(__dadd_rn(*p, __dmul_rn(sigma, z[h])));
    }
  }
}

__global__ void k_wrap(double* x, int rows, int cols, long long ld) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e - (long long)i * cols);
    x[(long long)i * ld + j] = wrap0(x[(long long)i * ld + j]);
  }
}

int grid_for(long long n) { return (int)std::min<long long>((n + 255) / 256, 148LL * 16); }

int check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  return pu::fail_ext(2, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
}

}  // namespace

extern "C" {

int pu_synth_bumps(double* out, int rows, int cols, int64_t ld, const double* params, int count, void* stream) {
  if (!out || rows < 1 || cols < 1 || ld < cols || count < 0 || (count > 0 && !params))
    return pu::fail_ext(1, "pu_synth_bumps: invalid arguments");
  k_bumps<<<grid_for((long long)rows * cols), 256, 0, (cudaStream_t)stream>>>(out, rows, cols, ld, params, count);
  return check(cudaGetLastError(), "pu_synth_bumps");
}

int pu_synth_fault(double* out, int rows, int cols, int64_t ld, const int64_t* seam, const double* lin,
                   double amplitude, void* stream) {
  if (!out || !seam || !lin || rows < 1 || cols < 1 || ld < cols) return pu::fail_ext(1, "pu_synth_fault: invalid arguments");
  k_fault<<<grid_for((long long)rows * cols), 256, 0, (cudaStream_t)stream>>>(
      out, rows, cols, ld, reinterpret_cast<const long long*>(seam), lin, amplitude);
  return check(cudaGetLastError(), "pu_synth_fault");
}

int pu_synth_wrap_noise(double* x, int rows, int cols, int64_t ld, double sigma, uint64_t seed, void* stream) {
  if (!x || rows < 1 || cols < 1 || ld < cols || !(sigma >= 0)) return pu::fail_ext(1, "pu_synth_wrap_noise: invalid arguments");
  const long long n = (long long)rows * cols;
  if (sigma == 0)
    k_wrap<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(x, rows, cols, ld);
  else
    k_noise_wrap<<<grid_for((n + 1) / 2), 256, 0, (cudaStream_t)stream>>>(x, rows, cols, ld, sigma,
                                                                          (unsigned long long)seed);
  return check(cudaGetLastError(), "pu_synth_wrap_noise");
}

}  // extern "C"
