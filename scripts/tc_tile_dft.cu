// Tensor-core tile-DFT experiment (north_star: "tensor cores used only if a
// dense DCT-matrix contraction is shown by ncu to win at the tile size").
//
// The preconditioner's column transform at 4096 points splits as 64 x 64
// (four-step); its inner work is a batch of 64-point complex DFTs.  This
// program times that stage both ways on the C3 volume (4096 x 4096 complex
// values = 262144 vectors of 64 points) and checks accuracy:
//
//   fp64  k_dft64_fft<double>  radix-8 x 8 FFT, 8 threads per vector, one
//                               shared-memory exchange (the production scheme)
//         k_dft64_dmma          dense 64 x 64 complex DFT matrix on the FP64
//                               tensor cores: mma.sync.m8n8k4.f64 (DMMA; the
//                               fp64 tensor path of sm_100 -- tcgen05 has no
//                               f64 kind), Y = [Fr -Fi; Fi Fr] [Xr; Xi]
//   fp32  k_dft64_fft<float>   as above
//         k_dft64_tf32x3        the same contraction on TF32 tensor cores,
//                               3xTF32 split (hi*hi + hi*lo + lo*hi) for
//                               fp32-level accuracy, mma.sync.m16n8k8.tf32
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        scripts/tc_tile_dft.cu -o scripts/tc_tile_dft && scripts/tc_tile_dft
//
// Prints one JSON line per kernel: ms per stage, achieved flop/s, bytes/s,
// max relative error against an fp64 host DFT on sampled vectors.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

// ---------------------------------------------------------------------------
// FFT path: 64 = 8 x 8.  Thread (vector v, lane r in 0..7) loads x[r + 8 s],
// s = 0..7 (stride 8), runs a radix-8 DFT, twiddles by W64^(r k1), exchanges
// through shared memory, and runs the second radix-8 on x'[8 r .. 8 r + 7].
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void dft8(typename C2<T>::t* a) {
  using C = typename C2<T>::t;
  const T h = (T)0.70710678118654752440;
  // radix-2 x 4 (DIT over even/odd)
  C e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
  auto dft4 = [](C* b) {
    C s0 = {b[0].x + b[2].x, b[0].y + b[2].y}, d0 = {b[0].x - b[2].x, b[0].y - b[2].y};
    C s1 = {b[1].x + b[3].x, b[1].y + b[3].y}, d1 = {b[1].y - b[3].y, -(b[1].x - b[3].x)};
    b[0] = {s0.x + s1.x, s0.y + s1.y};
    b[2] = {s0.x - s1.x, s0.y - s1.y};
    b[1] = {d0.x + d1.x, d0.y + d1.y};
    b[3] = {d0.x - d1.x, d0.y - d1.y};
  };
  dft4(e);
  dft4(o);
  C t1 = {h * (o[1].x + o[1].y), h * (o[1].y - o[1].x)};   // W8^1
  C t2 = {o[2].y, -o[2].x};                                 // W8^2 = -i
  C t3 = {h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)};  // W8^3
  a[0] = {e[0].x + o[0].x, e[0].y + o[0].y}; a[4] = {e[0].x - o[0].x, e[0].y - o[0].y};
  a[1] = {e[1].x + t1.x, e[1].y + t1.y};     a[5] = {e[1].x - t1.x, e[1].y - t1.y};
  a[2] = {e[2].x + t2.x, e[2].y + t2.y};     a[6] = {e[2].x - t2.x, e[2].y - t2.y};
  a[3] = {e[3].x + t3.x, e[3].y + t3.y};     a[7] = {e[3].x - t3.x, e[3].y - t3.y};
}

template <typename T>
__global__ void __launch_bounds__(256) k_dft64_fft(const typename C2<T>::t* __restrict__ x,
                                                   typename C2<T>::t* __restrict__ y, const typename C2<T>::t* tw,
                                                   int nvec) {
  using C = typename C2<T>::t;
  __shared__ C sm[32][65];  // 32 vectors per CTA, padded
  const int lv = threadIdx.x >> 3, r = threadIdx.x & 7;
  const long long v = (long long)blockIdx.x * 32 + lv;
  if (v >= nvec) return;
  const C* xv = x + v * 64;
  C a[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) a[s] = xv[r + 8 * s];
  dft8<T>(a);  // a[k1] = sum_s x[r + 8 s] W8^(s k1)
#pragma unroll
  for (int k1 = 1; k1 < 8; ++k1) {
    const C w = tw[r * k1];
    a[k1] = C{a[k1].x * w.x - a[k1].y * w.y, a[k1].x * w.y + a[k1].y * w.x};
  }
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) sm[lv][r + 8 * k1] = a[k1];  // [k1][r]
  __syncwarp();
  C b[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) b[s] = sm[lv][8 * r + s];  // k1 = r, over s = r'
  dft8<T>(b);  // X[k1 + 8 k2] = b[k2]
  C* yv = y + v * 64;
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) yv[r + 8 * k2] = b[k2];
}

// ---------------------------------------------------------------------------
// FP64 tensor path: one CTA = 64 vectors.  Real form: [Yr; Yi] (128 x 64) =
// A (128 x 128) B (128 x 64), A = [Fr -Fi; Fi Fr], B = [Xr; Xi] (k = 2 i + c
// interleaved so that B loads straight from the complex input).  8 warps,
// each a 16 x 64 output slab (2 x 8 tiles of m8n8), K in steps of 4.
// Fragment layouts (PTX ISA, mma.m8n8k4.f64): A row g = lane / 4, col
// t = lane % 4; B row t, col g; C rows g, cols 2 t, 2 t + 1.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) k_dft64_dmma(const double2* __restrict__ x, double2* __restrict__ y,
                                                       const double* __restrict__ Aglob, int nvec) {
  // persistent: the 128 x 128 matrix is staged once per CTA, vector tiles loop
  extern __shared__ __align__(16) double smd[];
  constexpr int SA = 132, SB = 68;  // strides = 4 (mod 16) doubles: conflict-free fragment loads
  double* As = smd;                 // 128 x SA
  double* Bs = smd + 128 * SA;      // 128 x SB (k x n)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int e = tid; e < 128 * 128; e += 256) As[(e >> 7) * SA + (e & 127)] = Aglob[e];
  const int ntiles = (nvec + 63) / 64;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long v0 = (long long)tile * 64;
    __syncthreads();
    for (int e = tid; e < 64 * 64; e += 256) {
      const int n = e >> 6, i = e & 63;
      const double2 xv = (v0 + n < nvec) ? x[(v0 + n) * 64 + i] : double2{0.0, 0.0};
      Bs[(2 * i) * SB + n] = xv.x;
      Bs[(2 * i + 1) * SB + n] = xv.y;
    }
    __syncthreads();
    double acc[2][8][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int m0 = warp * 16;
#pragma unroll 4
    for (int k0 = 0; k0 < 128; k0 += 4) {
      double af[2], bf[8];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = As[(m0 + 8 * a + g) * SA + k0 + t];
#pragma unroll
      for (int b = 0; b < 8; ++b) bf[b] = Bs[(k0 + t) * SB + 8 * b + g];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                       : "d"(af[a]), "d"(bf[b]));
    }
    // rows m < 64: Yr[m]; m >= 64: Yi[m - 64]
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int m = m0 + 8 * a + g;
      const bool im = m >= 64;
      const int kk = im ? m - 64 : m;
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const long long n = v0 + 8 * b + 2 * t + c;
          if (n < nvec) reinterpret_cast<double*>(y + n * 64 + kk)[im ? 1 : 0] = acc[a][b][c];
        }
    }
  }
}

// ---------------------------------------------------------------------------
// FP32 tensor path, 3xTF32: A = Ah + Al, B = Bh + Bl (each TF32), D = Ah Bh +
// Ah Bl + Al Bh.  mma.m16n8k8 tf32 layouts: A a0 (g, t), a1 (g+8, t), a2
// (g, t+4), a3 (g+8, t+4); B b0 (t, g), b1 (t+4, g); C c0 (g, 2t), c1 (g, 2t+1),
// c2 (g+8, 2t), c3 (g+8, 2t+1).  8 warps x 16 rows; 8 n-tiles of 8 = 64 vectors.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned tf32(float f) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return r;
}

__global__ void __launch_bounds__(256, 1) k_dft64_tf32x3(const float2* __restrict__ x, float2* __restrict__ y,
                                                         const float* __restrict__ Aglob, int nvec) {
  extern __shared__ __align__(16) float smf[];
  constexpr int SA = 132, SB = 72;  // conflict-free fragment loads for 4-byte elements
  float* As = smf;                  // 128 x SA
  float* Bs = smf + 128 * SA;       // 128 x SB
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int e = tid; e < 128 * 128; e += 256) As[(e >> 7) * SA + (e & 127)] = Aglob[e];
  const int ntiles = (nvec + 63) / 64;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long v0 = (long long)tile * 64;
    __syncthreads();
    for (int e = tid; e < 64 * 64; e += 256) {
      const int n = e >> 6, i = e & 63;
      const float2 xv = (v0 + n < nvec) ? x[(v0 + n) * 64 + i] : float2{0.f, 0.f};
      Bs[(2 * i) * SB + n] = xv.x;
      Bs[(2 * i + 1) * SB + n] = xv.y;
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[b][0] = acc[b][1] = acc[b][2] = acc[b][3] = 0.f;
    const int m0 = warp * 16;
#pragma unroll 2
    for (int k0 = 0; k0 < 128; k0 += 8) {
      const float a_[4] = {As[(m0 + g) * SA + k0 + t], As[(m0 + g + 8) * SA + k0 + t],
                           As[(m0 + g) * SA + k0 + t + 4], As[(m0 + g + 8) * SA + k0 + t + 4]};
      unsigned ah[4], al[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ah[q] = tf32(a_[q]);
        al[q] = tf32(a_[q] - __uint_as_float(ah[q]));
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const float b0 = Bs[(k0 + t) * SB + 8 * b + g], b1 = Bs[(k0 + t + 4) * SB + 8 * b + g];
        const unsigned bh0 = tf32(b0), bh1 = tf32(b1);
        const unsigned bl0 = tf32(b0 - __uint_as_float(bh0)), bl1 = tf32(b1 - __uint_as_float(bh1));
#define PU_MMA_TF32(A0, A1, A2, A3, B0, B1)                                                             \
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, " \
               "{%0,%1,%2,%3};"                                                                        \
               : "+f"(acc[b][0]), "+f"(acc[b][1]), "+f"(acc[b][2]), "+f"(acc[b][3])                    \
               : "r"(A0), "r"(A1), "r"(A2), "r"(A3), "r"(B0), "r"(B1))
        PU_MMA_TF32(al[0], al[1], al[2], al[3], bh0, bh1);
        PU_MMA_TF32(ah[0], ah[1], ah[2], ah[3], bl0, bl1);
        PU_MMA_TF32(ah[0], ah[1], ah[2], ah[3], bh0, bh1);
#undef PU_MMA_TF32
      }
    }
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int m = m0 + g + (c >= 2 ? 8 : 0);
        const long long n = v0 + 8 * b + 2 * t + (c & 1);
        const bool im = m >= 64;
        const int kk = im ? m - 64 : m;
        if (n < nvec) reinterpret_cast<float*>(y + n * 64 + kk)[im ? 1 : 0] = acc[b][c];
      }
  }
}

// ---------------------------------------------------------------------------
template <typename T>
static std::vector<T> dft_matrix_real() {  // [Fr -Fi; Fi Fr] with k interleaved (2 i + c)
  std::vector<T> A(128 * 128);
  for (int k = 0; k < 64; ++k)
    for (int i = 0; i < 64; ++i) {
      const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)((k * i) % 64) / 64.0L;
      const T fr = (T)cosl(ang), fi = (T)sinl(ang);
      A[k * 128 + 2 * i] = fr;             // Yr += Fr Xr
      A[k * 128 + 2 * i + 1] = -fi;        //      - Fi Xi
      A[(64 + k) * 128 + 2 * i] = fi;      // Yi += Fi Xr
      A[(64 + k) * 128 + 2 * i + 1] = fr;  //      + Fr Xi
    }
  return A;
}

template <typename T>
static double max_rel_err(const std::vector<typename C2<T>::t>& x, const std::vector<typename C2<T>::t>& y, int nvec) {
  double worst = 0.0;
  for (int v = 0; v < nvec; v += nvec / 97 + 1) {
    double num = 0.0, den = 0.0;
    for (int k = 0; k < 64; ++k) {
      long double re = 0, im = 0;
      for (int i = 0; i < 64; ++i) {
        const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)((k * i) % 64) / 64.0L;
        const long double c = cosl(ang), s = sinl(ang);
        re += (long double)x[v * 64 + i].x * c - (long double)x[v * 64 + i].y * s;
        im += (long double)x[v * 64 + i].x * s + (long double)x[v * 64 + i].y * c;
      }
      const double dr = (double)(re - (long double)y[v * 64 + k].x), di = (double)(im - (long double)y[v * 64 + k].y);
      num += dr * dr + di * di;
      den += (double)(re * re + im * im);
    }
    worst = std::max(worst, std::sqrt(num / den));
  }
  return worst;
}

template <typename T, typename Launch>
static void run(const char* name, const char* path, int nvec, Launch launch, double flops_per_vec) {
  using C = typename C2<T>::t;
  const size_t n = (size_t)nvec * 64;
  std::vector<C> hx(n);
  unsigned long long s = 12345;
  for (auto& c : hx) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    c.x = (T)((double)(s >> 11) / 9007199254740992.0 - 0.5);
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    c.y = (T)((double)(s >> 11) / 9007199254740992.0 - 0.5);
  }
  C *dx, *dy;
  CK(cudaMalloc(&dx, n * sizeof(C)));
  CK(cudaMalloc(&dy, n * sizeof(C)));
  CK(cudaMemcpy(dx, hx.data(), n * sizeof(C), cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const bool prof = std::getenv("TC_PROFILE") != nullptr;  // under ncu: one launch per kernel
  for (int i = 0; i < (prof ? 0 : 3); ++i) launch(dx, dy);
  CK(cudaDeviceSynchronize());
  const int reps = prof ? 1 : 20;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch(dx, dy);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  std::vector<C> hy(n);
  CK(cudaMemcpy(hy.data(), dy, n * sizeof(C), cudaMemcpyDeviceToHost));
  const double err = max_rel_err<T>(hx, hy, nvec);
  const double bytes = 2.0 * n * sizeof(C);
  std::printf("{\"kernel\": \"%s\", \"path\": \"%s\", \"dtype\": \"%s\", \"vectors\": %d, \"ms\": %.5f, "
              "\"tflops\": %.2f, \"gbs\": %.1f, \"max_rel_err\": %.3e}\n",
              name, path, sizeof(T) == 8 ? "f64" : "f32", nvec, ms, flops_per_vec * nvec / (ms * 1e-3) / 1e12,
              bytes / (ms * 1e-3) / 1e9, err);
  cudaFree(dx);
  cudaFree(dy);
}

int main() {
  const int nvec = 4096 * 4096 / 64;  // the C3 column stage: 16.7 M complex values
  // fft: 8 + 8 radix-8 DFTs of 8 points (~ 2 x 8 x (8 log2 8 x 5 / 2) real flops) + twiddles
  const double fft_flops = 2.0 * 8.0 * 60.0 + 49.0 * 6.0;
  const double mat_flops = 2.0 * 128.0 * 128.0;  // real 128 x 128 matrix-vector
  // twiddles W64^(r k1)
  std::vector<double2> tw64(64);
  std::vector<float2> tw32(64);
  for (int k = 0; k < 64; ++k) {
    const long double ang = -2.0L * 3.14159265358979323846264338327950288L * k / 64.0L;
    tw64[k] = double2{(double)cosl(ang), (double)sinl(ang)};
    tw32[k] = float2{(float)cosl(ang), (float)sinl(ang)};
  }
  double2* dtw64;
  float2* dtw32;
  CK(cudaMalloc(&dtw64, 64 * sizeof(double2)));
  CK(cudaMalloc(&dtw32, 64 * sizeof(float2)));
  CK(cudaMemcpy(dtw64, tw64.data(), 64 * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw32, tw32.data(), 64 * sizeof(float2), cudaMemcpyHostToDevice));
  auto A64 = dft_matrix_real<double>();
  auto A32 = dft_matrix_real<float>();
  double* dA64;
  float* dA32;
  CK(cudaMalloc(&dA64, A64.size() * sizeof(double)));
  CK(cudaMalloc(&dA32, A32.size() * sizeof(float)));
  CK(cudaMemcpy(dA64, A64.data(), A64.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA32, A32.data(), A32.size() * sizeof(float), cudaMemcpyHostToDevice));
  const size_t sm64 = (128 * 132 + 128 * 68) * sizeof(double), sm32 = (128 * 132 + 128 * 72) * sizeof(float);
  CK(cudaFuncSetAttribute(k_dft64_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64));
  CK(cudaFuncSetAttribute(k_dft64_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm32));
  const int gfft = (nvec + 31) / 32, gmat = 148;  // tensor kernels: persistent, one CTA per SM

  run<double>("k_dft64_fft<double>", "fft radix-8x8 (CUDA cores)", nvec,
              [&](double2* x, double2* y) { k_dft64_fft<double><<<gfft, 256>>>(x, y, dtw64, nvec); }, fft_flops);
  run<double>("k_dft64_dmma", "dense DFT matrix, FP64 tensor cores (DMMA m8n8k4)", nvec,
              [&](double2* x, double2* y) { k_dft64_dmma<<<gmat, 256, sm64>>>(x, y, dA64, nvec); }, mat_flops);
  run<float>("k_dft64_fft<float>", "fft radix-8x8 (CUDA cores)", nvec,
             [&](float2* x, float2* y) { k_dft64_fft<float><<<gfft, 256>>>(x, y, dtw32, nvec); }, fft_flops);
  run<float>("k_dft64_tf32x3", "dense DFT matrix, TF32 tensor cores (3xTF32, m16n8k8)", nvec,
             [&](float2* x, float2* y) { k_dft64_tf32x3<<<gmat, 256, sm32>>>(x, y, dA32, nvec); }, 3.0 * mat_flops);
  CK(cudaDeviceSynchronize());
  return 0;
}
