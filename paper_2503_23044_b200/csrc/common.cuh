// Shared device helpers for the vsx_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>

#include "../../include/vsx_b200.h"

#define VSX_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) {                                 \
      vsx_set_error("%s: %s", #expr, cudaGetErrorString(_e)); \
      return VSX_ERR_CUDA;                                   \
    }                                                        \
  } while (0)

void vsx_count_launch();

#define VSX_LAUNCH_CHECK(name)                                          \
  do {                                                                  \
    vsx_count_launch();                                                 \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) {                                            \
      vsx_set_error("%s launch: %s", name, cudaGetErrorString(_e));     \
      return VSX_ERR_CUDA;                                              \
    }                                                                   \
  } while (0)

#define VSX_REQUIRE(cond, ...)    \
  do {                            \
    if (!(cond)) {                \
      vsx_set_error(__VA_ARGS__); \
      return VSX_ERR_INVALID;     \
    }                             \
  } while (0)

void vsx_set_error(const char *fmt, ...);

namespace vsx {

constexpr int kTile = 16;
constexpr int kTilePixels = kTile * kTile;
constexpr int kEmbed = 32;
constexpr int kInDim = kEmbed + 4;
constexpr int kHidden = 64;
constexpr int kHeads = 3;

constexpr double kZNear = 0.01;
constexpr float kAlphaClamp = 0.99f;
constexpr float kEarlyStopT = 1e-4f;
constexpr float kAlphaValidMin = 1e-4f;
constexpr float kDenomGuard = 1e-6f;
constexpr double kLowpass = 0.3;
constexpr double kMinScale = 1e-6;

inline cudaStream_t as_stream(vsx_stream s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

// Row stride of the feature-major decoder caches ([rows][ld], anchors along a
// row): padded to 4 floats so rows are 16-byte aligned for vector loads.
__host__ __device__ __forceinline__ size_t cache_ld(int64_t n_active) {
  return (size_t)((n_active + 3) & ~int64_t(3));
}

// Gaussian-parallel decoder kernels stage the [rows x na] slice of a
// feature-major cache (anchors r0 .. r0+na) through shared memory
// ([rows][sp] floats). rows * na <= 11 * 256, so each of the 256 threads owns
// at most 11 elements; all of its loads are issued before the first smem store
// so their latencies overlap. Element e sits at row e / na, split with a float
// reciprocal: (e + 0.5) / na is >= 0.5 / na from any integer and e < 2^12, so
// the truncated product is the exact quotient.
__device__ __forceinline__ int tile_row(int e, float inv_na) {
  return __float2int_rz(((float)e + 0.5f) * inv_na);
}

__device__ __forceinline__ void stage_cache_tile(float *__restrict__ so, const float *__restrict__ src,
                                                 size_t ld, int r0, int na, int rows, int sp) {
  const int total = rows * na;
  const float inv = 1.0f / (float)na;
  float v[11];
#pragma unroll
  for (int i = 0; i < 11; ++i) {
    const int e = (int)threadIdx.x + 256 * i;
    const int row = tile_row(e, inv);
    if (e < total) v[i] = __ldg(src + (size_t)row * ld + r0 + (e - row * na));
  }
#pragma unroll
  for (int i = 0; i < 11; ++i) {
    const int e = (int)threadIdx.x + 256 * i;
    const int row = tile_row(e, inv);
    if (e < total) so[row * sp + (e - row * na)] = v[i];
  }
}

__device__ __forceinline__ void flush_cache_tile(float *__restrict__ dst, const float *__restrict__ so,
                                                 size_t ld, int r0, int na, int rows, int sp) {
  const int total = rows * na;
  const float inv = 1.0f / (float)na;
#pragma unroll
  for (int i = 0; i < 11; ++i) {
    const int e = (int)threadIdx.x + 256 * i;
    const int row = tile_row(e, inv);
    if (e < total) dst[(size_t)row * ld + r0 + (e - row * na)] = so[row * sp + (e - row * na)];
  }
}

// Explicitly rounded float64 ops: nvcc would otherwise contract a*b+c into an
// FMA, which numpy/torch elementwise code never does. Decisions that must be
// bit-exact against the reference (culling, projection keys, binning) use these.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// x_cam = R x + t, rounded exactly like the reference's `p @ R.T + t`: the
// host BLAS dgemm accumulates the K=3 dot product as fma(p2, r2, fma(p1, r1,
// p0*r0)) (verified bit-for-bit against numpy and torch on the build host),
// then the bias add is a separate rounded op.
__device__ __forceinline__ double dot3_blas(double a0, double a1, double a2, double b0, double b1,
                                            double b2) {
  return __fma_rn(a2, b2, __fma_rn(a1, b1, dmul(a0, b0)));
}

__device__ __forceinline__ void cam_transform(const vsx_camera &c, double x, double y, double z,
                                              double &ox, double &oy, double &oz) {
  ox = dadd(dot3_blas(x, y, z, c.r[0], c.r[1], c.r[2]), c.t[0]);
  oy = dadd(dot3_blas(x, y, z, c.r[3], c.r[4], c.r[5]), c.t[1]);
  oz = dadd(dot3_blas(x, y, z, c.r[6], c.r[7], c.r[8]), c.t[2]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Quaternion (w,x,y,z) -> row-major rotation, reference decoder.py:108-114.
template <typename T>
__device__ __forceinline__ void quat_to_rot(T w, T x, T y, T z, T *m) {
  m[0] = T(1) - T(2) * (y * y + z * z);
  m[1] = T(2) * (x * y - w * z);
  m[2] = T(2) * (x * z + w * y);
  m[3] = T(2) * (x * y + w * z);
  m[4] = T(1) - T(2) * (x * x + z * z);
  m[5] = T(2) * (y * z - w * x);
  m[6] = T(2) * (x * z - w * y);
  m[7] = T(2) * (y * z + w * x);
  m[8] = T(1) - T(2) * (x * x + y * y);
}

// tanh(x) = sign(x) (1 - 2 / (exp(2|x|) + 1)) on the MUFU ex2 / rcp units:
// six instructions instead of tanhf's ~20, absolute error < 3e-7 (|x| -> inf
// gives exactly +-1, x = 0 gives 0). The decoder's hidden layer feeds a
// 64-term product with |w2| <= 1/8, so this stays well inside the 1e-4
// image contract (the reference uses float64 torch.tanh, decoder.py:147).
__device__ __forceinline__ float tanh_fast(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(x) * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.f));
  return copysignf(__fmaf_rn(-2.f, r, 1.f), x);
}

// Index of the smallest of three scales, first index on ties (torch.argmin).
template <typename T>
__device__ __forceinline__ int argmin3(T a, T b, T c) {
  int i = 0;
  T best = a;
  if (b < best) { best = b; i = 1; }
  if (c < best) { i = 2; }
  return i;
}

// Tile rectangle of a splat (renderer.py:216-221), float64 floor semantics.
__device__ __forceinline__ bool tile_rect(double u, double v, double r, int txn, int tyn, int &x0,
                                          int &x1, int &y0, int &y1) {
  // x / 16 == x * 0.0625 exactly (power of two), without the f64 divide
  const double fx0 = fmax(floor(dmul(dsub(u, r), 0.0625)), 0.0);
  const double fx1 = fmin(floor(dmul(dadd(u, r), 0.0625)), (double)(txn - 1));
  const double fy0 = fmax(floor(dmul(dsub(v, r), 0.0625)), 0.0);
  const double fy1 = fmin(floor(dmul(dadd(v, r), 0.0625)), (double)(tyn - 1));
  if (!(fx1 >= fx0) || !(fy1 >= fy0)) return false;
  x0 = (int)fx0;
  x1 = (int)fx1;
  y0 = (int)fy0;
  y1 = (int)fy1;
  return true;
}

}  // namespace vsx
