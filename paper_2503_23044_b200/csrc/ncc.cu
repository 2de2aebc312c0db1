// f2 — multi-view patch NCC geometric loss, Eq. 10 (voxsplat losses.py:98-287).
//
// For a (reference, source) view pair and a set of patch centres on the
// source (chosen on the host with the reference's stratified RNG draw), each
// (2h+1)^2 source patch (grayscale of the rendered colour) is compared with
// the reference grayscale image warped through the homography of the source's
// rendered plane at the centre (normal n and depth at the centre pixel):
//   H = K_ref (R_rel + t_rel n^T / d) K_src^-1,  d = n . (depth * ray)
// term = 1 - NCC(src patch, bilinear(ref gray, H . pixel)), reference colours
// detached. One thread per patch, float64 throughout (64 patches per pair).
// The backward is written out by hand: NCC -> (src gray, warped coordinates)
// -> homography -> (n, d) -> (normal, depth) at the centre, and src gray ->
// rgb of every patch pixel. vsx_ncc_scatter adds the scaled per-patch
// gradients into the cotangent images the compositor backward consumes.
#include "common.cuh"

namespace vsx {

__constant__ double kGray[3] = {0.299, 0.587, 0.114};  // losses.py GRAY_WEIGHTS
constexpr double kNccStdGuard = 1e-6;                // NCC_STD_GUARD
constexpr double kPlaneGuard = 1e-6;                 // PLANE_D_GUARD
constexpr int kMaxPatch = 15 * 15;

__device__ __forceinline__ double gray_at(const float *rgb, size_t p) {
  return kGray[0] * (double)rgb[3 * p] + kGray[1] * (double)rgb[3 * p + 1] +
         kGray[2] * (double)rgb[3 * p + 2];
}

// status: 0 = plane through the source centre (rejected), 1 = warp leaves the
// reference image (rejected), 2 = used. grad_* hold d(1 - ncc)/d(input).
__global__ void ncc_patches_kernel(const float *__restrict__ src_rgb,
                                   const float *__restrict__ src_normal,
                                   const float *__restrict__ src_depth, int sw, int sh,
                                   const float *__restrict__ ref_rgb, int rw, int rh,
                                   vsx_ncc_geom G, const int32_t *__restrict__ centers, int P,
                                   int half, double *__restrict__ term,
                                   uint8_t *__restrict__ status, double *__restrict__ g_patch,
                                   double *__restrict__ g_n, double *__restrict__ g_dep,
                                   double *__restrict__ pair_sum, int32_t *__restrict__ pair_used,
                                   int32_t *__restrict__ pairs_used) {
  __shared__ double s_sum;
  __shared__ int s_used;
  if (threadIdx.x == 0) {
    s_sum = 0.0;
    s_used = 0;
  }
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int S = 2 * half + 1, N = S * S;
  if (p < P) {
    const int cu = centers[2 * p], cv = centers[2 * p + 1];
    const size_t c = (size_t)cv * sw + cu;
    const double n[3] = {(double)src_normal[3 * c], (double)src_normal[3 * c + 1],
                         (double)src_normal[3 * c + 2]};
    const double dep = (double)src_depth[c];
    const double ray[3] = {((double)cu - G.src_cx) / G.src_fx, ((double)cv - G.src_cy) / G.src_fy,
                           1.0};
    const double d = n[0] * dep * ray[0] + n[1] * dep * ray[1] + n[2] * dep * ray[2];
    uint8_t st = 0;
    double val = 0.0;
    if (fabs(d) > kPlaneGuard) {
      // M = R_rel + t_rel n^T / d ; H = K_ref M K_src^-1
      double M[9], H[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) M[3 * i + j] = G.r_rel[3 * i + j] + G.t_rel[i] * n[j] / d;
      const double K2[9] = {G.ref_fx, 0.0, G.ref_cx, 0.0, G.ref_fy, G.ref_cy, 0.0, 0.0, 1.0};
      const double K1i[9] = {1.0 / G.src_fx, 0.0, -G.src_cx / G.src_fx,
                             0.0, 1.0 / G.src_fy, -G.src_cy / G.src_fy, 0.0, 0.0, 1.0};
      double T[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          T[3 * i + j] = K2[3 * i] * M[j] + K2[3 * i + 1] * M[3 + j] + K2[3 * i + 2] * M[6 + j];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          H[3 * i + j] = T[3 * i] * K1i[j] + T[3 * i + 1] * K1i[3 + j] + T[3 * i + 2] * K1i[6 + j];
      // warp all patch pixels; every one must land inside the reference
      bool inside = true;
      double qu[kMaxPatch], qv[kMaxPatch], wz[kMaxPatch], x[kMaxPatch], y[kMaxPatch];
      for (int k = 0; k < N; ++k) {
        const double pu = (double)(cu + k % S - half), pv = (double)(cv + k / S - half);
        const double wx = H[0] * pu + H[1] * pv + H[2];
        const double wy = H[3] * pu + H[4] * pv + H[5];
        const double z = H[6] * pu + H[7] * pv + H[8];
        inside &= z > 1e-8;
        wz[k] = fmax(z, 1e-8);
        qu[k] = wx / wz[k];
        qv[k] = wy / wz[k];
        inside &= qu[k] >= 0.0 && qu[k] <= (double)(rw - 1) && qv[k] >= 0.0 &&
                  qv[k] <= (double)(rh - 1);
      }
      st = inside ? 2 : 1;
      if (inside) {
        double mx = 0.0, my = 0.0;
        double fu[kMaxPatch], fv[kMaxPatch];
        for (int k = 0; k < N; ++k) {
          const int pu = cu + k % S - half, pv = cv + k / S - half;
          x[k] = gray_at(src_rgb, (size_t)pv * sw + pu);
          const double u0 = fmin(fmax(floor(qu[k]), 0.0), (double)(rw - 2));
          const double v0 = fmin(fmax(floor(qv[k]), 0.0), (double)(rh - 2));
          fu[k] = qu[k] - u0;
          fv[k] = qv[k] - v0;
          const size_t i00 = (size_t)v0 * rw + (size_t)u0;
          const double a00 = gray_at(ref_rgb, i00), a01 = gray_at(ref_rgb, i00 + 1);
          const double a10 = gray_at(ref_rgb, i00 + rw), a11 = gray_at(ref_rgb, i00 + rw + 1);
          y[k] = a00 * (1 - fu[k]) * (1 - fv[k]) + a01 * fu[k] * (1 - fv[k]) +
                 a10 * (1 - fu[k]) * fv[k] + a11 * fu[k] * fv[k];
          // keep d y / d(qu, qv) in qu / qv (the coordinates are not needed again)
          qu[k] = (a01 - a00) * (1 - fv[k]) + (a11 - a10) * fv[k];
          qv[k] = (a10 - a00) * (1 - fu[k]) + (a11 - a01) * fu[k];
          mx += x[k];
          my += y[k];
        }
        mx /= N;
        my /= N;
        double cov = 0.0, vx = 0.0, vy = 0.0;
        for (int k = 0; k < N; ++k) {
          cov += (x[k] - mx) * (y[k] - my);
          vx += (x[k] - mx) * (x[k] - mx);
          vy += (y[k] - my) * (y[k] - my);
        }
        cov /= N;
        const double rsx = sqrt(vx / N), rsy = sqrt(vy / N);
        const bool cx = rsx < kNccStdGuard, cy = rsy < kNccStdGuard;  // clamped: no grad
        const double sx = cx ? kNccStdGuard : rsx, sy = cy ? kNccStdGuard : rsy;
        const double ncc = cov / (sx * sy);
        val = 1.0 - ncc;
        // d(1 - ncc): source gray, and warped coordinates through the sample
        double dH[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int k = 0; k < N; ++k) {
          const double xm = x[k] - mx, ym = y[k] - my;
          const double dx = -(ym / (N * sx * sy) - (cx ? 0.0 : ncc * xm / (N * sx * sx)));
          const double dy = -(xm / (N * sx * sy) - (cy ? 0.0 : ncc * ym / (N * sy * sy)));
          g_patch[(size_t)p * N + k] = dx;
          const double dqu = dy * qu[k], dqv = dy * qv[k];
          // qu = wx / wz, qv = wy / wz (wz > 1e-8 for an inside patch)
          const double iz = 1.0 / wz[k];
          const double dwx = dqu * iz, dwy = dqv * iz;
          const double pu = (double)(cu + k % S - half), pv = (double)(cv + k / S - half);
          // wz derivative needs the unnormalised warp: recompute it from H
          const double wx = H[0] * pu + H[1] * pv + H[2];
          const double wy = H[3] * pu + H[4] * pv + H[5];
          const double dwz = -(dqu * wx + dqv * wy) * iz * iz;
          const double hom[3] = {pu, pv, 1.0};
          for (int j = 0; j < 3; ++j) {
            dH[j] += dwx * hom[j];
            dH[3 + j] += dwy * hom[j];
            dH[6 + j] += dwz * hom[j];
          }
        }
        // H = K2 M K1i  ->  dM = K2^T dH K1i^T
        double dT[9], dM[9];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            dT[3 * i + j] = dH[3 * i] * K1i[3 * j] + dH[3 * i + 1] * K1i[3 * j + 1] +
                            dH[3 * i + 2] * K1i[3 * j + 2];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            dM[3 * i + j] = K2[i] * dT[j] + K2[3 + i] * dT[3 + j] + K2[6 + i] * dT[6 + j];
        // M = R + t n^T / d
        double dn[3] = {0, 0, 0}, dd = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            dn[j] += dM[3 * i + j] * G.t_rel[i] / d;
            dd -= dM[3 * i + j] * G.t_rel[i] * n[j] / (d * d);
          }
        // d = n . (dep * ray)
        for (int j = 0; j < 3; ++j) dn[j] += dd * dep * ray[j];
        g_n[3 * p + 0] = dn[0];
        g_n[3 * p + 1] = dn[1];
        g_n[3 * p + 2] = dn[2];
        g_dep[p] = dd * (n[0] * ray[0] + n[1] * ray[1] + n[2] * ray[2]);
      }
    }
    term[p] = val;
    status[p] = st;
    if (st == 2) {
      atomicAdd(&s_sum, val);
      atomicAdd(&s_used, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pair_sum[0] = s_sum;
    pair_used[0] = s_used;
    if (s_used > 0) atomicAdd(pairs_used, 1);
  }
}

// Adds scale * per-patch gradients into the source cotangent images, with
// scale = upstream / (pairs_used * patches used in this pair).
__global__ void ncc_scatter_kernel(const int32_t *__restrict__ centers, int P, int half, int sw,
                                   const uint8_t *__restrict__ status,
                                   const double *__restrict__ g_patch,
                                   const double *__restrict__ g_n,
                                   const double *__restrict__ g_dep,
                                   const int32_t *__restrict__ pair_used,
                                   const int32_t *__restrict__ pairs_used, double upstream,
                                   float *__restrict__ g_rgb, float *__restrict__ g_normal,
                                   float *__restrict__ g_depth) {
  const int p = blockIdx.x;
  if (p >= P || status[p] != 2) return;
  const double scale = upstream / ((double)pairs_used[0] * (double)pair_used[0]);
  const int S = 2 * half + 1, N = S * S;
  const int cu = centers[2 * p], cv = centers[2 * p + 1];
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const size_t q = (size_t)(cv + k / S - half) * sw + (cu + k % S - half);
    const double g = scale * g_patch[(size_t)p * N + k];
    for (int ch = 0; ch < 3; ++ch) atomicAdd(g_rgb + 3 * q + ch, (float)(g * kGray[ch]));
  }
  if (threadIdx.x == 0) {
    const size_t c = (size_t)cv * sw + cu;
    for (int j = 0; j < 3; ++j) atomicAdd(g_normal + 3 * c + j, (float)(scale * g_n[3 * p + j]));
    atomicAdd(g_depth + c, (float)(scale * g_dep[p]));
  }
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_ncc_patches(const float *src_rgb, const float *src_normal,
                               const float *src_depth, int32_t sw, int32_t sh,
                               const float *ref_rgb, int32_t rw, int32_t rh, vsx_ncc_geom geom,
                               const int32_t *centers, int32_t n_patches, int32_t half,
                               double *term, uint8_t *status, double *g_patch, double *g_normal,
                               double *g_depth, double *pair_sum, int32_t *pair_used,
                               int32_t *pairs_used, vsx_stream s) {
  VSX_REQUIRE(half >= 1 && (2 * half + 1) * (2 * half + 1) <= kMaxPatch,
              "ncc: patch half-size %d unsupported", half);
  VSX_REQUIRE(n_patches >= 0 && n_patches <= 1024 && rw >= 2 && rh >= 2 && sw >= 1 && sh >= 1,
              "ncc: bad arguments");
  ncc_patches_kernel<<<1, std::max(32, ((n_patches + 31) / 32) * 32), 0, as_stream(s)>>>(
      src_rgb, src_normal, src_depth, sw, sh, ref_rgb, rw, rh, geom, centers, n_patches, half,
      term, status, g_patch, g_normal, g_depth, pair_sum, pair_used, pairs_used);
  VSX_LAUNCH_CHECK("ncc_patches");
  return VSX_OK;
}

extern "C" int vsx_ncc_scatter(const int32_t *centers, int32_t n_patches, int32_t half,
                               int32_t sw, const uint8_t *status, const double *g_patch,
                               const double *g_normal, const double *g_depth,
                               const int32_t *pair_used, const int32_t *pairs_used,
                               double upstream, float *g_rgb, float *g_normal_img,
                               float *g_depth_img, vsx_stream s) {
  if (n_patches <= 0) return VSX_OK;
  ncc_scatter_kernel<<<n_patches, 64, 0, as_stream(s)>>>(
      centers, n_patches, half, sw, status, g_patch, g_normal, g_depth, pair_used, pairs_used,
      upstream, g_rgb, g_normal_img, g_depth_img);
  VSX_LAUNCH_CHECK("ncc_scatter");
  return VSX_OK;
}
