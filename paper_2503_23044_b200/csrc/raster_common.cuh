// Shared pieces of the compositing forward (K5) and backward (K6) kernels.
#pragma once

#include "common.cuh"

namespace vsx {

struct PixRay {
  float rx, ry;
};

// ((u - cx)/fx, (v - cy)/fy) of an integer pixel centre (renderer.py:274-275).
__device__ __forceinline__ PixRay pixel_ray(const vsx_camera &cam, int px, int py) {
  PixRay r;
  r.rx = (float)(((double)px - cam.cx) / cam.fx);
  r.ry = (float)(((double)py - cam.cy) / cam.fy);
  return r;
}

// Depth-quotient denominator raw_normal . ray, identically rounded in the
// forward and the backward (no FMA contraction) so validity decisions agree.
__device__ __forceinline__ float denom_of(float n0, float n1, float n2, PixRay ray) {
  return __fadd_rn(__fadd_rn(__fmul_rn(n0, ray.rx), __fmul_rn(n1, ray.ry)), n2);
}

// One splat record staged in tile-local float coordinates:
//   p0 = (mx, my, A2, B2)      A2 = -log2(e)/2 * A, B2 = -log2(e) * B
//   p1 = (C2, opacity, plane_d, A)   C2 = -log2(e)/2 * C
//   p2 = (r, g, b, B)
//   p3 = (nx, ny, nz, C)
// so that power * log2(e) = dx*(A2*dx + B2*dy) + C2*dy^2 feeds ex2 directly,
// while the unscaled conic (A, B, C) stays available for the gradients.
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void stage_splat(const vsx_splat &s, double ox, double oy, float4 &p0,
                                            float4 &p1, float4 &p2, float4 &p3) {
  p0 = make_float4((float)(s.mean2d[0] - ox), (float)(s.mean2d[1] - oy),
                   (-0.5f * kLog2e) * s.conic[0], (-kLog2e) * s.conic[1]);
  p1 = make_float4((-0.5f * kLog2e) * s.conic[2], s.opacity, s.plane_d, s.conic[0]);
  p2 = make_float4(s.color[0], s.color[1], s.color[2], s.conic[1]);
  p3 = make_float4(s.normal[0], s.normal[1], s.normal[2], s.conic[2]);
}

// 64-byte record as four 16-byte loads (rec is cudaMalloc'd, 64 B stride).
__device__ __forceinline__ vsx_splat load_splat(const vsx_splat *__restrict__ rec, uint32_t i) {
  union {
    float4 v[4];
    vsx_splat s;
  } u;
  const float4 *p = reinterpret_cast<const float4 *>(rec + i);
#pragma unroll
  for (int k = 0; k < 4; ++k) u.v[k] = __ldg(p + k);
  return u.s;
}

__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Gaussian falloff e = exp(min(power, 0)) and alpha = min(o * e, 0.99) for a
// pixel offset (dx, dy). Explicitly rounded so the forward and the backward
// recompute bit-identical alphas (the backward divides T by 1 - alpha).
__device__ __forceinline__ float splat_alpha(const float4 &p0, const float4 &p1, float dx,
                                             float dy, float &e, float &at) {
  const float q = __fmaf_rn(p0.z, dx, __fmul_rn(p0.w, dy));
  const float p2 = __fmaf_rn(q, dx, __fmul_rn(__fmul_rn(p1.x, dy), dy));
  e = ex2_ftz(fminf(p2, 0.f));
  at = __fmul_rn(p1.y, e);
  return fminf(at, 0.99f);
}

// Cotangent of the 8 blended channels of one pixel (finalize backward,
// renderer.py:282-301): alpha, rgb, raw normal (incl. depth-quotient and
// normal-renormalisation terms) and the plane-offset sum.
struct PixCot {
  float gA, gC0, gC1, gC2, gR0, gR1, gR2, gD;
};

__device__ __forceinline__ PixCot pixel_cotangent(
    const vsx_camera &cam, int px, int py, size_t p, const float *__restrict__ in_alpha,
    const float *__restrict__ in_depth, const float *__restrict__ in_raw,
    const float *__restrict__ g_rgb, const float *__restrict__ g_alpha,
    const float *__restrict__ g_depth, const float *__restrict__ g_normal,
    const float *__restrict__ g_raw) {
  PixCot c{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const float acc = in_alpha[p];
  const float n0 = in_raw[3 * p + 0], n1 = in_raw[3 * p + 1], n2 = in_raw[3 * p + 2];
  const PixRay ray = pixel_ray(cam, px, py);
  const float den = denom_of(n0, n1, n2, ray);
  const bool covered = acc >= kAlphaValidMin;
  const bool valid = covered && fabsf(den) >= kDenomGuard;
  if (g_alpha) c.gA = g_alpha[p];
  if (g_rgb) {
    c.gC0 = g_rgb[3 * p + 0];
    c.gC1 = g_rgb[3 * p + 1];
    c.gC2 = g_rgb[3 * p + 2];
  }
  if (g_depth && valid) {
    const float gd = g_depth[p];
    const float depth = in_depth[p];
    c.gD = gd / den;
    const float gden = -gd * depth / den;
    c.gR0 += gden * ray.rx;
    c.gR1 += gden * ray.ry;
    c.gR2 += gden;
  }
  if (g_raw) {
    c.gR0 += g_raw[3 * p + 0];
    c.gR1 += g_raw[3 * p + 1];
    c.gR2 += g_raw[3 * p + 2];
  }
  if (g_normal && covered) {
    const float gn0 = g_normal[3 * p + 0], gn1 = g_normal[3 * p + 1], gn2 = g_normal[3 * p + 2];
    const float len = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
    if (len >= 1e-12f) {
      const float il = 1.f / len;
      const float dot = (n0 * gn0 + n1 * gn1 + n2 * gn2) * il * il;
      c.gR0 += (gn0 - n0 * dot) * il;
      c.gR1 += (gn1 - n1 * dot) * il;
      c.gR2 += (gn2 - n2 * dot) * il;
    } else {
      c.gR0 += gn0 * 1e12f;
      c.gR1 += gn1 * 1e12f;
      c.gR2 += gn2 * 1e12f;
    }
  }
  return c;
}

__device__ __forceinline__ float sgn(float d) { return d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f); }

// Cotangents of the fused RGB-D-N objective (vsx_loss_desc) for one pixel,
// chained through the finalize backward exactly like pixel_cotangent.
__device__ __forceinline__ PixCot pixel_cotangent_loss(
    const vsx_camera &cam, int px, int py, size_t p, const float *__restrict__ in_alpha,
    const float *__restrict__ in_rgb, const float *__restrict__ in_depth,
    const float *__restrict__ in_normal, const float *__restrict__ in_raw,
    const vsx_loss_desc &L) {
  PixCot c{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const float acc = in_alpha[p];
  const float n0 = in_raw[3 * p + 0], n1 = in_raw[3 * p + 1], n2 = in_raw[3 * p + 2];
  const PixRay ray = pixel_ray(cam, px, py);
  const float den = denom_of(n0, n1, n2, ray);
  const bool covered = acc >= kAlphaValidMin;
  const bool valid = covered && fabsf(den) >= kDenomGuard;
  c.gC0 = sgn(in_rgb[3 * p + 0] - L.gt_rgb[3 * p + 0]) * L.rgb_scale;
  c.gC1 = sgn(in_rgb[3 * p + 1] - L.gt_rgb[3 * p + 1]) * L.rgb_scale;
  c.gC2 = sgn(in_rgb[3 * p + 2] - L.gt_rgb[3 * p + 2]) * L.rgb_scale;
  if (L.extra_rgb) {
    c.gC0 += L.extra_rgb[3 * p + 0];
    c.gC1 += L.extra_rgb[3 * p + 1];
    c.gC2 += L.extra_rgb[3 * p + 2];
  }
  float gd = 0.f;  // cotangent of the output depth (defined where valid)
  if (L.prior_depth && valid && L.prior_depth_valid[p])
    gd = sgn(in_depth[p] - L.prior_depth[p]) * L.depth_weight / (float)max(L.counts[0], 1u);
  if (L.extra_depth && valid) gd += L.extra_depth[p];
  if (gd != 0.f) {
    const float depth = in_depth[p];
    c.gD = gd / den;
    const float gden = -gd * depth / den;
    c.gR0 += gden * ray.rx;
    c.gR1 += gden * ray.ry;
    c.gR2 += gden;
  }
  // cotangent of the output (normalised) normal, defined where covered
  float gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
  if (L.prior_normal && valid && L.prior_normal_valid[p]) {
    const float sc = L.normal_weight / (float)max(L.counts[1], 1u);
    gn0 = sgn(in_normal[3 * p + 0] - L.prior_normal[3 * p + 0]) * sc;
    gn1 = sgn(in_normal[3 * p + 1] - L.prior_normal[3 * p + 1]) * sc;
    gn2 = sgn(in_normal[3 * p + 2] - L.prior_normal[3 * p + 2]) * sc;
  }
  if (L.extra_normal && covered) {
    gn0 += L.extra_normal[3 * p + 0];
    gn1 += L.extra_normal[3 * p + 1];
    gn2 += L.extra_normal[3 * p + 2];
  }
  if (gn0 != 0.f || gn1 != 0.f || gn2 != 0.f) {
    const float len = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
    if (len >= 1e-12f) {
      const float il = 1.f / len;
      const float dot = (n0 * gn0 + n1 * gn1 + n2 * gn2) * il * il;
      c.gR0 += (gn0 - n0 * dot) * il;
      c.gR1 += (gn1 - n1 * dot) * il;
      c.gR2 += (gn2 - n2 * dot) * il;
    } else {
      c.gR0 += gn0 * 1e12f;
      c.gR1 += gn1 * 1e12f;
      c.gR2 += gn2 * 1e12f;
    }
  }
  return c;
}

}  // namespace vsx
