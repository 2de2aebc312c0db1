// K5 / K6 — per-tile front-to-back RGB-D-N compositing and its backward.
//
// Forward restates voxsplat renderer.py:242-301 (_blend_padded + _finalize)
// and :390-449 (rasterize_view): one CTA per 16x16 tile, one thread per pixel,
// splat records staged through shared memory in chunks of 256, CTA-wide early
// exit once every pixel's transmittance fell below 1e-4 (__syncthreads_count).
// Semantics that differ from stock 3DGS and are kept exactly: every binned
// splat contributes (no 1/255 skip, no per-pixel 3-sigma cut), power is
// clamped at 0, alpha is clamped at 0.99, a splat is live iff T_prev >= 1e-4.
//
// Backward walks each tile back to front from the per-pixel live count,
// recovering T_k = T_{k+1} / (1 - alpha_k) from the stored final
// transmittance (the stable direction; see SURVEY.md §7 backward note).
#include "common.cuh"

namespace vsx {

constexpr int kChunk = 256;

struct PixRay {
  float rx, ry;
};

__device__ __forceinline__ PixRay pixel_ray(const vsx_camera &cam, int px, int py) {
  PixRay r;
  r.rx = (float)(((double)px - cam.cx) / cam.fx);
  r.ry = (float)(((double)py - cam.cy) / cam.fy);
  return r;
}

__device__ __noinline__ float denom_of(const float *rn, PixRay ray) {
  return __fadd_rn(__fadd_rn(__fmul_rn(rn[0], ray.rx), __fmul_rn(rn[1], ray.ry)), rn[2]);
}

// Stage one splat record into shared memory in tile-local float coordinates.
__device__ __forceinline__ void stage_splat(const vsx_splat &s, double ox, double oy, float4 &p0,
                                            float4 &p1, float4 &p2, float4 &p3) {
  p0 = make_float4((float)(s.mean2d[0] - ox), (float)(s.mean2d[1] - oy), s.conic[0], s.conic[1]);
  p1 = make_float4(s.conic[2], s.opacity, s.plane_d, 0.f);
  p2 = make_float4(s.color[0], s.color[1], s.color[2], 0.f);
  p3 = make_float4(s.normal[0], s.normal[1], s.normal[2], 0.f);
}

__global__ void __launch_bounds__(256) raster_fwd_kernel(
    const vsx_splat *__restrict__ rec, const uint32_t *__restrict__ tile_off,
    const uint32_t *__restrict__ tile_list, vsx_camera cam, float *__restrict__ out_rgb,
    float *__restrict__ out_alpha, float *__restrict__ out_depth, float *__restrict__ out_normal,
    float *__restrict__ out_raw, uint8_t *__restrict__ out_valid, float *__restrict__ out_T,
    int32_t *__restrict__ out_nc) {
  __shared__ float4 s0[kChunk], s1[kChunk], s2[kChunk], s3[kChunk];
  const int txn = gridDim.x;
  const int tile = blockIdx.y * txn + blockIdx.x;
  const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
  const int px = blockIdx.x * kTile + lx, py = blockIdx.y * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const double ox = (double)(blockIdx.x * kTile), oy = (double)(blockIdx.y * kTile);
  const uint32_t begin = tile_off[tile], end = tile_off[tile + 1];
  const float fx = (float)lx, fy = (float)ly;
  float T = 1.f, acc = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, n0 = 0.f, n1 = 0.f, n2 = 0.f, dist = 0.f;
  int32_t nc = 0;
  bool done = !inside;
  for (uint32_t cs = begin; cs < end; cs += kChunk) {
    if (__syncthreads_count(!done) == 0) break;
    const uint32_t idx = cs + threadIdx.x;
    if (idx < end) {
      const vsx_splat sp = rec[tile_list[idx]];
      stage_splat(sp, ox, oy, s0[threadIdx.x], s1[threadIdx.x], s2[threadIdx.x], s3[threadIdx.x]);
    }
    __syncthreads();
    const int cnt = (int)min((uint32_t)kChunk, end - cs);
    for (int j = 0; j < cnt && !done; ++j) {
      if (T < kEarlyStopT) {
        done = true;
        break;
      }
      const float4 p0 = s0[j], p1 = s1[j];
      const float dx = fx - p0.x, dy = fy - p0.y;
      const float power = -0.5f * (p0.z * dx * dx + 2.0f * p0.w * dx * dy + p1.x * dy * dy);
      const float alpha = fminf(p1.y * __expf(fminf(power, 0.f)), kAlphaClamp);
      const float w = alpha * T;
      const float4 p2 = s2[j], p3 = s3[j];
      acc += w;
      c0 = fmaf(w, p2.x, c0);
      c1 = fmaf(w, p2.y, c1);
      c2 = fmaf(w, p2.z, c2);
      n0 = fmaf(w, p3.x, n0);
      n1 = fmaf(w, p3.y, n1);
      n2 = fmaf(w, p3.z, n2);
      dist = fmaf(w, p1.z, dist);
      T = T * (1.f - alpha);
      nc = (int32_t)(cs - begin) + j + 1;
    }
  }
  if (!inside) return;
  const size_t p = (size_t)py * cam.width + px;
  const float rn[3] = {n0, n1, n2};
  const PixRay ray = pixel_ray(cam, px, py);
  const float den = denom_of(rn, ray);
  const bool covered = acc >= kAlphaValidMin;
  const bool valid = covered && fabsf(den) >= kDenomGuard;
  if (out_rgb) {
    out_rgb[3 * p + 0] = c0;
    out_rgb[3 * p + 1] = c1;
    out_rgb[3 * p + 2] = c2;
  }
  if (out_alpha) out_alpha[p] = acc;
  if (out_depth) out_depth[p] = valid ? dist / den : 0.f;
  if (out_raw) {
    out_raw[3 * p + 0] = n0;
    out_raw[3 * p + 1] = n1;
    out_raw[3 * p + 2] = n2;
  }
  if (out_normal) {
    const float nn = fmaxf(sqrtf(n0 * n0 + n1 * n1 + n2 * n2), 1e-12f);
    out_normal[3 * p + 0] = covered ? n0 / nn : 0.f;
    out_normal[3 * p + 1] = covered ? n1 / nn : 0.f;
    out_normal[3 * p + 2] = covered ? n2 / nn : 0.f;
  }
  if (out_valid) out_valid[p] = valid ? 1 : 0;
  out_T[p] = T;
  out_nc[p] = nc;
}

__global__ void __launch_bounds__(256) raster_bwd_kernel(
    const vsx_splat *__restrict__ rec, const uint32_t *__restrict__ tile_off,
    const uint32_t *__restrict__ tile_list, vsx_camera cam, const float *__restrict__ in_alpha,
    const float *__restrict__ in_depth, const float *__restrict__ in_raw,
    const float *__restrict__ in_T, const int32_t *__restrict__ in_nc,
    const float *__restrict__ g_rgb, const float *__restrict__ g_alpha,
    const float *__restrict__ g_depth, const float *__restrict__ g_normal,
    const float *__restrict__ g_raw, float *__restrict__ grad) {
  __shared__ float4 s0[kChunk], s1[kChunk], s2[kChunk], s3[kChunk];
  __shared__ uint32_t s_rank[kChunk];
  __shared__ int s_max;
  const int txn = gridDim.x;
  const int tile = blockIdx.y * txn + blockIdx.x;
  const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
  const int px = blockIdx.x * kTile + lx, py = blockIdx.y * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const double ox = (double)(blockIdx.x * kTile), oy = (double)(blockIdx.y * kTile);
  const uint32_t begin = tile_off[tile], end = tile_off[tile + 1];
  const float fx = (float)lx, fy = (float)ly;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  // ---- per-pixel cotangent of the blended channels (finalize backward)
  int nc = 0;
  float T = 1.f;
  float gA = 0.f, gC0 = 0.f, gC1 = 0.f, gC2 = 0.f, gR0 = 0.f, gR1 = 0.f, gR2 = 0.f, gD = 0.f;
  if (inside) {
    const size_t p = (size_t)py * cam.width + px;
    nc = in_nc[p];
    T = in_T[p];
    const float acc = in_alpha[p];
    const float rn[3] = {in_raw[3 * p + 0], in_raw[3 * p + 1], in_raw[3 * p + 2]};
    const PixRay ray = pixel_ray(cam, px, py);
    const float den = denom_of(rn, ray);
    const bool covered = acc >= kAlphaValidMin;
    const bool valid = covered && fabsf(den) >= kDenomGuard;
    if (g_alpha) gA = g_alpha[p];
    if (g_rgb) {
      gC0 = g_rgb[3 * p + 0];
      gC1 = g_rgb[3 * p + 1];
      gC2 = g_rgb[3 * p + 2];
    }
    if (g_depth && valid) {
      const float gd = g_depth[p];
      const float depth = in_depth[p];
      gD = gd / den;
      const float gden = -gd * depth / den;
      gR0 += gden * ray.rx;
      gR1 += gden * ray.ry;
      gR2 += gden;
    }
    if (g_raw) {
      gR0 += g_raw[3 * p + 0];
      gR1 += g_raw[3 * p + 1];
      gR2 += g_raw[3 * p + 2];
    }
    if (g_normal && covered) {
      const float gn0 = g_normal[3 * p + 0], gn1 = g_normal[3 * p + 1], gn2 = g_normal[3 * p + 2];
      const float len = sqrtf(rn[0] * rn[0] + rn[1] * rn[1] + rn[2] * rn[2]);
      if (len >= 1e-12f) {
        const float il = 1.f / len;
        const float dot = (rn[0] * gn0 + rn[1] * gn1 + rn[2] * gn2) * il * il;
        gR0 += (gn0 - rn[0] * dot) * il;
        gR1 += (gn1 - rn[1] * dot) * il;
        gR2 += (gn2 - rn[2] * dot) * il;
      } else {
        gR0 += gn0 * 1e12f;
        gR1 += gn1 * 1e12f;
        gR2 += gn2 * 1e12f;
      }
    }
    atomicMax(&s_max, nc);
  }
  __syncthreads();
  const uint32_t stop = begin + (uint32_t)s_max;
  float S = 0.f;  // sum over later live splats of s_i * w_i
  for (uint32_t ce = stop; ce > begin;) {
    const uint32_t cs = ce > begin + kChunk ? ce - kChunk : begin;
    const uint32_t idx = cs + threadIdx.x;
    if (idx < ce) {
      const uint32_t r = tile_list[idx];
      s_rank[threadIdx.x] = r;
      stage_splat(rec[r], ox, oy, s0[threadIdx.x], s1[threadIdx.x], s2[threadIdx.x], s3[threadIdx.x]);
    }
    __syncthreads();
    for (int j = (int)(ce - cs) - 1; j >= 0; --j) {
      const int k = (int)(cs - begin) + j;
      const bool live = k < nc;
      float g[13];
#pragma unroll
      for (int q = 0; q < 13; ++q) g[q] = 0.f;
      if (live) {
        const float4 p0 = s0[j], p1 = s1[j], p2 = s2[j], p3 = s3[j];
        const float dx = fx - p0.x, dy = fy - p0.y;
        const float power = -0.5f * (p0.z * dx * dx + 2.0f * p0.w * dx * dy + p1.x * dy * dy);
        const float e = __expf(fminf(power, 0.f));
        const float at = p1.y * e;
        const float alpha = fminf(at, kAlphaClamp);
        const float om = 1.f - alpha;
        const float Tk = T / om;
        const float w = alpha * Tk;
        const float sk = gA + gC0 * p2.x + gC1 * p2.y + gC2 * p2.z + gR0 * p3.x + gR1 * p3.y +
                         gR2 * p3.z + gD * p1.z;
        const float da = Tk * sk - S / om;
        S = fmaf(sk, w, S);
        T = Tk;
        g[6] = w * gC0;
        g[7] = w * gC1;
        g[8] = w * gC2;
        g[9] = w * gR0;
        g[10] = w * gR1;
        g[11] = w * gR2;
        g[12] = w * gD;
        const float dat = at <= kAlphaClamp ? da : 0.f;
        g[5] = dat * e;
        const float dp = power <= 0.f ? dat * p1.y * e : 0.f;
        g[2] = -0.5f * dp * dx * dx;
        g[3] = -dp * dx * dy;
        g[4] = -0.5f * dp * dy * dy;
        g[0] = dp * (p0.z * dx + p0.w * dy);
        g[1] = dp * (p0.w * dx + p1.x * dy);
      }
      if (__any_sync(0xffffffffu, live)) {
#pragma unroll
        for (int q = 0; q < 13; ++q) g[q] = warp_sum(g[q]);
        if (lane == 0) {
          float *dst = grad + (size_t)13 * s_rank[j];
#pragma unroll
          for (int q = 0; q < 13; ++q) atomicAdd(dst + q, g[q]);
        }
      }
    }
    __syncthreads();
    ce = cs;
  }
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_raster_fwd(const vsx_splat *rec, const uint32_t *tile_offsets,
                              const uint32_t *tile_list, vsx_camera cam, float *rgb,
                              float *alpha, float *depth, float *normal, float *raw_normal,
                              uint8_t *valid, float *t_final, int32_t *n_contrib,
                              vsx_stream s) {
  VSX_REQUIRE(cam.width > 0 && cam.height > 0 && t_final && n_contrib, "raster_fwd: bad args");
  dim3 grid((cam.width + kTile - 1) / kTile, (cam.height + kTile - 1) / kTile);
  raster_fwd_kernel<<<grid, 256, 0, as_stream(s)>>>(rec, tile_offsets, tile_list, cam, rgb, alpha,
                                                    depth, normal, raw_normal, valid, t_final,
                                                    n_contrib);
  VSX_LAUNCH_CHECK("raster_fwd");
  return VSX_OK;
}

extern "C" int vsx_raster_bwd(const vsx_splat *rec, const uint32_t *tile_offsets,
                              const uint32_t *tile_list, vsx_camera cam, const float *rgb,
                              const float *alpha, const float *depth, const float *raw_normal,
                              const float *t_final, const int32_t *n_contrib, const float *g_rgb,
                              const float *g_alpha, const float *g_depth, const float *g_normal,
                              const float *g_raw_normal, float *grad_splat, vsx_stream s) {
  (void)rgb;
  VSX_REQUIRE(cam.width > 0 && cam.height > 0 && alpha && raw_normal && t_final && n_contrib,
              "raster_bwd: bad args");
  VSX_REQUIRE(!g_depth || depth, "raster_bwd: depth cotangent needs the depth image");
  dim3 grid((cam.width + kTile - 1) / kTile, (cam.height + kTile - 1) / kTile);
  raster_bwd_kernel<<<grid, 256, 0, as_stream(s)>>>(rec, tile_offsets, tile_list, cam, alpha,
                                                    depth, raw_normal, t_final, n_contrib, g_rgb,
                                                    g_alpha, g_depth, g_normal, g_raw_normal,
                                                    grad_splat);
  VSX_LAUNCH_CHECK("raster_bwd");
  return VSX_OK;
}
