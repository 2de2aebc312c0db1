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
// It is split per chunk of kBC splats into
//   phase 1 (thread = pixel): the sequential back-to-front recursion, writing
//            the two per-(pixel, splat) scalars w = alpha*T and
//            q = dL/d(alpha_unclamped) * exp(power) to shared memory;
//   phase 2 (warp = splats, lane = pixels): per-splat sums over the tile's 256
//            pixels in registers, one warp reduction per splat and chunk, and
//            13 float atomics per (splat, tile) into the per-splat gradient.
// This replaces a 13-value warp reduction per (splat, warp) (round-1 v1, see
// profiles/r01_raster_bwd_v1_ncu.txt), which made the backward LSU-bound.
#include "raster_common.cuh"

namespace vsx {

constexpr int kChunk = 256;
constexpr int kBCMax = 32;  // largest backward splat chunk

__global__ void __launch_bounds__(256) raster_fwd_kernel(
    const vsx_splat *__restrict__ rec, const uint32_t *__restrict__ tile_off,
    const uint32_t *__restrict__ tile_list, vsx_camera cam, float *__restrict__ out_rgb,
    float *__restrict__ out_alpha, float *__restrict__ out_depth, float *__restrict__ out_normal,
    float *__restrict__ out_raw, uint8_t *__restrict__ out_valid, float *__restrict__ out_T,
    int32_t *__restrict__ out_nc, vsx_loss_desc L) {
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
    if (!done) {
      int j = 0;
#pragma unroll 4
      for (; j < cnt; ++j) {
        if (T < kEarlyStopT) break;  // T_prev < 1e-4: this and every later splat is dead
        const float4 p0 = s0[j], p1 = s1[j];
        float e, at;
        const float alpha = splat_alpha(p0, p1, fx - p0.x, fy - p0.y, e, at);
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
        T = __fmaf_rn(-alpha, T, T);
      }
      nc = (int32_t)(cs - begin) + j;
      done = j < cnt;
    }
  }
  // loss partial sums (fused K9): rgb |d|, masked depth |d|, masked normal |d|
  double l_rgb = 0.0, l_dep = 0.0, l_nrm = 0.0;
  uint32_t c_dep = 0, c_nrm = 0;
  if (inside) {
    const size_t p = (size_t)py * cam.width + px;
    const PixRay ray = pixel_ray(cam, px, py);
    const float den = denom_of(n0, n1, n2, ray);
    const bool covered = acc >= kAlphaValidMin;
    const bool valid = covered && fabsf(den) >= kDenomGuard;
    const float depth = valid ? dist / den : 0.f;
    const float nn = fmaxf(sqrtf(n0 * n0 + n1 * n1 + n2 * n2), 1e-12f);
    const float nx = covered ? n0 / nn : 0.f, ny = covered ? n1 / nn : 0.f,
                nz = covered ? n2 / nn : 0.f;
    if (out_rgb) {
      out_rgb[3 * p + 0] = c0;
      out_rgb[3 * p + 1] = c1;
      out_rgb[3 * p + 2] = c2;
    }
    if (out_alpha) out_alpha[p] = acc;
    if (out_depth) out_depth[p] = depth;
    if (out_raw) {
      out_raw[3 * p + 0] = n0;
      out_raw[3 * p + 1] = n1;
      out_raw[3 * p + 2] = n2;
    }
    if (out_normal) {
      out_normal[3 * p + 0] = nx;
      out_normal[3 * p + 1] = ny;
      out_normal[3 * p + 2] = nz;
    }
    if (out_valid) out_valid[p] = valid ? 1 : 0;
    out_T[p] = T;
    out_nc[p] = nc;
    if (L.gt_rgb) {
      l_rgb = fabs((double)(c0 - L.gt_rgb[3 * p + 0])) + fabs((double)(c1 - L.gt_rgb[3 * p + 1])) +
              fabs((double)(c2 - L.gt_rgb[3 * p + 2]));
      if (L.prior_depth && valid && L.prior_depth_valid[p]) {
        l_dep = fabs((double)(depth - L.prior_depth[p]));
        c_dep = 1;
      }
      if (L.prior_normal && valid && L.prior_normal_valid[p]) {
        l_nrm = fabs((double)(nx - L.prior_normal[3 * p + 0])) +
                fabs((double)(ny - L.prior_normal[3 * p + 1])) +
                fabs((double)(nz - L.prior_normal[3 * p + 2]));
        c_nrm = 1;
      }
    }
  }
  if (L.gt_rgb) {  // block-uniform
    l_rgb = warp_sum_d(l_rgb);
    l_dep = warp_sum_d(l_dep);
    l_nrm = warp_sum_d(l_nrm);
    const unsigned bd = __ballot_sync(0xffffffffu, c_dep), bn = __ballot_sync(0xffffffffu, c_nrm);
    if ((threadIdx.x & 31) == 0) {
      if (l_rgb != 0.0) atomicAdd(L.sums + 0, l_rgb);
      if (bd) {
        atomicAdd(L.sums + 1, l_dep);
        atomicAdd(L.counts + 0, (uint32_t)__popc(bd));
      }
      if (bn) {
        atomicAdd(L.sums + 2, l_nrm);
        atomicAdd(L.counts + 1, (uint32_t)__popc(bn));
      }
    }
  }
}

struct BwdArgs {
  const vsx_splat *rec;
  const uint32_t *tile_off;
  const uint32_t *tile_list;
  const float *alpha, *depth, *raw, *T, *g_rgb, *g_alpha, *g_depth, *g_normal, *g_raw;
  const int32_t *nc;
  float *grad;
  const float *rgb, *normal;  // forward outputs (fused-loss mode)
  vsx_loss_desc L;            // L.gt_rgb != NULL: cotangents from the fused objective
};

// ---------------------------------------------------------------- backward v2

template <int NS, int kBC>
__global__ void __launch_bounds__(256, (kBC == 16 ? 4 : 3))
    raster_bwd_kernel(BwdArgs a, vsx_camera cam) {
  __shared__ float4 s0[kBC], s1[kBC], s2[kBC], s3[kBC];
  __shared__ uint32_t s_rank[kBC];
  extern __shared__ float2 s_wq[];                // (w, q) per (splat, pixel): [kBC][256]
  __shared__ float4 s_ga[kTilePixels], s_gb[kTilePixels];  // pixel cotangents
  __shared__ int s_max;
  const int txn = gridDim.x;
  const int tile = blockIdx.y * txn + blockIdx.x;
  const int t = threadIdx.x;
  const int lx = t & 15, ly = t >> 4;
  const int px = blockIdx.x * kTile + lx, py = blockIdx.y * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const double ox = (double)(blockIdx.x * kTile), oy = (double)(blockIdx.y * kTile);
  const uint32_t begin = a.tile_off[tile];
  const float fx = (float)lx, fy = (float)ly;
  const int lane = t & 31, warp = t >> 5;
  if (t == 0) s_max = 0;
  __syncthreads();
  int nc = 0;
  float T = 1.f;
  PixCot c{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (inside) {
    const size_t p = (size_t)py * cam.width + px;
    nc = a.nc[p];
    T = a.T[p];
    if (a.L.gt_rgb)
      c = pixel_cotangent_loss(cam, px, py, p, a.alpha, a.rgb, a.depth, a.normal, a.raw, a.L);
    else
      c = pixel_cotangent(cam, px, py, p, a.alpha, a.depth, a.raw, a.g_rgb, a.g_alpha, a.g_depth,
                          a.g_normal, a.g_raw);
    if (nc > 0) atomicMax(&s_max, nc);
  }
  s_ga[t] = make_float4(c.gA, c.gC0, c.gC1, c.gC2);
  s_gb[t] = make_float4(c.gR0, c.gR1, c.gR2, c.gD);
  __syncthreads();
  const uint32_t stop = begin + (uint32_t)s_max;
  float S = 0.f;  // sum over later live splats of s_i * w_i
  for (uint32_t ce = stop; ce > begin;) {
    const uint32_t cs = ce > begin + kBC ? ce - kBC : begin;
    const int cnt = (int)(ce - cs);
    if (t < cnt) {
      const uint32_t r = a.tile_list[cs + t];
      s_rank[t] = r;
      stage_splat(a.rec[r], ox, oy, s0[t], s1[t], s2[t], s3[t]);
    }
    __syncthreads();
    // ---- phase 1: per-pixel back-to-front recursion
    const int kbase = (int)(cs - begin);
    // live splats of this pixel in the chunk are j < nc - kbase
    const int jlive = min(cnt, nc - kbase);
    // dead (and, in a partial chunk, padding) rows carry zeros into phase 2
    for (int j = kBC - 1; j >= max(jlive, 0); --j) s_wq[j * kTilePixels + t] = make_float2(0.f, 0.f);
#pragma unroll 2
    for (int j = jlive - 1; j >= 0; --j) {
      float2 wq;
      {
        const float4 p0 = s0[j], p1 = s1[j];
        const float4 p2 = s2[j], p3 = s3[j];
        float e, at;
        const float alpha = splat_alpha(p0, p1, fx - p0.x, fy - p0.y, e, at);
        const float rom = rcp_ftz(1.f - alpha);
        const float Tk = T * rom;
        const float w = alpha * Tk;
        const float sk = c.gA + c.gC0 * p2.x + c.gC1 * p2.y + c.gC2 * p2.z + c.gR0 * p3.x +
                         c.gR1 * p3.y + c.gR2 * p3.z + c.gD * p1.z;
        const float da = Tk * sk - S * rom;
        S = fmaf(sk, w, S);
        T = Tk;
        // power <= 0 for a positive-definite conic; where rounding makes it
        // slightly positive the clamped branch's zero d/dpower differs from
        // dat*e*op only by terms of order dx, dy ~ 0 (phase 2 multiplies them).
        const float dat = at <= kAlphaClamp ? da : 0.f;
        wq = make_float2(w, dat * e);
      }
      s_wq[j * kTilePixels + t] = wq;
    }
    __syncthreads();
    // ---- phase 2: warp w owns splats j = w + 8s (s < 4); lanes stride the 256
    // pixels. Per splat it accumulates 7 colour/normal/plane sums sum_p w*G(p)
    // and 6 pixel moments of q about the tile centre (1, x, y, x^2, xy, y^2);
    // the conic/mean/opacity gradients are polynomials of those moments.
    for (int jb = warp; jb < cnt; jb += 8 * NS) {
      float acc[NS][13];
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int q = 0; q < 13; ++q) acc[s][q] = 0.f;
      // pix = lane + 32 i: x = lane & 15 is fixed per lane, y = (lane >> 4) + 2 i
      const float xc = (float)(lane & 15) - 7.5f, xx = xc * xc;
#pragma unroll 2
      for (int i = 0; i < kTilePixels / 32; ++i) {
        const int pix = lane + 32 * i;
        const float4 ga = s_ga[pix], gb = s_gb[pix];
        const float yc = (float)((lane >> 4) + 2 * i) - 7.5f;
        const float xy = xc * yc, yy = yc * yc;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int j = jb + 8 * s;  // rows >= cnt are zero-padded by phase 1
          {
            const float2 wq = s_wq[j * kTilePixels + pix];
            acc[s][0] = fmaf(wq.x, ga.y, acc[s][0]);
            acc[s][1] = fmaf(wq.x, ga.z, acc[s][1]);
            acc[s][2] = fmaf(wq.x, ga.w, acc[s][2]);
            acc[s][3] = fmaf(wq.x, gb.x, acc[s][3]);
            acc[s][4] = fmaf(wq.x, gb.y, acc[s][4]);
            acc[s][5] = fmaf(wq.x, gb.z, acc[s][5]);
            acc[s][6] = fmaf(wq.x, gb.w, acc[s][6]);
            acc[s][7] += wq.y;
            acc[s][8] = fmaf(wq.y, xc, acc[s][8]);
            acc[s][9] = fmaf(wq.y, yc, acc[s][9]);
            acc[s][10] = fmaf(wq.y, xx, acc[s][10]);
            acc[s][11] = fmaf(wq.y, xy, acc[s][11]);
            acc[s][12] = fmaf(wq.y, yy, acc[s][12]);
          }
        }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int j = jb + 8 * s;
        if (j >= cnt) break;  // warp-uniform
#pragma unroll
        for (int q = 0; q < 13; ++q) acc[s][q] = warp_sum(acc[s][q]);
        const float4 p0 = s0[j], p1 = s1[j];
        const float op = p1.y, A = p1.w, B = s2[j].w, C = s3[j].w;
        const float mx = p0.x - 7.5f, my = p0.y - 7.5f;
        const float Q1 = acc[s][7];
        const float sx = acc[s][8] - mx * Q1;                 // sum q dx
        const float sy = acc[s][9] - my * Q1;                 // sum q dy
        const float sxx = acc[s][10] - 2.f * mx * acc[s][8] + mx * mx * Q1;
        const float sxy = acc[s][11] - mx * acc[s][9] - my * acc[s][8] + mx * my * Q1;
        const float syy = acc[s][12] - 2.f * my * acc[s][9] + my * my * Q1;
        float g[13];
        g[0] = op * (A * sx + B * sy);
        g[1] = op * (B * sx + C * sy);
        g[2] = -0.5f * op * sxx;
        g[3] = -op * sxy;
        g[4] = -0.5f * op * syy;
        g[5] = Q1;
#pragma unroll
        for (int q = 0; q < 7; ++q) g[6 + q] = acc[s][q];
        if (lane < 13) {
          float v = g[0];
#pragma unroll
          for (int q = 1; q < 13; ++q) v = (lane == q) ? g[q] : v;
          if (v != 0.f) atomicAdd(a.grad + (size_t)13 * s_rank[j] + lane, v);
        }
      }
    }
    __syncthreads();
    ce = cs;
  }
}

static int launch_bwd(const BwdArgs &a, const vsx_camera &cam, cudaStream_t st) {
  dim3 grid((cam.width + kTile - 1) / kTile, (cam.height + kTile - 1) / kTile);
  // VSX_RASTER_BWD="NS,BC" selects the phase-2 splats-per-pass and the splat
  // chunk for A/B timing (default 2,32).
  static int ns = 2, bc = 32;
  static bool attr = false;
  if (!attr) {
    if (const char *sel = getenv("VSX_RASTER_BWD")) sscanf(sel, "%d,%d", &ns, &bc);
    const int s32 = (int)(sizeof(float2) * 32 * kTilePixels);
    const int s16 = (int)(sizeof(float2) * 16 * kTilePixels);
    VSX_CUDA_TRY(cudaFuncSetAttribute(raster_bwd_kernel<1, 16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, s16));
    VSX_CUDA_TRY(cudaFuncSetAttribute(raster_bwd_kernel<2, 16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, s16));
    VSX_CUDA_TRY(cudaFuncSetAttribute(raster_bwd_kernel<1, 32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, s32));
    VSX_CUDA_TRY(cudaFuncSetAttribute(raster_bwd_kernel<2, 32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, s32));
    attr = true;
  }
  const int smem = (int)(sizeof(float2) * bc * kTilePixels);
  if (bc == 16) {
    if (ns == 1) raster_bwd_kernel<1, 16><<<grid, 256, smem, st>>>(a, cam);
    else raster_bwd_kernel<2, 16><<<grid, 256, smem, st>>>(a, cam);
  } else {
    if (ns == 1) raster_bwd_kernel<1, 32><<<grid, 256, smem, st>>>(a, cam);
    else raster_bwd_kernel<2, 32><<<grid, 256, smem, st>>>(a, cam);
  }
  VSX_LAUNCH_CHECK("raster_bwd");
  return VSX_OK;
}

static int launch_fwd(const vsx_splat *rec, const uint32_t *tile_offsets,
                      const uint32_t *tile_list, const vsx_camera &cam, float *rgb, float *alpha,
                      float *depth, float *normal, float *raw_normal, uint8_t *valid,
                      float *t_final, int32_t *n_contrib, const vsx_loss_desc &L,
                      cudaStream_t st) {
  VSX_REQUIRE(cam.width > 0 && cam.height > 0 && t_final && n_contrib, "raster_fwd: bad args");
  dim3 grid((cam.width + kTile - 1) / kTile, (cam.height + kTile - 1) / kTile);
  raster_fwd_kernel<<<grid, 256, 0, st>>>(rec, tile_offsets, tile_list, cam, rgb, alpha, depth,
                                          normal, raw_normal, valid, t_final, n_contrib, L);
  VSX_LAUNCH_CHECK("raster_fwd");
  return VSX_OK;
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_raster_fwd(const vsx_splat *rec, const uint32_t *tile_offsets,
                              const uint32_t *tile_list, vsx_camera cam, float *rgb,
                              float *alpha, float *depth, float *normal, float *raw_normal,
                              uint8_t *valid, float *t_final, int32_t *n_contrib,
                              vsx_stream s) {
  vsx_loss_desc none{};
  return launch_fwd(rec, tile_offsets, tile_list, cam, rgb, alpha, depth, normal, raw_normal,
                    valid, t_final, n_contrib, none, as_stream(s));
}

extern "C" int vsx_raster_fwd_loss(const vsx_splat *rec, const uint32_t *tile_offsets,
                                   const uint32_t *tile_list, vsx_camera cam, float *rgb,
                                   float *alpha, float *depth, float *normal, float *raw_normal,
                                   uint8_t *valid, float *t_final, int32_t *n_contrib,
                                   vsx_loss_desc loss, vsx_stream s) {
  VSX_REQUIRE(loss.gt_rgb && loss.sums && loss.counts, "raster_fwd_loss: gt_rgb/sums/counts");
  VSX_REQUIRE(rgb && depth && normal && valid, "raster_fwd_loss: needs rgb/depth/normal/valid");
  return launch_fwd(rec, tile_offsets, tile_list, cam, rgb, alpha, depth, normal, raw_normal,
                    valid, t_final, n_contrib, loss, as_stream(s));
}

extern "C" int vsx_raster_bwd(const vsx_splat *rec, const uint32_t *tile_offsets,
                              const uint32_t *tile_list, vsx_camera cam, const float *rgb,
                              const float *alpha, const float *depth, const float *raw_normal,
                              const float *t_final, const int32_t *n_contrib, const float *g_rgb,
                              const float *g_alpha, const float *g_depth, const float *g_normal,
                              const float *g_raw_normal, float *grad_splat, vsx_stream s) {
  VSX_REQUIRE(cam.width > 0 && cam.height > 0 && alpha && raw_normal && t_final && n_contrib,
              "raster_bwd: bad args");
  VSX_REQUIRE(!g_depth || depth, "raster_bwd: depth cotangent needs the depth image");
  BwdArgs a{rec, tile_offsets, tile_list, alpha, depth, raw_normal, t_final, g_rgb, g_alpha,
            g_depth, g_normal, g_raw_normal, n_contrib, grad_splat, rgb, nullptr, {}};
  return launch_bwd(a, cam, as_stream(s));
}

extern "C" int vsx_raster_bwd_loss(const vsx_splat *rec, const uint32_t *tile_offsets,
                                   const uint32_t *tile_list, vsx_camera cam, const float *rgb,
                                   const float *alpha, const float *depth, const float *normal,
                                   const float *raw_normal, const float *t_final,
                                   const int32_t *n_contrib, vsx_loss_desc loss,
                                   float *grad_splat, vsx_stream s) {
  VSX_REQUIRE(cam.width > 0 && cam.height > 0 && rgb && alpha && depth && normal && raw_normal &&
                  t_final && n_contrib && loss.gt_rgb && loss.counts,
              "raster_bwd_loss: bad args");
  BwdArgs a{rec, tile_offsets, tile_list, alpha, depth, raw_normal, t_final, nullptr, nullptr,
            nullptr, nullptr, nullptr, n_contrib, grad_splat, rgb, normal, loss};
  return launch_bwd(a, cam, as_stream(s));
}
