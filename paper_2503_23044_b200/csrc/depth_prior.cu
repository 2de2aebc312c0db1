// f1 — monocular depth-prior precompute (voxsplat depth_prior.py:85-214).
//
// The per-point and per-pixel float64 passes of the prior pipeline:
//   vsx_prior_sample        projection of the sparse points + bilinear sampling
//                           of the raw depth (fit_scale_shift, :85-110)
//   vsx_apply_scale_shift   metric = s * raw + b, masked (apply_scale_shift, :132-140)
//   vsx_reprojection_error  lift -> project -> resample -> lift -> project back
//                           round-trip error per source pixel (:143-187),
//                           optionally min-accumulated over neighbours (enhance)
//   vsx_enhance_finalize    keep pixels with min round-trip <= tau (:205-214)
// Arithmetic is float64 with explicit rounding, in the reference's operation
// order (numpy elementwise ops, BLAS dot order for the 3x3 products), so the
// masks agree with the reference up to ties at the tau / bounds comparisons.
#include "common.cuh"

namespace vsx {

constexpr double kZEps = 1e-9;  // depth_prior.py Z_EPS

// _bilinear_with_valid (depth_prior.py:62-74): sample requiring all four
// touched texels valid; u0 / v0 clipped to [0, w-2] / [0, h-2].
__device__ __forceinline__ double bilinear_valid(const double *__restrict__ vals,
                                                 const uint8_t *__restrict__ valid, int w, int h,
                                                 double u, double v, bool &ok) {
  const long long u0 = (long long)fmin(fmax(floor(u), 0.0), (double)(w - 2));
  const long long v0 = (long long)fmin(fmax(floor(v), 0.0), (double)(h - 2));
  const double fu = dsub(u, (double)u0), fv = dsub(v, (double)v0);
  const size_t i00 = (size_t)v0 * w + u0, i10 = i00 + w;
  ok = valid[i00] && valid[i00 + 1] && valid[i10] && valid[i10 + 1];
  const double gu = dsub(1.0, fu), gv = dsub(1.0, fv);
  double s = dmul(dmul(vals[i00], gu), gv);
  s = dadd(s, dmul(dmul(vals[i00 + 1], fu), gv));
  s = dadd(s, dmul(dmul(vals[i10], gu), fv));
  s = dadd(s, dmul(dmul(vals[i10 + 1], fu), fv));
  return s;
}

__global__ void prior_sample_kernel(const double *__restrict__ pts, int64_t n, vsx_camera cam,
                                    const double *__restrict__ depth,
                                    const uint8_t *__restrict__ valid, double *__restrict__ raw,
                                    double *__restrict__ zout, uint8_t *__restrict__ ok_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y, z;
  cam_transform(cam, pts[3 * i + 0], pts[3 * i + 1], pts[3 * i + 2], x, y, z);
  uint8_t ok = 0;
  double r = 0.0;
  if (z > kZEps) {
    const double u = dadd(ddiv(dmul(cam.fx, x), z), cam.cx);
    const double v = dadd(ddiv(dmul(cam.fy, y), z), cam.cy);
    if (u >= 0.0 && u <= (double)(cam.width - 1) && v >= 0.0 && v <= (double)(cam.height - 1)) {
      bool vok;
      r = bilinear_valid(depth, valid, cam.width, cam.height, u, v, vok);
      ok = vok ? 2 : 1;  // 1 = projected in bounds, 2 = and sampled on valid depth
    }
  }
  raw[i] = r;
  zout[i] = z;
  ok_out[i] = ok;
}

__global__ void apply_scale_shift_kernel(const double *__restrict__ raw,
                                         const uint8_t *__restrict__ valid, int64_t n, double s,
                                         double b, double *__restrict__ out,
                                         uint8_t *__restrict__ out_valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = raw[i];
  const bool v0 = valid ? valid[i] != 0 : (isfinite(d) && d > 0.0);
  const double m = dadd(dmul(s, d), b);
  const bool ok = v0 && isfinite(m) && m > 0.0;
  out[i] = ok ? m : 0.0;
  out_valid[i] = ok ? 1 : 0;
}

// Round trip of every valid source pixel through the reference view
// (depth_prior.py:143-187). err = +inf where the chain breaks. With
// accumulate != 0 the result is min-combined into err (enhance's emin).
__global__ void reprojection_error_kernel(const double *__restrict__ sv,
                                          const uint8_t *__restrict__ sok, vsx_camera vs,
                                          const double *__restrict__ rv,
                                          const uint8_t *__restrict__ rok, vsx_camera vr,
                                          double *__restrict__ err, int accumulate) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int w = vs.width, h = vs.height;
  if (p >= (int64_t)w * h) return;
  const int uu = (int)(p % w), vv = (int)(p / w);
  double e = INFINITY;
  if (sok[p]) {
    const double z = sv[p];
    const double x = dmul(ddiv(dsub((double)uu, vs.cx), vs.fx), z);
    const double y = dmul(ddiv(dsub((double)vv, vs.cy), vs.fy), z);
    // world = (cam_src - t) @ r
    const double c0 = dsub(x, vs.t[0]), c1 = dsub(y, vs.t[1]), c2 = dsub(z, vs.t[2]);
    const double wx = dot3_blas(c0, c1, c2, vs.r[0], vs.r[3], vs.r[6]);
    const double wy = dot3_blas(c0, c1, c2, vs.r[1], vs.r[4], vs.r[7]);
    const double wz = dot3_blas(c0, c1, c2, vs.r[2], vs.r[5], vs.r[8]);
    double rx, ry, rz;
    cam_transform(vr, wx, wy, wz, rx, ry, rz);
    bool ok = rz > kZEps;
    if (ok) {
      const double ur = dadd(ddiv(dmul(vr.fx, rx), rz), vr.cx);
      const double vrp = dadd(ddiv(dmul(vr.fy, ry), rz), vr.cy);
      ok = ur >= 0.0 && ur <= (double)(vr.width - 1) && vrp >= 0.0 &&
           vrp <= (double)(vr.height - 1);
      if (ok) {
        bool sok2;
        const double zs = bilinear_valid(rv, rok, vr.width, vr.height, ur, vrp, sok2);
        ok = sok2 && zs > 0.0;
        if (ok) {
          const double xr = dmul(ddiv(dsub(ur, vr.cx), vr.fx), zs);
          const double yr = dmul(ddiv(dsub(vrp, vr.cy), vr.fy), zs);
          const double d0 = dsub(xr, vr.t[0]), d1 = dsub(yr, vr.t[1]), d2 = dsub(zs, vr.t[2]);
          const double qx = dot3_blas(d0, d1, d2, vr.r[0], vr.r[3], vr.r[6]);
          const double qy = dot3_blas(d0, d1, d2, vr.r[1], vr.r[4], vr.r[7]);
          const double qz = dot3_blas(d0, d1, d2, vr.r[2], vr.r[5], vr.r[8]);
          double sx, sy, sz;
          cam_transform(vs, qx, qy, qz, sx, sy, sz);
          ok = sz > kZEps;
          if (ok) {
            const double u2 = dadd(ddiv(dmul(vs.fx, sx), sz), vs.cx);
            const double v2 = dadd(ddiv(dmul(vs.fy, sy), sz), vs.cy);
            e = hypot(dsub(u2, (double)uu), dsub(v2, (double)vv));
          }
        }
      }
    }
  }
  err[p] = accumulate ? fmin(err[p], e) : e;
}

__global__ void enhance_finalize_kernel(const double *__restrict__ vals,
                                        const uint8_t *__restrict__ valid,
                                        const double *__restrict__ emin, double tau, int64_t n,
                                        double *__restrict__ out, uint8_t *__restrict__ out_valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool ok = valid[i] && emin[i] <= tau;
  out[i] = ok ? vals[i] : 0.0;
  out_valid[i] = ok ? 1 : 0;
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_prior_sample(const double *points, int64_t n, vsx_camera cam,
                                const double *depth, const uint8_t *valid, double *raw,
                                double *z, uint8_t *ok, vsx_stream s) {
  VSX_REQUIRE(n >= 0 && cam.width >= 2 && cam.height >= 2, "prior_sample: bad arguments");
  if (n == 0) return VSX_OK;
  prior_sample_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(points, n, cam, depth, valid,
                                                                  raw, z, ok);
  VSX_LAUNCH_CHECK("prior_sample");
  return VSX_OK;
}

extern "C" int vsx_apply_scale_shift(const double *raw, const uint8_t *valid, int64_t n,
                                     double scale, double shift, double *out, uint8_t *out_valid,
                                     vsx_stream s) {
  VSX_REQUIRE(n >= 0, "apply_scale_shift: bad n");
  if (n == 0) return VSX_OK;
  apply_scale_shift_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(raw, valid, n, scale,
                                                                       shift, out, out_valid);
  VSX_LAUNCH_CHECK("apply_scale_shift");
  return VSX_OK;
}

extern "C" int vsx_reprojection_error(const double *src, const uint8_t *src_valid,
                                      vsx_camera view_src, const double *ref,
                                      const uint8_t *ref_valid, vsx_camera view_ref,
                                      double *err, int32_t accumulate_min, vsx_stream s) {
  VSX_REQUIRE(view_src.width >= 1 && view_src.height >= 1 && view_ref.width >= 2 &&
                  view_ref.height >= 2,
              "reprojection_error: bad view sizes");
  const int64_t n = (int64_t)view_src.width * view_src.height;
  reprojection_error_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      src, src_valid, view_src, ref, ref_valid, view_ref, err, accumulate_min);
  VSX_LAUNCH_CHECK("reprojection_error");
  return VSX_OK;
}

extern "C" int vsx_enhance_finalize(const double *src, const uint8_t *src_valid,
                                    const double *emin, double tau, int64_t n, double *out,
                                    uint8_t *out_valid, vsx_stream s) {
  VSX_REQUIRE(tau > 0.0, "enhance: tau must be positive");
  VSX_REQUIRE(n >= 0, "enhance: bad n");
  if (n == 0) return VSX_OK;
  enhance_finalize_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(src, src_valid, emin, tau,
                                                                      n, out, out_valid);
  VSX_LAUNCH_CHECK("enhance_finalize");
  return VSX_OK;
}
