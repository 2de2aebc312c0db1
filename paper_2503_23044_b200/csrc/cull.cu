// K1 — per-view frustum + LoD anchor culling.
//
// Restates voxsplat scene.py:239-259 (active_mask) and :232-236
// (lod_for_distance) over the level-major concatenation of all levels. All
// arithmetic is float64 with explicit rounding so the mask is bit-exact
// against the numpy reference. HBM-bound: 24 B centre + 4 B level in,
// 1 B mask out per anchor.
#include "common.cuh"

namespace vsx {

__global__ void __launch_bounds__(256) cull_kernel(const double *__restrict__ centers,
                                                   const int32_t *__restrict__ level, int64_t n,
                                                   int32_t lod_count, double lod_ref,
                                                   int32_t lod_bias, vsx_camera cam,
                                                   uint8_t *__restrict__ mask) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double cx = centers[3 * i + 0], cy = centers[3 * i + 1], cz = centers[3 * i + 2];
  double px, py, pz;
  cam_transform(cam, cx, cy, cz, px, py, pz);
  const bool front = pz > 1e-9;
  const double zs = front ? pz : 1.0;
  const double u = front ? dadd(ddiv(dmul(cam.fx, px), zs), cam.cx) : -1e9;
  const double v = front ? dadd(ddiv(dmul(cam.fy, py), zs), cam.cy) : -1e9;
  const double mx = dmul(0.1, (double)cam.width), my = dmul(0.1, (double)cam.height);
  const bool inside = front && u >= -mx && u <= dadd((double)cam.width, mx) && v >= -my &&
                      v <= dadd((double)cam.height, my);
  const double dx = dsub(cx, cam.center[0]), dy = dsub(cy, cam.center[1]),
               dz = dsub(cz, cam.center[2]);
  double dist = sqrt(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
  dist = fmax(dist, 1e-12);
  double lod = floor(dadd(log2(ddiv(lod_ref, dist)), (double)lod_bias));
  lod = fmin(fmax(lod, 0.0), (double)(lod_count - 1));
  mask[i] = (inside && (int)lod == level[i]) ? 1 : 0;
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_cull(const double *centers, const int32_t *level, int64_t n_anchors,
                        int32_t lod_count, double lod_ref, int32_t lod_bias, vsx_camera cam,
                        uint8_t *mask, vsx_stream s) {
  VSX_REQUIRE(n_anchors >= 0 && lod_count >= 1 && lod_ref > 0, "cull: bad arguments");
  if (n_anchors == 0) return VSX_OK;
  cull_kernel<<<grid_for(n_anchors, 256), 256, 0, as_stream(s)>>>(
      centers, level, n_anchors, lod_count, lod_ref, lod_bias, cam, mask);
  VSX_LAUNCH_CHECK("cull");
  return VSX_OK;
}
