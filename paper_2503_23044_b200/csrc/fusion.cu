// f4 — TSDF integration of a depth map into a dense volume
// (voxsplat fusion.py:102-133, TsdfVolume.integrate).
//
// One thread per voxel, float64 with the reference's operation order: the
// voxel centre (origin + index * voxel_size) is moved to the camera frame
// (BLAS dot order), projected, rounded half-to-even to the nearest pixel, and
// when the stored depth is valid, positive and not more than one truncation
// band in front of the voxel, the clamped, normalised signed distance is
// folded into the per-voxel running average. The voxel count touched is
// reduced per block and added to *touched.
#include "common.cuh"

namespace vsx {

constexpr double kFusionZEps = 1e-9;

__global__ void tsdf_integrate_kernel(double *__restrict__ tsdf, double *__restrict__ weight,
                                      int64_t d0, int64_t d1, int64_t d2, double ox, double oy,
                                      double oz, double vs, double trunc,
                                      const double *__restrict__ depth,
                                      const uint8_t *__restrict__ valid, vsx_camera cam,
                                      unsigned long long *__restrict__ touched) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool hit = false;
  if (idx < d0 * d1 * d2) {
    const int64_t i = idx / (d1 * d2), j = (idx / d2) % d1, k = idx % d2;
    const double px = dadd(ox, dmul((double)i, vs));
    const double py = dadd(oy, dmul((double)j, vs));
    const double pz = dadd(oz, dmul((double)k, vs));
    double x, y, z;
    cam_transform(cam, px, py, pz, x, y, z);
    if (z > kFusionZEps) {
      const double u = rint(dadd(ddiv(dmul(cam.fx, x), z), cam.cx));
      const double v = rint(dadd(ddiv(dmul(cam.fy, y), z), cam.cy));
      if (u >= 0.0 && u < (double)cam.width && v >= 0.0 && v < (double)cam.height) {
        const size_t p = (size_t)v * cam.width + (size_t)u;
        const double dd = depth[p];
        if (valid[p] && dd > 0.0) {
          const double sdf = dsub(dd, z);
          if (sdf >= -trunc) {
            const double val = ddiv(fmin(fmax(sdf, -trunc), trunc), trunc);
            const double w = weight[idx];
            tsdf[idx] = ddiv(dadd(dmul(tsdf[idx], w), val), dadd(w, 1.0));
            weight[idx] = dadd(w, 1.0);
            hit = true;
          }
        }
      }
    }
  }
  const unsigned c = __popc(__ballot_sync(0xffffffffu, hit));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(touched, (unsigned long long)c);
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_tsdf_integrate(double *tsdf, double *weight, const int64_t *dims,
                                  const double *origin, double voxel_size, double truncation,
                                  const double *depth, const uint8_t *valid, vsx_camera cam,
                                  unsigned long long *touched, vsx_stream s) {
  VSX_REQUIRE(dims[0] >= 2 && dims[1] >= 2 && dims[2] >= 2 && voxel_size > 0 &&
                  truncation >= voxel_size,
              "tsdf_integrate: bad volume");
  const int64_t n = dims[0] * dims[1] * dims[2];
  tsdf_integrate_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      tsdf, weight, dims[0], dims[1], dims[2], origin[0], origin[1], origin[2], voxel_size,
      truncation, depth, valid, cam, touched);
  VSX_LAUNCH_CHECK("tsdf_integrate");
  return VSX_OK;
}
