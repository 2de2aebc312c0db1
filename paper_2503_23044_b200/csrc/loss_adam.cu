// K9 — photometric / depth L1 losses with fused cotangents, and
// K10 — one-launch fused Adam over every parameter group.
//
// bl_rgb_loss restates voxsplat losses.py:43-53 (mean over views of mean
// |I_hat - I|; d/dI_hat = sign(diff) / (B*H*W*3), sign(0) = 0).
// e_depth_loss restates losses.py:65-84 (masked L1 over prior-valid &
// render-valid pixels, per-view mean, batch mean).
// Adam restates trainer.py:220-247 (bias-corrected, eps 1e-15), dense: every
// element moves every step, including zero-gradient anchors.
#include "common.cuh"

namespace vsx {

__device__ __forceinline__ float signf_(float d) { return d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f); }

__global__ void __launch_bounds__(256) l1_kernel(const float *__restrict__ r,
                                                 const float *__restrict__ g, int64_t n,
                                                 float scale, double *__restrict__ loss,
                                                 float *__restrict__ grad) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float d = r[i] - g[i];
    acc += fabs((double)d);
    if (grad) grad[i] = signf_(d) * scale;
  }
  acc = warp_sum_d(acc);
  __shared__ double ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < 8 ? ws[threadIdx.x] : 0.0;
    v = warp_sum_d(v);
    if (threadIdx.x == 0) atomicAdd(loss, v);
  }
}

__global__ void __launch_bounds__(256) depth_l1_kernel(
    const float *__restrict__ d, const uint8_t *__restrict__ valid, const float *__restrict__ p,
    const uint8_t *__restrict__ pv, int64_t n, double *__restrict__ sums,
    uint32_t *__restrict__ counts, const float *__restrict__ scale, float *__restrict__ grad) {
  double acc = 0.0;
  uint32_t cnt = 0;
  const float sc = (grad && scale) ? *scale : 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool m = valid[i] && pv[i];
    const float diff = d[i] - p[i];
    if (m) {
      acc += fabs((double)diff);
      ++cnt;
    }
    if (grad) grad[i] = m ? signf_(diff) * sc : 0.f;
  }
  acc = warp_sum_d(acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) {
    if (sums) atomicAdd(sums, acc);
    if (counts) atomicAdd(counts, cnt);
  }
}

// Masked multi-channel L1 (normal-prior term, same masking rule as the depth
// term): mask = valid & prior_valid per pixel, |x - p| summed over channels.
__global__ void __launch_bounds__(256) masked_l1_kernel(
    const float *__restrict__ x, const uint8_t *__restrict__ valid, const float *__restrict__ p,
    const uint8_t *__restrict__ pv, int64_t n_pix, int channels, double *__restrict__ sums,
    uint32_t *__restrict__ counts, const float *__restrict__ scale, float *__restrict__ grad) {
  double acc = 0.0;
  uint32_t cnt = 0;
  const float sc = (grad && scale) ? *scale : 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool m = valid[i] && pv[i];
    cnt += m ? 1u : 0u;
    for (int c = 0; c < channels; ++c) {
      const int64_t j = i * channels + c;
      const float diff = x[j] - p[j];
      if (m) acc += fabs((double)diff);
      if (grad) grad[j] = m ? signf_(diff) * sc : 0.f;
    }
  }
  acc = warp_sum_d(acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) {
    if (sums) atomicAdd(sums, acc);
    if (counts) atomicAdd(counts, cnt);
  }
}

constexpr int kMaxSeg = 16;
struct AdamSegs {
  int64_t begin[kMaxSeg + 1];
  double lr[kMaxSeg];
  int n;
};

// One thread per 4 consecutive parameters (segments start on 16-byte
// boundaries, so a float4 never straddles two learning-rate groups): three
// float4 loads + one scalar-free update + three float4 stores. The moment
// updates run in float32 (the parameters are float32; relative error ~1e-7
// of a step); the bias corrections come in from the host in float64.
__global__ void __launch_bounds__(256) adam_kernel(float *__restrict__ p,
                                                   const float *__restrict__ g,
                                                   float *__restrict__ m, float *__restrict__ v,
                                                   AdamSegs segs, double b1, double b2, double eps,
                                                   double bc1, double bc2,
                                                   const int32_t *__restrict__ guard) {
  if (guard && *guard) return;  // non-finite step: parameters and moments untouched
  const int64_t total = segs.begin[segs.n];
  const int64_t n4 = total >> 2;
  const float fb1 = (float)b1, fb2 = (float)b2, c1 = (float)(1.0 - b1), c2 = (float)(1.0 - b2);
  const float ibc1 = (float)(1.0 / bc1), ibc2 = (float)(1.0 / bc2), feps = (float)eps;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q << 2;
    int s = 0;
    while (s + 1 < segs.n && i >= segs.begin[s + 1]) ++s;
    const float lr = (float)segs.lr[s];
    const float4 gi = reinterpret_cast<const float4 *>(g)[q];
    float4 mi = reinterpret_cast<const float4 *>(m)[q];
    float4 vi = reinterpret_cast<const float4 *>(v)[q];
    float4 pi = reinterpret_cast<const float4 *>(p)[q];
    auto upd = [&](float gg, float &mm, float &vv, float &pp) {
      mm = fb1 * mm + c1 * gg;
      vv = fb2 * vv + c2 * gg * gg;
      pp = pp - lr * (mm * ibc1) / (sqrtf(vv * ibc2) + feps);
    };
    upd(gi.x, mi.x, vi.x, pi.x);
    upd(gi.y, mi.y, vi.y, pi.y);
    upd(gi.z, mi.z, vi.z, pi.z);
    upd(gi.w, mi.w, vi.w, pi.w);
    reinterpret_cast<float4 *>(m)[q] = mi;
    reinterpret_cast<float4 *>(v)[q] = vi;
    reinterpret_cast<float4 *>(p)[q] = pi;
  }
  // tail (total % 4) elements
  const int64_t t0 = n4 << 2;
  const int64_t i = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && i < total) {
    int s = 0;
    while (s + 1 < segs.n && i >= segs.begin[s + 1]) ++s;
    const float lr = (float)segs.lr[s];
    float mm = m[i], vv = v[i];
    const float gg = g[i];
    mm = fb1 * mm + c1 * gg;
    vv = fb2 * vv + c2 * gg * gg;
    m[i] = mm;
    v[i] = vv;
    p[i] = p[i] - lr * (mm * ibc1) / (sqrtf(vv * ibc2) + feps);
  }
}

}  // namespace vsx

using namespace vsx;

static int persistent_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min(grid_for(n, 256), sms * 8));
}

extern "C" int vsx_l1_loss(const float *rendered, const float *target, int64_t n, float scale,
                           double *loss_accum, float *grad, vsx_stream s) {
  VSX_REQUIRE(n >= 0 && loss_accum, "l1_loss: bad args");
  if (n == 0) return VSX_OK;
  l1_kernel<<<persistent_grid(n), 256, 0, as_stream(s)>>>(rendered, target, n, scale, loss_accum,
                                                          grad);
  VSX_LAUNCH_CHECK("l1_loss");
  return VSX_OK;
}

extern "C" int vsx_depth_loss(const float *depth, const uint8_t *valid, const float *prior,
                              const uint8_t *prior_valid, int64_t n, double *sums,
                              uint32_t *counts, const float *scale, float *grad, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "depth_loss: bad args");
  if (n == 0) return VSX_OK;
  depth_l1_kernel<<<persistent_grid(n), 256, 0, as_stream(s)>>>(depth, valid, prior, prior_valid,
                                                                n, sums, counts, scale, grad);
  VSX_LAUNCH_CHECK("depth_loss");
  return VSX_OK;
}

extern "C" int vsx_masked_l1(const float *x, const uint8_t *valid, const float *prior,
                             const uint8_t *prior_valid, int64_t n_pix, int32_t channels,
                             double *sums, uint32_t *counts, const float *scale, float *grad,
                             vsx_stream s) {
  VSX_REQUIRE(n_pix >= 0 && channels >= 1, "masked_l1: bad args");
  if (n_pix == 0) return VSX_OK;
  masked_l1_kernel<<<persistent_grid(n_pix), 256, 0, as_stream(s)>>>(
      x, valid, prior, prior_valid, n_pix, channels, sums, counts, scale, grad);
  VSX_LAUNCH_CHECK("masked_l1");
  return VSX_OK;
}

static int adam_impl(float *param, const float *grad, float *m, float *v, int32_t n_seg,
                     const int64_t *seg_begin, const double *lr, double beta1, double beta2,
                     double eps, int32_t step, const int32_t *guard, vsx_stream s) {
  VSX_REQUIRE(((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) |
                reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0,
              "adam: buffers must be 16-byte aligned");
  VSX_REQUIRE(n_seg >= 1 && n_seg <= kMaxSeg, "adam: 1..16 segments");
  AdamSegs segs{};
  segs.n = n_seg;
  for (int i = 0; i <= n_seg; ++i) segs.begin[i] = seg_begin[i];
  for (int i = 0; i < n_seg; ++i) {
    VSX_REQUIRE(seg_begin[i + 1] >= seg_begin[i], "adam: segments must be ascending");
    VSX_REQUIRE(seg_begin[i] % 4 == 0, "adam: segment %d must start on a 16-byte boundary", i);
    segs.lr[i] = lr[i];
  }
  const int64_t total = seg_begin[n_seg];
  if (total == 0) return VSX_OK;
  const int t = step + 1;
  const double bc1 = 1.0 - pow(beta1, (double)t), bc2 = 1.0 - pow(beta2, (double)t);
  adam_kernel<<<persistent_grid(total), 256, 0, as_stream(s)>>>(param, grad, m, v, segs, beta1,
                                                                beta2, eps, bc1, bc2, guard);
  VSX_LAUNCH_CHECK("adam");
  return VSX_OK;
}

extern "C" int vsx_adam(float *param, const float *grad, float *m, float *v, int32_t n_seg,
                        const int64_t *seg_begin, const double *lr, double beta1, double beta2,
                        double eps, int32_t step, vsx_stream s) {
  return adam_impl(param, grad, m, v, n_seg, seg_begin, lr, beta1, beta2, eps, step, nullptr, s);
}

extern "C" int vsx_adam_guarded(float *param, const float *grad, float *m, float *v,
                                int32_t n_seg, const int64_t *seg_begin, const double *lr,
                                double beta1, double beta2, double eps, int32_t step,
                                const int32_t *guard, vsx_stream s) {
  VSX_REQUIRE(guard, "adam_guarded: guard is required");
  return adam_impl(param, grad, m, v, n_seg, seg_begin, lr, beta1, beta2, eps, step, guard, s);
}
