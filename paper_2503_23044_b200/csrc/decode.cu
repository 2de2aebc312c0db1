// K2 / K8 — shared anchor decoder (3 tanh MLP heads 36 -> 64 -> {n,3n,7n}).
//
// Forward restates voxsplat decoder.py:142-180 (decode_inputs, _head_forward,
// decode_arrays) for the active anchors of one view, emitting gaussians in the
// canonical (anchor, slot) order of decode_active (decoder.py:210-250).
// Backward restates the autograd of that graph (decoder.py:267-292): an
// anchor-parallel kernel producing head-output and pre-activation cotangents
// plus per-anchor grads, then K-reduction GEMMs for the weight gradients.
//
// Layouts: per-anchor caches are FEATURE-major ([feature][anchor]) so warps
// read/write them coalesced and the weight-gradient reductions stream them.
#include "common.cuh"

namespace vsx {

struct DecSmem {
  // W1cat [36][192] (head h -> columns h*64..h*64+63), b1cat [192],
  // W2T per head [out_h][64] (transposed), b2cat [11n]
  float *w1, *b1, *w2t, *b2;
};

__host__ __device__ inline int dec_out_width(int n) { return 11 * n; }
__host__ __device__ inline int dec_head_off(int h, int n) { return h == 0 ? 0 : (h == 1 ? n : 4 * n); }
__host__ __device__ inline int dec_head_w(int h, int n) { return h == 0 ? n : (h == 1 ? 3 * n : 7 * n); }

inline size_t dec_smem_bytes(int n) {
  return sizeof(float) * (size_t)(kInDim * 192 + 192 + 64 * 11 * n + 11 * n);
}

__device__ __forceinline__ DecSmem dec_smem_carve(float *base, int n) {
  DecSmem s;
  s.w1 = base;
  s.b1 = s.w1 + kInDim * 192;
  s.w2t = s.b1 + 192;
  s.b2 = s.w2t + 64 * 11 * n;
  return s;
}

__device__ void dec_load_weights(const vsx_decoder &W, DecSmem s) {
  const int n = W.n;
  for (int h = 0; h < 3; ++h) {
    const int ow = dec_head_w(h, n), oo = dec_head_off(h, n);
    for (int e = threadIdx.x; e < kInDim * 64; e += blockDim.x) {
      const int i = e / 64, k = e % 64;
      s.w1[i * 192 + h * 64 + k] = W.w1[h][e];
    }
    for (int k = threadIdx.x; k < 64; k += blockDim.x) s.b1[h * 64 + k] = W.b1[h][k];
    for (int e = threadIdx.x; e < 64 * ow; e += blockDim.x) {
      const int k = e / ow, j = e % ow;  // w2 is (64, ow) row-major
      s.w2t[(oo + j) * 64 + k] = W.w2[h][e];
    }
    for (int j = threadIdx.x; j < ow; j += blockDim.x) s.b2[oo + j] = W.b2[h][j];
  }
  __syncthreads();
}

// Input block x = [emb | d/ref | (c - cam)/d] (decoder.py:142-147), float64
// geometry rounded to float32 for the MLP.
__device__ __forceinline__ void dec_inputs(const double *centers, const float *emb, int a,
                                           const vsx_camera &cam, double lod_ref, float *x) {
  const double rx = dsub(centers[3 * a + 0], cam.center[0]);
  const double ry = dsub(centers[3 * a + 1], cam.center[1]);
  const double rz = dsub(centers[3 * a + 2], cam.center[2]);
  double d = sqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), dmul(rz, rz)));
  d = fmax(d, 1e-12);
  const float4 *e4 = reinterpret_cast<const float4 *>(emb + (size_t)a * kEmbed);
#pragma unroll
  for (int q = 0; q < kEmbed / 4; ++q) {
    const float4 v = e4[q];
    x[4 * q + 0] = v.x;
    x[4 * q + 1] = v.y;
    x[4 * q + 2] = v.z;
    x[4 * q + 3] = v.w;
  }
  x[32] = (float)ddiv(d, lod_ref);
  x[33] = (float)ddiv(rx, d);
  x[34] = (float)ddiv(ry, d);
  x[35] = (float)ddiv(rz, d);
}

// hid[0:64] = W1_h^T x + b1_h (pre-activation)
__device__ __forceinline__ void dec_hidden(const DecSmem &s, int h, const float *x, float *hid) {
#pragma unroll
  for (int k = 0; k < 64; ++k) hid[k] = s.b1[h * 64 + k];
#pragma unroll
  for (int i = 0; i < kInDim; ++i) {
    const float xi = x[i];
    const float4 *w = reinterpret_cast<const float4 *>(s.w1 + i * 192 + h * 64);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const float4 wv = w[q];
      hid[4 * q + 0] = fmaf(xi, wv.x, hid[4 * q + 0]);
      hid[4 * q + 1] = fmaf(xi, wv.y, hid[4 * q + 1]);
      hid[4 * q + 2] = fmaf(xi, wv.z, hid[4 * q + 2]);
      hid[4 * q + 3] = fmaf(xi, wv.w, hid[4 * q + 3]);
    }
  }
}

__device__ __forceinline__ float dec_out(const DecSmem &s, int col, const float *hid) {
  const float4 *w = reinterpret_cast<const float4 *>(s.w2t + col * 64);
  float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
  for (int q = 0; q < 16; q += 2) {
    const float4 a = w[q], b = w[q + 1];
    acc0 = fmaf(hid[4 * q + 0], a.x, acc0);
    acc0 = fmaf(hid[4 * q + 1], a.y, acc0);
    acc0 = fmaf(hid[4 * q + 2], a.z, acc0);
    acc0 = fmaf(hid[4 * q + 3], a.w, acc0);
    acc1 = fmaf(hid[4 * q + 4], b.x, acc1);
    acc1 = fmaf(hid[4 * q + 5], b.y, acc1);
    acc1 = fmaf(hid[4 * q + 6], b.z, acc1);
    acc1 = fmaf(hid[4 * q + 7], b.w, acc1);
  }
  return s.b2[col] + (acc0 + acc1);
}

__device__ __forceinline__ float sigmoidf_(float v) { return 1.0f / (1.0f + expf(-v)); }

__global__ void __launch_bounds__(128) decode_fwd_kernel(
    vsx_decoder W, const int32_t *__restrict__ active, int32_t n_active,
    const double *__restrict__ centers, const float *__restrict__ emb,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, vsx_camera cam,
    double lod_ref, double max_scale, double *__restrict__ means, float *__restrict__ opacity,
    float *__restrict__ color, float *__restrict__ scale, float *__restrict__ quat,
    float *__restrict__ normal, float *__restrict__ cache_h, float *__restrict__ cache_o,
    int32_t *__restrict__ status) {
  extern __shared__ __align__(16) float smem[];
  const int n = W.n;
  DecSmem s = dec_smem_carve(smem, n);
  dec_load_weights(W, s);
  const float smax = (float)max_scale, smin = (float)kMinScale;
  const size_t ld = cache_ld(n_active);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_active; r += gridDim.x * blockDim.x) {
    const int a = active[r];
    float x[kInDim];
    dec_inputs(centers, emb, a, cam, lod_ref, x);
    bool bad = false;
    float hid[64];
    // opacity head
    dec_hidden(s, 0, x, hid);
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      hid[k] = tanhf(hid[k]);
      if (cache_h) cache_h[(size_t)k * ld + r] = hid[k];
    }
    for (int j = 0; j < n; ++j) {
      const float o = dec_out(s, j, hid);
      if (cache_o) cache_o[(size_t)j * ld + r] = o;
      const float op = sigmoidf_(o);
      bad |= !isfinite(op);
      opacity[(size_t)r * n + j] = op;
    }
    // color head
    dec_hidden(s, 1, x, hid);
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      hid[k] = tanhf(hid[k]);
      if (cache_h) cache_h[(size_t)(64 + k) * ld + r] = hid[k];
    }
    for (int j = 0; j < 3 * n; ++j) {
      const float o = dec_out(s, n + j, hid);
      if (cache_o) cache_o[(size_t)(n + j) * ld + r] = o;
      const float c = sigmoidf_(o);
      bad |= !isfinite(c);
      color[(size_t)r * 3 * n + j] = c;
    }
    // covariance head: per slot 3 log-scales + 4 raw quaternion entries
    dec_hidden(s, 2, x, hid);
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      hid[k] = tanhf(hid[k]);
      if (cache_h) cache_h[(size_t)(128 + k) * ld + r] = hid[k];
    }
    const double l0 = exp((double)log_scale[3 * a + 0]);
    const double l1 = exp((double)log_scale[3 * a + 1]);
    const double l2 = exp((double)log_scale[3 * a + 2]);
    for (int sl = 0; sl < n; ++sl) {
      float o[7];
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        o[c] = dec_out(s, 4 * n + 7 * sl + c, hid);
        if (cache_o) cache_o[(size_t)(4 * n + 7 * sl + c) * ld + r] = o[c];
      }
      const size_t g = (size_t)r * n + sl;
      float sc[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        sc[c] = fminf(fmaxf(expf(o[c]), smin), smax);
        scale[3 * g + c] = sc[c];
      }
      float qw = o[3] + 1.0f, qx = o[4], qy = o[5], qz = o[6];
      const float qn = fmaxf(sqrtf(qw * qw + qx * qx + qy * qy + qz * qz), 1e-12f);
      qw /= qn;
      qx /= qn;
      qy /= qn;
      qz /= qn;
      quat[4 * g + 0] = qw;
      quat[4 * g + 1] = qx;
      quat[4 * g + 2] = qy;
      quat[4 * g + 3] = qz;
      float R[9];
      quat_to_rot(qw, qx, qy, qz, R);
      const int ax = argmin3(sc[0], sc[1], sc[2]);
      normal[3 * g + 0] = R[0 + ax];
      normal[3 * g + 1] = R[3 + ax];
      normal[3 * g + 2] = R[6 + ax];
      const float *off = offsets + ((size_t)a * n + sl) * 3;
      const double m0 = dadd(centers[3 * a + 0], dmul((double)off[0], l0));
      const double m1 = dadd(centers[3 * a + 1], dmul((double)off[1], l1));
      const double m2 = dadd(centers[3 * a + 2], dmul((double)off[2], l2));
      means[3 * g + 0] = m0;
      means[3 * g + 1] = m1;
      means[3 * g + 2] = m2;
      bad |= !(isfinite(sc[0]) && isfinite(sc[1]) && isfinite(sc[2]) && isfinite(qw) &&
               isfinite(qx) && isfinite(qy) && isfinite(qz) && isfinite(m0) && isfinite(m1) &&
               isfinite(m2));
    }
    if (bad) atomicOr(status, VSX_STATUS_NONFINITE);
  }
}

// ---------------------------------------------------------------- backward

// dR/dq contraction: gq += sum_ij G_ij dR_ij/dq (row-major R of quat_to_rot).
__device__ __forceinline__ void rot_vjp(float w, float x, float y, float z, const float *G,
                                        float *gq) {
  gq[0] += 2.f * (-z * G[1] + y * G[2] + z * G[3] - x * G[5] - y * G[6] + x * G[7]);
  gq[1] += 2.f * (y * G[1] + z * G[2] + y * G[3] - 2.f * x * G[4] - w * G[5] + z * G[6] +
                  w * G[7] - 2.f * x * G[8]);
  gq[2] += 2.f * (-2.f * y * G[0] + x * G[1] + w * G[2] + x * G[3] + z * G[5] - w * G[6] +
                  z * G[7] - 2.f * y * G[8]);
  gq[3] += 2.f * (-2.f * z * G[0] - w * G[1] + x * G[2] + w * G[3] - 2.f * z * G[4] +
                  y * G[5] + x * G[6] + y * G[7]);
}

// Growth pressure (trainer.py:342-349): per active anchor r, the float64 sum
// of |dL/dmu| over its n gaussians (batch order g = r*n + sl) and n counts,
// added into the flat per-anchor accumulators. One thread per anchor; an
// anchor occurs once per view, so the adds do not contend.
__global__ void growth_accumulate_kernel(const float *__restrict__ g_means,
                                         const int32_t *__restrict__ active, int32_t n_active,
                                         int n, double *__restrict__ grow_sum,
                                         double *__restrict__ grow_cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_active) return;
  const float *gm = g_means + (size_t)r * n * 3;
  double acc = 0.0;
  for (int sl = 0; sl < n; ++sl) {
    const double x = gm[3 * sl], y = gm[3 * sl + 1], z = gm[3 * sl + 2];
    acc += sqrt(x * x + y * y + z * z);
  }
  const int a = active[r];
  atomicAdd(grow_sum + a, acc);
  atomicAdd(grow_cnt + a, (double)n);
}

// Backward, part 1 (gaussian-parallel): per-gaussian cotangents -> head-output
// cotangents g_o (feature-major, row = head output column) and the offsets
// grads. A block owns floor(256 / n) whole anchors (n gaussians each, thread =
// gaussian, so every per-gaussian array is read coalesced); the block's
// [11n x anchors] slice of the raw head outputs is staged through shared
// memory in, and the g_o slice out, so the feature-major rows move as
// contiguous runs instead of one scattered 4-byte access per (gaussian, row).
#ifndef VSX_DBG_MINB
#define VSX_DBG_MINB 4
#endif
__global__ void __launch_bounds__(256, VSX_DBG_MINB) decode_bwd_gauss_kernel(
    int n, const int32_t *__restrict__ active, int32_t n_active,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, double max_scale,
    const float *__restrict__ cache_o, const float *__restrict__ dscale,
    const float *__restrict__ dquat, const float *__restrict__ g_means,
    const float *__restrict__ g_opacity, const float *__restrict__ g_color,
    const float *__restrict__ g_scale, const float *__restrict__ g_quat,
    const float *__restrict__ g_normal, float *__restrict__ g_offsets,
    float *__restrict__ g_o_out) {
  extern __shared__ float so[];  // [11n][ab + 1]
  const int ab = 256 / n, sp = ab + 1;
  const int r0 = blockIdx.x * ab;
  const int na = min(ab, n_active - r0);
  const int rows = 11 * n;
  const size_t ld = cache_ld(n_active);
  const int t = threadIdx.x;
  const bool ok = t < na * n;
  const int ra = t / n, sl = t - ra * n;  // block-local anchor, slot
  const int r = r0 + ra;
  const size_t g = (size_t)r * n + sl;
  // per-gaussian operands are loaded before the staging barrier so their
  // latency overlaps the tile staging
  float gop = 0.f, gcol[3] = {0.f, 0.f, 0.f}, sc[3] = {0.f, 0.f, 0.f},
        gsc[3] = {0.f, 0.f, 0.f}, q4[4] = {0.f, 0.f, 0.f, 0.f}, gq[4] = {0.f, 0.f, 0.f, 0.f},
        gnr[3] = {0.f, 0.f, 0.f}, gmu[3] = {0.f, 0.f, 0.f}, ls[3] = {0.f, 0.f, 0.f};
  int a = 0;
  if (ok) {
    a = active[r];
    gop = g_opacity[g];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gcol[c] = g_color[3 * g + c];
      sc[c] = dscale[3 * g + c];
      gsc[c] = g_scale[3 * g + c];
      gnr[c] = g_normal[3 * g + c];
      gmu[c] = g_means[3 * g + c];
      ls[c] = log_scale[3 * a + c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      q4[c] = dquat[4 * g + c];
      gq[c] = g_quat[4 * g + c];
    }
  }
  stage_cache_tile(so, cache_o, ld, r0, na, rows, sp);
  __syncthreads();
  const float smax = (float)max_scale, smin = (float)kMinScale;
  float go[11];
  if (ok) {
    {
      const float sg = sigmoidf_(so[sl * sp + ra]);
      go[0] = gop * sg * (1.f - sg);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float sg = sigmoidf_(so[(n + 3 * sl + c) * sp + ra]);
      go[1 + c] = gcol[c] * sg * (1.f - sg);
    }
    float o[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) o[c] = so[(4 * n + 7 * sl + c) * sp + ra];
    // scales: clamp(exp(o), 1e-6, max) — gradient passes inside [min, max]
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float e = expf(o[c]);
      const bool pass = (e >= smin) && (e <= smax);
      go[4 + c] = pass ? gsc[c] * e : 0.f;
    }
    // quaternion: normalised (o[3:7] + (1,0,0,0)); normal = column argmin(s) of R(q)
    const float qw = q4[0], qx = q4[1], qy = q4[2], qz = q4[3];
    const int ax = argmin3(sc[0], sc[1], sc[2]);
    float G[9];
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // register selects: a dynamic index would spill G
#pragma unroll
      for (int k = 0; k < 3; ++k) G[3 * c + k] = k == ax ? gnr[c] : 0.f;
    }
    rot_vjp(qw, qx, qy, qz, G, gq);
    const float rw = o[3] + 1.0f, rx = o[4], ry = o[5], rz = o[6];
    const float rn = sqrtf(rw * rw + rx * rx + ry * ry + rz * rz);
    if (rn >= 1e-12f) {
      const float dot = qw * gq[0] + qx * gq[1] + qy * gq[2] + qz * gq[3];
      go[7] = (gq[0] - qw * dot) / rn;
      go[8] = (gq[1] - qx * dot) / rn;
      go[9] = (gq[2] - qy * dot) / rn;
      go[10] = (gq[3] - qz * dot) / rn;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) go[7 + c] = gq[c] / 1e-12f;
    }
    // means = c + offset * l  (each (anchor, slot) appears once per view);
    // float32 is ample for a gradient (the forward keeps mu in float64)
    float *goff = g_offsets + ((size_t)a * n + sl) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) atomicAdd(goff + c, gmu[c] * expf(ls[c]));
  }
  __syncthreads();  // the tile is reused for g_o
  if (ok) {
    so[sl * sp + ra] = go[0];
#pragma unroll
    for (int c = 0; c < 3; ++c) so[(n + 3 * sl + c) * sp + ra] = go[1 + c];
#pragma unroll
    for (int c = 0; c < 7; ++c) so[(4 * n + 7 * sl + c) * sp + ra] = go[4 + c];
  }
  __syncthreads();
  flush_cache_tile(g_o_out, so, ld, r0, na, rows, sp);
}

// Backward, part 2 (anchor-parallel): g_h = W2_h^T g_o, tanh backward ->
// g_pre (feature-major), embedding grads W1^T g_pre, log-scale grads, and the
// input block x (feature-major + a ones row) for the weight gradients.
__global__ void __launch_bounds__(128) decode_bwd_anchor_kernel(
    vsx_decoder W, const int32_t *__restrict__ active, int32_t n_active,
    const double *__restrict__ centers, const float *__restrict__ emb,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, vsx_camera cam,
    double lod_ref, const float *__restrict__ cache_h, const float *__restrict__ g_means,
    const float *__restrict__ g_o, float *__restrict__ g_emb, float *__restrict__ g_log_scale,
    float *__restrict__ xs, float *__restrict__ g_pre_out) {
  extern __shared__ __align__(16) float smem[];
  const int n = W.n;
  DecSmem s = dec_smem_carve(smem, n);
  dec_load_weights(W, s);
  const size_t ld = cache_ld(n_active);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_active; r += gridDim.x * blockDim.x) {
    const int a = active[r];
    {
      float x[kInDim];
      dec_inputs(centers, emb, a, cam, lod_ref, x);
#pragma unroll
      for (int i = 0; i < kInDim; ++i) xs[(size_t)i * ld + r] = x[i];
      xs[(size_t)kInDim * ld + r] = 1.0f;
    }
    // log-scale grads: sum over the anchor's slots of g_mean * offset
    {
      double gl[3] = {0.0, 0.0, 0.0};
      for (int sl = 0; sl < n; ++sl) {
        const size_t g = (size_t)r * n + sl;
        const float *off = offsets + ((size_t)a * n + sl) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) gl[c] += (double)g_means[3 * g + c] * (double)off[c];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
        atomicAdd(g_log_scale + 3 * a + c, (float)(gl[c] * exp((double)log_scale[3 * a + c])));
    }
    float gx[kEmbed];
#pragma unroll
    for (int i = 0; i < kEmbed; ++i) gx[i] = 0.f;
    for (int h = 0; h < 3; ++h) {
      const int ow = dec_head_w(h, n), oo = dec_head_off(h, n);
      float gh[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) gh[k] = 0.f;
      for (int j = 0; j < ow; ++j) {
        const float go = g_o[(size_t)(oo + j) * ld + r];
        const float4 *w = reinterpret_cast<const float4 *>(s.w2t + (oo + j) * 64);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 wv = w[q];
          gh[4 * q + 0] = fmaf(go, wv.x, gh[4 * q + 0]);
          gh[4 * q + 1] = fmaf(go, wv.y, gh[4 * q + 1]);
          gh[4 * q + 2] = fmaf(go, wv.z, gh[4 * q + 2]);
          gh[4 * q + 3] = fmaf(go, wv.w, gh[4 * q + 3]);
        }
      }
      // tanh backward, input-block cotangent
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const float hv = cache_h[(size_t)(h * 64 + k) * ld + r];
        gh[k] *= (1.f - hv * hv);
        g_pre_out[(size_t)(h * 64 + k) * ld + r] = gh[k];
      }
#pragma unroll
      for (int i = 0; i < kEmbed; ++i) {
        const float4 *w = reinterpret_cast<const float4 *>(s.w1 + i * 192 + h * 64);
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 wv = w[q];
          acc = fmaf(gh[4 * q + 0], wv.x, acc);
          acc = fmaf(gh[4 * q + 1], wv.y, acc);
          acc = fmaf(gh[4 * q + 2], wv.z, acc);
          acc = fmaf(gh[4 * q + 3], wv.w, acc);
        }
        gx[i] += acc;
      }
    }
#pragma unroll
    for (int i = 0; i < kEmbed; ++i) atomicAdd(g_emb + (size_t)a * kEmbed + i, gx[i]);
  }
}

// ------------------------------------------------- anchor backward on mma.sync
//
// The anchor part of the backward is two small GEMMs per anchor tile:
//   g_h  [16 x 64] = g_o_h [16 x ow_h] . W2_h^T         per head (block diagonal)
//   g_x  [16 x 32] = sum_h (g_h (.) (1 - h^2)) [16 x 64] . W1_h[0:32]^T
// One warp owns 16 anchors and runs both on the tensor cores with
// mma.sync.m16n8k8 tf32, 3xTF32 split (fp32-level accuracy). The second GEMM
// consumes the first's accumulators directly as its A operand: the C
// fragment of an n-tile (columns 2t, 2t+1) is the A fragment of a k-step whose
// K positions (t, t+4) are mapped to hidden units (2t, 2t+1) — the W1 image is
// laid out with that permutation. Weights live in shared memory as
// fragment-ordered hi/lo images (decoder_bwd_image_kernel), one float4 per
// (k-step, n-tile, lane).

// VSX_DECODE_IMG=smem copies the mma weight images into shared memory per CTA
// (A/B); by default fragments are read through L1, which leaves the SM's
// shared memory to the compositor kernels running concurrently.
inline int decode_image_in_smem() {
  static const int v = [] {
    const char *e = getenv("VSX_DECODE_IMG");
    return (e && e[0] == 's') ? 1 : 0;
  }();
  return v;
}

__host__ __device__ inline int dbw_ks(int h, int n) { return (dec_head_w(h, n) + 7) / 8; }
// staged floats per warp (decode_bwd_anchor_mma_kernel): g_o rows of the
// widest head + 64 hidden rows, 16 anchors each at the padded strides
__host__ __device__ inline int dbw_stage_floats(int n) {
  return 8 * dbw_ks(2, n) * 24 + 64 * 20;
}
__host__ __device__ inline int dbw_ks_total(int n) { return dbw_ks(0, n) + dbw_ks(1, n) + dbw_ks(2, n); }
__host__ __device__ inline size_t dbw_w2_floats(int n) { return (size_t)dbw_ks_total(n) * 8 * 32 * 4; }
constexpr size_t kDbwW1Floats = (size_t)24 * 4 * 32 * 4;
__host__ __device__ inline size_t dbw_image_floats(int n) { return dbw_w2_floats(n) + kDbwW1Floats; }

__device__ __forceinline__ void split_rna(float v, float &hi, float &lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
  hi = __uint_as_float(h);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(v - hi));
  lo = __uint_as_float(l);
}

__global__ void decoder_bwd_image_kernel(vsx_decoder W, float4 *__restrict__ img) {
  const int n = W.n;
  const int kst = dbw_ks_total(n);
  const int e_w2 = kst * 8 * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < e_w2 + 24 * 4 * 32;
       e += gridDim.x * blockDim.x) {
    float v0, v1;
    if (e < e_w2) {
      const int lane = e & 31, nt = (e >> 5) & 7, ksg = e >> 8;
      int h = 0, ks = ksg;
      while (ks >= dbw_ks(h, n)) ks -= dbw_ks(h++, n);
      const int ow = dec_head_w(h, n);
      const int g = lane >> 2, t = lane & 3;
      const int hid = nt * 8 + g, j0 = ks * 8 + t, j1 = j0 + 4;  // B[k=j][n=hidden]
      v0 = j0 < ow ? W.w2[h][hid * ow + j0] : 0.f;
      v1 = j1 < ow ? W.w2[h][hid * ow + j1] : 0.f;
    } else {
      const int e2 = e - e_w2;
      const int lane = e2 & 31, nt = (e2 >> 5) & 3, ks = e2 >> 7;  // ks over 192 hidden
      const int g = lane >> 2, t = lane & 3;
      const int i = nt * 8 + g;                                  // embedding input
      const int hid0 = ks * 8 + 2 * t, hid1 = hid0 + 1;          // K positions t, t+4
      v0 = W.w1[hid0 / 64][i * 64 + hid0 % 64];
      v1 = W.w1[hid1 / 64][i * 64 + hid1 % 64];
    }
    float h0, l0, h1, l1;
    split_rna(v0, h0, l0);
    split_rna(v1, h1, l1);
    img[e] = make_float4(h0, h1, l0, l1);
  }
}

__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], uint32_t a0, uint32_t a1,
                                                uint32_t a2, uint32_t a3, uint32_t b0,
                                                uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// d += a . b with a = (ah + al), b = (bh + bl): al.bh + ah.bl + ah.bh
__device__ __forceinline__ void mma3x(float (&d)[4], const uint32_t (&ah)[4],
                                      const uint32_t (&al)[4], float4 b) {
  const uint32_t bh0 = __float_as_uint(b.x), bh1 = __float_as_uint(b.y);
  const uint32_t bl0 = __float_as_uint(b.z), bl1 = __float_as_uint(b.w);
  mma_tf32_16x8x8(d, al[0], al[1], al[2], al[3], bh0, bh1);
  mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
  mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
}

__device__ __forceinline__ void split_trunc(float v, uint32_t &hi, uint32_t &lo) {
  hi = __float_as_uint(v) & 0xffffe000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
}

// 16-byte global -> shared copy, zero-filled beyond `bytes` (cp.async.cg)
__device__ __forceinline__ void cp_async16(float *dst, const float *src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}

#ifndef VSX_DBW_WARPS
#define VSX_DBW_WARPS 4
#endif
constexpr int kDbwWarps = VSX_DBW_WARPS;
constexpr int kDbwCtas = 16 / kDbwWarps;  // CTAs per SM: 16 warps at the 128-register budget
constexpr int kDbwGoStride = 24, kDbwHStride = 20;  // staged row strides (floats)

__global__ void __launch_bounds__(kDbwWarps * 32, kDbwCtas) decode_bwd_anchor_mma_kernel(
    int n, const float4 *__restrict__ img, const int32_t *__restrict__ active, int32_t n_active,
    const double *__restrict__ centers, const float *__restrict__ emb,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, vsx_camera cam,
    double lod_ref, const float *__restrict__ cache_h, const float *__restrict__ g_means,
    const float *__restrict__ g_o, float *__restrict__ g_emb, float *__restrict__ g_log_scale,
    float *__restrict__ xs, float *__restrict__ g_pre_out, int smem_img) {
  extern __shared__ __align__(16) float4 dimg[];
  const int kst = dbw_ks_total(n);
  const float4 *base = img;  // weight fragments read through L1 (shared with the compositor)
  const int nimg = smem_img ? (int)(dbw_image_floats(n) / 4) : 0;
  if (smem_img) {
    for (int e = threadIdx.x; e < nimg; e += blockDim.x) dimg[e] = img[e];
    __syncthreads();
    base = dimg;
  }
  const float4 *w2i = base, *w1i = base + kst * 8 * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-warp staging of one head's g_o rows and hidden activations for the
  // warp's 16 anchors: one round of coalesced loads per head instead of a
  // dependent global load in front of every k-step (the kernel was 76%
  // long-scoreboard stalls). Row strides 24 / 20 keep the fragment reads
  // bank-conflict free.
  const int go_rows = 8 * dbw_ks(2, n);
  float *s_go = reinterpret_cast<float *>(dimg + nimg) + (size_t)warp * dbw_stage_floats(n);
  float *s_h = s_go + go_rows * kDbwGoStride;
  const int g = lane >> 2, t = lane & 3;
  const size_t ld = cache_ld(n_active);
  const int n_tiles = (n_active + 15) / 16;
  for (int tile = blockIdx.x * kDbwWarps + warp; tile < n_tiles; tile += gridDim.x * kDbwWarps) {
    const int r0 = tile * 16;
    // ---- per-anchor scalar work: lanes 0-15 write the input block, 16-31 the log-scale grads
    {
      const int r = r0 + (lane & 15);
      if (r < n_active) {
        const int a = active[r];
        if (lane < 16) {
          float x[kInDim];
          dec_inputs(centers, emb, a, cam, lod_ref, x);
#pragma unroll
          for (int i = 0; i < kInDim; ++i) xs[(size_t)i * ld + r] = x[i];
          xs[(size_t)kInDim * ld + r] = 1.0f;
        } else {
          double gl[3] = {0.0, 0.0, 0.0};
          for (int sl = 0; sl < n; ++sl) {
            const size_t gg = (size_t)r * n + sl;
            const float *off = offsets + ((size_t)a * n + sl) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) gl[c] += (double)g_means[3 * gg + c] * (double)off[c];
          }
#pragma unroll
          for (int c = 0; c < 3; ++c)
            atomicAdd(g_log_scale + 3 * a + c, (float)(gl[c] * exp((double)log_scale[3 * a + c])));
        }
      }
    }
    const int ra = r0 + g, rb = r0 + g + 8;
    const bool va = ra < n_active, vb = rb < n_active;
    float dx[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) dx[q][0] = dx[q][1] = dx[q][2] = dx[q][3] = 0.f;
    int ksg = 0;
    for (int h = 0; h < 3; ++h) {
      const int ow = dec_head_w(h, n), oo = dec_head_off(h, n), nks = dbw_ks(h, n);
      float c[8][4];
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0.f;
      __syncwarp();  // the previous head's tiles are consumed
      {
        // every 16-byte piece of the head's g_o rows and hidden rows in flight
        // at once (cp.async, zero-filled past the last anchor / row): one
        // memory latency per head instead of one per unrolled load batch
        const int valid = min(16, n_active - r0);
        for (int c = lane; c < 8 * nks * 4; c += 32) {
          const int row = c >> 2, q = c & 3;
          const int bytes = row < ow ? 4 * max(0, min(4, valid - 4 * q)) : 0;
          cp_async16(s_go + row * kDbwGoStride + 4 * q,
                     g_o + (size_t)(oo + min(row, ow - 1)) * ld + r0 + 4 * q, bytes);
        }
        for (int c = lane; c < 64 * 4; c += 32) {
          const int k = c >> 2, q = c & 3;
          cp_async16(s_h + k * kDbwHStride + 4 * q,
                     cache_h + (size_t)(h * 64 + k) * ld + r0 + 4 * q,
                     4 * max(0, min(4, valid - 4 * q)));
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
      }
      __syncwarp();
      for (int ks = 0; ks < nks; ++ks, ++ksg) {
        const int j0 = ks * 8 + t, j1 = j0 + 4;
        const float a0 = s_go[j0 * kDbwGoStride + g];
        const float a1 = s_go[j0 * kDbwGoStride + g + 8];
        const float a2 = s_go[j1 * kDbwGoStride + g];
        const float a3 = s_go[j1 * kDbwGoStride + g + 8];
        uint32_t ah[4], al[4];
        split_trunc(a0, ah[0], al[0]);
        split_trunc(a1, ah[1], al[1]);
        split_trunc(a2, ah[2], al[2]);
        split_trunc(a3, ah[3], al[3]);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) mma3x(c[nt], ah, al, w2i[(ksg * 8 + nt) * 32 + lane]);
      }
      // tanh backward -> g_pre (stored), then the W1 GEMM over this head's 8 k-steps
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int k0 = h * 64 + nt * 8 + 2 * t;
        const float *h0 = s_h + (nt * 8 + 2 * t) * kDbwHStride, *h1 = h0 + kDbwHStride;
        float *p0 = g_pre_out + (size_t)k0 * ld, *p1 = p0 + ld;
        if (va) {
          const float x0 = h0[g], x1 = h1[g];
          c[nt][0] *= 1.f - x0 * x0;
          c[nt][1] *= 1.f - x1 * x1;
          p0[ra] = c[nt][0];
          p1[ra] = c[nt][1];
        } else {
          c[nt][0] = c[nt][1] = 0.f;
        }
        if (vb) {
          const float x0 = h0[g + 8], x1 = h1[g + 8];
          c[nt][2] *= 1.f - x0 * x0;
          c[nt][3] *= 1.f - x1 * x1;
          p0[rb] = c[nt][2];
          p1[rb] = c[nt][3];
        } else {
          c[nt][2] = c[nt][3] = 0.f;
        }
        // A fragment of k-step (h, nt): positions (t, t+4) = hidden (2t, 2t+1)
        uint32_t ah[4], al[4];
        split_trunc(c[nt][0], ah[0], al[0]);  // (row g,   k t)
        split_trunc(c[nt][2], ah[1], al[1]);  // (row g+8, k t)
        split_trunc(c[nt][1], ah[2], al[2]);  // (row g,   k t+4)
        split_trunc(c[nt][3], ah[3], al[3]);  // (row g+8, k t+4)
#pragma unroll
        for (int q = 0; q < 4; ++q) mma3x(dx[q], ah, al, w1i[((h * 8 + nt) * 4 + q) * 32 + lane]);
      }
    }
    // ---- embedding grads: D fragment (anchor g / g+8, input 8q + 2t, +1)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i0 = q * 8 + 2 * t;
      if (va) {
        float *ge = g_emb + (size_t)active[ra] * kEmbed + i0;
        atomicAdd(ge, dx[q][0]);
        atomicAdd(ge + 1, dx[q][1]);
      }
      if (vb) {
        float *ge = g_emb + (size_t)active[rb] * kEmbed + i0;
        atomicAdd(ge, dx[q][2]);
        atomicAdd(ge + 1, dx[q][3]);
      }
    }
  }
}

// ------------------------------------------------------- forward on mma.sync
//
// GEMM1 (per head)  Hpre[16 x 64] = [x | 1 | 0][16 x 40] . [W1_h ; b1_h ; 0]
// GEMM2 (per head)  O   [16 x ow] = tanh(Hpre)[16 x 64] . W2_h      (+ b2)
// One warp owns 16 anchors; the GEMM1 accumulators feed GEMM2 directly as
// its A operand (same K permutation as the backward's W1 image). Writes the
// feature-major caches (hidden activations, raw head outputs + b2); the
// per-gaussian activations run in decode_gauss_kernel.

__host__ __device__ inline int dfw_nt2(int h, int n) { return (dec_head_w(h, n) + 7) / 8; }
__host__ __device__ inline int dfw_nt2_total(int n) { return dfw_nt2(0, n) + dfw_nt2(1, n) + dfw_nt2(2, n); }
constexpr size_t kDfwW1Floats = (size_t)3 * 5 * 8 * 32 * 4;
__host__ __device__ inline size_t dfw_image_floats(int n) {
  return kDfwW1Floats + (size_t)8 * dfw_nt2_total(n) * 32 * 4;
}
__host__ __device__ inline bool dfw_supported(int n) { return dfw_nt2(2, n) <= 9; }

__global__ void decoder_fwd_image_kernel(vsx_decoder W, float4 *__restrict__ img) {
  const int n = W.n;
  const int e_w1 = 3 * 5 * 8 * 32;
  const int e_w2 = 8 * dfw_nt2_total(n) * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < e_w1 + e_w2;
       e += gridDim.x * blockDim.x) {
    const int lane = e & 31, g = lane >> 2, t = lane & 3;
    float v0, v1;
    if (e < e_w1) {
      const int nt = (e >> 5) & 7, ks = (e >> 8) % 5, h = (e >> 8) / 5;
      const int hid = nt * 8 + g;
      auto w1v = [&](int k) {
        if (k < kInDim) return W.w1[h][k * 64 + hid];
        if (k == kInDim) return W.b1[h][hid];
        return 0.f;
      };
      v0 = w1v(ks * 8 + t);
      v1 = w1v(ks * 8 + t + 4);
    } else {
      int e2 = e - e_w1;
      int h = 0;
      while (e2 >= 8 * dfw_nt2(h, n) * 32) e2 -= 8 * dfw_nt2(h++, n) * 32;
      const int nt2h = dfw_nt2(h, n), ow = dec_head_w(h, n);
      const int nt2 = (e2 >> 5) % nt2h, kk = (e2 >> 5) / nt2h;
      const int j = nt2 * 8 + g;
      const int hid0 = kk * 8 + 2 * t, hid1 = hid0 + 1;  // K positions t, t+4
      v0 = j < ow ? W.w2[h][hid0 * ow + j] : 0.f;
      v1 = j < ow ? W.w2[h][hid1 * ow + j] : 0.f;
    }
    float h0, l0, h1, l1;
    split_rna(v0, h0, l0);
    split_rna(v1, h1, l1);
    img[e] = make_float4(h0, h1, l0, l1);
  }
}

#ifndef VSX_DFW_WARPS
#define VSX_DFW_WARPS 8
#endif
#ifndef VSX_DFW_MINB
#define VSX_DFW_MINB 2
#endif
constexpr int kDfwWarps = VSX_DFW_WARPS;

__global__ void __launch_bounds__(kDfwWarps * 32, VSX_DFW_MINB) decode_fwd_mma_kernel(
    vsx_decoder W, const float4 *__restrict__ img, const int32_t *__restrict__ active,
    int32_t n_active, const double *__restrict__ centers, const float *__restrict__ emb,
    vsx_camera cam, double lod_ref, float *__restrict__ cache_h, float *__restrict__ cache_o,
    int smem_img) {
  extern __shared__ __align__(16) float4 fimg[];
  __shared__ float s_b2[11 * 10];
  const int n = W.n;
  const float4 *base = img;  // weight fragments read through L1 (shared with the compositor)
  if (smem_img) {
    const int nimg = (int)(dfw_image_floats(n) / 4);
    for (int e = threadIdx.x; e < nimg; e += blockDim.x) fimg[e] = img[e];
    base = fimg;
  }
  for (int j = threadIdx.x; j < 11 * n; j += blockDim.x)
    s_b2[j] = j < n ? W.b2[0][j] : (j < 4 * n ? W.b2[1][j - n] : W.b2[2][j - 4 * n]);
  __syncthreads();
  const float4 *w1i = base, *w2i = base + 3 * 5 * 8 * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const size_t ld = cache_ld(n_active);
  const int n_tiles = (n_active + 15) / 16;
  for (int tile = blockIdx.x * kDfwWarps + warp; tile < n_tiles; tile += gridDim.x * kDfwWarps) {
    const int r0 = tile * 16, ra = r0 + g, rb = r0 + g + 8;
    const bool va = ra < n_active, vb = rb < n_active;
    const int aa = va ? active[ra] : 0, ab = vb ? active[rb] : 0;
    // X fragments (raw): xa[ks] = {X[ra][8ks+t], X[rb][8ks+t], X[ra][8ks+t+4], X[rb][8ks+t+4]}
    float xa[5][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      xa[ks][0] = va ? emb[(size_t)aa * kEmbed + 8 * ks + t] : 0.f;
      xa[ks][1] = vb ? emb[(size_t)ab * kEmbed + 8 * ks + t] : 0.f;
      xa[ks][2] = va ? emb[(size_t)aa * kEmbed + 8 * ks + t + 4] : 0.f;
      xa[ks][3] = vb ? emb[(size_t)ab * kEmbed + 8 * ks + t + 4] : 0.f;
    }
    // columns 32..35 = (d/ref, (c - cam)/d) (decoder.py:142-147, float64), 36 = bias
    auto derived = [&](int a, bool v) {
      if (!v) return 0.f;
      const double rx = dsub(centers[3 * a + 0], cam.center[0]);
      const double ry = dsub(centers[3 * a + 1], cam.center[1]);
      const double rz = dsub(centers[3 * a + 2], cam.center[2]);
      const double d = fmax(sqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), dmul(rz, rz))), 1e-12);
      const double num = t == 0 ? d : (t == 1 ? rx : (t == 2 ? ry : rz));
      return (float)ddiv(num, t == 0 ? lod_ref : d);
    };
    xa[4][0] = derived(aa, va);
    xa[4][1] = derived(ab, vb);
    xa[4][2] = (t == 0 && va) ? 1.f : 0.f;
    xa[4][3] = (t == 0 && vb) ? 1.f : 0.f;
    int w2off = 0;
    for (int h = 0; h < 3; ++h) {
      const int nt2h = dfw_nt2(h, n), ow = dec_head_w(h, n), oo = dec_head_off(h, n);
      float c[8][4];
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 5; ++ks) {
        uint32_t ah[4], al[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_trunc(xa[ks][e], ah[e], al[e]);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) mma3x(c[nt], ah, al, w1i[((h * 5 + ks) * 8 + nt) * 32 + lane]);
      }
      float o[9][4];
#pragma unroll
      for (int q = 0; q < 9; ++q) o[q][0] = o[q][1] = o[q][2] = o[q][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const float v0 = tanh_fast(c[kk][0]), v1 = tanh_fast(c[kk][1]);
        const float v2 = tanh_fast(c[kk][2]), v3 = tanh_fast(c[kk][3]);
        if (cache_h) {
          const int k0 = h * 64 + kk * 8 + 2 * t;
          float *h0 = cache_h + (size_t)k0 * ld, *h1 = h0 + ld;
          if (va) {
            h0[ra] = v0;
            h1[ra] = v1;
          }
          if (vb) {
            h0[rb] = v2;
            h1[rb] = v3;
          }
        }
        uint32_t ah[4], al[4];
        split_trunc(v0, ah[0], al[0]);  // (row g,   k t)   = hidden 2t
        split_trunc(v2, ah[1], al[1]);  // (row g+8, k t)
        split_trunc(v1, ah[2], al[2]);  // (row g,   k t+4) = hidden 2t+1
        split_trunc(v3, ah[3], al[3]);  // (row g+8, k t+4)
#pragma unroll
        for (int q = 0; q < 9; ++q)
          if (q < nt2h) mma3x(o[q], ah, al, w2i[(w2off + kk * nt2h + q) * 32 + lane]);
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        if (q >= nt2h) break;
        const int j0 = q * 8 + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = j0 + e;
          if (j >= ow) continue;
          float *col = cache_o + (size_t)(oo + j) * ld;
          if (va) col[ra] = o[q][e] + s_b2[oo + j];
          if (vb) col[rb] = o[q][2 + e] + s_b2[oo + j];
        }
      }
      w2off += 8 * nt2h;
    }
  }
}

size_t decoder_fwd_image_floats(int n) { return dfw_image_floats(n); }

int decoder_fwd_image(vsx_decoder W, float *img, cudaStream_t st) {
  decoder_fwd_image_kernel<<<32, 256, 0, st>>>(W, reinterpret_cast<float4 *>(img));
  VSX_LAUNCH_CHECK("decoder_fwd_image");
  return VSX_OK;
}

// Returns 1 (not launched) when n is outside the mma path's register budget.
int decode_fwd_mma(vsx_decoder W, const float *img, const int32_t *active, int32_t n_active,
                   const double *centers, const float *emb, vsx_camera cam, double lod_ref,
                   float *cache_h, float *cache_o, cudaStream_t st) {
  if (!dfw_supported(W.n) || 11 * W.n > 110) return 1;
  const int smem_img = decode_image_in_smem();
  const size_t smem = smem_img ? sizeof(float) * dfw_image_floats(W.n) : 0;
  VSX_CUDA_TRY(cudaFuncSetAttribute(decode_fwd_mma_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(float) * dfw_image_floats(W.n))));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = (n_active + 15) / 16;
  const int grid = std::max(1, std::min(VSX_DFW_MINB * sms, (tiles + kDfwWarps - 1) / kDfwWarps));
  decode_fwd_mma_kernel<<<grid, kDfwWarps * 32, smem, st>>>(
      W, reinterpret_cast<const float4 *>(img), active, n_active, centers, emb, cam, lod_ref,
      cache_h, cache_o, smem_img);
  VSX_LAUNCH_CHECK("decode_fwd_mma");
  return VSX_OK;
}

// ----------------------------------------------- weight gradients on mma.sync
//
// dW2_h[k][j] = sum_r H_h[r][k] g_o[r][j] (+ db2 via a ones column) and
// dW1_h[i][k] = sum_r X[r][i] g_pre[r][k] (+ db1 via the ones row of X) as one
// K-split GEMM over the active anchors (K). Each CTA streams its K-chunks of
// the four feature-major operands into shared memory with cp.async (two
// stages, 16 anchors each) and its 8 warps own 144 output tiles (m16n8), 18
// each, accumulated in registers with mma.sync tf32 3xTF32. Per-CTA partial
// tiles go to a buffer that one reduction kernel folds into the gradients
// (no atomics). Head blocks of g_o are padded to 16 rows so every m-tile
// belongs to one head.

__host__ __device__ inline int wm_pad16(int x) { return (x + 15) / 16 * 16; }

constexpr int kWmKc = 16;       // anchors per stage
constexpr int kWmStride = 20;   // floats per staged row (bank-conflict-free fragments)
constexpr int kWmGo = 128;      // padded g_o rows (n <= 10: 16 + 32 + 80)
constexpr int kWmH = 200;       // cache_h rows + ones row (192) + zero rows
constexpr int kWmGp = 192;      // g_pre rows
constexpr int kWmX = 48;        // xs rows (36 = ones) + zero rows
constexpr int kWmRows = kWmGo + kWmH + kWmGp + kWmX;
constexpr int kWmStageFloats = kWmRows * kWmStride;
constexpr int kWmTiles = 144;
constexpr int kWmMaxCtas = 320;

__host__ __device__ inline bool wm_supported(int n) {
  return wm_pad16(n) + wm_pad16(3 * n) + wm_pad16(7 * n) <= kWmGo;
}

__device__ __forceinline__ void cp_async16_zfill(float *dst, const float *src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(256, 2) decoder_wgrad_mma_kernel(
    const float *__restrict__ g_o, const float *__restrict__ cache_h,
    const float *__restrict__ g_pre, const float *__restrict__ xs, int64_t K, size_t ld, int n,
    float *__restrict__ partial) {
  extern __shared__ __align__(16) float wms[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int np0 = wm_pad16(n), np1 = wm_pad16(3 * n);
  const int go_row0[3] = {0, np0, np0 + np1};
  const int oo[3] = {0, n, 4 * n};
  // zero both stages once (padding rows are never written again)
  for (int e = t; e < 2 * kWmStageFloats; e += 256) wms[e] = 0.f;
  __syncthreads();
  const int64_t nchunks = (K + kWmKc - 1) / kWmKc;
  auto stage_ptr = [&](int s) { return wms + s * kWmStageFloats; };
  // issue the copies of chunk c into stage s
  auto issue = [&](int64_t c, int s) {
    float *base = stage_ptr(s);
    const int64_t k0 = c * kWmKc;
    const int valid_rows = 11 * n + 192 + 192 + (kInDim + 1);
    for (int e = t; e < valid_rows * 4; e += 256) {
      const int row = e >> 2, q = e & 3;
      const float *src;
      int dst_row;
      if (row < 11 * n) {
        const int h = row < n ? 0 : (row < 4 * n ? 1 : 2);
        src = g_o + (size_t)row * ld;
        dst_row = go_row0[h] + (row - oo[h]);
      } else if (row < 11 * n + 192) {
        const int r = row - 11 * n;
        src = cache_h + (size_t)r * ld;
        dst_row = kWmGo + r;
      } else if (row < 11 * n + 384) {
        const int r = row - 11 * n - 192;
        src = g_pre + (size_t)r * ld;
        dst_row = kWmGo + kWmH + r;
      } else {
        const int r = row - 11 * n - 384;
        src = xs + (size_t)r * ld;
        dst_row = kWmGo + kWmH + kWmGp + r;
      }
      const int64_t k = k0 + 4 * q;
      const int bytes = (int)max((int64_t)0, min((int64_t)16, (K - k) * 4));
      cp_async16_zfill(base + dst_row * kWmStride + 4 * q, src + (bytes > 0 ? k : 0), bytes);
    }
  };
  float acc[18][4];
#pragma unroll
  for (int q = 0; q < 18; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
  int s = 0;
  if ((int64_t)blockIdx.x < nchunks) issue(blockIdx.x, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, s ^= 1) {
    const int64_t nx = c + gridDim.x;
    if (nx < nchunks) issue(nx, s ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    float *base = stage_ptr(s);
    if (t < kWmKc) base[(kWmGo + 192) * kWmStride + t] = (c * kWmKc + t < K) ? 1.f : 0.f;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kWmKc; kk += 8) {
      const int col = kk + tq;
      if (warp < 4) {
        // dW2: m-tiles 2w, 2w+1 over padded g_o rows; n-tiles 0..7 = head
        // hidden units, 8 = ones column (db2)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int mt = 2 * warp + mi;
          const int h = mt * 16 < go_row0[1] ? 0 : (mt * 16 < go_row0[2] ? 1 : 2);
          const float *A = base + (mt * 16 + g) * kWmStride + col;
          uint32_t ah[4], al[4];
          split_trunc(A[0], ah[0], al[0]);
          split_trunc(A[8 * kWmStride], ah[1], al[1]);
          split_trunc(A[4], ah[2], al[2]);
          split_trunc(A[8 * kWmStride + 4], ah[3], al[3]);
#pragma unroll
          for (int nt = 0; nt < 9; ++nt) {
            const int hrow = nt < 8 ? h * 64 + nt * 8 + g : 192 + g;
            const float *Bp = base + (kWmGo + hrow) * kWmStride + col;
            uint32_t bh0, bl0, bh1, bl1;
            split_trunc(Bp[0], bh0, bl0);
            split_trunc(Bp[4], bh1, bl1);
            float (&d)[4] = acc[mi * 9 + nt];
            mma_tf32_16x8x8(d, al[0], al[1], al[2], al[3], bh0, bh1);
            mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bl0, bl1);
            mma_tf32_16x8x8(d, ah[0], ah[1], ah[2], ah[3], bh0, bh1);
          }
        }
      } else {
        // dW1: m-tiles 0..2 over xs rows; n-tiles 6(w-4) .. +5 over g_pre rows
        uint32_t ah[3][4], al[3][4];
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
          const float *A = base + (kWmGo + kWmH + kWmGp + mt * 16 + g) * kWmStride + col;
          split_trunc(A[0], ah[mt][0], al[mt][0]);
          split_trunc(A[8 * kWmStride], ah[mt][1], al[mt][1]);
          split_trunc(A[4], ah[mt][2], al[mt][2]);
          split_trunc(A[8 * kWmStride + 4], ah[mt][3], al[mt][3]);
        }
#pragma unroll
        for (int ni = 0; ni < 6; ++ni) {
          const int nt = 6 * (warp - 4) + ni;
          const float *Bp = base + (kWmGo + kWmH + nt * 8 + g) * kWmStride + col;
          uint32_t bh0, bl0, bh1, bl1;
          split_trunc(Bp[0], bh0, bl0);
          split_trunc(Bp[4], bh1, bl1);
#pragma unroll
          for (int mt = 0; mt < 3; ++mt) {
            float (&d)[4] = acc[mt * 6 + ni];
            mma_tf32_16x8x8(d, al[mt][0], al[mt][1], al[mt][2], al[mt][3], bh0, bh1);
            mma_tf32_16x8x8(d, ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bl0, bl1);
            mma_tf32_16x8x8(d, ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bh0, bh1);
          }
        }
      }
    }
    __syncthreads();  // the stage is overwritten by the copies issued next iteration
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  // partial tiles in fragment order: tile index = dW2 mt*9+nt | 72 + dW1 mt*24+nt
  float4 *out = reinterpret_cast<float4 *>(partial) + (size_t)blockIdx.x * kWmTiles * 32;
#pragma unroll
  for (int q = 0; q < 18; ++q) {
    int tile;
    if (warp < 4) tile = (2 * warp + q / 9) * 9 + q % 9;
    else tile = 72 + (q / 6) * 24 + 6 * (warp - 4) + q % 6;
    out[tile * 32 + lane] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
  }
}

// Two fixed-order stages (no float atomics, so the weight gradients are
// bitwise reproducible): blockIdx.y = slice of the CTA partials summed into
// slice_sum, then one thread per element adds the kWmSlices slice sums in
// order into the gradient (each element has exactly one thread).
constexpr int kWmSlices = 8;

__global__ void decoder_wgrad_slices_kernel(const float *__restrict__ partial, int ctas,
                                            float *__restrict__ slice_sum) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // (tile, lane, e)
  if (idx >= kWmTiles * 128) return;
  const int per = (ctas + kWmSlices - 1) / kWmSlices;
  const int c0 = blockIdx.y * per, c1 = min(ctas, c0 + per);
  float sum = 0.f;
  for (int c = c0; c < c1; ++c) sum += partial[(size_t)c * kWmTiles * 128 + idx];
  slice_sum[(size_t)blockIdx.y * kWmTiles * 128 + idx] = sum;
}

__global__ void decoder_wgrad_reduce_kernel(const float *__restrict__ slice_sum, int n,
                                            vsx_decoder_grads dW) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // (tile, lane, e)
  if (idx >= kWmTiles * 128) return;
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kWmSlices; ++k) sum += slice_sum[(size_t)k * kWmTiles * 128 + idx];
  const int tile = idx >> 7, lane = (idx >> 2) & 31, e = idx & 3;
  const int g = lane >> 2, tq = lane & 3;
  const int row_in = g + 8 * (e >> 1), col_in = 2 * tq + (e & 1);
  if (tile < 72) {
    const int mt = tile / 9, nt = tile % 9;
    const int np0 = wm_pad16(n), np1 = wm_pad16(3 * n);
    const int row = mt * 16 + row_in;
    const int h = row < np0 ? 0 : (row < np0 + np1 ? 1 : 2);
    const int jh = row - (h == 0 ? 0 : (h == 1 ? np0 : np0 + np1));
    const int owh = h == 0 ? n : (h == 1 ? 3 * n : 7 * n);
    if (jh >= owh) return;
    const int col = nt * 8 + col_in;
    if (nt < 8) dW.w2[h][(size_t)col * owh + jh] += sum;
    else if (col == 64) dW.b2[h][jh] += sum;
  } else {
    const int tt = tile - 72, mt = tt / 24, nt = tt % 24;
    const int i = mt * 16 + row_in, col = nt * 8 + col_in;
    const int h = col / 64, hh = col % 64;
    if (i < kInDim) dW.w1[h][(size_t)i * 64 + hh] += sum;
    else if (i == kInDim) dW.b1[h][hh] += sum;
  }
}

// C[m][c] += sum_k A[m][k] * B[c][k] for a K-chunk per blockIdx.z, where A is
// (M x K) and B is (Ncols x K), both row-major with leading dim K (feature-
// major caches). Output column c maps to segment out[c / seg_w] with row
// stride ld_out; row M (== A_rows) is an implicit ones row written to
// bias[c] when bias != nullptr.
struct WgradOut {
  float *out[3];
  float *bias[3];
  int seg_w;
  int ld_out;
};

constexpr int kWgTile = 32;
constexpr int kWgK = 64;

__global__ void __launch_bounds__(256) wgrad_kernel(const float *__restrict__ A, int a_rows,
                                                    bool ones_row, const float *__restrict__ B,
                                                    int b_rows, int64_t K, int64_t k_chunk,
                                                    size_t ld, WgradOut o) {
  __shared__ float sa[kWgTile][kWgK + 1];
  __shared__ float sb[kWgTile][kWgK + 1];
  const int m0 = blockIdx.x * kWgTile, c0 = blockIdx.y * kWgTile;
  const int64_t k_begin = (int64_t)blockIdx.z * k_chunk;
  const int64_t k_end = min(K, k_begin + k_chunk);
  const int tm = threadIdx.x / 8;         // 0..31 row within tile
  const int tc = (threadIdx.x % 8) * 4;   // 4 consecutive columns
  const int m_total = a_rows + (ones_row ? 1 : 0);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t kk = k_begin; kk < k_end; kk += kWgK) {
    for (int e = threadIdx.x; e < kWgTile * kWgK; e += 256) {
      const int rr = e / kWgK, k = e % kWgK;
      const int64_t gk = kk + k;
      const int m = m0 + rr, c = c0 + rr;
      float av = 0.f, bv = 0.f;
      if (gk < k_end) {
        if (m < a_rows) av = A[(size_t)m * ld + gk];
        else if (m < m_total) av = 1.f;
        if (c < b_rows) bv = B[(size_t)c * ld + gk];
      }
      sa[rr][k] = av;
      sb[rr][k] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kWgK; ++k) {
      const float av = sa[tm][k];
      acc[0] = fmaf(av, sb[tc + 0][k], acc[0]);
      acc[1] = fmaf(av, sb[tc + 1][k], acc[1]);
      acc[2] = fmaf(av, sb[tc + 2][k], acc[2]);
      acc[3] = fmaf(av, sb[tc + 3][k], acc[3]);
    }
    __syncthreads();
  }
  const int m = m0 + tm;
  if (m >= m_total) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + tc + q;
    if (c >= b_rows) continue;
    const int seg = c / o.seg_w, cc = c % o.seg_w;
    if (m < a_rows) atomicAdd(o.out[seg] + (size_t)m * o.ld_out + cc, acc[q]);
    else if (o.bias[seg]) atomicAdd(o.bias[seg] + cc, acc[q]);
  }
}

static int launch_wgrad(const float *A, int a_rows, bool ones_row, const float *B, int b_rows,
                        int64_t K, size_t ld, WgradOut o, cudaStream_t st) {
  if (K == 0) return VSX_OK;
  const int gm = (a_rows + (ones_row ? 1 : 0) + kWgTile - 1) / kWgTile;
  const int gc = (b_rows + kWgTile - 1) / kWgTile;
  int64_t splits = std::max<int64_t>(1, (296 + gm * gc - 1) / (gm * gc));
  int64_t k_chunk = (K + splits - 1) / splits;
  k_chunk = ((k_chunk + kWgK - 1) / kWgK) * kWgK;
  splits = (K + k_chunk - 1) / k_chunk;
  dim3 grid(gm, gc, (unsigned)splits);
  wgrad_kernel<<<grid, 256, 0, st>>>(A, a_rows, ones_row, B, b_rows, K, k_chunk, ld, o);
  VSX_LAUNCH_CHECK("wgrad");
  return VSX_OK;
}

int decoder_wgrad_tc2(const float *g_o, const float *cache_h, const float *g_pre, const float *xs,
                      int64_t K, size_t ld, int n, vsx_decoder_grads dW, float *partial,
                      size_t partial_floats, cudaStream_t st);

}  // namespace vsx

using namespace vsx;

static int dec_grid(int32_t n_active, size_t smem) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = std::max<int>(1, (int)(200 * 1024 / std::max<size_t>(smem, 1)));
  return std::max(1, std::min(grid_for(n_active, 128), sms * std::min(per_sm, 4)));
}

extern "C" int vsx_decode_fwd(vsx_decoder W, const int32_t *active, int32_t n_active,
                              const double *centers, const float *emb, const float *log_scale,
                              const float *offsets, vsx_camera cam, double lod_ref,
                              double max_scale, double *means, float *opacity, float *color,
                              float *scale, float *quat, float *normal, float *cache_h,
                              float *cache_o, int32_t *status, vsx_stream s) {
  VSX_REQUIRE(W.n >= 1 && n_active >= 0 && lod_ref > 0, "decode_fwd: bad arguments");
  if (n_active == 0) return VSX_OK;
  const size_t smem = dec_smem_bytes(W.n);
  VSX_REQUIRE(smem <= 227 * 1024, "decode_fwd: n=%d too large for shared weights", W.n);
  VSX_CUDA_TRY(cudaFuncSetAttribute(decode_fwd_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  decode_fwd_kernel<<<dec_grid(n_active, smem), 128, smem, as_stream(s)>>>(
      W, active, n_active, centers, emb, log_scale, offsets, cam, lod_ref, max_scale, means,
      opacity, color, scale, quat, normal, cache_h, cache_o, status);
  VSX_LAUNCH_CHECK("decode_fwd");
  return VSX_OK;
}

extern "C" size_t vsx_decode_bwd_ws_bytes(int32_t n, int32_t n_active) {
  // xs [37][ld] + g_pre [192][ld] + g_o [11n][ld] + the mma weight image
  return sizeof(float) * cache_ld(n_active) * (size_t)(kInDim + 1 + 192 + 11 * n) +
         sizeof(float) * dbw_image_floats(n) +
         sizeof(float) * (size_t)(kWmMaxCtas + kWmSlices) * kWmTiles * 128 + 256;
}

extern "C" int vsx_decode_bwd(vsx_decoder W, vsx_decoder_grads dW, const int32_t *active,
                              int32_t n_active, const double *centers, const float *emb,
                              const float *log_scale, const float *offsets, vsx_camera cam,
                              double lod_ref, double max_scale, const float *cache_h,
                              const float *cache_o, const float *scale, const float *quat,
                              const float *g_means, const float *g_opacity, const float *g_color,
                              const float *g_scale, const float *g_quat, const float *g_normal,
                              float *g_emb, float *g_log_scale, float *g_offsets, void *ws,
                              size_t ws_bytes, vsx_stream s) {
  VSX_REQUIRE(W.n >= 1 && n_active >= 0, "decode_bwd: bad arguments");
  if (n_active == 0) return VSX_OK;
  VSX_REQUIRE(ws_bytes >= vsx_decode_bwd_ws_bytes(W.n, n_active), "decode_bwd: workspace");
  cudaStream_t st = as_stream(s);
  const int n = W.n;
  const size_t ld = cache_ld(n_active);
  float *xs = static_cast<float *>(ws);
  float *g_pre = xs + (size_t)(kInDim + 1) * ld;
  float *g_o = g_pre + (size_t)192 * ld;
  const int64_t ng = (int64_t)n_active * n;
  VSX_REQUIRE(n <= 256, "decode_bwd: n=%d > 256", n);
  const int ab = 256 / n;
  const size_t gsm = sizeof(float) * 11 * n * (ab + 1);
  (void)ng;
  decode_bwd_gauss_kernel<<<(unsigned)((n_active + ab - 1) / ab), 256, gsm, st>>>(
      n, active, n_active, log_scale, offsets, max_scale, cache_o, scale, quat, g_means,
      g_opacity, g_color, g_scale, g_quat, g_normal, g_offsets, g_o);
  VSX_LAUNCH_CHECK("decode_bwd_gauss");
  static const bool use_tc = [] {
    const char *e = getenv("VSX_DECODE_TC");
    return !(e && e[0] == '0');
  }();
  if (use_tc) {  // anchor GEMMs on mma.sync (tensor cores)
    float4 *dimg = reinterpret_cast<float4 *>(g_o + (size_t)11 * n * ld);
    decoder_bwd_image_kernel<<<32, 256, 0, st>>>(W, dimg);
    VSX_LAUNCH_CHECK("decoder_bwd_image");
    const int smem_img = decode_image_in_smem();
    const size_t smem_full = sizeof(float) * dbw_image_floats(n);
    VSX_REQUIRE(smem_full <= 113 * 1024, "decode_bwd: n=%d too large for the mma weight image", n);
    const size_t stage = sizeof(float) * (size_t)kDbwWarps * dbw_stage_floats(n);
    VSX_CUDA_TRY(cudaFuncSetAttribute(decode_bwd_anchor_mma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(smem_full + stage)));
    const size_t smem = (smem_img ? smem_full : 0) + stage;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int warps_needed = (n_active + 15) / 16;
    const int grid =
        std::max(1, std::min(kDbwCtas * sms, (warps_needed + kDbwWarps - 1) / kDbwWarps));
    decode_bwd_anchor_mma_kernel<<<grid, kDbwWarps * 32, smem, st>>>(
        n, dimg, active, n_active, centers, emb, log_scale, offsets, cam, lod_ref, cache_h,
        g_means, g_o, g_emb, g_log_scale, xs, g_pre, smem_img);
    VSX_LAUNCH_CHECK("decode_bwd_anchor_mma");
  } else {
    const size_t smem = dec_smem_bytes(n);
    VSX_CUDA_TRY(cudaFuncSetAttribute(decode_bwd_anchor_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    decode_bwd_anchor_kernel<<<dec_grid(n_active, smem), 128, smem, st>>>(
        W, active, n_active, centers, emb, log_scale, offsets, cam, lod_ref, cache_h, g_means, g_o,
        g_emb, g_log_scale, xs, g_pre);
    VSX_LAUNCH_CHECK("decode_bwd_anchor");
  }
  // weight gradients: the pipelined tcgen05 kernel (TMEM accumulators, one
  // fixed-order reduction) by default; VSX_WGRAD=mma selects the mma.sync
  // K-split kernel (A/B, and the path for 11 n > 128 outputs)
  static const bool wg_mma = [] {
    const char *e = getenv("VSX_WGRAD");
    return e && e[0] == 'm';
  }();
  float *partial = reinterpret_cast<float *>(
      reinterpret_cast<char *>(g_o + (size_t)11 * n * ld) + sizeof(float) * dbw_image_floats(n));
  if (use_tc && !wg_mma && 11 * n <= 128)
    return decoder_wgrad_tc2(g_o, cache_h, g_pre, xs, n_active, ld, n, dW, partial,
                             (size_t)(kWmMaxCtas + kWmSlices) * kWmTiles * 128, st);
  if (use_tc && wm_supported(n)) {  // mma.sync K-split + reduction
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nchunks = (n_active + kWmKc - 1) / kWmKc;
    const int ctas = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(2 * sms, kWmMaxCtas), nchunks));
    const size_t smem = sizeof(float) * 2 * kWmStageFloats;
    VSX_CUDA_TRY(cudaFuncSetAttribute(decoder_wgrad_mma_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    decoder_wgrad_mma_kernel<<<ctas, 256, smem, st>>>(g_o, cache_h, g_pre, xs, n_active, ld, n,
                                                       partial);
    VSX_LAUNCH_CHECK("decoder_wgrad_mma");
    float *slice_sum = partial + (size_t)kWmMaxCtas * kWmTiles * 128;
    decoder_wgrad_slices_kernel<<<dim3((kWmTiles * 128 + 255) / 256, kWmSlices), 256, 0, st>>>(
        partial, ctas, slice_sum);
    VSX_LAUNCH_CHECK("decoder_wgrad_slices");
    decoder_wgrad_reduce_kernel<<<(kWmTiles * 128 + 255) / 256, 256, 0, st>>>(slice_sum, n, dW);
    VSX_LAUNCH_CHECK("decoder_wgrad_reduce");
    return VSX_OK;
  }
  // dW1_h = X^T Gpre_h (+ db1 via the ones row of X)
  WgradOut o1{};
  for (int h = 0; h < 3; ++h) {
    o1.out[h] = dW.w1[h];
    o1.bias[h] = dW.b1[h];
  }
  o1.seg_w = 64;
  o1.ld_out = 64;
  int rc = launch_wgrad(xs, kInDim, true, g_pre, 192, n_active, ld, o1, st);
  if (rc) return rc;
  // dW2_h = H_h^T Go_h (+ db2 via an implicit ones row)
  for (int h = 0; h < 3; ++h) {
    const int ow = dec_head_w(h, n), oo = dec_head_off(h, n);
    WgradOut o2{};
    o2.out[0] = dW.w2[h];
    o2.bias[0] = dW.b2[h];
    o2.seg_w = ow;
    o2.ld_out = ow;
    rc = launch_wgrad(cache_h + (size_t)h * 64 * ld, 64, true, g_o + (size_t)oo * ld, ow,
                      n_active, ld, o2, st);
    if (rc) return rc;
  }
  return VSX_OK;
}

extern "C" int vsx_growth_accumulate(const float *g_means, const int32_t *active,
                                     int32_t n_active, int32_t n, double *grow_sum,
                                     double *grow_cnt, vsx_stream s) {
  VSX_REQUIRE(n >= 1 && n_active >= 0 && grow_sum && grow_cnt, "growth_accumulate: bad args");
  if (n_active == 0) return VSX_OK;
  growth_accumulate_kernel<<<grid_for(n_active, 256), 256, 0, as_stream(s)>>>(
      g_means, active, n_active, n, grow_sum, grow_cnt);
  VSX_LAUNCH_CHECK("growth_accumulate");
  return VSX_OK;
}
