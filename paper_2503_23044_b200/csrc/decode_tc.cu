// K2 on the 5th-gen tensor cores: the anchor decoder MLP with tcgen05.
//
// Same math as decode.cu (voxsplat decoder.py:142-180) but the two GEMMs per
// head run as kind::tf32 MMAs from shared memory into TMEM, with a 3xTF32
// split (hi*hi + lo*hi + hi*lo) so the result keeps fp32 accuracy (single
// TF32 misses the 1e-4 image bound, SURVEY §7 hard part 4):
//   GEMM1  Hpre[128 x 64] = [x | 1] [128 x 40] . [W1_h ; b1_h]^T   (bias folded in K)
//   GEMM2  O   [128 x Nh] = tanh(Hpre) [128 x 64] . W2_h^T         (+ b2 in the epilogue)
// One CTA (4 warps, thread = anchor row) loops persistently over tiles of 128
// active anchors; warp 0 lane 0 issues the MMAs; the epilogue reads TMEM with
// tcgen05.ld (warp w owns lanes 32w..32w+31) and applies the activations.
//
// Weights are pre-split once per optimizer step by decoder_image_kernel into
// the exact shared-memory image (hi/lo tiles in the K-major interleaved
// layout of umma.cuh), so tiles only copy them.
#include "common.cuh"
#include "umma.cuh"

namespace vsx {

constexpr int kTcK1 = 40;   // 36 inputs + bias column + zero pad (multiple of 8)
constexpr int kTcK2 = 64;   // hidden width
constexpr int kTcRows = 128;

__host__ __device__ inline int pad16(int x) { return (x + 15) / 16 * 16; }

struct TcDims {
  int n;          // gaussians per anchor
  int np[3];      // padded head widths (multiples of 16)
  int row0[3];    // row offset of each head inside the W2 image
  int np_total;
};

__host__ __device__ inline TcDims tc_dims(int n) {
  TcDims d;
  d.n = n;
  d.np[0] = pad16(n);
  d.np[1] = pad16(3 * n);
  d.np[2] = pad16(7 * n);
  d.row0[0] = 0;
  d.row0[1] = d.np[0];
  d.row0[2] = d.np[0] + d.np[1];
  d.np_total = d.np[0] + d.np[1] + d.np[2];
  return d;
}

// Floats of the weight image: 3 heads x (hi, lo) x [64 x 40] + (hi, lo) x [NP x 64].
__host__ __device__ inline size_t tc_image_floats(int n) {
  return (size_t)3 * 2 * 64 * kTcK1 + (size_t)2 * tc_dims(n).np_total * kTcK2;
}

__global__ void decoder_image_kernel(vsx_decoder W, float *__restrict__ img) {
  const TcDims d = tc_dims(W.n);
  const int w1_tile = 64 * kTcK1;
  const int total1 = 3 * 64 * kTcK1;
  const int total2 = d.np_total * kTcK2;
  float *w2img = img + 3 * 2 * w1_tile;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total1 + total2;
       e += gridDim.x * blockDim.x) {
    if (e < total1) {
      const int h = e / w1_tile, rem = e % w1_tile, n = rem / kTcK1, k = rem % kTcK1;
      float v = 0.f;
      if (k < kInDim) v = W.w1[h][k * 64 + n];
      else if (k == kInDim) v = W.b1[h][n];
      float hi, lo;
      umma::split_tf32(v, hi, lo);
      float *base = img + (size_t)h * 2 * w1_tile;
      const uint32_t off = umma::kmajor_offset(n, k, kTcK1) / 4;
      base[off] = hi;
      base[w1_tile + off] = lo;
    } else {
      const int e2 = e - total1, row = e2 / kTcK2, k = e2 % kTcK2;
      int h = 2;
      if (row < d.row0[1]) h = 0;
      else if (row < d.row0[2]) h = 1;
      const int j = row - d.row0[h];
      const int width = (h == 0 ? 1 : (h == 1 ? 3 : 7)) * d.n;
      const float v = j < width ? W.w2[h][k * width + j] : 0.f;
      float hi, lo;
      umma::split_tf32(v, hi, lo);
      const uint32_t off = umma::kmajor_offset(row, k, kTcK2) / 4;
      w2img[off] = hi;
      w2img[(size_t)d.np_total * kTcK2 + off] = lo;
    }
  }
}

__device__ __forceinline__ float sigm(float v) { return 1.0f / (1.0f + expf(-v)); }

struct TcSmem {
  float *x_hi, *x_lo, *w1_hi, *w1_lo, *h_hi, *h_lo, *w2_hi, *w2_lo;
};

__device__ __forceinline__ void st_split4(float *hi_base, float *lo_base, uint32_t off_bytes,
                                          float a, float b, float c, float d) {
  float4 h, l;
  umma::split_tf32(a, h.x, l.x);
  umma::split_tf32(b, h.y, l.y);
  umma::split_tf32(c, h.z, l.z);
  umma::split_tf32(d, h.w, l.w);
  *reinterpret_cast<float4 *>(reinterpret_cast<char *>(hi_base) + off_bytes) = h;
  *reinterpret_cast<float4 *>(reinterpret_cast<char *>(lo_base) + off_bytes) = l;
}

// 3xTF32 chain D (+)= A . B^T over K (in 8-element MMA steps).
__device__ __forceinline__ void mma3(uint32_t d, const float *a_hi, const float *a_lo,
                                     const float *b_hi, const float *b_lo, int K, uint32_t id) {
  const uint32_t ah = umma::smem_addr(a_hi), al = umma::smem_addr(a_lo);
  const uint32_t bh = umma::smem_addr(b_hi), bl = umma::smem_addr(b_lo);
  for (int s = 0; s < K / 8; ++s) {
    const uint32_t off = (uint32_t)s * 256;
    umma::mma_tf32(d, umma::desc_kmajor(ah + off, K), umma::desc_kmajor(bh + off, K), id, s > 0);
    umma::mma_tf32(d, umma::desc_kmajor(al + off, K), umma::desc_kmajor(bh + off, K), id, true);
    umma::mma_tf32(d, umma::desc_kmajor(ah + off, K), umma::desc_kmajor(bl + off, K), id, true);
  }
}

// Two warpgroups (256 threads): both own TMEM lanes 0-127 (thread row =
// tid % 128) and split every epilogue's columns / slots between them, which
// halves the serial per-thread epilogue chains that bound this kernel.
__global__ void __launch_bounds__(256, 1) decode_fwd_tc_kernel(
    vsx_decoder W, const float *__restrict__ img, const int32_t *__restrict__ active,
    int32_t n_active, const double *__restrict__ centers, const float *__restrict__ emb,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, vsx_camera cam,
    double lod_ref, double max_scale, double *__restrict__ means, float *__restrict__ opacity,
    float *__restrict__ color, float *__restrict__ scale, float *__restrict__ quat,
    float *__restrict__ normal, float *__restrict__ cache_h, float *__restrict__ cache_o,
    int32_t *__restrict__ status) {
  extern __shared__ __align__(1024) float tsm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ float s_b2[11 * 13];
  const int n = W.n;
  const TcDims dims = tc_dims(n);
  TcSmem s;
  s.x_hi = tsm;
  s.x_lo = s.x_hi + kTcRows * kTcK1;
  s.w1_hi = s.x_lo + kTcRows * kTcK1;
  s.w1_lo = s.w1_hi + 64 * kTcK1;
  s.h_hi = s.w1_lo + 64 * kTcK1;
  s.h_lo = s.h_hi + kTcRows * kTcK2;
  s.w2_hi = s.h_lo + kTcRows * kTcK2;
  s.w2_lo = s.w2_hi + dims.np_total * kTcK2;
  const int tid = threadIdx.x, t = tid & 127, wg = tid >> 7, warp = (tid >> 5) & 3;
  // resident W2 image (hi and lo back to back, same as the global image)
  {
    const float4 *src = reinterpret_cast<const float4 *>(img + 3 * 2 * 64 * kTcK1);
    float4 *dst = reinterpret_cast<float4 *>(s.w2_hi);
    const int n4 = 2 * dims.np_total * kTcK2 / 4;
    for (int i = tid; i < n4; i += 256) dst[i] = src[i];
  }
  for (int j = tid; j < 11 * n; j += 256)
    s_b2[j] = j < n ? W.b2[0][j] : (j < 4 * n ? W.b2[1][j - n] : W.b2[2][j - 4 * n]);
  if (tid < 32) umma::tmem_alloc(&tslot, 256);
  if (tid == 0) umma::mbar_init(&mbar, 1);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t lane = (uint32_t)(warp * 32) << 16;
  const uint32_t d1 = tbase, d2 = tbase + 64;
  uint32_t phase = 0;
  const int n_tiles = (n_active + kTcRows - 1) / kTcRows;
  const size_t ld = cache_ld(n_active);
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int r = tile * kTcRows + t;
    const bool valid = r < n_active;
    const int a = valid ? active[r] : 0;
    // ---- input block (decoder.py:142-147) + bias column, split into X tiles
    if (wg == 0) {
      float x[kTcK1];
#pragma unroll
      for (int i = 0; i < kTcK1; ++i) x[i] = 0.f;
      if (valid) {
        const double rx = dsub(centers[3 * a + 0], cam.center[0]);
        const double ry = dsub(centers[3 * a + 1], cam.center[1]);
        const double rz = dsub(centers[3 * a + 2], cam.center[2]);
        const double dd = fmax(sqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), dmul(rz, rz))), 1e-12);
        const float4 *e4 = reinterpret_cast<const float4 *>(emb + (size_t)a * kEmbed);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = e4[q];
          x[4 * q] = v.x;
          x[4 * q + 1] = v.y;
          x[4 * q + 2] = v.z;
          x[4 * q + 3] = v.w;
        }
        x[32] = (float)ddiv(dd, lod_ref);
        x[33] = (float)ddiv(rx, dd);
        x[34] = (float)ddiv(ry, dd);
        x[35] = (float)ddiv(rz, dd);
        x[36] = 1.f;
      }
#pragma unroll
      for (int q = 0; q < kTcK1 / 4; ++q)
        st_split4(s.x_hi, s.x_lo, umma::kmajor_offset(t, 4 * q, kTcK1), x[4 * q], x[4 * q + 1],
                  x[4 * q + 2], x[4 * q + 3]);
    }
    for (int h = 0; h < 3; ++h) {
      // W1_h image -> smem
      {
        const float4 *src = reinterpret_cast<const float4 *>(img + (size_t)h * 2 * 64 * kTcK1);
        float4 *dst = reinterpret_cast<float4 *>(s.w1_hi);
        for (int i = tid; i < 2 * 64 * kTcK1 / 4; i += 256) dst[i] = src[i];
      }
      umma::fence_async_smem();
      umma::fence_before_sync();
      __syncthreads();
      umma::fence_after_sync();
      if (tid == 0) {
        mma3(d1, s.x_hi, s.x_lo, s.w1_hi, s.w1_lo, kTcK1, umma::idesc_tf32(128, 64));
        umma::commit(&mbar);
      }
      umma::mbar_wait(&mbar, phase);
      phase ^= 1u;
      umma::fence_after_sync();
      // hidden activations -> cache + H tiles (warpgroup wg: columns 32wg..32wg+31)
#pragma unroll
      for (int c = 32 * wg; c < 32 * wg + 32; c += 16) {
        float v[16];
        umma::tmem_ld16(d1 + lane + (uint32_t)c, v);
        umma::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] = tanh_fast(v[i]);
          if (valid && cache_h) cache_h[(size_t)(h * 64 + c + i) * ld + r] = v[i];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_split4(s.h_hi, s.h_lo, umma::kmajor_offset(t, c + 4 * q, kTcK2), v[4 * q],
                    v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      umma::fence_async_smem();
      umma::fence_before_sync();
      __syncthreads();
      umma::fence_after_sync();
      if (tid == 0) {
        const int off = dims.row0[h] * kTcK2;  // row offset (multiple of 16 rows)
        mma3(d2, s.h_hi, s.h_lo, s.w2_hi + off, s.w2_lo + off, kTcK2,
             umma::idesc_tf32(128, dims.np[h]));
        umma::commit(&mbar);
      }
      umma::mbar_wait(&mbar, phase);
      phase ^= 1u;
      umma::fence_after_sync();
      // raw head outputs (+ b2) -> cache_o; the per-gaussian activations run
      // in decode_gauss_kernel with one thread per gaussian
      const int width = (h == 0 ? 1 : (h == 1 ? 3 : 7)) * n;
      const int oo = h == 0 ? 0 : (h == 1 ? n : 4 * n);
      for (int c = 16 * wg; c < dims.np[h]; c += 32) {
        float v[16];
        umma::tmem_ld16(d2 + lane + (uint32_t)c, v);
        umma::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = c + i;
          if (valid && j < width) cache_o[(size_t)(oo + j) * ld + r] = v[i] + s_b2[oo + j];
        }
      }
      umma::fence_before_sync();
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (tid < 32) umma::tmem_dealloc(tbase, 256);
}

// Per-gaussian activations of the decoded heads (decoder.py:160-180), one
// thread per gaussian g = r * n + sl (coalesced output rows). A block owns
// floor(256 / n) whole anchors and stages their [11n x anchors] slice of the
// feature-major cache_o through shared memory, so the raw outputs are read as
// contiguous row runs instead of one scattered 4-byte load per (gaussian, row).
#ifndef VSX_DG_MINB
#define VSX_DG_MINB 5
#endif
__global__ void __launch_bounds__(256, VSX_DG_MINB) decode_gauss_kernel(
    int n, const int32_t *__restrict__ active, int32_t n_active, const double *__restrict__ centers,
    const float *__restrict__ log_scale, const float *__restrict__ offsets, double max_scale,
    const float *__restrict__ cache_o, double *__restrict__ means, float *__restrict__ opacity,
    float *__restrict__ color, float *__restrict__ scale, float *__restrict__ quat,
    float *__restrict__ normal, int32_t *__restrict__ status) {
  extern __shared__ float so[];  // [11n][ab + 1]
  __shared__ double s_ls[3 * 256];  // exp(log_scale) of the block's anchors
  const int ab = 256 / n, sp = ab + 1;
  const int r0 = blockIdx.x * ab;
  const int na = min(ab, n_active - r0);
  const int rows = 11 * n;
  const size_t ld = cache_ld(n_active);
  const int t = threadIdx.x;
  const bool live = t < na * n;
  const int ra = t / n, sl = t - ra * n;
  const int r = r0 + ra;
  // per-gaussian global operands first (active -> offsets / centres /
  // log_scale is a dependent chain), so their latency overlaps the staging
  const int a = live ? active[r] : 0;
  float off[3] = {0.f, 0.f, 0.f};
  double cen[3] = {0.0, 0.0, 0.0};
  float ls[3] = {0.f, 0.f, 0.f};
  if (live) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      off[c] = offsets[((size_t)a * n + sl) * 3 + c];
      cen[c] = centers[3 * a + c];
      if (sl == 0) ls[c] = log_scale[3 * a + c];
    }
  }
  stage_cache_tile(so, cache_o, ld, r0, na, rows, sp);
  if (live && sl == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) s_ls[3 * ra + c] = exp((double)ls[c]);
  }
  __syncthreads();
  bool bad = false;
  if (live) {
    const int64_t g = (int64_t)r * n + sl;
    const float op = sigm(so[sl * sp + ra]);
    opacity[g] = op;
    bad |= !isfinite(op);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float v = sigm(so[(n + 3 * sl + c) * sp + ra]);
      color[3 * g + c] = v;
      bad |= !isfinite(v);
    }
    float o[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) o[c] = so[(4 * n + 7 * sl + c) * sp + ra];
    const float smax = (float)max_scale, smin = (float)kMinScale;
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
#pragma unroll
    for (int c = 0; c < 3; ++c)  // register selects: a dynamic index would spill R
      normal[3 * g + c] = ax == 0 ? R[3 * c] : (ax == 1 ? R[3 * c + 1] : R[3 * c + 2]);
    const double m0 = dadd(cen[0], dmul((double)off[0], s_ls[3 * ra + 0]));
    const double m1 = dadd(cen[1], dmul((double)off[1], s_ls[3 * ra + 1]));
    const double m2 = dadd(cen[2], dmul((double)off[2], s_ls[3 * ra + 2]));
    means[3 * g + 0] = m0;
    means[3 * g + 1] = m1;
    means[3 * g + 2] = m2;
    bad |= !(isfinite(sc[0]) && isfinite(sc[1]) && isfinite(sc[2]) && isfinite(qw) &&
             isfinite(qx) && isfinite(qy) && isfinite(qz) && isfinite(m0) && isfinite(m1) &&
             isfinite(m2));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, VSX_STATUS_NONFINITE);
}

// Resident-weight version (the default forward): W1 of all three heads
// ([192 x 40], one N = 192 MMA chain for the first layer) and W2 ([NP x 64])
// stay in shared memory for the CTA's lifetime, so a tile never copies
// weights; the hidden layer is fed to the second GEMM in two K halves of 32
// (the half tile is 32 KB, which keeps everything in 200 KB), and both
// warpgroups share every epilogue (thread row = tid % 128, columns split).
// TMEM: first-layer accumulators in columns [0, 192), second-layer head h at
// 192 + row0[h].
constexpr int kTcKH = 32;  // hidden columns per second-layer K half

__global__ void __launch_bounds__(256, 1) decode_fwd_tc2_kernel(
    vsx_decoder W, const float *__restrict__ img, const int32_t *__restrict__ active,
    int32_t n_active, const double *__restrict__ centers, const float *__restrict__ emb,
    vsx_camera cam, double lod_ref, float *__restrict__ cache_h, float *__restrict__ cache_o) {
  extern __shared__ __align__(1024) float tsm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  __shared__ float s_b2[11 * 13];
  const int n = W.n;
  const TcDims dims = tc_dims(n);
  float *x_hi = tsm, *x_lo = x_hi + kTcRows * kTcK1;
  float *w1_hi = x_lo + kTcRows * kTcK1, *w1_lo = w1_hi + 192 * kTcK1;
  float *h_hi = w1_lo + 192 * kTcK1, *h_lo = h_hi + kTcRows * kTcKH;
  float *w2_hi = h_lo + kTcRows * kTcKH, *w2_lo = w2_hi + dims.np_total * kTcK2;
  const int tid = threadIdx.x, t = tid & 127, wg = tid >> 7, warp = (tid >> 5) & 3;
  {
    // W1: the image holds (hi, lo) per head; the N = 192 operand wants the
    // three hi tiles back to back, then the three lo tiles
    const int tile4 = 64 * kTcK1 / 4;
    for (int i = tid; i < 3 * 2 * tile4; i += 256) {
      const int h = i / (2 * tile4), part = (i / tile4) & 1, e = i % tile4;
      float4 *dst = reinterpret_cast<float4 *>(part ? w1_lo : w1_hi) + h * tile4 + e;
      *dst = reinterpret_cast<const float4 *>(img)[i];
    }
    const float4 *src = reinterpret_cast<const float4 *>(img + 3 * 2 * 64 * kTcK1);
    float4 *dst = reinterpret_cast<float4 *>(w2_hi);
    const int n4 = 2 * dims.np_total * kTcK2 / 4;
    for (int i = tid; i < n4; i += 256) dst[i] = src[i];
  }
  for (int j = tid; j < 11 * n; j += 256)
    s_b2[j] = j < n ? W.b2[0][j] : (j < 4 * n ? W.b2[1][j - n] : W.b2[2][j - 4 * n]);
  if (tid < 32) umma::tmem_alloc(&tslot, 512);
  if (tid == 0) umma::mbar_init(&mbar, 1);
  umma::fence_async_smem();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t lane = (uint32_t)(warp * 32) << 16;
  const uint32_t d1 = tbase, d2 = tbase + 192;
  uint32_t phase = 0;
  const int n_tiles = (n_active + kTcRows - 1) / kTcRows;
  const size_t ld = cache_ld(n_active);
  auto sync_mma = [&]() {  // smem writes -> tensor core, all threads
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
  };
  auto wait_mma = [&]() {
    umma::mbar_wait(&mbar, phase);
    phase ^= 1u;
    umma::fence_after_sync();
  };
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int r = tile * kTcRows + t;
    const bool valid = r < n_active;
    // ---- input block (decoder.py:142-147) + bias column, split into X
    if (wg == 0) {
      float x[kTcK1];
#pragma unroll
      for (int i = 0; i < kTcK1; ++i) x[i] = 0.f;
      if (valid) {
        const int a = active[r];
        const double rx = dsub(centers[3 * a + 0], cam.center[0]);
        const double ry = dsub(centers[3 * a + 1], cam.center[1]);
        const double rz = dsub(centers[3 * a + 2], cam.center[2]);
        const double dd = fmax(sqrt(dadd(dadd(dmul(rx, rx), dmul(ry, ry)), dmul(rz, rz))), 1e-12);
        const float4 *e4 = reinterpret_cast<const float4 *>(emb + (size_t)a * kEmbed);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = e4[q];
          x[4 * q] = v.x;
          x[4 * q + 1] = v.y;
          x[4 * q + 2] = v.z;
          x[4 * q + 3] = v.w;
        }
        x[32] = (float)ddiv(dd, lod_ref);
        x[33] = (float)ddiv(rx, dd);
        x[34] = (float)ddiv(ry, dd);
        x[35] = (float)ddiv(rz, dd);
        x[36] = 1.f;
      }
#pragma unroll
      for (int q = 0; q < kTcK1 / 4; ++q)
        st_split4(x_hi, x_lo, umma::kmajor_offset(t, 4 * q, kTcK1), x[4 * q], x[4 * q + 1],
                  x[4 * q + 2], x[4 * q + 3]);
    }
    sync_mma();
    if (tid == 0) {  // first layer of all three heads: N = 192
      mma3(d1, x_hi, x_lo, w1_hi, w1_lo, kTcK1, umma::idesc_tf32(128, 192));
      umma::commit(&mbar);
    }
    wait_mma();
    for (int h = 0; h < 3; ++h) {
      for (int kh = 0; kh < 2; ++kh) {
        // hidden columns 32 kh .. 32 kh + 31 of head h: warpgroup wg takes 16
        const int c0 = kTcKH * kh + 16 * wg;
        float v[16];
        umma::tmem_ld16(d1 + lane + (uint32_t)(64 * h + c0), v);
        umma::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] = tanh_fast(v[i]);
          if (valid && cache_h) cache_h[(size_t)(h * 64 + c0 + i) * ld + r] = v[i];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_split4(h_hi, h_lo, umma::kmajor_offset(t, 16 * wg + 4 * q, kTcKH), v[4 * q],
                    v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        sync_mma();
        if (tid == 0) {
          const uint32_t ah = umma::smem_addr(h_hi), al = umma::smem_addr(h_lo);
          const uint32_t boff = (uint32_t)(dims.row0[h] * kTcK2 * 4) + (uint32_t)kh * 4 * 256;
          const uint32_t bh = umma::smem_addr(w2_hi) + boff, bl = umma::smem_addr(w2_lo) + boff;
          const uint32_t id = umma::idesc_tf32(128, dims.np[h]);
          const uint32_t dd2 = d2 + (uint32_t)dims.row0[h];
          for (int st = 0; st < kTcKH / 8; ++st) {
            const uint32_t oa = (uint32_t)st * 256;
            using umma::desc_kmajor;
            const bool acc = kh > 0 || st > 0;
            umma::mma_tf32(dd2, desc_kmajor(ah + oa, kTcKH), desc_kmajor(bh + oa, kTcK2), id, acc);
            umma::mma_tf32(dd2, desc_kmajor(al + oa, kTcKH), desc_kmajor(bh + oa, kTcK2), id, true);
            umma::mma_tf32(dd2, desc_kmajor(ah + oa, kTcKH), desc_kmajor(bl + oa, kTcK2), id, true);
          }
          umma::commit(&mbar);
        }
        wait_mma();  // the half tile is rewritten next
      }
      // raw head outputs (+ b2) -> cache_o
      const int width = (h == 0 ? 1 : (h == 1 ? 3 : 7)) * n;
      const int oo = h == 0 ? 0 : (h == 1 ? n : 4 * n);
      for (int c = 16 * wg; c < dims.np[h]; c += 32) {
        float v[16];
        umma::tmem_ld16(d2 + lane + (uint32_t)(dims.row0[h] + c), v);
        umma::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = c + i;
          if (valid && j < width) cache_o[(size_t)(oo + j) * ld + r] = v[i] + s_b2[oo + j];
        }
      }
    }
    umma::fence_before_sync();
    __syncthreads();  // TMEM columns are rewritten by the next tile
    umma::fence_after_sync();
  }
  umma::fence_before_sync();
  __syncthreads();
  if (tid < 32) umma::tmem_dealloc(tbase, 512);
}

size_t tc2_smem_bytes(int n) {
  const TcDims d = tc_dims(n);
  return sizeof(float) * ((size_t)2 * kTcRows * kTcK1 + 2 * 192 * kTcK1 + 2 * kTcRows * kTcKH +
                          (size_t)2 * d.np_total * kTcK2);
}

// ---------------------------------------------------------------- weight gradients
//
// All decoder weight gradients of one view as two K-split tcgen05 GEMMs over
// the active anchors (K), reading the feature-major caches directly (a row
// of each cache is contiguous along K, i.e. a K-major operand):
//   C1[j][n] = sum_r dO[r][j] * [H | 1][r][n]   M = 11n outputs (pad 128), N = 192 + 1 (pad 208)
//              -> dW2_h[n][j] (diagonal head blocks) and db2 (ones column)
//   C2[m][i] = sum_r dPre[r][m] * [X | 1][r][i] M = 192 hidden (two 128 tiles), N = 37 (pad 48)
//              -> dW1_h[i][m] and db1 (ones column)
// Each persistent CTA accumulates its K-chunks in TMEM (304 of 512 columns)
// and writes its partial sums to a slot of its own; one reduction kernel
// folds the slots in CTA order into the gradients (no float atomics, so the
// result is bitwise reproducible).

constexpr int kWgKc = 16;    // anchors per stage (2 MMA k-steps)
constexpr int kWgN1 = 208;   // 192 hidden + ones row, padded to 16
constexpr int kWgN2 = 48;    // 36 inputs + ones row, padded to 16

struct WgSmem {
  float *a1_hi, *a1_lo, *b1_hi, *b1_lo, *a2_hi, *a2_lo, *b2_hi, *b2_lo;
};

// The raw fp32 operand rows of K-chunks arrive by cp.async (16-byte pieces
// straight into the K-major core-matrix layout, eight threads per 128-byte
// column) two chunks ahead of the tensor core (three raw stages); the MMA
// reads the raw words as the "hi" tf32 operand (the tensor core keeps the
// top 19 bits: truncation), and one pass per chunk writes lo = x - trunc(x)
// into a double-buffered lo plane (3xTF32, the same split as the mma.sync
// kernel). Padding rows and the ones row of [H | 1] are written once. One
// mbarrier per raw stage orders its refill after the MMAs that read it.
__device__ __forceinline__ void wg_cp16(float *dst_base, uint32_t off, const float *src,
                                        int bytes) {
  const uint32_t d = umma::smem_addr(reinterpret_cast<char *>(dst_base) + off);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}

struct WgOp {
  float *hi, *lo;
  const float *src;
  int rows_valid;
};

__device__ __forceinline__ void wg_issue(const WgSmem &s, const float *g_o, const float *cache_h,
                                         const float *g_pre, const float *xs, int nout, int64_t K,
                                         size_t ld, int64_t k0) {
  const WgOp ops[4] = {{s.a1_hi, s.a1_lo, g_o, nout},
                       {s.b1_hi, s.b1_lo, cache_h, 192},
                       {s.a2_hi, s.a2_lo, g_pre, 192},
                       {s.b2_hi, s.b2_lo, xs, kInDim + 1}};
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    // piece e -> (8-row group, 16-byte column q, row in group): 8 consecutive
    // threads fill one contiguous 128-byte core-matrix column
    const int pieces = ((ops[o].rows_valid + 7) / 8) * 8 * (kWgKc / 4);
    for (int e = threadIdx.x; e < pieces; e += blockDim.x) {
      const int r = (e / (8 * (kWgKc / 4))) * 8 + (e & 7), q = (e >> 3) % (kWgKc / 4);
      if (r >= ops[o].rows_valid) continue;
      const int64_t k = k0 + 4 * q;
      const int64_t rem = K - k;
      const int bytes = rem <= 0 ? 0 : (rem >= 4 ? 16 : (int)(4 * rem));
      wg_cp16(ops[o].hi, umma::kmajor_offset(r, 4 * q, kWgKc),
              ops[o].src + (size_t)r * ld + (bytes > 0 ? k : 0), bytes);
    }
  }
}

__device__ __forceinline__ void wg_lo_pass(const WgSmem &s, int nout) {
  const WgOp ops[4] = {{s.a1_hi, s.a1_lo, nullptr, nout},
                       {s.b1_hi, s.b1_lo, nullptr, 192},
                       {s.a2_hi, s.a2_lo, nullptr, 192},
                       {s.b2_hi, s.b2_lo, nullptr, kInDim + 1}};
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int pieces = ((ops[o].rows_valid + 7) / 8) * 8 * (kWgKc / 4);
    for (int e = threadIdx.x; e < pieces; e += blockDim.x) {
      const int r = (e / (8 * (kWgKc / 4))) * 8 + (e & 7), q = (e >> 3) % (kWgKc / 4);
      if (r >= ops[o].rows_valid) continue;
      const uint32_t off = umma::kmajor_offset(r, 4 * q, kWgKc);
      const float4 x = *reinterpret_cast<const float4 *>(reinterpret_cast<const char *>(ops[o].hi) + off);
      float4 l;
      l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
      l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
      l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
      l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
      *reinterpret_cast<float4 *>(reinterpret_cast<char *>(ops[o].lo) + off) = l;
    }
  }
}

// Operand planes of one K-chunk (one plane: hi raw words or lo parts).
constexpr int kWgPlaneFloats = kWgKc * (128 + kWgN1 + 256 + kWgN2);
constexpr int kWgRaw = 3;  // raw-word stages in flight

__device__ __forceinline__ WgSmem wg_planes(float *hi, float *lo) {
  WgSmem s;
  s.a1_hi = hi;
  s.b1_hi = hi + 128 * kWgKc;
  s.a2_hi = s.b1_hi + kWgN1 * kWgKc;
  s.b2_hi = s.a2_hi + 256 * kWgKc;
  s.a1_lo = lo;
  s.b1_lo = lo + 128 * kWgKc;
  s.a2_lo = s.b1_lo + kWgN1 * kWgKc;
  s.b2_lo = s.a2_lo + 256 * kWgKc;
  return s;
}

constexpr int kWgPartial = 128 * kWgN1 + 256 * kWgN2;  // floats per CTA partial

__global__ void __launch_bounds__(256, 1) decoder_wgrad_tc2_kernel(
    const float *__restrict__ g_o, const float *__restrict__ cache_h,
    const float *__restrict__ g_pre, const float *__restrict__ xs, int64_t K, size_t ld, int n,
    float *__restrict__ partial) {
  extern __shared__ __align__(1024) float wsm[];
  __shared__ uint64_t mbar[kWgRaw];
  __shared__ uint32_t tslot;
  float *raw = wsm, *lo = wsm + kWgRaw * kWgPlaneFloats;
  const int t = threadIdx.x, warp = t >> 5;
  const int nout = 11 * n;
  // zero every plane once (padding rows, lo of the ones row), then the ones
  // row of [H | 1] (row 192 of B1) in each raw stage
  for (int e = t; e < (kWgRaw + 2) * kWgPlaneFloats; e += blockDim.x) wsm[e] = 0.f;
  __syncthreads();
  for (int b = 0; b < kWgRaw; ++b)
    for (int k = t; k < kWgKc; k += blockDim.x)
      *reinterpret_cast<float *>(reinterpret_cast<char *>(raw + b * kWgPlaneFloats +
                                                          128 * kWgKc) +
                                 umma::kmajor_offset(192, k, kWgKc)) = 1.f;
  if (warp == 0) umma::tmem_alloc(&tslot, 512);
  if (t == 0)
    for (int b = 0; b < kWgRaw; ++b) umma::mbar_init(&mbar[b], 1);
  __syncthreads();
  const int64_t nchunks = (K + kWgKc - 1) / kWgKc;
  const int64_t G = gridDim.x;
  // prologue: this CTA's chunks 0 and 1 in flight (one cp.async group each)
  for (int p = 0; p < kWgRaw - 1; ++p) {
    const int64_t ch = (int64_t)blockIdx.x + p * G;
    if (ch < nchunks)
      wg_issue(wg_planes(raw + p * kWgPlaneFloats, lo), g_o, cache_h, g_pre, xs, nout, K, ld,
               ch * kWgKc);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tbase = tslot;
  const uint32_t c1 = tbase, c2a = tbase + kWgN1, c2b = tbase + kWgN1 + kWgN2;
  uint32_t phase[kWgRaw] = {0u, 0u, 0u};
  int it = 0;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += G, ++it) {
    const int rb = it % kWgRaw, lb = it & 1;
    const WgSmem s = wg_planes(raw + rb * kWgPlaneFloats, lo + lb * kWgPlaneFloats);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // chunk ch landed
    __syncthreads();
    wg_lo_pass(s, nout);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (t == 0) {
      const uint32_t i1 = umma::idesc_tf32(128, kWgN1), i2 = umma::idesc_tf32(128, kWgN2);
      const uint32_t a1h = umma::smem_addr(s.a1_hi), a1l = umma::smem_addr(s.a1_lo);
      const uint32_t b1h = umma::smem_addr(s.b1_hi), b1l = umma::smem_addr(s.b1_lo);
      const uint32_t a2h = umma::smem_addr(s.a2_hi), a2l = umma::smem_addr(s.a2_lo);
      const uint32_t b2h = umma::smem_addr(s.b2_hi), b2l = umma::smem_addr(s.b2_lo);
      const uint32_t tile2 = 128 * kWgKc * 4;  // second 128-row tile of A2
      for (int st = 0; st < kWgKc / 8; ++st) {
        const uint32_t o = (uint32_t)st * 256;
        const bool acc0 = !(it == 0 && st == 0);
        using umma::desc_kmajor;
        umma::mma_tf32(c1, desc_kmajor(a1h + o, kWgKc), desc_kmajor(b1h + o, kWgKc), i1, acc0);
        umma::mma_tf32(c1, desc_kmajor(a1l + o, kWgKc), desc_kmajor(b1h + o, kWgKc), i1, true);
        umma::mma_tf32(c1, desc_kmajor(a1h + o, kWgKc), desc_kmajor(b1l + o, kWgKc), i1, true);
        for (int mt = 0; mt < 2; ++mt) {
          const uint32_t d = mt ? c2b : c2a, ao = mt ? tile2 : 0u;
          umma::mma_tf32(d, desc_kmajor(a2h + ao + o, kWgKc), desc_kmajor(b2h + o, kWgKc), i2,
                         acc0);
          umma::mma_tf32(d, desc_kmajor(a2l + ao + o, kWgKc), desc_kmajor(b2h + o, kWgKc), i2,
                         true);
          umma::mma_tf32(d, desc_kmajor(a2h + ao + o, kWgKc), desc_kmajor(b2l + o, kWgKc), i2,
                         true);
        }
      }
      umma::commit(&mbar[rb]);
    }
    // chunk ch + 2G goes to the raw stage chunk ch - G used: wait for its MMAs
    // (issued last iteration; the lo plane it used is rewritten next time)
    const int nb = (it + kWgRaw - 1) % kWgRaw;
    if (it >= 1) {
      umma::mbar_wait(&mbar[nb], phase[nb]);
      phase[nb] ^= 1u;
    }
    umma::fence_after_sync();
    if (ch + 2 * G < nchunks)
      wg_issue(wg_planes(raw + nb * kWgPlaneFloats, lo), g_o, cache_h, g_pre, xs, nout, K, ld,
               (ch + 2 * G) * kWgKc);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (it > 0) {  // the last chunk's MMAs
    const int lb = (it - 1) % kWgRaw;
    umma::mbar_wait(&mbar[lb], phase[lb]);
  }
  umma::fence_after_sync();
  // this CTA's sums to its partial slot (C1 [128][208] then C2 [256][48],
  // row-major), folded over the CTAs in order by decoder_wgrad_tc2_reduce
  if (t < 128) {
    float *part = partial + (size_t)blockIdx.x * kWgPartial;
    const uint32_t lane = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < kWgN1; c += 16) {
      float v[16];
      if (it > 0) {
        umma::tmem_ld16(c1 + lane + (uint32_t)c, v);
        umma::tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      float4 *dst = reinterpret_cast<float4 *>(part + (size_t)t * kWgN1 + c);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    for (int mt = 0; mt < 2; ++mt)
      for (int c = 0; c < kWgN2; c += 16) {
        float v[16];
        if (it > 0) {
          umma::tmem_ld16((mt ? c2b : c2a) + lane + (uint32_t)c, v);
          umma::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        float4 *dst = reinterpret_cast<float4 *>(part + 128 * kWgN1 +
                                                 (size_t)(mt * 128 + t) * kWgN2 + c);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tbase, 512);
}

// Element e of the partials summed over the CTAs in a fixed order
// (deterministic): four threads per element each sum a quarter of the CTAs
// in order, the quarters are added in order, and the result goes into the
// gradient it maps to (no atomics). 64 elements per 256-thread block.
__global__ void __launch_bounds__(256) decoder_wgrad_tc2_reduce(const float *__restrict__ partial,
                                                                int ctas, int n,
                                                                vsx_decoder_grads dW) {
  __shared__ float s_q[4][64];
  const int el = threadIdx.x & 63, qi = threadIdx.x >> 6;
  const int e = blockIdx.x * 64 + el;
  const int nout = 11 * n;
  int h = 0, col = 0, j = 0;
  bool w1 = false, valid = e < kWgPartial;
  if (valid) {
    if (e < 128 * kWgN1) {
      j = e / kWgN1;
      col = e % kWgN1;
      valid = j < nout && col <= 192;
    } else {
      const int f = e - 128 * kWgN1;
      j = f / kWgN2;        // hidden unit m
      col = f % kWgN2;      // input i (36 = bias)
      valid = j < 192 && col <= kInDim;
      w1 = true;
    }
  }
  float sum = 0.f;
  if (valid) {
    const int q = (ctas + 3) / 4;
    const int c0 = qi * q, c1 = min(ctas, c0 + q);
    int c = c0;
    // 8 independent loads in flight, summed in CTA order
    for (; c + 8 <= c1; c += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = partial[(size_t)(c + u) * kWgPartial + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; c < c1; ++c) sum += partial[(size_t)c * kWgPartial + e];
  }
  s_q[qi][el] = sum;
  __syncthreads();
  if (qi != 0 || !valid) return;
  sum = ((s_q[0][el] + s_q[1][el]) + s_q[2][el]) + s_q[3][el];
  if (w1) {
    const int hh = j / 64, mm = j % 64;
    if (col < kInDim) dW.w1[hh][(size_t)col * 64 + mm] += sum;
    else dW.b1[hh][mm] += sum;
  } else {
    h = j < n ? 0 : (j < 4 * n ? 1 : 2);
    const int oo = h == 0 ? 0 : (h == 1 ? n : 4 * n);
    const int width = (h == 0 ? 1 : (h == 1 ? 3 : 7)) * n;
    if (col == 192) dW.b2[h][j - oo] += sum;
    else if (col >= h * 64 && col < h * 64 + 64) dW.w2[h][(size_t)(col - h * 64) * width + (j - oo)] += sum;
  }
}

int decoder_wgrad_tc2(const float *g_o, const float *cache_h, const float *g_pre, const float *xs,
                      int64_t K, size_t ld, int n, vsx_decoder_grads dW, float *partial,
                      size_t partial_floats, cudaStream_t st) {
  if (K == 0) return VSX_OK;
  const size_t smem = sizeof(float) * (size_t)(kWgRaw + 2) * kWgPlaneFloats;
  VSX_CUDA_TRY(cudaFuncSetAttribute(decoder_wgrad_tc2_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t chunks = (K + kWgKc - 1) / kWgKc;
  const int ctas = (int)std::min<int64_t>(std::min<int64_t>(chunks, sms),
                                          (int64_t)(partial_floats / kWgPartial));
  VSX_REQUIRE(ctas >= 1, "decoder_wgrad_tc2: partial buffer too small");
  decoder_wgrad_tc2_kernel<<<ctas, 256, smem, st>>>(g_o, cache_h, g_pre, xs, K, ld, n, partial);
  VSX_LAUNCH_CHECK("decoder_wgrad_tc2");
  decoder_wgrad_tc2_reduce<<<(kWgPartial + 63) / 64, 256, 0, st>>>(partial, ctas, n, dW);
  VSX_LAUNCH_CHECK("decoder_wgrad_tc2_reduce");
  return VSX_OK;
}

size_t tc_smem_bytes(int n) {
  const TcDims d = tc_dims(n);
  return sizeof(float) * ((size_t)2 * kTcRows * kTcK1 + 2 * 64 * kTcK1 + 2 * kTcRows * kTcK2 +
                          (size_t)2 * d.np_total * kTcK2);
}

bool tc_supported(int n) { return n >= 1 && tc_smem_bytes(n) <= 220 * 1024 && 7 * n + 16 <= 176; }

}  // namespace vsx

using namespace vsx;

namespace vsx {
size_t decoder_fwd_image_floats(int n);
int decoder_fwd_image(vsx_decoder W, float *img, cudaStream_t st);
int decode_fwd_mma(vsx_decoder W, const float *img, const int32_t *active, int32_t n_active,
                   const double *centers, const float *emb, vsx_camera cam, double lod_ref,
                   float *cache_h, float *cache_o, cudaStream_t st);
}  // namespace vsx

// The image holds both weight layouts: the tcgen05 shared-memory tiles, then
// (16-byte aligned) the mma.sync fragment image of decode_fwd_mma.
static size_t mma_image_offset(int n) { return (tc_image_floats(n) + 3) / 4 * 4; }

extern "C" size_t vsx_decoder_image_floats(int32_t n) {
  return mma_image_offset(n) + decoder_fwd_image_floats(n);
}

extern "C" int vsx_decoder_image(vsx_decoder W, float *img, vsx_stream s) {
  VSX_REQUIRE(W.n >= 1, "decoder_image: bad n");
  decoder_image_kernel<<<64, 256, 0, as_stream(s)>>>(W, img);
  VSX_LAUNCH_CHECK("decoder_image");
  return decoder_fwd_image(W, img + mma_image_offset(W.n), as_stream(s));
}

extern "C" int vsx_decode_fwd_tc(vsx_decoder W, const float *img, const int32_t *active,
                                 int32_t n_active, const double *centers, const float *emb,
                                 const float *log_scale, const float *offsets, vsx_camera cam,
                                 double lod_ref, double max_scale, double *means, float *opacity,
                                 float *color, float *scale, float *quat, float *normal,
                                 float *cache_h, float *cache_o, int32_t *status, vsx_stream s) {
  VSX_REQUIRE(W.n >= 1 && n_active >= 0 && lod_ref > 0, "decode_fwd_tc: bad arguments");
  VSX_REQUIRE(cache_o, "decode_fwd_tc: cache_o is required (the activations read it back)");
  VSX_REQUIRE(tc_supported(W.n), "decode_fwd_tc: n=%d not supported by the tensor-core path",
              W.n);
  if (n_active == 0) return VSX_OK;
  // VSX_DECODE_FWD=tcgen05 selects the tcgen05 MLP (A/B); default is the
  // warp-per-16-anchors mma.sync kernel (falls back for large n)
  // VSX_DECODE_FWD: "tc2" = resident-weight tcgen05 MLP, "tcgen05" = the
  // per-tile-copy tcgen05 MLP (A/B); default: the warp-per-16-anchors mma.sync
  static const int fwd_impl = [] {
    const char *e = getenv("VSX_DECODE_FWD");
    if (!e) return 0;
    if (e[0] == 't' && e[1] == 'c' && e[2] == '2') return 2;
    return e[0] == 't' ? 1 : 0;
  }();
  int rc = 1;
  if (fwd_impl == 2 && tc2_smem_bytes(W.n) <= 227 * 1024) {
    const size_t smem = tc2_smem_bytes(W.n);
    VSX_CUDA_TRY(cudaFuncSetAttribute(decode_fwd_tc2_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = (n_active + kTcRows - 1) / kTcRows;
    decode_fwd_tc2_kernel<<<std::min(tiles, sms), 256, smem, as_stream(s)>>>(
        W, img, active, n_active, centers, emb, cam, lod_ref, cache_h, cache_o);
    VSX_LAUNCH_CHECK("decode_fwd_tc2");
    rc = 0;
  } else if (fwd_impl == 0) {
    rc = decode_fwd_mma(W, img + mma_image_offset(W.n), active, n_active, centers, emb, cam,
                        lod_ref, cache_h, cache_o, as_stream(s));
  }
  if (rc < 0) return rc;
  if (rc == 1) {
    const size_t smem = tc_smem_bytes(W.n);
    VSX_CUDA_TRY(cudaFuncSetAttribute(decode_fwd_tc_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = (n_active + kTcRows - 1) / kTcRows;
    decode_fwd_tc_kernel<<<std::min(tiles, sms), 256, smem, as_stream(s)>>>(
        W, img, active, n_active, centers, emb, log_scale, offsets, cam, lod_ref, max_scale,
        means, opacity, color, scale, quat, normal, cache_h, cache_o, status);
    VSX_LAUNCH_CHECK("decode_fwd_tc");
  }
  const int64_t total = (int64_t)n_active * W.n;
  VSX_REQUIRE(W.n <= 256, "decode_fwd: n=%d > 256", W.n);
  const int ab = 256 / W.n;
  const size_t gsm = sizeof(float) * 11 * W.n * (ab + 1);
  (void)total;
  decode_gauss_kernel<<<(unsigned)((n_active + ab - 1) / ab), 256, gsm, as_stream(s)>>>(
      W.n, active, n_active, centers, log_scale, offsets, max_scale, cache_o, means, opacity, color,
      scale, quat, normal, status);
  VSX_LAUNCH_CHECK("decode_gauss");
  return VSX_OK;
}
