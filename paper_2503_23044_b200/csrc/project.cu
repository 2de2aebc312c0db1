// K3 / K4 / K7 — EWA projection, tile binning, projection backward.
//
// Projection restates voxsplat renderer.py:144-204 in float64 (one thread per
// gaussian): z > 0.01 cull, J Sigma_c J^T + 0.3 I, conic, 3-sigma radius,
// camera normal flipped to face the camera, plane offset. The (z, gid) sort
// of renderer.py:197 is a stable radix sort of the float64 z bits over the
// ascending-gid batch (primitives.cu). Binning restates renderer.py:207-226.
#include "common.cuh"

namespace vsx {

struct ProjGeom {
  double x, y, z;      // mu_cam
  double Rq[9];        // rotation of the gaussian (world)
  double M[9];         // R * Rq (camera-frame rotation)
  double s2[3];        // squared scales
  double J00, J02, J11, J12;
  double S[6];         // Sigma_c symmetric (00,01,02,11,12,22)
  double a, b, c, det;
};

__device__ __forceinline__ void proj_geom(const vsx_camera &cam, const double *mu, const float *sc,
                                          const float *q, ProjGeom &g) {
  cam_transform(cam, mu[0], mu[1], mu[2], g.x, g.y, g.z);
  quat_to_rot<double>(q[0], q[1], q[2], q[3], g.Rq);
#pragma unroll
  for (int k = 0; k < 3; ++k) g.s2[k] = (double)sc[k] * (double)sc[k];
  // M = R * Rq, Sigma_c = M diag(s2) M^T
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      g.M[3 * i + j] = cam.r[3 * i + 0] * g.Rq[0 + j] + cam.r[3 * i + 1] * g.Rq[3 + j] +
                       cam.r[3 * i + 2] * g.Rq[6 + j];
  auto sig = [&](int i, int j) {
    return g.M[3 * i + 0] * g.s2[0] * g.M[3 * j + 0] + g.M[3 * i + 1] * g.s2[1] * g.M[3 * j + 1] +
           g.M[3 * i + 2] * g.s2[2] * g.M[3 * j + 2];
  };
  g.S[0] = sig(0, 0);
  g.S[1] = sig(0, 1);
  g.S[2] = sig(0, 2);
  g.S[3] = sig(1, 1);
  g.S[4] = sig(1, 2);
  g.S[5] = sig(2, 2);
  const double zi = 1.0 / g.z;
  g.J00 = cam.fx * zi;
  g.J02 = -cam.fx * g.x * zi * zi;
  g.J11 = cam.fy * zi;
  g.J12 = -cam.fy * g.y * zi * zi;
  // cov2d = J S J^T with J = [[J00, 0, J02], [0, J11, J12]]
  const double c00 = g.J00 * (g.J00 * g.S[0] + g.J02 * g.S[2]) + g.J02 * (g.J00 * g.S[2] + g.J02 * g.S[5]);
  const double c01 = g.J00 * (g.J11 * g.S[1] + g.J12 * g.S[2]) + g.J02 * (g.J11 * g.S[4] + g.J12 * g.S[5]);
  const double c11 = g.J11 * (g.J11 * g.S[3] + g.J12 * g.S[4]) + g.J12 * (g.J11 * g.S[4] + g.J12 * g.S[5]);
  g.a = c00 + kLowpass;
  g.b = c01;
  g.c = c11 + kLowpass;
  g.det = g.a * g.c - g.b * g.b;
}

__global__ void __launch_bounds__(256) project_fwd_kernel(
    const double *__restrict__ means, const float *__restrict__ opacity,
    const float *__restrict__ color, const float *__restrict__ scale,
    const float *__restrict__ quat, const float *__restrict__ normal, int32_t n, vsx_camera cam,
    vsx_splat *__restrict__ rec, uint64_t *__restrict__ zkey, double *__restrict__ radius,
    uint32_t *__restrict__ n_kept, int32_t *__restrict__ status) {
  __shared__ float4 s_rec[4 * 256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  if (i < n) {
    // every operand is loaded up front (one memory round trip instead of a
    // second one behind the near-plane test)
    const double mu[3] = {means[3 * i + 0], means[3 * i + 1], means[3 * i + 2]};
    const float sc[3] = {scale[3 * i + 0], scale[3 * i + 1], scale[3 * i + 2]};
    float qv[4];
    if ((reinterpret_cast<uintptr_t>(quat) & 15) == 0) {  // uniform branch
      const float4 q4 = reinterpret_cast<const float4 *>(quat)[i];
      qv[0] = q4.x, qv[1] = q4.y, qv[2] = q4.z, qv[3] = q4.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) qv[k] = quat[4 * i + k];
    }
    const float nrm[3] = {normal[3 * i + 0], normal[3 * i + 1], normal[3 * i + 2]};
    const float col[3] = {color[3 * i + 0], color[3 * i + 1], color[3 * i + 2]};
    const float op = opacity[i];
    double x, y, z;
    cam_transform(cam, mu[0], mu[1], mu[2], x, y, z);
    keep = z > kZNear;
    if (!keep) {
      zkey[i] = ~0ull;
      radius[i] = 0.0;
    } else {
      ProjGeom g;
      proj_geom(cam, mu, sc, qv, g);
      if (!(g.det > 0.0)) {
        if (g.det <= 0.0) atomicOr(status, VSX_STATUS_NONPD);
      }
      const double idet = 1.0 / g.det;
      const double mid = 0.5 * (g.a + g.c);
      const double disc = 0.25 * (g.a - g.c) * (g.a - g.c) + g.b * g.b;
      const double lam = mid + sqrt(fmax(disc, 0.0));
      radius[i] = 3.0 * sqrt(lam);
      // camera normal, flipped to face the camera (sign(n.mu) > 0 -> flip)
      const double n0 = nrm[0], n1 = nrm[1], n2 = nrm[2];
      double nc[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) nc[k] = cam.r[3 * k + 0] * n0 + cam.r[3 * k + 1] * n1 + cam.r[3 * k + 2] * n2;
      const double face = nc[0] * x + nc[1] * y + nc[2] * z;
      const double fl = face > 0.0 ? -1.0 : 1.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) nc[k] *= fl;
      vsx_splat r;
      r.mean2d[0] = dadd(ddiv(dmul(cam.fx, x), z), cam.cx);
      r.mean2d[1] = dadd(ddiv(dmul(cam.fy, y), z), cam.cy);
      r.conic[0] = (float)(g.c * idet);
      r.conic[1] = (float)(-g.b * idet);
      r.conic[2] = (float)(g.a * idet);
      r.opacity = op;
      r.color[0] = col[0];
      r.color[1] = col[1];
      r.color[2] = col[2];
      r.normal[0] = (float)nc[0];
      r.normal[1] = (float)nc[1];
      r.normal[2] = (float)nc[2];
      r.plane_d = (float)(nc[0] * x + nc[1] * y + nc[2] * z);
      r.src = (uint32_t)i;
      union {
        vsx_splat s;
        float4 v[4];
      } u;
      u.s = r;
#pragma unroll
      for (int k = 0; k < 4; ++k) s_rec[4 * threadIdx.x + k] = u.v[k];
      zkey[i] = (uint64_t)__double_as_longlong(z);
    }
  }
  const unsigned ball = __ballot_sync(0xffffffffu, keep);
  if ((threadIdx.x & 31) == 0 && ball) atomicAdd(n_kept, (uint32_t)__popc(ball));
  // records leave through shared memory as one contiguous run per CTA
  // (consecutive lanes, consecutive 16-byte pieces); the slots of culled
  // gaussians carry stale bytes, never read (they sort behind n_kept)
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x;
  const int nb = (int)min((int64_t)blockDim.x, (int64_t)n - b0);
  float4 *out4 = reinterpret_cast<float4 *>(rec) + 4 * b0;
  for (int e = threadIdx.x; e < 4 * nb; e += blockDim.x) out4[e] = s_rec[e];
}

__global__ void gather_splats_kernel(const vsx_splat *__restrict__ rec,
                                     const double *__restrict__ radius,
                                     const uint32_t *__restrict__ order, int32_t n,
                                     vsx_splat *__restrict__ out, double *__restrict__ rout) {
  // four threads per 64-byte record, one 16-byte piece each: full-line
  // gathers and fully coalesced stores
  const int64_t tq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = tq >> 2;
  const int part = (int)(tq & 3);
  if (i >= n) return;
  const uint32_t j = order[i];
  reinterpret_cast<float4 *>(out)[4 * i + part] = __ldg(reinterpret_cast<const float4 *>(rec) + 4 * (int64_t)j + part);
  if (part == 0) rout[i] = radius[j];
}

__global__ void bin_count_kernel(const vsx_splat *__restrict__ rec,
                                 const double *__restrict__ radius, int32_t n, int txn, int tyn,
                                 uint32_t *__restrict__ splat_tiles,
                                 uint32_t *__restrict__ tile_counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x0, x1, y0, y1;
  uint32_t cnt = 0;
  if (tile_rect(rec[i].mean2d[0], rec[i].mean2d[1], radius[i], txn, tyn, x0, x1, y0, y1)) {
    cnt = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
    if (tile_counts)
      for (int ty = y0; ty <= y1; ++ty)
        for (int tx = x0; tx <= x1; ++tx) atomicAdd(tile_counts + ty * txn + tx, 1u);
  }
  if (splat_tiles) splat_tiles[i] = cnt;
}

// Tile-major emission: every covered tile's next free slot (atomic cursor)
// gets the splat's rank. Order inside a tile is arbitrary here and restored
// by tile_segsort_kernel.
__global__ void bin_emit_tiles_kernel(const vsx_splat *__restrict__ rec,
                                      const double *__restrict__ radius, int32_t n, int txn,
                                      int tyn, const uint32_t *__restrict__ tile_off,
                                      uint32_t *__restrict__ cursor,
                                      uint32_t *__restrict__ tile_list) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x0, x1, y0, y1;
  if (!tile_rect(rec[i].mean2d[0], rec[i].mean2d[1], radius[i], txn, tyn, x0, x1, y0, y1)) return;
  for (int ty = y0; ty <= y1; ++ty)
    for (int tx = x0; tx <= x1; ++tx) {
      const int t = ty * txn + tx;
      tile_list[tile_off[t] + atomicAdd(cursor + t, 1u)] = (uint32_t)i;
    }
}

// One CTA per tile: bitonic sort of the tile's ranks in shared memory (ranks
// are unique, so ascending order is exactly the reference's emission order).
constexpr int kSegCap = 4096;

__global__ void __launch_bounds__(256) tile_segsort_kernel(const uint32_t *__restrict__ tile_off,
                                                           uint32_t *__restrict__ tile_list) {
  __shared__ uint32_t s[kSegCap];
  const uint32_t b = tile_off[blockIdx.x], n = tile_off[blockIdx.x + 1] - b;
  if (n <= 1) return;
  uint32_t N = 2;
  while (N < n) N <<= 1;
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) s[i] = i < n ? tile_list[b + i] : 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const uint32_t a = s[i], c = s[l];
          if ((a > c) == ((i & k) == 0)) {
            s[i] = c;
            s[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) tile_list[b + i] = s[i];
}

// tile_off[t] = lower_bound(sorted_tiles, t), tile_off[T] = n.
__global__ void tile_ranges_kernel(const uint32_t *__restrict__ keys, int64_t n, int T,
                                   uint32_t *__restrict__ tile_off) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < (uint32_t)t) lo = mid + 1;
    else hi = mid;
  }
  tile_off[t] = (uint32_t)(t == T ? n : lo);
}

// Block-cooperative emission: a CTA owns 256 consecutive splats; their pair
// offsets come from the global exclusive scan, so thread t emits pairs
// t, t+256, ... of the CTA's range (consecutive threads -> consecutive
// addresses, every lane busy), locating its splat by binary search over the
// CTA's 257 local offsets in shared memory. Row-major tile order inside a
// splat and splat order across pairs are the reference's (renderer.py:216-226).
__global__ void __launch_bounds__(256) bin_emit_block_kernel(
    const vsx_splat *__restrict__ rec, const double *__restrict__ radius, int32_t n, int txn,
    int tyn, const uint32_t *__restrict__ offs, uint32_t *__restrict__ tiles,
    uint32_t *__restrict__ ranks, uint32_t *__restrict__ hist) {
  __shared__ uint32_t s_off[257];
  __shared__ uint32_t s_h[2][256];  // digit histograms of the two radix passes
  if (hist) {
    s_h[0][threadIdx.x] = 0u;
    s_h[1][threadIdx.x] = 0u;
  }
  __shared__ int s_x0[256], s_y0[256], s_w[256];
  __shared__ float s_iw[256];
  const int t = threadIdx.x;
  const int s0 = blockIdx.x * 256;
  const int i = s0 + t;
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  bool ok = false;
  if (i < n) ok = tile_rect(rec[i].mean2d[0], rec[i].mean2d[1], radius[i], txn, tyn, x0, x1, y0, y1);
  const int w = ok ? x1 - x0 + 1 : 1;
  const uint32_t base = offs[s0];
  s_x0[t] = x0;
  s_y0[t] = y0;
  s_w[t] = w;
  s_iw[t] = 1.0f / (float)w;
  s_off[t] = offs[min(i, n)] - base;
  if (t == 0) s_off[256] = offs[min(s0 + 256, n)] - base;
  __syncthreads();
  const uint32_t total = s_off[256];
  for (uint32_t q = t; q < total; q += 256) {
    int lo = 0, hi = 255;  // largest k with s_off[k] <= q
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= q) lo = mid;
      else hi = mid - 1;
    }
    const int k = lo;
    const int e = (int)(q - s_off[k]);
    // e / w via the float reciprocal: exact for e < 2^22 (see tile_row)
    const int row = __float2int_rz(((float)e + 0.5f) * s_iw[k]);
    const int col = e - row * s_w[k];
    const uint32_t tile = (uint32_t)((s_y0[k] + row) * txn + s_x0[k] + col);
    tiles[base + q] = tile;
    ranks[base + q] = (uint32_t)(s0 + k);
    if (hist) {
      // low digit: consecutive tiles, few collisions; high digit: one tile row
      // shares it, so the lanes of a warp aggregate first
      atomicAdd(&s_h[0][tile & 255u], 1u);
      const uint32_t hi = (tile >> 8) & 255u;
      const unsigned peers = __match_any_sync(__activemask(), hi);
      if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&s_h[1][hi], __popc(peers));
    }
  }
  if (hist) {
    __syncthreads();
    const uint32_t a = s_h[0][threadIdx.x], b = s_h[1][threadIdx.x];
    if (a) atomicAdd(hist + threadIdx.x, a);
    if (b) atomicAdd(hist + 256 + threadIdx.x, b);
  }
}

__global__ void bin_emit_kernel(const vsx_splat *__restrict__ rec,
                                const double *__restrict__ radius, int32_t n, int txn, int tyn,
                                const uint32_t *__restrict__ offs, uint32_t *__restrict__ tiles,
                                uint32_t *__restrict__ ranks) {
  // Warp-cooperative emission: the warp walks its 32 splats in order and all
  // lanes write one splat's row-major tile run together, so every store
  // instruction covers consecutive addresses (a thread-per-splat loop made
  // each lane stream its own run: one 32-byte sector per 4-byte store).
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
  bool ok = false;
  uint32_t o = 0;
  if (i < n) {
    ok = tile_rect(rec[i].mean2d[0], rec[i].mean2d[1], radius[i], txn, tyn, x0, x1, y0, y1);
    o = offs[i];
  }
  const int w = ok ? x1 - x0 + 1 : 0, h = ok ? y1 - y0 + 1 : 0;
  const unsigned live = __ballot_sync(0xffffffffu, ok);
  const uint32_t first = (uint32_t)(i - lane);
  for (int sl = 0; sl < 32; ++sl) {
    if (!((live >> sl) & 1u)) continue;  // warp-uniform
    const int ws = __shfl_sync(0xffffffffu, w, sl), hs = __shfl_sync(0xffffffffu, h, sl);
    const int xs = __shfl_sync(0xffffffffu, x0, sl), ys = __shfl_sync(0xffffffffu, y0, sl);
    const uint32_t os = __shfl_sync(0xffffffffu, o, sl);
    const int cnt = ws * hs;
    for (int k = lane; k < cnt; k += 32) {
      const int ty = ys + k / ws, tx = xs + k % ws;
      tiles[os + k] = (uint32_t)(ty * txn + tx);
      ranks[os + k] = first + (uint32_t)sl;
    }
  }
}

// ---------------------------------------------------------------- K7 backward

// Per sorted splat: screen-space grads (mean2d 2, conic 3, opacity, color 3,
// normal 3, plane_d) -> gaussian grads, float64 internally. Writes (=) into
// the batch-order outputs at rec.src; culled gaussians keep the caller's zeros.
// kBatch = false: thread per sorted splat r, scattering into batch index
// rec[r].src (culled gaussians keep the caller's zeros). kBatch = true: thread
// per batch gaussian i with its sorted rank inv[i] (-1 = culled -> zeros), so
// the per-gaussian inputs and all six outputs are read / written in order and
// only the 64-byte record and the 13-float gradient row are gathered.
#ifndef VSX_PBW_MINB
#define VSX_PBW_MINB 6
#endif
template <bool kBatch>
__global__ void __launch_bounds__(128, VSX_PBW_MINB) project_bwd_kernel(
    const double *__restrict__ means, const float *__restrict__ scale,
    const float *__restrict__ quat, const float *__restrict__ normal,
    const vsx_splat *__restrict__ rec, const float *__restrict__ gs, int32_t n, vsx_camera cam,
    float *__restrict__ g_means, float *__restrict__ g_opacity, float *__restrict__ g_color,
    float *__restrict__ g_scale, float *__restrict__ g_quat, float *__restrict__ g_normal,
    const int32_t *__restrict__ inv, int32_t n_batch) {
  int r;
  uint32_t i;
  if (kBatch) {
    const int ib = blockIdx.x * blockDim.x + threadIdx.x;
    if (ib >= n_batch) return;
    i = (uint32_t)ib;
    r = inv[ib];
    if (r < 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        g_means[3 * i + k] = 0.f;
        g_color[3 * i + k] = 0.f;
        g_scale[3 * i + k] = 0.f;
        g_normal[3 * i + k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) g_quat[4 * i + k] = 0.f;
      g_opacity[i] = 0.f;
      return;
    }
  } else {
    r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    i = rec[r].src;
  }
  const float *G = gs + (size_t)13 * r;
  const double mu[3] = {means[3 * i + 0], means[3 * i + 1], means[3 * i + 2]};
  const float *sc = scale + 3 * i;
  const float *q = quat + 4 * i;
  ProjGeom g;
  proj_geom(cam, mu, sc, q, g);
  const double x = g.x, y = g.y, z = g.z;
  const double zi = 1.0 / z;
  // ---- conic -> (a, b, c)
  const double gA = G[2], gB = G[3], gC = G[4];
  const double idet = 1.0 / g.det;
  const double gdet = -(gA * g.c - gB * g.b + gC * g.a) * idet * idet;
  const double ga = gC * idet + gdet * g.c;
  const double gc = gA * idet + gdet * g.a;
  const double gb = -gB * idet - 2.0 * gdet * g.b;
  // symmetric cov2d cotangent Gs = [[ga, gb/2], [gb/2, gc]]
  const double G00 = ga, G01 = 0.5 * gb, G11 = gc;
  // J rows: j0 = (J00, 0, J02), j1 = (0, J11, J12)
  const double j0[3] = {g.J00, 0.0, g.J02}, j1[3] = {0.0, g.J11, g.J12};
  const double S[9] = {g.S[0], g.S[1], g.S[2], g.S[1], g.S[3], g.S[4], g.S[2], g.S[4], g.S[5]};
  // g_J = 2 Gs J S  (2x3)
  double JS0[3], JS1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    JS0[k] = j0[0] * S[k] + j0[1] * S[3 + k] + j0[2] * S[6 + k];
    JS1[k] = j1[0] * S[k] + j1[1] * S[3 + k] + j1[2] * S[6 + k];
  }
  const double gJ00 = 2.0 * (G00 * JS0[0] + G01 * JS1[0]);
  const double gJ02 = 2.0 * (G00 * JS0[2] + G01 * JS1[2]);
  const double gJ11 = 2.0 * (G01 * JS0[1] + G11 * JS1[1]);
  const double gJ12 = 2.0 * (G01 * JS0[2] + G11 * JS1[2]);
  // g_S = J^T Gs J (3x3 symmetric)
  double gS[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      gS[3 * a + b] = j0[a] * (G00 * j0[b] + G01 * j1[b]) + j1[a] * (G01 * j0[b] + G11 * j1[b]);
  // ---- mu_cam cotangent
  double gx = 0.0, gy = 0.0, gz = 0.0;
  const double gu = G[0], gv = G[1];
  gx += gu * cam.fx * zi;
  gy += gv * cam.fy * zi;
  gz += -gu * cam.fx * x * zi * zi - gv * cam.fy * y * zi * zi;
  gz += -gJ00 * cam.fx * zi * zi - gJ11 * cam.fy * zi * zi;
  gx += -gJ02 * cam.fx * zi * zi;
  gz += gJ02 * 2.0 * cam.fx * x * zi * zi * zi;
  gy += -gJ12 * cam.fy * zi * zi;
  gz += gJ12 * 2.0 * cam.fy * y * zi * zi * zi;
  // plane_d = n_c . mu_c, n_c = fl * R n
  const double nw[3] = {normal[3 * i + 0], normal[3 * i + 1], normal[3 * i + 2]};
  double nc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) nc[k] = cam.r[3 * k + 0] * nw[0] + cam.r[3 * k + 1] * nw[1] + cam.r[3 * k + 2] * nw[2];
  const double fl = (nc[0] * x + nc[1] * y + nc[2] * z) > 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) nc[k] *= fl;
  const double gpd = G[12];
  gx += gpd * nc[0];
  gy += gpd * nc[1];
  gz += gpd * nc[2];
  const double gnc[3] = {G[9] + gpd * x, G[10] + gpd * y, G[11] + gpd * z};
  // mu = R^T mu_c cotangent; n = fl R^T gnc
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g_means[3 * i + k] = (float)(cam.r[0 + k] * gx + cam.r[3 + k] * gy + cam.r[6 + k] * gz);
    g_normal[3 * i + k] = (float)(fl * (cam.r[0 + k] * gnc[0] + cam.r[3 + k] * gnc[1] + cam.r[6 + k] * gnc[2]));
  }
  // ---- Sigma_c = M D M^T, M = R Rq: gM = 2 gS M D ; gD_k = (M^T gS M)_kk
  double gM[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      gM[3 * a + k] = 2.0 * (gS[3 * a + 0] * g.M[0 + k] + gS[3 * a + 1] * g.M[3 + k] +
                             gS[3 * a + 2] * g.M[6 + k]) * g.s2[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) d += g.M[3 * a + k] * gS[3 * a + b] * g.M[3 * b + k];
    g_scale[3 * i + k] = (float)(d * 2.0 * (double)sc[k]);
  }
  // gRq = R^T gM
  double gRq[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      gRq[3 * a + k] = cam.r[0 + a] * gM[0 + k] + cam.r[3 + a] * gM[3 + k] + cam.r[6 + a] * gM[6 + k];
  const double w = q[0], qx = q[1], qy = q[2], qz = q[3];
  const double *Gq = gRq;
  g_quat[4 * i + 0] = (float)(2.0 * (-qz * Gq[1] + qy * Gq[2] + qz * Gq[3] - qx * Gq[5] - qy * Gq[6] + qx * Gq[7]));
  g_quat[4 * i + 1] = (float)(2.0 * (qy * Gq[1] + qz * Gq[2] + qy * Gq[3] - 2.0 * qx * Gq[4] - w * Gq[5] + qz * Gq[6] + w * Gq[7] - 2.0 * qx * Gq[8]));
  g_quat[4 * i + 2] = (float)(2.0 * (-2.0 * qy * Gq[0] + qx * Gq[1] + w * Gq[2] + qx * Gq[3] + qz * Gq[5] - w * Gq[6] + qz * Gq[7] - 2.0 * qy * Gq[8]));
  g_quat[4 * i + 3] = (float)(2.0 * (-2.0 * qz * Gq[0] - w * Gq[1] + qx * Gq[2] + w * Gq[3] - 2.0 * qz * Gq[4] + qy * Gq[5] + qx * Gq[6] + qy * Gq[7]));
  g_opacity[i] = G[5];
  g_color[3 * i + 0] = G[6];
  g_color[3 * i + 1] = G[7];
  g_color[3 * i + 2] = G[8];
}

__global__ void splat_rank_kernel(const vsx_splat *__restrict__ rec,
                                  const int32_t *__restrict__ src, int32_t n,
                                  int32_t *__restrict__ inv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) inv[src ? (uint32_t)src[r] : rec[r].src] = r;
}

}  // namespace vsx

using namespace vsx;

extern "C" int vsx_project_fwd(const double *means, const float *opacity, const float *color,
                               const float *scale, const float *quat, const float *normal,
                               int32_t n, vsx_camera cam, vsx_splat *rec, uint64_t *zkey,
                               double *radius, uint32_t *n_kept, int32_t *status, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "project_fwd: negative n");
  cudaStream_t st = as_stream(s);
  VSX_CUDA_TRY(cudaMemsetAsync(n_kept, 0, sizeof(uint32_t), st));
  if (n == 0) return VSX_OK;
  project_fwd_kernel<<<grid_for(n, 256), 256, 0, st>>>(means, opacity, color, scale, quat, normal,
                                                       n, cam, rec, zkey, radius, n_kept, status);
  VSX_LAUNCH_CHECK("project_fwd");
  return VSX_OK;
}

extern "C" int vsx_gather_splats(const vsx_splat *rec, const double *radius,
                                 const uint32_t *order, int32_t n, vsx_splat *rec_sorted,
                                 double *radius_sorted, vsx_stream s) {
  if (n <= 0) return VSX_OK;
  gather_splats_kernel<<<grid_for((int64_t)4 * n, 256), 256, 0, as_stream(s)>>>(
      rec, radius, order, n, rec_sorted, radius_sorted);
  VSX_LAUNCH_CHECK("gather_splats");
  return VSX_OK;
}

namespace vsx {
// C1 payload rows: 6 x 16-byte pieces per 96-byte row (record, then
// (z, radius), then (gid, pad)); one thread per piece, coalesced stores.
__global__ void pack_splat_rows_kernel(const vsx_splat *__restrict__ rec,
                                       const double *__restrict__ z,
                                       const double *__restrict__ radius,
                                       const int64_t *__restrict__ gid, int32_t n,
                                       uint8_t *__restrict__ out) {
  const int64_t tq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = tq / 6;
  const int part = (int)(tq - 6 * i);
  if (i >= n) return;
  longlong2 v;
  if (part < 4) {
    v = __ldg(reinterpret_cast<const longlong2 *>(rec) + 4 * i + part);
  } else if (part == 4) {
    v = make_longlong2(__double_as_longlong(z[i]), __double_as_longlong(radius[i]));
  } else {
    v = make_longlong2(gid[i], 0);
  }
  reinterpret_cast<longlong2 *>(out + i * VSX_SPLAT_ROW_BYTES)[part] = v;
}

__global__ void splat_rows_keys_kernel(const uint8_t *__restrict__ rows,
                                       const int32_t *__restrict__ rowmap, int32_t n,
                                       double *__restrict__ z, int64_t *__restrict__ gid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = rowmap ? rowmap[i] : i;
  const longlong2 *row = reinterpret_cast<const longlong2 *>(rows + r * VSX_SPLAT_ROW_BYTES);
  z[i] = __longlong_as_double(row[4].x);
  gid[i] = row[5].x;
}

__global__ void gather_splat_rows_kernel(const uint8_t *__restrict__ rows,
                                         const int32_t *__restrict__ rowmap,
                                         const uint32_t *__restrict__ order, int32_t n,
                                         vsx_splat *__restrict__ out, double *__restrict__ rout) {
  const int64_t tq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = tq >> 2;
  const int part = (int)(tq & 3);
  if (i >= n) return;
  const uint32_t j = order[i];
  const int64_t r = rowmap ? rowmap[j] : (int64_t)j;
  const float4 *row = reinterpret_cast<const float4 *>(rows + r * VSX_SPLAT_ROW_BYTES);
  reinterpret_cast<float4 *>(out)[4 * i + part] = __ldg(row + part);
  if (part == 0) rout[i] = __longlong_as_double(reinterpret_cast<const longlong2 *>(row)[4].y);
}

// Owner-side payload keys of the sharded step: for kept splat i (decode
// batch index src[i]) the global gaussian id active[src / n] * n + src % n
// and its float64 z bits.
__global__ void payload_keys_kernel(const int32_t *__restrict__ active,
                                    const uint32_t *__restrict__ src,
                                    const uint64_t *__restrict__ key, int32_t n_kept, int32_t n,
                                    int64_t *__restrict__ gid, uint64_t *__restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_kept) return;
  const uint32_t s = src[i];
  gid[i] = (int64_t)active[s / (uint32_t)n] * n + (int64_t)(s % (uint32_t)n);
  z[i] = key[s];
}

}  // namespace vsx

extern "C" int vsx_payload_keys(const int32_t *active, const uint32_t *src, const uint64_t *key,
                                int32_t n_kept, int32_t n, int64_t *gid, uint64_t *z,
                                vsx_stream s) {
  VSX_REQUIRE(n_kept >= 0 && n >= 1, "payload_keys: bad arguments");
  if (n_kept == 0) return VSX_OK;
  VSX_REQUIRE(active && src && key && gid && z, "payload_keys: null pointer");
  payload_keys_kernel<<<grid_for(n_kept, 256), 256, 0, as_stream(s)>>>(active, src, key, n_kept,
                                                                      n, gid, z);
  VSX_LAUNCH_CHECK("payload_keys");
  return VSX_OK;
}

extern "C" int vsx_pack_splat_rows(const vsx_splat *rec, const double *z, const double *radius,
                                   const int64_t *gid, int32_t n, uint8_t *out, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "pack_splat_rows: n < 0");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(rec && z && radius && gid && out, "pack_splat_rows: null pointer");
  VSX_REQUIRE(((uintptr_t)out & 15) == 0, "pack_splat_rows: out not 16-byte aligned");
  pack_splat_rows_kernel<<<grid_for((int64_t)6 * n, 256), 256, 0, as_stream(s)>>>(
      rec, z, radius, gid, n, out);
  VSX_LAUNCH_CHECK("pack_splat_rows");
  return VSX_OK;
}

extern "C" int vsx_splat_rows_keys(const uint8_t *rows, const int32_t *rowmap, int32_t n,
                                   double *z, int64_t *gid, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "splat_rows_keys: n < 0");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(rows && z && gid, "splat_rows_keys: null pointer");
  splat_rows_keys_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(rows, rowmap, n, z, gid);
  VSX_LAUNCH_CHECK("splat_rows_keys");
  return VSX_OK;
}

extern "C" int vsx_gather_splat_rows(const uint8_t *rows, const int32_t *rowmap,
                                     const uint32_t *order, int32_t n, vsx_splat *rec_sorted,
                                     double *radius_sorted, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "gather_splat_rows: n < 0");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(rows && order && rec_sorted && radius_sorted, "gather_splat_rows: null pointer");
  VSX_REQUIRE(((uintptr_t)rows & 15) == 0, "gather_splat_rows: rows not 16-byte aligned");
  gather_splat_rows_kernel<<<grid_for((int64_t)4 * n, 256), 256, 0, as_stream(s)>>>(
      rows, rowmap, order, n, rec_sorted, radius_sorted);
  VSX_LAUNCH_CHECK("gather_splat_rows");
  return VSX_OK;
}

extern "C" int vsx_bin_count(const vsx_splat *rec, const double *radius, int32_t n,
                             int32_t width, int32_t height, uint32_t *splat_tiles,
                             uint32_t *tile_counts, vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0, "bin_count: bad arguments");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  cudaStream_t st = as_stream(s);
  if (tile_counts) VSX_CUDA_TRY(cudaMemsetAsync(tile_counts, 0, sizeof(uint32_t) * txn * tyn, st));
  if (n == 0) return VSX_OK;
  bin_count_kernel<<<grid_for(n, 256), 256, 0, st>>>(rec, radius, n, txn, tyn, splat_tiles,
                                                     tile_counts);
  VSX_LAUNCH_CHECK("bin_count");
  return VSX_OK;
}

extern "C" int vsx_bin_emit(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                            int32_t height, const uint32_t *splat_offsets, uint32_t *isect_tile,
                            uint32_t *isect_rank, vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0, "bin_emit: bad arguments");
  if (n == 0) return VSX_OK;
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  static const bool warp_emit = [] {  // VSX_BIN_EMIT=warp: the warp-walk kernel (A/B)
    const char *e = getenv("VSX_BIN_EMIT");
    return e && e[0] == 'w';
  }();
  if (warp_emit)
    bin_emit_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(rec, radius, n, txn, tyn,
                                                                splat_offsets, isect_tile,
                                                                isect_rank);  // whole warps
  else
    bin_emit_block_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
        rec, radius, n, txn, tyn, splat_offsets, isect_tile, isect_rank, nullptr);
  VSX_LAUNCH_CHECK("bin_emit");
  return VSX_OK;
}

extern "C" int vsx_bin_emit_hist(const vsx_splat *rec, const double *radius, int32_t n,
                                 int32_t width, int32_t height, const uint32_t *splat_offsets,
                                 uint32_t *isect_tile, uint32_t *isect_rank, uint32_t *hist,
                                 vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0 && hist, "bin_emit_hist: bad arguments");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  VSX_REQUIRE((int64_t)txn * tyn <= 65536, "bin_emit_hist: more than 2^16 tiles");
  cudaStream_t st = as_stream(s);
  VSX_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 2 * 256, st));
  if (n == 0) return VSX_OK;
  bin_emit_block_kernel<<<grid_for(n, 256), 256, 0, st>>>(rec, radius, n, txn, tyn, splat_offsets,
                                                          isect_tile, isect_rank, hist);
  VSX_LAUNCH_CHECK("bin_emit_hist");
  return VSX_OK;
}

extern "C" int vsx_tile_ranges(const uint32_t *sorted_tiles, int64_t n, int32_t num_tiles,
                               uint32_t *tile_offsets, vsx_stream s) {
  VSX_REQUIRE(n >= 0 && num_tiles >= 1, "tile_ranges: bad args");
  tile_ranges_kernel<<<grid_for(num_tiles + 1, 256), 256, 0, as_stream(s)>>>(
      sorted_tiles, n, num_tiles, tile_offsets);
  VSX_LAUNCH_CHECK("tile_ranges");
  return VSX_OK;
}

__global__ void tile_max_len_kernel(const uint32_t *__restrict__ tile_off, int T,
                                    uint32_t *__restrict__ max_len) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t len = t < T ? tile_off[t + 1] - tile_off[t] : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  if ((threadIdx.x & 31) == 0 && len) atomicMax(max_len, len);
}

extern "C" int vsx_tile_max_len(const uint32_t *tile_offsets, int32_t num_tiles,
                                uint32_t *max_len, vsx_stream s) {
  VSX_REQUIRE(num_tiles >= 1 && max_len, "tile_max_len: bad args");
  tile_max_len_kernel<<<grid_for(num_tiles, 256), 256, 0, as_stream(s)>>>(tile_offsets,
                                                                          num_tiles, max_len);
  VSX_LAUNCH_CHECK("tile_max_len");
  return VSX_OK;
}

extern "C" int vsx_bin_emit_tiles(const vsx_splat *rec, const double *radius, int32_t n,
                                  int32_t width, int32_t height, const uint32_t *tile_offsets,
                                  uint32_t *cursor, uint32_t *tile_list, vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0, "bin_emit_tiles: bad arguments");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  cudaStream_t st = as_stream(s);
  VSX_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * txn * tyn, st));
  if (n == 0) return VSX_OK;
  bin_emit_tiles_kernel<<<grid_for(n, 256), 256, 0, st>>>(rec, radius, n, txn, tyn, tile_offsets,
                                                          cursor, tile_list);
  VSX_LAUNCH_CHECK("bin_emit_tiles");
  return VSX_OK;
}

extern "C" int vsx_tile_segsort(const uint32_t *tile_offsets, int32_t num_tiles,
                                uint32_t *tile_list, int32_t max_len, vsx_stream s) {
  VSX_REQUIRE(num_tiles >= 1, "tile_segsort: bad num_tiles");
  if (max_len > kSegCap) {
    vsx_set_error("tile_segsort: tile list of %d > %d entries", max_len, kSegCap);
    return VSX_ERR_CAPACITY;
  }
  tile_segsort_kernel<<<num_tiles, 256, 0, as_stream(s)>>>(tile_offsets, tile_list);
  VSX_LAUNCH_CHECK("tile_segsort");
  return VSX_OK;
}

extern "C" int vsx_project_bwd(const double *means, const float *scale, const float *quat,
                               const float *normal, const vsx_splat *rec_sorted,
                               const float *grad_splat, int32_t n_sorted, vsx_camera cam,
                               float *g_means, float *g_opacity, float *g_color, float *g_scale,
                               float *g_quat, float *g_normal, vsx_stream s) {
  if (n_sorted <= 0) return VSX_OK;
  project_bwd_kernel<false><<<grid_for(n_sorted, 128), 128, 0, as_stream(s)>>>(
      means, scale, quat, normal, rec_sorted, grad_splat, n_sorted, cam, g_means, g_opacity,
      g_color, g_scale, g_quat, g_normal, nullptr, 0);
  VSX_LAUNCH_CHECK("project_bwd");
  return VSX_OK;
}

extern "C" int vsx_project_bwd_batch(const double *means, const float *scale, const float *quat,
                                     const float *normal, const vsx_splat *rec_sorted,
                                     const float *grad_splat, int32_t n_sorted, int32_t n_batch,
                                     vsx_camera cam, float *g_means, float *g_opacity,
                                     float *g_color, float *g_scale, float *g_quat,
                                     float *g_normal, const int32_t *src_sorted, int32_t *inv_ws,
                                     vsx_stream s) {
  VSX_REQUIRE(n_sorted >= 0 && n_batch >= n_sorted && inv_ws, "project_bwd_batch: bad args");
  if (n_batch == 0) return VSX_OK;
  cudaStream_t st = as_stream(s);
  VSX_CUDA_TRY(cudaMemsetAsync(inv_ws, 0xFF, sizeof(int32_t) * n_batch, st));
  if (n_sorted > 0) {
    splat_rank_kernel<<<grid_for(n_sorted, 256), 256, 0, st>>>(rec_sorted, src_sorted, n_sorted,
                                                                inv_ws);
    VSX_LAUNCH_CHECK("splat_rank");
  }
  project_bwd_kernel<true><<<grid_for(n_batch, 128), 128, 0, st>>>(
      means, scale, quat, normal, rec_sorted, grad_splat, n_sorted, cam, g_means, g_opacity,
      g_color, g_scale, g_quat, g_normal, inv_ws, n_batch);
  VSX_LAUNCH_CHECK("project_bwd");
  return VSX_OK;
}
