// K5 / K6 — per-tile front-to-back RGB-D-N compositing and its backward.
//
// Forward restates voxsplat renderer.py:242-301 (_blend_padded + _finalize)
// and :390-449 (rasterize_view): one CTA of 128 threads per 16x16 tile, two
// horizontally adjacent pixels per thread as float2 lanes of paired FP32
// instructions (FFMA2 / FMUL2 / FADD2), splat records staged through
// shared memory in chunks of 256, CTA-wide early exit once every pixel's
// transmittance fell below 1e-4 (__syncthreads_count). Semantics that differ
// from stock 3DGS and are kept exactly: every binned splat contributes (no
// 1/255 skip, no per-pixel 3-sigma cut), power is clamped at 0, alpha is
// clamped at 0.99, a splat is live iff T_prev >= 1e-4.
//
// Backward (raster_bwd_tc_kernel) walks each tile back to front from the
// per-pixel live count, recovering T_k = T_{k+1} / (1 - alpha_k) from the
// stored final transmittance (the stable direction; SURVEY.md §7 backward
// note), in chunks of 16 splats:
//   phase 0 (tensor cores): the per-(pixel, splat) cotangent dot
//            s = F[p] . P[j], a [256 x 8] . [8 x 16] product (3xTF32);
//   phase 1 (thread = pixel): the sequential back-to-front recursion, writing
//            w = alpha*T and q = dL/d(alpha_unclamped) * exp(power) to two
//            shared-memory planes; the alphas of a splat pair are the lanes
//            of paired FP32 instructions;
//   phase 2 (tensor cores): the per-splat sums over the tile's 256 pixels,
//            [16 x 256] . [256 x 8] GEMMs of the w plane against the colour /
//            normal / plane cotangents and of the q plane against the pixel
//            moments (1, x, y, x^2, xy, y^2), then 13 float atomics per
//            (splat, tile) from closed-form polynomials of the moments.
// Records are prefetched one chunk ahead with cp.async; the next chunk is
// staged right after phase 2 (double-buffered), two CTA barriers per chunk.
// The measured alternatives (pixel-per-thread forward, a tensor-core
// forward, an FFMA phase 2, a warp-specialised backward) are in DESIGN.md §6.
#include <cuda_fp16.h>

#include "raster_common.cuh"

namespace vsx {

#ifndef VSX_FWD_CHUNK
#define VSX_FWD_CHUNK 256
#endif
constexpr int kChunk = VSX_FWD_CHUNK;

// Per-pixel finalize (renderer.py:282-301) + fused loss partial sums (K9),
// shared by both forward kernels. Block-uniform in L.gt_rgb.
template <bool kDet>
__device__ __forceinline__ void fwd_epilogue(const vsx_camera &cam, bool inside, int px, int py,
                                             float acc, float c0, float c1, float c2, float n0,
                                             float n1, float n2, float dist, float T, int32_t nc,
                                             float *__restrict__ out_rgb,
                                             float *__restrict__ out_alpha,
                                             float *__restrict__ out_depth,
                                             float *__restrict__ out_normal,
                                             float *__restrict__ out_raw,
                                             uint8_t *__restrict__ out_valid,
                                             float *__restrict__ out_T,
                                             int32_t *__restrict__ out_nc,
                                             const vsx_loss_desc &L) {
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
  if (L.live_pairs) {  // block-uniform
    unsigned long long lp = inside ? (unsigned long long)nc : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o);
    if ((threadIdx.x & 31) == 0 && lp) atomicAdd(L.live_pairs, lp);
  }
  if (L.gt_rgb) {  // block-uniform
    l_rgb = warp_sum_d(l_rgb);
    l_dep = warp_sum_d(l_dep);
    l_nrm = warp_sum_d(l_nrm);
    const unsigned bd = __ballot_sync(0xffffffffu, c_dep), bn = __ballot_sync(0xffffffffu, c_nrm);
    if ((threadIdx.x & 31) == 0) {
      if (kDet) {
        // deterministic mode: one slot per (tile, warp), reduced in order by
        // vsx_reduce_partials (the counts are integers: atomics are exact)
        const size_t slot = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * (blockDim.x / 32) +
                            (threadIdx.x >> 5);
        // += : a thread finalizes PX pixels, one epilogue call each, in order
        // (the buffer is zeroed by the caller)
        L.sum_partials[3 * slot + 0] += l_rgb;
        L.sum_partials[3 * slot + 1] += l_dep;
        L.sum_partials[3 * slot + 2] += l_nrm;
      } else {
        if (l_rgb != 0.0) atomicAdd(L.sums + 0, l_rgb);
        if (bd) atomicAdd(L.sums + 1, l_dep);
        if (bn) atomicAdd(L.sums + 2, l_nrm);
      }
      if (bd) atomicAdd(L.counts + 0, (uint32_t)__popc(bd));
      if (bn) atomicAdd(L.counts + 1, (uint32_t)__popc(bn));
    }
  }
}

__device__ __forceinline__ void copy_splat_async(vsx_splat *dst, const vsx_splat *src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * k),
                 "l"(reinterpret_cast<const char *>(src) + 16 * k)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Forward: one CTA of 128 threads per tile, two horizontally adjacent pixels
// per thread held as the lanes of float2 registers and advanced with the
// sm_100 paired FP32 instructions (FFMA2 / FMUL2 / FADD2; the staged splat
// value is the broadcast operand). Records are staged through shared memory
// kChunk at a time; per staged splat the two pixels share its loads and the dy
// terms of the falloff; the alphas of U splats are evaluated before the
// serial transmittance chain. Every lane performs the scalar operations with
// the same roundings (fma / mul / add are each correctly rounded), so alpha
// and T agree bit for bit with the backward's recompute. The scalar
// two-pixel kernel this replaced was issue-bound at 84% with 26 instructions
// per (pixel, splat) (profiles/r02_raster_final_ncu.txt); pairing removes a
// third of them (profiles/r02_raster_fwd_pk_ncu.txt).
__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }

struct FwdPair {
  float2 T = {1.f, 1.f}, acc = {0.f, 0.f}, c0 = {0.f, 0.f}, c1 = {0.f, 0.f}, c2 = {0.f, 0.f},
         n0 = {0.f, 0.f}, n1 = {0.f, 0.f}, n2 = {0.f, 0.f}, dist = {0.f, 0.f};
  // 1 + the chunk index of the last splat blended while live (T only
  // decreases, so the live splats are a prefix): one select per lane
  int32_t nl0 = 0, nl1 = 0;
  __device__ __forceinline__ void blend_if_live(float2 al, const float4 &p2, const float4 &p3,
                                                float pd, int32_t idx1) {
    const bool l0 = T.x >= kEarlyStopT, l1 = T.y >= kEarlyStopT;
    const float2 m = make_float2(l0 ? al.x : 0.f, l1 ? al.y : 0.f);
    const float2 w = __fmul2_rn(m, T);
    acc = __fadd2_rn(acc, w);
    c0 = __ffma2_rn(w, bc2(p2.x), c0);
    c1 = __ffma2_rn(w, bc2(p2.y), c1);
    c2 = __ffma2_rn(w, bc2(p2.z), c2);
    n0 = __ffma2_rn(w, bc2(p3.x), n0);
    n1 = __ffma2_rn(w, bc2(p3.y), n1);
    n2 = __ffma2_rn(w, bc2(p3.z), n2);
    dist = __ffma2_rn(w, bc2(pd), dist);
    T = __ffma2_rn(make_float2(-m.x, -m.y), T, T);
    nl0 = l0 ? idx1 : nl0;
    nl1 = l1 ? idx1 : nl1;
  }
};

__device__ __forceinline__ float2 falloff_alpha2(const float4 &p0, const float4 &p1, float2 fx,
                                                 float cy, float cyy) {
  const float2 dx = __fadd2_rn(fx, bc2(-p0.x));
  const float2 q = __ffma2_rn(bc2(p0.z), dx, bc2(cy));
  const float2 p = __ffma2_rn(q, dx, bc2(cyy));
  const float2 e = make_float2(ex2_ftz(fminf(p.x, 0.f)), ex2_ftz(fminf(p.y, 0.f)));
  const float2 a = __fmul2_rn(bc2(p1.y), e);
  return make_float2(fminf(a.x, 0.99f), fminf(a.y, 0.99f));
}

#ifndef VSX_FWD_PK_MINB
#define VSX_FWD_PK_MINB 1
#endif
template <int U, bool kDet>
__global__ void __launch_bounds__(128, VSX_FWD_PK_MINB) raster_fwd_pk_kernel(
    const vsx_splat *__restrict__ rec, const uint32_t *__restrict__ tile_off,
    const uint32_t *__restrict__ tile_list, vsx_camera cam, float *__restrict__ out_rgb,
    float *__restrict__ out_alpha, float *__restrict__ out_depth, float *__restrict__ out_normal,
    float *__restrict__ out_raw, uint8_t *__restrict__ out_valid, float *__restrict__ out_T,
    int32_t *__restrict__ out_nc, vsx_loss_desc L) {
  constexpr int kThreads = 128, kRowThreads = kTile / 2;
  __shared__ float4 s0[kChunk], s1[kChunk], s2[kChunk], s3[kChunk];
  const int txn = gridDim.x;
  const int by = (int)blockIdx.y + L.tile_row0;
  const int tile = by * txn + blockIdx.x;
  const int lx = 2 * (threadIdx.x % kRowThreads), ly = threadIdx.x / kRowThreads;
  const int px = blockIdx.x * kTile + lx, py = by * kTile + ly;
  const double ox = (double)(blockIdx.x * kTile), oy = (double)(by * kTile);
  const uint32_t begin = tile_off[tile], end = tile_off[tile + 1];
  const float fy = (float)ly;
  const float2 fx = make_float2((float)lx, (float)(lx + 1));
  const bool in0 = px < cam.width && py < cam.height, in1 = px + 1 < cam.width && py < cam.height;
  bool done0 = !in0, done1 = !in1;
  int32_t nc0 = 0, nc1 = 0;
  FwdPair A;
  for (uint32_t cs = begin; cs < end; cs += kChunk) {
    if (__syncthreads_count(!(done0 && done1)) == 0) break;
#pragma unroll
    for (int h = 0; h < kChunk / kThreads; ++h) {
      const int k = threadIdx.x + kThreads * h;
      const uint32_t idx = cs + k;
      if (idx < end) {
        const vsx_splat sp = load_splat(rec, tile_list[idx]);
        stage_splat(sp, ox, oy, s0[k], s1[k], s2[k], s3[k]);
      }
    }
    __syncthreads();
    const int cnt = (int)min((uint32_t)kChunk, end - cs);
    if (!(done0 && done1)) {
      A.nl0 = A.nl1 = 0;
      int j = 0;
      for (; j + U <= cnt && fmaxf(A.T.x, A.T.y) >= kEarlyStopT; j += U) {
        float2 al[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float4 p0 = s0[j + u], p1 = s1[j + u];
          const float dy = fy - p0.y;
          const float cy = __fmul_rn(p0.w, dy), cyy = __fmul_rn(__fmul_rn(p1.x, dy), dy);
          al[u] = falloff_alpha2(p0, p1, fx, cy, cyy);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          A.blend_if_live(al[u], s2[j + u], s3[j + u], s1[j + u].z, j + u + 1);
      }
      for (; j < cnt && fmaxf(A.T.x, A.T.y) >= kEarlyStopT; ++j) {
        const float4 p0 = s0[j], p1 = s1[j];
        const float dy = fy - p0.y;
        const float cy = __fmul_rn(p0.w, dy), cyy = __fmul_rn(__fmul_rn(p1.x, dy), dy);
        A.blend_if_live(falloff_alpha2(p0, p1, fx, cy, cyy), s2[j], s3[j], p1.z, j + 1);
      }
      if (!done0) {
        nc0 = (int32_t)(cs - begin) + A.nl0;
        done0 = A.T.x < kEarlyStopT;
      }
      if (!done1) {
        nc1 = (int32_t)(cs - begin) + A.nl1;
        done1 = A.T.y < kEarlyStopT;
      }
    }
  }
  fwd_epilogue<kDet>(cam, in0, px, py, A.acc.x, A.c0.x, A.c1.x, A.c2.x, A.n0.x, A.n1.x, A.n2.x,
                     A.dist.x, A.T.x, nc0, out_rgb, out_alpha, out_depth, out_normal, out_raw,
                     out_valid, out_T, out_nc, L);
  fwd_epilogue<kDet>(cam, in1, px + 1, py, A.acc.y, A.c0.y, A.c1.y, A.c2.y, A.n0.y, A.n1.y,
                     A.n2.y, A.dist.y, A.T.y, nc1, out_rgb, out_alpha, out_depth, out_normal,
                     out_raw, out_valid, out_T, out_nc, L);
}

__device__ __forceinline__ void mma_m16n8k8_tf32(float (&d)[4], const uint32_t (&a)[4],
                                                 uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// tf32 by truncation: one LOP3 (cvt.rna.tf32 is a 4-instruction sequence on
// sm_100a). With x = hi + (x - hi), the dropped bits of lo cost < 2^-21 |x|.
__device__ __forceinline__ uint32_t tf32_bits(float x) {
  return __float_as_uint(x) & 0xffffe000u;
}

// tf32 by rounding to nearest (ties away from zero): one IADD more. With hi
// rounded, |x - hi| <= 2^-11 |x| and the rounded lo leaves < 2^-22 |x|: the
// 3xTF32 product then carries float32-level error (truncation leaves up to
// 2^-20, which cancelling per-splat sums amplify past the 1e-3 bar).
__device__ __forceinline__ uint32_t tf32_rn(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}
#ifndef VSX_BWD_RN2
#define VSX_BWD_RN2 1
#endif

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

// ------------------------------------------------------- backward v3 (tensor)
//
// Phase 2 of v2 is two small GEMMs per chunk of kBC splats:
//   Gsum[j][f] = sum_p W[j][p] * Gw[p][f]   f = (rgb, raw normal, plane) cotangents
//   Mom[j][m]  = sum_p Q[j][p] * Mq[p][m]   m = (1, x, y, x^2, xy, y^2) about the centre
// run here on the tensor cores with mma.sync m16n8k8 tf32 (A = the w / q
// planes written by phase 1, B = per-tile constants). Precision is kept at
// fp32 level with the 3xTF32 split (a_hi b_hi + a_hi b_lo + a_lo b_hi) for
// Gw; Mq holds multiples of 1/4 below 64, exact in tf32, so q needs only
// a_hi + a_lo. Warps split (m-tile, plane, k-range); the KSPLIT partial sums
// meet in shared memory and one 8-lane group per splat forms its 13
// gradients (same polynomials as v2) and issues the atomics.
#ifndef VSX_BWD_KR7
#define VSX_BWD_KR7 5
#endif
#ifndef VSX_BWD_STAGE_WARP
#define VSX_BWD_STAGE_WARP 7
#endif
#ifndef VSX_BWD_SORTPIX
#define VSX_BWD_SORTPIX 1
#endif
#ifndef VSX_BWD_P0SKIP
#define VSX_BWD_P0SKIP 1
#endif
#ifndef VSX_BWD_MERGED
#define VSX_BWD_MERGED 1
#endif
#ifndef VSX_BWD_PREFIX
#define VSX_BWD_PREFIX 1
#endif
#ifndef VSX_BWD_EPI_HI
#define VSX_BWD_EPI_HI 1
#endif
// 4 CTAs per SM (56 KB of shared memory, 64 registers): the per-tile B
// fragments of phase 2 are kept raw and split per k-step (cotangents) or as
// exact half2 (pixel moments), the partial-sum rows are 18 floats, the
// prologue's sort scratch lives in the not yet used q plane.
#ifndef VSX_BWD_OCC4
#define VSX_BWD_OCC4 1
#endif
constexpr int kRedStride = VSX_BWD_OCC4 ? 18 : 24;
constexpr int kPlaneStride = kTilePixels + 4;  // 4 mod 32: conflict-free A fragments

// pixel moment m of tile pixel p (x, y about the tile centre)
__device__ __forceinline__ float pixel_moment(int p, int m) {
  const float xc = (float)(p & 15) - 7.5f, yc = (float)(p >> 4) - 7.5f;
  switch (m) {
    case 0: return 1.f;
    case 1: return xc;
    case 2: return yc;
    case 3: return xc * xc;
    case 4: return xc * yc;
    case 5: return yc * yc;
    default: return 0.f;
  }
}

// Phase 1 on splat pairs: the alphas of splats 2i and 2i + 1 are evaluated
// as the two lanes of paired FP32 instructions (FFMA2 / FMUL2 / FADD2) from
// the pair-interleaved staging sP; the T / S recursion stays sequential
// (T_2i+1 first, back to front). Per lane the operations and roundings are
// the scalar ones (splat_alpha), so alpha and T agree bit for bit with the
// forward. Writes w and q of rows [0, jlive) of this thread's plane column.
__device__ __forceinline__ void pair_alpha(const float4 (&P)[3], float fx, float fy, float2 &al,
                                           float2 &e, float2 &at) {
  const float2 dx = __fadd2_rn(bc2(fx), make_float2(P[0].x, P[0].y));
  const float2 dy = __fadd2_rn(bc2(fy), make_float2(P[0].z, P[0].w));
  const float2 cy = __fmul2_rn(make_float2(P[1].z, P[1].w), dy);
  const float2 cyy = __fmul2_rn(__fmul2_rn(make_float2(P[2].x, P[2].y), dy), dy);
  const float2 q = __ffma2_rn(make_float2(P[1].x, P[1].y), dx, cy);
  const float2 p = __ffma2_rn(q, dx, cyy);
  e = make_float2(ex2_ftz(fminf(p.x, 0.f)), ex2_ftz(fminf(p.y, 0.f)));
  at = __fmul2_rn(make_float2(P[2].z, P[2].w), e);
  al = make_float2(fminf(at.x, 0.99f), fminf(at.y, 0.99f));
}

__device__ __forceinline__ void bwd_phase1_pairs(const float4 (*__restrict__ sP)[3],
                                                 float *__restrict__ wpl, float *__restrict__ qpl,
                                                 int t, int jlive, float fx, float fy, float &T,
                                                 float &S) {
  int j = jlive - 1;
  if (j >= 0 && !(j & 1)) {  // an even top row: lane .x of its pair, alone
    const float *pp = reinterpret_cast<const float *>(&sP[j >> 1][0]);
    const float dx = fx + pp[0], dy = fy + pp[2];
    const float q = __fmaf_rn(pp[4], dx, __fmul_rn(pp[6], dy));
    const float p2 = __fmaf_rn(q, dx, __fmul_rn(__fmul_rn(pp[8], dy), dy));
    const float e = ex2_ftz(fminf(p2, 0.f));
    const float at = __fmul_rn(pp[10], e);
    const float alpha = fminf(at, 0.99f);
    const float rom = rcp_ftz(1.f - alpha);
    const float Tk = T * rom;
    const float w = alpha * Tk;
    const float sk = qpl[j * kPlaneStride + t];
    const float da = Tk * sk - S * rom;
    S = fmaf(sk, w, S);
    T = Tk;
    wpl[j * kPlaneStride + t] = w;
    qpl[j * kPlaneStride + t] = (at <= kAlphaClamp ? da : 0.f) * e;
    --j;
  }
  // j odd (or -1): pairs (j - 1, j), two per batch
  auto pair_step = [&](int i, float2 al, float2 e, float2 at, float2 sk) {
    const float2 om = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-al.x, -al.y));
    const float2 rm = make_float2(rcp_ftz(om.x), rcp_ftz(om.y));
    const float Thi = T * rm.y;
    const float Tlo = Thi * rm.x;
    const float2 Tk = make_float2(Tlo, Thi);
    const float2 w = __fmul2_rn(al, Tk);
    const float S1 = fmaf(sk.y, w.y, S);
    const float2 srm = __fmul2_rn(make_float2(S1, S), rm);
    const float2 da = __ffma2_rn(Tk, sk, make_float2(-srm.x, -srm.y));
    S = fmaf(sk.x, w.x, S1);
    T = Tlo;
    const float2 q = __fmul2_rn(make_float2(at.x <= kAlphaClamp ? da.x : 0.f,
                                            at.y <= kAlphaClamp ? da.y : 0.f), e);
    wpl[(2 * i + 1) * kPlaneStride + t] = w.y;
    qpl[(2 * i + 1) * kPlaneStride + t] = q.y;
    wpl[2 * i * kPlaneStride + t] = w.x;
    qpl[2 * i * kPlaneStride + t] = q.x;
  };
  for (; j >= 3; j -= 4) {
    const int i0 = j >> 1, i1 = i0 - 1;
    float2 al0, e0, at0, al1, e1, at1;
    pair_alpha(sP[i0], fx, fy, al0, e0, at0);
    pair_alpha(sP[i1], fx, fy, al1, e1, at1);
    const float2 sk0 = make_float2(qpl[2 * i0 * kPlaneStride + t], qpl[(2 * i0 + 1) * kPlaneStride + t]);
    const float2 sk1 = make_float2(qpl[2 * i1 * kPlaneStride + t], qpl[(2 * i1 + 1) * kPlaneStride + t]);
    pair_step(i0, al0, e0, at0, sk0);
    pair_step(i1, al1, e1, at1, sk1);
  }
  if (j >= 1) {
    const int i0 = j >> 1;
    float2 al0, e0, at0;
    pair_alpha(sP[i0], fx, fy, al0, e0, at0);
    const float2 sk0 = make_float2(qpl[2 * i0 * kPlaneStride + t], qpl[(2 * i0 + 1) * kPlaneStride + t]);
    pair_step(i0, al0, e0, at0, sk0);
  }
}

template <int kBC, bool kDet>
__global__ void __launch_bounds__(256, (kBC == 16 ? (VSX_BWD_OCC4 ? 4 : 3) : 2))
    raster_bwd_tc_kernel(BwdArgs a, vsx_camera cam) {
  constexpr int kMT = kBC / 16;          // m-tiles per chunk
  constexpr int kSplit = 8 / (2 * kMT);  // k-range split across warps
  constexpr int kKS = 32 / kSplit;       // k-steps (8 pixels) per warp
  // phase-1 operands of splat pair (2i, 2i + 1), lane .x / .y of each float2:
  // (-mx, -my), (A2, B2), (C2, opacity) as in stage_splat; the epilogue's
  // unscaled conic (A, B, C) per splat
  __shared__ float4 sP[2][kBC / 2][3];
  __shared__ float4 sC[2][kBC];
  __shared__ float4 s_ph[2][kBC][4];  // P B fragments per (splat, lane&3): hi b0, hi b1, lo b0, lo b1
  __shared__ uint32_t s_rank[2][kBC];
#if VSX_BWD_OCC4
  __shared__ float2 s_bw[32][32];   // Gw B fragment values per (k-step, lane): b0, b1 (split per use)
  __shared__ __half2 s_bq[32][32];  // Mq B fragments per (k-step, lane): exact in half
#else
  __shared__ float4 s_bw[32][32];  // Gw B fragments per (k-step, lane): hi b0, hi b1, lo b0, lo b1
  __shared__ float2 s_bq[32][32];  // Mq B fragments per (k-step, lane)
#endif
  __shared__ float s_red[kSplit][kBC][kRedStride];
  __shared__ __align__(16) vsx_splat s_raw[2][kBC];
  __shared__ int s_max;
  extern __shared__ float s_plane[];  // w plane [kBC][kPlaneStride], then q plane
  const int txn = gridDim.x;
  // optional heaviest-first schedule: CTA i takes tile_order[i]
  const int lin = ((int)blockIdx.y + a.L.tile_row0) * txn + blockIdx.x;  // tile_row0: a band
  const int tile = a.L.tile_order ? (int)a.L.tile_order[lin] : lin;
  const int bx = tile % txn, by = tile / txn;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int g = lane >> 2, tq = lane & 3;
#if VSX_BWD_SORTPIX
  // Slot t (thread, plane column) takes the pixel of rank t in descending
  // live count (8-splat buckets): pixels that stop compositing at similar
  // depths share a warp, so phase 1 runs fewer idle lanes and whole warps go
  // quiet together. Phases 0 / 2 follow the slot order through the per-tile
  // fragments (cotangents and pixel moments are staged per slot).
#if VSX_BWD_OCC4
  // sort scratch in the q plane (first written by phase 0 of the first chunk)
  uint32_t *s_bin = reinterpret_cast<uint32_t *>(s_plane + kBC * kPlaneStride);
  uint8_t *s_perm = reinterpret_cast<uint8_t *>(s_plane + kBC * kPlaneStride + 260);
  __shared__ uint16_t s_lp[257];  // first slot of each key ([256] = 256): the live prefix
#else
  __shared__ uint32_t s_bin[257];  // after the scan: first slot of each key; [256] = 256
  __shared__ uint8_t s_perm[256];  // slot -> pixel (t = 16 y + x)
#endif
  __shared__ uint32_t s_wsum[8];
  {
    const int x0 = bx * kTile + (t & 15), y0 = by * kTile + (t >> 4);
    const int nc0 = (x0 < cam.width && y0 < cam.height) ? a.nc[(size_t)y0 * cam.width + x0] : 0;
    const uint32_t key = 255u - (uint32_t)min(nc0 >> 3, 255);
    s_bin[t] = 0u;
    __syncthreads();
    uint32_t r;
    if (kDet) {
      // deterministic mode: pixels keep their index order inside a bucket
      // (the slot order is the phase-2 summation order): warps in turn, lanes
      // ranked among equal keys
      r = 0;
      for (int w = 0; w < 8; ++w) {
        if (warp == w) {
          const unsigned peers = __match_any_sync(0xffffffffu, key);
          const uint32_t base = s_bin[key];
          __syncwarp();
          if ((peers >> lane) == 1u) s_bin[key] = base + __popc(peers);
          r = base + __popc(peers & ((1u << lane) - 1u));
        }
        __syncthreads();
      }
    } else {
      r = atomicAdd(&s_bin[key], 1u);  // order inside a bucket is free
      __syncthreads();
    }
    // exclusive scan of the 256 bucket counts
    uint32_t v = s_bin[t], inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += s_wsum[w];
    s_bin[t] = base + inc - v;
    if (t == 0) s_bin[256] = 256u;
#if VSX_BWD_OCC4
    s_lp[t] = (uint16_t)(base + inc - v);
    if (t == 0) s_lp[256] = 256;
#endif
    __syncthreads();
    s_perm[s_bin[key] + r] = (uint8_t)t;
    __syncthreads();
  }
  const int pix = s_perm[t];
#else
  const int pix = t;
#endif
  const int lx = pix & 15, ly = pix >> 4;
  const int px = bx * kTile + lx, py = by * kTile + ly;
  const bool inside = px < cam.width && py < cam.height;
  const double ox = (double)(bx * kTile), oy = (double)(by * kTile);
  const uint32_t begin = a.tile_off[tile];
  const float fx = (float)lx, fy = (float)ly;
  if (t == 0) s_max = 0;
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
  }
  // per-tile B fragments: Gw[p][f] staged through the (not yet used) w plane
  {
    float *gw = s_plane + t * 9;
    gw[0] = c.gC0; gw[1] = c.gC1; gw[2] = c.gC2; gw[3] = c.gR0;
    gw[4] = c.gR1; gw[5] = c.gR2; gw[6] = c.gD; gw[7] = c.gA;
  }
  __syncthreads();
  if (inside && nc > 0) atomicMax(&s_max, nc);
  // F A fragments (pixel rows of this warp x the 8 pixel cotangents), split
  uint32_t fhi[2][4], flo[2][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int pix = 32 * warp + 16 * m + g + 8 * (r & 1), f = tq + 4 * (r >> 1);
      const float v = s_plane[pix * 9 + f];
      fhi[m][r] = tf32_rn(v);
      flo[m][r] = tf32_rn(v - __uint_as_float(fhi[m][r]));
    }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = t + 256 * i, ks = idx >> 5, ln = idx & 31;
    const int f = ln >> 2, p0 = 8 * ks + (ln & 3), p1 = p0 + 4;
    const float v0 = f < 7 ? s_plane[p0 * 9 + f] : 0.f, v1 = f < 7 ? s_plane[p1 * 9 + f] : 0.f;
    const float h0 = __uint_as_float(tf32_rn(v0)), h1 = __uint_as_float(tf32_rn(v1));
#if VSX_BWD_OCC4
    (void)h0;
    (void)h1;
    s_bw[ks][ln] = make_float2(v0, v1);
    s_bq[ks][ln] = __floats2half2_rn(pixel_moment(s_perm[p0], f), pixel_moment(s_perm[p1], f));
#else
    s_bw[ks][ln] = make_float4(h0, h1, __uint_as_float(tf32_rn(v0 - h0)),
                               __uint_as_float(tf32_rn(v1 - h1)));
#endif
#if VSX_BWD_SORTPIX
#if !VSX_BWD_OCC4
    s_bq[ks][ln] = make_float2(pixel_moment(s_perm[p0], f), pixel_moment(s_perm[p1], f));
#endif
#else
    s_bq[ks][ln] = make_float2(pixel_moment(p0, f), pixel_moment(p1, f));
#endif
  }
  __syncthreads();
  const uint32_t stop = begin + (uint32_t)s_max;
  if (a.L.tile_live && t == 0) a.L.tile_live[tile] = (uint32_t)s_max;  // rows written below stop
  float S = 0.f;  // sum over later live splats of s_i * w_i
  float *wpl = s_plane, *qpl = s_plane + kBC * kPlaneStride;
  // phase-2 role of this warp
  const int mt = warp % kMT, plane = (warp / kMT) & 1, kr = warp / (2 * kMT);
  int buf = 0;
  // Record prefetch: the raw 64-byte records of chunk i+1 are copied
  // (cp.async) into s_raw while chunk i is processed, and the tile-list ranks
  // of chunk i+2 are loaded into a register, so neither dependent global load
  // sits in front of a barrier.
  auto chunk_lo = [&](uint32_t e) { return e > begin + kBC ? e - kBC : begin; };
  // slot owner: thread t owns slot t - 32 * VSX_BWD_STAGE_WARP, a warp whose
  // phase-2 role has two tensor-core products per k-step, not three, and
  // which sits outside the epilogue's warps 0-3 (warp 0: 1503 us, 7: 1475 us)
  const int sl = t - 32 * VSX_BWD_STAGE_WARP;
  uint32_t rr = 0;  // rank of slot t in the chunk whose copy is in flight
  uint32_t nr = 0;  // rank of slot t in the chunk after it
  {
    const uint32_t cs = chunk_lo(stop);
    if (stop > begin && (unsigned)sl < (stop - cs)) {
      rr = a.tile_list[cs + sl];
      copy_splat_async(&s_raw[0][sl], a.rec + rr);
    }
    cp_async_commit();
    const uint32_t cs2 = chunk_lo(cs);
    if (cs > begin && (unsigned)sl < (cs - cs2)) nr = a.tile_list[cs2 + sl];
  }
  // Stage chunk [cs_, cs_ + cnt_) into buffer sb from its in-flight copy and
  // start the copy of the chunk after it.
  auto stage = [&](int sb, uint32_t cs_, int cnt_) {
    cp_async_wait_all();
    if ((unsigned)sl < (unsigned)cnt_) {
      s_rank[sb][sl] = rr;
      const vsx_splat &sp = s_raw[sb][sl];
      {
        float4 p0, p1, p2, p3;
        stage_splat(sp, ox, oy, p0, p1, p2, p3);
        float *pp = reinterpret_cast<float *>(&sP[sb][sl >> 1][0]) + (sl & 1);
        pp[0] = -p0.x;
        pp[2] = -p0.y;
        pp[4] = p0.z;
        pp[6] = p0.w;
        pp[8] = p1.x;
        pp[10] = p1.y;
        sC[sb][sl] = make_float4(p1.w, p2.w, p3.w, 0.f);
      }
      const float pv[8] = {sp.color[0], sp.color[1], sp.color[2], sp.normal[0],
                           sp.normal[1], sp.normal[2], sp.plane_d, 1.f};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float h0 = __uint_as_float(tf32_rn(pv[k])), h1 = __uint_as_float(tf32_rn(pv[k + 4]));
        s_ph[sb][sl][k] = make_float4(h0, h1, __uint_as_float(tf32_rn(pv[k] - h0)),
                                     __uint_as_float(tf32_rn(pv[k + 4] - h1)));
      }
    }
    const uint32_t cs2 = chunk_lo(cs_);
    if (cs_ > begin && (unsigned)sl < (cs_ - cs2)) {
      rr = nr;
      copy_splat_async(&s_raw[sb ^ 1][sl], a.rec + nr);
    }
    cp_async_commit();
    const uint32_t cs3 = chunk_lo(cs2);
    if (cs2 > begin && (unsigned)sl < (cs2 - cs3)) nr = a.tile_list[cs3 + sl];
  };
#if VSX_BWD_MERGED
  // Two barriers per chunk: the next chunk is staged (double-buffered) right
  // after phase 2, so the epilogue's atomics overlap the next chunk's phase 0/1.
  if (stop > begin) stage(0, chunk_lo(stop), (int)(stop - chunk_lo(stop)));
  __syncthreads();
#endif
  for (uint32_t ce = stop; ce > begin; buf ^= 1) {
    const uint32_t cs = chunk_lo(ce);
    const int cnt = (int)(ce - cs);
#if !VSX_BWD_MERGED
    stage(buf, cs, cnt);
    __syncthreads();
#endif
    const int kbase = (int)(cs - begin);
    const int jlive = min(cnt, nc - kbase);
#if VSX_BWD_SORTPIX && VSX_BWD_PREFIX
    // Live prefix: slots are in descending (live count >> 3) order, so every
    // pixel with nc >> 3 < kbase >> 3 (nc <= kbase: dead in this chunk and all
    // earlier ones) sits after the first s_bin[256 - (kbase >> 3)] slots.
    // Phases 1 / 2 only touch the k-steps (8 slots) that cover the prefix.
#if VSX_BWD_OCC4
    const int nks = ((int)s_lp[256 - min(kbase >> 3, 255)] + 7) >> 3;
#else
    const int nks = ((int)s_bin[256 - min(kbase >> 3, 255)] + 7) >> 3;
#endif
#else
    const int nks = 32;
#endif
    // ---- phase 0: sk[j][p] = F[p] . P[j] for this warp's 32 pixels on the
    // tensor cores (3xTF32), written into the q plane that phase 1 overwrites
    // in place with q (same thread, same slot). Skipped by a warp none of
    // whose pixels is live in this chunk (with pixels sorted by live count,
    // whole warps go quiet together): phase 1 then only writes its zeros.
    if (!VSX_BWD_P0SKIP || __any_sync(0xffffffffu, jlive > 0))
#pragma unroll
    for (int nt = 0; nt < kBC / 8; ++nt) {
      const float4 b = s_ph[buf][8 * nt + g][tq];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        mma_m16n8k8_tf32(d, flo[m], __float_as_uint(b.x), __float_as_uint(b.y));
        mma_m16n8k8_tf32(d, fhi[m], __float_as_uint(b.z), __float_as_uint(b.w));
        mma_m16n8k8_tf32(d, fhi[m], __float_as_uint(b.x), __float_as_uint(b.y));
        float *o = qpl + (8 * nt + 2 * tq) * kPlaneStride + 32 * warp + 16 * m + g;
        o[0] = d[0];
        o[kPlaneStride] = d[1];
        o[8] = d[2];
        o[kPlaneStride + 8] = d[3];
      }
    }
    __syncwarp();
    // ---- phase 1: per-pixel back-to-front recursion
    if (t < 8 * nks)
      for (int j = cnt - 1; j >= max(jlive, 0); --j) {
        wpl[j * kPlaneStride + t] = 0.f;
        qpl[j * kPlaneStride + t] = 0.f;
      }
    bwd_phase1_pairs(sP[buf], wpl, qpl, t, jlive, fx, fy, T, S);
    __syncthreads();
    // ---- phase 2: tensor-core sums over this warp's k-range
    {
      const float *A = (plane ? qpl : wpl) + (16 * mt + g) * kPlaneStride + tq;
      // independent accumulators per split term and k-step parity: the HMMA
      // chains overlap instead of serialising on one accumulator
      float d[4] = {0.f, 0.f, 0.f, 0.f}, e1[4] = {0.f, 0.f, 0.f, 0.f},
            e2[4] = {0.f, 0.f, 0.f, 0.f};
      // A fragment of k-step ks split hi/lo (3xTF32)
      auto a_frag = [&](int ks, uint32_t (&hi)[4], uint32_t (&lo)[4]) {
        const float x0 = A[8 * ks], x1 = A[8 * kPlaneStride + 8 * ks], x2 = A[8 * ks + 4],
                    x3 = A[8 * kPlaneStride + 8 * ks + 4];
#if VSX_BWD_RN2
        hi[0] = tf32_rn(x0);
        hi[1] = tf32_rn(x1);
        hi[2] = tf32_rn(x2);
        hi[3] = tf32_rn(x3);
#else
        hi[0] = tf32_bits(x0);
        hi[1] = tf32_bits(x1);
        hi[2] = tf32_bits(x2);
        hi[3] = tf32_bits(x3);
#endif
        // lo is passed as its float32 bits: the tensor core reads the tf32
        // part (truncation of a value already <= 2^-11 |x|)
        lo[0] = __float_as_uint(x0 - __uint_as_float(hi[0]));
        lo[1] = __float_as_uint(x1 - __uint_as_float(hi[1]));
        lo[2] = __float_as_uint(x2 - __uint_as_float(hi[2]));
        lo[3] = __float_as_uint(x3 - __uint_as_float(hi[3]));
      };
      // warp-uniform plane branch outside the k loop: no predicated HMMAs
      // (skipping the k-ranges of quiet pixel warps here measured 1,469 ->
      // 1,583 us: the branch costs more than the zero products it saves)
      if (plane == 0) {
        int k0 = kr * kKS, kn = kKS;
        if (kMT == 1 && nks != 32) {
          const int q = (nks + 3) >> 2;
          k0 = kr * q;
          kn = max(0, min(q, nks - k0));
        }
#pragma unroll 4
        for (int kk = 0; kk < kn; ++kk) {
          const int ks = k0 + kk;
          uint32_t hi[4], lo[4];
          a_frag(ks, hi, lo);
#if VSX_BWD_OCC4
          const float2 rb = s_bw[ks][lane];
          const uint32_t bh0 = tf32_rn(rb.x), bh1 = tf32_rn(rb.y);
          const uint32_t bl0 = tf32_rn(rb.x - __uint_as_float(bh0));
          const uint32_t bl1 = tf32_rn(rb.y - __uint_as_float(bh1));
          mma_m16n8k8_tf32(e1, lo, bh0, bh1);
          mma_m16n8k8_tf32(e2, hi, bl0, bl1);
          mma_m16n8k8_tf32(d, hi, bh0, bh1);
#else
          const float4 b = s_bw[ks][lane];
          mma_m16n8k8_tf32(e1, lo, __float_as_uint(b.x), __float_as_uint(b.y));
          mma_m16n8k8_tf32(e2, hi, __float_as_uint(b.z), __float_as_uint(b.w));
          mma_m16n8k8_tf32(d, hi, __float_as_uint(b.x), __float_as_uint(b.y));
#endif
        }
      } else {
        // q-plane k-ranges: the staging warp (kr = 3 at kBC = 16) takes 5 of
        // the 32 k-steps, the other three 9 each (VSX_BWD_KR7 = 8 / 5 / 2:
        // 1479 / 1467 / 1479 us per view)
        int k0 = kr * kKS, kn = kKS;
        if (kMT == 1 && VSX_BWD_KR7 != kKS) {
          const int q = (nks * (32 - VSX_BWD_KR7) / 32 + 2) / 3;
          k0 = kr * q;
          kn = max(0, min(kr == 3 ? nks - 3 * q : q, nks - k0));
        } else if (kMT == 1 && nks != 32) {
          const int q = (nks + 3) >> 2;
          k0 = kr * q;
          kn = max(0, min(q, nks - k0));
        }
#pragma unroll 4
        for (int kk = 0; kk < kn; ++kk) {
          const int ks = k0 + kk;
          uint32_t hi[4], lo[4];
          a_frag(ks, hi, lo);
#if VSX_BWD_OCC4
          const float2 b = __half22float2(s_bq[ks][lane]);
#else
          const float2 b = s_bq[ks][lane];
#endif
          mma_m16n8k8_tf32(e1, lo, __float_as_uint(b.x), __float_as_uint(b.y));
          mma_m16n8k8_tf32(d, hi, __float_as_uint(b.x), __float_as_uint(b.y));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = (e1[k] + e2[k]) + d[k];
      float *red = &s_red[kr][16 * mt + g][8 * plane + 2 * tq];
      *reinterpret_cast<float2 *>(red) = make_float2(d[0], d[1]);
      *reinterpret_cast<float2 *>(red + 8 * kRedStride) = make_float2(d[2], d[3]);
    }
#if VSX_BWD_MERGED
    if (cs > begin) stage(buf ^ 1, chunk_lo(cs), (int)(cs - chunk_lo(cs)));
#endif
    __syncthreads();
    // ---- epilogue: 8 lanes per splat, lane part holds features 2part, 2part+1.
    // It runs on the LAST 8 kBC threads (warps 4-7 at kBC = 16): with pixels
    // sorted by live count those warps hold the shortest-lived pixels, so the
    // epilogue stays off the critical path (warp 0's phase 1 of the next
    // chunk) instead of delaying it.
    const int te = VSX_BWD_EPI_HI ? t - (256 - 8 * kBC) : t;
    if (te >= 0 && te < 8 * kBC) {
      const int j = te >> 3, part = te & 7;
      float2 v = *reinterpret_cast<const float2 *>(&s_red[0][j][2 * part]);
#pragma unroll
      for (int k = 1; k < kSplit; ++k) {
        const float2 u = *reinterpret_cast<const float2 *>(&s_red[k][j][2 * part]);
        v.x += u.x;
        v.y += u.y;
      }
      // moments: part 4 = (1, x), 5 = (y, xx), 6 = (xy, yy)
      const float m2 = __shfl_down_sync(0xffffffffu, v.x, 1), m3 = __shfl_down_sync(0xffffffffu, v.y, 1);
      const float m4 = __shfl_down_sync(0xffffffffu, v.x, 2), m5 = __shfl_down_sync(0xffffffffu, v.y, 2);
      if (j < cnt) {
        // deterministic mode (L.isect_grad): this (splat, tile)'s 13 sums go
        // to the intersection's row, reduced per splat in tile order later
        float *row = kDet ? a.L.isect_grad + (size_t)13 * (cs + j) : nullptr;
        float *gp = a.grad + (size_t)13 * s_rank[buf][j];
        if (part < 4) {
          if (row) {
            row[6 + 2 * part] = v.x;
            if (part < 3) row[7 + 2 * part] = v.y;
          } else {
            if (v.x != 0.f) atomicAdd(gp + 6 + 2 * part, v.x);
            if (part < 3 && v.y != 0.f) atomicAdd(gp + 7 + 2 * part, v.y);
          }
        } else if (part == 4) {
          const float *pp = reinterpret_cast<const float *>(&sP[buf][j >> 1][0]) + (j & 1);
          const float4 cc = sC[buf][j];
          const float op = pp[10], A = cc.x, B = cc.y, C = cc.z;
          const float mx = -pp[0] - 7.5f, my = -pp[2] - 7.5f;
          const float Q1 = v.x, X = v.y, Y = m2, XX = m3, XY = m4, YY = m5;
          const float sx = X - mx * Q1, sy = Y - my * Q1;
          const float sxx = XX - 2.f * mx * X + mx * mx * Q1;
          const float sxy = XY - mx * Y - my * X + mx * my * Q1;
          const float syy = YY - 2.f * my * Y + my * my * Q1;
          const float g[6] = {op * (A * sx + B * sy), op * (B * sx + C * sy), -0.5f * op * sxx,
                              -op * sxy, -0.5f * op * syy, Q1};
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            if (row) row[k] = g[k];
            else if (g[k] != 0.f) atomicAdd(gp + k, g[k]);
          }
        }
      }
    }
    ce = cs;
  }
}

// cudaFuncSetAttribute is per device: set it once per device the process
// launches on (a multi-GPU process, or threaded ranks, use several).
template <typename K>
static int smem_opt_in(K kernel, int bytes, std::atomic<uint64_t> &done) {
  int dev = 0;
  VSX_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load() & bit)) {
    VSX_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.fetch_or(bit);
  }
  return VSX_OK;
}

// The tile rows a launch composites: all, or the band [tile_row0, tile_row0 +
// tile_rows) of vsx_loss_desc (a renderer rank's share of a view).
static int band_rows(const vsx_loss_desc &L, const vsx_camera &cam, int &rows) {
  const int tyn = (cam.height + kTile - 1) / kTile;
  rows = L.tile_rows > 0 ? L.tile_rows : tyn;
  VSX_REQUIRE(L.tile_row0 >= 0 && L.tile_row0 + rows <= tyn && (L.tile_rows == 0 || L.tile_rows > 0),
              "raster: tile band [%d, %d) outside the %d tile rows", L.tile_row0,
              L.tile_row0 + rows, tyn);
  VSX_REQUIRE(L.tile_rows == 0 || L.tile_order == nullptr, "raster: tile_order with a band");
  return VSX_OK;
}

static int launch_bwd(const BwdArgs &a, const vsx_camera &cam, cudaStream_t st) {
  constexpr int kBC = 16;
  int rows = 0;
  if (int rc = band_rows(a.L, cam, rows)) return rc;
  dim3 grid((cam.width + kTile - 1) / kTile, rows);
  const int smem = (int)(sizeof(float) * 2 * kBC * kPlaneStride);
  static std::atomic<uint64_t> done{0};
  if (a.L.isect_grad) {  // deterministic mode (separate instantiation)
    static std::atomic<uint64_t> done_det{0};
    if (int rc = smem_opt_in(raster_bwd_tc_kernel<kBC, true>, smem, done_det)) return rc;
    raster_bwd_tc_kernel<kBC, true><<<grid, 256, smem, st>>>(a, cam);
  } else {
    if (int rc = smem_opt_in(raster_bwd_tc_kernel<kBC, false>, smem, done)) return rc;
    raster_bwd_tc_kernel<kBC, false><<<grid, 256, smem, st>>>(a, cam);
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
  int rows = 0;
  if (int rc = band_rows(L, cam, rows)) return rc;
  dim3 grid((cam.width + kTile - 1) / kTile, rows);
  // two horizontally adjacent pixels per thread, alpha batches of 4 splats
  // (the measured optimum: DESIGN.md §3, scripts/ab_fwd.py)
  if (L.sum_partials)  // deterministic mode (a separate instantiation)
    raster_fwd_pk_kernel<4, true><<<grid, 128, 0, st>>>(rec, tile_offsets, tile_list, cam, rgb,
                                                        alpha, depth, normal, raw_normal, valid,
                                                        t_final, n_contrib, L);
  else
    raster_fwd_pk_kernel<4, false><<<grid, 128, 0, st>>>(rec, tile_offsets, tile_list, cam, rgb,
                                                         alpha, depth, normal, raw_normal, valid,
                                                         t_final, n_contrib, L);
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

// ------------------------------------------------------ deterministic mode
//
// With vsx_loss_desc.isect_grad / tile_live / sum_partials set, the compositor
// kernels write their per-(splat, tile) gradient sums and per-warp loss sums
// to fixed slots instead of adding them with float atomics; these kernels
// reduce the slots in a fixed order, so a step is bitwise reproducible (the
// reference's sums are order-fixed by construction, trainer.py:9-13).

namespace vsx {

// One thread per sorted splat: its tiles in row-major order over the
// rectangle (renderer.py:216-221), its position in each tile's ascending list
// by binary search, the row counted when the backward visited it.
__global__ void raster_grad_reduce_kernel(const vsx_splat *__restrict__ rec,
                                          const double *__restrict__ radius, int32_t n, int txn,
                                          int tyn, const uint32_t *__restrict__ toff,
                                          const uint32_t *__restrict__ tl,
                                          const uint32_t *__restrict__ tile_live,
                                          const float *__restrict__ isect,
                                          float *__restrict__ grad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int x0, x1, y0, y1;
  if (!tile_rect(rec[r].mean2d[0], rec[r].mean2d[1], radius[r], txn, tyn, x0, x1, y0, y1)) return;
  float acc[13];
#pragma unroll
  for (int f = 0; f < 13; ++f) acc[f] = 0.f;
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x) {
      const int t = y * txn + x;
      const uint32_t b = toff[t];
      uint32_t lo = b, hi = toff[t + 1];
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tl[mid] < (uint32_t)r) lo = mid + 1;
        else hi = mid;
      }
      if (lo - b < tile_live[t]) {
        const float *row = isect + (size_t)13 * lo;
#pragma unroll
        for (int f = 0; f < 13; ++f) acc[f] += row[f];
      }
    }
  float *g = grad + (size_t)13 * r;
#pragma unroll
  for (int f = 0; f < 13; ++f) g[f] += acc[f];
}

// One CTA: thread t sums slots t, t + 1024, ... in order, then a fixed tree.
__global__ void __launch_bounds__(1024) reduce_partials_kernel(const double *__restrict__ part,
                                                               int64_t slots,
                                                               double *__restrict__ sums) {
  __shared__ double s[3][1024];
  const int t = threadIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t i = t; i < slots; i += 1024) {
    a0 += part[3 * i + 0];
    a1 += part[3 * i + 1];
    a2 += part[3 * i + 2];
  }
  s[0][t] = a0;
  s[1][t] = a1;
  s[2][t] = a2;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (t < w) {
      s[0][t] += s[0][t + w];
      s[1][t] += s[1][t + w];
      s[2][t] += s[2][t + w];
    }
    __syncthreads();
  }
  if (t < 3) sums[t] += s[t][0];
}

}  // namespace vsx

extern "C" int vsx_reduce_partials(const double *partials, int64_t slots, double *sums,
                                   vsx_stream s) {
  VSX_REQUIRE(slots >= 0 && sums && (partials || slots == 0), "reduce_partials: bad args");
  reduce_partials_kernel<<<1, 1024, 0, as_stream(s)>>>(partials, slots, sums);
  VSX_LAUNCH_CHECK("reduce_partials");
  return VSX_OK;
}

extern "C" int vsx_raster_grad_reduce(const vsx_splat *rec, const double *radius, int32_t n,
                                      int32_t width, int32_t height, const uint32_t *tile_offsets,
                                      const uint32_t *tile_list, const uint32_t *tile_live,
                                      const float *isect_grad, float *grad_splat, vsx_stream s) {
  VSX_REQUIRE(n >= 0 && width > 0 && height > 0, "raster_grad_reduce: bad args");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(rec && radius && tile_offsets && tile_list && tile_live && isect_grad && grad_splat,
              "raster_grad_reduce: null buffer");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  raster_grad_reduce_kernel<<<grid_for(n, 128), 128, 0, as_stream(s)>>>(
      rec, radius, n, txn, tyn, tile_offsets, tile_list, tile_live, isect_grad, grad_splat);
  VSX_LAUNCH_CHECK("raster_grad_reduce");
  return VSX_OK;
}
