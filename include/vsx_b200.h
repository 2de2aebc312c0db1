/*
 * vsx_b200.h — C ABI of the B200-native CityGS-X training hot path.
 *
 * Every entry point takes caller-owned DEVICE buffers as raw pointers plus
 * explicit element counts, is asynchronous on the given CUDA stream, and
 * returns a status code (VSX_OK or a negative VSX_ERR_*). There are no torch
 * types in any signature. Host callers (the Python shim in
 * paper_2503_23044_b200/, or a ctypes/cgo binding) own allocation.
 *
 * Reference interface each group replaces (paths relative to
 * /root/reference/pkg/src/voxsplat):
 *   vsx_cull / vsx_select          scene.py:239-259 active_mask (+ lod_for_distance :232-236)
 *   vsx_decode_fwd(_tc)            decoder.py:142-180 decode_inputs/_head_forward/decode_arrays,
 *                                  decoder.py:210-250 decode_active (canonical order)
 *   vsx_project_fwd                renderer.py:144-204 project_splats (EWA + (z,gid) order)
 *   vsx_sort_splats_z              renderer.py:197 np.lexsort((gid, z)) (float32 proxy radix
 *                                  sort + exact run fix-up); vsx_sort_pairs_u64/_u32 generic
 *   vsx_bin_plan / vsx_bin_build   renderer.py:207-226 bin_splats (row-column counting sorts;
 *                                  vsx_bin_count / vsx_bin_emit(_hist) / vsx_tile_ranges +
 *                                  vsx_sort_pairs_u32 for images over 4096 px a side)
 *   vsx_raster_fwd(_loss)          renderer.py:242-301 _blend_padded + _finalize, :390-449 rasterize_view
 *   vsx_raster_bwd(_loss)          renderer.py:347-367 rasterize_backward (autograd of the blend)
 *   vsx_reduce_partials / vsx_raster_grad_reduce
 *                                  deterministic mode: fixed-order loss sums and per-splat
 *                                  gradient sums (the reference's sums are order-fixed,
 *                                  trainer.py:9-13)
 *   vsx_project_bwd(_batch)        autograd of project_splats (trainer.py:330)
 *   vsx_decode_bwd                 decoder.py:267-292 decoder_backward (autograd of decode)
 *   vsx_l1_loss / vsx_depth_loss   losses.py:43-53 bl_rgb_loss, losses.py:65-84 e_depth_loss
 *   vsx_adam / vsx_adam_guarded    trainer.py:220-247 TrainState._adam + apply_*_grads
 *                                  (guarded: skipped on the device after a non-finite step,
 *                                  trainer.py:317-321)
 *   vsx_growth_accumulate          trainer.py:342-349 (growth pressure accumulators)
 *   vsx_tile_max_len               trainer.py:373 StepReport.max_tile_splats
 *   vsx_sort_z_gid                 C1 merge of received splat rows in (z, gid) order
 *   vsx_tsdf_integrate             fusion.py:102-133 TSDF integration
 *   (C1 payload exchange)          renderer.py:452-477 transfer_gaussians: the 64-byte splat
 *                                  records are the payload; the all-to-all is NCCL (dist.py)
 *   vsx_pack_splat_rows / vsx_splat_rows_keys / vsx_gather_splat_rows
 *                                  C1 payload rows (96 B: record | z | radius | gid) packed
 *                                  for the all-to-all, and read back in (z, gid) order
 *   vsx_prior_sample / vsx_apply_scale_shift / vsx_reprojection_error / vsx_enhance_finalize
 *                                  depth_prior.py:85-214 (fit_scale_shift, apply_scale_shift,
 *                                  reprojection_error, enhance)
 *   vsx_ncc_patches / vsx_ncc_scatter
 *                                  losses.py:98-287 compute_homography .. bl_geo_loss (Eq. 10)
 */
#ifndef VSX_B200_H
#define VSX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSX_OK 0
#define VSX_ERR_INVALID -1   /* -> errors.InvalidInput */
#define VSX_ERR_NUMERICAL -2 /* -> errors.NumericalError */
#define VSX_ERR_CONTRACT -3  /* -> errors.ContractViolation */
#define VSX_ERR_CUDA -4      /* CUDA launch/runtime failure */
#define VSX_ERR_CAPACITY -5  /* workspace too small -> errors.ResourceError */

/* Device-status bits written by kernels into a caller-owned int32 word. */
#define VSX_STATUS_NONPD 1     /* det(cov2d) <= 0 (renderer.py:182-183) */
#define VSX_STATUS_NONFINITE 2 /* non-finite decoder output (decoder.py:246-249) */

typedef void *vsx_stream; /* cudaStream_t */

/* Pinhole camera: x_cam = R x_world + t (geometry.py:68-112). center = -R^T t
 * is computed on the host so it is bit-identical to CameraView.center. */
typedef struct vsx_camera {
  double r[9];
  double t[3];
  double center[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} vsx_camera;

/* Splat record, 64 bytes, one per projected gaussian (sorted order). The
 * mean is kept in float64 so per-tile local pixel offsets are exact even at
 * 4K; everything the compositor multiplies is float32. */
typedef struct vsx_splat {
  double mean2d[2];
  float conic[3]; /* (A, B, C) = inverse 2D covariance (c, -b, a)/det */
  float opacity;
  float color[3];
  float normal[3]; /* camera-frame normal, flipped to face the camera */
  float plane_d;   /* n_cam . mu_cam */
  uint32_t src;    /* index of the gaussian in the decode batch */
} vsx_splat;

/* Decoder weights, all float32 device pointers, reference layouts
 * (decoder.py:39-78): w1 (36,64) row-major, b1 (64), w2 (64,out), b2 (out),
 * out = n, 3n, 7n for opacity, color, cov. */
typedef struct vsx_decoder {
  const float *w1[3];
  const float *b1[3];
  const float *w2[3];
  const float *b2[3];
  int32_t n;
} vsx_decoder;

typedef struct vsx_decoder_grads {
  float *w1[3];
  float *b1[3];
  float *w2[3];
  float *b2[3];
} vsx_decoder_grads;

const char *vsx_last_error(void);
int vsx_version(void);
/* Number of kernels this library has launched so far (monotonic). */
uint64_t vsx_launch_count(void);

/* ---- generic device primitives ---------------------------------------- */
/* Workspace bytes needed by vsx_sort_pairs_* / vsx_select / vsx_scan for n items. */
size_t vsx_sort_ws_bytes(int64_t n);
size_t vsx_scan_ws_bytes(int64_t n);
/* Row scatter of float32 rows: dst[idx[i] * width + k] = src[i * width + k]
 * (idx a permutation of [0, n); the sharded step returns each merged view's
 * splat gradients to the received row order with it). */
int vsx_scatter_rows_f32(const float *src, const uint32_t *idx, int32_t n, int32_t width,
                         float *dst, vsx_stream s);
/* Exclusive scan of uint32 counts: out[i] = sum(in[0:i]); out[n] = total. */
int vsx_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *ws, size_t ws_bytes,
                 vsx_stream s);
/* Stable LSD radix sort of (key, value) pairs on key bits [begin_bit, end_bit).
 * flags & VSX_SORT_SKIP_CONSTANT: first reduce OR/AND of the keys and skip
 * 8-bit digits that are identical for every key (costs one host sync). */
#define VSX_SORT_SKIP_CONSTANT 1
/* flags & VSX_SORT_HIST_IN_WS: the per-pass digit histograms (pass p at
 * u32 [256 p, 256 p + 256)) are already in the workspace at
 * vsx_sort_hist_offset(n) (a producer such as vsx_bin_emit_hist built them);
 * the sort skips its own histogram read. Passes are every 8 bits of
 * [begin_bit, end_bit). */
#define VSX_SORT_HIST_IN_WS 2
size_t vsx_sort_hist_offset(int64_t n);
int vsx_sort_pairs_u64(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                       uint32_t *vals_out, int64_t n, int32_t begin_bit, int32_t end_bit,
                       int32_t flags, void *ws, size_t ws_bytes, vsx_stream s);
int vsx_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                       uint32_t *vals_out, int64_t n, int32_t begin_bit, int32_t end_bit,
                       int32_t flags, void *ws, size_t ws_bytes, vsx_stream s);
/* Stable order of projected splats by their float64 z keys (vsx_project_fwd
 * zkey; UINT64_MAX = culled, sorted last) without sorting 64-bit keys: a
 * 4-pass sort on a round-toward-zero float32 proxy, then runs of equal proxy
 * re-sorted by the exact key (ties by index). No host synchronisation. */
size_t vsx_sort_splats_ws_bytes(int64_t n);
int vsx_sort_splats_z(const uint64_t *zkey, int64_t n, uint32_t *order, void *ws,
                      size_t ws_bytes, vsx_stream s);
/* order = np.lexsort((gid, z)) for positive float64 z (renderer.py:197), used
 * by a renderer rank to merge splat segments received from several owners:
 * stable radix sort on the z bits, then runs of equal z reordered by gid. */
size_t vsx_sort_z_gid_ws_bytes(int64_t n);
int vsx_sort_z_gid(const double *z, const int64_t *gid, uint32_t *order, int64_t n, void *ws,
                   size_t ws_bytes, vsx_stream s);
/* Ordered stream compaction: out_idx = flatnonzero(flags), *out_count on device. */
int vsx_select(const uint8_t *flags, int64_t n, int32_t *out_idx, uint32_t *out_count,
               void *ws, size_t ws_bytes, vsx_stream s);

/* ---- K1: frustum + LoD culling (scene.py:232-259) --------------------- */
int vsx_cull(const double *centers, const int32_t *level, int64_t n_anchors, int32_t lod_count,
             double lod_ref, int32_t lod_bias, vsx_camera cam, uint8_t *mask, vsx_stream s);

/* ---- K2: anchor -> gaussian decode (decoder.py:142-180) --------------- */
/* active: ascending flat anchor ids (n_active). Per-anchor params are flat
 * level-major: emb (A,32) f32, log_scale (A,3) f32 (l_v = exp in float64),
 * offsets (A,n,3) f32, centers (A,3) f64. Outputs are gaussian-major
 * (n_active*n rows). cache_h [192][ld] and cache_o [11n][ld] (feature-major,
 * ld = n_active rounded up to a multiple of 4) keep the hidden activations
 * and raw head outputs for vsx_decode_bwd (may be NULL for inference). */
int vsx_decode_fwd(vsx_decoder W, const int32_t *active, int32_t n_active, const double *centers,
                   const float *emb, const float *log_scale, const float *offsets,
                   vsx_camera cam, double lod_ref, double max_scale, double *means,
                   float *opacity, float *color, float *scale, float *quat, float *normal,
                   float *cache_h, float *cache_o, int32_t *status, vsx_stream s);

/* Tensor-core (tcgen05, 3xTF32) variant of vsx_decode_fwd. `img` is the
 * decoder weight image built by vsx_decoder_image (vsx_decoder_image_floats(n)
 * floats) after every weight update. Supported for n <= 13. cache_o is
 * required here (the per-gaussian activations read the raw head outputs back
 * from it); cache_h may be NULL. */
size_t vsx_decoder_image_floats(int32_t n);
int vsx_decoder_image(vsx_decoder W, float *img, vsx_stream s);
int vsx_decode_fwd_tc(vsx_decoder W, const float *img, const int32_t *active, int32_t n_active,
                      const double *centers, const float *emb, const float *log_scale,
                      const float *offsets, vsx_camera cam, double lod_ref, double max_scale,
                      double *means, float *opacity, float *color, float *scale, float *quat,
                      float *normal, float *cache_h, float *cache_o, int32_t *status,
                      vsx_stream s);

/* ---- K3: projection (renderer.py:144-204) ----------------------------- */
/* Writes one unsorted record per gaussian plus a sort key (float64 z bits,
 * or UINT64_MAX when z <= 0.01) and the 3-sigma radius; *n_kept counts
 * z > 0.01. Sorting (key, index) stably gives the reference (z, gid) order
 * when the batch is in ascending-gid order. */
int vsx_project_fwd(const double *means, const float *opacity, const float *color,
                    const float *scale, const float *quat, const float *normal, int32_t n,
                    vsx_camera cam, vsx_splat *rec, uint64_t *zkey, double *radius,
                    uint32_t *n_kept, int32_t *status, vsx_stream s);
/* Gather records/radius into sorted order: dst[i] = src[order[i]], i < n. */
int vsx_gather_splats(const vsx_splat *rec, const double *radius, const uint32_t *order,
                      int32_t n, vsx_splat *rec_sorted, double *radius_sorted, vsx_stream s);
/* C1 payload rows (the sharded step, dist.py): 96 bytes per splat = the
 * 64-byte record, float64 z, float64 radius, int64 gid, 8 bytes of padding
 * (16-byte aligned rows for the all-to-all buffer). Pack n rows into out. */
#define VSX_SPLAT_ROW_BYTES 96
/* Owner-side payload keys: gid[i] = active[src[i] / n] * n + src[i] % n and
 * z[i] = key[src[i]] for the n_kept kept splats (src: decode batch indices). */
int vsx_payload_keys(const int32_t *active, const uint32_t *src, const uint64_t *key,
                     int32_t n_kept, int32_t n, int64_t *gid, uint64_t *z, vsx_stream s);
int vsx_pack_splat_rows(const vsx_splat *rec, const double *z, const double *radius,
                        const int64_t *gid, int32_t n, uint8_t *out, vsx_stream s);
/* Sort keys of n received rows: row i is rows[rowmap[i]] (rowmap NULL: rows[i]). */
int vsx_splat_rows_keys(const uint8_t *rows, const int32_t *rowmap, int32_t n, double *z,
                        int64_t *gid, vsx_stream s);
/* Records / radii in merge order: dst[i] = row(order[i]), row(j) = rows[rowmap[j]]
 * (rowmap NULL: rows[j]). */
int vsx_gather_splat_rows(const uint8_t *rows, const int32_t *rowmap, const uint32_t *order,
                          int32_t n, vsx_splat *rec_sorted, double *radius_sorted,
                          vsx_stream s);

/* ---- K4: tile binning (renderer.py:207-226) --------------------------- */
/* Phase 1: per-splat tile counts (+ per-tile histogram when tile_counts is
 * not NULL; the training path derives tile ranges from the sorted keys
 * instead and passes NULL). */
int vsx_bin_count(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                  int32_t height, uint32_t *splat_tiles, uint32_t *tile_counts, vsx_stream s);
/* Phase 2: emit (tile, rank) pairs at exclusive-scan offsets of splat_tiles
 * (splat_offsets has n+1 entries, the total last). */
int vsx_bin_emit(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                 int32_t height, const uint32_t *splat_offsets, uint32_t *isect_tile,
                 uint32_t *isect_rank, vsx_stream s);
/* Phase 2 with the tile-key digit histograms of both radix passes (bits
 * [0, 8) and [8, 16)) accumulated on the fly into hist (2 x 256 u32, zeroed
 * here): the following vsx_sort_pairs_u32(..., VSX_SORT_HIST_IN_WS) skips
 * its histogram read of the 8-byte pairs. */
int vsx_bin_emit_hist(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                      int32_t height, const uint32_t *splat_offsets, uint32_t *isect_tile,
                      uint32_t *isect_rank, uint32_t *hist, vsx_stream s);
/* Phase 3: CSR tile offsets (num_tiles+1) from the tile-sorted keys
 * (lower_bound per tile; no atomics). */
int vsx_tile_ranges(const uint32_t *sorted_tiles, int64_t n, int32_t num_tiles,
                    uint32_t *tile_offsets, vsx_stream s);
/* *max_len = max(*max_len, longest tile list) (device u32, accumulates across
 * calls: StepReport.max_tile_splats, trainer.py:373). */
int vsx_tile_max_len(const uint32_t *tile_offsets, int32_t num_tiles, uint32_t *max_len,
                     vsx_stream s);
/* Tile-major alternative to phases 2-3 (the training path): with
 * tile_offsets = exclusive scan of vsx_bin_count's tile_counts (splat_tiles
 * may be NULL), every covered tile's next slot (atomic cursor, num_tiles
 * u32 scratch, zeroed here) gets the splat rank; vsx_tile_segsort then sorts
 * each tile's ranks ascending (one CTA per tile, shared-memory bitonic sort;
 * VSX_ERR_CAPACITY when max_len > 4096 — the caller falls back to phases
 * 2-3). The result equals the sorted (tile, rank) lists bit for bit. */
int vsx_bin_emit_tiles(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                       int32_t height, const uint32_t *tile_offsets, uint32_t *cursor,
                       uint32_t *tile_list, vsx_stream s);
int vsx_tile_segsort(const uint32_t *tile_offsets, int32_t num_tiles, uint32_t *tile_list,
                     int32_t max_len, vsx_stream s);
/* Row-column binning (the training path; width and height <= 4096 pixels,
 * i.e. <= 256 tile rows and columns): two stable counting sorts with the
 * tile rectangle expanded on the fly, replacing phases 1-3. vsx_bin_plan
 * computes each splat's rectangle (renderer.py:216-221) into plan_ws and
 * totals[0] = row entries (sum of rectangle heights), totals[1] = pairs
 * (copied to `totals`, device or pinned host, when not NULL). After the
 * caller reads them, vsx_bin_build (once per plan) writes tile_offsets (T+1)
 * and tile_list (pairs) — bit for bit the sorted (tile, rank) lists of
 * phases 1-3 — using a build workspace of vsx_bin_build_ws_bytes(row_entries). */
size_t vsx_bin_plan_ws_bytes(int32_t n, int32_t width, int32_t height);
size_t vsx_bin_build_ws_bytes(int32_t width, int32_t height, int64_t row_entries);
int vsx_bin_plan(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                 int32_t height, void *plan_ws, size_t plan_bytes, uint64_t *totals, vsx_stream s);
int vsx_bin_build(int32_t n, int32_t width, int32_t height, int64_t row_entries, int64_t pairs,
                  void *plan_ws, size_t plan_bytes, void *build_ws, size_t build_bytes,
                  uint32_t *tile_offsets, uint32_t *tile_list, vsx_stream s);

/* ---- K5: compositing forward (renderer.py:242-301, 390-449) ----------- */
/* tile_offsets (T+1) CSR over tile_list (sorted ranks). Outputs are HWC
 * images (rgb/normal/raw_normal 3 channels) plus per-pixel backward state
 * (t_final, n_contrib). Any output pointer except t_final/n_contrib may be
 * NULL to skip it. */
int vsx_raster_fwd(const vsx_splat *rec, const uint32_t *tile_offsets, const uint32_t *tile_list,
                   vsx_camera cam, float *rgb, float *alpha, float *depth, float *normal,
                   float *raw_normal, uint8_t *valid, float *t_final, int32_t *n_contrib,
                   vsx_stream s);

/* Fused training objective of one view (K9 folded into K5/K6):
 *   L = rgb_scale * sum|rgb - gt|                              (losses.py:43-53)
 *     + depth_weight  * sum_mask |depth - prior| / count_depth  (losses.py:65-84)
 *     + normal_weight * sum_mask |normal - prior_n| / count_normal
 * with mask = render-valid & prior-valid. The forward accumulates the raw
 * sums (sums[0..2], float64) and counts (counts[0..1]); the backward forms
 * the pixel cotangents on the fly from the same inputs. Unused priors NULL. */
typedef struct vsx_loss_desc {
  const float *gt_rgb;
  const float *prior_depth;
  const uint8_t *prior_depth_valid;
  const float *prior_normal;
  const uint8_t *prior_normal_valid;
  float rgb_scale;
  float depth_weight;
  float normal_weight;
  double *sums;
  uint32_t *counts;
  /* optional additional cotangents of the rendered rgb (H,W,3), normal
   * (H,W,3) and depth (H,W) images (e.g. the NCC term, vsx_ncc_scatter);
   * NULL when absent. Used by vsx_raster_bwd_loss only. */
  const float *extra_rgb;
  const float *extra_normal;
  const float *extra_depth;
  /* optional: += sum over the view's pixels of n_contrib (live (pixel, splat)
   * pairs), reduced in the forward epilogue; NULL when not wanted. */
  unsigned long long *live_pairs;
  /* optional schedule for vsx_raster_bwd_loss: CTA i composites tile
   * tile_order[i] (a permutation of the tiles, e.g. longest list first so the
   * heavy tiles do not form the kernel's tail); NULL = row-major. */
  const uint32_t *tile_order;
  /* optional deterministic mode (bitwise run-to-run reproducible sums):
   * sum_partials (3 doubles per (tile, forward warp): T * 4 * 3) takes the
   * forward's loss sums instead of float atomics, reduced in order by
   * vsx_reduce_partials; isect_grad (13 floats per intersection) and
   * tile_live (one u32 per tile) take the backward's per-(splat, tile)
   * gradient sums instead of float atomics into grad_splat, reduced per
   * splat in row-major tile order by vsx_raster_grad_reduce. NULL = atomics. */
  double *sum_partials;
  float *isect_grad;
  uint32_t *tile_live;
  /* optional band (the sharded step's split of a view over ranks when the
   * batch has fewer views than ranks): composite only tile rows
   * [tile_row0, tile_row0 + tile_rows); tile_rows = 0 = all rows. Outputs
   * outside the band are not written; the loss counts and sums cover the
   * band only. Not combined with tile_order. */
  int32_t tile_row0;
  int32_t tile_rows;
} vsx_loss_desc;

int vsx_raster_fwd_loss(const vsx_splat *rec, const uint32_t *tile_offsets,
                        const uint32_t *tile_list, vsx_camera cam, float *rgb, float *alpha,
                        float *depth, float *normal, float *raw_normal, uint8_t *valid,
                        float *t_final, int32_t *n_contrib, vsx_loss_desc loss, vsx_stream s);
int vsx_raster_bwd_loss(const vsx_splat *rec, const uint32_t *tile_offsets,
                        const uint32_t *tile_list, vsx_camera cam, const float *rgb,
                        const float *alpha, const float *depth, const float *normal,
                        const float *raw_normal, const float *t_final, const int32_t *n_contrib,
                        vsx_loss_desc loss, float *grad_splat, vsx_stream s);

/* Deterministic-mode reductions. vsx_reduce_partials: sums[k] += the
 * fixed-order sum over `slots` of partials[3 * slot + k], k < 3.
 * vsx_raster_grad_reduce: per sorted splat r (n of them, radius the binning
 * radius), grad_splat[13 r + f] += the sum over the tiles of its rectangle in
 * row-major order of isect_grad[13 * pos + f], pos = r's position in the
 * tile's list, for the positions the backward visited (< tile_live). */
int vsx_reduce_partials(const double *partials, int64_t slots, double *sums, vsx_stream s);
int vsx_raster_grad_reduce(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                           int32_t height, const uint32_t *tile_offsets,
                           const uint32_t *tile_list, const uint32_t *tile_live,
                           const float *isect_grad, float *grad_splat, vsx_stream s);

/* ---- K6: compositing backward ------------------------------------------ */
/* Pixel cotangents (any may be NULL = zero) -> per-splat gradients
 * (sorted order, float32 x 13: mean2d 2, conic 3, opacity, color 3,
 * normal 3, plane_d), accumulated (+=) into grad_splat. */
int vsx_raster_bwd(const vsx_splat *rec, const uint32_t *tile_offsets, const uint32_t *tile_list,
                   vsx_camera cam, const float *rgb, const float *alpha, const float *depth,
                   const float *raw_normal, const float *t_final, const int32_t *n_contrib,
                   const float *g_rgb, const float *g_alpha, const float *g_depth,
                   const float *g_normal, const float *g_raw_normal, float *grad_splat,
                   vsx_stream s);

/* ---- K7: projection backward ------------------------------------------- */
/* grad_splat (sorted, 13 floats) -> per-gaussian grads (+=, batch order):
 * means 3, opacity, color 3, scale 3, quat 4 (w.r.t. the normalised quat),
 * normal 3. */
int vsx_project_bwd(const double *means, const float *scale, const float *quat,
                    const float *normal, const vsx_splat *rec_sorted, const float *grad_splat,
                    int32_t n_sorted, vsx_camera cam, float *g_means, float *g_opacity,
                    float *g_color, float *g_scale, float *g_quat, float *g_normal,
                    vsx_stream s);
/* Same gradients in batch order: thread per decoded gaussian with its sorted
 * rank (inv_ws: n_batch int32 scratch); writes every output row, zeros for
 * gaussians culled by the projection (no zero-initialised outputs needed).
 * src_sorted (optional) = the records' src field as a dense int32 array. */
int vsx_project_bwd_batch(const double *means, const float *scale, const float *quat,
                          const float *normal, const vsx_splat *rec_sorted,
                          const float *grad_splat, int32_t n_sorted, int32_t n_batch,
                          vsx_camera cam, float *g_means, float *g_opacity, float *g_color,
                          float *g_scale, float *g_quat, float *g_normal,
                          const int32_t *src_sorted, int32_t *inv_ws, vsx_stream s);

/* ---- K8: decode backward ------------------------------------------------ */
/* Per-gaussian grads -> decoder weight grads (+=) and per-anchor grads (+=)
 * for emb (A,32), log_scale (A,3), offsets (A,n,3). scale/quat are the
 * decoded (clamped) scales and normalised quaternions of the forward. */
size_t vsx_decode_bwd_ws_bytes(int32_t n, int32_t n_active);
int vsx_decode_bwd(vsx_decoder W, vsx_decoder_grads dW, const int32_t *active, int32_t n_active,
                   const double *centers, const float *emb, const float *log_scale,
                   const float *offsets, vsx_camera cam, double lod_ref, double max_scale,
                   const float *cache_h, const float *cache_o, const float *scale,
                   const float *quat, const float *g_means, const float *g_opacity,
                   const float *g_color, const float *g_scale, const float *g_quat,
                   const float *g_normal, float *g_emb, float *g_log_scale, float *g_offsets,
                   void *ws, size_t ws_bytes, vsx_stream s);

/* Growth pressure (trainer.py:342-349, f3): grow_sum[active[r]] += sum over
 * the n gaussians of anchor r of |g_means| (float64), grow_cnt[...] += n.
 * g_means is the (n_active*n, 3) mean gradient of the decode batch. */
int vsx_growth_accumulate(const float *g_means, const int32_t *active, int32_t n_active,
                          int32_t n, double *grow_sum, double *grow_cnt, vsx_stream s);

/* ---- K9: losses --------------------------------------------------------- */
/* L1: loss_accum[0] += sum|r - g| (float64); grad = sign(r - g) * scale. */
int vsx_l1_loss(const float *rendered, const float *target, int64_t n, float scale,
                double *loss_accum, float *grad, vsx_stream s);
/* Masked depth L1 (losses.py:65-84): mask = prior_valid & valid;
 * sums[0] += sum |d - p| * mask, counts[0] += sum mask; with grad != NULL
 * writes grad = sign(d - p) * mask * (*scale) where scale is a DEVICE
 * float (w2 / (B_depth * count)), so no host sync is needed. */
int vsx_depth_loss(const float *depth, const uint8_t *valid, const float *prior,
                   const uint8_t *prior_valid, int64_t n, double *sums, uint32_t *counts,
                   const float *scale, float *grad, vsx_stream s);

/* Generic masked L1 over `channels` values per pixel (normal-prior term of
 * the RGB-D-N objective; channels = 1 reproduces vsx_depth_loss). */
int vsx_masked_l1(const float *x, const uint8_t *valid, const float *prior,
                  const uint8_t *prior_valid, int64_t n_pix, int32_t channels, double *sums,
                  uint32_t *counts, const float *scale, float *grad, vsx_stream s);

/* ---- K10: fused Adam (trainer.py:220-247) ------------------------------- */
/* One launch over n_seg contiguous segments (16-byte aligned buffers, each
 * segment starting on a multiple of 4 elements); seg_begin (n_seg+1, host) are
 * element offsets into the flat param/grad/m/v buffers, lr (n_seg, host). */
int vsx_adam(float *param, const float *grad, float *m, float *v, int32_t n_seg,
             const int64_t *seg_begin, const double *lr, double beta1, double beta2, double eps,
             int32_t step, vsx_stream s);
/* Same update, skipped on the device when *guard (device int32) is nonzero:
 * the trainer queues it before its single host read, with guard = status bits
 * | non-finite loss, so the non-finite check still precedes the update
 * (trainer.py:317-321) without a host round trip in front of Adam. */
int vsx_adam_guarded(float *param, const float *grad, float *m, float *v, int32_t n_seg,
                     const int64_t *seg_begin, const double *lr, double beta1, double beta2,
                     double eps, int32_t step, const int32_t *guard, vsx_stream s);

/* ---- f1: depth-prior precompute (depth_prior.py:85-214) ------------------ */
/* float64 device maps (H, W) row-major with uint8 validity. Replaces the
 * numpy passes of fit_scale_shift (:85-110; the 2x2 normal equations and the
 * MAD refit stay on the host), apply_scale_shift (:132-140),
 * reprojection_error (:143-187) and enhance (:205-214). */
/* Per point: camera z, and the bilinearly sampled raw depth when the point
 * projects in front (z > 1e-9) inside [0, W-1] x [0, H-1]; ok = 0 (not
 * projected), 1 (projected, some touched texel invalid), 2 (sampled). */
int vsx_prior_sample(const double *points, int64_t n, vsx_camera cam, const double *depth,
                     const uint8_t *valid, double *raw, double *z, uint8_t *ok, vsx_stream s);
/* metric = scale * raw + shift where valid (NULL: finite and > 0) and the
 * result is finite and > 0; 0 elsewhere. */
int vsx_apply_scale_shift(const double *raw, const uint8_t *valid, int64_t n, double scale,
                          double shift, double *out, uint8_t *out_valid, vsx_stream s);
/* Pixel round-trip error src -> ref -> src for every valid source pixel
 * (+inf where the chain breaks); accumulate_min != 0 min-combines into err. */
int vsx_reprojection_error(const double *src, const uint8_t *src_valid, vsx_camera view_src,
                           const double *ref, const uint8_t *ref_valid, vsx_camera view_ref,
                           double *err, int32_t accumulate_min, vsx_stream s);
/* Enhanced prior: keep valid source pixels with min round trip <= tau. */
int vsx_enhance_finalize(const double *src, const uint8_t *src_valid, const double *emin,
                         double tau, int64_t n, double *out, uint8_t *out_valid, vsx_stream s);

/* ---- f2: multi-view patch NCC loss, Eq. 10 (losses.py:98-287) ----------- */
/* Relative pose (R_rel = R_ref R_src^T, t_rel = t_ref - R_rel t_src, row-major)
 * and both intrinsics of a (reference, source) pair (losses.py:118-128). */
typedef struct vsx_ncc_geom {
  double r_rel[9];
  double t_rel[3];
  double src_fx, src_fy, src_cx, src_cy;
  double ref_fx, ref_fy, ref_cx, ref_cy;
} vsx_ncc_geom;

/* Per patch centre (int32 (u, v) pairs chosen by the host's stratified draw,
 * losses.py:184-206): term = 1 - NCC of the (2h+1)^2 source grayscale patch
 * against the reference grayscale warped by the plane homography of the
 * rendered source normal/depth at the centre; status 0 plane rejected,
 * 1 warp outside the reference, 2 used; the per-patch gradients of the term
 * w.r.t. the patch pixels' grayscale, the centre normal and the centre depth.
 * pair_sum / pair_used get the pair's sum of terms and used count, and
 * pairs_used (device counter) is incremented when the pair used a patch. */
int vsx_ncc_patches(const float *src_rgb, const float *src_normal, const float *src_depth,
                    int32_t src_width, int32_t src_height, const float *ref_rgb,
                    int32_t ref_width, int32_t ref_height, vsx_ncc_geom geom,
                    const int32_t *centers, int32_t n_patches, int32_t half, double *term,
                    uint8_t *status, double *g_patch, double *g_normal, double *g_depth,
                    double *pair_sum, int32_t *pair_used, int32_t *pairs_used, vsx_stream s);
/* Adds upstream / (pairs_used * pair_used) times the per-patch gradients into
 * the source cotangent images g_rgb (H,W,3), g_normal (H,W,3), g_depth (H,W). */
int vsx_ncc_scatter(const int32_t *centers, int32_t n_patches, int32_t half, int32_t src_width,
                    const uint8_t *status, const double *g_patch, const double *g_normal,
                    const double *g_depth, const int32_t *pair_used, const int32_t *pairs_used,
                    double upstream, float *g_rgb, float *g_normal_img, float *g_depth_img,
                    vsx_stream s);

/* ---- f4: TSDF fusion (fusion.py:102-133) --------------------------------- */
/* Folds one depth map (float64 (H, W) + uint8 valid, device) into a dense
 * volume: tsdf / weight are float64 device arrays of dims[0]*dims[1]*dims[2]
 * voxels (ij-indexed, voxel (i,j,k) at origin + (i,j,k)*voxel_size); dims
 * (3 int64) and origin (3 double) are HOST arrays. *touched (device u64) is
 * incremented by the number of voxels updated. */
int vsx_tsdf_integrate(double *tsdf, double *weight, const int64_t *dims, const double *origin,
                       double voxel_size, double truncation, const double *depth,
                       const uint8_t *valid, vsx_camera cam, unsigned long long *touched,
                       vsx_stream s);

/* ---- diagnostics --------------------------------------------------------- */
/* tcgen05 self-test: D[128 x N] = A[128 x K] . B[N x K]^T, kind::tf32 from
 * shared memory into TMEM (three != 0: 3xTF32 split). */
int vsx_umma_selftest(const float *A, const float *B, float *D, int32_t N, int32_t K,
                      int32_t three, vsx_stream s);

#ifdef __cplusplus
}
#endif
#endif /* VSX_B200_H */
