// K4 — tile binning as two stable counting sorts (rows, then columns).
//
// The reference lists, for every 16x16 tile, the depth-sorted splats whose
// tile rectangle covers it, in ascending depth rank (renderer.py:216-226:
// per splat the row-major tiles of its rectangle, then a stable sort by tile
// id). Since every splat covers a rectangle, the (tile, rank) order factors
// into a row pass and a column pass, each a stable counting sort over at
// most 256 buckets with the rectangle expanded on the fly:
//
//   plan  bin_rect_kernel        rectangle per splat (float64, renderer.py
//                                :216-221); per-CTA row counts; per-row pair
//                                totals; row-entry and pair totals
//   rows  bin_rows_scan_kernel   CTA-order offsets per row (CTA per row); the
//                                last CTA: row starts, pair bases, chunking
//         bin_rows_emit_kernel   row lists (rank, x0 | x1 << 16), ascending
//                                rank within each row
//   cols  bin_cols_count_kernel  per (row chunk, column) counts
//         bin_cols_scan_kernel   per-row chunk-order offsets and tile_offsets
//         bin_cols_emit_kernel   tile_list
//
// Stability: CTAs take consecutive ranges (offsets by CTA order), warps
// consecutive sub-ranges (offsets by warp order), and a warp expands its
// items in order, 32 expanded elements per round, ranking equal buckets with
// a per-warp bucket mask. Counts come from difference arrays (two shared atomics per
// interval). The emit kernels place their output bucket-grouped in shared
// memory first and then store runs (one per bucket) with consecutive lanes
// on consecutive addresses; a CTA whose output exceeds the staging buffer
// stores directly. The output is the reference's order exactly (ranks are
// unique). Traffic per view: n rectangles, E = sum of rectangle heights row
// entries (8 B, written once, read twice), P pairs (4 B, written once).
#include "common.cuh"

namespace vsx {

constexpr int kBinSplats = 512;   // splats per CTA in the plan / row passes
constexpr int kBinChunk = 1024;   // row entries per CTA in the column passes
constexpr int kBinWarps = 8;
constexpr int kRowCap = 2560;     // staged row entries per CTA (rows pass)
constexpr int kColCap = 5120;     // staged pairs per CTA (columns pass)

struct BinWs {
  uint2 *rect;                   // [n] (x0 | x1 << 16, y0 | y1 << 16); empty: y0 > y1
  uint32_t *mrow;                // [ctas][tyn] row counts -> offsets
  unsigned long long *totals;    // [2] row entries, pairs
  uint32_t *rowpairs;            // [tyn] pairs per row
  uint32_t *rowtot;              // [tyn] row entries per row
  uint32_t *ticket;              // [1] finished rows-scan CTAs
  uint32_t *rowstart;            // [tyn + 1]
  uint32_t *pairbase;            // [tyn + 1] first pair of each row
  uint32_t *cpre;                // [tyn + 1] first chunk of each row
  uint2 *rows;                   // [E] (rank, x0 | x1 << 16)
  uint32_t *mcol;                // [chunks][txn] column counts -> per-row offsets
};

static size_t a256(size_t b) { return (b + 255) & ~size_t(255); }
static int64_t rect_ctas(int64_t n) { return std::max<int64_t>((n + kBinSplats - 1) / kBinSplats, 1); }
static int64_t col_chunks(int64_t E, int tyn) { return (E + kBinChunk - 1) / kBinChunk + tyn; }

static size_t bin_plan_bytes(int64_t n, int tyn) {
  return a256(8 * (size_t)n) + a256(4 * (size_t)rect_ctas(n) * tyn) + a256(16) +
         3 * a256(4 * (size_t)tyn) + 3 * a256(4 * (size_t)(tyn + 1));
}

static size_t bin_build_bytes(int txn, int tyn, int64_t E) {
  return a256(8 * (size_t)E) + a256(4 * (size_t)col_chunks(E, tyn) * txn);
}

// plan workspace (rectangles, row counts, totals, row starts, chunking) and
// build workspace (row lists, column counts)
static BinWs carve_bin_ws(void *plan, int64_t n, int tyn, void *build, int txn, int64_t E) {
  char *p = static_cast<char *>(plan);
  BinWs w;
  w.rect = reinterpret_cast<uint2 *>(p);
  p += a256(8 * (size_t)n);
  w.mrow = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)rect_ctas(n) * tyn);
  w.totals = reinterpret_cast<unsigned long long *>(p);
  p += a256(16);
  w.rowpairs = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)tyn);
  w.rowtot = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)tyn);
  w.ticket = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)tyn);
  w.rowstart = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)(tyn + 1));
  w.pairbase = reinterpret_cast<uint32_t *>(p);
  p += a256(4 * (size_t)(tyn + 1));
  w.cpre = reinterpret_cast<uint32_t *>(p);
  char *q = static_cast<char *>(build);
  w.rows = reinterpret_cast<uint2 *>(q);
  w.mcol = q ? reinterpret_cast<uint32_t *>(q + a256(8 * (size_t)E)) : nullptr;
  return w;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Exclusive scan over a 256-thread CTA (all threads call); *total = sum.
__device__ __forceinline__ uint32_t block_excl_256(uint32_t v, uint32_t *s_w, uint32_t &total) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t inc = warp_incl_scan(v, lane);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint32_t base = 0;
  total = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t s = s_w[k];
    base += k < warp ? s : 0u;
    total += s;
  }
  __syncthreads();
  return base + inc - v;
}

// Expand the warp's 32 items (item on lane k covers buckets lo_k .. lo_k +
// cnt_k - 1, payload pay_k) in item order, 32 expanded (bucket, payload)
// elements per round; f(bucket, payload, valid) is called by every lane each
// round. Items with cnt > 0 are first compacted to lanes 0..np-1, so within
// a round the item of element e is found from the bitmask of the items that
// start in the round (one REDUX) and a running count of earlier starts.
template <typename F>
__device__ __forceinline__ void warp_expand(int lo, int cnt, uint32_t pay, int lane,
                                            uint32_t *s_cmp, F &&f) {
  const unsigned pos = __ballot_sync(0xffffffffu, cnt > 0);
  const int np = __popc(pos);
  if (np == 0) return;
  // compaction through shared memory (3 words per item)
  if (cnt > 0) {
    const int d = __popc(pos & ((1u << lane) - 1u));
    s_cmp[d] = (uint32_t)lo;
    s_cmp[32 + d] = (uint32_t)cnt;
    s_cmp[64 + d] = pay;
  }
  __syncwarp();
  cnt = lane < np ? (int)s_cmp[32 + lane] : 0;
  lo = (int)s_cmp[lane];
  pay = s_cmp[64 + lane];
  __syncwarp();
  const uint32_t incl = warp_incl_scan((uint32_t)cnt, lane);
  const uint32_t excl = incl - (uint32_t)cnt;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const int base = lo - (int)excl;  // bucket of element e of this item = base + e
  const unsigned upto = 0xffffffffu >> (31 - lane);
  int started = 0;  // items starting before this round
  for (uint32_t e0 = 0; e0 < total; e0 += 32) {
    const uint32_t d = excl - e0;
    const unsigned M = __reduce_or_sync(0xffffffffu, (lane < np && d < 32u) ? 1u << d : 0u);
    const int r = started - 1 + __popc(M & upto);
    started += __popc(M);
    const int b = __shfl_sync(0xffffffffu, base, r);
    const uint32_t p = __shfl_sync(0xffffffffu, pay, r);
    const uint32_t e = e0 + (uint32_t)lane;
    f(b + (int)e, p, e < total);
  }
}

// Stable rank of this lane's element among the warp's elements of the same
// bucket. Peers come from a per-warp bucket mask: every lane ORs its bit in
// and reads the group's mask back (one shared atomic; MATCH.ANY measured
// 79 us and eight ballots 57 us for this kernel, against 49.5 us); the last
// peer advances the warp counter wh[bucket] and clears the mask.
__device__ __forceinline__ uint32_t warp_rank(uint32_t *wh, uint32_t *wm, int bucket, bool valid,
                                              int lane) {
  if (valid) atomicOr(wm + bucket, 1u << lane);
  __syncwarp();
  const unsigned peers = valid ? wm[bucket] : 1u << lane;
  const uint32_t cur = valid ? wh[bucket] : 0u;
  __syncwarp();
  if (valid && (peers >> lane) == 1u) {
    wh[bucket] = cur + __popc(peers);
    wm[bucket] = 0u;
  }
  __syncwarp();
  return cur + __popc(peers & ((1u << lane) - 1u));
}

// Per-bucket counts of intervals [lo, hi] by a difference array (two shared
// atomics per interval) followed by a prefix sum: d has 257 entries, zeroed.
__device__ __forceinline__ void diff_add(uint32_t *d, int lo, int hi, uint32_t wgt = 1u) {
  if (hi >= lo) {
    atomicAdd(d + lo, wgt);
    atomicAdd(d + hi + 1, 0u - wgt);
  }
}

// In-place prefix of one warp's 256-entry difference array (8 per lane).
__device__ __forceinline__ void warp_diff_to_counts(uint32_t *d, int lane) {
  uint32_t v[8], s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = d[8 * lane + k];
    s += v[k];
  }
  uint32_t run = warp_incl_scan(s, lane) - s;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    run += v[k];
    d[8 * lane + k] = run;
  }
}

// A CTA takes kRectSub consecutive row-pass chunks of kBinSplats splats:
// one row histogram per chunk (the row pass's CTA granularity), one pair
// histogram for all of them.
constexpr int kRectSub = 4;

__global__ void __launch_bounds__(256) bin_rect_kernel(const vsx_splat *__restrict__ rec,
                                                       const double *__restrict__ radius,
                                                       int32_t n, int txn, int tyn, BinWs w,
                                                       int chunks) {
  __shared__ uint32_t h[kRectSub][257], hp[257];
  const int t = threadIdx.x;
#pragma unroll
  for (int c = 0; c < kRectSub; ++c) h[c][t] = 0u;
  hp[t] = 0u;
  if (t < kRectSub) h[t][256] = 0u;
  if (t == 0) hp[256] = 0u;
  __syncthreads();
  unsigned long long rows = 0, pairs = 0;
  for (int c = 0; c < kRectSub; ++c) {
    const int chunk = blockIdx.x * kRectSub + c;
#pragma unroll
    for (int k = 0; k < kBinSplats / 256; ++k) {
      const int i = chunk * kBinSplats + k * 256 + t;
      if (i >= n) break;
      int x0 = 0, x1 = -1, y0 = 1, y1 = 0;
      if (tile_rect(rec[i].mean2d[0], rec[i].mean2d[1], radius[i], txn, tyn, x0, x1, y0, y1)) {
        diff_add(h[c], y0, y1);
        diff_add(hp, y0, y1, (uint32_t)(x1 - x0 + 1));
        rows += (unsigned long long)(y1 - y0 + 1);
        pairs += (unsigned long long)(y1 - y0 + 1) * (unsigned long long)(x1 - x0 + 1);
        w.rect[i] = make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
      } else {
        w.rect[i] = make_uint2(0u, 1u);  // y0 = 1 > y1 = 0: no rows
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rows += __shfl_xor_sync(0xffffffffu, rows, o);
    pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
  }
  if ((t & 31) == 0) {
    if (rows) atomicAdd(&w.totals[0], rows);
    if (pairs) atomicAdd(&w.totals[1], pairs);
  }
  __syncthreads();
  const int warp = t >> 5;
  if (warp < kRectSub) warp_diff_to_counts(h[warp], t & 31);
  else if (warp == kRectSub) warp_diff_to_counts(hp, t & 31);
  __syncthreads();
  if (t < tyn) {
#pragma unroll
    for (int c = 0; c < kRectSub; ++c) {
      const int chunk = blockIdx.x * kRectSub + c;
      if (chunk < chunks) w.mrow[(size_t)chunk * tyn + t] = h[c][t];
    }
    if (hp[t]) atomicAdd(&w.rowpairs[t], hp[t]);
  }
}

// CTA per tile row: CTA-order exclusive prefix of the row's counts (thread t
// takes a contiguous run of CTAs). The last CTA to finish derives the row
// starts, the pair base of every row and the column-pass chunking.
__global__ void __launch_bounds__(256) bin_rows_scan_kernel(int ctas, int tyn, BinWs w) {
  __shared__ uint32_t s_w[8];
  __shared__ bool s_last;
  const int y = blockIdx.x, t = threadIdx.x;
  const int per = (ctas + 255) / 256, c0 = t * per;
  uint32_t sum = 0;
  for (int k = 0; k < per; ++k)
    if (c0 + k < ctas) sum += w.mrow[(size_t)(c0 + k) * tyn + y];
  uint32_t tot;
  uint32_t run = block_excl_256(sum, s_w, tot);
  for (int k = 0; k < per; ++k)
    if (c0 + k < ctas) {
      uint32_t *m = w.mrow + (size_t)(c0 + k) * tyn + y;
      const uint32_t v = *m;
      *m = run;
      run += v;
    }
  if (t == 0) {
    w.rowtot[y] = tot;
    __threadfence();
    s_last = atomicAdd(w.ticket, 1u) == (uint32_t)tyn - 1u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA: rows 8 per lane in warp 0
  if (t < 32) {
    const int lane = t;
    uint32_t len[8], nch[8], prs[8], sl = 0, sc = 0, sp = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 8 * lane + k;
      len[k] = r < tyn ? __ldcg(w.rowtot + r) : 0u;
      prs[k] = r < tyn ? __ldcg(w.rowpairs + r) : 0u;
      nch[k] = (len[k] + kBinChunk - 1) / kBinChunk;
      sl += len[k];
      sc += nch[k];
      sp += prs[k];
    }
    const uint32_t il = warp_incl_scan(sl, lane), ic = warp_incl_scan(sc, lane),
                   ip = warp_incl_scan(sp, lane);
    uint32_t rl = il - sl, rc = ic - sc, rp = ip - sp;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 8 * lane + k;
      if (r < tyn) {
        w.rowstart[r] = rl;
        w.cpre[r] = rc;
        w.pairbase[r] = rp;
      }
      rl += len[k];
      rc += nch[k];
      rp += prs[k];
    }
    if (lane == 31) {
      w.rowstart[tyn] = il;
      w.cpre[tyn] = ic;
      w.pairbase[tyn] = ip;
    }
  }
}

// Warp-private counts of a warp's intervals (wh[warp], 257 entries zeroed by
// the caller) turned into per-warp bases: thread b < nb of the CTA folds the
// warps of bucket b starting at base(b). Returns through wh.
__device__ __forceinline__ void warp_bases(uint32_t (*wh)[257], int nb, uint32_t base_b) {
  const int t = threadIdx.x;
  if (t < nb) {
    uint32_t run = base_b;
#pragma unroll
    for (int k = 0; k < kBinWarps; ++k) {
      const uint32_t v = wh[k][t];
      wh[k][t] = run;
      run += v;
    }
  }
}

__global__ void __launch_bounds__(256) bin_rows_emit_kernel(int32_t n, int tyn, BinWs w) {
  __shared__ uint32_t wh[kBinWarps][257];
  __shared__ uint32_t s_cmp[kBinWarps][96];
  __shared__ uint32_t wm[kBinWarps][256];
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_g[256];  // global minus local position per row
  __shared__ uint2 s_val[kRowCap];
  __shared__ uint8_t s_b[kRowCap];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int k = 0; k < kBinWarps; ++k) wh[k][t] = 0u;
  if (t < kBinWarps) wh[t][256] = 0u;
#pragma unroll
  for (int k = 0; k < kBinWarps; ++k) wm[k][t] = 0u;
  __syncthreads();
  constexpr int kPer = kBinSplats / kBinWarps;
  const int wbase = blockIdx.x * kBinSplats + warp * kPer;
  for (int g = 0; g < kPer; g += 32) {
    const int i = wbase + g + lane;
    if (i < n) {
      const uint2 r = w.rect[i];
      diff_add(wh[warp], (int)(r.y & 0xffffu), (int)(r.y >> 16));
    }
  }
  __syncwarp();
  warp_diff_to_counts(wh[warp], lane);
  __syncthreads();
  uint32_t cnt = 0;
  if (t < tyn)
#pragma unroll
    for (int k = 0; k < kBinWarps; ++k) cnt += wh[k][t];
  uint32_t total;
  const uint32_t loc = block_excl_256(cnt, s_w, total);
  const bool staged = total <= (uint32_t)kRowCap;
  const uint32_t glob = t < tyn ? w.rowstart[t] + w.mrow[(size_t)blockIdx.x * tyn + t] : 0u;
  s_g[t] = glob - loc;
  warp_bases(wh, tyn, staged ? loc : glob);
  __syncthreads();
  for (int g = 0; g < kPer; g += 32) {
    const int i = wbase + g + lane;
    uint2 r = make_uint2(0u, 1u);
    if (i < n) r = w.rect[i];
    const int y0 = (int)(r.y & 0xffffu), y1 = (int)(r.y >> 16);
    // payload: the lane (the splat is wbase + g + lane, its x range in r.x)
    warp_expand(y0, y1 >= y0 ? y1 - y0 + 1 : 0, (uint32_t)lane, lane, s_cmp[warp],
                [&](int y, uint32_t k, bool valid) {
      const uint32_t xs = __shfl_sync(0xffffffffu, r.x, (int)k);
      const uint32_t pos = warp_rank(wh[warp], wm[warp], y, valid, lane);
      const uint2 v = make_uint2((uint32_t)(wbase + g) + k, xs);
      if (valid) {
        if (staged) {
          s_val[pos] = v;
          s_b[pos] = (uint8_t)y;
        } else {
          w.rows[pos] = v;
        }
      }
    });
  }
  if (staged) {
    __syncthreads();
    for (uint32_t j = t; j < total; j += 256) w.rows[s_g[s_b[j]] + j] = s_val[j];
  }
}

// Row y and entry range of column-pass CTA c (c < cpre[tyn]).
__device__ __forceinline__ bool col_chunk(const BinWs &w, int tyn, int c, int &y, uint32_t &b,
                                          uint32_t &e) {
  if ((uint32_t)c >= w.cpre[tyn]) return false;
  int lo = 0, hi = tyn - 1;  // last row with cpre[y] <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (w.cpre[mid] <= (uint32_t)c) lo = mid;
    else hi = mid - 1;
  }
  y = lo;
  b = w.rowstart[y] + (uint32_t)(c - (int)w.cpre[y]) * kBinChunk;
  e = min(b + (uint32_t)kBinChunk, w.rowstart[y + 1]);
  return true;
}

__global__ void __launch_bounds__(256) bin_cols_count_kernel(int txn, int tyn, BinWs w) {
  __shared__ uint32_t h[257];
  const int t = threadIdx.x;
  int y;
  uint32_t b, e;
  if (!col_chunk(w, tyn, blockIdx.x, y, b, e)) return;
  h[t] = 0u;
  if (t == 0) h[256] = 0u;
  __syncthreads();
  for (uint32_t q = b + t; q < e; q += 256) {
    const uint32_t xs = w.rows[q].y;
    diff_add(h, (int)(xs & 0xffffu), (int)(xs >> 16));
  }
  __syncthreads();
  if (t < 32) warp_diff_to_counts(h, t);
  __syncthreads();
  if (t < txn) w.mcol[(size_t)blockIdx.x * txn + t] = h[t];
}

// CTA per tile row, thread x = column: chunk-order offsets within the row,
// then tile_offsets of the row = pair base of the row + exclusive scan of
// its tile counts (tile_offsets[T] = all pairs, from the last row).
__global__ void __launch_bounds__(256) bin_cols_scan_kernel(int txn, int tyn, BinWs w,
                                                            uint32_t *__restrict__ toff) {
  __shared__ uint32_t s_w[8];
  const int y = blockIdx.x, x = threadIdx.x;
  uint32_t run = 0;
  if (x < txn) {
    const uint32_t c1 = w.cpre[y + 1];
    for (uint32_t c0 = w.cpre[y]; c0 < c1; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = c0 + k < c1 ? w.mcol[(size_t)(c0 + k) * txn + x] : 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (c0 + k < c1) w.mcol[(size_t)(c0 + k) * txn + x] = run;
        run += v[k];
      }
    }
  }
  uint32_t tot;
  const uint32_t ex = block_excl_256(run, s_w, tot);
  if (x < txn) toff[y * txn + x] = w.pairbase[y] + ex;
  if (y == tyn - 1 && x == 0) toff[tyn * txn] = w.pairbase[tyn];
}

__global__ void __launch_bounds__(256) bin_cols_emit_kernel(int txn, int tyn, BinWs w,
                                                            const uint32_t *__restrict__ toff,
                                                            uint32_t *__restrict__ tile_list) {
  __shared__ uint32_t wh[kBinWarps][257];
  __shared__ uint32_t s_cmp[kBinWarps][96];
  __shared__ uint32_t wm[kBinWarps][256];
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_g[256];  // global minus local position per column
  __shared__ uint32_t s_val[kColCap];
  __shared__ uint8_t s_b[kColCap];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int y;
  uint32_t b, e;
  if (!col_chunk(w, tyn, blockIdx.x, y, b, e)) return;
#pragma unroll
  for (int k = 0; k < kBinWarps; ++k) wh[k][t] = 0u;
  if (t < kBinWarps) wh[t][256] = 0u;
#pragma unroll
  for (int k = 0; k < kBinWarps; ++k) wm[k][t] = 0u;
  __syncthreads();
  constexpr int kPer = kBinChunk / kBinWarps;
  const uint32_t wb = b + (uint32_t)warp * kPer;
  const uint32_t we = min(wb + (uint32_t)kPer, e);
  for (uint32_t q = wb + lane; q < we; q += 32) {
    const uint32_t xs = w.rows[q].y;
    diff_add(wh[warp], (int)(xs & 0xffffu), (int)(xs >> 16));
  }
  __syncwarp();
  warp_diff_to_counts(wh[warp], lane);
  __syncthreads();
  uint32_t cnt = 0;
  if (t < txn)
#pragma unroll
    for (int k = 0; k < kBinWarps; ++k) cnt += wh[k][t];
  uint32_t total;
  const uint32_t loc = block_excl_256(cnt, s_w, total);
  const bool staged = total <= (uint32_t)kColCap;
  const uint32_t glob = t < txn ? toff[y * txn + t] + w.mcol[(size_t)blockIdx.x * txn + t] : 0u;
  s_g[t] = glob - loc;
  warp_bases(wh, txn, staged ? loc : glob);
  __syncthreads();
  for (uint32_t q0 = wb; q0 < we; q0 += 32) {
    const uint32_t q = q0 + lane;
    uint2 ent = make_uint2(0u, 1u);  // x0 = 1 > x1 = 0: nothing
    if (q < we) ent = w.rows[q];
    const int x0 = (int)(ent.y & 0xffffu), x1 = (int)(ent.y >> 16);
    warp_expand(x0, x1 >= x0 ? x1 - x0 + 1 : 0, ent.x, lane, s_cmp[warp],
                [&](int x, uint32_t rank, bool valid) {
      const uint32_t pos = warp_rank(wh[warp], wm[warp], x, valid, lane);
      if (valid) {
        if (staged) {
          s_val[pos] = rank;
          s_b[pos] = (uint8_t)x;
        } else {
          tile_list[pos] = rank;
        }
      }
    });
  }
  if (staged) {
    __syncthreads();
    for (uint32_t j = t; j < total; j += 256) tile_list[s_g[s_b[j]] + j] = s_val[j];
  }
}

}  // namespace vsx

using namespace vsx;

extern "C" size_t vsx_bin_plan_ws_bytes(int32_t n, int32_t width, int32_t height) {
  const int tyn = (height + kTile - 1) / kTile;
  return bin_plan_bytes(std::max(n, 0), tyn);
}

extern "C" size_t vsx_bin_build_ws_bytes(int32_t width, int32_t height, int64_t row_entries) {
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  return bin_build_bytes(txn, tyn, std::max<int64_t>(row_entries, 0));
}

extern "C" int vsx_bin_plan(const vsx_splat *rec, const double *radius, int32_t n, int32_t width,
                            int32_t height, void *plan_ws, size_t plan_bytes, uint64_t *totals,
                            vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0 && plan_ws, "bin_plan: bad arguments");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  VSX_REQUIRE(txn <= 256 && tyn <= 256, "bin_plan: more than 256 tile rows or columns");
  VSX_REQUIRE(plan_bytes >= bin_plan_bytes(n, tyn), "bin_plan: workspace too small");
  cudaStream_t st = as_stream(s);
  BinWs w = carve_bin_ws(plan_ws, n, tyn, nullptr, txn, 0);
  // totals, rowpairs, rowtot and the ticket are contiguous
  VSX_CUDA_TRY(cudaMemsetAsync(w.totals, 0,
                               reinterpret_cast<char *>(w.rowstart) -
                                   reinterpret_cast<char *>(w.totals), st));
  if (n > 0) {
    const int chunks = (int)rect_ctas(n);
    bin_rect_kernel<<<(chunks + kRectSub - 1) / kRectSub, 256, 0, st>>>(rec, radius, n, txn, tyn, w,
                                                                       chunks);
    VSX_LAUNCH_CHECK("bin_rect");
  }
  if (totals) VSX_CUDA_TRY(cudaMemcpyAsync(totals, w.totals, 16, cudaMemcpyDefault, st));
  return VSX_OK;
}

extern "C" int vsx_bin_build(int32_t n, int32_t width, int32_t height, int64_t row_entries,
                             int64_t pairs, void *plan_ws, size_t plan_bytes, void *build_ws,
                             size_t build_bytes, uint32_t *tile_offsets, uint32_t *tile_list,
                             vsx_stream s) {
  VSX_REQUIRE(width > 0 && height > 0 && n >= 0 && row_entries >= 0 && pairs >= 0 && plan_ws &&
                  tile_offsets, "bin_build: bad arguments");
  VSX_REQUIRE(pairs < ((int64_t)1 << 32) && row_entries < ((int64_t)1 << 32),
              "bin_build: more than 2^32 pairs");
  const int txn = (width + kTile - 1) / kTile, tyn = (height + kTile - 1) / kTile;
  VSX_REQUIRE(txn <= 256 && tyn <= 256, "bin_build: more than 256 tile rows or columns");
  VSX_REQUIRE(plan_bytes >= bin_plan_bytes(n, tyn), "bin_build: plan workspace too small");
  cudaStream_t st = as_stream(s);
  if (n == 0 || row_entries == 0 || pairs == 0) {
    VSX_CUDA_TRY(cudaMemsetAsync(tile_offsets, 0, sizeof(uint32_t) * (txn * tyn + 1), st));
    return VSX_OK;
  }
  VSX_REQUIRE(build_ws && build_bytes >= bin_build_bytes(txn, tyn, row_entries) && tile_list,
              "bin_build: build workspace too small");
  BinWs w = carve_bin_ws(plan_ws, n, tyn, build_ws, txn, row_entries);
  const int ctas = (int)rect_ctas(n);
  bin_rows_scan_kernel<<<tyn, 256, 0, st>>>(ctas, tyn, w);
  VSX_LAUNCH_CHECK("bin_rows_scan");
  bin_rows_emit_kernel<<<ctas, 256, 0, st>>>(n, tyn, w);
  VSX_LAUNCH_CHECK("bin_rows_emit");
  const int chunks = (int)col_chunks(row_entries, tyn);
  bin_cols_count_kernel<<<chunks, 256, 0, st>>>(txn, tyn, w);
  VSX_LAUNCH_CHECK("bin_cols_count");
  bin_cols_scan_kernel<<<tyn, 256, 0, st>>>(txn, tyn, w, tile_offsets);
  VSX_LAUNCH_CHECK("bin_cols_scan");
  bin_cols_emit_kernel<<<chunks, 256, 0, st>>>(txn, tyn, w, tile_offsets, tile_list);
  VSX_LAUNCH_CHECK("bin_cols_emit");
  return VSX_OK;
}
