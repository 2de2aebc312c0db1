// Generic device primitives: error state, exclusive scan, ordered select,
// stable LSD radix sort. Hand-written (no CUB) so the sort's stability —
// which carries the reference's (z, gid) tie-break — is explicit.
#include <atomic>
#include <cstdarg>

#include "common.cuh"

static thread_local char g_err[512] = "";

void vsx_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char *vsx_last_error(void) { return g_err; }
extern "C" int vsx_version(void) { return 1; }

// Every kernel launch of this library bumps one counter (VSX_LAUNCH_CHECK),
// so callers can report how many of OUR kernels ran in a timed region.
static std::atomic<unsigned long long> g_launches{0};
void vsx_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" uint64_t vsx_launch_count(void) { return g_launches.load(); }

namespace vsx {

// ------------------------------------------------------------------ scan

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t &total) {
  __shared__ uint32_t warp_tot[kScanBlock / 32];
  __shared__ uint32_t tot_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kScanBlock / 32 ? warp_tot[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kScanBlock / 32) warp_tot[lane] = wi - w;
    if (lane == kScanBlock / 32 - 1) tot_s = wi;
  }
  __syncthreads();
  const uint32_t res = warp_tot[warp] + inc - v;
  total = tot_s;
  __syncthreads();
  return res;
}

// Tile-local exclusive scan; tile total goes to sums[blockIdx.x].
__global__ void scan_tiles_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                  int64_t n, uint32_t *__restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0u;
    acc += v[i];
  }
  uint32_t total = 0;
  uint32_t pre = block_exclusive_scan(acc, total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = pre;
    pre += v[i];
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void scan_add_kernel(uint32_t *__restrict__ out, int64_t n,
                                const uint32_t *__restrict__ tile_off, int64_t n_tiles) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / kScanTile];
  if (i == 0) out[n] = tile_off[n_tiles];
}

static size_t scan_ws_elems(int64_t n) {
  if (n <= kScanTile) return 0;
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  return (size_t)(2 * nt + 1) + scan_ws_elems(nt);
}

static int scan_impl(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *ws,
                     cudaStream_t st) {
  if (n <= kScanTile) {
    scan_tiles_kernel<<<1, kScanBlock, 0, st>>>(in, out, n, out + n);
    VSX_LAUNCH_CHECK("scan_tiles");
    return VSX_OK;
  }
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  uint32_t *sums = ws;
  uint32_t *sums_scan = ws + nt;
  scan_tiles_kernel<<<(unsigned)nt, kScanBlock, 0, st>>>(in, out, n, sums);
  VSX_LAUNCH_CHECK("scan_tiles");
  int rc = scan_impl(sums, sums_scan, nt, ws + 2 * nt + 1, st);
  if (rc) return rc;
  scan_add_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, sums_scan, nt);
  VSX_LAUNCH_CHECK("scan_add");
  return VSX_OK;
}

// ------------------------------------------------------------------ select

// ------------------------------------------------------------------ radix sort

template <typename K>
__global__ void rs_minmax_kernel(const K *__restrict__ keys, int64_t n,
                                 unsigned long long *__restrict__ or_and) {
  unsigned long long o = 0ull, a = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = (unsigned long long)keys[i];
    o |= k;
    a &= k;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    o |= __shfl_xor_sync(0xffffffffu, o, s);
    a &= __shfl_xor_sync(0xffffffffu, a, s);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&or_and[0], o);
    atomicAnd(&or_and[1], a);
  }
}

__global__ void rs_init_or_and(unsigned long long *or_and) {
  or_and[0] = 0ull;
  or_and[1] = ~0ull;
}

// ------------------------------------------------ single-pass (onesweep) passes
//
// One kernel per 8-bit digit pass. Each CTA takes the next tile index from an
// atomic counter (so every lower tile has started and will finish), ranks its
// 4096 keys with warp-private digit counters (match_any, no CTA barriers in
// the ranking loop), publishes its per-digit counts, and obtains the exclusive
// per-digit prefix of all earlier tiles by decoupled look-back on a
// (flag:2 | count:30) status word per (tile, digit). A single histogram kernel
// up front supplies the global digit totals of every pass. Launches per sort:
// memset + histogram + one per pass (the older multi-kernel LSD sort needed
// histogram + 3-level scan + scatter per pass).

constexpr int kOsBlock = 256;
constexpr int kOsItems = 16;
constexpr int kOsTile = kOsBlock * kOsItems;  // 4096 keys, 512 per warp
// Smaller tiles for small sorts (kOsItemsSmall, below kOsSmallN keys) are
// kept as an A/B switch.
constexpr int kOsItemsSmall = 4;
#ifndef VSX_OS_WIN
#define VSX_OS_WIN 8
#endif
constexpr int kOsWin = VSX_OS_WIN;  // look-back window (predecessor tiles per step)
#ifndef VSX_OS_SMALL_ON
#define VSX_OS_SMALL_ON 0
#endif
constexpr int64_t kOsSmallN = VSX_OS_SMALL_ON ? ((int64_t)1 << 21) : 0;  // disabled: 1024-key tiles measured 21.2 us per pass at 0.6 M keys, 4096-key 15.5 (the look-back chain grows with the tile count)
__host__ __device__ inline int os_items(int64_t n) { return n <= kOsSmallN ? kOsItemsSmall : kOsItems; }
constexpr int kOsWarps = kOsBlock / 32;
constexpr uint32_t kOsAgg = 1u << 30, kOsPre = 2u << 30, kOsMask = kOsAgg - 1u;

struct OsShifts {
  int s[16];
  int np;
};

// Lanes of the warp holding the same 8-bit digit as this lane (8 ballots;
// cheaper and more predictable than MATCH.ANY), restricted to `valid`.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, unsigned valid) {
  unsigned m = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bal : ~bal;
  }
  return m;
}

// Global digit histograms of every pass in one read. Each thread takes 16
// consecutive keys and run-length merges equal digits before its shared
// atomic: emitted (tile, rank) keys come in long runs of equal high digits,
// which would otherwise serialise on one shared-memory address.
template <typename K>
__global__ void __launch_bounds__(256) os_hist_kernel(const K *__restrict__ keys, int64_t n,
                                                      OsShifts sh, uint32_t *__restrict__ gh) {
  constexpr int kPer = 16;
  __shared__ uint32_t h[8][256];
  for (int p = 0; p < sh.np; ++p) h[p][threadIdx.x] = 0u;
  __syncthreads();
  for (int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPer; b0 < n;
       b0 += (int64_t)gridDim.x * blockDim.x * kPer) {
    K kk[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) kk[j] = b0 + j < n ? keys[b0 + j] : K(0);
    const int m = (int)min((int64_t)kPer, n - b0);
    for (int p = 0; p < sh.np; ++p) {
      uint32_t cur = (uint32_t)(kk[0] >> sh.s[p]) & 255u, c = 1;
#pragma unroll
      for (int j = 1; j < kPer; ++j) {
        if (j < m) {
          const uint32_t d = (uint32_t)(kk[j] >> sh.s[p]) & 255u;
          if (d == cur) {
            ++c;
          } else {
            atomicAdd(&h[p][cur], c);
            cur = d;
            c = 1;
          }
        }
      }
      atomicAdd(&h[p][cur], c);
    }
  }
  __syncthreads();
  for (int p = 0; p < sh.np; ++p) {
    const uint32_t c = h[p][threadIdx.x];
    if (c) atomicAdd(&gh[p * 256 + threadIdx.x], c);
  }
}

// The look-back words carry their own payload (flag | count), so relaxed
// (L2-coherent) accesses suffice: no other data is published through them.
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename K, int kItems>
__global__ void __launch_bounds__(kOsBlock) os_pass_kernel(
    const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const uint32_t *__restrict__ gh,
    uint32_t *__restrict__ status, uint32_t *__restrict__ counter) {
  // input tile and digit-grouped output tile live in separate buffers, so
  // keys / values are never held in registers across the ranking
  constexpr int kT = kOsBlock * kItems;
  extern __shared__ __align__(16) unsigned char os_smem[];
  K *sk = reinterpret_cast<K *>(os_smem);
  K *ok_ = sk + kT;
  uint32_t *sv = reinterpret_cast<uint32_t *>(ok_ + kT);
  uint32_t *ov = sv + kT;
  __shared__ uint32_t whist[kOsWarps][256];
  __shared__ uint32_t s_lstart[256], s_dst[256];
  __shared__ uint32_t s_bid;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_bid = atomicAdd(counter, 1u);
#pragma unroll
  for (int w = 0; w < kOsWarps; ++w) whist[w][t] = 0u;
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t base = (int64_t)bid * kT;
  const unsigned lt = (1u << lane) - 1u;
  const int nvalid = (int)min((int64_t)kT, n - base);
  // ---- stage the tile with 16-byte loads, all in flight at once
  {
    const bool vec = nvalid == kT &&
                     ((reinterpret_cast<uintptr_t>(kin) | reinterpret_cast<uintptr_t>(vin)) & 15) == 0;
    if (vec) {
      constexpr int kKV = kT * (int)sizeof(K) / 16 / kOsBlock;  // uint4 per thread
      constexpr int kVV = kT * 4 / 16 / kOsBlock;
      const uint4 *gk = reinterpret_cast<const uint4 *>(kin + base);
      const uint4 *gv = reinterpret_cast<const uint4 *>(vin + base);
      uint4 bk[kKV], bv[kVV];
#pragma unroll
      for (int q = 0; q < kKV; ++q) bk[q] = __ldg(gk + q * kOsBlock + t);
#pragma unroll
      for (int q = 0; q < kVV; ++q) bv[q] = __ldg(gv + q * kOsBlock + t);
#pragma unroll
      for (int q = 0; q < kKV; ++q) reinterpret_cast<uint4 *>(sk)[q * kOsBlock + t] = bk[q];
#pragma unroll
      for (int q = 0; q < kVV; ++q) reinterpret_cast<uint4 *>(sv)[q * kOsBlock + t] = bv[q];
    } else {
      for (int s = t; s < nvalid; s += kOsBlock) {
        sk[s] = kin[base + s];
        sv[s] = vin[base + s];
      }
    }
    __syncthreads();
  }
  // ---- warp-private ranking, keys in input order (warp, round, lane)
  uint32_t rk[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int s = warp * (32 * kItems) + r * 32 + lane;
    const bool ok = s < nvalid;
    const uint32_t d = ok ? ((uint32_t)(sk[s] >> shift) & 255u) : 0u;
    const unsigned peers = digit_peers(d, __ballot_sync(0xffffffffu, ok));
    uint32_t cur = 0;
    if (ok) cur = whist[warp][d];
    __syncwarp();
    if (ok && (peers & lt) == 0u) whist[warp][d] = cur + __popc(peers);
    __syncwarp();
    rk[r] = cur + __popc(peers & lt);
  }
  __syncthreads();
  // ---- thread t = digit t: per-warp offsets, tile count, publish aggregate
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kOsWarps; ++w) {
    const uint32_t c = whist[w][t];
    whist[w][t] = cnt;
    cnt += c;
  }
  uint32_t *my = status + (size_t)bid * 256 + t;
  st_relaxed_u32(my, (bid == 0 ? kOsPre : kOsAgg) | cnt);
  uint32_t tot = 0;
  const uint32_t lstart = block_exclusive_scan(cnt, tot);
  const uint32_t gstart = block_exclusive_scan(gh[t], tot);
  s_lstart[t] = lstart;
  // ---- decoupled look-back over earlier tiles (per digit)
  // A window of kOsWin predecessors is read per step (independent loads in
  // flight), consumed nearest-first up to the first inclusive prefix or the
  // first tile that has not published yet (re-read next step).
  uint32_t excl = 0;
  if (bid > 0) {
    int64_t p = (int64_t)bid - 1;
    while (true) {
      uint32_t w[kOsWin];
#pragma unroll
      for (int j = 0; j < kOsWin; ++j)
        w[j] = p - j >= 0 ? ld_relaxed_u32(status + (size_t)(p - j) * 256 + t) : kOsPre;
      int used = 0;
      bool done = false;
#pragma unroll
      for (int j = 0; j < kOsWin; ++j) {
        if (!done && used == j && w[j] != 0u) {
          excl += w[j] & kOsMask;
          ++used;
          done = (w[j] & kOsPre) != 0u;
        }
      }
      if (done) break;
      p -= used;
    }
    st_relaxed_u32(my, kOsPre | (excl + cnt));
  }
  s_dst[t] = gstart + excl - lstart;
  __syncthreads();
  // ---- place keys digit-grouped in the output tile, then coalesced stores
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int s = warp * (32 * kItems) + r * 32 + lane;
    if (s < nvalid) {
      const K kk = sk[s];
      const uint32_t d = (uint32_t)(kk >> shift) & 255u;
      const uint32_t pos = s_lstart[d] + whist[warp][d] + rk[r];
      ok_[pos] = kk;
      ov[pos] = sv[s];
    }
  }
  __syncthreads();
  for (int s = t; s < nvalid; s += kOsBlock) {
    const K kk = ok_[s];
    const uint32_t pos = s_dst[(uint32_t)(kk >> shift) & 255u] + (uint32_t)s;
    kout[pos] = kk;
    vout[pos] = ov[s];
  }
}

// Ordered stream compaction in one pass: 2048 flags per CTA (8 per thread),
// CTA prefix by decoupled look-back over the earlier tiles (tile ids from a
// ticket, so every predecessor is already running), indices written at
// their global rank. Replaces flags -> u32, a two-level scan and a scatter.
constexpr int kSelItems = 8, kSelTile = 256 * kSelItems;
__global__ void __launch_bounds__(256) select_onepass_kernel(const uint8_t *__restrict__ f,
                                                             int64_t n, int32_t *__restrict__ out,
                                                             uint32_t *__restrict__ count,
                                                             uint32_t *__restrict__ status,
                                                             uint32_t *__restrict__ ticket) {
  __shared__ uint32_t s_bid, s_excl, s_w[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_bid = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t i0 = bid * kSelTile + (int64_t)t * kSelItems;
  uint32_t bits = 0;
  if (i0 + kSelItems <= n && (reinterpret_cast<uintptr_t>(f + i0) & 7) == 0) {
    const uint64_t v = *reinterpret_cast<const uint64_t *>(f + i0);
#pragma unroll
    for (int k = 0; k < kSelItems; ++k) bits |= ((v >> (8 * k)) & 0xffu) ? (1u << k) : 0u;
  } else {
#pragma unroll
    for (int k = 0; k < kSelItems; ++k)
      if (i0 + k < n && f[i0 + k]) bits |= 1u << k;
  }
  const uint32_t c = __popc(bits);
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    // CTA total and per-warp bases, then the look-back: 32 predecessors per
    // step, one per lane, consumed up to the nearest inclusive prefix
    const uint32_t x = lane < 8 ? s_w[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < 8) s_w[lane] = xi - x;
    const uint32_t agg = __shfl_sync(0xffffffffu, xi, 7);
    uint32_t *my = status + bid;
    if (lane == 0) st_relaxed_u32(my, (bid == 0 ? kOsPre : kOsAgg) | agg);
    uint32_t excl = 0;
    if (bid > 0) {
      int64_t p = bid - 1;
      while (true) {
        const int64_t q = p - lane;
        const uint32_t w = q >= 0 ? ld_relaxed_u32(status + q) : kOsPre;  // before tile 0: prefix 0
        const unsigned pre = __ballot_sync(0xffffffffu, (w & kOsPre) != 0u);
        const unsigned zero = __ballot_sync(0xffffffffu, w == 0u);
        const int lim = pre ? __ffs(pre) - 1 : 31;
        const unsigned need = lim == 31 ? 0xffffffffu : ((1u << (lim + 1)) - 1u);
        if (zero & need) continue;  // a predecessor has not published: re-read
        uint32_t v = lane <= lim ? (w & kOsMask) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pre) break;
        p -= 32;
      }
      if (lane == 0) st_relaxed_u32(my, kOsPre | (excl + agg));
    }
    if (lane == 0) {
      s_excl = excl;
      if ((bid + 1) * kSelTile >= n) *count = excl + agg;
    }
  }
  __syncthreads();
  uint32_t pos = s_excl + s_w[warp] + inc - c;
#pragma unroll
  for (int k = 0; k < kSelItems; ++k)
    if (bits & (1u << k)) out[pos++] = (int32_t)(i0 + k);
}

struct SortWs {
  void *alt_keys;
  uint32_t *alt_vals;
  uint32_t *gh;       // [16][256] global digit histograms
  uint32_t *status;   // [nb][256] look-back words, per pass
  uint32_t *counter;  // [16] tile-index counters
  unsigned long long *or_and;
};

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

static int64_t os_tiles(int64_t n) {
  const int64_t t = (int64_t)kOsBlock * os_items(n);
  return std::max<int64_t>((n + t - 1) / t, 1);
}

static size_t sort_ws_bytes(int64_t n) {
  return align256(sizeof(uint64_t) * n) + align256(sizeof(uint32_t) * n) +
         align256(sizeof(uint32_t) * 16 * 256) + align256(sizeof(uint32_t) * 256 * os_tiles(n)) +
         align256(sizeof(uint32_t) * 16) + 256;
}

static SortWs carve_sort_ws(void *ws, int64_t n) {
  char *p = static_cast<char *>(ws);
  SortWs w;
  w.alt_keys = p;
  p += align256(sizeof(uint64_t) * n);
  w.alt_vals = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  w.gh = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * 16 * 256);
  w.status = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * 256 * os_tiles(n));
  w.counter = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * 16);
  w.or_and = reinterpret_cast<unsigned long long *>(p);
  return w;
}

template <typename K>
static int sort_pairs(const K *kin, const uint32_t *vin, K *kout, uint32_t *vout, int64_t n,
                      int begin_bit, int end_bit, int flags, void *ws, size_t ws_bytes,
                      cudaStream_t st) {
  VSX_REQUIRE(n >= 0 && n < (int64_t)1 << 30, "sort: bad n %lld", (long long)n);
  VSX_REQUIRE(begin_bit >= 0 && end_bit <= (int)(8 * sizeof(K)) && begin_bit <= end_bit,
              "sort: bad bit range");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(ws_bytes >= sort_ws_bytes(n), "sort: workspace %zu < %zu", ws_bytes,
              sort_ws_bytes(n));
  SortWs w = carve_sort_ws(ws, n);
  const int items = os_items(n);
  const int smem = (int)(2 * (sizeof(K) + sizeof(uint32_t)) * kOsBlock * items);
  {
    // the opt-in is a per-device attribute: once per device this process uses
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    VSX_CUDA_TRY(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done.load() & bit)) {
      VSX_CUDA_TRY(cudaFuncSetAttribute(os_pass_kernel<uint64_t, kOsItems>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(24 * kOsTile)));
      VSX_CUDA_TRY(cudaFuncSetAttribute(os_pass_kernel<uint32_t, kOsItems>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(16 * kOsTile)));
      done.fetch_or(bit);
    }
  }
  unsigned long long varying = ~0ull;
  if (flags & VSX_SORT_SKIP_CONSTANT) {
    // Which digit bytes actually vary? (one tiny D2H read)
    rs_init_or_and<<<1, 1, 0, st>>>(w.or_and);
    rs_minmax_kernel<K><<<std::min(grid_for(n, 256), 1184), 256, 0, st>>>(kin, n, w.or_and);
    VSX_LAUNCH_CHECK("rs_minmax");
    unsigned long long oa[2];
    VSX_CUDA_TRY(cudaMemcpyAsync(oa, w.or_and, sizeof(oa), cudaMemcpyDeviceToHost, st));
    VSX_CUDA_TRY(cudaStreamSynchronize(st));
    varying = oa[0] ^ oa[1];
  }
  int shifts[16];
  int np = 0;
  for (int sh = begin_bit - (begin_bit % 8); sh < end_bit; sh += 8) {
    unsigned long long m = (0xFFull << sh);
    if (varying & m) shifts[np++] = sh;
  }
  if (np == 0) {
    if (kout != kin) VSX_CUDA_TRY(cudaMemcpyAsync(kout, kin, sizeof(K) * n, cudaMemcpyDeviceToDevice, st));
    if (vout != vin) VSX_CUDA_TRY(cudaMemcpyAsync(vout, vin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
    return VSX_OK;
  }
  const int64_t nb = os_tiles(n);
  K *alt_k = static_cast<K *>(w.alt_keys);
  const K *src_k = kin;
  const uint32_t *src_v = vin;
  OsShifts sh{};
  sh.np = np;
  for (int p = 0; p < np; ++p) sh.s[p] = shifts[p];
  VSX_CUDA_TRY(cudaMemsetAsync(w.counter, 0, sizeof(uint32_t) * 16, st));
  if (!(flags & VSX_SORT_HIST_IN_WS)) {
    VSX_CUDA_TRY(cudaMemsetAsync(w.gh, 0, sizeof(uint32_t) * 16 * 256, st));
    os_hist_kernel<K><<<(unsigned)std::min<int64_t>(grid_for(n, 256), 8 * 148), 256, 0, st>>>(
        kin, n, sh, w.gh);
    VSX_LAUNCH_CHECK("os_hist");
  } else {
    VSX_REQUIRE(!(flags & VSX_SORT_SKIP_CONSTANT), "sort: HIST_IN_WS excludes SKIP_CONSTANT");
  }
  for (int p = 0; p < np; ++p) {
    const bool to_out = ((np - 1 - p) % 2) == 0;
    K *dk = to_out ? kout : alt_k;
    uint32_t *dv = to_out ? vout : w.alt_vals;
    VSX_CUDA_TRY(cudaMemsetAsync(w.status, 0, sizeof(uint32_t) * 256 * nb, st));
    if (items == kOsItems)
      os_pass_kernel<K, kOsItems><<<(unsigned)nb, kOsBlock, smem, st>>>(
          src_k, src_v, dk, dv, n, shifts[p], w.gh + 256 * p, w.status, w.counter + p);
    else
      os_pass_kernel<K, kOsItemsSmall><<<(unsigned)nb, kOsBlock, smem, st>>>(
          src_k, src_v, dk, dv, n, shifts[p], w.gh + 256 * p, w.status, w.counter + p);
    VSX_LAUNCH_CHECK("os_pass");
    src_k = dk;
    src_v = dv;
  }
  return VSX_OK;
}

// 32-bit monotone proxy of a positive float64 z: round toward zero to float32
// (order-preserving, never reverses two keys); ~0 marks culled entries.
// Proxies + identity values + the four 8-bit digit histograms in one
// pass (the sort then runs with VSX_SORT_HIST_IN_WS): 8 consecutive items
// per thread, vector loads / stores, run-compressed shared-memory counts as
// os_hist_kernel (the high digits come in long runs).
#ifndef VSX_ZPROXY_PER
#define VSX_ZPROXY_PER 8
#endif
__global__ void __launch_bounds__(256) z_proxy_hist_kernel(const uint64_t *__restrict__ zkey,
                                                           int64_t n, uint32_t *__restrict__ k32,
                                                           uint32_t *__restrict__ iota,
                                                           uint32_t *__restrict__ gh) {
  constexpr int kPer = VSX_ZPROXY_PER;
  __shared__ uint32_t h[4][256];
  for (int p = 0; p < 4; ++p) h[p][threadIdx.x] = 0u;
  __syncthreads();
  for (int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPer; b0 < n;
       b0 += (int64_t)gridDim.x * blockDim.x * kPer) {
    const int m = (int)min((int64_t)kPer, n - b0);
    uint32_t kk[kPer];
    if (m == kPer) {
      const ulonglong2 *z2 = reinterpret_cast<const ulonglong2 *>(zkey + b0);
#pragma unroll
      for (int j = 0; j < kPer / 2; ++j) {
        const ulonglong2 v = z2[j];
        kk[2 * j] = v.x == ~0ull ? 0xFFFFFFFFu
                                 : __float_as_uint(__double2float_rz(__longlong_as_double((long long)v.x)));
        kk[2 * j + 1] = v.y == ~0ull ? 0xFFFFFFFFu
                                     : __float_as_uint(__double2float_rz(__longlong_as_double((long long)v.y)));
      }
      uint4 *k4 = reinterpret_cast<uint4 *>(k32 + b0);
      uint4 *i4 = reinterpret_cast<uint4 *>(iota + b0);
#pragma unroll
      for (int j = 0; j < kPer / 4; ++j) {
        k4[j] = make_uint4(kk[4 * j], kk[4 * j + 1], kk[4 * j + 2], kk[4 * j + 3]);
        const uint32_t b = (uint32_t)b0 + 4 * j;
        i4[j] = make_uint4(b, b + 1, b + 2, b + 3);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        kk[j] = 0u;
        if (j < m) {
          const uint64_t k = zkey[b0 + j];
          kk[j] = k == ~0ull ? 0xFFFFFFFFu
                             : __float_as_uint(__double2float_rz(__longlong_as_double((long long)k)));
          k32[b0 + j] = kk[j];
          iota[b0 + j] = (uint32_t)(b0 + j);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      uint32_t cur = (kk[0] >> (8 * p)) & 255u, c = 1;
#pragma unroll
      for (int j = 1; j < kPer; ++j) {
        if (j < m) {
          const uint32_t d = (kk[j] >> (8 * p)) & 255u;
          if (d == cur) {
            ++c;
          } else {
            atomicAdd(&h[p][cur], c);
            cur = d;
            c = 1;
          }
        }
      }
      atomicAdd(&h[p][cur], c);
    }
  }
  __syncthreads();
  for (int p = 0; p < 4; ++p)
    if (h[p][threadIdx.x]) atomicAdd(gh + 256 * p + threadIdx.x, h[p][threadIdx.x]);
}

// Runs of equal 32-bit proxies (float32 collisions) are re-sorted by the exact
// float64 key, ties by index: the final order is the stable float64 order.
__global__ void fix_proxy_runs_kernel(const uint32_t *__restrict__ k32,
                                      const uint64_t *__restrict__ zkey,
                                      uint32_t *__restrict__ order, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (i > 0 && k32[i] == k32[i - 1])) return;
  int64_t j = i + 1;
  while (j < n && k32[j] == k32[i]) ++j;
  for (int64_t a = i + 1; a < j; ++a) {
    const uint32_t o = order[a];
    const uint64_t z = zkey[o];
    int64_t b = a - 1;
    while (b >= i && (zkey[order[b]] > z || (zkey[order[b]] == z && order[b] > o))) {
      order[b + 1] = order[b];
      --b;
    }
    order[b + 1] = o;
  }
}

// Same fix-up, exact order (z, gid): the merge of C1-received splat rows.
__global__ void fix_proxy_runs_zgid_kernel(const uint32_t *__restrict__ k32,
                                           const uint64_t *__restrict__ zkey,
                                           const int64_t *__restrict__ gid,
                                           uint32_t *__restrict__ order, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (i > 0 && k32[i] == k32[i - 1])) return;
  int64_t j = i + 1;
  while (j < n && k32[j] == k32[i]) ++j;
  for (int64_t a = i + 1; a < j; ++a) {
    const uint32_t o = order[a];
    const uint64_t z = zkey[o];
    const int64_t g = gid[o];
    int64_t b = a - 1;
    while (b >= i && (zkey[order[b]] > z || (zkey[order[b]] == z && gid[order[b]] > g))) {
      order[b + 1] = order[b];
      --b;
    }
    order[b + 1] = o;
  }
}

}  // namespace vsx

using namespace vsx;

// float32 proxies + identity values + digit histograms in one kernel, then
// the four onesweep passes on the proxies (histograms taken from the
// workspace)
static int proxy_and_sort(const uint64_t *zkey, int64_t n, uint32_t *k32, uint32_t *iota,
                          uint32_t *k32s, uint32_t *order, char *sort_ws, size_t sort_ws_bytes,
                          cudaStream_t st) {
  uint32_t *gh = reinterpret_cast<uint32_t *>(sort_ws + vsx_sort_hist_offset(n));
  VSX_CUDA_TRY(cudaMemsetAsync(gh, 0, sizeof(uint32_t) * 4 * 256, st));
  const int64_t per_block = 256 * VSX_ZPROXY_PER;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + per_block - 1) / per_block, 8 * 148);
  z_proxy_hist_kernel<<<blocks, 256, 0, st>>>(zkey, n, k32, iota, gh);
  VSX_LAUNCH_CHECK("z_proxy_hist");
  return sort_pairs<uint32_t>(k32, iota, k32s, order, n, 0, 32, VSX_SORT_HIST_IN_WS, sort_ws,
                              sort_ws_bytes, st);
}

extern "C" size_t vsx_sort_splats_ws_bytes(int64_t n) {
  return 2 * align256(sizeof(uint32_t) * n) + align256(sizeof(uint32_t) * n) + sort_ws_bytes(n);
}

extern "C" int vsx_sort_splats_z(const uint64_t *zkey, int64_t n, uint32_t *order, void *ws,
                                 size_t ws_bytes, vsx_stream s) {
  cudaStream_t st = as_stream(s);
  if (n <= 0) return VSX_OK;
  VSX_REQUIRE(ws_bytes >= vsx_sort_splats_ws_bytes(n), "sort_splats_z: workspace too small");
  char *p = static_cast<char *>(ws);
  uint32_t *k32 = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  uint32_t *k32s = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  uint32_t *iota = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  int rc = proxy_and_sort(zkey, n, k32, iota, k32s, order, p,
                          ws_bytes - 3 * align256(sizeof(uint32_t) * n), st);
  if (rc) return rc;
  fix_proxy_runs_kernel<<<grid_for(n, 256), 256, 0, st>>>(k32s, zkey, order, n);
  VSX_LAUNCH_CHECK("fix_proxy_runs");
  return VSX_OK;
}

extern "C" int vsx_sort_z_gid(const double *z, const int64_t *gid, uint32_t *order, int64_t n,
                              void *ws, size_t ws_bytes, vsx_stream s) {
  // positive float64 z: float32 round-toward-zero proxy, 4 radix passes, then
  // runs of equal proxies re-sorted by the exact (z, gid) key. No host read
  // (the 64-bit sort needed the varying-bit mask on the host).
  cudaStream_t st = as_stream(s);
  if (n <= 0) return VSX_OK;
  VSX_REQUIRE(ws_bytes >= vsx_sort_z_gid_ws_bytes(n), "sort_z_gid: workspace too small");
  const uint64_t *zkey = reinterpret_cast<const uint64_t *>(z);
  char *p = static_cast<char *>(ws);
  uint32_t *k32 = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  uint32_t *k32s = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  uint32_t *iota = reinterpret_cast<uint32_t *>(p);
  p += align256(sizeof(uint32_t) * n);
  int rc = proxy_and_sort(zkey, n, k32, iota, k32s, order, p,
                          ws_bytes - 3 * align256(sizeof(uint32_t) * n), st);
  if (rc) return rc;
  fix_proxy_runs_zgid_kernel<<<grid_for(n, 256), 256, 0, st>>>(k32s, zkey, gid, order, n);
  VSX_LAUNCH_CHECK("fix_proxy_runs_zgid");
  return VSX_OK;
}

extern "C" size_t vsx_sort_z_gid_ws_bytes(int64_t n) {
  return 3 * align256(sizeof(uint32_t) * n) + sort_ws_bytes(n);
}

extern "C" size_t vsx_scan_ws_bytes(int64_t n) { return sizeof(uint32_t) * (scan_ws_elems(n) + 1); }

extern "C" size_t vsx_sort_ws_bytes(int64_t n) {
  const size_t a = sort_ws_bytes(n);
  const size_t b = sizeof(uint32_t) * (n + 1) + vsx_scan_ws_bytes(n) + 512;  // select
  return a > b ? a : b;
}

extern "C" int vsx_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, void *ws,
                            size_t ws_bytes, vsx_stream s) {
  VSX_REQUIRE(n >= 0, "scan: negative n");
  VSX_REQUIRE(ws_bytes >= vsx_scan_ws_bytes(n), "scan: workspace too small");
  if (n == 0) {
    VSX_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint32_t), as_stream(s)));
    return VSX_OK;
  }
  return scan_impl(in, out, n, static_cast<uint32_t *>(ws), as_stream(s));
}

extern "C" int vsx_select(const uint8_t *flags, int64_t n, int32_t *out_idx,
                          uint32_t *out_count, void *ws, size_t ws_bytes, vsx_stream s) {
  cudaStream_t st = as_stream(s);
  VSX_REQUIRE(n >= 0, "select: negative n");
  if (n == 0) {
    VSX_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(uint32_t), st));
    return VSX_OK;
  }
  const int64_t nt = (n + kSelTile - 1) / kSelTile;
  const size_t need = sizeof(uint32_t) * (nt + 1);
  VSX_REQUIRE(ws_bytes >= need, "select: workspace %zu < %zu", ws_bytes, need);
  VSX_REQUIRE(n < ((int64_t)1 << 30), "select: n >= 2^30");
  uint32_t *status = static_cast<uint32_t *>(ws);
  VSX_CUDA_TRY(cudaMemsetAsync(status, 0, need, st));
  select_onepass_kernel<<<(unsigned)nt, 256, 0, st>>>(flags, n, out_idx, out_count, status,
                                                       status + nt);
  VSX_LAUNCH_CHECK("select");
  return VSX_OK;
}

extern "C" int vsx_sort_pairs_u64(const uint64_t *keys_in, const uint32_t *vals_in,
                                  uint64_t *keys_out, uint32_t *vals_out, int64_t n,
                                  int32_t begin_bit, int32_t end_bit, int32_t flags, void *ws,
                                  size_t ws_bytes, vsx_stream s) {
  return sort_pairs<uint64_t>(keys_in, vals_in, keys_out, vals_out, n, begin_bit, end_bit, flags,
                              ws, ws_bytes, as_stream(s));
}

extern "C" size_t vsx_sort_hist_offset(int64_t n) {
  return align256(sizeof(uint64_t) * n) + align256(sizeof(uint32_t) * n);
}

extern "C" int vsx_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in,
                                  uint32_t *keys_out, uint32_t *vals_out, int64_t n,
                                  int32_t begin_bit, int32_t end_bit, int32_t flags, void *ws,
                                  size_t ws_bytes, vsx_stream s) {
  return sort_pairs<uint32_t>(keys_in, vals_in, keys_out, vals_out, n, begin_bit, end_bit, flags,
                              ws, ws_bytes, as_stream(s));
}

namespace vsx {
__global__ void scatter_rows_f32_kernel(const float *__restrict__ src,
                                        const uint32_t *__restrict__ idx, int32_t n, int width,
                                        float *__restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * width) return;
  const int64_t i = e / width;
  dst[(int64_t)idx[i] * width + (e - i * width)] = src[e];
}

}  // namespace vsx

extern "C" int vsx_scatter_rows_f32(const float *src, const uint32_t *idx, int32_t n,
                                    int32_t width, float *dst, vsx_stream s) {
  VSX_REQUIRE(n >= 0 && width > 0, "scatter_rows_f32: bad arguments");
  if (n == 0) return VSX_OK;
  VSX_REQUIRE(src && idx && dst, "scatter_rows_f32: null pointer");
  scatter_rows_f32_kernel<<<grid_for((int64_t)n * width, 256), 256, 0, as_stream(s)>>>(
      src, idx, n, width, dst);
  VSX_LAUNCH_CHECK("scatter_rows_f32");
  return VSX_OK;
}
