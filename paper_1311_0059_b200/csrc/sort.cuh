// sort.cuh — the sort path (sort_based.py:24-211): LSD radix sort of the
// records by key words, then a segmented reduction over runs of equal keys.
//
//   k_sort_append    copies pushed columns into the sort buffers and gathers
//                    256-bin histograms of every key byte on the way (decides
//                    which digit passes are needed: a byte equal in every key
//                    needs no pass)
//   k_tile_hist      per-tile digit counts for one pass   -> counts[d][tile]
//   k_scan_*         3-phase exclusive scan of the digit-major counts
//   k_scatter        stable scatter of one pass (warp match_any ranking)
//   k_heads / k_seg  segment heads -> compaction -> per-segment reduction
//                    (thread per short segment, block per long segment)
//
// Records are SoA arrays of 8-byte words (KW key words, then payload words)
// ping-ponged between two buffers.  The key order is unsigned word order,
// which is the reference's byte order (_kernels.py:121-131).
#pragma once
#include "kernels.cuh"
#include "wc2.cuh"  // CompactProg (compile-time COUNT/SUM/MIN/MAX programs)

namespace aggb {

constexpr int SORT_BLOCK = 256;
constexpr int SORT_IPT = 16;                       // items per thread
constexpr int SORT_TILE = SORT_BLOCK * SORT_IPT;   // 4096

struct SortBuf {
  uint64_t* w[MAX_STATES + 2];  // word columns (KW key words first)
  int nw;
};

__global__ void k_tile_hist(const uint64_t* key, int shift, int64_t n, uint32_t* counts /* [256][ntiles] */,
                            int64_t ntiles) {
  __shared__ unsigned int sh[256];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int64_t base = t * SORT_TILE;
    for (int j = threadIdx.x; j < SORT_TILE; j += blockDim.x) {
      int64_t i = base + j;
      if (i < n) atomicAdd(&sh[(key[i] >> shift) & 255], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) counts[(int64_t)d * ntiles + t] = sh[d];
    __syncthreads();
  }
}

// ---- 3-phase exclusive scan (u32 in, u64 out) ------------------------------

constexpr int SCAN_CHUNK = 8192;

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long x) {
  __shared__ unsigned long long sw[32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) sw[wid] = x;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; w++) t += sw[w];
  __syncthreads();
  if (threadIdx.x == 0) sw[0] = t;
  __syncthreads();
  t = sw[0];
  __syncthreads();
  return t;
}

__global__ void k_scan_reduce(const uint32_t* in, int64_t n, unsigned long long* bsum) {
  int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
  unsigned long long s = 0;
  for (int j = threadIdx.x; j < SCAN_CHUNK; j += blockDim.x)
    if (base + j < n) s += in[base + j];
  s = block_sum_u64(s);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

// single block: exclusive scan of nb block sums (in place), total at [nb]
__global__ void k_scan_top(unsigned long long* bsum, int64_t nb) {
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    unsigned long long x = i < nb ? bsum[i] : 0;
    // block inclusive scan
    __shared__ unsigned long long sw[33];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) sw[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long acc = 0;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; w++) {
        unsigned long long t = sw[w];
        sw[w] = acc;
        acc += t;
      }
      sw[32] = acc;
    }
    __syncthreads();
    unsigned long long excl = carry + sw[wid] + v - x;
    if (i < nb) bsum[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += sw[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void k_scan_down(const uint32_t* in, int64_t n, const unsigned long long* bsum, unsigned long long* out) {
  int64_t base = (int64_t)blockIdx.x * SCAN_CHUNK;
  __shared__ unsigned long long carry;
  __shared__ unsigned long long sw[33];
  if (threadIdx.x == 0) carry = bsum[blockIdx.x];
  __syncthreads();
  for (int j0 = 0; j0 < SCAN_CHUNK; j0 += blockDim.x) {
    int64_t i = base + j0 + threadIdx.x;
    unsigned long long x = i < n ? in[i] : 0;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) sw[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long acc = 0;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; w++) {
        unsigned long long t = sw[w];
        sw[w] = acc;
        acc += t;
      }
      sw[32] = acc;
    }
    __syncthreads();
    if (i < n) out[i] = carry + sw[wid] + v - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += sw[32];
    __syncthreads();
  }
}

// ---- stable scatter of one digit pass --------------------------------------
// Thread t of a tile holds items t*IPT .. t*IPT+IPT-1 (consecutive), so the
// tile order is thread-major and ranks are computed in that order: per item
// slot j, warps rank their lanes' digits with match_any, and a running SMEM
// counter per digit carries the order across (slot, warp) steps.

__global__ void __launch_bounds__(SORT_BLOCK) k_scatter(SortBuf src, SortBuf dst, int key_word, int shift, int64_t n,
                                                        const unsigned long long* offs /* [256][ntiles] excl */,
                                                        int64_t ntiles) {
  __shared__ unsigned int run[256];          // running count per digit within the tile
  __shared__ unsigned int wcnt[SORT_BLOCK / 32][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = SORT_BLOCK / 32;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) run[i] = 0;
    __syncthreads();
    const int64_t base = t * SORT_TILE;
    // items of this thread: base + threadIdx.x * IPT + j; ranks in (thread, j) order require
    // ordering by thread first, so process slot by slot but count a thread's earlier slots:
    // instead use the layout index = base + j * SORT_BLOCK + threadIdx.x (slot-major order).
    for (int j = 0; j < SORT_IPT; j++) {
      const int64_t i = base + (int64_t)j * SORT_BLOCK + threadIdx.x;
      const bool live = i < n;
      uint64_t kw = live ? src.w[key_word][i] : 0;
      int d = live ? (int)((kw >> shift) & 255) : 256;
      unsigned peers = __match_any_sync(0xffffffffu, d);
      unsigned lower = peers & ((1u << lane) - 1);
      int rank_in_warp = __popc(lower);
      int leader = __ffs(peers) - 1;
      for (int q = threadIdx.x; q < nwarps * 256; q += blockDim.x) (&wcnt[0][0])[q] = 0;
      __syncthreads();
      if (live && lane == leader) wcnt[wid][d] = __popc(peers);
      __syncthreads();
      // exclusive prefix over warps per digit, plus the running count
      for (int dd = threadIdx.x; dd < 256; dd += blockDim.x) {
        unsigned acc = run[dd];
        for (int w = 0; w < nwarps; w++) {
          unsigned c = wcnt[w][dd];
          wcnt[w][dd] = acc;
          acc += c;
        }
        run[dd] = acc;
      }
      __syncthreads();
      if (live) {
        unsigned long long pos = offs[(int64_t)d * ntiles + t] + wcnt[wid][d] + rank_in_warp;
        for (int w = 0; w < src.nw; w++) dst.w[w][pos] = (w == key_word) ? kw : src.w[w][i];
      }
      __syncthreads();
    }
  }
}

// ---- tile-local radix rank + SMEM reorder (two-word records) -----------------
// Records of two 8-byte words (key word + one payload word: the C4 shape).  Warp
// w owns tile items [512 w, 512 w + 512), slot j its items 512 w + 32 j + lane,
// so (warp, slot, lane) order is index order and the ranks are stable:
//   1. per slot, match_any ranks the lanes of each digit; a per-warp SMEM
//      counter carries the digit's running count across slots (no block barrier);
//   2. per digit, an exclusive prefix over warps and a scan over digits give
//      every record its tile-local rank;
//   3. records are reordered in SMEM by rank, then written out in rank order:
//      consecutive threads write consecutive records of a digit run to
//      consecutive addresses (coalesced), instead of one scattered write each.
constexpr int S2_BLOCK = 512, S2_IPT = SORT_TILE / S2_BLOCK, S2_WARPS = S2_BLOCK / 32;

__global__ void __launch_bounds__(S2_BLOCK, 2) k_scatter2(SortBuf src, SortBuf dst, int key_word, int shift, int64_t n,
                                                       const unsigned long long* offs /* [256][ntiles] excl */,
                                                       int64_t ntiles) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* sk = (uint64_t*)smem;               // SORT_TILE key words (rank order)
  uint64_t* sv = sk + SORT_TILE;                // SORT_TILE payload words
  __shared__ uint32_t wcnt[S2_WARPS][256];      // per-warp digit counts -> per-warp exclusive bases
  __shared__ uint32_t dbase[256];               // tile-local exclusive base of each digit
  __shared__ unsigned long long goff[256];      // global base of each digit for this tile
  __shared__ uint32_t wsum[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int other = 1 - key_word;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
#pragma unroll
    for (int q = lane; q < 256; q += 32) wcnt[wid][q] = 0;
    __syncwarp();
    const int64_t base = t * SORT_TILE + (int64_t)wid * (S2_IPT * 32);
    uint64_t kk[S2_IPT], vv[S2_IPT];
    uint32_t rk[S2_IPT];
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      const int64_t i = base + j * 32 + lane;
      const bool live = i < n;
      kk[j] = live ? src.w[key_word][i] : 0ull;
      vv[j] = live ? src.w[other][i] : 0ull;
    }
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      const bool live = base + j * 32 + lane < n;
      const int d = live ? (int)((kk[j] >> shift) & 255) : 256 + lane;  // dead lanes: unique, not counted
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const unsigned run = live ? wcnt[wid][d] : 0u;
      rk[j] = run + __popc(peers & ((1u << lane) - 1u));
      __syncwarp();
      if (live && lane == __ffs(peers) - 1) wcnt[wid][d] = run + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // per digit (threads 0..255): exclusive prefix over warps; digit totals -> scan over digits
    const int d0 = threadIdx.x;
    uint32_t acc = 0, x = 0;
    if (d0 < 256) {
#pragma unroll
      for (int w = 0; w < S2_WARPS; w++) {
        const uint32_t c = wcnt[w][d0];
        wcnt[w][d0] = acc;
        acc += c;
      }
      x = acc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      goff[d0] = offs[(int64_t)d0 * ntiles + t];
    }
    __syncthreads();
    if (d0 < 256) {
      uint32_t pre = 0;
      for (int w = 0; w < wid; w++) pre += wsum[w];
      dbase[d0] = pre + x - acc;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      if (base + j * 32 + lane >= n) continue;
      const int d = (int)((kk[j] >> shift) & 255);
      const uint32_t r = dbase[d] + wcnt[wid][d] + rk[j];
      sk[r] = kk[j];
      sv[r] = vv[j];
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)SORT_TILE, n - t * SORT_TILE);
    for (int q = threadIdx.x; q < cnt; q += S2_BLOCK) {
      const uint64_t k = sk[q];
      const int d = (int)((k >> shift) & 255);
      const unsigned long long pos = goff[d] + (q - dbase[d]);
      dst.w[key_word][pos] = k;
      dst.w[other][pos] = sv[q];
    }
    __syncthreads();
  }
}

// ---- one-sweep digit pass (two-word records) ----------------------------------
// The same tile-local ranking and shared-memory reorder as k_scatter2, but the
// tile's global digit offsets come from a chained scan with decoupled look-back
// (Merrill & Garland's single-pass scan, as in onesweep radix sort) instead of a
// per-tile histogram kernel and a 3-phase scan per pass: tiles take tickets in
// order; a tile publishes its 256 digit counts (flag AGG), sums its
// predecessors' statuses backwards until one carries an inclusive prefix (flag
// INCL) and publishes its own inclusive prefix.  The global base of every digit
// comes from the byte histograms k_sort_append gathered.  Status words are 32
// bits (2 flag bits + 30 count bits: n < 2^30 records).
constexpr uint32_t OS_AGG = 1u << 30, OS_INCL = 2u << 30, OS_MASK = (1u << 30) - 1u;

__global__ void __launch_bounds__(S2_BLOCK, 2) k_onesweep2(SortBuf src, SortBuf dst, int key_word, int shift, int64_t n,
                                                        const unsigned long long* gbase /* [256] exclusive */,
                                                        uint32_t* status /* [ntiles][256], zeroed */,
                                                        unsigned long long* ticket, int64_t ntiles, int nowrite) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* sk = (uint64_t*)smem;               // SORT_TILE key words (rank order)
  uint64_t* sv = sk + SORT_TILE;                // SORT_TILE payload words
  __shared__ uint32_t wcnt[S2_WARPS][256];      // per-warp digit counts -> per-warp exclusive bases
  __shared__ uint32_t dbase[256];               // tile-local exclusive base of each digit
  __shared__ unsigned long long goff[256];      // global base of each digit for this tile
  __shared__ uint32_t wsum[8];
  __shared__ long long s_tile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int other = 1 - key_word;
  // One tile per CTA, in ticket order (a tile only ever waits for lower tickets, and
  // those CTAs are running).  The ticket is a returning global atomic (~1 us): with a
  // persistent loop all 512 threads waited for it at the top of every tile (30% of the
  // stall samples), and taking it a tile ahead stalls every later tile's look-back for
  // a whole tile; here the other resident CTA of the SM covers it.
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(ticket, 1ull);
#pragma unroll
  for (int q = lane; q < 256; q += 32) wcnt[wid][q] = 0;
  __syncthreads();
  {
    const int64_t t = s_tile;
    if (t >= ntiles) return;
    const int64_t base = t * SORT_TILE + (int64_t)wid * (S2_IPT * 32);
    uint64_t kk[S2_IPT], vv[S2_IPT];
    uint32_t rk[S2_IPT];
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      const int64_t i = base + j * 32 + lane;
      const bool live = i < n;
      kk[j] = live ? __ldcs(src.w[key_word] + i) : 0ull;
      vv[j] = live ? __ldcs(src.w[other] + i) : 0ull;
    }
    // ranks: lanes of equal digit are ranked by match_any; the group's leader adds the
    // group to the warp's digit counter with one returning shared atomic (same-address
    // atomics of a warp apply in program order, so the slots' atomics are independent
    // instructions: no read-modify-write chain through the counters between slots)
    uint32_t old[S2_IPT], low[S2_IPT];
    int ldr[S2_IPT];
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      const bool live = base + j * 32 + lane < n;
      const int d = live ? (int)((kk[j] >> shift) & 255) : 256 + lane;  // dead lanes: unique, not counted
      // lanes with the same digit: eight ballots (one per digit bit) instead of MATCH.ANY,
      // whose result the warp waited for (17% of the kernel's stall samples)
      unsigned peers = __ballot_sync(0xffffffffu, live);
      if (!live) peers = 1u << lane;
#pragma unroll
      for (int b = 0; b < 8; b++) {
        const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1);
        peers &= ((d >> b) & 1) ? bal : ~bal;
      }
      ldr[j] = __ffs(peers) - 1;
      low[j] = __popc(peers & ((1u << lane) - 1u));
      old[j] = 0;
      if (live && lane == ldr[j]) old[j] = atomicAdd(&wcnt[wid][d], (uint32_t)__popc(peers));
    }
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) rk[j] = __shfl_sync(0xffffffffu, old[j], ldr[j]) + low[j];
    __syncthreads();
    // per digit (threads 0..255): exclusive prefix over warps; digit totals -> scan over digits
    const int d0 = threadIdx.x;
    uint32_t acc = 0, x = 0;
    if (d0 < 256) {
#pragma unroll
      for (int w = 0; w < S2_WARPS; w++) {
        const uint32_t c = wcnt[w][d0];
        wcnt[w][d0] = acc;
        acc += c;
      }
      volatile uint32_t* st = status + (size_t)t * 256 + d0;
      *st = OS_AGG | acc;
      x = acc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
    }
    // Decoupled look-back, S2_WARPS predecessors per step: warp w fetches all 256
    // statuses of tile t - 1 - w - 16 step (one round trip to L2 for the whole step;
    // a digit thread walking its predecessors one load at a time cost a round trip
    // per tile looked at: a third of the kernel's stall samples), the digit threads
    // then add up their columns in shared memory until one holds an inclusive prefix.
    uint32_t excl = 0;
    bool fin = d0 >= 256;
    uint32_t* lb = (uint32_t*)sk;  // [S2_WARPS][256] (the reorder buffer is not in use yet)
    for (int64_t first = t - 1;; first -= S2_WARPS) {
      const int64_t tt = first - wid;
      uint32_t v[8];
      if (tt >= 0) {
        volatile const uint32_t* ps = status + (size_t)tt * 256 + lane;
        bool ready;
        do {
          ready = true;
#pragma unroll
          for (int q = 0; q < 8; q++) {
            v[q] = ps[q * 32];
            ready &= (v[q] >> 30) != 0;
          }
        } while (!__all_sync(0xffffffffu, ready));
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = OS_INCL;  // before the first tile: inclusive prefix 0
      }
#pragma unroll
      for (int q = 0; q < 8; q++) lb[wid * 256 + q * 32 + lane] = v[q];
      __syncthreads();
      if (!fin) {
#pragma unroll 4
        for (int w = 0; w < S2_WARPS; w++) {
          const uint32_t u = lb[w * 256 + d0];
          excl += u & OS_MASK;
          if ((u >> 30) == 2) {
            fin = true;
            break;
          }
        }
      }
      if (__syncthreads_and(fin)) break;
    }
    if (d0 < 256) {
      *(volatile uint32_t*)(status + (size_t)t * 256 + d0) = OS_INCL | (excl + acc);
      goff[d0] = gbase[d0] + excl;
    }
    __syncthreads();
    if (d0 < 256) {
      uint32_t pre = 0;
      for (int w = 0; w < wid; w++) pre += wsum[w];
      dbase[d0] = pre + x - acc;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < S2_IPT; j++) {
      if (base + j * 32 + lane >= n) continue;
      const int d = (int)((kk[j] >> shift) & 255);
      const uint32_t r = dbase[d] + wcnt[wid][d] + rk[j];
      sk[r] = kk[j];
      sv[r] = vv[j];
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)SORT_TILE, n - t * SORT_TILE);
    for (int q = threadIdx.x; q < cnt; q += S2_BLOCK) {
      const uint64_t k = sk[q];
      const int d = (int)((k >> shift) & 255);
      const unsigned long long pos = goff[d] + (q - dbase[d]);
      if (nowrite) continue;  // (experiment)
      dst.w[key_word][pos] = k;
      dst.w[other][pos] = sv[q];
    }
    __syncthreads();
  }
}

// ---- segmented reduction ----------------------------------------------------

template <int KW>
__global__ void k_head_count(const SortBuf s, int64_t n, uint32_t* tile_heads, int64_t ntiles) {
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    unsigned c = 0;
    for (int j = threadIdx.x; j < SORT_TILE; j += blockDim.x) {
      int64_t i = t * SORT_TILE + j;
      if (i >= n) continue;
      bool head = (i == 0);
      if (!head)
        for (int w = 0; w < KW; w++) head = head || (s.w[w][i] != s.w[w][i - 1]);
      c += head;
    }
    unsigned long long tot = block_sum_u64(c);
    if (threadIdx.x == 0) tile_heads[t] = (uint32_t)tot;
  }
}

template <int KW>
__global__ void k_head_compact(const SortBuf s, int64_t n, const unsigned long long* tile_off, int64_t ntiles,
                               int64_t* heads) {
  __shared__ unsigned long long sbase;
  __shared__ unsigned int wsum[SORT_BLOCK / 32 + 1];
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0) sbase = tile_off[t];
    __syncthreads();
    for (int j0 = 0; j0 < SORT_TILE; j0 += blockDim.x) {
      int64_t i = t * SORT_TILE + j0 + threadIdx.x;
      bool head = false;
      if (i < n) {
        head = (i == 0);
        if (!head)
          for (int w = 0; w < KW; w++) head = head || (s.w[w][i] != s.w[w][i - 1]);
      }
      unsigned m = __ballot_sync(0xffffffffu, head);
      int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      if (lane == 0) wsum[wid] = __popc(m);
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int w = 0; w < SORT_BLOCK / 32; w++) {
          unsigned c = wsum[w];
          wsum[w] = acc;
          acc += c;
        }
        wsum[SORT_BLOCK / 32] = acc;
      }
      __syncthreads();
      if (head) heads[sbase + wsum[wid] + __popc(m & ((1u << lane) - 1))] = i;
      __syncthreads();
      if (threadIdx.x == 0) sbase += wsum[SORT_BLOCK / 32];
      __syncthreads();
    }
  }
}

constexpr int64_t SEG_SHORT = 256;

// contribution of sorted record i (payload words from the SoA buffer)
template <int KW, int NWT>
__device__ __forceinline__ void seg_load(const SortBuf& s, int64_t i, int nw, uint64_t (&v)[NWT]) {
#pragma unroll
  for (int w = 0; w < NWT; w++) v[w] = (w < nw) ? s.w[KW + w][i] : 0ull;
}

template <int KW, int NWT>
__global__ void k_seg_reduce(const SortBuf s, DevSpec sp, int kind, int64_t n, const int64_t* heads, int64_t G,
                             OutBuf o, int64_t* long_list, unsigned long long* nlong) {
  const int ns = sp.ns;
  __shared__ uint32_t s_fd[MAX_STATES];
  if (threadIdx.x < ns) s_fd[threadIdx.x] = field_desc(sp, threadIdx.x);
  __syncthreads();
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = heads[g], b = (g + 1 < G) ? heads[g + 1] : n;
    if (b - a > SEG_SHORT) {
      long_list[atomicAdd(nlong, 1ull)] = g;
      continue;
    }
    uint64_t st[MAX_STATES];
    for (int j = 0; j < ns; j++) st[j] = state_identity(sp.op[j], sp.ty[j]);
    for (int64_t i = a; i < b; i++) {
      uint64_t v[NWT];
      seg_load<KW, NWT>(s, i, s.nw - KW, v);
      for (int j = 0; j < ns; j++) {
        uint32_t fd = s_fd[j];
        st[j] = merge_word(st[j], contrib_fd<NWT>(fd, kind, j, v), fd & 3, (fd >> 2) & 3);
      }
    }
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = s.w[w][a];
    emit_group<KW>(sp, o, g, k, st);
  }
}

// block per long segment: strided partial states, then a shared reduction
template <int KW, int NWT>
__global__ void k_seg_reduce_long(const SortBuf s, DevSpec sp, int kind, int64_t n, const int64_t* heads, int64_t G,
                                  OutBuf o, const int64_t* long_list, const unsigned long long* nlong) {
  const int ns = sp.ns;
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ uint64_t part[SORT_BLOCK];
  if (threadIdx.x < ns) s_fd[threadIdx.x] = field_desc(sp, threadIdx.x);
  __syncthreads();
  for (unsigned long long q = blockIdx.x; q < *nlong; q += gridDim.x) {
    int64_t g = long_list[q];
    int64_t a = heads[g], b = (g + 1 < G) ? heads[g + 1] : n;
    uint64_t st_out[MAX_STATES];
    for (int j = 0; j < ns; j++) {
      uint32_t fd = s_fd[j];
      uint64_t acc = state_identity(fd & 3, (fd >> 2) & 3);
      for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        uint64_t v[NWT];
        seg_load<KW, NWT>(s, i, s.nw - KW, v);
        acc = merge_word(acc, contrib_fd<NWT>(fd, kind, j, v), fd & 3, (fd >> 2) & 3);
      }
      part[threadIdx.x] = acc;
      __syncthreads();
      for (int stp = blockDim.x / 2; stp; stp >>= 1) {
        if (threadIdx.x < stp) part[threadIdx.x] = merge_word(part[threadIdx.x], part[threadIdx.x + stp], fd & 3, (fd >> 2) & 3);
        __syncthreads();
      }
      st_out[j] = part[0];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      uint64_t k[KW];
#pragma unroll
      for (int w = 0; w < KW; w++) k[w] = s.w[w][a];
      emit_group<KW>(sp, o, g, k, st_out);
    }
    __syncthreads();
  }
}

// ---- fused segmented reduction (one-word keys, one int64 value, COUNT/SUM/MIN/MAX) ----
// One pass over the sorted records after the per-tile head counts are scanned:
// thread t of a tile holds 8 consecutive records in registers, finds the segment
// heads among them, and reduces every segment that STARTS in its records — a
// segment that runs past them is followed through global memory (the next
// threads' records: cache hits), up to SEG_WALK records; a longer one is listed
// for k_seg_long2 (a block per segment).  Threads inside a longer segment do
// nothing.  A head's output row is tile_off[tile] + its rank in the tile, so the
// output is in key order.  (The generic path compacts the head positions into an
// 8-byte-per-group array and gathers from it: 37 ms per 1B records on C4.)
constexpr int SEG_IPT = 8, SEG_BLOCK = SORT_TILE / SEG_IPT;  // 512 threads x 8 records
constexpr int SEG_WALK = 256;

template <class CP>
struct SegAgg {
  uint64_t cnt;
  long long sum, mn, mx;
  __device__ __forceinline__ void start(uint64_t v) {
    cnt = 1;
    sum = mn = mx = (long long)v;
  }
  __device__ __forceinline__ void add(uint64_t v) {
    cnt++;
    sum += (long long)v;
    mn = min(mn, (long long)v);
    mx = max(mx, (long long)v);
  }
  __device__ __forceinline__ void emit(const DevSpec& sp, const OutBuf& o, int64_t idx, uint64_t key) const {
    uint64_t st[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < CP::N; j++) {
      const uint32_t F = CP::fd(j);
      if (j < 4) st[j] = CP::is_count(j) ? cnt : CP::is_sum(j) ? (uint64_t)sum : (F & 3) == OP_MIN ? (uint64_t)mn : (uint64_t)mx;
    }
    const uint64_t kk[1] = {key};
    emit_group4<1>(sp, o, idx, kk, st);
  }
};

template <class CP>
__global__ void __launch_bounds__(SEG_BLOCK) k_seg_emit2(const uint64_t* __restrict__ key, const uint64_t* __restrict__ val,
                                                         int64_t n, const unsigned long long* tile_off, int64_t ntiles,
                                                         DevSpec sp, OutBuf o, long long* long_list,
                                                         unsigned long long* nlong) {
  __shared__ uint32_t wsum[SEG_BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool aligned = (((uintptr_t)key | (uintptr_t)val) & 15) == 0;  // (a word column starts at any 8-byte offset)
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t base = t * SORT_TILE + (int64_t)threadIdx.x * SEG_IPT;
    uint64_t k[SEG_IPT], v[SEG_IPT];
    const int nvalid = (int)max((int64_t)0, min((int64_t)SEG_IPT, n - base));
    if (nvalid == SEG_IPT && aligned) {
#pragma unroll
      for (int j = 0; j < SEG_IPT; j += 2) {
        const ulonglong2 a = __ldcs((const ulonglong2*)(key + base + j));
        const ulonglong2 b = __ldcs((const ulonglong2*)(val + base + j));
        k[j] = a.x;
        k[j + 1] = a.y;
        v[j] = b.x;
        v[j + 1] = b.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < SEG_IPT; j++) {
        k[j] = j < nvalid ? key[base + j] : 0ull;
        v[j] = j < nvalid ? val[base + j] : 0ull;
      }
    }
    // the record before this thread's first: the previous lane's last record
    uint64_t prev = __shfl_up_sync(0xffffffffu, k[SEG_IPT - 1], 1);
    if (lane == 0 && base > 0 && nvalid > 0) prev = key[base - 1];
    uint32_t hm = 0;
#pragma unroll
    for (int j = 0; j < SEG_IPT; j++) {
      const bool head = j < nvalid && (j == 0 ? (base == 0 || k[0] != prev) : k[j] != k[j - 1]);
      hm |= (uint32_t)head << j;
    }
    // rank of this thread's first head in the tile
    const uint32_t nh = __popc(hm);
    uint32_t x = nh;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    __syncthreads();  // (wsum of the previous tile is read)
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < wid; w++) pre += wsum[w];
    int64_t g = (int64_t)tile_off[t] + pre + x - nh;
    if (!hm) continue;
    SegAgg<CP> ag;
    bool open = false;
    uint64_t ck = 0;
    int64_t cstart = 0;
#pragma unroll
    for (int j = 0; j < SEG_IPT; j++) {
      if (j >= nvalid) break;
      if ((hm >> j) & 1u) {
        if (open) ag.emit(sp, o, g++, ck);
        open = true;
        ck = k[j];
        cstart = base + j;
        ag.start(v[j]);
      } else if (open) {
        ag.add(v[j]);
      }
    }
    // the last segment may run on past this thread's records
    int64_t i = base + nvalid;
    int steps = 0;
    while (i < n && steps < SEG_WALK && key[i] == ck) {
      ag.add(val[i]);
      i++;
      steps++;
    }
    if (i < n && steps == SEG_WALK && key[i] == ck) {  // a long segment: a block takes it from its start
      const unsigned long long at = atomicAdd(nlong, 1ull);
      long_list[2 * at] = (long long)cstart;
      long_list[2 * at + 1] = (long long)g;
    } else {
      ag.emit(sp, o, g, ck);
    }
  }
}

// block per long segment: strided accumulation while the key lasts, then a block reduction
template <class CP>
__global__ void __launch_bounds__(256) k_seg_long2(const uint64_t* __restrict__ key, const uint64_t* __restrict__ val,
                                                   int64_t n, DevSpec sp, OutBuf o, const long long* long_list,
                                                   const unsigned long long* nlong) {
  __shared__ unsigned long long s_cnt[8];
  __shared__ long long s_sum[8], s_mn[8], s_mx[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (unsigned long long q = blockIdx.x; q < *nlong; q += gridDim.x) {
    const int64_t start = long_list[2 * q], g = long_list[2 * q + 1];
    const uint64_t k0 = key[start];
    unsigned long long cnt = 0;
    long long sum = 0, mn = 0x7FFFFFFFFFFFFFFFll, mx = (long long)0x8000000000000000ull;
    for (int64_t c = start;; c += blockDim.x) {
      const int64_t i = c + threadIdx.x;
      const bool in = i < n && key[i] == k0;
      if (in) {
        const long long x = (long long)val[i];
        cnt++;
        sum += x;
        mn = min(mn, x);
        mx = max(mx, x);
      }
      if (!__syncthreads_and(in)) break;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      sum += __shfl_xor_sync(0xffffffffu, sum, d);
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, d));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    }
    if (lane == 0) {
      s_cnt[wid] = cnt;
      s_sum[wid] = sum;
      s_mn[wid] = mn;
      s_mx[wid] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      SegAgg<CP> ag;
      ag.cnt = 0;
      ag.sum = 0;
      ag.mn = 0x7FFFFFFFFFFFFFFFll;
      ag.mx = (long long)0x8000000000000000ull;
      for (int w = 0; w < (int)blockDim.x / 32; w++) {
        ag.cnt += s_cnt[w];
        ag.sum += s_sum[w];
        ag.mn = min(ag.mn, s_mn[w]);
        ag.mx = max(ag.mx, s_mx[w]);
      }
      ag.emit(sp, o, g, k0);
    }
    __syncthreads();
  }
}

// input_sorted: any key[i] < key[i-1] sets the flag (k_stream_fold order check,
// _kernels.py:655-694 -> MergeOrderError)
template <int KW>
__global__ void k_check_sorted(const SortBuf s, int64_t n, int* bad) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool lt = false, eq = true;
#pragma unroll
    for (int w = 0; w < KW; w++) {
      uint64_t x = s.w[w][i], y = s.w[w][i - 1];
      if (eq && x != y) {
        lt = x < y;
        eq = false;
      }
    }
    if (lt) atomicExch(bad, 1);
  }
}

// append a columnar batch to the sort buffer as words (keys, payload words)
template <int KW, int NWT>
__global__ void k_sort_append(ColSrc c, int nv, SortBuf s, int64_t at, unsigned long long* hist /* [16][256] */) {
  // the byte histograms are gathered here while the keys pass through registers
  // (a separate histogram pass re-read every key at finish: 4 ms per 1B records)
  __shared__ unsigned int sh[KW * 8][256];
  for (int i = threadIdx.x; i < KW * 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
    col_key<KW>(c, i, k);
#pragma unroll
    for (int w = 0; w < KW; w++) {
      s.w[w][at + i] = k[w];
#pragma unroll
      for (int b = 0; b < 8; b++) atomicAdd(&sh[w * 8 + b][(k[w] >> (8 * b)) & 255], 1u);
    }
    for (int w = 0; w < nv; w++) {
      const uint8_t* p = c.val[w] + i * c.vstride[w];
      s.w[KW + w][at + i] =
          (c.vty[w] == TY_I32) ? (uint64_t)(long long)*(const int*)p : (uint64_t)*(const long long*)p;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < KW * 8 * 256; i += blockDim.x)
    if ((&sh[0][0])[i]) atomicAdd(&hist[i], (unsigned long long)(&sh[0][0])[i]);
}

}  // namespace aggb
