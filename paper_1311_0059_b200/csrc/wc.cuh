// wc.cuh — the level-0 PROBE of pre-partitioning with bulk-copy input staging
// and shared-memory write-combining of the spill (k_probe_wc), and the
// one-wave compact child that aggregates its partitions (k_child_wc).
//
// Replaces, for one-word keys and one dense int64/f64 value column (the C1-C3
// record shape, 16-byte spill records):
//   k_pp_probe   /root/reference/pkg/src/aggbench/_kernels.py:917-962
//                (frozen table: hits aggregate in place, misses spill to
//                hash % P partitions; the bloom byte :938-942)
//   PrePartitioning stage 2 + _drain_runs
//                /root/reference/pkg/src/aggbench/operators/hybrid.py:518-552,
//                :244-277 (each spilled run re-aggregated by a child)
//
// k_probe_wc (one CTA per SM, persistent):
//   * input tiles (1024 keys + 1024 values) arrive by cp.async.bulk (the TMA
//     engine, SASS UBLKCP) into an NS-stage shared-memory ring with mbarrier
//     completion; thread 0 grabs tiles dynamically and keeps NS in flight;
//   * a record's table hash gives its bloom block (SMEM), its partition (top
//     bits) and its table bucket (low bits); bloom positives issue their
//     bucket loads at once and are resolved at the start of the NEXT tile
//     (latency hidden behind a whole tile), hits update with L2 REDs;
//   * a spilled record claims its position x in its partition's CTA-private
//     chain with one shared atomic (cnt[p]); inside the partition's window of
//     LINES 128-byte lines it is written into a shared-memory ring, and the
//     claimer of a line's 8th record queues the line; after the tile's barrier
//     warps copy whole queued lines to HBM (8 lanes x 16 B = one 128-byte
//     line per store group).  A record beyond the window (a partition that got
//     more than the window in one tile: skew) is written straight to its page
//     after the barrier when its line is complete, or parked in registers and
//     written into the ring at the start of the next tile when it belongs to
//     the chain's open line;
//   * pages (8 KB, 512 records) are CTA-private; each new page is appended to
//     its partition's device-side page list, so children need no host round
//     trip to find their input.
//
// k_child_wc (one CTA per partition, one wave): the partition's records from
// its page list into a shared-memory table of compact 32-bit states: COUNT as
// u32, integer SUM of (v - vmin) as u32 (or a u32 pair with carry when the
// partition's records x value range can pass 2^32), MIN/MAX of (v - vmin) as
// u32 (native ATOMS.MIN/MAX).  vmin/vmax come from the level-0 pass.  A
// partition whose groups do not fit is flagged and left to the generic drain
// (its pages are untouched).
#pragma once
#include "pass.cuh"
#ifndef WC_EXP
#define WC_EXP 0
#endif

namespace aggb {

// ---------------------------------------------------------------------------
// PTX: mbarrier + 1-D bulk copy global -> shared (TMA engine)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void st_v2(void* p, ulonglong2 v) {
  asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v.x), "l"(v.y) : "memory");
}

// bloom of the frozen table for k_probe_wc: any number of 64-bit blocks (block
// from the low 32 hash bits by multiply-high; the table bucket uses bits 0-15,
// the partition the top bits, the four bit positions bits 34-53)
__device__ __forceinline__ uint32_t wc_bloom_block(uint64_t h, uint32_t nblk) { return __umulhi((uint32_t)h, nblk); }
// the block's bit pattern: one of 1024 four-bit patterns, chosen by hash bits 34-43
// (k_probe_wc looks it up in an 8 KB shared table instead of building it per record)
constexpr int WC_NPAT = 1024;
__host__ __device__ __forceinline__ uint64_t wc_pattern(uint32_t i) {
  uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 29;
  return (1ull << (z & 63)) | (1ull << ((z >> 6) & 63)) | (1ull << ((z >> 12) & 63)) | (1ull << ((z >> 18) & 63));
}
__device__ __forceinline__ uint32_t wc_pat_index(uint64_t h) { return (uint32_t)(h >> 34) & (WC_NPAT - 1); }

__global__ void k_bloom_build_wc(GTable t, uint64_t* bloom, uint32_t nblk) {
  const uint64_t n = t.mask + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k[1] = {t.keys[i]};
    if (k[0] == EMPTY) continue;
    const uint64_t h = hash_key<1>(k, t.seed);
    atomicOr((unsigned long long*)&bloom[wc_bloom_block(h, nblk)], (unsigned long long)wc_pattern(wc_pat_index(h)));
  }
}

struct WcArgs {
  DevSpec sp;
  GTable t;                               // the frozen level-0 table
  const unsigned long long* key;          // dense 8-byte key column (16-byte aligned)
  const unsigned long long* val;          // dense 8-byte value column (16-byte aligned)
  int64_t n;                              // records in the columns
  const unsigned long long* start_tiles;  // FILL consumed rows [0, *start_tiles * start_T)
  int64_t start_T;
  const unsigned long long* lkey;         // FILL's deferral list (SoA), nullable
  const unsigned long long* lval;
  const unsigned long long* lcount;
  const uint64_t* bloom;                  // nblk 64-bit blocks
  uint32_t nblk;
  PagePool pool;
  SpillSet ss;                            // rw = 2, per_page = 512
  uint32_t* plist;                        // [P][plist_cap] page ids per partition
  uint32_t* plist_n;                      // [P]
  uint32_t plist_cap;
  unsigned long long* part_recs;          // [P] records spilled per partition
  unsigned long long* tile_counter;
  unsigned long long* stats;              // ST_* counters
  long long* vrange;                      // [0] min, [1] max of the spilled values (int64 columns)
  uint32_t* fail;                         // page list overflow / page map error
  int32_t stash;                          // pages per CTA stash refill
};

template <int BLK, int NS, int LINES>
struct WcLayout {
  static constexpr int T = BLK;  // records per tile: one per thread
  static constexpr int RING = LINES * 8;
  static constexpr int NE = 8;
  // bytes: stages, ring, bloom + bit patterns, cnt + lb + page maps
  static __host__ __device__ size_t stage_bytes() { return (size_t)NS * 2 * T * 8; }
  static __host__ __device__ size_t ring_bytes(int P) { return (size_t)P * RING * 16; }
  static __host__ __device__ size_t meta_bytes(int P) { return ((size_t)P * (2 + NE) * 4 + 15) & ~(size_t)15; }
  static __host__ __device__ size_t bytes(int P, uint32_t nblk) {
    return stage_bytes() + ring_bytes(P) + (size_t)(nblk + WC_NPAT) * 8 + meta_bytes(P);
  }
};

// One CTA per SM, one record per thread per tile.  Per tile:
//   [A] wait for the stage; resolve the lane's carried bloom positive (its
//       bucket arrived during the last tile): hit -> REDs, miss -> spill; then
//       the lane's new record: hash -> bloom -> positive (issue its bucket
//       loads, carry it) or spill (claim x in its partition's chain; window
//       records into the ring, others held in registers);
//   barrier 1 (stage consumed -> its next tile is issued; claims visible);
//   [B] every complete line of every window is copied out (8 lanes x 16 B per
//       line); held records of complete lines go straight to their page, those
//       of the open line are parked for the next tile; windows move on;
//   barrier 2 (the ring lines are out before the next tile writes the ring).
template <class PG, int BLK, int NS, int LINES>
__global__ void __launch_bounds__(BLK, 1) k_probe_wc(WcArgs a) {
  using L = WcLayout<BLK, NS, LINES>;
  constexpr int T = L::T, RING = L::RING, NE = L::NE;
  constexpr int SLOG = 9, S = 1 << SLOG;  // 16-byte records per 8 KB page
  constexpr int NWARP = BLK / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int P = a.ss.nparts;
  const uint32_t nblk = a.nblk;
  unsigned long long* stg = (unsigned long long*)smem;
  ulonglong2* ring = (ulonglong2*)(smem + L::stage_bytes());
  uint64_t* sbloom = (uint64_t*)(smem + L::stage_bytes() + L::ring_bytes(P));
  uint64_t* spat = sbloom + nblk;  // WC_NPAT bit patterns
  uint32_t* cnt = (uint32_t*)(spat + WC_NPAT);
  uint32_t* lb = cnt + P;
  uint32_t* ent = lb + P;
  __shared__ __align__(8) uint64_t mbar[NS];
  __shared__ int s_tcnt[NS];
  __shared__ uint32_t s_sb, s_su, s_sc, s_nb, s_nv;
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_cnt[ST_NSTATS];

  const int64_t n = a.n;
  const int64_t col_start =
      a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t nlin = a.lcount ? (int64_t)*a.lcount : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (nlin + T - 1) / T);

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  for (int p = tid; p < P; p += BLK) cnt[p] = lb[p] = 0;
  for (int i = tid; i < P * NE; i += BLK) ent[i] = 0xFFFFFF00u | (uint32_t)(((i & (NE - 1)) + 1) & (NE - 1));
  for (uint32_t i = tid; i < nblk; i += BLK) sbloom[i] = __ldcg((const unsigned long long*)a.bloom + i);
  for (int i = tid; i < WC_NPAT; i += BLK) spat[i] = wc_pattern((uint32_t)i);
  if (tid == 0) {
    s_sb = s_su = s_sc = s_nb = s_nv = 0;
    for (int s = 0; s < NS; s++) mbar_init(&mbar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // producer (thread 0): tiles round-robin over the CTAs (uniform work per tile;
  // no returning global atomic on the barrier's path)
  unsigned long long next_tile = blockIdx.x;
  auto issue = [&](int s) {
    const unsigned long long tile = next_tile;
    next_tile += gridDim.x;
    int c = 0;
    const unsigned long long *kp = nullptr, *vp = nullptr;
    if (tile < (unsigned long long)col_tiles) {
      const int64_t b = col_start + (int64_t)tile * T;
      c = (int)(n - b < (int64_t)T ? n - b : (int64_t)T);
      kp = a.key + b;
      vp = a.val + b;
    } else if (tile < total) {
      const int64_t b = (int64_t)(tile - col_tiles) * T;
      c = (int)(nlin - b < (int64_t)T ? nlin - b : (int64_t)T);
      kp = a.lkey + b;
      vp = a.lval + b;
    }
    s_tcnt[s] = c;
    unsigned long long* sk = stg + (size_t)s * 2 * T;
    unsigned long long* sv = sk + T;
    const int c2 = c & ~1;  // bulk copies move multiples of 16 bytes
    if (c & 1) {
      sk[c - 1] = kp[c - 1];
      sv[c - 1] = vp[c - 1];
    }
    if (c2) {
      mbar_arrive_tx(&mbar[s], (uint32_t)c2 * 16u);
      bulk_g2s(sk, kp, (uint32_t)c2 * 8u, &mbar[s]);
      bulk_g2s(sv, vp, (uint32_t)c2 * 8u, &mbar[s]);
    } else {
      mbar_arrive(&mbar[s]);
    }
  };
  if (tid == 0)
    for (int s = 0; s < NS; s++) issue(s);

  uint64_t* const pool = (uint64_t*)a.pool.base;
  auto page_of = [&](int p, uint32_t j) -> uint32_t {
    const uint32_t e = ent[p * NE + (j & (NE - 1))];
    if ((e & 0xFFu) != (j & 0xFFu)) {
      atomicExch(a.fail, 2u);  // cannot happen: a page is published before the barrier that precedes its use
      return 0xFFFFFFu;
    }
    return e >> 8;
  };
  auto rec_ptr = [&](uint32_t pg, uint32_t x) { return pool + (((size_t)pg << SLOG) + (x & (S - 1))) * 2; };
  auto alloc_page = [&](int p, uint32_t j) {
    const uint32_t off = atomicAdd(&s_su, 1u);
    uint32_t pg;
    if (off < s_sc) {
      pg = s_sb + off;
    } else {
      pg = atomicAdd(a.pool.next_page, 1u);
      if (pg >= a.pool.capacity) {
        atomicExch(a.pool.overflow, 1u);
        pg = 0xFFFFFFu;
      }
    }
    if (pg < 0xFFFFFFu) {
      a.pool.page_part[pg] = p;
      a.pool.page_set[pg] = a.ss.id;
      a.pool.page_fill[pg] = S;
      const uint32_t li = atomicAdd(&a.plist_n[p], 1u);
      if (li < a.plist_cap) a.plist[(size_t)p * a.plist_cap + li] = pg;
      else atomicExch(a.fail, 1u);
    }
    ent[p * NE + (j & (NE - 1))] = (pg << 8) | (j & 0xFFu);
  };

  // the lane's bloom positive in flight (bucket loads issued, resolved next tile)
  bool cf = false;
  uint64_t ck = 0, cv = 0;
  uint32_t cb = 0;
  int cp = 0;
  ulonglong2 cx = make_ulonglong2(0, 0), cy = cx;
  // records beyond their window: pending (after barrier 1) / parked (open line, next tile)
  uint32_t opend = 0, opark = 0;
  uint32_t ox[2] = {0, 0};
  int op[2] = {0, 0};
  uint64_t okk[2] = {0, 0}, ovv[2] = {0, 0};
  long long vlo = LLONG_MAX, vhi = LLONG_MIN;
  uint32_t c_hit = 0, c_rec = 0, c_sp = 0;
  uint32_t nb_pending = 0;  // thread 0: next stash base in flight
  bool nb_busy = false;

  auto spill = [&](uint64_t k, uint64_t v, int p, int q) {
    c_sp++;
    const uint32_t x = atomicAdd(&cnt[p], 1u);
    if (__builtin_expect((x & (S - 1)) == 0, 0)) alloc_page(p, x >> SLOG);
    if (__builtin_expect(x < lb[p] + RING, 1)) {
      ring[p * RING + (x & (RING - 1))] = make_ulonglong2(k, v);
    } else {
      opend |= 1u << q;
      ox[q] = x;
      op[q] = p;
      okk[q] = k;
      ovv[q] = v;
    }
  };

  for (int it = 0;; it++) {
    const int s = it % NS;
    mbar_wait(&mbar[s], (uint32_t)((it / NS) & 1));
    const int c = s_tcnt[s];
    if (tid == 0 && a.stash && !nb_busy && !s_nv && 2 * s_su >= s_sc) {  // next stash, taken after barrier 1
      nb_pending = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
      nb_busy = true;
    }
    // ---- [A1] parked open-line records of the last tile into the ring
    if (__builtin_expect(opark != 0, 0)) {
#pragma unroll
      for (int q = 0; q < 2; q++)
        if ((opark >> q) & 1u) ring[op[q] * RING + (ox[q] & (RING - 1))] = make_ulonglong2(okk[q], ovv[q]);
      opark = 0;
    }
    // ---- [A2] the carried positive
    if (cf) {
      int64_t sl = -1;
      if (ck == EMPTY) {
        if (*(volatile int*)&a.t.hdr->esc) sl = (int64_t)a.t.mask + 1;
      } else {
        uint64_t b = cb;
        ulonglong2 x = cx, y = cy;
        for (;;) {
          if (x.x == ck) { sl = (int64_t)(b * 4); break; }
          if (x.y == ck) { sl = (int64_t)(b * 4 + 1); break; }
          if (y.x == ck) { sl = (int64_t)(b * 4 + 2); break; }
          if (y.y == ck) { sl = (int64_t)(b * 4 + 3); break; }
          if ((x.x == EMPTY) | (x.y == EMPTY) | (y.x == EMPTY) | (y.y == EMPTY)) break;
          b = (b + 1) & a.t.bmask;
          const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(a.t.keys + b * 4);
          x = __ldcg(pp);
          y = __ldcg(pp + 1);
        }
      }
      if (sl >= 0) {
        const uint64_t vv[1] = {cv};
        Upd<PG>::template g<1>(a.t.states, a.t.fstride, (uint64_t)sl * a.t.sstride, 0, s_fd, ns, vv);
        c_hit++;
      } else {
        spill(ck, cv, cp, 0);
      }
      cf = false;
    }
    // ---- [A3] the lane's record of this tile
    if (tid < c) {
      const unsigned long long* sk = stg + (size_t)s * 2 * T;
      const uint64_t k = sk[tid], v = sk[T + tid];
      c_rec++;
      vlo = min(vlo, (long long)v);
      vhi = max(vhi, (long long)v);
      const uint64_t kk[1] = {k};
      const uint64_t h = hash_key<1>(kk, a.t.seed);
      const int p = k == EMPTY ? 0 : (int)reduce32(h, (uint32_t)P);
      const uint64_t bits = spat[wc_pat_index(h)];
      const bool pos = k == EMPTY || (sbloom[wc_bloom_block(h, nblk)] & bits) == bits;
      if (pos) {
        cf = true;
        ck = k;
        cv = v;
        cp = p;
        if (k != EMPTY) {
          cb = (uint32_t)(h & a.t.bmask);
          const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(a.t.keys + (uint64_t)cb * 4);
          cx = __ldcg(pp);
          cy = __ldcg(pp + 1);
        }
      } else {
        spill(k, v, p, 1);
      }
    }
    const bool more = c != 0;
    const bool pending = cf || opend != 0;
    __syncthreads();  // ---- barrier 1: claims, ring writes and page maps are visible; the stage is consumed
    if (tid == 0) {
      issue(s);  // the tile NS ahead goes into stage s (an empty tile past the last)
      if (nb_busy) {
        s_nb = nb_pending;
        s_nv = 1;
        nb_busy = false;
      }
      if (s_nv && s_su >= s_sc) {
        const bool fits = s_nb + (uint32_t)a.stash <= a.pool.capacity;
        if (!fits)
          for (uint32_t x = s_nb; x < min(s_nb + (uint32_t)a.stash, a.pool.capacity); x++) a.pool.page_set[x] = -1;
        s_sb = s_nb;
        s_sc = fits ? (uint32_t)a.stash : 0u;
        s_su = 0;
        s_nv = 0;
      }
    }
    // ---- [B1] complete lines of the windows: lane l of warp w looks at partition
    // l * NWARP + w; the warp copies its lines 4 at a time, 8 lanes (16 B each) per line
    {
      const int p = lane * NWARP + wid;
      uint32_t l0 = 0, nl = 0;
      if (p < P) {
        const uint32_t w = lb[p], ce = cnt[p];
        l0 = w >> 3;
        nl = (min(ce, w + RING) >> 3) - l0;
        lb[p] = ce & ~7u;  // the window moves to the open line (read again after barrier 2)
      }
#pragma unroll
      for (int i = 0; i < LINES; i++) {
        uint32_t m = __ballot_sync(0xffffffffu, nl > (uint32_t)i);
        while (m) {
          uint32_t mm = m;
          int src = -1;
#pragma unroll
          for (int g = 0; g < 4; g++) {  // group g = lane >> 3 takes the g-th set bit
            const int b = __ffs(mm) - 1;
            if (g == (lane >> 3)) src = b;
            if (mm) mm &= mm - 1;
          }
          m = mm;
          const int sp = __shfl_sync(0xffffffffu, p, src < 0 ? 0 : src);
          const uint32_t sl = __shfl_sync(0xffffffffu, l0, src < 0 ? 0 : src) + (uint32_t)i;
          if (src >= 0) {
            const uint32_t x = (sl << 3) | (lane & 7);
            const ulonglong2 rec = ring[sp * RING + (x & (RING - 1))];
            const uint32_t pg = page_of(sp, x >> SLOG);
            if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, x), rec);
          }
        }
      }
    }
    // ---- [B2] held records: complete lines go straight to their page, the open line waits
    if (__builtin_expect(opend != 0, 0)) {
#pragma unroll
      for (int q = 0; q < 2; q++) {
        if (!((opend >> q) & 1u)) continue;
        const uint32_t cend = cnt[op[q]];
        if ((ox[q] >> 3) < (cend >> 3)) {
          const uint32_t pg = page_of(op[q], ox[q] >> SLOG);
          if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, ox[q]), make_ulonglong2(okk[q], ovv[q]));
        } else {
          opark |= 1u << q;
        }
      }
      opend = 0;
    }
    // ---- barrier 2: the ring lines are out before the next tile writes the ring
    if (!more) {
      if (!__syncthreads_or(pending || opark != 0)) break;
    } else {
      __syncthreads();
    }
  }
  // ---- close: every chain's open line (all in the ring), then the page fills
  for (int p = tid; p < P; p += BLK) {
    const uint32_t cc = cnt[p];
    if (!cc) continue;
    for (uint32_t x = cc & ~7u; x < cc; x++) {
      const uint32_t pg = page_of(p, x >> SLOG);
      if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, x), ring[p * RING + (x & (RING - 1))]);
    }
    const uint32_t pg = page_of(p, (cc - 1) >> SLOG);
    if (pg < 0xFFFFFFu) a.pool.page_fill[pg] = (int32_t)(((cc - 1) & (S - 1)) + 1);
    atomicAdd(&a.part_recs[p], (unsigned long long)cc);
  }
  if (tid == 0) {  // unused stash pages leave the set
    for (uint32_t x = min(s_su, s_sc); x < s_sc; x++) a.pool.page_set[s_sb + x] = -1;
    if (s_nv)
      for (uint32_t x = s_nb; x < min(s_nb + (uint32_t)a.stash, a.pool.capacity); x++) a.pool.page_set[x] = -1;
    if (nb_busy)
      for (uint32_t x = nb_pending; x < min(nb_pending + (uint32_t)a.stash, a.pool.capacity); x++)
        a.pool.page_set[x] = -1;
  }
  if (c_sp) atomicExch(&a.t.hdr->frozen, 1);
  // value range of the probed records (compact child states)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    vlo = min(vlo, __shfl_xor_sync(0xffffffffu, vlo, o));
    vhi = max(vhi, __shfl_xor_sync(0xffffffffu, vhi, o));
  }
  if (lane == 0 && vlo <= vhi) {
    atomicMin(&a.vrange[0], vlo);
    atomicMax(&a.vrange[1], vhi);
  }
  uint32_t cs[3] = {c_sp, c_hit, c_rec};
  const int ids[3] = {ST_SPILLED, ST_HITS, ST_RECORDS};
#pragma unroll
  for (int q = 0; q < 3; q++) {
    uint32_t x = cs[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && x) atomicAdd(&s_cnt[ids[q]], (unsigned long long)x);
  }
  __syncthreads();
  if (tid < ST_NSTATS && s_cnt[tid]) atomicAdd(&a.stats[tid], s_cnt[tid]);
}

// ---------------------------------------------------------------------------
// k_child_wc: one CTA per spilled partition, compact 32-bit states
// ---------------------------------------------------------------------------

struct CwArgs {
  DevSpec sp;
  PagePool pool;
  const uint32_t* plist;
  const uint32_t* plist_n;
  uint32_t plist_cap;
  const unsigned long long* part_recs;
  const long long* vrange;      // [0] vmin, [1] vmax of the spilled values
  int32_t P;
  int32_t table_bytes;          // dynamic shared memory for the table
  uint64_t seed;                // slot hash seed of the child level
  OutBuf out;
  uint32_t* failed;             // [P]: 1 = groups did not fit, left to the generic drain
  unsigned long long* stats;
};

// Compact field programs: every state field an integer COUNT / SUM / MIN / MAX
// of the one value column (descriptor op | ty<<2 | srck<<4 | vty<<6 | src<<8).
template <uint32_t... F>
struct CompactProg {
  static constexpr int N = sizeof...(F);
  __host__ __device__ static constexpr uint32_t fd(int j) {
    constexpr uint32_t a[N] = {F...};
    return a[j];
  }
  __host__ __device__ static constexpr bool is_count(int j) { return ((fd(j) >> 4) & 3) == SRC_ONE; }
  __host__ __device__ static constexpr bool is_sum(int j) { return (fd(j) & 3) == OP_ADD && !is_count(j); }
  // u32 word array of field j (0 = the count word, shared by COUNT fields)
  __host__ __device__ static constexpr int arr(int j) {
    int x = 1;
    for (int i = 0; i < j; i++) x += !is_count(i);
    return is_count(j) ? 0 : x;
  }
  __host__ __device__ static constexpr int na() {
    int x = 1;
    for (int i = 0; i < N; i++) x += !is_count(i);
    return x;
  }
  __host__ __device__ static constexpr int nsum() {
    int x = 0;
    for (int i = 0; i < N; i++) x += is_sum(i);
    return x;
  }
};
using CpC1 = CompactProg<0x000, 0x010>;                 // COUNT, SUM
using CpC2 = CompactProg<0x000, 0x010, 0x011, 0x012>;   // COUNT, SUM, MIN, MAX

template <class CP, int BLK, int RL>
__global__ void __launch_bounds__(BLK, 1) k_child_wc(CwArgs a) {
  constexpr int N = CP::N;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NWARP = BLK / 32;
  __shared__ int s_groups, s_fail, s_esc;
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_wsum[NWARP];
  const long long vmin = a.vrange[0], vmax = a.vrange[1];
  const uint64_t range = (uint64_t)(vmax - vmin);
  constexpr int NA = CP::na(), NSUM = CP::nsum();
  for (int p = blockIdx.x; p < a.P; p += gridDim.x) {
    const unsigned long long np = a.part_recs[p];
    if (np == 0) continue;
    // wide sums (u32 pair with carry) only when the partition's biased sum can pass 2^32
    const bool wide = (vmax >= vmin) && (range >= (1ull << 32) || (double)np * (double)range >= 4294967295.0);
    const bool rfit = vmax < vmin || range < (1ull << 32);
    const int words = 2 + NA + (wide ? NSUM : 0);  // key (2 x u32), count, one u32 per other field (+ hi words)
    // keys in 32-byte buckets of 4 slots (one bucket = two LDS.128; the warp runs
    // the longest probe of its lanes, and buckets keep that short)
    const int nbk = ((a.table_bytes / 4 - 2) / words - 1) / 4;
    const int nslots = nbk * 4;
    const int maxg = (int)(0.85 * nslots);
    uint64_t* skeys = (uint64_t*)smem;                      // nslots + 1 (escape slot last)
    uint32_t* sw = (uint32_t*)(skeys + (nslots + 1));       // [field][slot] u32 words
    const int stride = nslots + 1;
    // word arrays: 0 = count (COUNT fields), CP::arr(j) = field j, then the hi words of wide sums
    for (int i = tid; i < stride; i += BLK) {
      skeys[i] = EMPTY;
      sw[i] = 0;
#pragma unroll
      for (int j = 0; j < N; j++)
        if (!CP::is_count(j)) sw[CP::arr(j) * stride + i] = (CP::fd(j) & 3) == OP_MIN ? 0xFFFFFFFFu : 0u;
      for (int j = 0; j < (wide ? NSUM : 0); j++) sw[(NA + j) * stride + i] = 0u;
    }
    if (tid == 0) {
      s_groups = 0;
      s_fail = !rfit;
      s_esc = 0;
    }
    __syncthreads();
    const uint32_t npg = min(a.plist_n[p], a.plist_cap);
    const uint32_t* pl = a.plist + (size_t)p * a.plist_cap;
    // warp per page, lane l takes slots l, l + 32, ... (RL records per lane in flight)
    for (uint32_t q = wid; q < npg; q += NWARP) {
      if (__any_sync(0xffffffffu, *(volatile int*)&s_fail)) break;  // warp-uniform
      const uint32_t pg = pl[q];
      const int fill = a.pool.page_fill[pg];
      const ulonglong2* pb = (const ulonglong2*)page_ptr(a.pool, pg);
      for (int s0 = 0; s0 < fill; s0 += RL * 32) {
        ulonglong2 rec[RL];
#pragma unroll
        for (int r = 0; r < RL; r++) {
          const int sl = s0 + r * 32 + lane;
          rec[r] = sl < fill ? __ldcs(pb + sl) : make_ulonglong2(0, 0);
        }
#pragma unroll
        for (int r = 0; r < RL; r++) {
          const int sl = s0 + r * 32 + lane;
          int slot = -1;
          if (sl < fill) {
            const uint64_t k = rec[r].x;
            if (k == EMPTY) {
              slot = nslots;
              if (!*(volatile int*)&s_esc) atomicExch(&s_esc, 1);
            } else {
              const uint64_t kk[1] = {k};
              const uint64_t h = hash_key<1>(kk, a.seed);
              int b = (int)__umulhi((uint32_t)h, (uint32_t)nbk);
              for (;;) {
                const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(skeys + b * 4);
                const ulonglong2 x = bp[0], y = bp[1];
                const int hit = x.x == k ? 0 : x.y == k ? 1 : y.x == k ? 2 : y.y == k ? 3 : -1;
                if (hit >= 0) { slot = b * 4 + hit; break; }
                const int emp = x.x == EMPTY ? 0 : x.y == EMPTY ? 1 : y.x == EMPTY ? 2 : y.y == EMPTY ? 3 : -1;
                if (emp < 0) {  // full bucket: the next one
                  if (++b == nbk) b = 0;
                  continue;
                }
                if (atomicAdd(&s_groups, 1) >= maxg) {
                  s_fail = 1;
                  break;
                }
                const unsigned long long prev = atomicCAS((unsigned long long*)&skeys[b * 4 + emp], EMPTY, k);
                if (prev == EMPTY) { slot = b * 4 + emp; break; }
                atomicSub(&s_groups, 1);  // the slot went to another insert: look at the bucket again
              }
            }
          }
          __syncwarp();
          if (slot >= 0) {
            const uint32_t cb = (uint32_t)((long long)rec[r].y - vmin);
            atomicAdd(&sw[slot], 1u);
            int js = 0;
#pragma unroll
            for (int j = 0; j < N; j++) {
              const uint32_t F = CP::fd(j);
              if (((F >> 4) & 3) == SRC_ONE) continue;  // COUNT: the count word
              uint32_t* w = &sw[CP::arr(j) * stride + slot];
              if ((F & 3) == OP_ADD) {
                if (wide) {
                  const uint32_t old = atomicAdd(w, cb);
                  if (old + cb < old) atomicAdd(&sw[(NA + js) * stride + slot], 1u);
                } else {
                  atomicAdd(w, cb);
                }
                js++;
              } else if ((F & 3) == OP_MIN) {
                atomicMin(w, cb);
              } else {
                atomicMax(w, cb);
              }
            }
          }
        }
      }
    }
    __syncthreads();
    if (s_fail) {
      if (tid == 0) a.failed[p] = 1;
      __syncthreads();
      continue;
    }
    // emit: block compaction, one output reservation per partition
    const int per = (stride + BLK - 1) / BLK;
    const int lo = tid * per, hi = min(stride, lo + per);
    uint32_t mine = 0;
    for (int s = lo; s < hi; s++) mine += (s == nslots) ? (s_esc != 0) : (skeys[s] != EMPTY);
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int w = 0; w < NWARP; w++) {
        const uint32_t t2 = s_wsum[w];
        s_wsum[w] = acc;
        acc += t2;
      }
      s_base = acc ? atomicAdd(a.out.count, (unsigned long long)acc) : 0ull;
    }
    __syncthreads();
    int64_t idx = (int64_t)s_base + s_wsum[wid] + (x - mine);
    for (int s = lo; s < hi; s++) {
      const bool occ = (s == nslots) ? (s_esc != 0) : (skeys[s] != EMPTY);
      if (!occ) continue;
      const uint64_t kk[1] = {s == nslots ? EMPTY : skeys[s]};
      const uint64_t cntw = sw[s];
      uint64_t st[4] = {0, 0, 0, 0};
      int js = 0;
#pragma unroll
      for (int j = 0; j < N; j++) {
        const uint32_t F = CP::fd(j);
        uint64_t w;
        if (((F >> 4) & 3) == SRC_ONE) {
          w = cntw;
        } else if ((F & 3) == OP_ADD) {
          uint64_t b = sw[CP::arr(j) * stride + s];
          if (wide) b |= (uint64_t)sw[(NA + js) * stride + s] << 32;
          w = b + cntw * (uint64_t)vmin;  // sum(v) = sum(v - vmin) + count * vmin (mod 2^64: exact)
          js++;
        } else {
          w = (uint64_t)((long long)sw[CP::arr(j) * stride + s] + vmin);
        }
        if (j < 4) st[j] = w;
      }
      emit_group4<1>(a.sp, a.out, idx++, kk, st);
    }
    __syncthreads();
  }
}

}  // namespace aggb
