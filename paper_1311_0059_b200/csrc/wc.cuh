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
#include "ptx.cuh"

namespace aggb {


// bloom of the frozen table for k_probe_wc: any number of 64-bit blocks (block
// from the low 32 hash bits by multiply-high; the table bucket uses bits 0-15,
// the partition the top bits, the four bit positions bits 34-53)
__device__ __forceinline__ uint32_t wc_bloom_block(uint64_t h, uint32_t nblk) { return __umulhi((uint32_t)h, nblk); }
// the block's bit pattern: bloom_bits(h) (four bits from hash bits 34-53)

__global__ void k_bloom_build_wc(GTable t, uint64_t* bloom, uint32_t nblk) {
  const uint64_t n = t.mask + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k[1] = {t.keys[i]};
    if (k[0] == EMPTY) continue;
    const uint64_t h = hash_key<1>(k, t.seed);
    atomicOr((unsigned long long*)&bloom[wc_bloom_block(h, nblk)], (unsigned long long)bloom_bits(h));
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
  unsigned int* vinfo;                    // [0] some probed value is outside int32, [1] max |v| (int64 columns)
  uint32_t* fail;                         // page list overflow / page map error
  int32_t stash;                          // pages per CTA stash refill
  // bloom positives: WC_SCAN writes CTA c's keys to pos[c * pos_stride ...] and
  // values pos_regions * pos_stride words further, their number to pos_count[c];
  // WC_RESOLVE reads them
  uint64_t* pos;
  int64_t pos_stride;
  unsigned long long* pos_count;
  int32_t pos_regions;
  int32_t pf;   // L2 prefetch of the batch tiles ahead
  int32_t pf2;  // WC_RESOLVE: load the second bucket with the first
};

template <int BLK, int R, int NS, int LINES>
struct WcLayout {
  static constexpr int T = BLK * R;
  static constexpr int RING = LINES * 8;
  static constexpr int RS = RING + 1;  // ring stride per partition (16-byte slots): one slot of skew per
                                       // partition spreads the same ring position over the banks
  static constexpr int NE = 8;
  // bytes: stages, ring, bloom + bit patterns, cnt + lb + page maps, positive index list
  static __host__ __device__ size_t stage_bytes() { return (size_t)NS * 2 * T * 8; }
  static __host__ __device__ size_t ring_bytes(int P) { return (size_t)P * RS * 16; }
  static __host__ __device__ size_t meta_bytes(int P) { return ((size_t)P * (1 + NE) * 4 + 15) & ~(size_t)15; }
  // + per-warp lists: the tile's positives (u16 stage index) and completed lines (u32)
  static __host__ __device__ size_t bytes(int P, uint32_t nblk) {
    return stage_bytes() + ring_bytes(P) + (size_t)nblk * 8 + meta_bytes(P) + (size_t)T * 2 + (size_t)T * 4;
  }
};

// k_probe_wc<MODE>: level-0 PROBE in two launches of one kernel.
//   WC_SCAN    the batch: hash -> bloom.  A positive (resident key or filter
//              false positive) is copied, coalesced, to this CTA's positive
//              region (SoA); any other record spills.
//   WC_RESOLVE the positive regions: every record probes the frozen table (its
//              first bucket loads are issued for all R records at once): a hit
//              aggregates with L2 REDs, a miss (filter false positive) spills.
// A spill claims chain position x of its partition (one shared atomic): inside
// the partition's window -> the ring (the claimer of a line's 8th slot owns the
// line), beyond -> held in registers.  Per tile: [A] classify + claims;
// barrier 1; [B] owned lines leave as 128-byte bulk copies (UBLKCP), held
// records of complete lines go straight to their page, those of the open line
// are parked for the next tile, windows move on; barrier 2 (ring, positive
// list and stage free again; the stage's next tile is issued).
constexpr int WC_SCAN = 0, WC_RESOLVE = 1;
constexpr int WC_PF = 6;  // k_probe_wc: L2 prefetch distance in tiles (rounds of the grid)
template <class PG, int BLK, int R, int NS, int LINES, int MODE>
__global__ void __launch_bounds__(BLK, 1) k_probe_wc(WcArgs a) {
  using L = WcLayout<BLK, R, NS, LINES>;
  constexpr int T = L::T, RING = L::RING, NE = L::NE;
  constexpr int SLOG = 9, S = 1 << SLOG;  // 16-byte records per 8 KB page
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int P = a.ss.nparts;
  const uint32_t nblk = MODE == WC_SCAN ? a.nblk : 0u;
  unsigned long long* stg = (unsigned long long*)smem;
  ulonglong2* ring = (ulonglong2*)(smem + L::stage_bytes());
  uint64_t* sbloom = (uint64_t*)(smem + L::stage_bytes() + L::ring_bytes(P));
  // cw[p]: the chain's claim counter (bits 0-22) and its window's first line mod 512
  // (bits 23-31): one shared atomic returns both the position and the window
  uint32_t* cw = (uint32_t*)(sbloom + nblk);
  uint32_t* ent = cw + P;
  uint16_t* plist_t = (uint16_t*)((unsigned char*)cw + L::meta_bytes(P));  // this tile's positives (stage indices)
  const uint32_t a_stg = smem_u32(smem), a_ring = smem_u32(ring), a_bloom = smem_u32(sbloom), a_cw = smem_u32(cw),
                 a_pl = smem_u32(plist_t), a_lq = a_pl + 2u * T;
  const int wid = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  // this warp's list of completed lines: entry = partition << 20 | line index (x >> 3)
  const uint32_t a_wq = a_lq + 4u * (uint32_t)(wid * R * 32);
  uint32_t nlq = 0;
  constexpr uint32_t CWM = (1u << 23) - 1;  // count bits
  constexpr int RS = L::RS;
  __shared__ __align__(8) uint64_t mbar[NS];
  __shared__ int s_tcnt[NS];
  __shared__ uint32_t s_wpos[BLK / 32];  // WC_SCAN: positives per warp of the tile
  __shared__ uint32_t s_sb, s_su, s_sc, s_nb, s_nv;
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_cnt[ST_NSTATS];
  __shared__ unsigned long long s_maxch;

  // inputs.  WC_SCAN: the batch rows [col_start, n), then FILL's deferral list.
  // WC_RESOLVE: region g holds pos_count[g] positives; tile = g * maxch + chunk.
  const int64_t n = a.n;
  int64_t col_start = 0, col_tiles = 0, nlin = 0;
  unsigned long long total = 0, maxch = 0;
  if constexpr (MODE == WC_SCAN) {
    col_start = a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
    col_tiles = (n - col_start + T - 1) / T;
    nlin = a.lcount ? (int64_t)*a.lcount : 0;
    total = (unsigned long long)(col_tiles + (nlin + T - 1) / T);
  } else {
    if (tid == 0) s_maxch = 0;
    __syncthreads();
    for (int g = tid; g < a.pos_regions; g += BLK) atomicMax(&s_maxch, (a.pos_count[g] + T - 1) / T);
    __syncthreads();
    maxch = s_maxch;
    total = maxch * (unsigned long long)a.pos_regions;
  }

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  for (int p = tid; p < P; p += BLK) cw[p] = 0;
  for (int i = tid; i < P * NE; i += BLK) ent[i] = 0xFFFFFF00u | (uint32_t)(((i & (NE - 1)) + 1) & (NE - 1));
  for (uint32_t i = tid; i < nblk; i += BLK) sbloom[i] = __ldcg((const unsigned long long*)a.bloom + i);
  if (tid == 0) {
    s_sb = s_su = s_sc = s_nb = s_nv = 0;
    for (int s = 0; s < NS; s++) mbar_init(&mbar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // producer (thread 0): tiles round-robin over the CTAs (no returning global
  // atomic on the barrier's path); WC_RESOLVE skips the empty chunks of short regions
  unsigned long long next_tile = blockIdx.x;
  auto issue = [&](int s) {
    int c = 0;
    const unsigned long long *kp = nullptr, *vp = nullptr;
    while (next_tile < total) {
      const unsigned long long tile = next_tile;
      next_tile += gridDim.x;
      if constexpr (MODE == WC_SCAN) {
        if (tile < (unsigned long long)col_tiles) {
          const int64_t b = col_start + (int64_t)tile * T;
          c = (int)(n - b < (int64_t)T ? n - b : (int64_t)T);
          kp = a.key + b;
          vp = a.val + b;
        } else {
          const int64_t b = (int64_t)(tile - col_tiles) * T;
          c = (int)(nlin - b < (int64_t)T ? nlin - b : (int64_t)T);
          kp = a.lkey + b;
          vp = a.lval + b;
        }
      } else {
        const unsigned long long g = tile / maxch;
        const int64_t b = (int64_t)(tile - g * maxch) * T;
        const int64_t np = (int64_t)a.pos_count[g];
        if (b >= np) continue;
        c = (int)(np - b < (int64_t)T ? np - b : (int64_t)T);
        kp = (const unsigned long long*)a.pos + (size_t)g * a.pos_stride + b;
        vp = kp + (size_t)a.pos_regions * a.pos_stride;
      }
      break;
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
    if constexpr (MODE == WC_SCAN) {  // the tile WC_PF rounds ahead into L2
      const unsigned long long pt = next_tile + (unsigned long long)(WC_PF - 1) * gridDim.x;
      if (a.pf && pt < (unsigned long long)col_tiles) {
        const int64_t b = col_start + (int64_t)pt * T;
        const uint32_t cb = (uint32_t)((n - b < (int64_t)T ? n - b : (int64_t)T) & ~1ll) * 8u;
        if (cb) {
          bulk_prefetch_l2(a.key + b, cb);
          bulk_prefetch_l2(a.val + b, cb);
        }
      }
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

  uint32_t opend = 0, opark = 0, lf = 0;
  uint32_t xs[R];
  int ps[R];
  uint64_t hk[R], hv[R];  // held records (beyond the window)
#pragma unroll
  for (int r = 0; r < R; r++) {
    xs[r] = 0;
    ps[r] = 0;
    hk[r] = hv[r] = 0;
  }
  uint32_t vbad = 0, vabs = 0;  // value range of the probed records (compact children)
  uint32_t c_rec = 0, c_sp = 0, c_hit = 0;
  unsigned long long pcur = 0;  // WC_SCAN: positives written to this CTA's region
  uint32_t nb_pending = 0;      // thread 0: next stash base in flight
  bool nb_busy = false;

  auto spill = [&](uint64_t k, uint64_t v, int p, int q) {
    c_sp++;
    const uint32_t old = atoms_add(a_cw + 4u * (uint32_t)p, 1u);
    const uint32_t x = old & CWM;
    if (__builtin_expect((x & (S - 1)) == 0, 0)) alloc_page(p, x >> SLOG);
    xs[q] = x;
    ps[q] = p;
    if (__builtin_expect((((x >> 3) - (old >> 23)) & 511u) < (uint32_t)LINES, 1)) {
      sts128(a_ring + 16u * ((uint32_t)p * RS + (x & (RING - 1))), k, v);
      lf |= (uint32_t)((x & 7u) == 7u) << q;  // the line is complete: queued, sent after barrier 1
    } else {
      opend |= 1u << q;
      hk[q] = k;
      hv[q] = v;
    }
  };
  // (warp-uniform) a line slot q completed goes to the warp's line list
  auto queue_line = [&](int q) {
    const bool has = (lf >> q) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    if (has) sts32(a_wq + 4u * (nlq + __popc(m & lt_mask)), ((uint32_t)ps[q] << 20) | ((xs[q] >> 3) & 0xFFFFFu));
    nlq += __popc(m);
  };

  // WC_RESOLVE: the records of the tile being processed and their first two
  // buckets, loaded one iteration ahead (software pipeline: a tile's L2 bucket
  // latency hides behind the previous tile's work)
  uint64_t rk[R], rv[R], rh[R];
  ulonglong2 rb[R][4];
  int rc = 0;
  auto resolve_fetch = [&](int t) {  // wait for tile t's stage, load its records, request their buckets
    const int st = t % NS;
    mbar_wait(&mbar[st], (uint32_t)((t / NS) & 1));
    rc = s_tcnt[st];
    const uint32_t a_k = a_stg + (uint32_t)st * 2u * T * 8u, a_v = a_k + T * 8u;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int idx = r * BLK + tid;
      rk[r] = lds64(a_k + 8u * (uint32_t)idx);
      rv[r] = lds64(a_v + 8u * (uint32_t)idx);
      const uint64_t kk[1] = {rk[r]};
      rh[r] = hash_key<1>(kk, a.t.seed);
      const uint64_t b = rh[r] & a.t.bmask;
      if (idx < rc && rk[r] != EMPTY) {
        ld_bucket32(a.t.keys + b * 4, rb[r][0], rb[r][1]);
        if (a.pf2) ld_bucket32(a.t.keys + ((b + 1) & a.t.bmask) * 4, rb[r][2], rb[r][3]);
        else rb[r][2] = rb[r][3] = make_ulonglong2(0, 0);  // (not EMPTY, no key: the chain walk below decides)
      }
    }
  };
  if constexpr (MODE == WC_RESOLVE) resolve_fetch(0);

  for (int it = 0;; it++) {
    const int s = it % NS;
    int c;
    if constexpr (MODE == WC_SCAN) {
      mbar_wait(&mbar[s], (uint32_t)((it / NS) & 1));
      c = s_tcnt[s];
    } else {
      c = rc;
    }
    if (tid == 0 && a.stash && !nb_busy && !s_nv && 2 * s_su >= s_sc) {  // next stash, taken after barrier 1
      nb_pending = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
      nb_busy = true;
    }
    // ---- [A1] parked open-line records of the last tile into the ring
    if (__builtin_expect(opark != 0, 0)) {
#pragma unroll
      for (int r = 0; r < R; r++)
        if ((opark >> r) & 1u) ring[ps[r] * RS + (xs[r] & (RING - 1))] = make_ulonglong2(hk[r], hv[r]);
      opark = 0;
    }
    // ---- [A2] this tile's records
    const unsigned long long* sk = stg + (size_t)s * 2 * T;
    const unsigned long long* sv = sk + T;
    const uint32_t a_sk = a_stg + (uint32_t)s * 2u * T * 8u, a_sv = a_sk + T * 8u;
    uint64_t k3[R], v3[R], h3[R];
    bool val3[R];
#pragma unroll
    for (int r = 0; r < R; r++) {  // loads and hashes of all R records first (ILP)
      const int idx = r * BLK + tid;
      val3[r] = idx < c;
      if constexpr (MODE == WC_SCAN) {
        k3[r] = lds64(a_sk + 8u * (uint32_t)idx);
        v3[r] = lds64(a_sv + 8u * (uint32_t)idx);
        const uint64_t kk[1] = {k3[r]};
        h3[r] = hash_key<1>(kk, a.t.seed);
      } else {
        k3[r] = rk[r];
        v3[r] = rv[r];
        h3[r] = rh[r];
      }
    }
    if constexpr (MODE == WC_SCAN) {
      bool pos3[R];
#pragma unroll
      for (int r = 0; r < R; r++) {
        const uint64_t bits = bloom_bits(h3[r]);
        const uint64_t blk = lds64(a_bloom + 8u * wc_bloom_block(h3[r], nblk));
        pos3[r] = val3[r] & ((k3[r] == EMPTY) | ((blk & bits) == bits));
      }
      // positives: this warp's slice of the tile's list (R * 32 entries per warp)
      const uint32_t a_wl = a_pl + 2u * (uint32_t)(wid * R * 32);
      uint32_t wpos = 0;
#pragma unroll
      for (int r = 0; r < R; r++) {
        // value range (compact children): some |v| >= 2^31, and max |v| otherwise
        const uint32_t lo = val3[r] ? (uint32_t)v3[r] : 0u, hi = val3[r] ? (uint32_t)(v3[r] >> 32) : 0u;
        vbad |= hi ^ (uint32_t)((int)lo >> 31);
        vabs = max(vabs, (uint32_t)abs((int)lo));
        const uint32_t m = __ballot_sync(0xffffffffu, pos3[r]);
        if (pos3[r]) sts16(a_wl + 2u * (wpos + __popc(m & lt_mask)), (uint16_t)(r * BLK + tid));
        wpos += __popc(m);
        if (val3[r] & !pos3[r]) spill(k3[r], v3[r], (int)reduce32(h3[r], (uint32_t)P), r);
        queue_line(r);
      }
      if (lane == 0) s_wpos[wid] = wpos;
      c_rec += c > tid ? (uint32_t)min(R, (c - tid + BLK - 1) / BLK) : 0u;  // this thread's records of the tile
    } else {
      // probe the frozen table: all R first buckets in flight together
      {
      // the first two buckets (64 B) of every record arrived during the last
      // tile: a miss must reach an empty slot and a displaced key the next bucket
      uint64_t bb[R];
      ulonglong2 bx[R][4];
#pragma unroll
      for (int r = 0; r < R; r++) {
        bb[r] = h3[r] & a.t.bmask;
#pragma unroll
        for (int i = 0; i < 4; i++) bx[r][i] = rb[r][i];
      }
      if (c) resolve_fetch(it + 1);  // the next tile's records and buckets go in flight now
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (!val3[r]) continue;
        const uint64_t k = k3[r];
        int64_t sl = -1;
        if (k == EMPTY) {
          if (*(volatile int*)&a.t.hdr->esc) sl = (int64_t)a.t.mask + 1;
        } else {
          // the two loaded buckets, branch-free; a longer chain (rare) continues below
          const ulonglong2 x0 = bx[r][0], y0 = bx[r][1], x1 = bx[r][2], y1 = bx[r][3];
          const uint32_t hm = (uint32_t)(x0.x == k) | ((uint32_t)(x0.y == k) << 1) | ((uint32_t)(y0.x == k) << 2) |
                              ((uint32_t)(y0.y == k) << 3) | ((uint32_t)(x1.x == k) << 4) | ((uint32_t)(x1.y == k) << 5) |
                              ((uint32_t)(y1.x == k) << 6) | ((uint32_t)(y1.y == k) << 7);
          const uint32_t em = (uint32_t)(x0.x == EMPTY) | ((uint32_t)(x0.y == EMPTY) << 1) |
                              ((uint32_t)(y0.x == EMPTY) << 2) | ((uint32_t)(y0.y == EMPTY) << 3) |
                              ((uint32_t)(x1.x == EMPTY) << 4) | ((uint32_t)(x1.y == EMPTY) << 5) |
                              ((uint32_t)(y1.x == EMPTY) << 6) | ((uint32_t)(y1.y == EMPTY) << 7);
          // (a key sits before the first empty slot of its chain)
          const uint32_t known = a.pf2 ? 0xFFu : 0x0Fu;  // buckets loaded
          const uint32_t hmk = hm & known, emk = em & known;
          const uint32_t hbit = hmk & -hmk, ebit = emk & -emk;
          if (hmk && (!emk || hbit < ebit)) {
            const int i = __ffs(hmk) - 1;
            sl = (int64_t)(((bb[r] + (uint32_t)(i >> 2)) & a.t.bmask) * 4 + (uint32_t)(i & 3));
          } else if (!emk) {  // the loaded buckets are full and hold no match: walk on
            uint64_t b = (bb[r] + (a.pf2 ? 2u : 1u)) & a.t.bmask;
            for (;;) {
              ulonglong2 x, y;
              ld_bucket32(a.t.keys + b * 4, x, y);
              if (x.x == k) { sl = (int64_t)(b * 4); break; }
              if (x.y == k) { sl = (int64_t)(b * 4 + 1); break; }
              if (y.x == k) { sl = (int64_t)(b * 4 + 2); break; }
              if (y.y == k) { sl = (int64_t)(b * 4 + 3); break; }
              if ((x.x == EMPTY) | (x.y == EMPTY) | (y.x == EMPTY) | (y.y == EMPTY)) break;
              b = (b + 1) & a.t.bmask;
            }
          }
        }
        if (sl >= 0) {
          const uint64_t vv[1] = {v3[r]};
          Upd<PG>::template g<1>(a.t.states, a.t.fstride, (uint64_t)sl * a.t.sstride, 0, s_fd, ns, vv);
          c_hit++;
        } else {
          spill(k, v3[r], k == EMPTY ? 0 : (int)reduce32(h3[r], (uint32_t)P), r);
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R; r++) queue_line(r);
      }
    }
    const bool more = c != 0;
    fence_proxy_async_smem();  // ring writes before the bulk copies that read them
    __syncthreads();           // ---- barrier 1
    if (tid == 0) {
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
    // ---- [B1] the warp's completed lines: 128-byte bulk copies (TMA engine), one per lane
    bool sent = false;
    for (uint32_t i = (uint32_t)lane; i < nlq; i += 32) {
      const uint32_t e = lds32(a_wq + 4u * i);
      const int p = (int)(e >> 20);
      const uint32_t x0 = (e & 0xFFFFFu) << 3;
      const uint32_t pg = page_of(p, x0 >> SLOG);
      if (pg < 0xFFFFFFu) bulk_s2g(rec_ptr(pg, x0), &ring[p * RS + (x0 & (RING - 1))], 128u);
      sent = true;
    }
    if (sent) bulk_commit();
    nlq = 0;
    lf = 0;
    if constexpr (MODE == WC_SCAN) {
      // ---- [B2] the tile's positives to this CTA's region (SoA), coalesced: warp w
      // writes its list after the lists of warps 0 .. w-1
      constexpr int NW = BLK / 32;
      const uint32_t wc_l = lane < NW ? s_wpos[lane] : 0u;
      uint32_t before = lane < wid ? wc_l : 0u, all = wc_l;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        before += __shfl_xor_sync(0xffffffffu, before, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
      }
      const uint32_t mine = __shfl_sync(0xffffffffu, wc_l, wid);
      unsigned long long* pk = (unsigned long long*)a.pos + (size_t)blockIdx.x * a.pos_stride + pcur + before;
      unsigned long long* pv = pk + (size_t)a.pos_regions * a.pos_stride;
      const uint32_t a_wl = a_pl + 2u * (uint32_t)(wid * R * 32);
      for (uint32_t i = (uint32_t)lane; i < mine; i += 32) {
        uint16_t idx;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(idx) : "r"(a_wl + 2u * i));
        __stcg(pk + i, sk[idx]);
        __stcg(pv + i, sv[idx]);
      }
      pcur += all;
    }
    // ---- [B3] held records: complete lines straight to their page, the open line waits
    if (__builtin_expect(opend != 0, 0)) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (!((opend >> r) & 1u)) continue;
        if ((xs[r] >> 3) < ((cw[ps[r]] & CWM) >> 3)) {
          const uint32_t pg = page_of(ps[r], xs[r] >> SLOG);
          if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, xs[r]), make_ulonglong2(hk[r], hv[r]));
        } else {
          opark |= 1u << r;
        }
      }
      opend = 0;
    }
    for (int p = tid; p < P; p += BLK) {  // the windows move to the open lines
      const uint32_t cc = cw[p] & CWM;
      cw[p] = ((cc >> 3) << 23) | cc;
    }
    if (sent) bulk_wait_read0();  // the ring slots are read before barrier 2
    // ---- barrier 2: ring, positive list and stage are free again
    if (!more) {
      if (!__syncthreads_or(opark != 0)) break;
    } else {
      __syncthreads();
    }
    if (tid == 0) issue(s);  // the tile NS ahead goes into stage s (an empty tile past the last)
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // this thread's bulk copies are complete
  // ---- close: every chain's open line (all in the ring), then the page fills
  for (int p = tid; p < P; p += BLK) {
    const uint32_t cc = cw[p] & CWM;
    if (!cc) continue;
    for (uint32_t x = cc & ~7u; x < cc; x++) {
      const uint32_t pg = page_of(p, x >> SLOG);
      if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, x), ring[p * RS + (x & (RING - 1))]);
    }
    const uint32_t pg = page_of(p, (cc - 1) >> SLOG);
    if (pg < 0xFFFFFFu) a.pool.page_fill[pg] = (int32_t)(((cc - 1) & (S - 1)) + 1);
    atomicAdd(&a.part_recs[p], (unsigned long long)cc);
  }
  if (tid == 0) {
    if (MODE == WC_SCAN) a.pos_count[blockIdx.x] = pcur;
    // unused stash pages leave the set
    for (uint32_t x = min(s_su, s_sc); x < s_sc; x++) a.pool.page_set[s_sb + x] = -1;
    if (s_nv)
      for (uint32_t x = s_nb; x < min(s_nb + (uint32_t)a.stash, a.pool.capacity); x++) a.pool.page_set[x] = -1;
    if (nb_busy)
      for (uint32_t x = nb_pending; x < min(nb_pending + (uint32_t)a.stash, a.pool.capacity); x++)
        a.pool.page_set[x] = -1;
  }
  if (c_sp) atomicExch(&a.t.hdr->frozen, 1);  // the resident set is final from now on
  if (MODE == WC_SCAN) {
    vbad = __reduce_or_sync(0xffffffffu, vbad);
    vabs = __reduce_max_sync(0xffffffffu, vabs);
    if (lane == 0) {
      if (vbad) atomicOr(&a.vinfo[0], 1u);
      atomicMax(&a.vinfo[1], vabs);
    }
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
  const unsigned int* vinfo;    // [0] some value outside int32, [1] max |v| (k_probe_wc)
  int32_t P;
  int32_t table_bytes;          // dynamic shared memory for the table
  uint64_t seed;                // slot hash seed of the child level
  OutBuf out;
  uint32_t* failed;             // [P]: 1 = groups did not fit, left to the generic drain
  uint32_t* fail;               // bit 2: some partition failed (the host runs the fallback)
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
  const bool rfit = a.vinfo[0] == 0;  // every value is an int32
  const uint32_t vabs = a.vinfo[1];
  constexpr int NA = CP::na(), NSUM = CP::nsum();
  for (int p = blockIdx.x; p < a.P; p += gridDim.x) {
    const unsigned long long np = a.part_recs[p];
    if (np == 0) continue;
    // wide sums (a u32 pair with carry) only when a partition sum can leave int32
    const bool wide = (double)np * (double)vabs >= 2147483647.0;
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
        if (!CP::is_count(j))
          sw[CP::arr(j) * stride + i] =
              (CP::fd(j) & 3) == OP_MIN ? 0x7FFFFFFFu : (CP::fd(j) & 3) == OP_MAX ? 0x80000000u : 0u;
      for (int j = 0; j < (wide ? NSUM : 0); j++) sw[(NA + j) * stride + i] = 0u;
    }
    if (tid == 0) {
      s_groups = 0;
      s_fail = !rfit || a.plist_n[p] > a.plist_cap;  // (a page list that overflowed is incomplete)
      s_esc = 0;
    }
    __syncthreads();
    const uint32_t npg = min(a.plist_n[p], a.plist_cap);
    const uint32_t* pl = a.plist + (size_t)p * a.plist_cap;
    // Warp w takes pages w, w + NWARP, ...; lane l takes slots l, l + 32, ... of
    // the page, RL records per lane in flight.
    for (uint32_t q = wid; q < npg; q += NWARP) {
      if (__any_sync(0xffffffffu, *(volatile int*)&s_fail)) break;  // warp-uniform
      const uint32_t pg = pl[q];
      const int fill = a.pool.page_fill[pg];
      const ulonglong2* pb = (const ulonglong2*)page_ptr(a.pool, pg);
      for (int s0 = 0; s0 < fill; s0 += RL * 32) {
      ulonglong2 cur[RL];
#pragma unroll
      for (int r = 0; r < RL; r++) {
        const int sl = s0 + r * 32 + lane;
        cur[r] = sl < fill ? __ldcs(pb + sl) : make_ulonglong2(0, 0);
      }
#pragma unroll
      for (int r = 0; r < RL; r++) {
        int slot = -1;
        if (s0 + r * 32 + lane < fill) {
          const uint64_t k = cur[r].x;
          if (__builtin_expect(k == EMPTY, 0)) {
            slot = nslots;
            s_esc = 1;  // (idempotent; read after the barrier)
          } else {
            const uint64_t kk[1] = {k};
            const uint64_t h = hash_key<1>(kk, a.seed);
            int b = (int)__umulhi((uint32_t)h, (uint32_t)nbk);
            for (;;) {
              const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(skeys + b * 4);
              const ulonglong2 x = bp[0], y = bp[1];
              const int hit = x.x == k ? 0 : x.y == k ? 1 : y.x == k ? 2 : y.y == k ? 3 : -1;
              if (hit >= 0) {
                slot = b * 4 + hit;
                break;
              }
              const int emp = x.x == EMPTY ? 0 : x.y == EMPTY ? 1 : y.x == EMPTY ? 2 : y.y == EMPTY ? 3 : -1;
              if (emp < 0) {  // full bucket: the next one
                if (++b == nbk) b = 0;
                continue;
              }
              if (atomicAdd(&s_groups, 1) >= maxg) {
                s_fail = 1;
                break;
              }
              const int e = b * 4 + emp;
              const unsigned long long prev = atomicCAS((unsigned long long*)&skeys[e], EMPTY, k);
              if (prev == EMPTY) {
                slot = e;
                break;
              }
              atomicSub(&s_groups, 1);  // the slot went to another insert: look at the bucket again
            }
          }
        }
        __syncwarp();
        if (slot >= 0) {
          const int cb = (int)(uint32_t)cur[r].y;  // an int32 (vinfo)
          atomicAdd(&sw[slot], 1u);
          int js = 0;
#pragma unroll
          for (int j = 0; j < N; j++) {
            const uint32_t F = CP::fd(j);
            if (((F >> 4) & 3) == SRC_ONE) continue;  // COUNT: the count word
            uint32_t* w = &sw[CP::arr(j) * stride + slot];
            if ((F & 3) == OP_ADD) {
              if (wide) {  // 64-bit two's complement sum in (lo, hi) words
                const uint32_t old = atomicAdd(w, (uint32_t)cb);
                const uint32_t hi = (uint32_t)(old + (uint32_t)cb < old) + (cb < 0 ? 0xFFFFFFFFu : 0u);
                if (hi) atomicAdd(&sw[(NA + js) * stride + slot], hi);
              } else {
                atomicAdd(w, (uint32_t)cb);
              }
              js++;
            } else if ((F & 3) == OP_MIN) {
              atomicMin((int*)w, cb);
            } else {
              atomicMax((int*)w, cb);
            }
          }
        }
      }
      }
    }
    __syncthreads();
    if (s_fail) {
      if (tid == 0) {
        a.failed[p] = 1;
        atomicOr(a.fail, 4u);
      }
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
      // reserve the rows only if they fit (else the partition goes to the fallback)
      unsigned long long base = 0;
      if (acc) {
        unsigned long long old = *(volatile unsigned long long*)a.out.count;
        for (;;) {
          if (old + acc > (unsigned long long)a.out.cap) {
            base = ~0ull;
            break;
          }
          const unsigned long long prev = atomicCAS(a.out.count, old, old + acc);
          if (prev == old) {
            base = old;
            break;
          }
          old = prev;
        }
      }
      s_base = base;
    }
    __syncthreads();
    if (s_base == ~0ull) {
      if (tid == 0) {
        a.failed[p] = 1;
        atomicOr(a.fail, 4u);
      }
      __syncthreads();
      continue;
    }
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
          const uint32_t lo = sw[CP::arr(j) * stride + s];
          w = wide ? ((uint64_t)sw[(NA + js) * stride + s] << 32 | lo) : (uint64_t)(long long)(int)lo;
          js++;
        } else {
          w = (uint64_t)(long long)(int)sw[CP::arr(j) * stride + s];
        }
        if (j < 4) st[j] = w;
      }
      emit_group4<1>(a.sp, a.out, idx++, kk, st);
    }
    __syncthreads();
  }
}

}  // namespace aggb

namespace aggb {
// Fallback after k_child_wc: the pages of every partition a child completed
// leave the spill set, so drain (the generic recursion) sees only the
// partitions that did not fit (their pages are untouched).
__global__ void k_wc_retire(const uint32_t* plist, const uint32_t* plist_n, uint32_t cap, const uint32_t* failed,
                            int P, int32_t* page_set) {
  for (int p = blockIdx.x; p < P; p += gridDim.x) {
    if (failed[p]) continue;
    const uint32_t n = plist_n[p];
    if (n > cap) continue;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) page_set[plist[(size_t)p * cap + i]] = -1;
  }
}
}  // namespace aggb
