// wc2.cuh — level 0 of budgeted pre-partitioning for 16-byte records (one-word
// key, one int64 value; the C1/C2 record shape) after the table froze, in two
// kernels:
//
//   k_scan_wc   one pass over the batch that only ROUTES: every record is
//               hashed and appended to the run of its hash range.  Runs are
//               written through per-run shared-memory write-combining rings as
//               whole 128-byte lines; input tiles arrive by cp.async.bulk (the
//               TMA engine, SASS UBLKCP) from a producer warp.
//   k_child2_wc one CTA per run, a compact shared-memory table (u32 states),
//               seeded with the resident keys of the run's hash range (the
//               level-0 table's keys, listed per run by k_wc2_build).  The
//               aggregates of the seeded keys are merged into the level-0 table
//               (L2 REDs, once per group) and not emitted, so resident keys are
//               emitted once, by the table flush, and their records do not count
//               as spilled; every other key of the run is a spilled group the
//               child emits.
//
// Replaces k_pp_probe (/root/reference/pkg/src/aggbench/_kernels.py:917-962:
// frozen table, hits aggregate in place, misses spill to hash % P partitions,
// bloom byte :938-942), PrePartitioning stage 2 and _drain_runs
// (/root/reference/pkg/src/aggbench/operators/hybrid.py:518-552, :244-277).
//
// Why routing only: resolving each record against the L2 table cost one bucket
// load and four REDs per hit (k_probe_wc's resolve pass: 0.71 ms for 27M filter
// positives on C2, 750 instructions per positive) and a filter in shared memory
// (64 KB, ~14 instructions per record) to keep the misses away from it.  Here
// the table sees 4 REDs per resident GROUP, the filter is gone, and its shared
// memory holds a third input stage.
#pragma once
#include "pass.cuh"
#include "ptx.cuh"
#include <type_traits>

namespace aggb {

__device__ __forceinline__ uint32_t fmix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}
// 32-bit hash of a one-word key (the high word folded in by an odd multiply); the
// routing hash and the children's slot hash are this function under different seeds
__device__ __forceinline__ uint32_t hash32(uint64_t k, uint32_t seed) {
  return fmix32((uint32_t)k ^ seed ^ ((uint32_t)(k >> 32) * 0x9E3779B1u));
}
// the routing hash: run = top bits (9 instructions; the 64-bit fmix was 16 per record)
__device__ __forceinline__ uint32_t wc2_run(uint64_t k, uint32_t seed, uint32_t NP) { return __umulhi(hash32(k, seed), NP); }

// the runs' lists of resident slots: one pass over the frozen table's key array
__global__ void k_wc2_build(GTable t, uint32_t seed, uint32_t* olist, uint32_t* olist_n, uint32_t ocap, uint32_t NP) {
  const uint64_t n = t.mask + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = t.keys[i];
    if (k == EMPTY) continue;
    const uint32_t o = wc2_run(k, seed, NP);
    const uint32_t at = atomicAdd(&olist_n[o], 1u);
    if (at < ocap) olist[(size_t)o * ocap + at] = (uint32_t)i;
  }
}

struct Wc2Args {
  GTable t;                               // the frozen level-0 table (header only)
  uint32_t seed;                          // routing hash seed
  const unsigned long long* key;          // dense 8-byte key column (16-byte aligned)
  const unsigned long long* val;          // dense 8-byte value column (16-byte aligned)
  int64_t n;                              // records in the columns
  const unsigned long long* start_tiles;  // FILL consumed rows [0, *start_tiles * start_T)
  int64_t start_T;
  const unsigned long long* lkey;         // FILL's deferral list (SoA), nullable
  const unsigned long long* lval;
  const unsigned long long* lcount;
  PagePool pool;
  int32_t set_id;                         // spill set of the runs' pages
  int32_t NP;                             // runs
  uint32_t* plist;                        // [NP][plist_cap] page ids per run
  uint32_t* plist_n;                      // [NP]
  uint32_t plist_cap;
  unsigned long long* ovf;                // pages past a run's list (skew): run << 32 | page, one list for all runs
  unsigned long long* ovf_n;
  uint32_t ovf_cap;
  uint32_t plist_blk;                     // page-list entries a CTA reserves per run at a time
  unsigned long long* part_recs;          // [NP] records per run
  unsigned long long* stats;              // ST_* counters
  unsigned int* vinfo;                    // [0] some value outside int32, [1] OR of the magnitudes, [2] OR of the keys' high words
  uint32_t* fail;                         // page list overflow / page map error
  int32_t stash;                          // pages per CTA stash refill
  int32_t nosend;                         // (experiment) lines are not written
  int32_t nohot;                          // (experiment / test) no heavy-hitter handling
  int32_t prog;                           // 1 COUNT, SUM; 2 COUNT, SUM, MIN, MAX (state fields of the level-0 table)
};

template <int BLK, int R, int NS>
struct Wc2Layout {
  static_assert(R % 2 == 0, "records are loaded in pairs");
  static constexpr int T = BLK * R;
  static constexpr int LINES = 2, RING = LINES * 8;
  static constexpr int RS = RING + 1;  // ring stride per run (16-byte slots): one slot of skew per run
                                       // spreads the same ring position over the banks
  static constexpr int NE = 8;         // page map entries per run (pages a run can open in one tile)
  static __host__ __device__ size_t stage_bytes() { return (size_t)NS * 2 * T * 8; }
  static __host__ __device__ size_t ring_bytes(int NP) { return (size_t)NP * RS * 16; }
  static __host__ __device__ size_t meta_bytes(int NP) { return ((size_t)NP * (3 + NE) * 4 + 15) & ~(size_t)15; }
  static __host__ __device__ size_t send_bytes() { return (size_t)(BLK / 32) * 32 * 16; }  // per warp: 32 lines to send
  static __host__ __device__ size_t bytes(int NP) { return stage_bytes() + ring_bytes(NP) + meta_bytes(NP) + send_bytes(); }
};

__device__ __forceinline__ void lds128(uint32_t a, uint64_t& x, uint64_t& y) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
}

// One CTA per SM, persistent.  Per tile (T = BLK * R records):
//   [A] every thread routes its R records: hash, run id, one shared
//       atomic on the run's claim word cw[run] (claim counter in bits 0-22, the
//       run's window start (line index mod 512) in bits 23-31).  A claim
//       inside the window (LINES lines from the run's open line) is written
//       into the run's ring; a claim beyond it (a burst: more than a window of
//       one run in one tile) is held.  The claimer of a page's first slot opens
//       the page (CTA-private, appended to the run's device-side page list).
//   barrier 1
//   [B] held records of lines that are complete go straight to their page;
//       those of the run's open line are parked in registers and written into
//       the ring at the start of the next tile.  One thread per run sends the
//       window lines the tile completed, one 128-byte bulk copy shared -> global
//       each, and moves the run's window to its open line.
//   barrier 2 (ring and stage free again; thread 0 issues the stage's next tile)
template <int BLK, int R, int NS>
__global__ void __launch_bounds__(BLK + 32, 1) k_scan_wc(Wc2Args a) {
  using L = Wc2Layout<BLK, R, NS>;
  constexpr int T = L::T, RING = L::RING, NE = L::NE, LINES = L::LINES, RS = L::RS;
  constexpr int SLOG = 9, S = 1 << SLOG;  // 16-byte records per 8 KB page
  constexpr uint32_t CWM = (1u << 23) - 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int NP = a.NP;
  unsigned long long* stg = (unsigned long long*)smem;
  ulonglong2* ring = (ulonglong2*)(smem + L::stage_bytes());
  uint32_t* cw = (uint32_t*)(smem + L::stage_bytes() + L::ring_bytes(NP));
  uint32_t* ent = cw + NP;
  uint32_t* lbase = ent + NP * NE;  // this CTA's block of the run's page list ...
  uint32_t* lused = lbase + NP;     // ... and the entries of it in use
  uint4* sendq = (uint4*)((unsigned char*)cw + L::meta_bytes(NP));  // per warp: (ring address, -, destination) of the lines to send
  const uint32_t a_stg = smem_u32(smem), a_ring = smem_u32(ring), a_cw = smem_u32(cw);
  __shared__ __align__(8) uint64_t mbar[NS];    // stage full (the tile's bytes have landed)
  __shared__ __align__(8) uint64_t mbar_e[NS];  // stage empty (every consumer is past barrier 2 of its tile)
  __shared__ int s_tcnt[NS];
  __shared__ uint32_t s_sb, s_su, s_sc, s_nb, s_nv, s_want, s_pdone;
  // Heavy hitters (a key holding percents of the input would make its run, and the
  // one CTA that aggregates it, the whole step: 30% of C2's records on 3 keys ran
  // 18.6 ms).  The resident ones among the sampled hot keys are not routed: their
  // records are reduced per warp into these accumulators and merged into the
  // level-0 table when the CTA ends.
  __shared__ unsigned long long s_hk[8];
  __shared__ unsigned long long s_hacc[8][4];  // count, sum, min, max
  __shared__ uint32_t s_hslot[8];
  __shared__ unsigned char s_hdir[64];         // 6 hash bits -> hot key index
  __shared__ int s_nhot;

  const int64_t n = a.n;
  const int64_t col_start = a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t nlin = a.lcount ? (int64_t)*a.lcount : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (nlin + T - 1) / T);
  // tiles of this CTA (round-robin), plus one empty tile that lets parked records into the ring
  const int ntiles = total > blockIdx.x ? (int)((total - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;

  // page-list entries are reserved per run in blocks, up front: opening a page then
  // needs no returning global atomic (a ~1 us round trip that every other warp of
  // the tile waited for at barrier 1, about four times per tile)
  // (entries left unused stay 0xFFFFFFFF; a run that needs more than its block takes
  // single entries with the atomic)
  constexpr int NT = BLK + 32;  // all threads (set-up only)
  for (int p = tid; p < NP; p += NT) {
    cw[p] = 0;
    lbase[p] = atomicAdd(&a.plist_n[p], a.plist_blk);
    lused[p] = 0;
  }
  for (int i = tid; i < NP * NE; i += NT) ent[i] = 0xFFFFFF00u | (uint32_t)(((i & (NE - 1)) + 1) & (NE - 1));
  if (tid == 0) {
    s_sb = s_su = s_sc = s_nb = s_nv = s_want = s_pdone = 0;
    for (int s = 0; s < NS; s++) {
      mbar_init(&mbar[s], 1);
      mbar_init(&mbar_e[s], 1);
    }
    mbar_fence_init();
    s_nhot = 0;
  }
  if (tid < 64) s_hdir[tid] = 0xFF;
  if (tid < 8) {
    s_hacc[tid][0] = s_hacc[tid][1] = 0;
    s_hacc[tid][2] = 0x7FFFFFFFFFFFFFFFull;
    s_hacc[tid][3] = 0x8000000000000000ull;
    s_hslot[tid] = 0xFFFFFFFFu;
  }
  __syncthreads();
  int nhot = 0;  // resident heavy hitters this CTA found in its first tile (set below, by the consumers)

  // producer (thread 0): tiles round-robin over the CTAs
  unsigned long long next_tile = blockIdx.x;
  unsigned long long n_rec = 0;  // thread 0: records of the tiles issued
  auto issue = [&](int s) {
    int c = 0;
    const unsigned long long *kp = nullptr, *vp = nullptr;
    if (next_tile < total) {
      const unsigned long long tile = next_tile;
      next_tile += gridDim.x;
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
    }
    s_tcnt[s] = c;
    n_rec += (unsigned long long)c;
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
  // The producer is a warp of its own (thread BLK).  As thread 0 of the consumers
  // it issued a stage's next tile between barrier 2 and its own phase A, started
  // every tile ~1,000 cycles late and made the other 15 warps wait at barrier 1
  // (measured: 1,330 cycles of arrival skew per tile).  It also fetches the page
  // stash refills (a returning global atomic) off the consumers' path.
  if (tid >= BLK) {
    if (tid == BLK) {
      for (int it = 0; it < ntiles + 1; it++) {
        const int s = it % NS;
        if (it >= NS) mbar_wait(&mbar_e[s], (uint32_t)((it / NS - 1) & 1));  // (try_wait suspends the thread)
        issue(s);
        if (a.stash && *(volatile uint32_t*)&s_want && !*(volatile uint32_t*)&s_nv) {
          const uint32_t nb = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
          *(volatile uint32_t*)&s_nb = nb;
          __threadfence_block();
          *(volatile uint32_t*)&s_nv = 1;
          *(volatile uint32_t*)&s_want = 0;
        }
      }
      if (n_rec) {
        atomicExch(&a.t.hdr->frozen, 1);  // the resident set is final from now on
        // every routed record counts as spilled until an owner child finds its key resident
        atomicAdd(&a.stats[ST_SPILLED], n_rec);
        atomicAdd(&a.stats[ST_RECORDS], n_rec);
      }
      __threadfence_block();
      *(volatile uint32_t*)&s_pdone = 1;
    }
    return;
  }
  auto bar_consumers = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(BLK) : "memory"); };
  auto rec_idx0 = [&](int r) { return 2 * ((r >> 1) * BLK + tid) + (r & 1); };
  // ---- heavy hitters: every CTA counts the keys of its first tile in a scratch table
  // (the rings' shared memory, not in use yet), keeps up to 8 keys seen >= 16 times
  // (~0.8% of the tile) that are resident in the frozen table, and from then on reduces
  // their records per warp instead of routing them.  No sampling kernel, no host round
  // trip; the CTAs need not agree on the set.
  if (ntiles > 0 && !a.nohot) {
    constexpr int HS = 2048;  // scratch slots: key u64 + count u32 (24 KB: the rings of >= 91 runs)
    unsigned long long* hkeys = (unsigned long long*)ring;
    uint32_t* hcnt = (uint32_t*)(hkeys + HS);
    const bool room = (size_t)HS * 12 <= L::ring_bytes(NP);
    if (room) {
      for (int i = tid; i < HS; i += BLK) {
        hkeys[i] = EMPTY;
        hcnt[i] = 0;
      }
      mbar_wait(&mbar[0], 0u);  // the first tile has landed (it stays in its stage: the loop below takes it)
      const int c0 = s_tcnt[0];
      bar_consumers();
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int idx = rec_idx0(r);
        if (idx >= c0) continue;
        const uint64_t k = stg[idx];
        if (k == EMPTY) continue;
        uint32_t b = hash32(k, a.seed ^ 0x5bd1e995u) & (HS - 1);
        for (int t = 0; t < 8; t++, b = (b + 1) & (HS - 1)) {
          unsigned long long prev = hkeys[b];
          if (prev == EMPTY) prev = atomicCAS(&hkeys[b], EMPTY, (unsigned long long)k);
          if (prev == EMPTY || prev == k) {
            atomicAdd(&hcnt[b], 1u);
            break;
          }
        }
      }
      bar_consumers();
      for (int i = tid; i < HS; i += BLK)
        if (hcnt[i] >= 16u) {
          const int j = atomicAdd(&s_nhot, 1);
          if (j < 8) s_hk[j] = hkeys[i];
        }
      bar_consumers();
      const int nc = min(s_nhot, 8);
      if (tid < nc) {  // resident?  (probe the frozen table)
        const uint64_t k = s_hk[tid];
        const uint64_t kk[1] = {k};
        uint64_t b = hash_key<1>(kk, a.t.seed) & a.t.bmask;
        for (int step = 0; step < 64; step++) {
          uint64_t w[4];
          ld_bucket(a.t.keys, b, w);
          int hit = -1;
          bool emp = false;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            if (w[j] == k) hit = j;
            emp |= w[j] == EMPTY;
          }
          if (hit >= 0) {
            s_hslot[tid] = (uint32_t)(b * 4 + hit);
            break;
          }
          if (emp) break;
          b = (b + 1) & a.t.bmask;
        }
      }
      bar_consumers();
      if (tid == 0) {
        int nh = 0;
        for (int j = 0; j < nc; j++) {
          if (s_hslot[j] == 0xFFFFFFFFu) continue;
          const uint32_t d = hash32(s_hk[j], a.seed) >> 26;
          if (s_hdir[d] == 0xFF) {
            s_hdir[d] = (unsigned char)j;
            nh++;
          } else {
            s_hslot[j] = 0xFFFFFFFFu;  // (directory collision: this one is routed like any key)
          }
        }
        s_nhot = nh;
      }
      bar_consumers();
      nhot = s_nhot;
      bar_consumers();  // (the scratch is the rings' memory again)
    }
  }

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
      a.pool.page_set[pg] = a.set_id;
      a.pool.page_fill[pg] = S;
      const uint32_t u = atomicAdd(&lused[p], 1u);
      const uint32_t li = u < a.plist_blk ? lbase[p] + u : atomicAdd(&a.plist_n[p], 1u);
      if (li < a.plist_cap) {
        a.plist[(size_t)p * a.plist_cap + li] = pg;
      } else {  // a run far above the mean (skew): the shared overflow list
        const unsigned long long oi = atomicAdd(a.ovf_n, 1ull);
        if (oi < a.ovf_cap) a.ovf[oi] = ((unsigned long long)(uint32_t)p << 32) | pg;
        else atomicExch(a.fail, 1u);
      }
    }
    ent[p * NE + (j & (NE - 1))] = (pg << 8) | (j & 0xFFu);
  };

  // per-thread state of the tile: claim words and runs of its R records
  uint32_t old[R];
  int pid[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    old[r] = 0;
    pid[r] = 0;
  }
  uint32_t held = 0;   // ... claimed beyond their run's window
  uint32_t opark = 0;  // ... parked for the next tile (open line)
  uint64_t hk[R], hv[R];
#pragma unroll
  for (int r = 0; r < R; r++) hk[r] = hv[r] = 0;
  uint64_t vm = 0;  // OR of v ^ (v >> 63): bounds the magnitudes (compact children)
  uint32_t km = 0;  // OR of the keys' high words (32-bit child tables when zero)

  // stage index of record r of this thread: pairs (2i, 2i + 1), i = (r / 2) * BLK + tid
  auto rec_idx = [&](int r) { return 2 * ((r >> 1) * BLK + tid) + (r & 1); };
  auto in_window = [&](uint32_t o) { return ((((o & CWM) >> 3) - (o >> 23)) & 511u) < (uint32_t)LINES; };

  for (int it = 0; it < ntiles + 1; it++) {
    const int s = it % NS;
    mbar_wait(&mbar[s], (uint32_t)((it / NS) & 1));
    const int c = s_tcnt[s];
    if (tid == 0 && a.stash && !*(volatile uint32_t*)&s_nv && !*(volatile uint32_t*)&s_want && 2 * s_su >= s_sc)
      *(volatile uint32_t*)&s_want = 1;  // the producer fetches the next stash
    // ---- [A1] parked open-line records of the last tile into the ring
    if (__builtin_expect(opark != 0, 0)) {
#pragma unroll
      for (int r = 0; r < R; r++)
        if ((opark >> r) & 1u) ring[pid[r] * RS + (old[r] & (RING - 1))] = make_ulonglong2(hk[r], hv[r]);
      opark = 0;
    }
    // ---- [A2] route this tile's records
    const uint32_t a_sk = a_stg + (uint32_t)s * 2u * T * 8u, a_sv = a_sk + T * 8u;
    held = 0;
    auto route = [&](auto full, auto hot_t) {
      constexpr bool FULL = decltype(full)::value;
      constexpr bool HOT = decltype(hot_t)::value;  // (its own instantiation: the common path's code is unchanged)
      uint64_t k[R], v[R];
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        const uint32_t o = 16u * (uint32_t)((r >> 1) * BLK + tid);
        lds128(a_sk + o, k[r], k[r + 1]);
        lds128(a_sv + o, v[r], v[r + 1]);
      }
      uint32_t vm_ = FULL ? (1u << R) - 1u : 0u;
      if (!FULL) {
#pragma unroll
        for (int r = 0; r < R; r++) vm_ |= (uint32_t)(rec_idx(r) < c) << r;
        if (HOT) {  // records of resident heavy hitters: reduced per warp, not routed
#pragma unroll
          for (int r = 0; r < R; r++) {
            const uint32_t d = s_hdir[hash32(k[r], a.seed) >> 26];
            const bool hot = ((vm_ >> r) & 1u) && d != 0xFFu && s_hk[d & 7u] == k[r];
            unsigned hm = __ballot_sync(0xffffffffu, hot);
            while (hm) {
              const int l = __ffs(hm) - 1;
              const uint32_t j = __shfl_sync(0xffffffffu, d, l);
              const bool mine = hot && d == j;
              const unsigned grp = __ballot_sync(0xffffffffu, mine);
              hm &= ~grp;
              long long sv = mine ? (long long)v[r] : 0ll;
              long long mn = mine ? (long long)v[r] : 0x7FFFFFFFFFFFFFFFll;
              long long mx = mine ? (long long)v[r] : (long long)0x8000000000000000ull;
#pragma unroll
              for (int o = 16; o; o >>= 1) {
                sv += __shfl_xor_sync(0xffffffffu, sv, o);
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              }
              if (lane == l) {
                atomicAdd(&s_hacc[j][0], (unsigned long long)__popc(grp));
                atomicAdd(&s_hacc[j][1], (unsigned long long)sv);
                atomicMin((long long*)&s_hacc[j][2], mn);
                atomicMax((long long*)&s_hacc[j][3], mx);
              }
            }
            if (hot) vm_ &= ~(1u << r);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; r++) {
        pid[r] = (int)wc2_run(k[r], a.seed, (uint32_t)NP);
        const uint64_t m = v[r] ^ (uint64_t)((long long)v[r] >> 63);
        vm |= FULL ? m : (((vm_ >> r) & 1u) ? m : 0ull);
        km |= FULL ? (uint32_t)(k[r] >> 32) : (((vm_ >> r) & 1u) ? (uint32_t)(k[r] >> 32) : 0u);
      }
#pragma unroll
      for (int r = 0; r < R; r++)
        if (FULL || ((vm_ >> r) & 1u)) old[r] = atoms_add(a_cw + 4u * (uint32_t)pid[r], 1u);
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (!FULL && !((vm_ >> r) & 1u)) continue;
        const uint32_t x = old[r] & CWM;
        if (__builtin_expect((x & (S - 1)) == 0, 0)) alloc_page(pid[r], x >> SLOG);
        if (__builtin_expect(in_window(old[r]), 1))
          sts128(a_ring + 16u * ((uint32_t)pid[r] * RS + (x & (RING - 1))), k[r], v[r]);
        else
          held |= 1u << r;
      }
    };
    if (__builtin_expect(nhot != 0, 0)) route(std::false_type{}, std::true_type{});
    else if (c == T) route(std::true_type{}, std::false_type{});
    else route(std::false_type{}, std::false_type{});
    bar_consumers();  // ---- barrier 1
    if (tid == 0) {
      if (*(volatile uint32_t*)&s_nv && s_su >= s_sc) {
        const uint32_t nb = *(volatile uint32_t*)&s_nb;
        const bool fits = nb + (uint32_t)a.stash <= a.pool.capacity;
        if (!fits)
          for (uint32_t x = nb; x < min(nb + (uint32_t)a.stash, a.pool.capacity); x++) a.pool.page_set[x] = -1;
        s_sb = nb;
        s_sc = fits ? (uint32_t)a.stash : 0u;
        s_su = 0;
        *(volatile uint32_t*)&s_nv = 0;
      }
    }
    // ---- [B1] held records: complete lines straight to their page, the open line waits
    if (__builtin_expect(held != 0, 0)) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        if (!((held >> r) & 1u)) continue;
        const uint32_t x = old[r] & CWM;
        const uint32_t o = 8u * (uint32_t)rec_idx(r);
        const uint64_t k = lds64(a_sk + o), v = lds64(a_sv + o);
        if ((x >> 3) < ((cw[pid[r]] & CWM) >> 3)) {
          const uint32_t pg = page_of(pid[r], x >> SLOG);
          if (pg < 0xFFFFFFu) st_v2(rec_ptr(pg, x), make_ulonglong2(k, v));
        } else {
          hk[r] = k;
          hv[r] = v;
          opark |= 1u << r;
        }
      }
    }
    // ---- [B2] one lane per run (run p belongs to warp p % NW): the lines of the
    // run's window that this tile completed leave through the warp, four lines
    // per step (8 lanes x 16 bytes = one 128-byte line per store group), and the
    // window moves to the run's open line.  (Lines completed beyond the window
    // were all held.  A 128-byte bulk copy per line through the TMA engine
    // measured ~16 cycles per copy and SM: 57% of the tile.)
    {
      constexpr int NW = BLK / 32;
      const int wid = tid >> 5;
      const int sub = lane & 7, grp = lane >> 3;
      for (int p0 = wid; p0 < NP; p0 += 32 * NW) {
        const int p = p0 + NW * lane;
        uint32_t nl = 0, ln = 0;
        if (p < NP) {
          const uint32_t w = cw[p];
          const uint32_t cc = w & CWM;
          ln = cc >> 3;
          nl = (ln - (w >> 23)) & 511u;  // lines completed since the window opened
          if (nl) cw[p] = (ln << 23) | cc;
        }
        const uint32_t ns = nl < (uint32_t)LINES ? nl : (uint32_t)LINES;
        uint4* wq = sendq + 32 * wid;
        const uint32_t a_wq = smem_u32(wq);
#pragma unroll
        for (int round = 0; round < LINES; round++) {
          const bool has = ns > (uint32_t)round;
          const uint32_t mask = __ballot_sync(0xffffffffu, has);
          if (!mask) break;
          if (has) {  // the lane's line into the warp's list: where it is and where it goes
            const uint32_t x0 = (ln - nl + (uint32_t)round) << 3;
            const uint32_t pg = page_of(p, x0 >> SLOG);
            const unsigned long long dst = pg < 0xFFFFFFu ? (unsigned long long)rec_ptr(pg, x0) : 0ull;
            wq[__popc(mask & ((1u << lane) - 1u))] =
                make_uint4(a_ring + 16u * ((uint32_t)p * RS + (x0 & (RING - 1))), 0u, (uint32_t)dst, (uint32_t)(dst >> 32));
          }
          __syncwarp();
          const int n = __popc(mask);
          // lane group g copies lines g, g + 4, ...: 8 lanes x 16 bytes per line
#pragma unroll 2
          for (int i = grp; i < n; i += 4) {
            uint32_t src, pad;
            unsigned long long dst;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%3];\n\tld.shared.u64 %2, [%3 + 8];"
                         : "=r"(src), "=r"(pad), "=l"(dst)
                         : "r"(a_wq + 16u * (uint32_t)i));
            if (dst && !a.nosend) {
              uint64_t x, y;
              lds128(src + 16u * (uint32_t)sub, x, y);
              st_v2((void*)(dst + 16u * (uint32_t)sub), make_ulonglong2(x, y));
            }
          }
          __syncwarp();
        }
      }
    }
    bar_consumers();  // ---- barrier 2: ring and stage are free again
    if (tid == 0) mbar_arrive(&mbar_e[s]);
  }
  // ---- close: every run's open line (all in the ring), then the page fills
  for (int p = tid; p < NP; p += BLK) {
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
  // the entries of this CTA's page-list blocks it did not need are marked unused (every
  // entry below a run's count is then written by this run: the lists need no clearing)
  for (int p = tid; p < NP; p += BLK)
    for (uint32_t u = lused[p]; u < a.plist_blk; u++)
      if (lbase[p] + u < a.plist_cap) a.plist[(size_t)p * a.plist_cap + lbase[p] + u] = 0xFFFFFFFFu;
  if (tid == 0) {
    // unused stash pages leave the set (the producer is done: no refill in flight)
    while (!*(volatile uint32_t*)&s_pdone) {
    }
    for (uint32_t x = min(s_su, s_sc); x < s_sc; x++) a.pool.page_set[s_sb + x] = -1;
    if (*(volatile uint32_t*)&s_nv) {
      const uint32_t nb = *(volatile uint32_t*)&s_nb;
      for (uint32_t x = nb; x < min(nb + (uint32_t)a.stash, a.pool.capacity); x++) a.pool.page_set[x] = -1;
    }
  }
  if (nhot) {  // the heavy hitters' aggregates into the level-0 table; their records were not spilled
    bar_consumers();
    if (tid < 8 && s_hslot[tid] != 0xFFFFFFFFu && s_hacc[tid][0]) {
      uint64_t* st = a.t.states + (uint64_t)s_hslot[tid] * a.t.sstride;
      gupdate(st, OP_ADD, TY_I64, s_hacc[tid][0]);
      gupdate(st + a.t.fstride, OP_ADD, TY_I64, s_hacc[tid][1]);
      if (a.prog == 2) {
        gupdate(st + 2 * a.t.fstride, OP_MIN, TY_I64, s_hacc[tid][2]);
        gupdate(st + 3 * a.t.fstride, OP_MAX, TY_I64, s_hacc[tid][3]);
      }
      atomicAdd(&a.stats[ST_HITS], s_hacc[tid][0]);
      atomicAdd(&a.stats[ST_SPILLED], (unsigned long long)(-(long long)s_hacc[tid][0]));
    }
  }
  {
    uint32_t mlo = (uint32_t)vm, mhi = (uint32_t)(vm >> 32);
    mlo = __reduce_or_sync(0xffffffffu, mlo);
    mhi = __reduce_or_sync(0xffffffffu, mhi);
    km = __reduce_or_sync(0xffffffffu, km);
    if (lane == 0) {
      if (mhi | (mlo >> 31)) atomicOr(&a.vinfo[0], 1u);
      if (mlo) atomicOr(&a.vinfo[1], mlo & 0x7FFFFFFFu);
      if (km) atomicOr(&a.vinfo[2], km);
    }
  }
}

// ---------------------------------------------------------------------------
// k_child2_wc: one CTA per run, compact 32-bit states
// ---------------------------------------------------------------------------

struct Cw2Args {
  DevSpec sp;
  PagePool pool;
  const uint32_t* plist;
  const uint32_t* plist_n;
  uint32_t plist_cap;
  const unsigned long long* ovf;  // pages past the runs' lists: run << 32 | page
  const unsigned long long* ovf_n;
  uint32_t ovf_cap;
  const unsigned long long* part_recs;
  const unsigned int* vinfo;    // [0] some value outside int32, [1] OR of the magnitudes, [2] OR of the keys' high words (k_scan_wc)
  int32_t NP;                   // runs
  int32_t table_bytes;          // dynamic shared memory for the table
  uint64_t seed;                // slot hash seed of the child level
  OutBuf out;
  uint32_t* failed;             // [NP]: 1 = did not fit, left to the fallback
  uint32_t* fail;               // bit 2: some run failed (the host runs the fallback)
  unsigned long long* stats;
  GTable t;                     // the level-0 table (the runs merge their resident groups into it)
  const uint32_t* olist;        // [NP][ocap] resident slots per run
  const uint32_t* olist_n;      // [NP]
  uint32_t ocap;
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

__device__ __forceinline__ void reds_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void reds_min_s32(uint32_t a, int v) {
  asm volatile("red.shared.min.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void reds_max_s32(uint32_t a, int v) {
  asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// word layout of a slot's compact states (u32 words, slot-major so that every
// offset below is an immediate): MIN / MAX fields first (one LDS.64 reads a
// MIN-MAX pair), the count word, one word per SUM; the extended layout (wide
// sums and owner runs) adds the sums' high words and the level-0 slot of a
// seeded key.  Both strides are even (8-byte aligned slots).
template <class CP>
struct CwWords {
  static constexpr int N = CP::N;
  __host__ __device__ static constexpr bool is_mm(int j) { return !CP::is_count(j) && !CP::is_sum(j); }
  __host__ __device__ static constexpr int nmm() {
    int x = 0;
    for (int i = 0; i < N; i++) x += is_mm(i);
    return x;
  }
  static constexpr int NMM = nmm(), NSUM = CP::nsum();
  static constexpr int W_CNT = NMM;
  static constexpr int WB = NMM + 1 + NSUM;        // base words
  static constexpr int W_HI = WB;                  // + k: high word of sum k
  static constexpr int W_ORG = WB + NSUM;          // level-0 slot of a seeded key
  static constexpr int W_NARROW = (WB + 1) & ~1, W_EXT = (WB + NSUM + 1 + 1) & ~1;
  // word of field j (COUNT fields share the count word)
  __host__ __device__ static constexpr int word(int j) {
    if (CP::is_count(j)) return W_CNT;
    int x = 0;
    if (is_mm(j)) {
      for (int i = 0; i < j; i++) x += is_mm(i);
      return x;
    }
    for (int i = 0; i < j; i++) x += CP::is_sum(i);
    return NMM + 1 + x;
  }
  __host__ __device__ static constexpr int sum_rank(int j) {
    int x = 0;
    for (int i = 0; i < j; i++) x += CP::is_sum(i);
    return x;
  }
  __host__ __device__ static constexpr uint32_t identity(int w) {  // initial value of base word w
    for (int j = 0; j < N; j++)
      if (is_mm(j) && word(j) == w) return (CP::fd(j) & 3) == OP_MIN ? 0x7FFFFFFFu : 0x80000000u;
    return 0u;
  }
  // a MIN field at word 0 and a MAX field at word 1: read together
  __host__ __device__ static constexpr bool mm_pair() {
    if (NMM != 2) return false;
    bool mn = false, mx = false;
    for (int j = 0; j < N; j++) {
      if (is_mm(j) && word(j) == 0 && (CP::fd(j) & 3) == OP_MIN) mn = true;
      if (is_mm(j) && word(j) == 1 && (CP::fd(j) & 3) == OP_MAX) mx = true;
    }
    return mn && mx;
  }
};

// slot hash of a child table (independent of the level-0 routing hash: another seed)
__device__ __forceinline__ uint32_t cw_hash(uint64_t k, uint32_t seed) { return hash32(k, seed); }

// One run through a child table.  Template flags: K32 = every key the scan saw
// fits in 32 bits (keys are stored as u32: a bucket of 4 is one LDS.128 and four
// 32-bit compares; the one key equal to the empty marker 0xFFFFFFFF lives in the
// escape slot), WIDE = sums as u32 pairs with carry, EXT = the extended word
// layout (wide sums and seeded runs), V64 = some value is beyond int32 (64-bit
// MIN/MAX words, the sums take the value's high word).
//   table: keys[nslots + 1] (u32 or u64; 4-slot buckets; escape slot last), then
//          (nslots + 1) x W u32 state words
// A record compares its key with the four keys of its bucket, the buckets of RL
// records in flight together; a record that did not hit looks at the next bucket
// (a displaced key: warp-uniform second stage) and only then takes the general
// loop (first occurrence -> CAS insert, longer chains, the escape key).  COUNT,
// SUM, MIN and MAX are fire-and-forget shared-memory REDs (no read before the
// update: the kernel is bound by shared-memory latency, not by its atomic rate).
struct CwShared {
  int groups, fail, esc;
  unsigned int next;  // next page-list entry to hand out
  unsigned long long base;
  uint32_t wsum[32];
};

template <class CP, int BLK, int RL, bool K32, bool WIDE, bool EXT, bool V64 = false>
__device__ __forceinline__ void child_run(const Cw2Args& a, int p, bool owner, unsigned char* smem, CwShared& sh,
                                          uint32_t seed32) {
  using CW = CwWords<CP>;
  using KT = typename std::conditional<K32, uint32_t, uint64_t>::type;
  constexpr int N = CP::N;
  constexpr int NWARP = BLK / 32;
  constexpr int W = EXT ? CW::W_EXT : CW::W_NARROW;
  constexpr int KB = K32 ? 4 : 8;
  constexpr KT KEMPTY = K32 ? (KT)0xFFFFFFFFu : (KT)EMPTY;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // V64 (some value beyond int32): MIN / MAX live in 64-bit word arrays after the u32
  // ones (native 64-bit shared-memory MIN/MAX atomics), sums take the value's high word
  constexpr int MM64 = V64 ? CW::NMM : 0;
  const int nbk = ((a.table_bytes - 64) / (KB + 4 * W + 8 * MM64) - 1) / 4;
  const int nslots = nbk * 4;
  const int maxg = (int)(0.85 * nslots);
  const int stride = nslots + 1;
  KT* skeys = (KT*)smem;                                                     // stride keys (escape slot last)
  uint32_t* sst = (uint32_t*)(smem + (((size_t)stride * KB + 15) & ~(size_t)15));  // stride x W state words
  unsigned long long* smm = (unsigned long long*)(((uintptr_t)(sst + (size_t)stride * W) + 15) & ~(uintptr_t)15);  // MM64 x stride
  const uint32_t a_keys = smem_u32(skeys), a_st = smem_u32(sst), a_mm = smem_u32(smm);
  const uint32_t sbytes = 4u * (uint32_t)stride;  // bytes between a slot's consecutive words
  for (int i = tid; i < stride; i += BLK) {
    skeys[i] = KEMPTY;
#pragma unroll
    for (int w = 0; w < CW::WB; w++) sst[w * stride + i] = CW::identity(w);
    if (EXT) {
#pragma unroll
      for (int w = CW::WB; w < CW::W_EXT; w++) sst[w * stride + i] = w == CW::W_ORG ? 0xFFFFFFFFu : 0u;
    }
    if (V64) {
#pragma unroll
      for (int j = 0; j < N; j++)
        if (CW::is_mm(j))
          smm[CW::word(j) * stride + i] = (CP::fd(j) & 3) == OP_MIN ? 0x7FFFFFFFFFFFFFFFull : 0x8000000000000000ull;
    }
  }
  if (tid == 0) {
    sh.groups = 0;
    sh.fail = a.plist_n[p] > a.plist_cap && *a.ovf_n > a.ovf_cap;  // (the overflow list overflowed too: incomplete)
    sh.esc = 0;
    sh.next = 0;
  }
  __syncthreads();
  auto bucket_of = [&](uint64_t k) { return (int)__umulhi(cw_hash(k, seed32), (uint32_t)nbk); };
  // the general probe: hit, insert into the bucket chain's first empty slot, or fail (table full)
  auto probe_slow = [&](KT k, int b) -> int {
    for (;;) {
      const KT* bp = skeys + b * 4;
      const KT q0 = bp[0], q1 = bp[1], q2 = bp[2], q3 = bp[3];
      const int hit = q0 == k ? 0 : q1 == k ? 1 : q2 == k ? 2 : q3 == k ? 3 : -1;
      if (hit >= 0) return b * 4 + hit;
      const int emp = q0 == KEMPTY ? 0 : q1 == KEMPTY ? 1 : q2 == KEMPTY ? 2 : q3 == KEMPTY ? 3 : -1;
      if (emp < 0) {  // full bucket: the next one
        if (++b == nbk) b = 0;
        continue;
      }
      if (atomicAdd(&sh.groups, 1) >= maxg) {
        sh.fail = 1;
        return -1;
      }
      const int e = b * 4 + emp;
      KT prev;
      if constexpr (K32) prev = atomicCAS((unsigned int*)&skeys[e], KEMPTY, k);
      else prev = atomicCAS((unsigned long long*)&skeys[e], (unsigned long long)KEMPTY, (unsigned long long)k);
      if (prev == KEMPTY) return e;
      atomicSub(&sh.groups, 1);  // the slot went to another insert: look at the bucket again
    }
  };
  if (owner) {  // seed: the resident keys this owner answers for, with their level-0 slots
    const int o = p;
    const uint32_t nres = a.olist_n[o];
    if (nres > a.ocap || (int)nres > maxg) {
      if (tid == 0) sh.fail = 1;
    } else {
      for (uint32_t i = tid; i < nres; i += BLK) {
        const uint32_t ls = a.olist[(size_t)o * a.ocap + i];
        const uint64_t k = a.t.keys[ls];
        int sl;
        if (K32) {
          // (a resident key beyond 32 bits came in through FILL; no record of the runs can match it)
          if (k >> 32) continue;
          sl = (uint32_t)k == 0xFFFFFFFFu ? nslots : probe_slow((KT)k, bucket_of(k));
        } else {
          sl = probe_slow((KT)k, bucket_of(k));
        }
        if (sl >= 0) sst[CW::W_ORG * stride + sl] = ls;
      }
      if (!K32 && tid == 0 && *(volatile int*)&a.t.hdr->esc) sst[CW::W_ORG * stride + nslots] = (uint32_t)(a.t.mask + 1);
    }
    __syncthreads();
  }
  const uint32_t nown = min(a.plist_n[p], a.plist_cap);
  // entries: the run's own list, then (a run past its list only) every entry of the overflow list
  const uint32_t npg = nown + (a.plist_n[p] > a.plist_cap ? (uint32_t)min(*a.ovf_n, (unsigned long long)a.ovf_cap) : 0u);
  const uint32_t* pl = a.plist + (size_t)p * a.plist_cap;
  // Warps take the list's entries as they come free (pages differ in fill, and a
  // static split left the warps ~10% apart at the end of a run); the first lanes look at
  // one entry each of a small batch, the used ones are processed in turn with the next
  // one's page already on its way into L2.  Lane l takes slots l, l + 32, ... of a
  // page, RL records per lane in flight.
  for (;;) {
    uint32_t q0 = 0;
    constexpr uint32_t NB = 8;  // entries per batch (about four pages: the warps end a run within a few pages of each other)
    if (lane == 0) q0 = atomicAdd(&sh.next, NB);
    q0 = __shfl_sync(0xffffffffu, q0, 0);
    if (q0 >= npg || __any_sync(0xffffffffu, *(volatile int*)&sh.fail)) break;  // warp-uniform
    uint32_t mypg = 0xFFFFFFFFu;
    if ((uint32_t)lane < NB && q0 + lane < npg) {
      if (q0 + lane < nown) {
        mypg = pl[q0 + lane];
      } else {
        const unsigned long long e = a.ovf[q0 + lane - nown];
        if ((uint32_t)(e >> 32) == (uint32_t)p) mypg = (uint32_t)e;
      }
    }
    const int myfill = mypg != 0xFFFFFFFFu ? a.pool.page_fill[mypg] : 0;
    uint32_t used = __ballot_sync(0xffffffffu, myfill > 0);
    if (used) {  // the first page of the batch
      const int l0 = __ffs(used) - 1;
      if (lane == l0) bulk_prefetch_l2(page_ptr(a.pool, mypg), ((uint32_t)myfill * 16u + 15u) & ~15u);
    }
    while (used) {
      const int l = __ffs(used) - 1;
      used &= used - 1;
      if (used) {  // the next page into L2 while this one is processed
        const int ln = __ffs(used) - 1;
        if (lane == ln) bulk_prefetch_l2(page_ptr(a.pool, mypg), ((uint32_t)myfill * 16u + 15u) & ~15u);
      }
      const uint32_t pg = __shfl_sync(0xffffffffu, mypg, l);
      const int fill = __shfl_sync(0xffffffffu, myfill, l);
      const ulonglong2* pb = (const ulonglong2*)page_ptr(a.pool, pg);
    for (int s0 = 0; s0 < fill; s0 += RL * 32) {
      ulonglong2 cur[RL];
#pragma unroll
      for (int r = 0; r < RL; r++) {
        const int sl = s0 + r * 32 + lane;
        cur[r] = sl < fill ? __ldcs(pb + sl) : make_ulonglong2((uint64_t)KEMPTY, 0);  // (padding: the escape key, skipped below)
      }
      int bk[RL], slot[RL];
      bool need[RL];
      if constexpr (K32) {
        uint32_t q0[RL], q1[RL], q2[RL], q3[RL];
#pragma unroll
        for (int r = 0; r < RL; r++) {
          bk[r] = bucket_of(cur[r].x);
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(q0[r]), "=r"(q1[r]), "=r"(q2[r]), "=r"(q3[r])
                       : "r"(a_keys + 16u * (uint32_t)bk[r]));
        }
#pragma unroll
        for (int r = 0; r < RL; r++) {
          const uint32_t k = (uint32_t)cur[r].x;
          const bool e1 = q1[r] == k, e2 = q2[r] == k, e3 = q3[r] == k;
          const bool hit = ((q0[r] == k) | e1 | e2 | e3) & (k != KEMPTY);
          slot[r] = hit ? bk[r] * 4 + (int)e1 + 2 * (int)e2 + 3 * (int)e3 : -1;
          need[r] = !hit && s0 + r * 32 + lane < fill;
        }
      } else {
#pragma unroll
        for (int r0 = 0; r0 < RL; r0 += 2) {  // (two 32-byte buckets in flight: registers)
          uint64_t bx[2][4];
#pragma unroll
          for (int u = 0; u < 2; u++) {
            bk[r0 + u] = bucket_of(cur[r0 + u].x);
            lds128(a_keys + 32u * (uint32_t)bk[r0 + u], bx[u][0], bx[u][1]);
            lds128(a_keys + 32u * (uint32_t)bk[r0 + u] + 16u, bx[u][2], bx[u][3]);
          }
#pragma unroll
          for (int u = 0; u < 2; u++) {
            const int r = r0 + u;
            const uint64_t k = cur[r].x;
            const bool e1 = bx[u][1] == k, e2 = bx[u][2] == k, e3 = bx[u][3] == k;
            const bool hit = ((bx[u][0] == k) | e1 | e2 | e3) & (k != EMPTY);
            slot[r] = hit ? bk[r] * 4 + (int)e1 + 2 * (int)e2 + 3 * (int)e3 : -1;
            need[r] = !hit && s0 + r * 32 + lane < fill;
          }
        }
      }
      bool any_need = false;
#pragma unroll
      for (int r = 0; r < RL; r++) any_need |= need[r];
      if (__any_sync(0xffffffffu, any_need)) {  // warp-uniform second stage
#pragma unroll
        for (int r = 0; r < RL; r++) {
          if (!need[r]) continue;
          const KT k = (KT)cur[r].x;
          if (__builtin_expect(k == KEMPTY, 0)) {
            slot[r] = nslots;
            sh.esc = 1;  // (idempotent; read after the barrier)
          } else {
            const int b2 = bk[r] + 1 == nbk ? 0 : bk[r] + 1;
            const KT* bp = skeys + b2 * 4;
            const KT c0 = bp[0], c1 = bp[1], c2 = bp[2], c3 = bp[3];
            const bool f0 = c0 == k, f1 = c1 == k, f2 = c2 == k, f3 = c3 == k;
            if (f0 | f1 | f2 | f3) slot[r] = b2 * 4 + (f0 ? 0 : f1 ? 1 : f2 ? 2 : 3);
            else slot[r] = probe_slow(k, bk[r]);
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int r = 0; r < RL; r++) {
        if (slot[r] < 0) continue;
        const int cb = (int)(uint32_t)cur[r].y;  // the value (V64: its low word)
        // (word arrays, not slot-major: a warp's updates of one field spread over all 32
        // banks; slot-major states put them on 8 and tripled the atomics' wavefronts)
        const uint32_t a_s = a_st + 4u * (uint32_t)slot[r];
        reds_add(a_s + sbytes * CW::W_CNT, 1u);
#pragma unroll
        for (int j = 0; j < N; j++) {
          const uint32_t F = CP::fd(j);
          if (CP::is_count(j)) continue;
          const uint32_t a_w = a_s + sbytes * (uint32_t)CW::word(j);
          if (CP::is_sum(j)) {
            if (WIDE) {  // 64-bit two's complement sum in (lo, hi) words
              const uint32_t o = atoms_add(a_w, (uint32_t)cb);
              const uint32_t vhi = V64 ? (uint32_t)(cur[r].y >> 32) : (cb < 0 ? 0xFFFFFFFFu : 0u);
              const uint32_t hi = (uint32_t)(o + (uint32_t)cb < o) + vhi;
              if (hi) reds_add(a_s + sbytes * (uint32_t)(CW::W_HI + CW::sum_rank(j)), hi);
            } else {
              reds_add(a_w, (uint32_t)cb);
            }
          } else if (V64) {
            const uint32_t a_q = a_mm + 8u * (uint32_t)(CW::word(j) * stride + slot[r]);
            if ((F & 3) == OP_MIN) asm volatile("red.shared.min.s64 [%0], %1;" ::"r"(a_q), "l"((long long)cur[r].y) : "memory");
            else asm volatile("red.shared.max.s64 [%0], %1;" ::"r"(a_q), "l"((long long)cur[r].y) : "memory");
          } else if ((F & 3) == OP_MIN) {
            reds_min_s32(a_w, cb);
          } else {
            reds_max_s32(a_w, cb);
          }
        }
      }
    }
    }
  }
  __syncthreads();
  if (sh.fail) {
    if (tid == 0) {
      a.failed[p] = 1;
      atomicOr(a.fail, 4u);
    }
    __syncthreads();
    return;
  }
  // state word j of slot s as a 64-bit native state
  auto state_of = [&](int s, int j) -> uint64_t {
    const uint32_t* w = sst + s;
    if (CP::is_count(j)) return (uint64_t)w[CW::W_CNT * stride];
    if (CP::is_sum(j)) {
      const uint32_t lo = w[CW::word(j) * stride];
      return WIDE ? ((uint64_t)w[(CW::W_HI + CW::sum_rank(j)) * stride] << 32 | lo) : (uint64_t)(long long)(int)lo;
    }
    if (V64) return (uint64_t)smm[CW::word(j) * stride + s];
    return (uint64_t)(long long)(int)w[CW::word(j) * stride];
  };
  // rows this run emits: its groups, minus the seeded (resident) ones of an owner run
  auto emits = [&](int s) -> bool {
    if (EXT && owner && sst[CW::W_ORG * stride + s] != 0xFFFFFFFFu) return false;
    return (s == nslots) ? (sh.esc != 0 && sst[CW::W_CNT * stride + s] != 0) : (skeys[s] != KEMPTY);
  };
  // block compaction, one output reservation per run
  const int per = (stride + BLK - 1) / BLK;
  const int lo = tid * per, hi = min(stride, lo + per);
  uint32_t mine = 0;
  for (int s = lo; s < hi; s++) mine += emits(s);
  uint32_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.wsum[wid] = x;
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < NWARP; w++) {
      const uint32_t t2 = sh.wsum[w];
      sh.wsum[w] = acc;
      acc += t2;
    }
    // reserve the rows only if they fit (else the run goes to the fallback)
    unsigned long long base = 0;
    if (acc) {
      unsigned long long o = *(volatile unsigned long long*)a.out.count;
      for (;;) {
        if (o + acc > (unsigned long long)a.out.cap) {
          base = ~0ull;
          break;
        }
        const unsigned long long prev = atomicCAS(a.out.count, o, o + acc);
        if (prev == o) {
          base = o;
          break;
        }
        o = prev;
      }
    }
    sh.base = base;
  }
  __syncthreads();
  if (sh.base == ~0ull) {  // (nothing merged or emitted yet: the fallback redoes the whole run)
    if (tid == 0) {
      a.failed[p] = 1;
      atomicOr(a.fail, 4u);
    }
    __syncthreads();
    return;
  }
  if (EXT && owner) {
    // resident groups: merged into the level-0 table (its flush emits them), and
    // their records were not spilled after all
    unsigned long long hits = 0;
    for (int s = tid; s < stride; s += BLK) {
      const uint32_t ls = sst[CW::W_ORG * stride + s];
      const uint32_t cnt = sst[CW::W_CNT * stride + s];
      if (ls == 0xFFFFFFFFu || cnt == 0) continue;
      hits += cnt;
#pragma unroll
      for (int j = 0; j < N; j++) {
        const uint32_t F = CP::fd(j);
        gupdate(a.t.states + (uint64_t)j * a.t.fstride + (uint64_t)ls * a.t.sstride, F & 3, (F >> 2) & 3, state_of(s, j));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
    if (lane == 0 && hits) {
      atomicAdd(&a.stats[ST_HITS], hits);
      atomicAdd(&a.stats[ST_SPILLED], (unsigned long long)(-(long long)hits));
    }
  }
  int64_t idx = (int64_t)sh.base + sh.wsum[wid] + (x - mine);
  for (int s = lo; s < hi; s++) {
    if (!emits(s)) continue;
    const uint64_t kk[1] = {s == nslots ? (K32 ? 0xFFFFFFFFull : EMPTY) : (uint64_t)skeys[s]};
    uint64_t st[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < N; j++)
      if (j < 4) st[j] = state_of(s, j);
    emit_group4<1>(a.sp, a.out, idx++, kk, st);
  }
  __syncthreads();
}

template <class CP, int BLK, int RL>
__global__ void __launch_bounds__(BLK, 1) k_child2_wc(Cw2Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CwShared sh;
  const uint32_t vabs = a.vinfo[1] + 1u;
  const bool k32 = a.vinfo[2] == 0;  // every key of the runs fits in 32 bits
  const uint32_t seed32 = (uint32_t)a.seed ^ (uint32_t)(a.seed >> 32);
  const int NP = a.NP;
  for (int p = blockIdx.x; p < NP; p += gridDim.x) {
    const unsigned long long np = a.part_recs[p];
    if (np == 0) continue;
    const bool owner = true;  // every run answers for the resident keys of its hash range
    // wide sums (a u32 pair with carry) only when a run's sum can leave int32
    const bool wide = CP::nsum() > 0 && (double)np * (double)vabs >= 2147483647.0;
    if (a.vinfo[0]) {  // some value beyond int32: 64-bit MIN/MAX words, sums with the value's high word
      if (k32) child_run<CP, BLK, RL, true, true, true, true>(a, p, owner, smem, sh, seed32);
      else child_run<CP, BLK, RL, false, true, true, true>(a, p, owner, smem, sh, seed32);
    } else if (k32) {
      if (wide) child_run<CP, BLK, RL, true, true, true>(a, p, owner, smem, sh, seed32);
      else if (owner) child_run<CP, BLK, RL, true, false, true>(a, p, owner, smem, sh, seed32);
      else child_run<CP, BLK, RL, true, false, false>(a, p, owner, smem, sh, seed32);
    } else {
      if (wide) child_run<CP, BLK, RL, false, true, true>(a, p, owner, smem, sh, seed32);
      else if (owner) child_run<CP, BLK, RL, false, false, true>(a, p, owner, smem, sh, seed32);
      else child_run<CP, BLK, RL, false, false, false>(a, p, owner, smem, sh, seed32);
    }
  }
}

// Fallback after k_child2_wc: the runs that did not fit are re-probed by the host
// (gathered, then the generic PROBE); then every run's pages leave the spill set.
__global__ void k_wc2_retire(const uint32_t* plist, const uint32_t* plist_n, uint32_t cap, int NP,
                             const unsigned long long* ovf, const unsigned long long* ovf_n, uint32_t ovf_cap,
                             int32_t* page_set) {
  for (int p = blockIdx.x; p < NP; p += gridDim.x) {
    const uint32_t n = min(plist_n[p], cap);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t pg = plist[(size_t)p * cap + i];
      if (pg != 0xFFFFFFFFu) page_set[pg] = -1;
    }
  }
  const unsigned long long no = min(*ovf_n, (unsigned long long)ovf_cap);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < no;
       i += (unsigned long long)gridDim.x * blockDim.x)
    page_set[(uint32_t)ovf[i]] = -1;
}

// one run's pages -> dense key / value columns (a run the host re-probes)
__global__ void k_wc2_gather(PagePool pool, const uint32_t* pl, uint32_t nown, const unsigned long long* ovf,
                             uint32_t novf, uint32_t run, unsigned long long* keys, unsigned long long* vals,
                             unsigned long long* count) {
  __shared__ unsigned long long s_base;
  for (uint32_t q = blockIdx.x; q < nown + novf; q += gridDim.x) {
    uint32_t pg = 0xFFFFFFFFu;
    if (q < nown) {
      pg = pl[q];
    } else {
      const unsigned long long e = ovf[q - nown];
      if ((uint32_t)(e >> 32) == run) pg = (uint32_t)e;
    }
    if (pg == 0xFFFFFFFFu) continue;  // (uniform over the CTA)
    const int fill = pool.page_fill[pg];
    if (threadIdx.x == 0) s_base = atomicAdd(count, (unsigned long long)fill);
    __syncthreads();
    const ulonglong2* pb = (const ulonglong2*)page_ptr(pool, pg);
    for (int i = threadIdx.x; i < fill; i += blockDim.x) {
      const ulonglong2 r = pb[i];
      keys[s_base + i] = r.x;
      vals[s_base + i] = r.y;
    }
    __syncthreads();
  }
}

}  // namespace aggb
