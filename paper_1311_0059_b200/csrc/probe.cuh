// probe.cuh — k_probe: the PROBE pass specialised for one-word keys and one
// 8-byte value column (records of 16 bytes: the C1-C3 benchmark shapes).
//
// Same contract as k_pass in MODE_PROBE (_kernels.py k_pp_probe :917-962):
// every record of the batch remainder (and of the FILL deferral list) either
// aggregates into its resident group with L2 atomics or spills to its
// partition's page, and the spill layout (CTA-private AoS pages, sector-complete
// writes through an SMEM residual) is the one k_child reads.
//
// What differs is how a warp spends its instructions.  ~85% of records are
// rejected by the SMEM bloom filter; the ~15% that pass it (resident hits and
// false positives) are pushed into a per-warp SMEM ring and resolved 32 at a
// time by all lanes together, so the bucket probe and the four atomics of a hit
// run with full warps instead of 4-5 active lanes per record slot.  Results go
// back to the owning lanes as ballot masks; owners keep their records in
// registers and claim spill ranks themselves.  Record width, sector group and
// page size are compile-time constants.
#pragma once
#include "pass.cuh"

namespace aggb {

constexpr int PQ_RING = 64;  // per-warp ring of bloom-positive records (two rounds of 32)

// Resolve key k (value v) against the frozen table: aggregate with L2 atomics if
// resident.  The first bucket (b, x, y) was loaded by the caller.
template <class PG>
__device__ __forceinline__ int64_t probe_finish(const PassArgs& a, uint64_t k, uint64_t v, uint64_t b, ulonglong2 x,
                                             ulonglong2 y, const uint32_t* s_fd, int ns) {
  int64_t s = -1;
  if (k == EMPTY) {  // escape slot: the key whose word equals the sentinel
    if (*(volatile int*)&a.t.hdr->esc) s = (int64_t)a.t.mask + 1;
  } else {
    for (;;) {
      if (x.x == k) { s = (int64_t)(b * 4); break; }
      if (x.y == k) { s = (int64_t)(b * 4 + 1); break; }
      if (y.x == k) { s = (int64_t)(b * 4 + 2); break; }
      if (y.y == k) { s = (int64_t)(b * 4 + 3); break; }
      if ((x.x == EMPTY) | (x.y == EMPTY) | (y.x == EMPTY) | (y.y == EMPTY)) break;
      b = (b + 1) & a.t.bmask;
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(a.t.keys + b * 4);
      x = __ldcg(p);
      y = __ldcg(p + 1);
    }
  }
  if (s < 0) return -1;
  const uint64_t vv[1] = {v};
  Upd<PG>::template g<1>(a.t.states, a.t.fstride, (uint64_t)s * a.t.sstride, 0, s_fd, ns, vv);
  return s;
}

__device__ __forceinline__ uint64_t probe_issue(const PassArgs& a, uint64_t k, uint64_t& b, ulonglong2& x, ulonglong2& y) {
  const uint64_t kk[1] = {k};
  const uint64_t hh = hash_key<1>(kk, a.t.seed);
  b = hh & a.t.bmask;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(a.t.keys + b * 4);
  x = __ldca(p);  // L1: prefetched by the owner lane at classification
  y = __ldca(p + 1);
  return hh;
}

// Spill layout: each CTA appends a partition's records to its own chain of
// 8 KB pages (512 records).  A record claims its index in the chain with one
// shared-memory atomic (cnt[p]); the claimer of a page's first slot allocates
// the page (from a CTA-local stash) and publishes it in the partition's page
// map ent[p][j mod 8] tagged with j; everyone else writes straight into the
// page the map names.  A record whose page is not published yet (its
// allocator is still in flight) is written after the tile's barrier, when
// every allocation of the tile is visible.  8 map entries cover a tile: a map
// entry is reused only 7 pages (3584 records) later, more than a tile holds.
//
// Phases (PM):
//   PM_ONE     one pass: bloom positives resolved through the per-warp ring.
//   PM_SCAN    two-phase PROBE, phase 1: a pure streaming partition pass.  Bloom
//              positives (~15% on C2) are appended to NREG candidate regions
//              (one atomic per warp and tile; warp w writes region w mod NREG,
//              which bounds a region by a quarter of the records) and every
//              other record spills.  No probe latency sits inside the tile
//              loop.  The chains stay open: each CTA saves {cnt, last page}
//              per partition.
//   PM_RESOLVE phase 2 (same grid): CTA c reopens CTA c's chains, resolves the
//              candidates 32 at a time through the ring (every lane busy),
//              spills the misses (bloom false positives) into the same chains
//              and seals them.
constexpr int PM_ONE = 0, PM_SCAN = 1, PM_RESOLVE = 2;
constexpr int NREG = 4;

template <int R, int BLK, class PG, int PM, int NH = 0>
__global__ void __launch_bounds__(BLK, 1) k_probe(PassArgs a) {
  constexpr int T = R * BLK, NWARP = BLK / 32;
  constexpr int SLOG = 9, S = 1 << SLOG;  // 16-byte records per 8 KB page
  constexpr int NE = 8;                   // page-map entries per partition
  static_assert((NE - 1) * S >= T, "a page-map entry must outlive a tile");
  static_assert(NWARP % NREG == 0, "candidate regions split the warps evenly");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int P = a.ss.nparts;
  const int nbw = (PM != PM_RESOLVE && a.bloom.words) ? (int)a.bloom.mask + 1 : 0;
  uint64_t* sbloom = (uint64_t*)smem;
  constexpr int RING = PM == PM_SCAN ? 0 : PQ_RING;                          // phase 1 has no ring
  ulonglong2* ring = (ulonglong2*)(sbloom + ((nbw + 1) & ~1)) + wid * RING;  // this warp's ring (16-B aligned)
  uint32_t* cnt = (uint32_t*)((ulonglong2*)(sbloom + ((nbw + 1) & ~1)) + NWARP * RING);  // P
  uint32_t* ent = cnt + P;                                                                 // P * NE
  // PM_SCAN sector pairs: records 2m and 2m+1 of a chain leave as one 32-byte
  // store.  The even one parks in pk[p] (tag ptag[p] = m) and the odd one takes
  // it; when the slot is busy the even one is written alone, and an odd one
  // that does not find its partner parked (after the tile's barrier, every
  // even record has parked or been written) is written alone too.
  const bool PAIR = PM == PM_SCAN && a.pairs;  // one-pass: measured slower with pairs (2.15 -> 2.48 ms)
  ulonglong2* pk = (ulonglong2*)(((uintptr_t)(ent + P * NE) + 15) & ~(uintptr_t)15);  // P (PAIR)
  uint32_t* ptag = (uint32_t*)(pk + (PM != PM_RESOLVE ? P : 0));                        // P (PAIR)
  constexpr uint32_t FREE = 0xFFFFFFFFu, BUSY = 0x80000000u;
  __shared__ uint32_t s_hm[NWARP][R];
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_grab[2];
  __shared__ uint32_t s_sb[2], s_su[2], s_sc[2];  // page stash by tile parity: base, used, capacity
  __shared__ unsigned long long s_cnt[ST_NSTATS];
  __shared__ unsigned long long s_rt[NREG + 1];    // PM_RESOLVE: first tile of each candidate region
  __shared__ unsigned long long s_rn[NREG];        // PM_RESOLVE: candidates per region
  // heavy-hitter tier (NH > 0, pass.cuh): directory, resolved slots, per-thread columns
  using HO = HotOps<PG>;
  uint64_t* hdk = (uint64_t*)(((uintptr_t)(PAIR ? (void*)(ptag + P) : (void*)(ent + P * NE)) + 15) & ~(uintptr_t)15);
  int32_t* hdi = (int32_t*)(hdk + HOT_DIR);
  long long* hsl = (long long*)(hdi + HOT_DIR);
  uint64_t* hacc = (uint64_t*)(hsl + HOT_MAX);
  if constexpr (NH > 0) {
    for (int i = tid; i < HOT_DIR; i += BLK) {
      hdk[i] = EMPTY;
      hdi[i] = -1;
    }
    if (tid < HOT_MAX) hsl[tid] = -1;
    for (int q = 0; q < HOT_MAX; q++)
      for (int j = 0; j < HO::N; j++) {
        const uint32_t F = HO::desc(j);
        hacc[((size_t)q * HO::N + j) * BLK + tid] = state_identity(F & 3, (F >> 2) & 3);
      }
    __syncthreads();
    if (tid == 0) {
      const int nh = a.hot[HOT_MAX] < (uint64_t)HOT_MAX ? (int)a.hot[HOT_MAX] : HOT_MAX;
      for (int q = 0; q < nh; q++) {
        const uint64_t k[1] = {a.hot[q]};
        const int d = (int)(hash_key<1>(k, a.t.seed) >> 58) & (HOT_DIR - 1);
        if (hdi[d] < 0) {
          hdk[d] = k[0];
          hdi[d] = q;
        }
      }
    }
  }

  const int64_t n = PM == PM_RESOLVE ? 0 : a.col.n;
  const int64_t col_start = (PM != PM_RESOLVE && a.start_tiles)
                                ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T)
                                : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t n_lin = (PM != PM_RESOLVE && a.lin_count) ? (int64_t)*a.lin_count : 0;

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  for (int p = tid; p < P; p += BLK) cnt[p] = 0;
  for (int i = tid; i < P * NE; i += BLK) ent[i] = 0xFFFFFF00u | (uint32_t)(((i & (NE - 1)) + 1) & (NE - 1));
  if (PAIR)
    for (int p = tid; p < P; p += BLK) ptag[p] = FREE;
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  if (PM == PM_RESOLVE && tid == 0) {
    unsigned long long acc = 0;
    for (int g = 0; g < NREG; g++) {
      s_rt[g] = acc;
      s_rn[g] = a.cand_count[g];
      acc += (s_rn[g] + T - 1) / T;
    }
    s_rt[NREG] = acc;
  }
  for (int i = tid; i < nbw; i += BLK) sbloom[i] = __ldcg((const unsigned long long*)a.bloom.words + i);
  __syncthreads();
  if (PM == PM_RESOLVE) {  // reopen the chains phase 1 left in this CTA's name
    for (int p = tid; p < P; p += BLK) {
      const uint2 c = a.chains[(size_t)blockIdx.x * P + p];
      cnt[p] = c.x;
      if (c.x) {
        const uint32_t j = (c.x - 1) >> SLOG;
        ent[p * NE + (j & (NE - 1))] = (c.y << 8) | (j & 0xFFu);
      }
    }
  }
  const unsigned long long total =
      PM == PM_RESOLVE ? s_rt[NREG] : (unsigned long long)(col_tiles + (n_lin + T - 1) / T);
  uint64_t* const pool = (uint64_t*)a.pool.base;

  auto load_tile = [&](unsigned long long tile, uint64_t (&k)[R], uint64_t (&v)[R], bool (&live)[R]) {
    int64_t base, end;
    const long long *kp, *vp;
    if constexpr (PM == PM_RESOLVE) {
      int g = 0;
#pragma unroll
      for (int q = 1; q < NREG; q++)
        if (tile >= s_rt[q]) g = q;
      base = (int64_t)(tile - s_rt[g]) * T;
      end = (int64_t)s_rn[g];
      kp = (const long long*)a.cand + (size_t)g * a.cand_stride;
      vp = kp + (size_t)NREG * a.cand_stride;
    } else {
      const int src = (int64_t)tile < col_tiles ? 0 : 1;
      base = src == 0 ? col_start + (int64_t)tile * T : ((int64_t)tile - col_tiles) * T;
      end = src == 0 ? n : n_lin;
      kp = (const long long*)(src == 0 ? a.col.key[0] : a.lin.key[0]);
      vp = (const long long*)(src == 0 ? a.col.val[0] : a.lin.val[0]);
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t i = base + r * BLK + tid;
      live[r] = (tile < total) && (i < end);
      if (live[r]) {
        k[r] = (uint64_t)__ldcs(kp + i);
        v[r] = (uint64_t)__ldcs(vp + i);
      }
    }
  };
  auto put2 = [&](uint32_t pg, uint32_t slot_even, ulonglong2 e, uint64_t k, uint64_t v) {  // one full sector
    if (pg < 0xFFFFFFu)
      asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(pool + (((size_t)pg << SLOG) + slot_even) * 2),
                   "l"(e.x), "l"(e.y), "l"(k), "l"(v)
                   : "memory");
  };
  auto put = [&](uint32_t pg, uint32_t slot, uint64_t k, uint64_t v) {
    if (pg < 0xFFFFFFu) __stcg((ulonglong2*)(pool + (((size_t)pg << SLOG) + slot) * 2), make_ulonglong2(k, v));
  };

  // tiles are grabbed two ahead: s_grab[t & 1] holds the index of this CTA's tile t
  if (tid == 0) {
    s_sb[0] = s_sb[1] = s_su[0] = s_su[1] = s_sc[0] = s_sc[1] = 0;
    s_grab[0] = total ? atomicAdd(a.tile_counter, 1ull) : 0ull;
    s_grab[1] = total ? atomicAdd(a.tile_counter, 1ull) : 0ull;
  }
  __syncthreads();
  unsigned long long cur = s_grab[0], nxt = s_grab[1];
  uint64_t kc[R], vc[R];
  bool lc[R];
  load_tile(cur, kc, vc, lc);

  uint32_t c_hit = 0, c_rec = 0, c_sp = 0;
  int par = 0;
  const uint32_t lt_mask = (1u << lane) - 1u;
  while (cur < total) {
    // thread 0 grabs tile t + 2 (into s_grab[t & 1], read by all before the last
    // barrier) and refills the other parity's page stash (idle during this tile);
    // the atomics' latency hides behind phase A
    unsigned long long g_next = 0;
    uint32_t ref_first = 0;
    bool refill = false;
    if (tid == 0) {
      g_next = atomicAdd(a.tile_counter, 1ull);
      const int q = par ^ 1;
      refill = a.stash && s_su[q] >= s_sc[q];  // refill a used-up stash only: no page is dropped
      if (refill) ref_first = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
    }
    // ---- [A] classify: one hash; partition from its high bits, bloom from a remix
    int part[R];
    uint32_t seq[R];  // ring sequence number of a bloom-positive record, ~0u otherwise
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t kk[1] = {kc[r]};
      const uint64_t h = hash_key<1>(kk, a.t.seed);
      part[r] = kc[r] == EMPTY ? 0 : (int)reduce32(h, (uint32_t)P);
      if constexpr (NH > 0) {  // heavy hitter with a resolved slot: this thread's column
        const int d = (int)(h >> 58) & (HOT_DIR - 1);
        if (lc[r] && hdk[d] == kc[r] && kc[r] != EMPTY) {
          const int q = hdi[d];
          if (*(volatile long long*)&hsl[q] >= 0) {
            const uint64_t vv[1] = {vc[r]};
            HO::template add<1>(hacc + (size_t)q * HO::N * BLK + tid, BLK, 0, vv);
            c_rec++;
            c_hit++;
            lc[r] = false;
          }
        }
      }
      bool posv = lc[r];
      if (nbw && kc[r] != EMPTY) {
        const uint64_t bits = bloom_bits(h);
        posv = posv && (sbloom[bloom_block(h, a.bloom.mask)] & bits) == bits;
      }
      // a positive is resolved by some lane of the warp shortly: pull its first
      // bucket into L1 now (the frozen table is read-only for this kernel)
      if (PM == PM_ONE && posv && kc[r] != EMPTY)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.t.keys + (h & a.t.bmask) * 4));
      seq[r] = posv ? 0u : ~0u;
    }
    // ---- PM_SCAN: reserve this warp's candidate slots now (one atomic per warp
    // and tile); the result is consumed after the claims, which hide its latency
    uint32_t mk[R], ctot = 0;
    unsigned long long cbase = 0;
    if constexpr (PM == PM_SCAN) {
#pragma unroll
      for (int r = 0; r < R; r++) {
        mk[r] = __ballot_sync(0xffffffffu, seq[r] == 0u);
        ctot += __popc(mk[r]);
      }
      if (ctot && lane == 0) cbase = atomicAdd(&a.cand_count[wid & (NREG - 1)], (unsigned long long)ctot);
    }
    // ---- prefetch the next tile
    uint64_t kn[R], vn[R];
    bool ln[R];
    load_tile(nxt, kn, vn, ln);
    if constexpr (PM != PM_SCAN) {
      // ---- resolve the bloom positives 32 at a time
      uint32_t qt = 0, qh = 0;  // warp-uniform ring tail / head
      auto round = [&](uint32_t cnt_in) {  // resolve ring entries [qh, qh + cnt_in)
        __syncwarp();
        bool hit = false;
        if (lane < (int)cnt_in) {
          const ulonglong2 e = ring[(qh + lane) & (PQ_RING - 1)];
          uint64_t b = 0, hh = 0;
          ulonglong2 x = make_ulonglong2(0, 0), y = x;
          if (e.x != EMPTY) hh = probe_issue(a, e.x, b, x, y);
          const int64_t sl = probe_finish<PG>(a, e.x, e.y, b, x, y, s_fd, ns);
          hit = sl >= 0;
          if constexpr (NH > 0) {  // a resolved heavy hitter: this CTA's columns take it from now on
            const int d = (int)(hh >> 58) & (HOT_DIR - 1);
            if (hit && e.x != EMPTY && hdk[d] == e.x) *(volatile long long*)&hsl[hdi[d]] = sl;
          }
        }
        const uint32_t hb = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_hm[wid][qh >> 5] = hb;
        __syncwarp();
      };
#pragma unroll
      for (int r = 0; r < R; r++) {
        const bool posv = seq[r] == 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, posv);
        if (posv) {
          seq[r] = qt + __popc(m & lt_mask);
          ring[seq[r] & (PQ_RING - 1)] = make_ulonglong2(kc[r], vc[r]);
        }
        qt += __popc(m);
        if (qt - qh >= 32) {
          round(32);
          qh += 32;
        }
      }
      if (qt != qh) round(qt - qh);
      __syncwarp();
    }
    // ---- claim chain positions and write the spilled records (one record at a
    // time: batching the R claim atomics measured no faster, 2.08 vs 2.15 ms)
    uint32_t pend = 0, pidx[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      pidx[r] = 0;
      if (PM != PM_RESOLVE) c_rec += lc[r];
      bool spill = lc[r];
      if (seq[r] != ~0u) {
        if constexpr (PM == PM_SCAN) {
          spill = false;  // a candidate: phase 2 resolves it
        } else {
          const bool hit = (s_hm[wid][seq[r] >> 5] >> (seq[r] & 31)) & 1u;
          c_hit += hit;
          spill = !hit;
        }
      }
      if (!spill) continue;
      c_sp++;
      const int p = part[r];
      const uint32_t idx = atomicAdd(&cnt[p], 1u);
      const uint32_t j = idx >> SLOG, slot = idx & (S - 1);
      uint32_t* ep = &ent[p * NE + (j & (NE - 1))];
      uint32_t pg;
      if (slot == 0) {  // first record of page j: allocate it and publish it
        const uint32_t off = atomicAdd(&s_su[par], 1u);
        if (off < s_sc[par]) {
          pg = s_sb[par] + off;
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
        }
        *(volatile uint32_t*)ep = (pg << 8) | (j & 0xFFu);
      } else {
        const uint32_t e = *(volatile uint32_t*)ep;
        pg = ((e & 0xFFu) == (j & 0xFFu)) ? (e >> 8) : 0xFFFFFFFFu;
      }
      pidx[r] = idx;
      if (PAIR) {
        const uint32_t m = idx >> 1;
        if (!(idx & 1u)) {  // even: park for the partner, or go alone
          // (no fence: the partner reads the slot only after the tile's barrier)
          if (atomicCAS(&ptag[p], FREE, m | BUSY) == FREE) {
            pk[p] = make_ulonglong2(kc[r], vc[r]);
            *(volatile uint32_t*)&ptag[p] = m;
          } else if (pg == 0xFFFFFFFFu) {
            pend |= 1u << r;
          } else {
            put(pg, slot, kc[r], vc[r]);
          }
        } else {
          pend |= 1u << r;  // odd: decided after the barrier
        }
      } else if (pg == 0xFFFFFFFFu) {
        pend |= 1u << r;
      } else {
        put(pg, slot, kc[r], vc[r]);
      }
    }
    if constexpr (PM == PM_SCAN) {
      if (ctot) {
        cbase = __shfl_sync(0xffffffffu, cbase, 0);
        const int g = wid & (NREG - 1);
        uint64_t* ck = a.cand + (size_t)g * a.cand_stride;
        uint64_t* cv = a.cand + (size_t)(NREG + g) * a.cand_stride;
#pragma unroll
        for (int r = 0; r < R; r++) {
          if (seq[r] == 0u) {
            const unsigned long long i = cbase + __popc(mk[r] & lt_mask);
            __stcg((unsigned long long*)ck + i, (unsigned long long)kc[r]);
            __stcg((unsigned long long*)cv + i, (unsigned long long)vc[r]);
          }
          cbase += __popc(mk[r]);
        }
      }
    }
    if (tid == 0) {
      s_grab[par] = g_next;
      if (refill) {
        const int q = par ^ 1;
        for (uint32_t x = min(s_su[q], s_sc[q]); x < s_sc[q]; x++) a.pool.page_set[s_sb[q] + x] = -1;
        const bool fits = ref_first + (uint32_t)a.stash <= a.pool.capacity;
        if (!fits)
          for (uint32_t x = ref_first; x < min(ref_first + (uint32_t)a.stash, a.pool.capacity); x++)
            a.pool.page_set[x] = -1;
        s_sb[q] = ref_first;
        s_sc[q] = fits ? (uint32_t)a.stash : 0u;
        s_su[q] = 0;
      }
    }
    __syncthreads();
    // ---- records whose page was published by another thread after they looked
#pragma unroll
    for (int r = 0; r < R; r++) {
      if (!((pend >> r) & 1u)) continue;
      const uint32_t idx = pidx[r], j = idx >> SLOG;
      const uint32_t e = ent[part[r] * NE + (j & (NE - 1))];
      if ((e & 0xFFu) != (j & 0xFFu)) {
        atomicExch(a.pool.overflow, 3u);  // cannot happen: the allocation precedes the barrier
        continue;
      }
      if (PAIR && (idx & 1u)) {
        const int p = part[r];
        if (*(volatile uint32_t*)&ptag[p] == (idx >> 1)) {  // the partner parked before the barrier: take it
          ulonglong2 pe;
          asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
                       : "=l"(pe.x), "=l"(pe.y)
                       : "r"((uint32_t)__cvta_generic_to_shared(&pk[p])));
          *(volatile uint32_t*)&ptag[p] = FREE;  // after the read (in-order shared-memory pipe)
          put2(e >> 8, idx & (S - 1) & ~1u, pe, kc[r], vc[r]);
          continue;
        }
      }
      put(e >> 8, idx & (S - 1), kc[r], vc[r]);
    }
    cur = nxt;
    nxt = s_grab[par];
    par ^= 1;
#pragma unroll
    for (int r = 0; r < R; r++) {
      lc[r] = ln[r];
      kc[r] = kn[r];
      vc[r] = vn[r];
    }
  }
  __syncthreads();
  if constexpr (NH > 0) {  // heavy-hitter columns: warp-reduced, one L2 update per warp and field
    for (int q = 0; q < HOT_MAX; q++) {
      const long long sl = hsl[q];
      if (sl < 0) continue;  // CTA-uniform (after the barrier above)
#pragma unroll
      for (int j = 0; j < HO::N; j++) {
        const uint32_t F = HO::desc(j);
        uint64_t v = hacc[((size_t)q * HO::N + j) * BLK + tid];
#pragma unroll
        for (int o = 16; o; o >>= 1) v = merge_word(v, __shfl_xor_sync(0xffffffffu, v, o), F & 3, (F >> 2) & 3);
        if (lane == 0 && v != state_identity(F & 3, (F >> 2) & 3))
          gupdate(a.t.states + (uint64_t)j * a.t.fstride + (uint64_t)sl * a.t.sstride, F & 3, (F >> 2) & 3, v);
      }
    }
  }
  if (PAIR) {
    // a parked even record whose partner never came is the last of its chain
    for (int p = tid; p < P; p += BLK) {
      const uint32_t t = ptag[p];
      if (t == FREE) continue;
      const uint32_t idx = 2u * t, j = idx >> SLOG;
      const uint32_t e = ent[p * NE + (j & (NE - 1))];
      if ((t & BUSY) || idx + 1 != cnt[p] || (e & 0xFFu) != (j & 0xFFu)) {
        atomicExch(a.pool.overflow, 3u);  // cannot happen
        continue;
      }
      const ulonglong2 pe = pk[p];
      put(e >> 8, idx & (S - 1), pe.x, pe.y);
    }
  }
  if constexpr (PM == PM_SCAN) {
    // leave the chains open for phase 2: {records claimed, page of the last claim}
    for (int p = tid; p < P; p += BLK) {
      const uint32_t c = cnt[p];
      uint32_t pg = 0xFFFFFFu;
      if (c) {
        const uint32_t j = (c - 1) >> SLOG;
        const uint32_t e = ent[p * NE + (j & (NE - 1))];
        if ((e & 0xFFu) == (j & 0xFFu)) pg = e >> 8;
      }
      a.chains[(size_t)blockIdx.x * P + p] = make_uint2(c, pg);
    }
  } else {
    // seal: the last page of every chain holds cnt mod S records
    for (int p = tid; p < P; p += BLK) {
      const uint32_t c = cnt[p];
      if (!c) continue;
      const uint32_t j = (c - 1) >> SLOG;
      const uint32_t e = ent[p * NE + (j & (NE - 1))];
      if ((e >> 8) < 0xFFFFFFu) a.pool.page_fill[e >> 8] = (int32_t)(c - (j << SLOG));
    }
  }
  // unused stash pages leave the set
  for (int q = 0; q < 2; q++)
    for (uint32_t x = min(s_su[q], s_sc[q]) + tid; x < s_sc[q]; x += BLK) a.pool.page_set[s_sb[q] + x] = -1;
  if (c_sp) atomicExch(&a.t.hdr->frozen, 1);  // the resident set is final from now on
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
// k_probe_w: the PROBE pass for wider records — two-word keys and several
// payload words read from strided, typed columns (C5's 64-byte rows: int64 ||
// int32 key, 4 values; 48-byte spill records).  Same page chains, claims and
// page map as k_probe.  Bloom positives are rare here (the table holds ~2% of
// the groups), so they are resolved inline; a record's words leave as 16-byte
// stores (a 48-byte record covers 1.5 sectors, so partial sectors are few).
// ---------------------------------------------------------------------------
constexpr int gcd_c(int x, int y) { return y ? gcd_c(y, x % y) : x; }

template <int KW, int NW, int R, int BLK, class PG>
__global__ void __launch_bounds__(BLK, 1) k_probe_w(PassArgs a) {
  constexpr int RW = KW + NW;
  constexpr int GRP = 4 / gcd_c(RW, 4);
  constexpr int S = (8192 / (RW * 8)) / GRP * GRP;  // records per page, as make_set
  constexpr int T = R * BLK;
  constexpr int NE = 8;
  static_assert((NE - 1) * S >= T, "a page-map entry must outlive a tile");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int P = a.ss.nparts;
  const int nbw = a.bloom.words ? (int)a.bloom.mask + 1 : 0;
  uint64_t* sbloom = (uint64_t*)smem;
  uint32_t* cnt = (uint32_t*)(sbloom + ((nbw + 1) & ~1));  // P
  uint32_t* ent = cnt + P;                                  // P * NE
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_grab[2];
  __shared__ uint32_t s_sb[2], s_su[2], s_sc[2];
  __shared__ unsigned long long s_cnt[ST_NSTATS];
  __shared__ int s_dummy[4];
  const CapCache cc{&s_dummy[0], (unsigned*)&s_dummy[1], &s_dummy[2], &s_dummy[3], 0u, 0ull};

  const int64_t n = a.col.n;
  const int64_t col_start =
      a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t n_lin = a.lin_count ? (int64_t)*a.lin_count : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (n_lin + T - 1) / T);
  if (total == 0) return;

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  for (int p = tid; p < P; p += BLK) cnt[p] = 0;
  for (int i = tid; i < P * NE; i += BLK) ent[i] = 0xFFFFFF00u | (uint32_t)(((i & (NE - 1)) + 1) & (NE - 1));
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  for (int i = tid; i < nbw; i += BLK) sbloom[i] = __ldcg((const unsigned long long*)a.bloom.words + i);
  uint64_t* const pool = (uint64_t*)a.pool.base;

  auto load_tile = [&](unsigned long long tile, uint64_t (&k)[R][KW], uint64_t (&v)[R][NW], bool (&live)[R]) {
    const bool lin = (int64_t)tile >= col_tiles;
    const int64_t base = lin ? ((int64_t)tile - col_tiles) * T : col_start + (int64_t)tile * T;
    const int64_t end = lin ? n_lin : n;
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t i = base + r * BLK + tid;
      live[r] = (tile < total) && (i < end);
      if (live[r]) {
        if constexpr (KW == 2 && NW == 4) {
          if (!lin && a.rows64) {
            // the row's 48 live bytes as three 16-byte loads through L1 (separate
            // per-field streaming loads re-fetched sectors: 10.7 GB read for 6.4)
            const uint8_t* rp = a.col.key[0] + i * a.col.kstride[0];
            const ulonglong2 A = __ldg((const ulonglong2*)rp);
            const ulonglong2 Bv = __ldg((const ulonglong2*)(rp + 16));
            const ulonglong2 C = __ldg((const ulonglong2*)(rp + 32));
            k[r][0] = A.x;
            k[r][1] = ((uint64_t)(uint32_t)A.y) << 32;  // col_key's int32 key word
            v[r][0] = Bv.x;
            v[r][1] = Bv.y;
            v[r][2] = C.x;
            v[r][3] = C.y;
            continue;
          }
        }
        col_key<KW>(lin ? a.lin : a.col, i, k[r]);
        col_vals<NW>(lin ? a.lin : a.col, i, v[r]);
      }
    }
  };
  auto put = [&](uint32_t pg, uint32_t slot, const uint64_t (&k)[KW], const uint64_t (&v)[NW]) {
    if (pg >= 0xFFFFFFu) return;
    uint64_t* d = pool + ((size_t)pg * (8192 / 8) + (size_t)slot * RW);
    uint64_t w[RW];
#pragma unroll
    for (int q = 0; q < KW; q++) w[q] = k[q];
#pragma unroll
    for (int q = 0; q < NW; q++) w[KW + q] = v[q];
    if constexpr (RW % 2 == 0) {
#pragma unroll
      for (int q = 0; q < RW; q += 2) __stcg((ulonglong2*)(d + q), make_ulonglong2(w[q], w[q + 1]));
    } else {
#pragma unroll
      for (int q = 0; q < RW; q++) __stcg((unsigned long long*)d + q, (unsigned long long)w[q]);
    }
  };

  if (tid == 0) {
    s_sb[0] = s_sb[1] = s_su[0] = s_su[1] = s_sc[0] = s_sc[1] = 0;
    s_grab[0] = atomicAdd(a.tile_counter, 1ull);
    s_grab[1] = atomicAdd(a.tile_counter, 1ull);
  }
  __syncthreads();
  unsigned long long cur = s_grab[0], nxt = s_grab[1];
  uint64_t kc[R][KW], vc[R][NW];
  bool lc[R];
  load_tile(cur, kc, vc, lc);

  uint32_t c_hit = 0, c_rec = 0, c_sp = 0;
  int par = 0;
  while (cur < total) {
    unsigned long long g_next = 0;
    uint32_t ref_first = 0;
    bool refill = false;
    if (tid == 0) {
      g_next = atomicAdd(a.tile_counter, 1ull);
      const int q = par ^ 1;
      refill = a.stash && s_su[q] >= s_sc[q];
      if (refill) ref_first = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
    }
    uint64_t kn[R][KW], vn[R][NW];
    bool ln[R];
    load_tile(nxt, kn, vn, ln);
    uint32_t pend = 0, pidx[R];
    int part[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      pidx[r] = 0;
      part[r] = 0;
      if (!lc[r]) continue;
      c_rec++;
      const bool sent = is_sentinel<KW>(kc[r]);
      const uint64_t h = hash_key<KW>(kc[r], a.t.seed);
      part[r] = sent ? 0 : (int)reduce32(h, (uint32_t)P);
      bool posv = true;
      if (nbw && !sent) {
        const uint64_t bits = bloom_bits(h);
        posv = (sbloom[bloom_block(h, a.bloom.mask)] & bits) == bits;
      }
      if (posv) {  // rare: resolve inline against the frozen table
        int res = R_MISS;
        int64_t sl;
        if (sent) {
          sl = gt_escape<KW>(a.t, false, cc, res);
        } else {
          const uint64_t b = h & a.t.bmask;
          uint64_t w[4];
          ld_bucket(a.t.keys, b, w);
          sl = gt_resolve<KW>(a.t, kc[r], b, w, false, cc, res);
        }
        if (res == R_HIT) {
          Upd<PG>::template g<NW>(a.t.states, a.t.fstride, (uint64_t)sl * a.t.sstride, 0, s_fd, ns, vc[r]);
          c_hit++;
          continue;
        }
      }
      c_sp++;
      const int p = part[r];
      const uint32_t idx = atomicAdd(&cnt[p], 1u);
      const uint32_t j = idx / S, slot = idx - j * S;
      uint32_t* ep = &ent[p * NE + (j & (NE - 1))];
      uint32_t pg;
      if (slot == 0) {
        const uint32_t off = atomicAdd(&s_su[par], 1u);
        if (off < s_sc[par]) {
          pg = s_sb[par] + off;
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
        }
        *(volatile uint32_t*)ep = (pg << 8) | (j & 0xFFu);
      } else {
        const uint32_t e = *(volatile uint32_t*)ep;
        pg = ((e & 0xFFu) == (j & 0xFFu)) ? (e >> 8) : 0xFFFFFFFFu;
      }
      if (pg == 0xFFFFFFFFu) {
        pend |= 1u << r;
        pidx[r] = idx;
      } else {
        put(pg, slot, kc[r], vc[r]);
      }
    }
    if (tid == 0) {
      s_grab[par] = g_next;
      if (refill) {
        const int q = par ^ 1;
        for (uint32_t x = min(s_su[q], s_sc[q]); x < s_sc[q]; x++) a.pool.page_set[s_sb[q] + x] = -1;
        const bool fits = ref_first + (uint32_t)a.stash <= a.pool.capacity;
        if (!fits)
          for (uint32_t x = ref_first; x < min(ref_first + (uint32_t)a.stash, a.pool.capacity); x++)
            a.pool.page_set[x] = -1;
        s_sb[q] = ref_first;
        s_sc[q] = fits ? (uint32_t)a.stash : 0u;
        s_su[q] = 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; r++) {
      if (!((pend >> r) & 1u)) continue;
      const uint32_t idx = pidx[r], j = idx / S;
      const uint32_t e = ent[part[r] * NE + (j & (NE - 1))];
      if ((e & 0xFFu) != (j & 0xFFu)) {
        atomicExch(a.pool.overflow, 3u);  // cannot happen: the allocation precedes the barrier
        continue;
      }
      put(e >> 8, idx - j * S, kc[r], vc[r]);
    }
    cur = nxt;
    nxt = s_grab[par];
    par ^= 1;
#pragma unroll
    for (int r = 0; r < R; r++) {
      lc[r] = ln[r];
#pragma unroll
      for (int q = 0; q < KW; q++) kc[r][q] = kn[r][q];
#pragma unroll
      for (int q = 0; q < NW; q++) vc[r][q] = vn[r][q];
    }
  }
  __syncthreads();
  for (int p = tid; p < P; p += BLK) {
    const uint32_t c = cnt[p];
    if (!c) continue;
    const uint32_t j = (c - 1) / S;
    const uint32_t e = ent[p * NE + (j & (NE - 1))];
    if ((e >> 8) < 0xFFFFFFu) a.pool.page_fill[e >> 8] = (int32_t)(c - j * S);
  }
  for (int q = 0; q < 2; q++)
    for (uint32_t x = min(s_su[q], s_sc[q]) + tid; x < s_sc[q]; x += BLK) a.pool.page_set[s_sb[q] + x] = -1;
  if (c_sp) atomicExch(&a.t.hdr->frozen, 1);
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

}  // namespace aggb
