// pass.cuh — the two record-streaming kernels of the hot path (sm_100a).
//
//   k_pass   level-0 pass over a batch against the L2-resident table
//            (_kernels.py k_table_insert :353-392 / k_pp_probe :917-962 /
//            k_hh_push :865-914), spilling misses to per-partition HBM pages
//   k_child  one recursion level: each CTA aggregates one spilled partition
//            in a shared-memory table (hybrid.py:244-277 _drain_runs child)
//
// Both are templated on a field program PG (device.cuh): PS<...> for the
// benchmark specs (straight-line updates), PD for any other spec.
#pragma once
#include "kernels.cuh"

namespace aggb {

struct PassArgs {
  DevSpec sp;
  int32_t mode;
  GTable t;
  // source 1: columnar batch rows [start, n), start = min(n, *start_tiles * start_T)
  ColSrc col;
  int32_t col_dense;                      // all key/value columns 8-byte, stride 8
  int32_t col_kind;                       // 0 raw payload, 1 native partial states
  const unsigned long long* start_tiles;  // nullable
  int64_t start_T;
  // source 2: SoA list (deferred / overflow records) described as dense columns
  ColSrc lin;                             // lin.nv = payload words of the list
  const unsigned long long* lin_count;    // nullable -> no list
  int32_t lin_kind;                       // 0 raw payload, 1 native partial
  // spill target
  PagePool pool;
  SpillSet ss;
  int32_t group;                          // records per whole-sector group (4 / gcd(rw, 4))
  // ROUTE (original_hh): u32 part hash < cut0 -> partition 0 (table)
  uint32_t cut0;
  uint64_t part_seed;
  // PROBE: bloom filter of the frozen resident keys (copied into SMEM)
  Bloom bloom;
  // FILL deferral target (raw records, SoA, KW + nv words)
  uint64_t* defer;
  int64_t defer_stride;
  unsigned long long* defer_count;
  unsigned long long* tile_counter;
  unsigned long long* stats;
  int32_t stash;                          // pages per CTA-local page-stash refill (0: global atomics only)
  int32_t cache_log2;                     // FILL, one-word keys: SMEM pre-aggregation slots (0: off)
  uint32_t cap_chunk;                     // table reservations per CTA chunk (0: exact path only)
  unsigned long long cap_chunked;         // capacity handed out in chunks (kernels.cuh CapCache)
  // two-phase PROBE (probe.cuh, k_probe PM_SCAN / PM_RESOLVE)
  uint64_t* cand;                         // bloom positives: NREG regions of keys, then NREG of values
  int64_t cand_stride;                    // records per region
  unsigned long long* cand_count;         // [NREG]
  uint2* chains;                          // per (CTA, partition): {records claimed, page of the last claim}
  int32_t pairs;                          // k_probe: sector pairs on (shared memory permitting)
  const uint64_t* hot;                    // heavy-hitter keys (k_hot_sample): hot[0..7] keys, hot[8] count
  int32_t rows64;                         // k_probe_w: columns are C5's 64-byte rows (k0 i64 | k1 i32 | v0..v3 at +16)
  const uint8_t* dd_spilled;              // MODE_DD: partitions destaged so far (their records spill raw)
};

// ---------------------------------------------------------------------------
// Heavy-hitter tier (k_pass NH > 0; in-memory and L2-capped plans of one-word
// keys).  Under Zipf s = 1.5 (C3) the hottest key is ~38% of the records and
// the next few several percent each: in the SMEM pre-aggregation tier every CTA
// serialises on a handful of shared addresses (f64 ADD is a CAS loop there;
// ncu: 60% of the FILL's stalls).  k_hot_sample finds up to 8 keys above 0.4% of
// a strided sample.  k_pass gives every thread a private accumulator column per
// hot key in shared memory (no atomics, no contention), reached through a
// 64-entry directory indexed by the record's table hash; a record takes it once
// its key is known resident in this CTA (slot resolved through the table, as
// for the SMEM tier).  At exit the columns are warp-reduced and merged into
// the table with one L2 update per warp and field.
// ---------------------------------------------------------------------------
constexpr int HOT_MAX = 8;
constexpr int HOT_DIR = 64;  // directory entries (power of two)
template <class PG>
struct HotOps {
  static constexpr int N = 1;
  static __device__ __forceinline__ uint32_t desc(int) { return 0; }
  template <int NWT>
  static __device__ __forceinline__ void add(uint64_t*, int, int, const uint64_t (&)[NWT]) {}
};
template <uint32_t... F>
struct HotOps<PS<F...>> {
  static constexpr int N = sizeof...(F);
  static __device__ __forceinline__ uint32_t desc(int j) {
    constexpr uint32_t fd[N] = {F...};
    return fd[j];
  }
  // col: this thread's column of hot key q (field j at col[j * stride])
  template <int NWT>
  static __device__ __forceinline__ void add(uint64_t* col, int stride, int kind, const uint64_t (&v)[NWT]) {
    constexpr uint32_t fd[N] = {F...};
#pragma unroll
    for (int j = 0; j < N; j++)
      col[j * stride] = merge_word(col[j * stride], contrib_fd<NWT>(fd[j], kind, j, v), fd[j] & 3, (fd[j] >> 2) & 3);
  }
};
// dynamic shared memory of the tier: directory keys, directory hot index, slots, accumulators
template <class PG>
constexpr size_t hot_smem(int blk) {
  return HOT_DIR * 8 + HOT_DIR * 4 + HOT_MAX * 8 + (size_t)HOT_MAX * HotOps<PG>::N * blk * 8;
}

// one CTA: count the keys of a strided sample in a shared-memory table, then
// pick up to 8 keys seen at least min_count times, most frequent first
constexpr int HOT_SLOTS = 2048;
__global__ void __launch_bounds__(1024) k_hot_sample(ColSrc c, int64_t n, int64_t sample, uint32_t min_count,
                                                     uint64_t* out) {
  __shared__ unsigned long long sk[HOT_SLOTS];
  __shared__ uint32_t sc[HOT_SLOTS];
  __shared__ unsigned long long s_best[32];
  const int tid = threadIdx.x;
  for (int i = tid; i < HOT_SLOTS; i += blockDim.x) {
    sk[i] = EMPTY;
    sc[i] = 0;
  }
  __syncthreads();
  const int64_t step = sample > 0 ? (n / sample > 1 ? n / sample : 1) : 1;
  for (int64_t q = tid; q < sample; q += blockDim.x) {
    const int64_t i = q * step;
    if (i >= n) break;
    uint64_t k[1];
    col_key<1>(c, i, k);
    if (k[0] == EMPTY) continue;
    uint32_t b = (uint32_t)fmix64(k[0]) & (HOT_SLOTS - 1);
    for (int t = 0; t < 16; t++, b = (b + 1) & (HOT_SLOTS - 1)) {
      unsigned long long prev = sk[b];
      if (prev == EMPTY) prev = atomicCAS(&sk[b], EMPTY, (unsigned long long)k[0]);
      if (prev == EMPTY || prev == k[0]) {
        atomicAdd(&sc[b], 1u);
        break;
      }
    }
  }
  if (tid == 0) out[HOT_MAX + 1] = 0;
  __syncthreads();
  int found = 0;
  for (int r = 0; r < HOT_MAX; r++) {
    unsigned long long best = 0;  // count << 32 | slot
    for (int i = tid; i < HOT_SLOTS; i += blockDim.x)
      if (sc[i] >= min_count) best = max(best, ((unsigned long long)sc[i] << 32) | (unsigned)i);
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((tid & 31) == 0) s_best[tid >> 5] = best;
    __syncthreads();
    if (tid < 32) {
      best = tid < (int)(blockDim.x >> 5) ? s_best[tid] : 0ull;
      for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (tid == 0) {
        if (best >> 32) {
          out[HOT_MAX + 1] += best >> 32;  // sample records the hot keys cover
          out[found] = sk[(uint32_t)best];
          sc[(uint32_t)best] = 0;
        }
        s_best[0] = best;
      }
    }
    __syncthreads();
    const bool any = (s_best[0] >> 32) != 0;
    __syncthreads();
    if (!any) break;
    found++;
  }
  if (tid == 0) {
    for (int r = found; r < HOT_MAX; r++) out[r] = EMPTY;
    out[HOT_MAX] = (uint64_t)found;
  }
}


template <int KW, int NWT>
__device__ __forceinline__ void load_rec(const ColSrc& c, bool dense, int nv, int64_t i, uint64_t (&k)[KW],
                                         uint64_t (&v)[NWT]) {
  if (dense) {
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = (uint64_t)__ldcs((const long long*)c.key[w] + i);
#pragma unroll
    for (int w = 0; w < NWT; w++) v[w] = (w < nv) ? (uint64_t)__ldcs((const long long*)c.val[w] + i) : 0ull;
  } else {
    col_key<KW>(c, i, k);
#pragma unroll
    for (int w = 0; w < NWT; w++) {
      if (w < nv) {
        const uint8_t* p = c.val[w] + i * c.vstride[w];
        v[w] = (c.vty[w] == TY_I32) ? (uint64_t)(long long)__ldcs((const int*)p) : (uint64_t)__ldcs((const long long*)p);
      } else {
        v[w] = 0ull;
      }
    }
  }
}

// write one record (key words + nw payload words) at slot `slot` of an AoS page
template <int KW, int NWT>
__device__ __forceinline__ void put_rec(uint64_t* dst, const uint64_t (&k)[KW], const uint64_t (&v)[NWT], int nw) {
#pragma unroll
  for (int w = 0; w < KW; w++) dst[w] = k[w];
#pragma unroll
  for (int w = 0; w < NWT; w++)
    if (w < nw) dst[KW + w] = v[w];
}

// ---------------------------------------------------------------------------
// k_pass
//
// Persistent, tile-scheduled.  Per tile of T = R * BLK records:
//  [A] issue the first-bucket loads of the current records, prefetch the next
//      tile's records into registers, then resolve: hits aggregate with L2
//      atomics (RED), misses get a rank in their partition (SMEM atomic);
//  [B] one thread per touched partition reserves page space in the CTA's own
//      page for that partition (one global atomic per new page) for the
//      records that complete whole 32-byte sectors, and copies the partition's
//      sector residual (< group records, kept in SMEM) in front of them;
//  [C] every thread writes its records from registers: into the page when
//      they complete a sector group, otherwise into the SMEM residual.
// Records therefore reach L2 as complete sectors within one tile, so L2
// never evicts a half-written sector (which ECC DRAM would read-modify-write).
// ---------------------------------------------------------------------------

template <int KW, int NWT, int R, int BLK, int MINB, class PG, int NH = 0>
__global__ void __launch_bounds__(BLK, MINB) k_pass(PassArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = BLK, tid = threadIdx.x;
  const int T = R * BLK;
  const bool spills = (a.mode != MODE_FILL);
  const int P = spills ? a.ss.nparts : 1;
  const int S = spills ? a.ss.per_page : 1;
  const int G = spills ? a.group : 1;
  const int rw = spills ? a.ss.rw : 1;
  const int nw = rw - KW;

  const bool use_bloom = (a.mode == MODE_PROBE) && a.bloom.words != nullptr;
  const int nbw = use_bloom ? (int)a.bloom.mask + 1 : 0;
  uint64_t* sbloom = (uint64_t*)smem;                        // nbw words
  uint64_t* resid = sbloom + nbw;                            // P * (G - 1) * rw words
  uint32_t* hist = (uint32_t*)(resid + (size_t)P * (G - 1) * rw);
  int32_t* pcur = (int32_t*)(hist + P);
  int32_t* pfill = pcur + P;
  int32_t* bpg = pfill + P;
  int32_t* bslot = bpg + P;
  int32_t* pnew = bslot + P;
  uint32_t* rcnt = (uint32_t*)(pnew + P);
  uint32_t* rprev = rcnt + P;
  uint32_t* emitn = rprev + P;
  uint16_t* touched = (uint16_t*)(emitn + P);                // P: partitions touched by the tile
  // SMEM pre-aggregation tier (FILL / ROUTE): per-CTA cache of resident keys.
  // A key enters it only after its global lookup/insert succeeded (slot cgs);
  // later records of that key update the cache's states in shared memory, which
  // merge into the global slot at exit.  Hot (skewed) keys stop contending on
  // one L2 address; the table's capacity semantics are untouched.
  const int CH = (KW == 1 && a.cache_log2) ? 1 << a.cache_log2 : 0;
  uint64_t* ckeys = (uint64_t*)(((uintptr_t)(touched + P) + 15) & ~(uintptr_t)15);  // CH
  uint64_t* cst = ckeys + CH;                                                        // ns * CH
  uint32_t* cgs = (uint32_t*)(cst + (size_t)a.sp.ns * CH);                           // CH
  __shared__ int s_ccount;
  __shared__ uint32_t s_ntouched[2];  // by tile parity: A fills one while the other is reset
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_grab, s_defer_base;
  __shared__ uint32_t s_ndefer;
  __shared__ uint32_t s_sbase, s_sused, s_scap;  // CTA-local page stash [s_sbase, s_sbase + s_scap)
  __shared__ int s_avail;                         // table reservations given back in this CTA
  __shared__ unsigned s_commits;                  // keys this CTA inserted
  __shared__ int s_refused, s_refilling;
  const CapCache cc{&s_avail, &s_commits, &s_refused, &s_refilling, a.cap_chunk, a.cap_chunked};
  __shared__ unsigned long long s_cnt[ST_NSTATS];

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  for (int p = tid; p < P; p += B) {
    hist[p] = 0;
    pcur[p] = -1;
    pfill[p] = S;
    rcnt[p] = 0;
  }
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  for (int i = tid; i < nbw; i += B) sbloom[i] = __ldcg((const unsigned long long*)a.bloom.words + i);
  for (int i = tid; i < CH; i += B) {
    ckeys[i] = EMPTY;
    for (int j = 0; j < a.sp.ns; j++) cst[(size_t)j * CH + i] = state_identity(a.sp.op[j], a.sp.ty[j]);
  }
  if (tid == 0) s_ccount = 0;
  // heavy-hitter tier (NH > 0): directory, resolved slots, per-thread accumulator columns
  using HO = HotOps<PG>;
  uint64_t* hdk = (uint64_t*)(((uintptr_t)(cgs + CH) + 15) & ~(uintptr_t)15);  // HOT_DIR keys
  int32_t* hdi = (int32_t*)(hdk + HOT_DIR);                                     // HOT_DIR hot index
  long long* hsl = (long long*)(hdi + HOT_DIR);                                 // HOT_MAX slots
  uint64_t* hacc = (uint64_t*)(hsl + HOT_MAX);                                  // [HOT_MAX][N][BLK]
  if constexpr (NH > 0) {
    for (int i = tid; i < HOT_DIR; i += B) {
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
    if (tid == 0) {  // hot keys into the directory (a colliding later key is left out)
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
  const int64_t n = a.col.n;
  const int64_t col_start =
      a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t n_lin = a.lin_count ? (int64_t)*a.lin_count : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (n_lin + T - 1) / T);
  const bool use_table = (a.mode == MODE_FILL || a.mode == MODE_PROBE || a.mode == MODE_ROUTE || a.mode == MODE_DD);
  const bool insert = (a.mode != MODE_PROBE);
  const int nvc = a.col.nv, nvl = a.lin.nv;

  auto grab = [&]() -> unsigned long long {
    if ((a.mode == MODE_FILL || a.mode == MODE_DD) && *(volatile int*)&a.t.hdr->frozen) return ~0ull;
    return atomicAdd(a.tile_counter, 1ull);
  };
  auto load_tile = [&](unsigned long long tile, uint64_t (&k)[R][KW], uint64_t (&v)[R][NWT], bool (&live)[R]) {
    const bool fc = (int64_t)tile < col_tiles;
    const int64_t base = fc ? col_start + (int64_t)tile * T : ((int64_t)tile - col_tiles) * T;
    const int64_t end = fc ? n : n_lin;
#pragma unroll
    for (int r = 0; r < R; r++) {
      int64_t i = base + (int64_t)r * B + tid;
      live[r] = (tile < total) && (i < end);
      if (live[r]) {
        if (fc) load_rec<KW, NWT>(a.col, a.col_dense != 0, nvc, i, k[r], v[r]);
        else load_rec<KW, NWT>(a.lin, true, nvl, i, k[r], v[r]);
      }
    }
  };
  // emission position -> (page, slot) for partition p in this tile
  auto emit_at = [&](int p, int pos, int32_t& pg, int& slot) -> bool {
    int room = S - bslot[p];
    if (pos < room) {
      pg = bpg[p];
      slot = bslot[p] + pos;
      return pg >= 0;
    }
    if (pnew[p] < 0) return false;
    int j = pos - room;
    pg = pnew[p] + j / S;
    slot = j % S;
    return true;
  };

  if (tid == 0) {
    s_ndefer = 0;
    s_avail = 0;
    s_commits = 0;
    s_refused = 0;
    s_refilling = 0;
    s_sbase = s_sused = s_scap = 0;
    s_ntouched[0] = s_ntouched[1] = 0;
    s_grab = grab();
  }
  __syncthreads();
  unsigned long long cur = s_grab;
  __syncthreads();
  if (tid == 0) s_grab = (cur < total) ? grab() : ~0ull;
  uint64_t kc[R][KW], vc[R][NWT];
  bool lc[R];
  load_tile(cur, kc, vc, lc);
  __syncthreads();
  unsigned long long nxt = s_grab;

  uint32_t c_hit = 0, c_ins = 0, c_rec = 0, c_sp = 0, c_def = 0;
  int par = 0;
  while (cur < total) {
    const int kind = ((int64_t)cur < col_tiles) ? a.col_kind : a.lin_kind;
    // page-stash refill: phase A never overlaps phase B (the only consumer),
    // the atomic's latency hides behind this warp's phase A
    const bool refill = spills && a.stash && tid == 0 && s_sused >= s_scap;  // refill only when used up
    uint32_t ref_first = 0;
    if (refill) ref_first = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
    // ---- [A] first-bucket loads for the current records
    uint64_t bk[R];
    uint64_t bw[R][4];
    int part[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      part[r] = -2;
      if (!lc[r]) continue;
      part[r] = -1;
      if (a.mode == MODE_ROUTE) {
        uint32_t u = (uint32_t)(hash_key<KW>(kc[r], a.part_seed) >> 32);
        if (u >= a.cut0) {
          int pp = 1 + (int)(((uint64_t)(u - a.cut0) * (uint64_t)(P - 1)) / (0x100000000ull - a.cut0));
          part[r] = pp > P - 1 ? P - 1 : pp;
        }
      } else if (a.mode == MODE_GRACE) {
        part[r] = (int)reduce32(hash_key<KW>(kc[r], a.ss.seed), (uint32_t)P);
      } else if (a.mode == MODE_DD) {  // destaged partitions spill raw, the others aggregate
        const int pp = (int)reduce32(hash_key<KW>(kc[r], a.ss.seed), (uint32_t)P);  // GRACE's partition
        if (a.dd_spilled[pp]) part[r] = pp;
      }
      if (use_table && part[r] == -1 && !is_sentinel<KW>(kc[r])) {
        // one 64-bit hash per record at this level: bucket from the low bits,
        // spill partition from the high bits, bloom probe from a remix
        const uint64_t h = hash_key<KW>(kc[r], a.t.seed);
        bk[r] = h;
        if constexpr (NH > 0) {  // heavy hitter with a resolved slot: this thread's column
          const int d = (int)(h >> 58) & (HOT_DIR - 1);
          if (hdk[d] == kc[r][0]) {
            const int q = hdi[d];
            if (*(volatile long long*)&hsl[q] >= 0) {
              HO::template add<NWT>(hacc + (size_t)q * HO::N * BLK + tid, BLK, kind, vc[r]);
              c_rec++;
              c_hit++;
              part[r] = -2;
              continue;
            }
          }
        }
        if (CH) {  // pre-aggregation tier: a cached key never leaves the SM
          const int c0 = (int)(h >> 40) & (CH - 1);
          int hit = -1;
          for (int q = 0; q < 4; q++) {
            const int c = (c0 + q) & (CH - 1);
            const uint64_t ck = *(volatile uint64_t*)&ckeys[c];
            if (ck == kc[r][0]) { hit = c; break; }
            if (ck == EMPTY) break;
          }
          if (hit >= 0) {
            part[r] = -3 - hit;
            continue;
          }
        }
        if (use_bloom) {
          const uint64_t bits = bloom_bits(h);
          if ((sbloom[bloom_block(h, a.bloom.mask)] & bits) != bits) {  // definitely not resident
            part[r] = (int)reduce32(h, (uint32_t)P);
            continue;
          }
        }
        ld_bucket(a.t.keys, h & a.t.bmask, bw[r]);
      }
    }
    // ---- prefetch the next tile while the buckets are in flight
    uint64_t kn[R][KW], vn[R][NWT];
    bool ln[R];
    load_tile(nxt, kn, vn, ln);
    // ---- resolve
    uint32_t tag[R];  // spill: (p << 16 | rank) + 1; defer: 0x80000000 | rank; 0 done
#pragma unroll
    for (int r = 0; r < R; r++) {
      tag[r] = 0;
      int res = R_MISS;
      int64_t s = -1;
      if (part[r] != -2) c_rec++;
      if (part[r] == -1)
        s = is_sentinel<KW>(kc[r]) ? gt_escape<KW>(a.t, insert, cc, res)
                                   : gt_resolve<KW>(a.t, kc[r], bk[r] & a.t.bmask, bw[r], insert, cc, res);
      __syncwarp();  // reconverge after the divergent probe before the updates
      if (part[r] <= -3) {  // cached key: shared-memory update
        Upd<PG>::template sm<NWT>(cst, CH, -3 - part[r], kind, s_fd, ns, vc[r]);
        c_hit++;
        part[r] = -2;
      }
      if (part[r] == -1) {
        if (res == R_HIT || res == R_INSERTED) {
          Upd<PG>::template g<NWT>(a.t.states, a.t.fstride, (uint64_t)s * a.t.sstride, kind, s_fd, ns, vc[r]);
          c_hit += (res == R_HIT);
          c_ins += (res == R_INSERTED);
          part[r] = -2;
          if constexpr (NH > 0) {
            const int d = (int)(bk[r] >> 58) & (HOT_DIR - 1);
            if (hdk[d] == kc[r][0] && !is_sentinel<KW>(kc[r])) *(volatile long long*)&hsl[hdi[d]] = s;
          }
          // resident now: cache the key for its later records (first come, no eviction)
          if (CH && !is_sentinel<KW>(kc[r]) && *(volatile int*)&s_ccount < (CH * 3) / 4) {
            const int c0 = (int)(bk[r] >> 40) & (CH - 1);
            for (int q = 0; q < 4; q++) {
              const int c = (c0 + q) & (CH - 1);
              const unsigned long long prev = atomicCAS((unsigned long long*)&ckeys[c], EMPTY, kc[r][0]);
              if (prev == EMPTY) {
                cgs[c] = (uint32_t)s;
                atomicAdd(&s_ccount, 1);
                break;
              }
              if (prev == kc[r][0]) break;
            }
          }
        } else if (res == R_MISS) {
          part[r] = is_sentinel<KW>(kc[r]) ? 0 : (int)reduce32(bk[r], (uint32_t)P);
        } else if (a.mode == MODE_FILL || a.mode == MODE_DD) {
          tag[r] = 0x80000000u | atomicAdd(&s_ndefer, 1u);
          c_def++;
          part[r] = -2;
        } else {
          part[r] = 0;  // ROUTE overflow: partition 0 spills raw (hybrid.py:431-451)
        }
      }
      if (part[r] >= 0) {
        uint32_t rank = atomicAdd(&hist[part[r]], 1u);
        if (rank == 0) touched[atomicAdd(&s_ntouched[par], 1u)] = (uint16_t)part[r];
        tag[r] = (((uint32_t)part[r] << 16) | rank) + 1u;
        c_sp++;
      }
      __syncwarp();
    }
    if (refill) {
      for (uint32_t q = min(s_sused, s_scap); q < s_scap; q++) a.pool.page_set[s_sbase + q] = -1;  // leftover
      if (ref_first + (uint32_t)a.stash <= a.pool.capacity) {
        s_sbase = ref_first;
        s_scap = (uint32_t)a.stash;
      } else {
        for (uint32_t q = ref_first; q < min(ref_first + (uint32_t)a.stash, a.pool.capacity); q++)
          a.pool.page_set[q] = -1;
        s_scap = 0;
      }
      s_sused = 0;
    }
    __syncthreads();
    // ---- [B] per touched partition: reserve whole sector groups, drain the residual
    if (spills) {
      const int nt = (int)s_ntouched[par];
      for (int ti = tid; ti < nt; ti += B) {
        const int p = touched[ti];
        int c = (int)hist[p];
        hist[p] = 0;
        int r0 = (int)rcnt[p];
        int t = r0 + c;
        int e = (t / G) * G;
        rprev[p] = (uint32_t)r0;
        emitn[p] = (uint32_t)e;
        rcnt[p] = (uint32_t)(t - e);
        if (!e) continue;
        int room = S - pfill[p];
        bpg[p] = pcur[p];
        bslot[p] = pfill[p];
        pnew[p] = -1;
        if (e > room) {
          int need = (e - room + S - 1) / S;
          // single pages come from the CTA's stash (a taker past its end takes
          // nothing from it); runs of pages are contiguous: one global atomic
          uint32_t first = 0xFFFFFFFFu;
          if (need == 1) {
            const uint32_t off = atomicAdd(&s_sused, 1u);
            if (off < s_scap) first = s_sbase + off;
          }
          if (first == 0xFFFFFFFFu) first = atomicAdd(a.pool.next_page, (uint32_t)need);
          if (first + need > a.pool.capacity) {
            atomicExch(a.pool.overflow, 1u);
            pcur[p] = -1;
            pfill[p] = S;
          } else {
            for (int q = 0; q < need; q++) {
              a.pool.page_part[first + q] = p;
              a.pool.page_set[first + q] = a.ss.id;
              a.pool.page_fill[first + q] = S;
            }
            pnew[p] = (int32_t)first;
            pcur[p] = (int32_t)(first + need - 1);
            pfill[p] = (e - room) - (need - 1) * S;
          }
          if (bpg[p] >= 0) a.pool.page_fill[bpg[p]] = S;
        } else {
          pfill[p] += e;
        }
        // the residual records lead this tile's emission
        for (int q = 0; q < r0; q++) {
          int32_t pg;
          int slot;
          if (!emit_at(p, q, pg, slot)) continue;
          uint64_t* dst = (uint64_t*)page_ptr(a.pool, (uint32_t)pg) + (size_t)slot * rw;
          const uint64_t* src = resid + ((size_t)p * (G - 1) + q) * rw;
          for (int w = 0; w < rw; w++) dst[w] = src[w];
        }
      }
    }
    if (tid == 0) {
      if (s_ndefer) {
        s_defer_base = atomicAdd(a.defer_count, (unsigned long long)s_ndefer);
        // deferral pressure (transient refusals while the table is not full):
        // freeze early so the rest of the batch goes to PROBE — budget-safe
        if (s_defer_base + s_ndefer > (unsigned long long)a.defer_stride / 2) atomicExch(&a.t.hdr->frozen, 1);
        s_ndefer = 0;
      }
      s_grab = (nxt < total) ? grab() : ~0ull;
      s_ntouched[par ^ 1] = 0;  // last read in the previous tile's phase B
    }
    __syncthreads();
    // ---- [C] write spilled / deferred records from registers
#pragma unroll
    for (int r = 0; r < R; r++) {
      uint32_t tg = tag[r];
      if (!tg) continue;
      if (tg & 0x80000000u) {
        int64_t d = (int64_t)s_defer_base + (tg & 0x7FFFFFFFu);
        if (d >= a.defer_stride) {  // cannot happen with the early freeze; never write out of bounds
          atomicExch(a.pool.overflow, 2u);
          continue;
        }
#pragma unroll
        for (int w = 0; w < KW; w++) a.defer[w * a.defer_stride + d] = kc[r][w];
#pragma unroll
        for (int w = 0; w < NWT; w++)
          if (w < nvc) a.defer[(KW + w) * a.defer_stride + d] = vc[r][w];
        continue;
      }
      tg -= 1u;
      int p = (int)(tg >> 16);
      int pos = (int)rprev[p] + (int)(tg & 0xFFFFu);
      int e = (int)emitn[p];
      if (pos < e) {
        int32_t pg;
        int slot;
        if (emit_at(p, pos, pg, slot))
          put_rec<KW, NWT>((uint64_t*)page_ptr(a.pool, (uint32_t)pg) + (size_t)slot * rw, kc[r], vc[r], nw);
      } else {
        put_rec<KW, NWT>(resid + ((size_t)p * (G - 1) + (pos - e)) * rw, kc[r], vc[r], nw);
      }
    }
    // ---- rotate
    par ^= 1;
    cur = nxt;
    nxt = s_grab;
#pragma unroll
    for (int r = 0; r < R; r++) {
      lc[r] = ln[r];
#pragma unroll
      for (int w = 0; w < KW; w++) kc[r][w] = kn[r][w];
#pragma unroll
      for (int w = 0; w < NWT; w++) vc[r][w] = vn[r][w];
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
        if ((tid & 31) == 0 && v != state_identity(F & 3, (F >> 2) & 3))
          gupdate(a.t.states + (uint64_t)j * a.t.fstride + (uint64_t)sl * a.t.sstride, F & 3, (F >> 2) & 3, v);
      }
    }
  }
  // merge the pre-aggregation tier into the table (skip identity states: keys cached late)
  for (int i = tid; i < CH; i += B) {
    if (ckeys[i] == EMPTY) continue;
    const uint64_t gs = cgs[i];
    for (int j = 0; j < ns; j++) {
      const uint64_t v = cst[(size_t)j * CH + i];
      const uint32_t F = s_fd[j];
      if (v == state_identity(F & 3, (F >> 2) & 3)) continue;
      gupdate(a.t.states + (uint64_t)j * a.t.fstride + gs * a.t.sstride, F & 3, (F >> 2) & 3, v);
    }
  }
  if (spills)
    for (uint32_t q = min(s_sused, s_scap) + tid; q < s_scap; q += B) a.pool.page_set[s_sbase + q] = -1;
  // drain the residuals (partial sectors, once per partition) and seal the pages
  if (spills) {
    for (int p = tid; p < P; p += B) {
      int r0 = (int)rcnt[p];
      if (r0) {
        if (S - pfill[p] < r0) {
          uint32_t pg = atomicAdd(a.pool.next_page, 1u);
          if (pg >= a.pool.capacity) {
            atomicExch(a.pool.overflow, 1u);
            continue;
          }
          a.pool.page_part[pg] = p;
          a.pool.page_set[pg] = a.ss.id;
          if (pcur[p] >= 0) a.pool.page_fill[pcur[p]] = pfill[p];
          pcur[p] = (int32_t)pg;
          pfill[p] = 0;
        }
        uint64_t* dst = (uint64_t*)page_ptr(a.pool, (uint32_t)pcur[p]) + (size_t)pfill[p] * rw;
        const uint64_t* src = resid + (size_t)p * (G - 1) * rw;
        for (int w = 0; w < r0 * rw; w++) dst[w] = src[w];
        pfill[p] += r0;
      }
      if (pcur[p] >= 0) a.pool.page_fill[pcur[p]] = pfill[p];
    }
  }
  // PROBE spilled records: the resident set is final from now on (a later
  // push's FILL must not insert a key that already went to a partition)
  if (a.mode == MODE_PROBE && c_sp) atomicExch(&a.t.hdr->frozen, 1);
  // counters: warp reduce then one shared atomic per warp
  uint32_t cs[5] = {c_sp, c_hit, c_ins, c_def, c_rec};
  const int ids[5] = {ST_SPILLED, ST_HITS, ST_INSERTS, ST_DEFERRED, ST_RECORDS};
#pragma unroll
  for (int q = 0; q < 5; q++) {
    uint32_t x = cs[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((tid & 31) == 0 && x) atomicAdd(&s_cnt[ids[q]], (unsigned long long)x);
  }
  __syncthreads();
  if (tid < ST_NSTATS && s_cnt[tid]) atomicAdd(&a.stats[tid], s_cnt[tid]);
  if (tid == 0 && s_commits) atomicAdd(&a.t.hdr->committed, (unsigned long long)s_commits);
  if (tid == 0 && s_refused) atomicExch((int*)&a.t.hdr->pad, 1);
}

// ---------------------------------------------------------------------------
// k_child
// ---------------------------------------------------------------------------

struct ChildArgs {
  DevSpec sp;
  PagePool pool;
  SpillSet sets[2];         // pages of item i: sets[0] in [off[2i], off[2i+1]), sets[1] in [off[2i+1], off[2i+2])
  const uint2* plist;       // {page id, records in it}, grouped by item (set 0 pages first)
  const int64_t* item_off;  // [2 * nitems + 1]
  int32_t nitems;
  int32_t slots_log2;       // SMEM table slots
  int32_t cap;              // group capacity (<= budget)
  uint64_t seed;            // slot hash seed of this level
  int32_t nsub;             // sub-passes per item (1: one table holds the partition)
  uint64_t sub_seed;        // sub-pass hash seed (independent of the slot and spill seeds)
  OutBuf out;
  uint64_t* ovf;            // overflow list: native partial records, SoA KW + ns words
  int64_t ovf_stride;
  unsigned long long* ovf_count;
  unsigned long long* item_counter;
  unsigned long long* stats;
};

// One CTA aggregates one spilled partition (a child operator at level + 1,
// hybrid.py:244-277) in a shared-memory table.  Threads map onto (page, slot)
// across B / per_page pages per row and R rows per round; the next round's
// records are prefetched into registers while the current one aggregates.
// There is no barrier per round.  An insert refused because the table is full
// (the child's budget: the reference's TABLE_FULL + freeze) waits until no
// insert is in flight — the key set is then final — and re-probes: resident
// keys aggregate in place, the rest go to the overflow list (next level).
template <int KW, int NWT, int R, class PG, int MINB = 2>
__global__ void __launch_bounds__(512, MINB) k_child(ChildArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = blockDim.x, tid = threadIdx.x;
  const int nslots = 1 << a.slots_log2;
  const int stride = nslots + 1;
  const int ns = a.sp.ns;
  uint64_t* skeys = (uint64_t*)smem;                       // stride * KW
  uint64_t* sst = skeys + (size_t)stride * KW;             // ns * stride
  __shared__ int s_groups[2], s_frozen, s_esc, s_inflight;
  __shared__ unsigned long long s_item;
  __shared__ unsigned long long s_cnt[ST_NSTATS];
  __shared__ uint32_t s_fd[MAX_STATES];
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  uint32_t nrec = 0, novf = 0;

  const int nsub = max(1, a.nsub);
  int sub = nsub - 1;
  for (;;) {
    // an item runs nsub sub-passes, each in a fresh table (one flush each)
    if (++sub == nsub) sub = 0;
    if (tid == 0 && sub == 0) s_item = atomicAdd(a.item_counter, 1ull);
    for (int i = tid; i < stride; i += B) {
#pragma unroll
      for (int w = 0; w < KW; w++) skeys[(size_t)i * KW + w] = EMPTY;
      for (int j = 0; j < ns; j++) sst[(size_t)j * stride + i] = state_identity(a.sp.op[j], a.sp.ty[j]);
    }
    if (tid == 0) {
      s_groups[0] = s_groups[1] = 0;
      s_frozen = 0;
      s_esc = 0;
      s_inflight = 0;
    }
    __syncthreads();
    unsigned long long item = s_item;
    if (item >= (unsigned long long)a.nitems) break;
    for (int sidx = 0; sidx < 2; sidx++) {
      const int64_t qa = a.item_off[2 * item + sidx], qb = a.item_off[2 * item + sidx + 1];
      if (qa >= qb) continue;
      const SpillSet ss = a.sets[sidx];
      const int kind = ss.kind;
      const int nw = ss.rw - KW;
      const int rw = ss.rw;
      // Warp-per-page mapping: warp w takes pages qa + w, qa + w + NWARPS, ...;
      // lane l handles slots l, l + 32, ... of the page (no page search, one
      // base address per page; ~15 records per lane for the ~484-record pages
      // CTA-private chains leave).  The next chunk of R records per lane is
      // prefetched while the current one aggregates; the next page's list
      // entry is loaded one page ahead.
      const int lane = tid & 31, wid = tid >> 5, nwarps = B >> 5;
      auto load_chunk = [&](const uint64_t* pbase, int fill, int s0, uint64_t (&k)[R][KW], uint64_t (&v)[R][NWT],
                            bool (&live)[R]) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int slot = s0 + r * 32 + lane;
          live[r] = slot < fill;
          if (live[r]) {
            const unsigned long long* src = (const unsigned long long*)pbase + (size_t)slot * rw;
#pragma unroll
            for (int w = 0; w < KW; w++) k[r][w] = __ldcs(src + w);
#pragma unroll
            for (int w = 0; w < NWT; w++) v[r][w] = (w < nw) ? (uint64_t)__ldcs(src + KW + w) : 0ull;
          }
        }
      };
      uint2 pe_next = (qa + wid < qb) ? a.plist[qa + wid] : make_uint2(0, 0);
      for (int64_t q = qa + wid; q < qb; q += nwarps) {
        const uint2 pe = pe_next;
        if (q + nwarps < qb) pe_next = a.plist[q + nwarps];
        const uint64_t* pbase = (const uint64_t*)page_ptr(a.pool, pe.x);
        const int fill = (int)pe.y;
        uint64_t kc[R][KW], vc[R][NWT];
        bool lc[R];
        load_chunk(pbase, fill, 0, kc, vc, lc);
        for (int s0 = 0; s0 < fill; s0 += R * 32) {
          uint64_t kn[R][KW], vn[R][NWT];
          bool ln[R];
          load_chunk(pbase, fill, s0 + R * 32, kn, vn, ln);
#pragma unroll
          for (int r = 0; r < R; r++) {
            int res = R_MISS, s = -1;
            if (nsub > 1 && lc[r]) lc[r] = reduce32(hash_key<KW>(kc[r], a.sub_seed), (uint32_t)nsub) == (uint32_t)sub;
            if (lc[r]) {
              nrec++;
              s = stable_lookup<KW>(skeys, nslots, a.cap, kc[r], a.seed, true, s_groups, &s_frozen, &s_esc,
                                    &s_inflight, res);
              if (res == R_REFUSED)
                s = stable_resolve_refused<KW>(skeys, nslots, a.cap, kc[r], a.seed, s_groups, &s_frozen, &s_esc,
                                               &s_inflight, res);
            }
            __syncwarp();  // reconverge after the divergent probe before the updates
            if (res == R_HIT || res == R_INSERTED) {
              Upd<PG>::template sm<NWT>(sst, stride, s, kind, s_fd, ns, vc[r]);
            } else if (lc[r]) {  // not resident: the next recursion level
              unsigned long long d = atomicAdd(a.ovf_count, 1ull);
              novf++;
              if (d < (unsigned long long)a.ovf_stride) {  // past the list: counted, reported by the host
#pragma unroll
                for (int w = 0; w < KW; w++) a.ovf[w * a.ovf_stride + d] = kc[r][w];
                for (int j = 0; j < ns; j++)
                  a.ovf[(KW + j) * a.ovf_stride + d] = contrib_fd<NWT>(s_fd[j], kind, j, vc[r]);
              }
            }
            __syncwarp();
          }
#pragma unroll
          for (int r = 0; r < R; r++) {
            lc[r] = ln[r];
#pragma unroll
            for (int w = 0; w < KW; w++) kc[r][w] = kn[r][w];
#pragma unroll
            for (int w = 0; w < NWT; w++) vc[r][w] = vn[r][w];
          }
        }
      }
    }
    __syncthreads();
    // flush the item's groups: block compaction then one global reservation
    {
      __shared__ unsigned long long s_base;
      __shared__ uint32_t s_wsum[33];
      int per = (stride + B - 1) / B;
      int lo = tid * per, hi = min(stride, lo + per);
      uint32_t mine = 0;
      for (int s = lo; s < hi; s++) {
        uint64_t kk[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) kk[w] = skeys[(size_t)s * KW + w];
        mine += (s == nslots) ? (s_esc != 0) : !is_sentinel<KW>(kk);
      }
      int lane = tid & 31, wid = tid >> 5;
      uint32_t x = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[wid] = x;
      __syncthreads();
      if (tid == 0) {
        uint32_t acc = 0;
        int nwp = (B + 31) >> 5;
        for (int w = 0; w < nwp; w++) {
          uint32_t t2 = s_wsum[w];
          s_wsum[w] = acc;
          acc += t2;
        }
        s_base = acc ? atomicAdd(a.out.count, (unsigned long long)acc) : 0ull;
      }
      __syncthreads();
      int64_t idx = (int64_t)s_base + s_wsum[wid] + (x - mine);
      for (int s = lo; s < hi; s++) {
        uint64_t kk[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) kk[w] = skeys[(size_t)s * KW + w];
        bool occ = (s == nslots) ? (s_esc != 0) : !is_sentinel<KW>(kk);
        if (!occ) continue;
        uint64_t st[MAX_STATES];
        for (int j = 0; j < ns; j++) st[j] = sst[(size_t)j * stride + s];
        emit_group<KW>(a.sp, a.out, idx++, kk, st);
      }
    }
    __syncthreads();
  }
  uint32_t cs[2] = {nrec, novf};
  const int ids[2] = {ST_RECORDS, ST_OVERFLOW};
#pragma unroll
  for (int q = 0; q < 2; q++) {
    uint32_t x = cs[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((tid & 31) == 0 && x) atomicAdd(&s_cnt[ids[q]], (unsigned long long)x);
  }
  __syncthreads();
  if (tid < ST_NSTATS && s_cnt[tid]) atomicAdd(&a.stats[tid], s_cnt[tid]);
}

}  // namespace aggb

namespace aggb {

// ---------------------------------------------------------------------------
// k_split: one more grace level for partitions too large for a child table
// (hybrid.py:281-318 grace partitioning, fresh seed per level).  A CTA takes a
// spilled partition (item) and re-partitions it into S sub-partitions:
//   1. count the item's records per sub-partition (keys only),
//   2. reserve whole pages per sub-partition (one global atomic each), so a
//      sub-partition is a page-aligned run the children read like any other,
//   3. scatter: lanes with the same sub-partition claim consecutive slots
//      (match_any + one shared atomic), so a warp's record writes coalesce.
// The item is read twice; a child would otherwise read it once per sub-pass.
// ---------------------------------------------------------------------------

struct SplitArgs {
  PagePool pool;
  SpillSet in;              // input set (one live set)
  const uint2* plist;       // {page id, records} grouped by item
  const int64_t* item_off;  // [2 * nitems + 1] (child layout: set 0 range, set 1 range)
  int32_t nitems;
  int32_t S;                // sub-partitions per item (<= 1024)
  uint64_t sub_seed;
  SpillSet out;             // output set: partition = item * S + sub
  unsigned long long* item_counter;
};

// RWC: record width known at compile time (registers), 0: any width (per-word copies)
template <int KW, int RWC>
__global__ void __launch_bounds__(512) k_split(SplitArgs a) {
  __shared__ uint32_t s_hist[1024], s_base[1024], s_cur[1024];
  __shared__ unsigned long long s_item;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const int S = a.S, rw = RWC ? RWC : a.in.rw, per = a.out.per_page;
  constexpr int NR = RWC ? RWC : KW;  // words held in registers
  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.item_counter, 1ull);
    for (int s = tid; s < S; s += blockDim.x) s_hist[s] = s_cur[s] = 0;
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= (unsigned long long)a.nitems) break;
    const int64_t qa = a.item_off[2 * item], qb = a.item_off[2 * item + 2];
    // 1. histogram
    for (int64_t q = qa + wid; q < qb; q += nwarps) {
      const uint2 pe = a.plist[q];
      const uint64_t* pb = (const uint64_t*)page_ptr(a.pool, pe.x);
      for (int slot = lane; slot < (int)pe.y; slot += 32) {
        uint64_t k[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) k[w] = __ldcg(pb + (size_t)slot * rw + w);
        atomicAdd(&s_hist[reduce32(hash_key<KW>(k, a.sub_seed), (uint32_t)S)], 1u);
      }
    }
    __syncthreads();
    // 2. whole pages per sub-partition
    for (int s = tid; s < S; s += blockDim.x) {
      const uint32_t n = s_hist[s];
      const uint32_t np = (n + per - 1) / per;
      uint32_t b = 0xFFFFFFFFu;
      if (np) {
        b = atomicAdd(a.pool.next_page, np);
        if (b + np > a.pool.capacity) {
          atomicExch(a.pool.overflow, 1u);
          b = 0xFFFFFFFFu;
        } else {
          const int part = (int)(item * (unsigned long long)S + s);
          for (uint32_t x = 0; x < np; x++) {
            a.pool.page_part[b + x] = part;
            a.pool.page_set[b + x] = a.out.id;
            a.pool.page_fill[b + x] = (int32_t)min((uint32_t)per, n - x * per);
          }
        }
      }
      s_base[s] = b;
    }
    __syncthreads();
    // 3. scatter
    for (int64_t q = qa + wid; q < qb; q += nwarps) {
      const uint2 pe = a.plist[q];
      const uint64_t* pb = (const uint64_t*)page_ptr(a.pool, pe.x);
      for (int s0 = 0; s0 < (int)pe.y; s0 += 32) {
        const int slot = s0 + lane;
        const bool live = slot < (int)pe.y;
        // the whole record in registers (16-byte loads when records are 16-byte
        // aligned: streaming per-word loads re-fetched each line from L2)
        uint64_t rec[NR];
        const uint64_t* src = pb + (size_t)slot * rw;
        if (live) {
          if constexpr (NR % 2 == 0) {
#pragma unroll
            for (int w = 0; w < NR; w += 2) {
              const ulonglong2 x = __ldcs((const ulonglong2*)(src + w));
              rec[w] = x.x;
              rec[w + 1] = x.y;
            }
          } else {
#pragma unroll
            for (int w = 0; w < NR; w++) rec[w] = __ldcs((const unsigned long long*)src + w);
          }
        }
        uint64_t k[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) k[w] = live ? rec[w] : 0ull;
        const uint32_t sub = live ? reduce32(hash_key<KW>(k, a.sub_seed), (uint32_t)S) : 0xFFFFFFFFu;
        const uint32_t grp = __match_any_sync(0xffffffffu, sub);
        const int leader = __ffs(grp) - 1;
        uint32_t at = 0;
        if (live && lane == leader) at = atomicAdd(&s_cur[sub], (uint32_t)__popc(grp));
        at = __shfl_sync(0xffffffffu, at, leader) + __popc(grp & ((1u << lane) - 1u));
        if (!live || s_base[sub] == 0xFFFFFFFFu) continue;
        uint64_t* dst = (uint64_t*)page_ptr(a.pool, s_base[sub] + at / per) + (size_t)(at % per) * rw;
        if constexpr (NR % 2 == 0) {
#pragma unroll
          for (int w = 0; w < NR; w += 2) __stcg((ulonglong2*)(dst + w), make_ulonglong2(rec[w], rec[w + 1]));
        } else {
#pragma unroll
          for (int w = 0; w < NR; w++) __stcg((unsigned long long*)dst + w, (unsigned long long)rec[w]);
        }
        for (int w = NR; w < rw; w++)  // RWC == 0: the payload words beyond the key
          __stcg((unsigned long long*)dst + w, __ldcg((const unsigned long long*)src + w));
      }
    }
    __syncthreads();
  }
}

}  // namespace aggb
