// kernels.cuh — sm_100a kernels of the group-by hot path.
//
//   k_table_init   table reset (slots EMPTY, states at their identities)
//   k_pass         persistent, tile-scheduled pass over a batch against the
//                  level-0 L2-resident table.  Modes (the reference kernels
//                  they restate, /root/reference/pkg/src/aggbench/_kernels.py):
//                    FILL   insert-or-aggregate with a capacity and a sticky
//                           freeze; refused records are deferred     (k_table_insert :353-392)
//                    PROBE  frozen table: hits aggregate, misses spill to
//                           hash(spill_seed) partitions               (k_pp_probe :917-962)
//                    ROUTE  partition-0 table + raw spill of the other
//                           partitions; overflow spills partition 0  (k_hh_push :865-914)
//                    GRACE  pure hash partitioning                    (k_hh_push, table_on=0)
//                  Spills go through SMEM staging (per-tile counting sort by
//                  partition) into CTA-private HBM pages, so writes are
//                  contiguous runs and there is one global atomic per page.
//   k_flush_table  compaction of occupied slots + finalize (AVG division)
//                  into output columns, or native partial states  (k_flush_slots :473-519)
//   k_child        recursion step: one CTA aggregates one spilled partition in
//                  a shared-memory table (the child operator's table), frozen
//                  on overflow; misses go to the next level       (hybrid.py:244-277)
//   k_gen          seeded counter-based generators (datagen.py)
#pragma once
#include "device.cuh"

namespace aggb {

enum { MODE_FILL = 0, MODE_PROBE = 1, MODE_ROUTE = 2, MODE_GRACE = 3, MODE_DD = 4 };
enum { R_HIT = 0, R_INSERTED = 1, R_MISS = 2, R_REFUSED = 3 };
enum { ST_SPILLED = 0, ST_HITS = 1, ST_INSERTS = 2, ST_DEFERRED = 3, ST_RECORDS = 4, ST_OVERFLOW = 5,
       ST_NSTATS = 8 };

struct TableHdr {
  unsigned long long groups;     // exact-region reservations granted (may pass the region's size)
  int frozen;
  int esc;
  unsigned long long committed;  // keys actually inserted (each CTA adds its count at exit)
  unsigned long long pad;        // some insert was refused
  unsigned long long chunked;    // chunk-region reservations handed to CTAs
};

struct GTable {
  uint64_t* keys;    // (nslots + 2) * KW words; slots grouped in 32-byte buckets
                     // (4 one-word keys or 2 two-word keys), escape slot last
  uint64_t* states;  // ns * stride words: state j of slot s at states[j * fstride + s * sstride]
  uint64_t stride;   // nslots + 1 (slot nslots = escape slot of the sentinel key)
  uint64_t fstride;  // field-major (SoA, fstride = stride, sstride = 1) for L2-resident tables;
  uint64_t sstride;  // slot-major (AoS, fstride = 1, sstride = ns) for tables beyond L2 (one sector per slot)
  uint64_t mask;     // nslots - 1
  uint64_t bmask;    // nbuckets - 1
  uint64_t cap;      // group capacity (budget)
  uint64_t seed;
  TableHdr* hdr;
};

template <int KW>
struct Bkt {
  static constexpr int N = (KW == 1) ? 4 : 2;  // slots per 32-byte bucket
};

// ---------------------------------------------------------------------------
// global table lookup: bucketized linear probing (one 32-byte sector per probe
// step, so nearly every lookup resolves in its first bucket and warps do not
// diverge on long probe chains), CAS-claimed keys, capacity-bounded inserts.
// ---------------------------------------------------------------------------

// Capacity reservations are aggregated per warp: the lanes that need one at
// the same time take their count from the table's counter with one atomic by
// a leader lane, so ~inserts / (lanes per event) global atomics replace one
// same-address atomic per insert (which serialised at the L2 and dominated
// FILL).  Grants never pass `cap`.  A reservation given back (the key turned
// out to be present) goes to a per-CTA shared cache that later reservations
// use first.  When the counter reaches the capacity the table freezes (FILL
// stops grabbing tiles; the key set is final at the kernel boundary) and a
// lane left without a reservation is refused without waiting — FILL defers the
// record to the PROBE pass, ROUTE spills it to partition 0 and marks the table
// for the overflow cut.  Never wait here: a lane spinning on a reservation
// held by a lane of its own warp deadlocks at the loop's reconvergence point.
// Large tables add a chunk region: capacity [0, cap_chunked) is handed to CTAs
// `chunk` reservations at a time (one refilling thread per CTA), the rest
// [cap_chunked, cap) through the exact per-warp path, so the table still fills
// to within the CTAs' unused chunks (the host keeps that under 1% of cap).
struct CapCache {
  int* avail;          // shared: reservations held by this CTA (given back or chunked)
  unsigned* commits;   // shared: keys this CTA inserted (added to hdr->committed at exit)
  int* refused;        // shared: some insert of this CTA was refused (hdr->pad at exit)
  int* refilling;      // shared: a thread of this CTA is taking a chunk
  uint32_t chunk;      // 0: no chunk region
  unsigned long long cap_chunked;
};

__device__ __forceinline__ bool reserve_capacity(const GTable& t, const CapCache& cc) {
  if (*(volatile int*)cc.avail > 0) {
    if (atomicSub(cc.avail, 1) > 0) return true;
    atomicAdd(cc.avail, 1);
  }
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  const unsigned n = __popc(m), rank = __popc(m & ((1u << lane) - 1u));
  // (the leader reads the counter and broadcasts it: a per-lane volatile load could
  // split the lanes of m across the branch and leave __shfl_sync lanes missing)
  unsigned long long chunked = 0;
  if (cc.chunk && lane == leader) chunked = *(volatile unsigned long long*)&t.hdr->chunked;
  chunked = __shfl_sync(m, chunked, leader);
  if (cc.chunk && chunked < cc.cap_chunked) {
    // chunk region: the lanes here take one each; the leader also takes a chunk
    // for its CTA when no other thread of the CTA is doing so
    unsigned long long c = ~0ull;
    if (lane == leader) {
      const bool extra = atomicCAS(cc.refilling, 0, 1) == 0;
      const unsigned long long want = n + (extra ? cc.chunk : 0u);
      c = atomicAdd(&t.hdr->chunked, want);
      if (c + want <= cc.cap_chunked) {
        if (extra) atomicAdd(cc.avail, (int)cc.chunk);
      } else {
        c = ~0ull;  // region exhausted (its tail is left unused): the exact path decides
      }
      if (extra) atomicExch(cc.refilling, 0);
    }
    c = __shfl_sync(m, c, leader);
    if (c != ~0ull) return true;
  }
  const unsigned long long exact = t.cap - cc.cap_chunked;  // size of the exact region
  unsigned long long g = ~0ull;
  if (lane == leader && !*(volatile int*)&t.hdr->frozen) {
    g = atomicAdd(&t.hdr->groups, (unsigned long long)n);
    if (g + n >= exact) atomicExch(&t.hdr->frozen, 1);  // the counter reached the capacity
  }
  g = __shfl_sync(m, g, leader);
  if (g != ~0ull && g + rank < exact) return true;
  *(volatile int*)cc.refused = 1;  // published once per CTA (ROUTE: cut the table at close)
  return false;
}

__device__ __forceinline__ void release_capacity(const CapCache& cc) { atomicAdd(cc.avail, 1); }
__device__ __forceinline__ void commit_insert(const CapCache& cc) { atomicAdd(cc.commits, 1u); }

__device__ __forceinline__ void ld_bucket(const uint64_t* keys, uint64_t b, uint64_t (&w)[4]) {
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(keys + b * 4);
  ulonglong2 x = __ldcg(p), y = __ldcg(p + 1);
  w[0] = x.x;
  w[1] = x.y;
  w[2] = y.x;
  w[3] = y.y;
}

// escape slot: the one key whose words all equal EMPTY
template <int KW>
__device__ __forceinline__ int64_t gt_escape(const GTable& t, bool insert, const CapCache& cc, int& res) {
  int64_t s = (int64_t)t.mask + 1;
  if (*(volatile int*)&t.hdr->esc) { res = R_HIT; return s; }
  if (!insert) { res = R_MISS; return -1; }
  if (!reserve_capacity(t, cc)) { res = R_REFUSED; return -1; }
  if (atomicCAS(&t.hdr->esc, 0, 1) == 0) { commit_insert(cc); res = R_INSERTED; return s; }
  release_capacity(cc);
  res = R_HIT;
  return s;
}

// Resolve key k whose first bucket b was already loaded into w[].
template <int KW>
__device__ __forceinline__ int64_t gt_resolve(const GTable& t, const uint64_t (&k)[KW], uint64_t b,
                                              uint64_t (&w)[4], bool insert, const CapCache& cc, int& res) {
  constexpr int BK = Bkt<KW>::N;
  bool reserved = false;
  int from = 0;
  for (;;) {
    int hit = -1, emp = -1;
#pragma unroll
    for (int j = 0; j < BK; j++) {
      if (j < from || hit >= 0 || emp >= 0) continue;
      uint64_t a0 = w[j * KW], a1 = (KW == 2) ? w[j * KW + 1] : 0ull;
      if (KW == 2 && insert && ((a0 == EMPTY) != (a1 == EMPTY))) {
        uint64_t x, y;  // possibly torn while another thread inserts: read atomically
        cas128(t.keys + (b * BK + j) * KW, EMPTY, EMPTY, EMPTY, EMPTY, x, y);
        a0 = x;
        a1 = y;
      }
      if (a0 == k[0] && (KW == 1 || a1 == k[KW - 1])) hit = j;
      else if (a0 == EMPTY && (KW == 1 || a1 == EMPTY)) emp = j;
    }
    if (hit >= 0) {
      if (reserved) release_capacity(cc);
      res = R_HIT;
      return (int64_t)(b * BK + hit);
    }
    if (emp >= 0) {
      if (!insert) { res = R_MISS; return -1; }
      if (!reserved) {
        if (!reserve_capacity(t, cc)) { res = R_REFUSED; return -1; }
        reserved = true;
      }
      uint64_t* kp = t.keys + (b * BK + emp) * KW;
      if (KW == 1) {
        unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k[0]);
        if (prev == EMPTY) { commit_insert(cc); res = R_INSERTED; return (int64_t)(b * BK + emp); }
        if (prev == k[0]) { release_capacity(cc); res = R_HIT; return (int64_t)(b * BK + emp); }
      } else {
        uint64_t x, y;
        cas128(kp, EMPTY, EMPTY, k[0], k[KW - 1], x, y);
        if (x == EMPTY && y == EMPTY) { commit_insert(cc); res = R_INSERTED; return (int64_t)(b * BK + emp); }
        if (x == k[0] && y == k[KW - 1]) { release_capacity(cc); res = R_HIT; return (int64_t)(b * BK + emp); }
      }
      // another key took the slot: rescan this bucket after it
      ld_bucket(t.keys, b, w);
      from = emp + 1;
      if (from < BK) continue;
    }
    b = (b + 1) & t.bmask;
    from = 0;
    ld_bucket(t.keys, b, w);
  }
}


// ---------------------------------------------------------------------------
// blocked bloom filter of the frozen resident keys (the reference keeps a
// bloom byte per slot for pre-partitioning's probe stage, _kernels.py:388-390,
// :938-942; here one 64-bit block per key, 4 bits, held in SMEM by k_pass)
// ---------------------------------------------------------------------------

struct Bloom {
  const uint64_t* words;  // nullptr: disabled
  uint32_t mask;          // nblocks - 1 (blocks are 64-bit words)
  uint64_t seed;
};

// The filter is keyed off the table's own 64-bit hash h (k_pass / k_probe
// derive bucket, spill partition and bloom probe from one hash): bucket from
// bits 0..16 (the filter is off for tables large enough to use more), block
// from bits 20..33, four bit positions from bits 34..53 (two per 32-bit half of
// the block; 32-bit shifts only); the partition comes from the top bits.
__device__ __forceinline__ uint32_t bloom_block(uint64_t h, uint32_t mask) { return (uint32_t)(h >> 20) & mask; }
__device__ __forceinline__ uint64_t bloom_bits(uint64_t h) {
  const uint32_t x = (uint32_t)(h >> 34);
  const uint32_t lo = (1u << (x & 31)) | (1u << ((x >> 5) & 31));
  const uint32_t hi = (1u << ((x >> 10) & 31)) | (1u << ((x >> 15) & 31));
  return ((uint64_t)hi << 32) | lo;
}

template <int KW>
__global__ void k_bloom_build(GTable t, uint64_t* bloom, uint32_t mask) {
  uint64_t n = t.mask + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = t.keys[i * KW + w];
    if (is_sentinel<KW>(k)) continue;
    const uint64_t h = hash_key<KW>(k, t.seed);
    atomicOr((unsigned long long*)&bloom[bloom_block(h, mask)], (unsigned long long)bloom_bits(h));
  }
}

__global__ void k_table_init(GTable t, int kw, DevSpec sp) {
  // one array at a time, one identity per array, 16-byte stores (a per-slot loop
  // over the fields indexed the spec dynamically: 1.7 TB/s on C4's 24 GB table)
  const uint64_t n = t.stride;
  const uint64_t gt = (uint64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  auto fill = [&](uint64_t* p, uint64_t cnt, uint64_t v) {
    const uint64_t head = ((16 - ((uintptr_t)p & 15)) & 15) / 8;  // 8-byte words before 16-byte alignment
    if (t0 < head && t0 < cnt) p[t0] = v;
    ulonglong2* q = (ulonglong2*)(p + min(head, cnt));
    const uint64_t pairs = cnt > head ? (cnt - head) / 2 : 0;
    const ulonglong2 vv = make_ulonglong2(v, v);
    for (uint64_t i = t0; i < pairs; i += gt) q[i] = vv;
    const uint64_t tail = cnt > head ? (cnt - head) % 2 : 0;
    if (tail && t0 == 0) p[cnt - 1] = v;
  };
  fill(t.keys, n * (uint64_t)kw, EMPTY);
  if (t.sstride == 1) {
    for (int j = 0; j < sp.ns; j++) fill(t.states + (uint64_t)j * n, n, state_identity(sp.op[j], sp.ty[j]));
  } else {  // slot-major: the identities repeat with period ns
    uint64_t id[MAX_STATES];
    bool zero = true;
    for (int j = 0; j < sp.ns; j++) {
      id[j] = state_identity(sp.op[j], sp.ty[j]);
      zero = zero && id[j] == 0;
    }
    const uint64_t words = n * (uint64_t)sp.ns;
    if (zero) {
      fill(t.states, words, 0ull);
    } else {
      for (uint64_t i = t0; i < words; i += gt) t.states[i] = id[i % (uint64_t)sp.ns];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    t.hdr->groups = 0;
    t.hdr->frozen = 0;
    t.hdr->esc = 0;
    t.hdr->committed = 0;
    t.hdr->pad = 0;
    t.hdr->chunked = 0;
  }
}

// ---------------------------------------------------------------------------
// record sources
// ---------------------------------------------------------------------------

struct ColSrc {
  int64_t n;
  const uint8_t* key[2];
  int64_t kstride[2];
  uint8_t kty[2];
  int32_t nv;
  const uint8_t* val[MAX_VALS];
  int64_t vstride[MAX_VALS];
  uint8_t vty[MAX_VALS];  // input types (I32 widened on load)
};

template <int KW>
__device__ __forceinline__ void col_key(const ColSrc& c, int64_t i, uint64_t (&k)[KW]) {
#pragma unroll
  for (int w = 0; w < KW; w++) {
    const uint8_t* p = c.key[w] + i * c.kstride[w];
    if (c.kty[w] == TY_I32) k[w] = ((uint64_t)(uint32_t)__ldcs((const int*)p)) << 32;
    else k[w] = (uint64_t)__ldcs((const long long*)p);
  }
}

template <int NWT>
__device__ __forceinline__ void col_vals(const ColSrc& c, int64_t i, uint64_t (&v)[NWT]) {
#pragma unroll
  for (int w = 0; w < NWT; w++) {
    if (w < c.nv) {
      const uint8_t* p = c.val[w] + i * c.vstride[w];
      if (c.vty[w] == TY_I32) v[w] = (uint64_t)(long long)__ldcs((const int*)p);
      else v[w] = (uint64_t)__ldcs((const long long*)p);
    } else {
      v[w] = 0;
    }
  }
}

// SoA record block: word w of record i at base[w * stride + i]
template <int KW, int NWT>
__device__ __forceinline__ void soa_load(const uint64_t* base, int64_t stride, int64_t i, int nw, uint64_t (&k)[KW],
                                         uint64_t (&v)[NWT]) {
#pragma unroll
  for (int w = 0; w < KW; w++) k[w] = __ldcs((const unsigned long long*)base + w * stride + i);
#pragma unroll
  for (int w = 0; w < NWT; w++)
    v[w] = (w < nw) ? (uint64_t)__ldcs((const unsigned long long*)base + (KW + w) * stride + i) : 0ull;
}

// contribution of record payload v[] (raw or native partial) to state field j
__device__ __forceinline__ uint64_t contrib(const DevSpec& sp, int kind, int j, const uint64_t* v) {
  return kind ? v[j] : contribution(sp, j, v);
}

// ---------------------------------------------------------------------------
// block helpers
// ---------------------------------------------------------------------------

// exclusive scan of a[0..n) in shared memory (n arbitrary), returns total
__device__ uint32_t block_exscan(uint32_t* a, int n, uint32_t* scratch /* >= 33 */) {
  int tid = threadIdx.x, B = blockDim.x;
  int per = (n + B - 1) / B;
  int lo = tid * per, hi = min(n, lo + per);
  uint32_t sum = 0;
  for (int i = lo; i < hi; i++) sum += a[i];
  // warp inclusive scan of per-thread sums
  uint32_t x = sum;
  int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int nw = (B + 31) >> 5;
    uint32_t s = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) scratch[lane] = s;  // inclusive per warp
    if (lane == nw - 1) scratch[32] = s;
  }
  __syncthreads();
  uint32_t run = x - sum + (wid ? scratch[wid - 1] : 0);
  for (int i = lo; i < hi; i++) {
    uint32_t t = a[i];
    a[i] = run;
    run += t;
  }
  uint32_t total = scratch[32];
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------------------
// k_pass
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// output buffers + table flush
// ---------------------------------------------------------------------------

struct OutBuf {
  uint64_t* keys;   // KW word columns: keys[w * cap + i]
  uint64_t* vals;   // finalized: nout columns; partial: ns columns
  int64_t cap;
  unsigned long long* count;
  int32_t partial;  // 1: write native partial states instead of finished values
};

__device__ __forceinline__ uint64_t finish_value(const DevSpec& sp, int j, const uint64_t* st) {
  uint64_t a = st[sp.fin_a[j]];
  int fa = sp.fin_a[j];
  if (sp.fin_div[j]) {
    double num = (sp.ty[fa] == TY_F64) ? __longlong_as_double((long long)a) : (double)(long long)a;
    double den = (double)(long long)st[sp.fin_b[j]];
    return (uint64_t)__double_as_longlong(num / den);
  }
  if (sp.ty[fa] == TY_F64 && sp.op[fa] != OP_ADD) return ord_f64(a);
  return a;
}

template <int KW>
__device__ __forceinline__ void emit_group(const DevSpec& sp, const OutBuf& o, int64_t idx, const uint64_t (&k)[KW],
                                           const uint64_t* st) {
  if (idx >= o.cap) return;
#pragma unroll
  for (int w = 0; w < KW; w++) o.keys[w * o.cap + idx] = k[w];
  if (o.partial) {
    for (int j = 0; j < sp.ns; j++) o.vals[j * o.cap + idx] = st[j];
  } else {
    for (int j = 0; j < sp.nout; j++) o.vals[j * o.cap + idx] = finish_value(sp, j, st);
  }
}

// the same for specs of at most 4 state fields and 4 outputs, states in
// registers (the generic path indexes a 32-entry state array dynamically, which
// lives in local memory: C4's 0.5B-group flush ran at 1.2 TB/s)
__device__ __forceinline__ uint64_t sel4(const uint64_t (&v)[4], int i) {
  return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
}
template <int KW>
__device__ __forceinline__ void emit_group4(const DevSpec& sp, const OutBuf& o, int64_t idx, const uint64_t (&k)[KW],
                                            const uint64_t (&st)[4]) {
  if (idx >= o.cap) return;
#pragma unroll
  for (int w = 0; w < KW; w++) o.keys[w * o.cap + idx] = k[w];
  if (o.partial) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (j < sp.ns) o.vals[j * o.cap + idx] = st[j];
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; j++) {
    if (j >= sp.nout) break;
    const int fa = sp.fin_a[j];
    const uint64_t a = sel4(st, fa);
    uint64_t v = a;
    if (sp.fin_div[j]) {
      const double num = (sp.ty[fa] == TY_F64) ? __longlong_as_double((long long)a) : (double)(long long)a;
      const double den = (double)(long long)sel4(st, sp.fin_b[j]);
      v = (uint64_t)__double_as_longlong(num / den);
    } else if (sp.ty[fa] == TY_F64 && sp.op[fa] != OP_ADD) {
      v = ord_f64(a);
    }
    o.vals[j * o.cap + idx] = v;
  }
}

// CLEAR: also reset every slot it emits (keys EMPTY, states at identity), so
// a table cut by hash_sort is empty again without a full k_table_init pass
// (the header is reset separately, after the kernel)
// the flush of a table by the CTAs of a grid (k_flush_table, and the cut step of
// k_blind_cuts): tiles of 8 x 256 slots: warp w scans slots [base + 256 j + 32 w, +32)
// for j < 8 (coalesced), the CTA reserves its tile's output with ONE atomic (one
// per warp and 32 slots was 33.5M same-address atomics on C4's 2^30-slot table:
// 69 ms of flush).  BLK threads per CTA (s_wc holds BLK / 32 words).
template <int KW, bool CLEAR, int BLK = 256, int J = 8>
__device__ __forceinline__ void flush_tiles(const GTable& t, const DevSpec& sp, const OutBuf& o, uint32_t* s_wc,
                                            unsigned long long* s_base_p) {
  constexpr int TILE = BLK * J, NWF = BLK / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t n = t.stride;
  for (uint64_t base = (uint64_t)blockIdx.x * TILE; base < n; base += (uint64_t)gridDim.x * TILE) {
    unsigned m[J];
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < J; j++) {
      const uint64_t s = base + (uint64_t)j * BLK + (uint64_t)wid * 32 + lane;
      bool occ = false;
      if (s < n) {
        uint64_t k[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) k[w] = __ldcg(t.keys + s * KW + w);  // (L2: a persistent caller's L1 may hold the last cut's keys)
        occ = (s == n - 1) ? (*(volatile int*)&t.hdr->esc != 0) : !is_sentinel<KW>(k);
      }
      m[j] = __ballot_sync(0xffffffffu, occ);
      cnt += __popc(m[j]);
    }
    if (lane == 0) s_wc[wid] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (int w = 0; w < NWF; w++) {
        const uint32_t c = s_wc[w];
        s_wc[w] = acc;
        acc += c;
      }
      *s_base_p = acc ? atomicAdd(o.count, (unsigned long long)acc) : 0ull;
    }
    __syncthreads();
    int64_t at = (int64_t)(*s_base_p + s_wc[wid]);
#pragma unroll
    for (int j = 0; j < J; j++) {
      if (!m[j]) continue;  // warp-uniform
      const uint64_t s = base + (uint64_t)j * BLK + (uint64_t)wid * 32 + lane;
      if ((m[j] >> lane) & 1u) {
        uint64_t k[KW];
#pragma unroll
        for (int w = 0; w < KW; w++) k[w] = __ldcg(t.keys + s * KW + w);  // (L2: a persistent caller's L1 may hold the last cut's keys)
        const int64_t idx = at + __popc(m[j] & ((1u << lane) - 1));
        if (sp.ns <= 4 && sp.nout <= 4) {
          uint64_t st4[4];
#pragma unroll
          for (int q = 0; q < 4; q++) st4[q] = q < sp.ns ? __ldcg(t.states + (uint64_t)q * t.fstride + s * t.sstride) : 0ull;
          emit_group4<KW>(sp, o, idx, k, st4);
        } else {
          uint64_t st[MAX_STATES];
          // eight state words in flight at a time (a word-by-word loop through the local
          // array serialised an L2 round trip per field)
          for (int q0 = 0; q0 < sp.ns; q0 += 8) {
            uint64_t r[8];
#pragma unroll
            for (int j2 = 0; j2 < 8; j2++)
              r[j2] = q0 + j2 < sp.ns ? __ldcg(t.states + (uint64_t)(q0 + j2) * t.fstride + s * t.sstride) : 0ull;
#pragma unroll
            for (int j2 = 0; j2 < 8; j2++)
              if (q0 + j2 < sp.ns) st[q0 + j2] = r[j2];
          }
          emit_group<KW>(sp, o, idx, k, st);
        }
        if (CLEAR) {
#pragma unroll
          for (int w = 0; w < KW; w++) t.keys[s * KW + w] = EMPTY;
          for (int q = 0; q < sp.ns; q++) t.states[(uint64_t)q * t.fstride + s * t.sstride] = state_identity(sp.op[q], sp.ty[q]);
          if (s == n - 1) t.hdr->esc = 0;  // (the escape slot's only reader: the table is empty again)
        }
      }
      at += __popc(m[j]);
    }
    __syncthreads();  // s_wc / s_base reused by the next tile
  }
}


template <int KW, bool CLEAR = false>
__global__ void __launch_bounds__(256) k_flush_table(GTable t, DevSpec sp, OutBuf o) {
  __shared__ uint32_t s_wc[8];
  __shared__ unsigned long long s_base;
  flush_tiles<KW, CLEAR>(t, sp, o, s_wc, &s_base);
}

// ---------------------------------------------------------------------------
// k_child: per-partition shared-memory aggregation (one recursion level)
// ---------------------------------------------------------------------------

// Shared-memory table lookup of the child operators.  `s_inflight` counts
// threads between a capacity reservation and the end of their key CAS; once
// the table is frozen no reservation succeeds, so when a refused thread sees
// `s_inflight == 0` the key set is final and its re-probe is exact — a key is
// either resident (aggregate) or not (overflow), never both.
template <int KW>
__device__ __forceinline__ int stable_lookup(uint64_t* keys, int nslots, int cap, const uint64_t (&k)[KW], uint64_t seed,
                                             bool insert, int* s_groups, int* s_frozen, int* s_esc, int* s_inflight,
                                             int& res) {
  // s_groups[0]: reservations + committed inserts; s_groups[1]: committed inserts.
  // A transient excess (racing reservations) refuses without freezing; the
  // caller re-probes once no insert is in flight (stable_resolve_refused).
  auto reserve = [&]() -> bool {
    atomicAdd(s_inflight, 1);
    if (!*(volatile int*)s_frozen) {
      int old = atomicAdd(s_groups, 1);
      if (old < cap) return true;  // s_inflight released by the caller after the key CAS
      atomicSub(s_groups, 1);
      if (*(volatile int*)(s_groups + 1) + max(1, cap / 32) > cap) atomicExch(s_frozen, 1);
    }
    atomicSub(s_inflight, 1);
    return false;
  };
  if (is_sentinel<KW>(k)) {
    if (*(volatile int*)s_esc) { res = R_HIT; return nslots; }
    if (!insert) { res = R_MISS; return -1; }
    if (!reserve()) { res = R_REFUSED; return -1; }
    int won = atomicCAS(s_esc, 0, 1) == 0;
    if (!won) atomicSub(s_groups, 1);
    else atomicAdd(s_groups + 1, 1);
    atomicSub(s_inflight, 1);  // after the CAS: same-thread shared atomics complete in order
    res = won ? R_INSERTED : R_HIT;
    return nslots;
  }
  int mask = nslots - 1;
  bool reserved = false;
  if (KW == 1) {
    // slots probed in aligned pairs, one 16-byte shared load per pair; the probe
    // sequence starts at the pair of the home slot (inserts and lookups agree)
    int s = (int)(hash_key<KW>(k, seed) & (uint64_t)mask) & ~1;
    const uint32_t keys_sh = (uint32_t)__cvta_generic_to_shared(keys);
    for (;;) {
      uint64_t w0, w1;
      asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "r"(keys_sh + 8u * (uint32_t)s));
      int at = -1;
      if (w0 == k[0]) at = s;
      else if (w1 == k[0]) at = s + 1;
      if (at >= 0) {
        if (reserved) {
          atomicSub(s_groups, 1);
          atomicSub(s_inflight, 1);
        }
        res = R_HIT;
        return at;
      }
      const int e = (w0 == EMPTY) ? s : ((w1 == EMPTY) ? s + 1 : -1);
      if (e >= 0) {
        if (!insert) { res = R_MISS; return -1; }
        if (!reserved) {
          if (!reserve()) { res = R_REFUSED; return -1; }
          reserved = true;
        }
        const unsigned long long prev = atomicCAS((unsigned long long*)(keys + e), EMPTY, k[0]);
        if (prev == EMPTY || prev == k[0]) {
          if (prev == k[0]) atomicSub(s_groups, 1);
          else atomicAdd(s_groups + 1, 1);
          atomicSub(s_inflight, 1);  // after the CAS: same-thread shared atomics complete in order
          res = prev == EMPTY ? R_INSERTED : R_HIT;
          return e;
        }
        continue;  // another key took the slot: re-read the pair
      }
      s = (s + 2) & mask;
    }
  }
  int s = (int)(hash_key<KW>(k, seed) & (uint64_t)mask);
  for (;;) {
    uint64_t* kp = keys + (size_t)s * KW;
    uint64_t w0 = *(volatile uint64_t*)kp;
    uint64_t w1 = (KW == 2) ? *(volatile uint64_t*)(kp + 1) : 0ull;
    bool match = (w0 == k[0]) && (KW == 1 || w1 == k[KW - 1]);
    bool empty = (w0 == EMPTY) && (KW == 1 || w1 == EMPTY);
    if (KW == 2 && !match && !empty && (w0 == EMPTY || w1 == EMPTY || w0 == k[0])) {
      uint64_t a, b;
      cas128(kp, EMPTY, EMPTY, EMPTY, EMPTY, a, b);
      match = (a == k[0]) && (b == k[KW - 1]);
      empty = (a == EMPTY) && (b == EMPTY);
    }
    if (match) {
      if (reserved) {
        atomicSub(s_groups, 1);
        atomicSub(s_inflight, 1);
      }
      res = R_HIT;
      return s;
    }
    if (empty) {
      if (!insert) { res = R_MISS; return -1; }
      if (!reserved) {
        if (!reserve()) { res = R_REFUSED; return -1; }
        reserved = true;
      }
      bool won, same;
      if (KW == 1) {
        unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k[0]);
        won = prev == EMPTY;
        same = prev == k[0];
      } else {
        uint64_t a, b;
        cas128(kp, EMPTY, EMPTY, k[0], k[KW - 1], a, b);
        won = (a == EMPTY && b == EMPTY);
        same = (a == k[0] && b == k[KW - 1]);
      }
      if (won || same) {
        if (same) atomicSub(s_groups, 1);
        else atomicAdd(s_groups + 1, 1);
        atomicSub(s_inflight, 1);  // after the CAS: same-thread shared atomics complete in order
        res = won ? R_INSERTED : R_HIT;
        return s;
      }
    }
    s = (s + 1) & mask;
  }
}

// A refused record may go to the overflow list only when the table can no
// longer change for its key: the table is frozen and no insert is in flight.
// A transient refusal (racing reservations, table not frozen) retries the
// insert once the in-flight inserts have drained; if that keeps failing the
// table is frozen explicitly, which makes the final probe exact.
template <int KW>
__device__ __forceinline__ int stable_resolve_refused(uint64_t* keys, int nslots, int cap, const uint64_t (&k)[KW],
                                                      uint64_t seed, int* s_groups, int* s_frozen, int* s_esc,
                                                      int* s_inflight, int& res) {
  for (int tries = 0;; tries++) {
    for (int spin = 0; *(volatile int*)s_inflight > 0 && spin < (1 << 22); spin++) __nanosleep(32);
    __threadfence_block();
    const bool frozen = *(volatile int*)s_frozen != 0;
    int s = stable_lookup<KW>(keys, nslots, cap, k, seed, !frozen, s_groups, s_frozen, s_esc, s_inflight, res);
    if (res != R_REFUSED) return s;  // hit, inserted, or (frozen) a final miss
    if (tries >= 16) atomicExch(s_frozen, 1);
  }
}

// ---------------------------------------------------------------------------
// page bookkeeping: bucket a page range by partition (counting sort)
// ---------------------------------------------------------------------------

__global__ void k_page_hist(PagePool pool, uint32_t first, const uint32_t* last_ptr, int set_id, int nparts,
                            unsigned long long* part_records, uint32_t* part_pages /* [nparts] for this set */) {
  uint32_t last = min(*last_ptr, pool.capacity);
  for (uint32_t pg = first + blockIdx.x * blockDim.x + threadIdx.x; pg < last; pg += gridDim.x * blockDim.x) {
    if (pool.page_set[pg] != set_id) continue;
    int p = pool.page_part[pg];
    if (p < 0 || p >= nparts) continue;
    if (pool.page_fill[pg] == 0) continue;  // the same filter as k_page_scatter (its lists count these pages)
    atomicAdd(&part_records[p], (unsigned long long)pool.page_fill[pg]);
    atomicAdd(&part_pages[p], 1u);
  }
}

__global__ void k_page_scatter(PagePool pool, uint32_t first, const uint32_t* last_ptr, int set_id, int nparts,
                               uint32_t* cursor /* exclusive offsets, advanced */, uint2* plist) {
  uint32_t last = min(*last_ptr, pool.capacity);
  for (uint32_t pg = first + blockIdx.x * blockDim.x + threadIdx.x; pg < last; pg += gridDim.x * blockDim.x) {
    if (pool.page_set[pg] != set_id) continue;
    int p = pool.page_part[pg];
    if (p < 0 || p >= nparts) continue;
    if (pool.page_fill[pg] == 0) continue;
    uint32_t at = atomicAdd(&cursor[p], 1u);
    plist[at] = make_uint2(pg, (uint32_t)pool.page_fill[pg]);  // fill travels with the id
  }
}

// ---------------------------------------------------------------------------
// output egress: key words -> typed key columns
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// multi-GPU exchange: pack partial groups by destination rank (AoS records)
// ---------------------------------------------------------------------------

template <int KW>
__global__ void k_exch_count(const uint64_t* keys, int64_t cap, int64_t n, uint64_t seed, int nranks,
                             unsigned long long* counts) {
  __shared__ unsigned int sh[256];
  for (int i = threadIdx.x; i < nranks; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = keys[w * cap + i];
    atomicAdd(&sh[reduce32(hash_key<KW>(k, seed), (uint32_t)nranks)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nranks; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

template <int KW>
__global__ void k_exch_scatter(const uint64_t* keys, const uint64_t* states, int64_t cap, int64_t n, int ns,
                               uint64_t seed, int nranks, unsigned long long* cursor, uint64_t* send) {
  const int rw = KW + ns;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = keys[w * cap + i];
    unsigned d = reduce32(hash_key<KW>(k, seed), (uint32_t)nranks);
    unsigned long long at = atomicAdd(&cursor[d], 1ull);
    uint64_t* dst = send + at * rw;
#pragma unroll
    for (int w = 0; w < KW; w++) dst[w] = k[w];
    for (int j = 0; j < ns; j++) dst[KW + j] = states[(int64_t)j * cap + i];
  }
}

// raw-first exchange (C4-like inputs, little local collapse): input rows are
// packed by destination before any aggregation, one 8-byte slot per key and
// value column (4-byte columns in the slot's low half), so the receiver pushes
// the buffer as strided columns of the same types
template <int KW>
__global__ void k_exch_raw_count(ColSrc c, uint64_t seed, int nranks, unsigned long long* counts) {
  __shared__ unsigned int sh[256];
  for (int i = threadIdx.x; i < nranks; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
    col_key<KW>(c, i, k);
    atomicAdd(&sh[reduce32(hash_key<KW>(k, seed), (uint32_t)nranks)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nranks; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

__device__ __forceinline__ uint64_t raw_slot(const uint8_t* base, int64_t stride, int ty, int64_t i) {
  const uint8_t* p = base + i * stride;
  return ty == TY_I32 ? (uint64_t)(uint32_t)*(const int32_t*)p : *(const uint64_t*)p;
}

template <int KW>
__global__ void k_exch_raw_scatter(ColSrc c, uint64_t seed, int nranks, unsigned long long* cursor, uint64_t* send) {
  const int rw = KW + c.nv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
    col_key<KW>(c, i, k);
    const unsigned d = reduce32(hash_key<KW>(k, seed), (uint32_t)nranks);
    const unsigned long long at = atomicAdd(&cursor[d], 1ull);
    uint64_t* dst = send + at * rw;
#pragma unroll
    for (int w = 0; w < KW; w++) dst[w] = raw_slot(c.key[w], c.kstride[w], c.kty[w], i);
    for (int w = 0; w < c.nv; w++) dst[KW + w] = raw_slot(c.val[w], c.vstride[w], c.vty[w], i);
  }
}

// dynamic destaging (hybrid.py:974-1149): groups of a flushed table (SoA
// partial list, `n` records, column stride `cap`) counted per partition, and
// split into the evicted partitions' groups and the kept ones
template <int KW>
__global__ void k_dd_hist(const uint64_t* keys, int64_t cap, const unsigned long long* n, uint64_t seed, int P,
                          unsigned long long* hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = keys[w * cap + i];
    const int p = (int)reduce32(hash_key<KW>(k, seed), (uint32_t)P);  // GRACE's partition
    atomicAdd(&hist[p], 1ull);
  }
}

template <int KW>
__global__ void k_dd_split(const uint64_t* src, int64_t cap, const unsigned long long* n, int words, uint64_t seed,
                           int P, const uint8_t* evict, uint64_t* ev, uint64_t* kept, unsigned long long* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k[KW];
#pragma unroll
    for (int w = 0; w < KW; w++) k[w] = src[w * cap + i];
    const int p = (int)reduce32(hash_key<KW>(k, seed), (uint32_t)P);
    const int e = evict[p] ? 0 : 1;
    uint64_t* dst = e == 0 ? ev : kept;
    const unsigned long long at = atomicAdd(&counts[e], 1ull);
    for (int w = 0; w < words; w++) dst[w * cap + at] = src[w * cap + i];
  }
}

// AoS partial records -> SoA (the pass kernels' list layout)
__global__ void k_aos_to_soa(const uint64_t* in, int64_t n, int rw, uint64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int w = 0; w < rw; w++) out[(int64_t)w * n + i] = in[i * rw + w];
}

// Gather one item's records (AoS pages of rw words) into dense columns
// (SoA, column stride `stride`) for an L2-table child; pages land in any order
// (aggregation is order-free), each page's records contiguously.
__global__ void k_gather_pages(PagePool pool, const uint2* plist, int64_t npages, int rw, uint64_t* out,
                               int64_t stride, unsigned long long* count) {
  __shared__ unsigned long long s_base;
  for (int64_t q = blockIdx.x; q < npages; q += gridDim.x) {
    const uint2 pe = plist[q];
    if (threadIdx.x == 0) s_base = atomicAdd(count, (unsigned long long)pe.y);
    __syncthreads();
    const unsigned long long* src = (const unsigned long long*)page_ptr(pool, pe.x);
    const int64_t base = (int64_t)s_base;
    for (int i = threadIdx.x; i < (int)pe.y * rw; i += blockDim.x)
      out[(int64_t)(i % rw) * stride + base + i / rw] = __ldcs(src + i);
    __syncthreads();
  }
}

__global__ void k_key_to_i32(const uint64_t* w, int32_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)(uint32_t)(w[i] >> 32);
}

// ---------------------------------------------------------------------------
// generators (paper_1311_0059_b200/datagen.py restated)
// ---------------------------------------------------------------------------

__host__ __device__ __forceinline__ uint64_t mix64_sm(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_gen(int kind, uint64_t base, uint64_t base2, int64_t start, int64_t n, int64_t lo, int64_t range,
                      const double* cdf, int64_t K, uint64_t pa, uint64_t pb, uint8_t* out, int64_t stride) {
  const uint64_t G = 0x9E3779B97F4A7C15ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = mix64_sm(base + (uint64_t)(start + i + 1) * G);
    uint8_t* dst = out + i * stride;
    if (kind == 0) {
      *(int64_t*)dst = (int64_t)(x % (uint64_t)range) + lo;
    } else if (kind == 4) {
      *(int32_t*)dst = (int32_t)((int64_t)(x % (uint64_t)range) + lo);
    } else if (kind == 1) {
      *(double*)dst = (double)(x >> 11) * 0x1.0p-53;
    } else if (kind == 2) {
      uint64_t x2 = mix64_sm(base2 + (uint64_t)(start + i + 1) * G);
      double u1 = ((double)(x >> 11) + 1.0) * 0x1.0p-53;
      double u2 = (double)(x2 >> 11) * 0x1.0p-53;
      *(double*)dst = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
    } else {  // zipf: first rank with cdf[rank] > u (np.searchsorted side='right')
      double u = (double)(x >> 11) * 0x1.0p-53;
      int64_t lo2 = 0, hi2 = K;
      while (lo2 < hi2) {
        int64_t mid = (lo2 + hi2) >> 1;
        if (cdf[mid] <= u) lo2 = mid + 1;
        else hi2 = mid;
      }
      uint64_t rank = (uint64_t)min(lo2, K - 1);
      *(int64_t*)dst = (int64_t)((rank * pa + pb) % (uint64_t)K);
    }
  }
}

__global__ void k_l2flush(uint4* p, int64_t n, uint32_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((uint32_t)i, salt, 0u, 0u);
}

}  // namespace aggb
