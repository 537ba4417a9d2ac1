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

enum { MODE_FILL = 0, MODE_PROBE = 1, MODE_ROUTE = 2, MODE_GRACE = 3 };
enum { R_HIT = 0, R_INSERTED = 1, R_MISS = 2, R_REFUSED = 3 };
enum { ST_SPILLED = 0, ST_HITS = 1, ST_INSERTS = 2, ST_DEFERRED = 3, ST_RECORDS = 4, ST_OVERFLOW = 5,
       ST_NSTATS = 8 };

struct TableHdr {
  unsigned long long groups;
  int frozen;
  int esc;
  unsigned long long pad[2];
};

struct GTable {
  uint64_t* keys;    // (nslots + 2) * KW words; slots grouped in 32-byte buckets
                     // (4 one-word keys or 2 two-word keys), escape slot last
  uint64_t* states;  // ns * stride, field-major
  uint64_t stride;   // nslots + 1 (slot nslots = escape slot of the sentinel key)
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

__device__ __forceinline__ bool reserve_capacity(const GTable& t) {
  if (*(volatile int*)&t.hdr->frozen) return false;
  unsigned long long old = atomicAdd(&t.hdr->groups, 1ull);
  if (old >= t.cap) {
    atomicAdd(&t.hdr->groups, ~0ull);
    atomicExch(&t.hdr->frozen, 1);
    return false;
  }
  return true;
}

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
__device__ __forceinline__ int64_t gt_escape(const GTable& t, bool insert, int& res) {
  int64_t s = (int64_t)t.mask + 1;
  if (*(volatile int*)&t.hdr->esc) { res = R_HIT; return s; }
  if (!insert) { res = R_MISS; return -1; }
  if (!reserve_capacity(t)) { res = R_REFUSED; return -1; }
  if (atomicCAS(&t.hdr->esc, 0, 1) == 0) { res = R_INSERTED; return s; }
  atomicAdd(&t.hdr->groups, ~0ull);
  res = R_HIT;
  return s;
}

// Resolve key k whose first bucket b was already loaded into w[].
template <int KW>
__device__ __forceinline__ int64_t gt_resolve(const GTable& t, const uint64_t (&k)[KW], uint64_t b,
                                              uint64_t (&w)[4], bool insert, int& res) {
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
      if (reserved) atomicAdd(&t.hdr->groups, ~0ull);
      res = R_HIT;
      return (int64_t)(b * BK + hit);
    }
    if (emp >= 0) {
      if (!insert) { res = R_MISS; return -1; }
      if (!reserved) {
        if (!reserve_capacity(t)) { res = R_REFUSED; return -1; }
        reserved = true;
      }
      uint64_t* kp = t.keys + (b * BK + emp) * KW;
      if (KW == 1) {
        unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k[0]);
        if (prev == EMPTY) { res = R_INSERTED; return (int64_t)(b * BK + emp); }
        if (prev == k[0]) { atomicAdd(&t.hdr->groups, ~0ull); res = R_HIT; return (int64_t)(b * BK + emp); }
      } else {
        uint64_t x, y;
        cas128(kp, EMPTY, EMPTY, k[0], k[KW - 1], x, y);
        if (x == EMPTY && y == EMPTY) { res = R_INSERTED; return (int64_t)(b * BK + emp); }
        if (x == k[0] && y == k[KW - 1]) { atomicAdd(&t.hdr->groups, ~0ull); res = R_HIT; return (int64_t)(b * BK + emp); }
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

template <int KW>
__device__ __forceinline__ int64_t gtable_lookup(const GTable& t, const uint64_t (&k)[KW], bool insert, int& res) {
  if (is_sentinel<KW>(k)) return gt_escape<KW>(t, insert, res);
  uint64_t b = hash_key<KW>(k, t.seed) & t.bmask;
  uint64_t w[4];
  ld_bucket(t.keys, b, w);
  return gt_resolve<KW>(t, k, b, w, insert, res);
}

__global__ void k_table_init(GTable t, int kw, DevSpec sp) {
  uint64_t n = t.stride;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    for (int w = 0; w < kw; w++) t.keys[i * kw + w] = EMPTY;
    for (int j = 0; j < sp.ns; j++) t.states[j * n + i] = state_identity(sp.op[j], sp.ty[j]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    t.hdr->groups = 0;
    t.hdr->frozen = 0;
    t.hdr->esc = 0;
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

struct PassArgs {
  DevSpec sp;
  int32_t mode;
  GTable t;
  // source 1: columnar batch rows [start, n), start = min(n, *start_tiles * start_T)
  ColSrc col;
  int32_t col_dense;                      // all key/value columns 8-byte, stride 8
  const unsigned long long* start_tiles;  // nullable
  int64_t start_T;
  // source 2: SoA list (deferred / overflow records) described as dense columns
  ColSrc lin;                             // lin.nv = payload words of the list
  const unsigned long long* lin_count;    // nullable -> no list
  int32_t lin_kind;                       // 0 raw payload, 1 native partial
  // spill target
  PagePool pool;
  SpillSet ss;
  // ROUTE (original_hh): u32 part hash < cut0 -> partition 0 (table)
  uint32_t cut0;
  uint64_t part_seed;
  // FILL deferral target (raw records, SoA, KW + nv words)
  uint64_t* defer;
  int64_t defer_stride;
  unsigned long long* defer_count;
  unsigned long long* tile_counter;
  unsigned long long* stats;
};

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

// Persistent, tile-scheduled pass.  Per tile: [A] issue the first-bucket loads
// of the current tile's records and prefetch the next tile's records into
// registers, resolve the current records (aggregate hits, rank misses per
// partition in SMEM); [B] one thread per partition reserves page space (CTA-
// private pages, one global atomic per new page) and thread 0 grabs the tile
// after next; [C] every thread writes its spilled / deferred records straight
// from registers.  Two barriers per tile.
template <int KW, int NWT, int R, int BLK = 512, int MINB = 2>
__global__ void __launch_bounds__(BLK, MINB) k_pass(PassArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = BLK, tid = threadIdx.x;
  const int T = R * BLK;
  const bool spills = (a.mode != MODE_FILL);
  const int P = spills ? a.ss.nparts : 1;
  const int S = spills ? a.ss.per_page : 1;

  uint32_t* hist = (uint32_t*)smem;       // P: records of the tile per partition (ranks)
  int32_t* pcur = (int32_t*)(hist + P);   // P: CTA's current page per partition
  int32_t* pfill = pcur + P;              // P: records in that page
  int32_t* bpg = pfill + P;               // P: tile write base: page
  int32_t* bslot = bpg + P;               // P: tile write base: slot (room = S - bslot)
  int32_t* pnew = bslot + P;              // P: first page allocated for this tile
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_grab, s_defer_base;
  __shared__ uint32_t s_ndefer;
  __shared__ unsigned long long s_cnt[ST_NSTATS];

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  for (int p = tid; p < P; p += B) {
    hist[p] = 0;
    pcur[p] = -1;
    pfill[p] = S;
  }
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  const int64_t n = a.col.n;
  const int64_t col_start =
      a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t n_lin = a.lin_count ? (int64_t)*a.lin_count : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (n_lin + T - 1) / T);
  const bool use_table = (a.mode == MODE_FILL || a.mode == MODE_PROBE || a.mode == MODE_ROUTE);
  const bool insert = (a.mode != MODE_PROBE);
  const int nvc = a.col.nv, nvl = a.lin.nv;

  auto grab = [&]() -> unsigned long long {
    if (a.mode == MODE_FILL && *(volatile int*)&a.t.hdr->frozen) return ~0ull;
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

  if (tid == 0) {
    s_ndefer = 0;
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
  while (cur < total) {
    const int kind = ((int64_t)cur < col_tiles) ? 0 : a.lin_kind;
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
      }
      if (use_table && part[r] == -1 && !is_sentinel<KW>(kc[r])) {
        bk[r] = hash_key<KW>(kc[r], a.t.seed) & a.t.bmask;
        ld_bucket(a.t.keys, bk[r], bw[r]);
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
      if (part[r] == -2) continue;
      c_rec++;
      if (part[r] == -1) {
        int res;
        int64_t s = is_sentinel<KW>(kc[r]) ? gt_escape<KW>(a.t, insert, res)
                                            : gt_resolve<KW>(a.t, kc[r], bk[r], bw[r], insert, res);
        if (res == R_HIT || res == R_INSERTED) {
          for (int j = 0; j < ns; j++) {
            uint32_t fd = s_fd[j];
            gupdate(a.t.states + (uint64_t)j * a.t.stride + s, fd & 3, (fd >> 2) & 3,
                    contrib_fd<NWT>(fd, kind, j, vc[r]));
          }
          c_hit += (res == R_HIT);
          c_ins += (res == R_INSERTED);
          continue;
        }
        if (res == R_MISS) {
          part[r] = (int)reduce32(hash_key<KW>(kc[r], a.ss.seed), (uint32_t)P);
        } else if (a.mode == MODE_FILL) {
          tag[r] = 0x80000000u | atomicAdd(&s_ndefer, 1u);
          c_def++;
          continue;
        } else {
          part[r] = 0;  // ROUTE overflow: partition 0 spills raw (hybrid.py:431-451)
        }
      }
      tag[r] = (((uint32_t)part[r] << 16) | atomicAdd(&hist[part[r]], 1u)) + 1u;
      c_sp++;
    }
    __syncthreads();
    // ---- [B] reserve page space per partition; grab the tile after next
    if (spills) {
      for (int p = tid; p < P; p += B) {
        int cnt = (int)hist[p];
        if (!cnt) continue;
        hist[p] = 0;
        int room = S - pfill[p];
        bpg[p] = pcur[p];
        bslot[p] = pfill[p];
        if (cnt > room) {
          int need = (cnt - room + S - 1) / S;
          uint32_t first = atomicAdd(a.pool.next_page, (uint32_t)need);
          if (first + need > a.pool.capacity) {
            atomicExch(a.pool.overflow, 1u);
            pnew[p] = -1;
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
            pfill[p] = (cnt - room) - (need - 1) * S;
          }
          if (bpg[p] >= 0) a.pool.page_fill[bpg[p]] = S;
        } else {
          pfill[p] += cnt;
        }
      }
    }
    if (tid == 0) {
      if (s_ndefer) {
        s_defer_base = atomicAdd(a.defer_count, (unsigned long long)s_ndefer);
        s_ndefer = 0;
      }
      s_grab = (nxt < total) ? grab() : ~0ull;
    }
    __syncthreads();
    // ---- [C] write spilled / deferred records from registers
#pragma unroll
    for (int r = 0; r < R; r++) {
      uint32_t tg = tag[r];
      if (!tg) continue;
      if (tg & 0x80000000u) {
        int64_t d = (int64_t)s_defer_base + (tg & 0x7FFFFFFFu);
#pragma unroll
        for (int w = 0; w < KW; w++) a.defer[w * a.defer_stride + d] = kc[r][w];
#pragma unroll
        for (int w = 0; w < NWT; w++)
          if (w < nvc) a.defer[(KW + w) * a.defer_stride + d] = vc[r][w];
        continue;
      }
      tg -= 1u;
      int p = (int)(tg >> 16);
      int rank = (int)(tg & 0xFFFFu);
      int room = S - bslot[p];
      int32_t pg;
      int slot;
      if (rank < room) {
        pg = bpg[p];
        slot = bslot[p] + rank;
      } else {
        if (pnew[p] < 0) continue;
        int j = rank - room;
        pg = pnew[p] + j / S;
        slot = j % S;
      }
      uint64_t* dst = (uint64_t*)page_ptr(a.pool, (uint32_t)pg) + slot;
#pragma unroll
      for (int w = 0; w < KW; w++) dst[(size_t)w * S] = kc[r][w];
      const int nw = a.ss.rw - KW;
#pragma unroll
      for (int w = 0; w < NWT; w++)
        if (w < nw) dst[(size_t)(KW + w) * S] = vc[r][w];
    }
    // ---- rotate
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
  // seal partially filled pages
  if (spills)
    for (int p = tid; p < P; p += B)
      if (pcur[p] >= 0) a.pool.page_fill[pcur[p]] = pfill[p];
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
}

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

template <int KW>
__global__ void k_flush_table(GTable t, DevSpec sp, OutBuf o) {
  int lane = threadIdx.x & 31;
  uint64_t n = t.stride;
  for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x) & ~31ull; base < n;
       base += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = base + lane + (threadIdx.x & ~31);
    bool occ = false;
    uint64_t k[KW];
    if (s < n) {
#pragma unroll
      for (int w = 0; w < KW; w++) k[w] = t.keys[s * KW + w];
      occ = (s == n - 1) ? (t.hdr->esc != 0) : !is_sentinel<KW>(k);
    }
    unsigned m = __ballot_sync(0xffffffffu, occ);
    if (!m) continue;
    unsigned long long wbase = 0;
    if (lane == 0) wbase = atomicAdd(o.count, (unsigned long long)__popc(m));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (occ) {
      uint64_t st[MAX_STATES];
      for (int j = 0; j < sp.ns; j++) st[j] = t.states[(uint64_t)j * n + s];
      emit_group<KW>(sp, o, (int64_t)(wbase + __popc(m & ((1u << lane) - 1))), k, st);
    }
  }
}

// ---------------------------------------------------------------------------
// k_child: per-partition shared-memory aggregation (one recursion level)
// ---------------------------------------------------------------------------

struct ChildArgs {
  DevSpec sp;
  PagePool pool;
  SpillSet sets[2];         // pages of item i: sets[0] in [off[2i], off[2i+1]), sets[1] in [off[2i+1], off[2i+2])
  const int32_t* plist;     // page ids, grouped by item (set 0 pages first)
  const int64_t* item_off;  // [2 * nitems + 1]
  int32_t nitems;
  int32_t slots_log2;       // SMEM table slots
  int32_t cap;              // group capacity (<= budget)
  uint64_t seed;            // slot hash seed of this level
  OutBuf out;
  uint64_t* ovf;            // overflow list: native partial records, SoA KW + ns words
  int64_t ovf_stride;
  unsigned long long* ovf_count;
  unsigned long long* item_counter;
  unsigned long long* stats;
};

template <int KW>
__device__ __forceinline__ int stable_lookup(uint64_t* keys, int nslots, int cap, const uint64_t (&k)[KW], uint64_t seed,
                                             bool insert, int* s_groups, int* s_frozen, int* s_esc, int& res) {
  if (is_sentinel<KW>(k)) {
    if (*(volatile int*)s_esc) { res = R_HIT; return nslots; }
    if (!insert) { res = R_MISS; return -1; }
    if (*(volatile int*)s_frozen) { res = R_REFUSED; return -1; }
    int old = atomicAdd(s_groups, 1);
    if (old >= cap) { atomicSub(s_groups, 1); atomicExch(s_frozen, 1); res = R_REFUSED; return -1; }
    if (atomicCAS(s_esc, 0, 1) == 0) { res = R_INSERTED; return nslots; }
    atomicSub(s_groups, 1);
    res = R_HIT;
    return nslots;
  }
  int mask = nslots - 1;
  int s = (int)(hash_key<KW>(k, seed) & (uint64_t)mask);
  bool reserved = false;
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
      if (reserved) atomicSub(s_groups, 1);
      res = R_HIT;
      return s;
    }
    if (empty) {
      if (!insert) { res = R_MISS; return -1; }
      if (!reserved) {
        if (*(volatile int*)s_frozen) { res = R_REFUSED; return -1; }
        int old = atomicAdd(s_groups, 1);
        if (old >= cap) { atomicSub(s_groups, 1); atomicExch(s_frozen, 1); res = R_REFUSED; return -1; }
        reserved = true;
      }
      if (KW == 1) {
        unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k[0]);
        if (prev == EMPTY) { res = R_INSERTED; return s; }
        if (prev == k[0]) { atomicSub(s_groups, 1); res = R_HIT; return s; }
      } else {
        uint64_t a, b;
        cas128(kp, EMPTY, EMPTY, k[0], k[KW - 1], a, b);
        if (a == EMPTY && b == EMPTY) { res = R_INSERTED; return s; }
        if (a == k[0] && b == k[KW - 1]) { atomicSub(s_groups, 1); res = R_HIT; return s; }
      }
    }
    s = (s + 1) & mask;
  }
}

// One CTA aggregates one spilled partition (a child operator at level + 1,
// hybrid.py:244-277) in a shared-memory table.  Threads map onto (page, slot)
// across B / per_page pages per row and R rows per round, and the next round's
// records are prefetched into registers while the current round aggregates.
// A refused insert (table full) freezes the table; after the round's barrier
// the key set is immutable, so refused records re-probe and either aggregate
// or go to the overflow list (the next recursion level).
template <int KW, int NWT, int R>
__global__ void __launch_bounds__(512) k_child(ChildArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = blockDim.x, tid = threadIdx.x;
  const int nslots = 1 << a.slots_log2;
  const int stride = nslots + 1;
  const int ns = a.sp.ns;
  uint64_t* skeys = (uint64_t*)smem;                       // stride * KW
  uint64_t* sst = skeys + (size_t)stride * KW;             // ns * stride
  __shared__ int s_groups, s_frozen, s_esc;
  __shared__ unsigned long long s_item;
  __shared__ unsigned long long s_cnt[ST_NSTATS];
  __shared__ uint32_t s_fd[MAX_STATES];
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  uint32_t nrec = 0, novf = 0;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.item_counter, 1ull);
    for (int i = tid; i < stride; i += B) {
#pragma unroll
      for (int w = 0; w < KW; w++) skeys[(size_t)i * KW + w] = EMPTY;
      for (int j = 0; j < ns; j++) sst[(size_t)j * stride + i] = state_identity(a.sp.op[j], a.sp.ty[j]);
    }
    if (tid == 0) {
      s_groups = 0;
      s_frozen = 0;
      s_esc = 0;
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
      const int S = ss.per_page;
      const int ppr = B / S;                   // pages per row
      const int prow = tid / S, slot = tid % S;
      const int64_t per_round = (int64_t)R * ppr;
      auto load_round = [&](int64_t q0, uint64_t (&k)[R][KW], uint64_t (&v)[R][NWT], bool (&live)[R]) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          int64_t q = q0 + (int64_t)r * ppr + prow;
          live[r] = false;
          if (prow < ppr && q < qb) {
            uint32_t pg = (uint32_t)a.plist[q];
            if (slot < a.pool.page_fill[pg]) {
              live[r] = true;
              soa_load<KW, NWT>((const uint64_t*)page_ptr(a.pool, pg), S, slot, nw, k[r], v[r]);
            }
          }
        }
      };
      uint64_t kc[R][KW], vc[R][NWT];
      bool lc[R];
      load_round(qa, kc, vc, lc);
      for (int64_t q0 = qa; q0 < qb; q0 += per_round) {
        uint64_t kn[R][KW], vn[R][NWT];
        bool ln[R];
        load_round(q0 + per_round, kn, vn, ln);
        bool refused[R];
        bool any_ref = false;
#pragma unroll
        for (int r = 0; r < R; r++) {
          refused[r] = false;
          if (!lc[r]) continue;
          nrec++;
          int res;
          int s = stable_lookup<KW>(skeys, nslots, a.cap, kc[r], a.seed, true, &s_groups, &s_frozen, &s_esc, res);
          if (res == R_REFUSED) {
            refused[r] = true;
            any_ref = true;
            continue;
          }
          for (int j = 0; j < ns; j++) {
            uint32_t fd = s_fd[j];
            supdate(sst + (size_t)j * stride + s, fd & 3, (fd >> 2) & 3, contrib_fd<NWT>(fd, kind, j, vc[r]));
          }
        }
        // the table's key set is immutable once frozen and this barrier has passed
        if (__syncthreads_or(any_ref)) {
#pragma unroll
          for (int r = 0; r < R; r++) {
            if (!refused[r]) continue;
            int res;
            int s = stable_lookup<KW>(skeys, nslots, a.cap, kc[r], a.seed, false, &s_groups, &s_frozen, &s_esc, res);
            if (res == R_HIT) {
              for (int j = 0; j < ns; j++) {
                uint32_t fd = s_fd[j];
                supdate(sst + (size_t)j * stride + s, fd & 3, (fd >> 2) & 3, contrib_fd<NWT>(fd, kind, j, vc[r]));
              }
            } else {
              unsigned long long d = atomicAdd(a.ovf_count, 1ull);
              novf++;
#pragma unroll
              for (int w = 0; w < KW; w++) a.ovf[w * a.ovf_stride + d] = kc[r][w];
              for (int j = 0; j < ns; j++) a.ovf[(KW + j) * a.ovf_stride + d] = contrib_fd<NWT>(s_fd[j], kind, j, vc[r]);
            }
          }
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
    atomicAdd(&part_records[p], (unsigned long long)pool.page_fill[pg]);
    atomicAdd(&part_pages[p], 1u);
  }
}

__global__ void k_page_scatter(PagePool pool, uint32_t first, const uint32_t* last_ptr, int set_id, int nparts,
                               uint32_t* cursor /* exclusive offsets, advanced */, int32_t* plist) {
  uint32_t last = min(*last_ptr, pool.capacity);
  for (uint32_t pg = first + blockIdx.x * blockDim.x + threadIdx.x; pg < last; pg += gridDim.x * blockDim.x) {
    if (pool.page_set[pg] != set_id) continue;
    int p = pool.page_part[pg];
    if (p < 0 || p >= nparts) continue;
    if (pool.page_fill[pg] == 0) continue;
    uint32_t at = atomicAdd(&cursor[p], 1u);
    plist[at] = (int32_t)pg;
  }
}

// ---------------------------------------------------------------------------
// output egress: key words -> typed key columns
// ---------------------------------------------------------------------------

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
