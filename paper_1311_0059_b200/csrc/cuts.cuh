// cuts.cuh — hash_sort's blind cuts as one persistent launch (hash_sort.py:40-78:
// aggregate until the table is full, cut it to a run of partial states, go on).
//
// When the table holds far fewer groups than the input has (C5: 84K of 4.19M),
// every chunk of `cap` records fills it, and a launch pair per cut (FILL + flush
// and clear: ~66 us for 84K records) made the 6,000 cuts of a 500M-record batch
// slow (FILL 217 ms + flush 181 ms; not the launches themselves: each of the small
// kernels is a chain of L2 round trips).  k_blind_cuts keeps the cut loop on the
// device, one 1,024-thread CTA per SM (the grid barrier costs per CTA; more CTAs
// measured slower), two table slots per thread in the flush: the grid aggregates one chunk into the L2-resident table, meets at
// a grid barrier, flushes the table as a run of partial states into the
// accumulation buffer while clearing it, meets again, and takes the next chunk.
// A chunk has at most `cap` records, so it can hold at most `cap` keys: no
// capacity reservations (the table has >= 2 slots per key).  The runs are
// hash-partitioned and merged exactly as the host-driven cuts' runs are.
#pragma once
#include "pass.cuh"

namespace aggb {

struct CutArgs {
  GTable t;
  DevSpec sp;
  ColSrc col;                  // the batch
  int64_t first, chunk;        // chunk k covers records [first + k * chunk, first + (k + 1) * chunk)
  int64_t nchunks;
  OutBuf o;                    // accumulation buffer (partial states), count appended across chunks
  unsigned* bar;               // [2] grid barrier: arrivals, generation
  unsigned long long* stats;   // ST_* counters
};

// all CTAs of the (co-resident, cooperatively launched) grid
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned gen = *(volatile unsigned*)(bar + 1);
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      *(volatile unsigned*)bar = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*(volatile unsigned*)(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// find or insert key k (first bucket b loaded into w): no capacity bound
template <int KW>
__device__ __forceinline__ int64_t blind_insert(const GTable& t, const uint64_t (&k)[KW], uint64_t b, uint64_t (&w)[4]) {
  constexpr int BK = Bkt<KW>::N;
  int from = 0;
  for (;;) {
    int hit = -1, emp = -1;
#pragma unroll
    for (int j = 0; j < BK; j++) {
      if (j < from || hit >= 0 || emp >= 0) continue;
      uint64_t a0 = w[j * KW], a1 = (KW == 2) ? w[j * KW + 1] : 0ull;
      if (KW == 2 && ((a0 == EMPTY) != (a1 == EMPTY))) {
        uint64_t x, y;  // possibly torn while another thread inserts: read atomically
        cas128(t.keys + (b * BK + j) * KW, EMPTY, EMPTY, EMPTY, EMPTY, x, y);
        a0 = x;
        a1 = y;
      }
      if (a0 == k[0] && (KW == 1 || a1 == k[KW - 1])) hit = j;
      else if (a0 == EMPTY && (KW == 1 || a1 == EMPTY)) emp = j;
    }
    if (hit >= 0) return (int64_t)(b * BK + hit);
    if (emp >= 0) {
      uint64_t* kp = t.keys + (b * BK + emp) * KW;
      if (KW == 1) {
        const unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k[0]);
        if (prev == EMPTY || prev == k[0]) return (int64_t)(b * BK + emp);
      } else {
        uint64_t x, y;
        cas128(kp, EMPTY, EMPTY, k[0], k[KW - 1], x, y);
        if ((x == EMPTY && y == EMPTY) || (x == k[0] && y == k[KW - 1])) return (int64_t)(b * BK + emp);
      }
      ld_bucket(t.keys, b, w);  // another key took the slot: rescan this bucket after it
      from = emp + 1;
      if (from < BK) continue;
    }
    b = (b + 1) & t.bmask;
    from = 0;
    ld_bucket(t.keys, b, w);
  }
}

constexpr int CUT_BLK = 1024;  // one CTA per SM: the grid barrier costs per CTA, the chunk needs threads

template <int KW, int NWT, class PG>
__global__ void __launch_bounds__(CUT_BLK, 1) k_blind_cuts(CutArgs a) {
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ uint32_t s_wc[CUT_BLK / 32];
  __shared__ unsigned long long s_base;
  const int ns = a.sp.ns;
  if (threadIdx.x < ns) s_fd[threadIdx.x] = field_desc(a.sp, threadIdx.x);
  __syncthreads();
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x, gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long nrec = 0;
  for (int64_t c = 0; c < a.nchunks; c++) {
    const int64_t lo = a.first + c * a.chunk, hi = min(a.col.n, lo + a.chunk);
    // ---- aggregate the chunk (L2 table: CAS-claimed keys, RED updates)
    for (int64_t i = lo + gtid; i < hi; i += gsize) {
      uint64_t k[KW], v[NWT];
      col_key<KW>(a.col, i, k);
      col_vals<NWT>(a.col, i, v);
      int64_t sl;
      if (is_sentinel<KW>(k)) {
        sl = (int64_t)a.t.mask + 1;
        if (!*(volatile int*)&a.t.hdr->esc) atomicExch(&a.t.hdr->esc, 1);
      } else {
        const uint64_t b = hash_key<KW>(k, a.t.seed) & a.t.bmask;
        uint64_t w[4];
        ld_bucket(a.t.keys, b, w);
        sl = blind_insert<KW>(a.t, k, b, w);
      }
      Upd<PG>::template g<NWT>(a.t.states, a.t.fstride, (uint64_t)sl * a.t.sstride, 0, s_fd, ns, v);
      nrec++;
    }
    grid_barrier(a.bar, gridDim.x);
    // ---- cut: the table as a run of partial states, cleared on the way
    flush_tiles<KW, true, CUT_BLK, 2>(a.t, a.sp, a.o, s_wc, &s_base);  // (2 slots per thread: every CTA has a tile)
    grid_barrier(a.bar, gridDim.x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nrec += __shfl_xor_sync(0xffffffffu, nrec, o);
  if ((threadIdx.x & 31) == 0 && nrec) atomicAdd(&a.stats[ST_RECORDS], nrec);
}

}  // namespace aggb
