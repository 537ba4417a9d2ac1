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

template <class PG>
__device__ __forceinline__ bool probe_resolve(const PassArgs& a, uint64_t k, uint64_t v, const uint32_t* s_fd, int ns) {
  int64_t s = -1;
  if (k == EMPTY) {  // escape slot: the key whose word equals the sentinel
    if (*(volatile int*)&a.t.hdr->esc) s = (int64_t)a.t.mask + 1;
  } else {
    const uint64_t kk[1] = {k};
    uint64_t b = hash_key<1>(kk, a.t.seed) & a.t.bmask;
    for (;;) {
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(a.t.keys + b * 4);
      const ulonglong2 x = __ldcg(p), y = __ldcg(p + 1);
      if (x.x == k) { s = (int64_t)(b * 4); break; }
      if (x.y == k) { s = (int64_t)(b * 4 + 1); break; }
      if (y.x == k) { s = (int64_t)(b * 4 + 2); break; }
      if (y.y == k) { s = (int64_t)(b * 4 + 3); break; }
      if ((x.x == EMPTY) | (x.y == EMPTY) | (y.x == EMPTY) | (y.y == EMPTY)) break;
      b = (b + 1) & a.t.bmask;
    }
  }
  if (s < 0) return false;
  const uint64_t vv[1] = {v};
  Upd<PG>::template g<1>(a.t.states, a.t.stride, (uint64_t)s, 0, s_fd, ns, vv);
  return true;
}

template <int R, int BLK, class PG>
__global__ void __launch_bounds__(BLK, 1) k_probe(PassArgs a) {
  constexpr int T = R * BLK, NWARP = BLK / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int P = a.ss.nparts, S = a.ss.per_page;
  const int nbw = a.bloom.words ? (int)a.bloom.mask + 1 : 0;
  uint64_t* sbloom = (uint64_t*)smem;
  ulonglong2* ring = (ulonglong2*)(sbloom + ((nbw + 1) & ~1)) + wid * PQ_RING;  // this warp's ring (16-B aligned)
  ulonglong2* resid = (ulonglong2*)(sbloom + ((nbw + 1) & ~1)) + NWARP * PQ_RING;  // P: one pending record each
  uint32_t* hist = (uint32_t*)(resid + P);
  int32_t* pcur = (int32_t*)(hist + P);
  int32_t* pfill = pcur + P;
  int32_t* bpg = pfill + P;
  int32_t* bslot = bpg + P;
  int32_t* pnew = bslot + P;
  uint32_t* rcnt = (uint32_t*)(pnew + P);
  uint32_t* rprev = rcnt + P;
  uint32_t* emitn = rprev + P;
  uint16_t* touched = (uint16_t*)(emitn + P);
  __shared__ uint32_t s_ntouched[2];
  __shared__ uint32_t s_fd[MAX_STATES];
  __shared__ unsigned long long s_grab;
  __shared__ uint32_t s_sbase, s_sused, s_scap;
  __shared__ unsigned long long s_cnt[ST_NSTATS];

  const int64_t n = a.col.n;
  const int64_t col_start =
      a.start_tiles ? (int64_t)min((unsigned long long)n, *a.start_tiles * (unsigned long long)a.start_T) : 0;
  const int64_t col_tiles = (n - col_start + T - 1) / T;
  const int64_t n_lin = a.lin_count ? (int64_t)*a.lin_count : 0;
  const unsigned long long total = (unsigned long long)(col_tiles + (n_lin + T - 1) / T);
  if (total == 0) return;  // FILL took the whole batch: no spill state to seal

  const int ns = a.sp.ns;
  if (tid < ns) s_fd[tid] = field_desc(a.sp, tid);
  for (int p = tid; p < P; p += BLK) {
    hist[p] = 0;
    pcur[p] = -1;
    pfill[p] = S;
    rcnt[p] = 0;
  }
  if (tid < ST_NSTATS) s_cnt[tid] = 0;
  for (int i = tid; i < nbw; i += BLK) sbloom[i] = __ldcg((const unsigned long long*)a.bloom.words + i);

  auto load_tile = [&](unsigned long long tile, uint64_t (&k)[R], uint64_t (&v)[R], bool (&live)[R]) {
    const int src = (int64_t)tile < col_tiles ? 0 : 1;
    const int64_t base = src == 0 ? col_start + (int64_t)tile * T : ((int64_t)tile - col_tiles) * T;
    const int64_t end = src == 0 ? n : n_lin;
    const long long* kp = (const long long*)(src == 0 ? a.col.key[0] : a.lin.key[0]);
    const long long* vp = (const long long*)(src == 0 ? a.col.val[0] : a.lin.val[0]);
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
  auto emit_at = [&](int p, int pos, int32_t& pg, int& slot) -> bool {
    const int room = S - bslot[p];
    if (pos < room) {
      pg = bpg[p];
      slot = bslot[p] + pos;
      return pg >= 0;
    }
    if (pnew[p] < 0) return false;
    const int j = pos - room;
    pg = pnew[p] + j / S;
    slot = j % S;
    return true;
  };

  if (tid == 0) {
    s_sbase = s_sused = s_scap = 0;
    s_ntouched[0] = s_ntouched[1] = 0;
    s_grab = atomicAdd(a.tile_counter, 1ull);
  }
  __syncthreads();
  unsigned long long cur = s_grab;
  __syncthreads();
  if (tid == 0) s_grab = (cur < total) ? atomicAdd(a.tile_counter, 1ull) : ~0ull;
  uint64_t kc[R], vc[R];
  bool lc[R];
  load_tile(cur, kc, vc, lc);
  __syncthreads();
  unsigned long long nxt = s_grab;

  uint32_t c_hit = 0, c_rec = 0, c_sp = 0;
  int par = 0;
  const uint32_t lt_mask = (1u << lane) - 1u;
  while (cur < total) {
    const bool refill = a.stash && tid == 0 && s_scap - min(s_sused, s_scap) < (uint32_t)a.stash / 2;
    uint32_t ref_first = 0;
    if (refill) ref_first = atomicAdd(a.pool.next_page, (uint32_t)a.stash);
    // ---- [A] classify: hash once, partition from the high bits, bloom from a remix
    int part[R];
    uint32_t seq[R];  // ring sequence number of a bloom-positive record, ~0u otherwise
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t kk[1] = {kc[r]};
      const uint64_t h = hash_key<1>(kk, a.t.seed);
      part[r] = kc[r] == EMPTY ? 0 : (int)reduce32(h, (uint32_t)P);
      bool posv = lc[r];
      if (nbw && kc[r] != EMPTY) {
        const uint64_t hb = bloom_remix(h);
        const uint64_t bits = bloom_bits(hb);
        posv = posv && (sbloom[(hb >> 8) & a.bloom.mask] & bits) == bits;
      }
      seq[r] = posv ? 0u : ~0u;
    }
    // ---- prefetch the next tile
    uint64_t kn[R], vn[R];
    bool ln[R];
    load_tile(nxt, kn, vn, ln);
    // ---- resolve the bloom positives 32 at a time
    uint32_t hm[R];  // hit mask of round q (records with seq in [32q, 32q + 32))
#pragma unroll
    for (int q = 0; q < R; q++) hm[q] = 0;
    uint32_t qt = 0, qh = 0;  // warp-uniform ring tail / head
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
        __syncwarp();
        const ulonglong2 e = ring[(qh + lane) & (PQ_RING - 1)];
        const bool hit = probe_resolve<PG>(a, e.x, e.y, s_fd, ns);
        const uint32_t hb = __ballot_sync(0xffffffffu, hit);
#pragma unroll
        for (int q = 0; q < R; q++)
          if ((int)(qh >> 5) == q) hm[q] = hb;
        qh += 32;
        __syncwarp();
      }
    }
    if (qt != qh) {
      __syncwarp();
      bool hit = false;
      if (lane < (int)(qt - qh)) {
        const ulonglong2 e = ring[(qh + lane) & (PQ_RING - 1)];
        hit = probe_resolve<PG>(a, e.x, e.y, s_fd, ns);
      }
      const uint32_t hb = __ballot_sync(0xffffffffu, hit);
#pragma unroll
      for (int q = 0; q < R; q++)
        if ((int)(qh >> 5) == q) hm[q] = hb;
      __syncwarp();
    }
    // ---- claim spill ranks
    uint32_t tag[R];  // (p << 16 | rank) + 1, 0 = nothing to write
#pragma unroll
    for (int r = 0; r < R; r++) {
      tag[r] = 0;
      c_rec += lc[r];
      bool spill = lc[r];
      if (seq[r] != ~0u) {
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < R; q++)
          if ((int)(seq[r] >> 5) == q) m = hm[q];
        const bool hit = (m >> (seq[r] & 31)) & 1u;
        c_hit += hit;
        spill = !hit;
      }
      if (spill) {
        const uint32_t rank = atomicAdd(&hist[part[r]], 1u);
        if (rank == 0) touched[atomicAdd(&s_ntouched[par], 1u)] = (uint16_t)part[r];
        tag[r] = (((uint32_t)part[r] << 16) | rank) + 1u;
        c_sp++;
      }
    }
    if (refill) {
      for (uint32_t q = min(s_sused, s_scap); q < s_scap; q++) a.pool.page_set[s_sbase + q] = -1;
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
    // ---- [B] per touched partition: reserve whole sectors (pairs), drain the residual
    {
      const int nt = (int)s_ntouched[par];
      for (int ti = tid; ti < nt; ti += BLK) {
        const int p = touched[ti];
        const int c = (int)hist[p];
        hist[p] = 0;
        const int r0 = (int)rcnt[p];
        const int t = r0 + c;
        const int e = t & ~1;
        rprev[p] = (uint32_t)r0;
        emitn[p] = (uint32_t)e;
        rcnt[p] = (uint32_t)(t & 1);
        if (!e) continue;
        const int room = S - pfill[p];
        bpg[p] = pcur[p];
        bslot[p] = pfill[p];
        pnew[p] = -1;
        if (e > room) {
          const int need = (e - room + S - 1) / S;
          uint32_t first;
          const uint32_t off = atomicAdd(&s_sused, (uint32_t)need);
          if (off + need <= s_scap) {
            first = s_sbase + off;
          } else {
            for (uint32_t q = off; q < min(off + (uint32_t)need, s_scap); q++) a.pool.page_set[s_sbase + q] = -1;
            first = atomicAdd(a.pool.next_page, (uint32_t)need);
          }
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
        if (r0) {  // the pending record leads this tile's emission
          int32_t pg;
          int slot;
          if (emit_at(p, 0, pg, slot)) *((ulonglong2*)page_ptr(a.pool, (uint32_t)pg) + slot) = resid[p];
        }
      }
    }
    if (tid == 0) {
      s_grab = (nxt < total) ? atomicAdd(a.tile_counter, 1ull) : ~0ull;
      s_ntouched[par ^ 1] = 0;
    }
    __syncthreads();
    // ---- [C] write the spilled records from registers
#pragma unroll
    for (int r = 0; r < R; r++) {
      uint32_t tg = tag[r];
      if (!tg) continue;
      tg -= 1u;
      const int p = (int)(tg >> 16);
      const int pos = (int)rprev[p] + (int)(tg & 0xFFFFu);
      const ulonglong2 rec = make_ulonglong2(kc[r], vc[r]);
      if (pos < (int)emitn[p]) {
        int32_t pg;
        int slot;
        if (emit_at(p, pos, pg, slot)) *((ulonglong2*)page_ptr(a.pool, (uint32_t)pg) + slot) = rec;
      } else {
        resid[p] = rec;
      }
    }
    par ^= 1;
    cur = nxt;
    nxt = s_grab;
#pragma unroll
    for (int r = 0; r < R; r++) {
      lc[r] = ln[r];
      kc[r] = kn[r];
      vc[r] = vn[r];
    }
  }
  __syncthreads();
  for (uint32_t q = min(s_sused, s_scap) + tid; q < s_scap; q += BLK) a.pool.page_set[s_sbase + q] = -1;
  // flush the pending records (one per partition at most) and seal the pages
  for (int p = tid; p < P; p += BLK) {
    if (rcnt[p]) {
      if (S - pfill[p] < 1) {
        const uint32_t pg = atomicAdd(a.pool.next_page, 1u);
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
      *((ulonglong2*)page_ptr(a.pool, (uint32_t)pcur[p]) + pfill[p]) = resid[p];
      pfill[p] += 1;
    }
    if (pcur[p] >= 0) a.pool.page_fill[pcur[p]] = pfill[p];
  }
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

}  // namespace aggb
