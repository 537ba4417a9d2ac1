// proto_c2.cu — standalone measurement of k_probe_wc + k_child_wc on the C2
// shape (100M int64 records, keys uniform over 1M, values in [0, 1000),
// COUNT/SUM/MIN/MAX, a 125K-group resident table), checked against a direct
// per-key ground truth.  Not part of the product; build with tools/proto/build.sh.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include "../../paper_1311_0059_b200/csrc/wc.cuh"

using namespace aggb;

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));      \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

__global__ void k_gen_proto(unsigned long long* key, unsigned long long* val, int64_t n, uint64_t G, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = fmix64((uint64_t)i * 2 + 1 + seed * 0x9E3779B97F4A7C15ull);
    const uint64_t b = fmix64(a ^ 0xABCDEF12345ull);
    key[i] = a % G;
    val[i] = b % 1000;
  }
}

// toy FILL: first F records; first-come inserts until cap, the rest deferred
__global__ void k_fill_proto(GTable t, DevSpec sp, const unsigned long long* key, const unsigned long long* val,
                             int64_t F, unsigned long long* lkey, unsigned long long* lval, unsigned long long* lcount) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i], v = val[i];
    const uint64_t kk[1] = {k};
    const uint64_t h = hash_key<1>(kk, t.seed);
    uint64_t b = h & t.bmask;
    int64_t slot = -1;
    bool deferred = false;
    for (int guard = 0; guard < 1 << 20 && slot < 0 && !deferred; guard++) {
      for (int j = 0; j < 4; j++) {
        uint64_t* kp = t.keys + b * 4 + j;
        uint64_t cur = *(volatile uint64_t*)kp;
        if (cur == k) { slot = b * 4 + j; break; }
        if (cur == EMPTY) {
          if (atomicAdd(&t.hdr->groups, 1ull) >= t.cap) { deferred = true; break; }
          unsigned long long prev = atomicCAS((unsigned long long*)kp, EMPTY, k);
          if (prev == EMPTY) { slot = b * 4 + j; break; }
          atomicAdd(&t.hdr->groups, (unsigned long long)-1ll);  // give the reservation back
          if (prev == k) { slot = b * 4 + j; break; }
          j--;  // re-read this slot
          continue;
        }
      }
      b = (b + 1) & t.bmask;
    }
    if (deferred) {
      unsigned long long d = atomicAdd(lcount, 1ull);
      lkey[d] = k;
      lval[d] = v;
      continue;
    }
    const uint64_t vv[1] = {v};
    Upd<ProgC2>::g<1>(t.states, t.fstride, (uint64_t)slot * t.sstride, 0, nullptr, 4, vv);
  }
}

__global__ void k_truth(const unsigned long long* key, const unsigned long long* val, int64_t n, unsigned long long* tc,
                        long long* ts, long long* tmin, long long* tmax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    const long long v = (long long)val[i];
    atomicAdd(&tc[k], 1ull);
    atomicAdd((unsigned long long*)&ts[k], (unsigned long long)v);
    atomicMin(&tmin[k], v);
    atomicMax(&tmax[k], v);
  }
}

__global__ void k_flush_proto(GTable t, OutBuf o) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= t.mask; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = t.keys[s];
    if (k == EMPTY) continue;
    unsigned long long i = atomicAdd(o.count, 1ull);
    o.keys[i] = k;
    for (int j = 0; j < 4; j++) o.vals[j * o.cap + i] = t.states[j * t.fstride + s * t.sstride];
  }
}

__global__ void k_verify(OutBuf o, int64_t nout, const unsigned long long* tc, const long long* ts, const long long* tmin,
                         const long long* tmax, unsigned int* seen, unsigned long long* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nout; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = o.keys[i];
    if (k >= (1ull << 20)) { atomicAdd(&bad[0], 1ull); continue; }
    atomicAdd(&seen[k], 1u);
    const long long c = (long long)o.vals[0 * o.cap + i], s = (long long)o.vals[1 * o.cap + i];
    const long long mn = (long long)o.vals[2 * o.cap + i], mx = (long long)o.vals[3 * o.cap + i];
    if (c != (long long)tc[k]) atomicAdd(&bad[1], 1ull);
    if (s != ts[k]) atomicAdd(&bad[2], 1ull);
    if (mn != tmin[k] || mx != tmax[k]) atomicAdd(&bad[3], 1ull);
  }
}
__global__ void k_verify2(const unsigned long long* tc, const unsigned int* seen, int64_t G, unsigned long long* bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < G; k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned e = tc[k] ? 1u : 0u;
    if (seen[k] != e) atomicAdd(&bad[4], 1ull);
  }
}

template <class T>
T* dalloc(size_t n) {
  T* p;
  CK(cudaMalloc(&p, n * sizeof(T) + 256));
  return p;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 100000000LL;
  const int P = argc > 2 ? atoi(argv[2]) : 148;
  const int variant = argc > 3 ? atoi(argv[3]) : 0;  // 0: LINES 2 bloom 96K; 1: LINES 4 bloom 64K; 2: LINES 2 bloom 128K
  const int iters = argc > 4 ? atoi(argv[4]) : 5;
  const uint64_t G = 1000000;
  const int64_t F = 262144;  // FILL prefix
  const uint64_t cap = 125000;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  printf("N=%lld P=%d variant=%d sms=%d\n", (long long)N, P, variant, sms);

  unsigned long long* key = dalloc<unsigned long long>(N);
  unsigned long long* val = dalloc<unsigned long long>(N);
  k_gen_proto<<<sms * 8, 512>>>(key, val, N, G, 2);
  // table
  const uint64_t slots = 262144;
  GTable t;
  memset(&t, 0, sizeof(t));
  t.stride = slots + 1;
  t.mask = slots - 1;
  t.fstride = slots + 1;
  t.sstride = 1;
  t.bmask = slots / 4 - 1;
  t.cap = cap;
  t.seed = 0x1234567ull;
  t.keys = dalloc<uint64_t>((slots + 2));
  t.states = dalloc<uint64_t>((slots + 1) * 4);
  t.hdr = dalloc<TableHdr>(1);
  DevSpec sp;
  memset(&sp, 0, sizeof(sp));
  sp.ns = 4;
  sp.nv = 1;
  const uint8_t ops[4] = {OP_ADD, OP_ADD, OP_MIN, OP_MAX};
  for (int j = 0; j < 4; j++) {
    sp.op[j] = ops[j];
    sp.ty[j] = TY_I64;
    sp.srck[j] = j == 0 ? SRC_ONE : SRC_VAL;
    sp.src[j] = 0;
  }
  sp.vty[0] = TY_I64;
  sp.nout = 4;
  for (int j = 0; j < 4; j++) {
    sp.fin_div[j] = 0;
    sp.fin_a[j] = j;
    sp.out_ty[j] = TY_I64;
  }
  std::vector<uint64_t> hinit((slots + 1) * 4);
  for (uint64_t s = 0; s <= slots; s++) {
    hinit[0 * (slots + 1) + s] = 0;
    hinit[1 * (slots + 1) + s] = 0;
    hinit[2 * (slots + 1) + s] = 0x7FFFFFFFFFFFFFFFull;
    hinit[3 * (slots + 1) + s] = 0x8000000000000000ull;
  }
  unsigned long long* lkey = dalloc<unsigned long long>(F);
  unsigned long long* lval = dalloc<unsigned long long>(F);
  unsigned long long* ctr = dalloc<unsigned long long>(64);
  // bloom
  const int lines = variant == 1 ? 4 : 2;
  const uint32_t nblk = variant == 1 ? 8192 : variant == 2 ? 10240 : 11264;
  uint64_t* bloom = dalloc<uint64_t>(nblk);
  // pool
  const uint32_t page_bytes = 8192;
  const uint64_t pool_pages = (uint64_t)(N / 512) + (uint64_t)sms * P * 2 + 100000;
  uint8_t* pbase = dalloc<uint8_t>(pool_pages * page_bytes);
  int32_t* page_part = dalloc<int32_t>(pool_pages);
  int32_t* page_fill = dalloc<int32_t>(pool_pages);
  int32_t* page_set = dalloc<int32_t>(pool_pages);
  const uint32_t plist_cap = (uint32_t)((N / 512) / P * 2 + 2 * sms + 64);
  uint32_t* plist = dalloc<uint32_t>((size_t)P * plist_cap);
  uint32_t* plist_n = dalloc<uint32_t>(P);
  unsigned long long* part_recs = dalloc<unsigned long long>(P);
  unsigned int* vinfo = dalloc<unsigned int>(2);
  const int64_t pos_stride = ((N / 1024 + 1) / sms + 2) * 1024;
  uint64_t* posb = dalloc<uint64_t>((size_t)pos_stride * 2 * sms);
  unsigned long long* pos_count = dalloc<unsigned long long>(sms);
  uint32_t* failw = dalloc<uint32_t>(4);
  uint32_t* failed = dalloc<uint32_t>(P);
  // output
  const int64_t ocap = 1100000;
  OutBuf o;
  o.keys = dalloc<uint64_t>(ocap);
  o.vals = dalloc<uint64_t>(ocap * 4);
  o.cap = ocap;
  o.count = dalloc<unsigned long long>(1);
  o.partial = 0;
  // truth
  unsigned long long* tc = dalloc<unsigned long long>(G);
  long long* ts = dalloc<long long>(G);
  long long* tmin = dalloc<long long>(G);
  long long* tmax = dalloc<long long>(G);
  unsigned int* seen = dalloc<unsigned int>(G);
  unsigned long long* bad = dalloc<unsigned long long>(8);
  CK(cudaMemset(tc, 0, G * 8));
  CK(cudaMemset(ts, 0, G * 8));
  {
    std::vector<long long> mn(G, LLONG_MAX), mx(G, LLONG_MIN);
    CK(cudaMemcpy(tmin, mn.data(), G * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(tmax, mx.data(), G * 8, cudaMemcpyHostToDevice));
  }
  k_truth<<<sms * 8, 512>>>(key, val, N, tc, ts, tmin, tmax);
  CK(cudaDeviceSynchronize());

  #ifndef PBLK
#define PBLK 512
#endif
#ifndef PNS
#define PNS 3
#endif
  constexpr int BLK = PBLK, NS = PNS, RR = 1024 / PBLK;
  auto* fn0 = k_probe_wc<ProgC2, BLK, RR, NS, 2>;
  auto* fn1 = k_probe_wc<ProgC2, BLK, RR, NS, 4>;
  auto* fnp = lines == 4 ? fn1 : fn0;
  const size_t psmem = lines == 4 ? WcLayout<BLK, RR, NS, 4>::bytes(P, nblk) : WcLayout<BLK, RR, NS, 2>::bytes(P, nblk);
  printf("probe smem %zu bytes\n", psmem);
  CK(cudaFuncSetAttribute((const void*)fnp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
  auto* fnr = k_resolve_wc<ProgC2, 512, 4>;
  const size_t rsmem = (size_t)P * 4 * 9;
  constexpr int CBLK = 1024;
  #ifndef CRL
#define CRL 4
#endif
  auto* fnc = k_child_wc<CpC2, CBLK, CRL>;
  const int csmem = 220 * 1024;
  CK(cudaFuncSetAttribute((const void*)fnc, cudaFuncAttributeMaxDynamicSharedMemorySize, csmem));

  cudaEvent_t e[8];
  for (int i = 0; i < 8; i++) CK(cudaEventCreate(&e[i]));
  double tp = 0, tc_ = 0, tf = 0, tall = 0;
  int meas = 0;
  for (int itx = 0; itx < iters; itx++) {
    // reset
    CK(cudaMemset(t.keys, 0x00, (slots + 2) * 8));
    {
      std::vector<uint64_t> ek(slots + 2, EMPTY);
      CK(cudaMemcpy(t.keys, ek.data(), (slots + 2) * 8, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(t.states, hinit.data(), hinit.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(t.hdr, 0, sizeof(TableHdr)));
    CK(cudaMemset(ctr, 0, 64 * 8));
    CK(cudaMemset(bloom, 0, nblk * 8));
    CK(cudaMemset(plist_n, 0, P * 4));
    CK(cudaMemset(part_recs, 0, P * 8));
    CK(cudaMemset(failw, 0, 16));
    CK(cudaMemset(failed, 0, P * 4));
    CK(cudaMemset(o.count, 0, 8));
    CK(cudaMemset(vinfo, 0, 8));
    CK(cudaMemset(page_set, 0xFF, pool_pages * 4));
    // ctr: [0] lcount [1] tile counter [2] next_page [3] overflow(u32) [8..15] stats
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e[0]));
    k_fill_proto<<<sms * 4, 256>>>(t, sp, key, val, F, lkey, lval, ctr + 0);
    k_bloom_build_wc<<<sms * 4, 256>>>(t, bloom, nblk);
    CK(cudaEventRecord(e[1]));
    WcArgs a;
    memset(&a, 0, sizeof(a));
    a.sp = sp;
    a.t = t;
    a.key = key;
    a.val = val;
    a.n = N;
    a.start_tiles = ctr + 20;  // holds 1
    a.start_T = F;
    a.lkey = lkey;
    a.lval = lval;
    a.lcount = ctr + 0;
    a.bloom = bloom;
    a.nblk = nblk;
    a.pool.base = pbase;
    a.pool.page_bytes = page_bytes;
    a.pool.next_page = (uint32_t*)(ctr + 2);
    a.pool.capacity = (uint32_t)pool_pages;
    a.pool.page_part = page_part;
    a.pool.page_fill = page_fill;
    a.pool.page_set = page_set;
    a.pool.overflow = (uint32_t*)(ctr + 3);
    a.ss.id = 1;
    a.ss.nparts = P;
    a.ss.rw = 2;
    a.ss.per_page = 512;
    a.plist = plist;
    a.plist_n = plist_n;
    a.plist_cap = plist_cap;
    a.part_recs = part_recs;
    a.tile_counter = ctr + 1;
    a.stats = ctr + 8;
    a.vinfo = vinfo;
    a.fail = failw;
    a.stash = 32;
    a.pos = posb;
    a.pos_stride = pos_stride;
    a.pos_count = pos_count;
    a.pos_regions = sms;
    {
      unsigned long long one = 1;
      CK(cudaMemcpy(ctr + 20, &one, 8, cudaMemcpyHostToDevice));
    }
    CK(cudaEventRecord(e[1]));
    fnp<<<sms, BLK, psmem>>>(a);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e[5]));
    a.tile_counter = ctr + 30;
    fnr<<<sms, 512, rsmem>>>(a);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e[2]));
    CwArgs ca;
    memset(&ca, 0, sizeof(ca));
    ca.sp = sp;
    ca.pool = a.pool;
    ca.plist = plist;
    ca.plist_n = plist_n;
    ca.plist_cap = plist_cap;
    ca.part_recs = part_recs;
    ca.vinfo = vinfo;
    ca.P = P;
    ca.table_bytes = csmem;
    ca.seed = 0x9876543ull;
    ca.out = o;
    ca.failed = failed;
    ca.fail = failw + 1;
    ca.stats = ctr + 8;
    fnc<<<std::min(P, sms), CBLK, csmem>>>(ca);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e[3]));
    k_flush_proto<<<sms * 4, 256>>>(t, o);
    CK(cudaEventRecord(e[4]));
    CK(cudaDeviceSynchronize());
    float m1, m2, m3, m4, m5;
    CK(cudaEventElapsedTime(&m1, e[1], e[2]));
    CK(cudaEventElapsedTime(&m5, e[1], e[5]));
    CK(cudaEventElapsedTime(&m2, e[2], e[3]));
    CK(cudaEventElapsedTime(&m3, e[3], e[4]));
    CK(cudaEventElapsedTime(&m4, e[0], e[4]));
    unsigned long long hc[24];
    CK(cudaMemcpy(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost));
    uint32_t hf[4];
    CK(cudaMemcpy(hf, failw, 16, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> hfd(P);
    CK(cudaMemcpy(hfd.data(), failed, P * 4, cudaMemcpyDeviceToHost));
    int nfailed = 0;
    for (int p = 0; p < P; p++) nfailed += hfd[p] != 0;
    unsigned long long nout;
    CK(cudaMemcpy(&nout, o.count, 8, cudaMemcpyDeviceToHost));
    printf("  (partition %.3f ms, resolve %.3f ms)\n", m5, m1 - m5);
    printf("iter %d: probe %.3f ms  child %.3f ms  flush %.3f ms  all %.3f ms | deferred %llu spilled %llu hits %llu recs %llu "
           "pages %llu ovf %u fail %u failed_parts %d out %llu\n",
           itx, m1, m2, m3, m4, hc[0], hc[8 + ST_SPILLED], hc[8 + ST_HITS], hc[8 + ST_RECORDS], hc[2],
           (unsigned)(hc[3] & 0xFFFFFFFF), hf[0], nfailed, nout);
    if (itx > 0) {
      tp += m1;
      tc_ += m2;
      tf += m3;
      tall += m4;
      meas++;
    }
    if (itx == iters - 1) {
      CK(cudaMemset(seen, 0, G * 4));
      CK(cudaMemset(bad, 0, 64));
      k_verify<<<sms * 8, 256>>>(o, (int64_t)nout, tc, ts, tmin, tmax, seen, bad);
      k_verify2<<<sms * 8, 256>>>(tc, seen, G, bad);
      unsigned long long hb[8];
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hb, bad, 64, cudaMemcpyDeviceToHost));
      printf("verify: badkey %llu count %llu sum %llu minmax %llu seen %llu -> %s\n", hb[0], hb[1], hb[2], hb[3], hb[4],
             (hb[0] | hb[1] | hb[2] | hb[3] | hb[4]) ? "FAIL" : "OK");
    }
  }
  if (meas) {
    const double alg_probe = (16.0 * N + 16.0 * 0.875 * N);
    printf("mean: probe %.3f ms (%.0f GB/s alg, %.3f of 6543)  child %.3f ms (%.0f GB/s)  all %.3f ms\n", tp / meas,
           alg_probe / (tp / meas) / 1e6, alg_probe / (tp / meas) / 1e6 / 6543.4, tc_ / meas,
           16.0 * 0.875 * N / (tc_ / meas) / 1e6, tall / meas);
  }
  return 0;
}
