// aggb200.cu — host orchestrator + C ABI (include/aggb200.h) of the B200
// group-by hot path.
//
// Planning restates the reference's (operators/hybrid.py:89-163,
// hash_table.py:31-45, operators/base.py:141-147): the frame budget M x p
// becomes a resident-table capacity in groups; Formula-1 partition counts are a
// lower bound on the spill fan-out, which is raised until every child
// partition fits a shared-memory table.
#include <cuda.h>  // driver-API types for the VMM page pool (entry points via cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <time.h>

#include "../../include/aggb200.h"
#include "pass.cuh"
#include "probe.cuh"
#include "sort.cuh"
#include "cuts.cuh"
#include "wc2.cuh"

using namespace aggb;

namespace {

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

thread_local std::string g_err;

// AGGB_TRACE=1: host-side phase timings on stderr (synchronizes the stream)
struct Trace {
  bool on;
  double t0;
  Trace() : on(getenv("AGGB_TRACE") != nullptr), t0(now()) {}
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  void mark(cudaStream_t st, const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    double t = now();
    fprintf(stderr, "[aggb] %-28s %8.3f ms\n", what, t - t0);
    t0 = t;
  }
};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) return fail(AGGB_CUDA_ERROR, "%s: %s (%s:%d)", #x,            \
                                       cudaGetErrorString(e_), __FILE__, __LINE__);      \
  } while (0)

#define TRY(x)                  \
  do {                          \
    int s_ = (x);               \
    if (s_ != AGGB_OK) return s_; \
  } while (0)

// grow-only device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need, size_t* hw) {
    if (need <= bytes) return AGGB_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t nb = std::max(need + need / 4, (size_t)256);  // headroom: sizes vary run to run
    cudaError_t e = cudaMalloc(&p, nb);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();  // do not leave the failure to a later launch check
      return fail(AGGB_CUDA_ERROR, "cudaMalloc(%zu): %s", nb, cudaGetErrorString(e));
    }
    bytes = nb;
    if (hw) *hw += nb;
    return AGGB_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return (T*)p; }
};

// Pinned host staging for the planning round trips: the D2H copies queue
// without the driver's pageable bounce (one blocking copy each) and complete
// behind a single stream synchronize.
struct HPin {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return AGGB_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    size_t nb = std::max(need + need / 4, (size_t)4096);
    cudaError_t e = cudaHostAlloc(&p, nb, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return fail(AGGB_CUDA_ERROR, "cudaHostAlloc(%zu): %s", nb, cudaGetErrorString(e));
    }
    bytes = nb;
    return AGGB_OK;
  }
  ~HPin() {
    if (p) cudaFreeHost(p);
  }
  template <class T>
  T* as() const { return (T*)p; }
};

// Spill page pool memory: one virtual address range reserved for twice the
// device's memory, physical memory mapped onto its end as the pool grows (CUDA
// VMM): HBM first, then pinned host memory once HBM is exhausted (SURVEY §8(f)
// f3, the external RunWriter/RunReader analog: runs larger than HBM).  Growth never copies and never holds old + new at once: a pool that
// doubles to 60+ GB (C5 hash_sort at 500M records) only maps the difference.
struct VPool {
  CUdeviceptr va = 0;
  size_t reserved = 0, mapped = 0, gran = 0;
  size_t dev_mapped = 0, host_mapped = 0, dev_limit = ~(size_t)0;
  int dev = -1;
  std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;
  struct Api {
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*afree)(CUdeviceptr, size_t);
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*release)(CUmemGenericAllocationHandle);
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*unmap)(CUdeviceptr, size_t);
    CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    bool ok = false;
  };
  static const Api& api() {
    static Api a = [] {
      Api x;
      memset(&x, 0, sizeof(x));
      cudaDriverEntryPointQueryResult q;
      bool ok = true;
      auto get = [&](const char* name, void** fn) {
        if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
            !*fn)
          ok = false;
      };
      get("cuMemAddressReserve", (void**)&x.reserve);
      get("cuMemAddressFree", (void**)&x.afree);
      get("cuMemCreate", (void**)&x.create);
      get("cuMemRelease", (void**)&x.release);
      get("cuMemMap", (void**)&x.map);
      get("cuMemUnmap", (void**)&x.unmap);
      get("cuMemSetAccess", (void**)&x.access);
      get("cuMemGetAllocationGranularity", (void**)&x.granularity);
      cudaGetLastError();
      x.ok = ok;
      return x;
    }();
    return a;
  }
  CUmemAllocationProp host_prop() const {
    CUmemAllocationProp pr;
    memset(&pr, 0, sizeof(pr));
    pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    pr.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
    // the host NUMA node nearest this GPU (2-socket nodes: GPUs of socket 1
    // would otherwise reach their spilled pages across the socket link)
    int numa = -1;
    if (cudaDeviceGetAttribute(&numa, cudaDevAttrHostNumaId, dev) != cudaSuccess || numa < 0) {
      cudaGetLastError();
      numa = 0;
    }
    pr.location.id = numa;
    return pr;
  }
  CUmemAllocationProp prop() const {
    CUmemAllocationProp pr;
    memset(&pr, 0, sizeof(pr));
    pr.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    pr.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    pr.location.id = dev;
    return pr;
  }
  // make [va, va + need) usable, [va, va + want) if memory allows (headroom
  // keeps growth steps few)
  int grow(size_t need, size_t want, size_t* hw) {
    if (need <= mapped) return AGGB_OK;
    const Api& A = api();
    if (!A.ok) return fail(AGGB_CUDA_ERROR, "CUDA VMM entry points unavailable");
    if (!va) {
      cudaGetDevice(&dev);
      CUmemAllocationProp pr = prop(), ph = host_prop();
      size_t gh = 0;
      if (A.granularity(&gran, &pr, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran) gran = 2u << 20;
      if (A.granularity(&gh, &ph, CU_MEM_ALLOC_GRANULARITY_MINIMUM) == CUDA_SUCCESS && gh > gran && gh % gran == 0)
        gran = gh;
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      // the device's memory, then as much again of pinned host memory
      reserved = ((std::max(2 * tot, need) + gran - 1) / gran) * gran;
      if (A.reserve(&va, reserved, gran, 0, 0) != CUDA_SUCCESS) {
        va = 0;
        return fail(AGGB_CUDA_ERROR, "cuMemAddressReserve(%zu) failed", reserved);
      }
      const char* e = getenv("AGGB_POOL_DEVICE_LIMIT_MB");  // test hook: overflow to host early
      dev_limit = e ? (size_t)atoll(e) << 20 : ~(size_t)0;
    }
    if (need > reserved) return fail(AGGB_CAPACITY_EXCEEDED, "spill pool of %zu bytes exceeds its address range", need);
    want = std::min(reserved, std::max(std::max(want, need), mapped + ((size_t)512 << 20)));
    auto up = [&](size_t x) { return ((x + gran - 1) / gran) * gran; };
    while (mapped < need) {
      CUmemGenericAllocationHandle hd;
      size_t sz = 0;
      bool host = false;
      CUmemAllocationProp pr = prop();
      if (dev_mapped < dev_limit) {
        const size_t room = dev_limit == ~(size_t)0 ? ~(size_t)0 : ((dev_limit - dev_mapped) / gran) * gran;
        const size_t tries[2] = {std::min(up(want - mapped), reserved - mapped), up(need - mapped)};
        for (size_t t : tries) {
          t = std::min(t, room);
          if (t && A.create(&hd, t, &pr, 0) == CUDA_SUCCESS) {
            sz = t;
            break;
          }
        }
      }
      if (!sz) {
        // HBM exhausted (or capped): pinned host memory mapped into the same
        // range; the kernels reach those pages over the host link unchanged
        pr = host_prop();
        sz = std::min(up(need - mapped), reserved - mapped);
        if (A.create(&hd, sz, &pr, 0) != CUDA_SUCCESS)
          return fail(AGGB_CUDA_ERROR, "cuMemCreate(%zu): out of device and host memory (pool %zu mapped)", sz,
                      mapped);
        host = true;
      }
      if (A.map(va + mapped, sz, 0, hd, 0) != CUDA_SUCCESS) {
        A.release(hd);
        return fail(AGGB_CUDA_ERROR, "cuMemMap failed");
      }
      CUmemAccessDesc ad;
      memset(&ad, 0, sizeof(ad));
      ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ad.location.id = dev;
      ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      if (A.access(va + mapped, sz, &ad, 1) != CUDA_SUCCESS) {
        A.unmap(va + mapped, sz);
        A.release(hd);
        return fail(AGGB_CUDA_ERROR, "cuMemSetAccess failed");
      }
      chunks.push_back({hd, sz});
      mapped += sz;
      (host ? host_mapped : dev_mapped) += sz;
      if (hw && !host) *hw += sz;
    }
    return AGGB_OK;
  }
  void release() {
    if (!va) return;
    const Api& A = api();
    size_t off = 0;
    for (auto& c : chunks) {
      A.unmap(va + off, c.second);
      A.release(c.first);
      off += c.second;
    }
    A.afree(va, reserved);
    chunks.clear();
    va = 0;
    reserved = mapped = dev_mapped = host_mapped = 0;
  }
  template <class T>
  T* as() const { return (T*)va; }
};

uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// role salts as in the reference (hybrid.py:57-60, hash_sort.py:32-33)
enum { SALT_PART = 0x11, SALT_SLOT = 0x22, SALT_SPILL = 0x33, SALT_SUB = 0x44, SALT_EXCH = 0x77 };
uint64_t level_seed(uint64_t seed, int salt, int level) {
  return splitmix(splitmix(seed) ^ ((uint64_t)salt + ((uint64_t)level << 8)));
}

int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---------------------------------------------------------------------------
// reference planning, restated (hybrid.py:89-132, hash_table.py:31-45)
// ---------------------------------------------------------------------------

double ref_group_bytes(const aggb_config& c, int ref_width, double G, double G_t) {
  double floor_b = 2 + 1 + 8.0 * ref_width;
  if (G_t > 0 && G > 0) return std::max(G * c.frame_size / G_t, floor_b);
  return 2 + 16 + 8.0 * ref_width;
}

double fudge_factor(double gb, double extra, double slot_ratio, bool bloom) {
  double per = gb + 8 + slot_ratio * (8 + (bloom ? 1 : 0));
  return per * extra / std::max(gb, 1e-300);
}

int plan_partitions(double gf, int M) {
  if (gf <= M) return 0;
  double p = std::ceil((gf - M) / (M - 2));
  return (int)std::max(1.0, std::min(p, (double)(M - 2)));
}

int64_t plan_table_cap(int n_frames, int p, double gb, double slot_ratio, bool bloom) {
  double per = gb + 8 + slot_ratio * (8 + (bloom ? 1 : 0));
  return (int64_t)(n_frames * (double)p / per);
}

struct Compiled {
  DevSpec ds;
  int kw = 1;
  int nv = 0;
  int ref_width = 0;  // reference state width (core.py:137)
  int out_type[AGGB_MAX_FNS];
};

int compile_spec(const aggb_spec& s, Compiled& c) {
  memset(&c.ds, 0, sizeof(c.ds));
  if (s.n_fns < 1 || s.n_fns > AGGB_MAX_FNS) return fail(AGGB_SPEC_ERROR, "need 1..%d aggregate functions", AGGB_MAX_FNS);
  if (s.n_keys < 1 || s.n_keys > 2) return fail(AGGB_SPEC_ERROR, "need 1 or 2 key columns");
  if (s.n_vals < 0 || s.n_vals > AGGB_MAX_VALS) return fail(AGGB_SPEC_ERROR, "too many value columns");
  for (int i = 0; i < s.n_keys; i++)
    if (s.key_type[i] != AGGB_I64 && s.key_type[i] != AGGB_I32) return fail(AGGB_SPEC_ERROR, "key columns must be int64/int32");
  c.kw = s.n_keys;
  DevSpec& d = c.ds;
  bool states = s.input_kind == AGGB_INPUT_STATES;
  d.nv = s.n_vals;
  for (int w = 0; w < s.n_vals; w++) d.vty[w] = (s.val_type[w] == AGGB_F64) ? TY_F64 : TY_I64;
  auto add_field = [&](uint8_t op, uint8_t ty, uint8_t sk, int8_t src, bool dedup) -> int {
    if (dedup)
      for (int j = 0; j < d.ns; j++)
        if (d.op[j] == op && d.ty[j] == ty && d.srck[j] == sk && d.src[j] == src) return j;
    if (d.ns >= MAX_STATES) return -1;
    d.op[d.ns] = op;
    d.ty[d.ns] = ty;
    d.srck[d.ns] = sk;
    d.src[d.ns] = src;
    return d.ns++;
  };
  int soff = 0;
  c.ref_width = 0;
  for (int i = 0; i < s.n_fns; i++) {
    int fn = s.fn[i];
    int col = s.col[i];
    int a = -1, b = -1;
    bool div = false;
    if (fn < 0 || fn > 4) return fail(AGGB_SPEC_ERROR, "unknown aggregate function id %d", fn);
    int width = (fn == AGGB_FN_AVG) ? 2 : 1;
    c.ref_width += width;
    if (states) {
      if (soff + width > s.n_vals) return fail(AGGB_SPEC_ERROR, "state columns do not cover the spec");
      if (fn == AGGB_FN_COUNT) a = add_field(OP_ADD, TY_I64, SRC_STATE_F64, soff, false);
      else if (fn == AGGB_FN_SUM) a = add_field(OP_ADD, TY_F64, SRC_STATE_F64, soff, false);
      else if (fn == AGGB_FN_MIN) a = add_field(OP_MIN, TY_F64, SRC_STATE_F64, soff, false);
      else if (fn == AGGB_FN_MAX) a = add_field(OP_MAX, TY_F64, SRC_STATE_F64, soff, false);
      else {
        a = add_field(OP_ADD, TY_F64, SRC_STATE_F64, soff, false);
        b = add_field(OP_ADD, TY_I64, SRC_STATE_F64, soff + 1, false);
        div = true;
      }
      soff += width;
    } else {
      if (fn != AGGB_FN_COUNT && (col < 0 || col >= s.n_vals))
        return fail(AGGB_SPEC_ERROR, "function %d bound to missing value column %d", i, col);
      uint8_t ty = (fn == AGGB_FN_COUNT) ? TY_I64 : d.vty[col];
      if (fn == AGGB_FN_COUNT) a = add_field(OP_ADD, TY_I64, SRC_ONE, -1, true);
      else if (fn == AGGB_FN_SUM) a = add_field(OP_ADD, ty, SRC_VAL, (int8_t)col, true);
      else if (fn == AGGB_FN_MIN) a = add_field(OP_MIN, ty, SRC_VAL, (int8_t)col, true);
      else if (fn == AGGB_FN_MAX) a = add_field(OP_MAX, ty, SRC_VAL, (int8_t)col, true);
      else {
        a = add_field(OP_ADD, ty, SRC_VAL, (int8_t)col, true);
        b = add_field(OP_ADD, TY_I64, SRC_ONE, -1, true);
        div = true;
      }
    }
    if (a < 0 || (div && b < 0)) return fail(AGGB_SPEC_ERROR, "more than %d state fields", MAX_STATES);
    d.fin_div[i] = div;
    d.fin_a[i] = (uint8_t)a;
    d.fin_b[i] = (uint8_t)(b < 0 ? 0 : b);
    uint8_t oty = div ? TY_F64 : d.ty[a];
    d.out_ty[i] = oty;
    c.out_type[i] = (oty == TY_F64) ? AGGB_F64 : AGGB_I64;
  }
  d.nout = s.n_fns;
  c.nv = states ? s.n_vals : s.n_vals;
  return AGGB_OK;
}

int nwt_for(int words) {
  int w = 1;
  while (w < words) w <<= 1;
  return w;
}

// ---------------------------------------------------------------------------
// kernel dispatch tables
// ---------------------------------------------------------------------------

typedef void (*pass_fn)(PassArgs);
typedef void (*child_fn)(ChildArgs);
constexpr int BLOCK = 512;

// field-program ids: 0 runtime (PD), 1 C1/C4, 2 C2, 3 C3, 5 C5
int detect_prog(const DevSpec& d, int kw) {
  static const uint32_t c1[] = {0x000, 0x010};
  static const uint32_t c2[] = {0x000, 0x010, 0x011, 0x012};
  static const uint32_t c3[] = {0x000, 0x054};
  static const uint32_t c5[] = {0x000, 0x010, 0x011, 0x012, 0x110, 0x111, 0x112,
                                0x254, 0x255, 0x256, 0x354, 0x355, 0x356};
  auto eq = [&](const uint32_t* f, int n) {
    if (d.ns != n) return false;
    for (int j = 0; j < n; j++)
      if (field_desc(d, j) != f[j]) return false;
    return true;
  };
  if (kw == 1 && d.nv == 1 && eq(c1, 2)) return 1;
  if (kw == 1 && d.nv == 1 && eq(c2, 4)) return 2;
  if (kw == 1 && d.nv == 1 && eq(c3, 2)) return 3;
  if (kw == 2 && d.nv == 4 && eq(c5, 13)) return 5;
  return 0;
}

struct PassCfg {
  pass_fn fn;
  int R, blk;
};

template <int KW, int NWT, int R, int BLK, class PG, int NH = 0>
PassCfg pc() { return PassCfg{k_pass<KW, NWT, R, BLK, 1, PG, NH>, R, BLK}; }

constexpr int NHOT = 1;  // k_pass heavy-hitter tier on (pass.cuh HotOps; up to HOT_MAX keys)

template <int KW>
PassCfg pass_kernel(int nwt, int prog, bool hot = false) {
  // 512 threads x 4 records, up to 128 registers, 1 CTA/SM: the 1024 x 2 shape
  // spilled at its 64-register cap (profiles/r01_notes.md)
  if (KW == 1 && nwt == 1 && hot) {
    if (prog == 1) return pc<1, 1, 4, 512, ProgC1, NHOT>();
    if (prog == 3) return pc<1, 1, 4, 512, ProgC3, NHOT>();
  }
  if (KW == 1 && nwt == 1) {
    if (prog == 1) return pc<1, 1, 4, 512, ProgC1>();
    if (prog == 2) return pc<1, 1, 4, 512, ProgC2>();
    if (prog == 3) return pc<1, 1, 4, 512, ProgC3>();
  }
  if (KW == 2 && nwt == 4 && prog == 5) return pc<2, 4, 2, 512, ProgC5>();
  switch (nwt) {
    case 1: return pc<KW, 1, 4, 512, PD>();
    case 2: return pc<KW, 2, KW == 1 ? 4 : 2, 512, PD>();
    case 4: return pc<KW, 4, 2, 512, PD>();
    case 8: return pc<KW, 8, 1, 512, PD>();
    case 16: return pc<KW, 16, 1, 512, PD>();
    default: return pc<KW, 32, 1, 256, PD>();
  }
}

// PROBE specialised for one-word keys and one dense 8-byte value column (probe.cuh)
template <int PM, int R = 4, int BLK = 512>
PassCfg probe_kernel_pm(int prog, bool hot = false) {
  if (PM == PM_ONE && hot && prog == 1) return PassCfg{k_probe<R, BLK, ProgC1, PM, 1>, R, BLK};
  if (PM == PM_ONE && hot && prog == 3) return PassCfg{k_probe<R, BLK, ProgC3, PM, 1>, R, BLK};
  if (prog == 1) return PassCfg{k_probe<R, BLK, ProgC1, PM>, R, BLK};
  if (prog == 2) return PassCfg{k_probe<R, BLK, ProgC2, PM>, R, BLK};
  if (prog == 3) return PassCfg{k_probe<R, BLK, ProgC3, PM>, R, BLK};
  return PassCfg{k_probe<R, BLK, PD, PM>, R, BLK};
}
PassCfg probe_kernel(int prog, int pm) {
  if (pm == PM_SCAN) {
    const char* e = getenv("AGGB_SCAN_CFG");  // launch-shape experiments
    if (e && !strcmp(e, "4x768")) return probe_kernel_pm<PM_SCAN, 4, 768>(prog);
    if (e && !strcmp(e, "2x1024")) return probe_kernel_pm<PM_SCAN, 2, 1024>(prog);
    if (e && !strcmp(e, "3x1024")) return probe_kernel_pm<PM_SCAN, 3, 1024>(prog);
    if (e && !strcmp(e, "8x256")) return probe_kernel_pm<PM_SCAN, 8, 256>(prog);
    return probe_kernel_pm<PM_SCAN>(prog);
  }
  if (pm == PM_RESOLVE) return probe_kernel_pm<PM_RESOLVE>(prog);
  return probe_kernel_pm<PM_ONE>(prog);
}

size_t probe_smem(int P, int bloom_words, int blk, int pm, bool pairs) {
  const size_t ring = pm == PM_SCAN ? 0 : (size_t)(blk / 32) * PQ_RING * 16;
  const size_t pk = (pairs && pm != PM_RESOLVE) ? (size_t)P * (16 + 4) + 16 : 0;  // parked record + tag
  return (size_t)((bloom_words + 1) & ~1) * 8 + ring + (size_t)P * (4 + 4 * 8) + pk + 64;
}

template <int KW>
child_fn child_kernel(int nwt, int prog) {
  // R = 2 records per thread in flight (R = 4 spilled registers at the 64-register
  // cap of 2 CTAs/SM and ran 2.7x slower, profiles/r01_notes.md)
  if (KW == 1 && nwt == 1) {
    if (prog == 1) return k_child<1, 1, 2, ProgC1>;
    if (prog == 2) return k_child<1, 1, 2, ProgC2>;
    if (prog == 3) return k_child<1, 1, 2, ProgC3>;
  }
  // C5 (13 fields): R = 1 — R = 2 spilled 268 B at the 64-register cap (child 16.5 -> 13.8 ms per 500M)
  if (KW == 2 && nwt == 4 && prog == 5) return getenv("AGGB_C5_R2") ? k_child<2, 4, 2, ProgC5> : k_child<2, 4, 1, ProgC5>;
  switch (nwt) {
    case 1: return k_child<KW, 1, 2, PD>;
    case 2: return k_child<KW, 2, 2, PD>;
    case 4: return k_child<KW, 4, 2, PD>;
    // wide payloads (partial-state merges of wide specs: C5 hash_sort runs) take
    // up to 128 registers at one CTA per SM: at 64 they spilled 200-1,360 bytes
    case 8: return getenv("AGGB_CHILD_MINB2") ? k_child<KW, 8, 1, PD> : k_child<KW, 8, 1, PD, 1>;
    case 16: return getenv("AGGB_CHILD_MINB2") ? k_child<KW, 16, 1, PD> : k_child<KW, 16, 1, PD, 1>;
    default: return getenv("AGGB_CHILD_MINB2") ? k_child<KW, 32, 1, PD> : k_child<KW, 32, 1, PD, 1>;
  }
}

constexpr uint32_t PAGE_BYTES = 8192;
size_t child_smem_budget() {
  const char* e = getenv("AGGB_CHILD_SMEM_KB");
  return (size_t)(e ? atoi(e) : 100) * 1024;
}

int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }
int group_of(int rw) { return 4 / gcd_i(rw, 4); }
// largest fan-out whose per-partition SMEM state (sector residual + page
// bookkeeping) fits one CTA of k_pass
int max_parts_for(int rw) {
  size_t per = (size_t)(group_of(rw) - 1) * rw * 8 + 38;
  return (int)std::min<size_t>(4096, (200 * 1024) / per);
}
constexpr int MAX_PARTS = 4096;

struct SetInfo {
  SpillSet ss;
  uint32_t first_page;  // pages of this set start at or after here
};

struct Handle {
  int device = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  aggb_config cfg{};
  aggb_spec spec{};
  Compiled cs;
  int kw = 1;
  int sms = 148;
  size_t hw = 0;
  // plan
  int64_t budget = 0;       // resident capacity (groups)
  bool unlimited = false;
  bool l2_children = false; // spilled partitions aggregate in the budget-sized L2 table (drain)
  int P0 = 1;               // level-0 spill fan-out
  int nsub0 = 1;            // sub-passes per level-1 child (fan-out beyond one spill pass)
  bool l2_capped = false;   // in-memory plan run budgeted at an L2-sized table
  int64_t fanout_need = 1;  // level-0 fan-out the child capacity asks for (P0 x nsub0)
  int child_slots_log2 = 11;
  int child_cap = 1024;
  // level-0 table
  GTable tab{};
  DBuf tkeys, tstates, thdr;
  bool has_table = false;
  // page pool
  VPool pool_base;
  DBuf page_part, page_fill, page_set, pool_ctr;  // pool_ctr: [0]=next_page [1]=overflow
  uint32_t pool_cap = 0;
  uint64_t pool_bound = 0;  // upper bound of pages used since reset
  // spill sets
  int next_set_id = 1;
  SetInfo raw0{}, part0{};
  bool raw0_live = false, part0_live = false;
  // deferral
  DBuf defer;
  int64_t defer_cap = 0;
  int defer_words = 0;      // words per record the deferral buffer holds
  unsigned long long last_cap_chunked = 0;  // chunk-region size of the last inserting pass
  unsigned long long reopen[2] = {0, 0};    // host staging for a hash_sort table reopen
  unsigned long long tail_sc[16] = {};      // scratch counters read after the last child pass
  uint32_t tail_ovfl = 0;
  bool tail_valid = false;
  HPin hpin;  // pinned staging of the drain's planning reads
  // scratch: [0..7] stats, [8] tile counter A, [9] tile counter B, [10] defer count, [11] ovf count,
  // [12] item counter, [13] out count
  DBuf scratch;
  DBuf hscratch_dev;
  // output
  DBuf out_keys, out_vals, out_i32[2];
  int64_t out_cap = 0;
  // host-side state
  int64_t records = 0;
  int launches = 0;
  bool finished = false;
  aggb_result result{};
  aggb_metrics met{};
  int64_t hash_sort_runs = 0;
  // recursion scratch
  DBuf part_records, part_pages, cursor, plist, item_off, ovf, pend, l2stage, cut_tmp;
  DBuf hot;                 // heavy-hitter keys of the current push (k_hot_sample)
  DBuf sort_hist;           // sort path: byte histograms of the appended keys
  DBuf dd_spilled, dd_tmp;  // dynamic destaging: destaged-partition flags, eviction lists
  std::vector<uint8_t> dd_host;
  int64_t dd_evictions = 0;
  int sh_stage = 0;  // shared_hash: overflows seen (0: shared table, 1: original_hh shape, 2: pure routing)
  bool hot_ready = false;
  bool hot_no_tier = false;  // the hot keys cover most records: no SMEM pre-aggregation tier
  int64_t skew_cap = 0;      // L2-capped plans: the capacity a heavily skewed push may use
  bool aos_planned = false;  // slot-major states planned (in-memory table beyond L2)
  bool l0_deferred = false;  // level-0 metrics ride on the tail's read (finish without a round trip)
  bool first_push = true;
  int prog = 0;
  // blocked bloom filter of the frozen level-0 table (PROBE)
  DBuf bloom;
  int64_t bloom_words = 0;
  uint64_t bloom_seed = 0;
  int64_t ovf_cap = 0;
  // two-phase PROBE: candidate regions (bloom positives), open chains per (CTA, partition)
  DBuf cand, chains;
  // write-combined level-0 PROBE + one-wave compact children (wc.cuh): planned
  // for budgeted pre-partitioning of one-word keys and one int64 column with an
  // integer COUNT/SUM(/MIN/MAX) spec; children find their pages through device
  // page lists (no host round trip), a partition they cannot hold goes to drain
  bool wc = false;
  bool wc_used = false;       // some PROBE of this run went through k_probe_wc
  int wc_table_bytes = 0;     // child shared-memory table
  uint32_t wc_plist_cap = 0;  // page-list entries per partition
  int64_t wc_fallbacks = 0;   // finishes that needed drain for some partition (tests)
  uint32_t wc_ocap = 0;       // resident slots per owner list
  size_t wc_scan_smem = 0;    // dynamic shared memory k_scan_wc was last configured for
  bool wc_child_attr = false; // k_child2_wc's shared-memory attribute is set
  int64_t wc_launches = 0;    // k_scan_wc launches of this run
  int64_t wc_entries = 0;     // page-list entries per run the launches so far may have taken
  DBuf cut_bar;  // grid barrier of k_blind_cuts
  DBuf wc_ovf;   // [0] count, then run << 32 | page: pages past the runs' page lists (skew)
  uint32_t wc_ovf_cap = 0;
  DBuf wc_plist, wc_meta, wc_olist, wc_olist_n, wc_gather;  // wc_meta: per-run records / page counts / failed flags, value info, fail word (one memset per run)
  DBuf partials_soa;  // aggb_push_partials: received partial records in the list layout
  // sort path
  DBuf sort_keys, sort_vals;
  int64_t sort_n = 0, sort_cap = 0;
  // staging for host inputs (grow-only)
  DBuf stage;
  // pipelined host pushes: copy stream, two staging buffers, their events
  cudaStream_t cst = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  cudaEvent_t ev_staged = nullptr;  // end of a host push's copies out of the caller's memory
  DBuf pstage[2];
  bool pstage_busy[2] = {false, false};  // an aggregation reading pstage[b] may still run (ev_used[b])
  // per-kernel CUDA-event timing (aggb_profile)
  bool prof = false;
  struct Ev { int kid; cudaEvent_t a, b; };
  std::vector<Ev> evs;
  std::vector<cudaEvent_t> free_events;
  double kms[24] = {0};
  int64_t kcount[24] = {0};
};

// views into Handle::wc_meta ([NP] u64 records | [NP] u32 pages | [NP] u32 failed | 4 u32 value info | 2 u32 fail)
inline size_t wc_meta_bytes(int NP) { return (size_t)NP * 16 + 32; }
inline unsigned long long* wc_recs(Handle* h) { return h->wc_meta.as<unsigned long long>(); }
inline uint32_t* wc_pn(Handle* h) { return (uint32_t*)(wc_recs(h) + h->P0); }
inline uint32_t* wc_failed(Handle* h) { return wc_pn(h) + h->P0; }
inline unsigned int* wc_vinfo(Handle* h) { return wc_failed(h) + h->P0; }
inline uint32_t* wc_fail(Handle* h) { return wc_vinfo(h) + 4; }

const char* KNAMES[] = {"k_pass<FILL>", "k_pass<PROBE>", "k_pass<ROUTE>", "k_pass<GRACE>", "k_child",
                        "k_flush_table", "k_table_init", "k_page_bucket", "k_key_egress", "k_sort",
                        "k_exchange_pack", "k_segreduce", "k_bloom_build", "k_pass<PROBE:resolve>", "k_split",
                        "k_scan_wc", "k_wc_build", "k_child_wc", "k_blind_cuts"};
constexpr int NKINDS = 19;

int prof_begin(Handle* h, int kid) {
  if (!h->prof) return -1;
  Handle::Ev e;
  e.kid = kid;
  for (cudaEvent_t* x : {&e.a, &e.b}) {
    if (!h->free_events.empty()) {
      *x = h->free_events.back();
      h->free_events.pop_back();
    } else {
      cudaEventCreate(x);
    }
  }
  cudaEventRecord(e.a, h->st);
  h->evs.push_back(e);
  return (int)h->evs.size() - 1;
}
void prof_end(Handle* h, int idx) {
  if (idx < 0) return;
  cudaEventRecord(h->evs[idx].b, h->st);
}
void prof_collect(Handle* h) {
  if (h->evs.empty()) return;
  cudaStreamSynchronize(h->st);
  for (auto& e : h->evs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e.a, e.b);
    h->kms[e.kid] += ms;
    h->kcount[e.kid]++;
    h->free_events.push_back(e.a);
    h->free_events.push_back(e.b);
  }
  h->evs.clear();
}

unsigned long long* SC(Handle* h) { return h->scratch.as<unsigned long long>(); }

int pool_ensure(Handle* h, uint64_t extra_pages) {
  uint64_t need = h->pool_bound + extra_pages;
  if (need > h->pool_cap && h->pool_cap) {
    // the running bound is loose (it sums every pass's worst case): before growing,
    // tighten it to the pages actually allocated so far plus this pass's bound
    uint32_t now = 0;
    CU(cudaMemcpyAsync(&now, h->pool_ctr.p, 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    need = std::min<uint64_t>(need, (uint64_t)std::min<uint32_t>(now, h->pool_cap) + extra_pages);
  }
  if (need > 0xFFFFFFF0ull) return fail(AGGB_CAPACITY_EXCEEDED, "spill pool would exceed 2^32 pages");
  h->pool_bound = need;
  if (need <= h->pool_cap) return AGGB_OK;
  // grow: one contiguous allocation; used pages and metadata are copied over
  uint64_t cap = std::max<uint64_t>(need + (need > (2u << 20) ? need / 16 : need / 4), 4096);  // less slack past 16 GB
  uint32_t used = 0;
  if (h->pool_cap) {
    CU(cudaMemcpyAsync(&used, h->pool_ctr.p, 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    used = std::min<uint32_t>(used, h->pool_cap);
  }
  // page memory grows in place (VPool: mapped onto a reserved range, pages stay
  // where they are); the 12 bytes of metadata per page are copied over
  CU(cudaStreamSynchronize(h->st));
  TRY(h->pool_base.grow(need * (size_t)PAGE_BYTES, cap * (size_t)PAGE_BYTES, &h->hw));
  cap = std::min<uint64_t>(h->pool_base.mapped / PAGE_BYTES, 0xFFFFFFF0ull);
  DBuf np, nf, ns;
  TRY(np.ensure(cap * 4, &h->hw));
  TRY(nf.ensure(cap * 4, &h->hw));
  TRY(ns.ensure(cap * 4, &h->hw));
  if (used) {
    CU(cudaMemcpyAsync(np.p, h->page_part.p, (size_t)used * 4, cudaMemcpyDeviceToDevice, h->st));
    CU(cudaMemcpyAsync(nf.p, h->page_fill.p, (size_t)used * 4, cudaMemcpyDeviceToDevice, h->st));
    CU(cudaMemcpyAsync(ns.p, h->page_set.p, (size_t)used * 4, cudaMemcpyDeviceToDevice, h->st));
  }
  CU(cudaStreamSynchronize(h->st));
  h->page_part.release();
  h->page_fill.release();
  h->page_set.release();
  h->page_part = np;
  h->page_fill = nf;
  h->page_set = ns;
  h->pool_cap = (uint32_t)cap;
  return AGGB_OK;
}

PagePool pool_of(Handle* h) {
  PagePool pp;
  pp.base = h->pool_base.as<uint8_t>();
  pp.page_bytes = PAGE_BYTES;
  pp.next_page = h->pool_ctr.as<uint32_t>();
  pp.overflow = h->pool_ctr.as<uint32_t>() + 1;
  pp.capacity = h->pool_cap;
  pp.page_part = h->page_part.as<int32_t>();
  pp.page_fill = h->page_fill.as<int32_t>();
  pp.page_set = h->page_set.as<int32_t>();
  return pp;
}

SpillSet make_set(Handle* h, int nparts, int payload_words, int kind, uint64_t seed) {
  SpillSet s;
  s.id = h->next_set_id++;
  s.nparts = nparts;
  s.rw = h->kw + payload_words;
  int G = group_of(s.rw);
  s.per_page = (int)(PAGE_BYTES / (8u * s.rw)) / G * G;
  s.seed = seed;
  s.kind = kind;
  return s;
}

int grid_for(const void* fn, size_t smem, int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BLOCK, smem);
  return std::max(1, occ) * sms;
}

size_t pass_smem(int P, int G, int rw, int bloom_words) {
  return (size_t)bloom_words * 8 + (size_t)P * (G - 1) * rw * 8 + (size_t)P * 38 + 64;
}

bool dense8(const ColSrc& c, int kw) {
  for (int w = 0; w < kw; w++)
    if (c.kty[w] == TY_I32 || c.kstride[w] != 8) return false;
  for (int w = 0; w < c.nv; w++)
    if (c.vty[w] == TY_I32 || c.vstride[w] != 8) return false;
  return true;
}

// one k_pass launch
struct PassPlan {
  int mode;
  const aggb_input* in;      // columnar source (may be null)
  ColSrc col{};
  int col_kind = 0;          // 0 raw payload, 1 native partial states
  bool use_start = false;    // start from tile counter A (after FILL)
  const uint64_t* lin = nullptr;
  int64_t lin_stride = 0;
  const unsigned long long* lin_count = nullptr;
  int lin_kind = 0;
  int lin_words = 0;
  SpillSet ss{};
  uint32_t cut0 = 0;
  uint64_t part_seed = 0;
  unsigned long long* counter = nullptr;
};

int launch_pass(Handle* h, PassPlan& pp) {
  int payload = std::max(pp.col.nv, pp.lin_words);
  if (pp.mode != MODE_FILL) payload = std::max(payload, pp.ss.rw - h->kw);
  int nwt = nwt_for(std::max(payload, 1));
  if (nwt > 32) return fail(AGGB_SPEC_ERROR, "record payload of %d words exceeds 32", payload);
  bool hot = h->hot_ready && h->kw == 1 && nwt == 1 && (pp.mode == MODE_FILL || pp.mode == MODE_PROBE);
  PassCfg pcfg = h->kw == 1 ? pass_kernel<1>(nwt, h->prog, hot) : pass_kernel<2>(nwt, h->prog);
  int P = pp.mode == MODE_FILL ? 1 : pp.ss.nparts;
  int G = pp.mode == MODE_FILL ? 1 : group_of(pp.ss.rw);
  int rw = pp.mode == MODE_FILL ? 1 : pp.ss.rw;
  // k_probe: 16-byte raw records from dense 8-byte columns (and the SoA deferral list)
  const bool fast_probe = pp.mode == MODE_PROBE && h->kw == 1 && pp.col.nv == 1 && pp.ss.rw == 2 && pp.col_kind == 0 &&
                          pp.ss.kind == 0 && (!pp.lin || (pp.lin_words == 1 && pp.lin_kind == 0)) &&
                          dense8(pp.col, 1) && pp.ss.per_page == 512 && (!h->l2_capped || !getenv("AGGB_L2CAP_WIDE")) &&
                          // page ids are 24-bit in k_probe's page map (conservative pool estimate)
                          h->pool_bound + (uint64_t)(pp.col.n + pp.lin_stride) / 256 +
                                  (uint64_t)h->sms * (2ull * pp.ss.nparts + 128) < 0xFFFFF0ull &&
                          !getenv("AGGB_GENERIC_PROBE");
  const int T_fill = pcfg.R * pcfg.blk;  // tile size of the FILL pass (start_tiles counts its tiles)
  // k_probe_w: two-word keys + 4 payload words (C5 rows), raw records
  const bool wide_probe = !fast_probe && pp.mode == MODE_PROBE && h->kw == 2 && pp.col.nv == 4 && pp.ss.rw == 6 &&
                          pp.col_kind == 0 && pp.ss.kind == 0 && (!pp.lin || (pp.lin_words == 4 && pp.lin_kind == 0)) &&
                          pp.ss.per_page == 170 &&
                          h->pool_bound + (uint64_t)(pp.col.n + pp.lin_stride) / 64 +
                                  (uint64_t)h->sms * (2ull * pp.ss.nparts + 128) < 0xFFFFF0ull &&
                          !getenv("AGGB_GENERIC_PROBE");
  if (wide_probe)
    pcfg = h->prog == 5 ? PassCfg{k_probe_w<2, 4, 2, 512, ProgC5>, 2, 512} : PassCfg{k_probe_w<2, 4, 2, 512, PD>, 2, 512};
  // two-phase PROBE (probe.cuh): a streaming partition pass, then the bloom positives
  const bool split = fast_probe && h->bloom_words && getenv("AGGB_SPLIT");
  if (fast_probe) pcfg = split ? probe_kernel(h->prog, PM_SCAN) : probe_kernel_pm<PM_ONE>(h->prog, hot);
  pass_fn fn = pcfg.fn;
  int R = pcfg.R, blk = pcfg.blk;
  int T = R * blk;
  Bloom bl{nullptr, 0, 0};
  if (pp.mode == MODE_PROBE && h->bloom_words) {
    bl.words = h->bloom.as<uint64_t>();
    bl.mask = (uint32_t)h->bloom_words - 1;
    bl.seed = h->bloom_seed;
  }
  // sector pairs pay off in the split scan only (C2: scan 1.83 -> 1.68 ms); in the
  // one-pass kernel the deferred odd records lengthen the tile (2.15 -> 2.48 ms)
  bool pairs = fast_probe && split && !getenv("AGGB_NO_PAIRS");
  auto smem_of = [&](int bw) {
    if (wide_probe) return (size_t)((bw + 1) & ~1) * 8 + (size_t)P * (4 + 8 * 4) + 64;
    return fast_probe ? probe_smem(P, bw, blk, split ? PM_SCAN : PM_ONE, pairs) : pass_smem(P, G, rw, bw);
  };
  size_t smem = smem_of(bl.words ? (int)h->bloom_words : 0);
  if (smem > 226 * 1024 && pairs) {  // no room for sector pairs: the bloom filter matters more
    pairs = false;
    smem = smem_of(bl.words ? (int)h->bloom_words : 0);
  }
  if (smem > 227 * 1024 && bl.words) {  // no room: probe without the filter
    bl.words = nullptr;
    smem = smem_of(0);
  }
  if (smem > 227 * 1024) return fail(AGGB_SPEC_ERROR, "pass needs %zu bytes of shared memory", smem);
  // SMEM pre-aggregation tier for inserting passes over one-word keys (pass.cuh)
  int cache_log2 = 0;
  if (wide_probe || (fast_probe && split)) hot = false;  // k_probe_w / the split PROBE: no heavy-hitter tier
  if (hot && smem + hot_smem<ProgC1>(blk) + 16 <= (fast_probe ? 220 : 200) * 1024) {
    smem += hot_smem<ProgC1>(blk) + 16;  // ProgC1 and ProgC3 both hold 2 fields
  } else if (hot) {                      // no room next to the partitions: the plain pass
    hot = false;
    pcfg = fast_probe ? probe_kernel_pm<PM_ONE>(h->prog, false) : pass_kernel<1>(nwt, h->prog, false);
    fn = pcfg.fn;
  }
  // (an L2-capped in-memory plan probes hot keys: the tier serves PROBE too)
  if (!fast_probe && (pp.mode == MODE_FILL || (pp.mode == MODE_PROBE && h->l2_capped)) && h->kw == 1 &&
      !getenv("AGGB_NO_CACHE") && !(hot && h->hot_no_tier)) {
    const size_t per = 12 + 8 * (size_t)h->cs.ds.ns;
    const size_t room = std::min<size_t>(160 * 1024, 224 * 1024 - std::min<size_t>(smem + 16, 224 * 1024));
    int L = 0;
    while (L < 14 && ((size_t)1 << (L + 1)) * per <= room) L++;
    if (L >= 8) {
      cache_log2 = L;
      smem += ((size_t)1 << L) * per + 16;
    }
  }
  CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, blk, smem);
  int grid = std::max(1, occ) * h->sms;
  if (pp.mode == MODE_GRACE || (pp.mode != MODE_FILL && pp.col.n == 0)) {
    // small list passes: every CTA opens a page per partition it touches, so
    // give each CTA at least ~4 tiles of records
    const int64_t recs = pp.col.n + (pp.lin_count ? pp.lin_stride : 0);
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (recs + 4LL * T - 1) / (4LL * T)));
  }
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.sp = h->cs.ds;
  a.mode = pp.mode;
  a.t = h->tab;
  a.col = pp.col;
  a.col_dense = dense8(pp.col, h->kw) ? 1 : 0;
  a.col_kind = pp.col_kind;
  a.start_tiles = pp.use_start ? SC(h) + 8 : nullptr;
  a.start_T = T_fill;
  if (pp.lin) {
    a.lin.n = 0;
    for (int w = 0; w < h->kw; w++) {
      a.lin.key[w] = (const uint8_t*)(pp.lin + (size_t)w * pp.lin_stride);
      a.lin.kstride[w] = 8;
      a.lin.kty[w] = TY_I64;
    }
    a.lin.nv = pp.lin_words;
    for (int w = 0; w < pp.lin_words; w++) {
      a.lin.val[w] = (const uint8_t*)(pp.lin + (size_t)(h->kw + w) * pp.lin_stride);
      a.lin.vstride[w] = 8;
      a.lin.vty[w] = TY_I64;
    }
  }
  a.lin_count = pp.lin ? pp.lin_count : nullptr;
  a.lin_kind = pp.lin_kind;
  a.pool = pool_of(h);
  a.ss = pp.ss;
  a.bloom = bl;
  a.group = G;
  a.cut0 = pp.cut0;
  a.part_seed = pp.part_seed;
  a.defer = h->defer.as<uint64_t>();
  a.defer_stride = h->defer_cap;
  a.defer_count = SC(h) + 10;
  a.tile_counter = pp.counter;
  a.stats = SC(h);
  a.cache_log2 = cache_log2;
  a.pairs = pairs ? 1 : 0;
  a.hot = hot ? h->hot.as<uint64_t>() : nullptr;
  a.dd_spilled = pp.mode == MODE_DD ? h->dd_spilled.as<uint8_t>() : nullptr;
  if (wide_probe) {  // C5's row layout read as three 16-byte loads per row
    const ColSrc& c = pp.col;
    const int64_t st = c.kstride[0];
    bool ok = c.kty[0] == TY_I64 && c.kty[1] == TY_I32 && c.key[1] == c.key[0] + 8 && st % 16 == 0 &&
              c.kstride[1] == st && ((uintptr_t)c.key[0] & 15) == 0 && c.nv == 4;
    for (int w = 0; ok && w < 4; w++)
      ok = c.val[w] == c.key[0] + 16 + 8 * w && c.vstride[w] == st && c.vty[w] != TY_I32;
    a.rows64 = ok ? 1 : 0;
  }
  // chunked reservations for large tables: unused chunks (< grid * chunk) stay under 1% of cap
  {
    const uint64_t cap = h->tab.cap;
    const uint64_t chunk = std::min<uint64_t>(64, cap / (100ull * (uint64_t)grid));
    if (chunk >= 32) {
      a.cap_chunk = (uint32_t)chunk;
      a.cap_chunked = cap - std::min<uint64_t>(cap, 2ull * (uint64_t)grid * chunk);
    }
    h->last_cap_chunked = a.cap_chunked;
  }
  if (pp.mode != MODE_FILL) {
    // upper bound of pages this pass can allocate
    int64_t recs = pp.col.n + (pp.lin_count ? (pp.lin_stride) : 0);
    // each (CTA, partition) pair that receives a record may hold one partly
    // filled page plus one residual-flush page: at most 2 per record
    uint64_t pairs = std::min<uint64_t>(2ull * grid * P, 2ull * (uint64_t)recs);
    uint64_t pages = (uint64_t)((recs + pp.ss.per_page - 1) / pp.ss.per_page) + pairs + 16;
    // CTA-local page stash: worth it when a CTA fills several pages per refill
    // window; each CTA may leave one unused refill behind
    const uint64_t per_cta = pages / (uint64_t)grid;
    a.stash = per_cta >= 64 ? 32 : 0;
    pages += (uint64_t)grid * 2 * a.stash * (split ? 2 : 1);
    TRY(pool_ensure(h, pages));
    a.pool = pool_of(h);
  }
  size_t smem_b = 0;
  pass_fn fn_b = nullptr;
  if (split) {
    const int64_t recs = pp.col.n + (pp.lin_count ? pp.lin_stride : 0);
    a.cand_stride = recs / NREG + 2 * T + 64;
    TRY(h->cand.ensure((size_t)a.cand_stride * 2 * NREG * 8, &h->hw));
    TRY(h->chains.ensure((size_t)grid * P * sizeof(uint2), &h->hw));
    a.cand = h->cand.as<uint64_t>();
    a.cand_count = SC(h) + 24;
    a.chains = h->chains.as<uint2>();
    CU(cudaMemsetAsync(a.cand_count, 0, NREG * 8, h->st));
    fn_b = probe_kernel(h->prog, PM_RESOLVE).fn;
    smem_b = probe_smem(P, 0, 512, PM_RESOLVE, false);
    CU(cudaFuncSetAttribute((const void*)fn_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b));
  }
  CU(cudaMemsetAsync(pp.counter, 0, 8, h->st));
  int pe = prof_begin(h, pp.mode);
  fn<<<grid, blk, smem, h->st>>>(a);
  prof_end(h, pe);
  h->launches++;
  CU(cudaGetLastError());
  if (split) {
    // phase 2 on the same grid: CTA c reopens CTA c's chains
    a.tile_counter = SC(h) + 20;
    CU(cudaMemsetAsync(a.tile_counter, 0, 8, h->st));
    pe = prof_begin(h, 13);
    fn_b<<<grid, 512, smem_b, h->st>>>(a);
    prof_end(h, pe);
    h->launches++;
    CU(cudaGetLastError());
  }
  return AGGB_OK;
}

int ensure_out(Handle* h, int64_t need) {
  if (need <= h->out_cap) return AGGB_OK;
  int64_t cap = std::max<int64_t>(need, 1024);
  int wv = std::max(h->cs.ds.nout, h->cs.ds.ns);
  unsigned long long cnt = 0;
  if (h->out_cap) {
    CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
  }
  DBuf nk, nv;
  TRY(nk.ensure((size_t)cap * h->kw * 8, &h->hw));
  TRY(nv.ensure((size_t)cap * wv * 8, &h->hw));
  if (cnt) {
    int64_t c = std::min<int64_t>((int64_t)cnt, h->out_cap);
    for (int w = 0; w < h->kw; w++)
      CU(cudaMemcpyAsync(nk.as<uint64_t>() + w * cap, h->out_keys.as<uint64_t>() + w * h->out_cap, c * 8,
                         cudaMemcpyDeviceToDevice, h->st));
    for (int j = 0; j < wv; j++)
      CU(cudaMemcpyAsync(nv.as<uint64_t>() + j * cap, h->out_vals.as<uint64_t>() + j * h->out_cap, c * 8,
                         cudaMemcpyDeviceToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
  }
  h->out_keys.release();
  h->out_vals.release();
  h->out_keys = nk;
  h->out_vals = nv;
  h->out_cap = cap;
  return AGGB_OK;
}

OutBuf outbuf(Handle* h, int partial) {
  OutBuf o;
  o.keys = h->out_keys.as<uint64_t>();
  o.vals = h->out_vals.as<uint64_t>();
  o.cap = h->out_cap;
  o.count = SC(h) + 13;
  o.partial = partial;
  return o;
}

int flush_table(Handle* h, bool partial, OutBuf* dst, bool clear = false) {
  int64_t cap_needed;
  OutBuf o;
  if (dst) {
    o = *dst;
  } else {
    unsigned long long cnt = 0;
    CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    cap_needed = (int64_t)cnt + (int64_t)h->tab.cap + 2;
    TRY(ensure_out(h, cap_needed));
    o = outbuf(h, partial ? 1 : 0);
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->sms * 8, (int64_t)((h->tab.stride + 2047) / 2048)));
  int pe = prof_begin(h, 5);
  if (clear) {
    if (h->kw == 1) k_flush_table<1, true><<<grid, 256, 0, h->st>>>(h->tab, h->cs.ds, o);
    else k_flush_table<2, true><<<grid, 256, 0, h->st>>>(h->tab, h->cs.ds, o);
  } else {
    if (h->kw == 1) k_flush_table<1><<<grid, 256, 0, h->st>>>(h->tab, h->cs.ds, o);
    else k_flush_table<2><<<grid, 256, 0, h->st>>>(h->tab, h->cs.ds, o);
  }
  prof_end(h, pe);
  h->launches++;
  CU(cudaGetLastError());
  if (clear) CU(cudaMemsetAsync(h->tab.hdr, 0, sizeof(TableHdr), h->st));
  return AGGB_OK;
}

int table_reset(Handle* h) {
  int grid = std::min<int64_t>((int64_t)h->sms * 8, (int64_t)((h->tab.stride + 255) / 256));
  int pe = prof_begin(h, 6);
  k_table_init<<<std::max(grid, 1), 256, 0, h->st>>>(h->tab, h->kw, h->cs.ds);
  prof_end(h, pe);
  h->launches++;
  CU(cudaGetLastError());
  return AGGB_OK;
}

ColSrc col_of(Handle* h, const aggb_input* in, const void* const* kptr, const void* const* vptr) {
  ColSrc c;
  memset(&c, 0, sizeof(c));
  c.n = in->n_rows;
  for (int w = 0; w < h->kw; w++) {
    c.key[w] = (const uint8_t*)kptr[w];
    c.kty[w] = h->spec.key_type[w] == AGGB_I32 ? TY_I32 : TY_I64;
    c.kstride[w] = in->key_stride[w] ? in->key_stride[w] : (c.kty[w] == TY_I32 ? 4 : 8);
  }
  c.nv = h->spec.n_vals;
  for (int w = 0; w < c.nv; w++) {
    c.val[w] = (const uint8_t*)vptr[w];
    c.vty[w] = h->spec.val_type[w] == AGGB_I32 ? TY_I32 : (h->spec.val_type[w] == AGGB_F64 ? TY_F64 : TY_I64);
    c.vstride[w] = in->val_stride[w] ? in->val_stride[w] : (c.vty[w] == TY_I32 ? 4 : 8);
  }
  return c;
}

// ---------------------------------------------------------------------------
// planning
// ---------------------------------------------------------------------------

void wc_plan(Handle* h, double spill_groups);
int plan(Handle* h) {
  const aggb_config& c = h->cfg;
  int M = c.memory_frames;
  int algo = c.algo;
  if (algo < 0 || algo > 5) return fail(AGGB_SPEC_ERROR, "unknown algorithm id %d", algo);
  double G = c.stats_G, G_t = c.stats_G_t;
  if (c.group_estimate >= 0 && c.level == 0) {  // _effective_stats (hybrid.py:193-203)
    double bg = ref_group_bytes(c, h->cs.ref_width, G, G_t);
    double gt = std::max(1.0, c.group_estimate);
    G = gt * bg / std::max(c.frame_size, 1);
    G_t = gt;
  }
  int ns = h->cs.ds.ns;
  // child shared-memory table geometry
  size_t per_slot = (size_t)(h->kw + ns) * 8;
  int lg = 6;
  while (((size_t)(1 << (lg + 1)) + 1) * per_slot <= child_smem_budget() && lg < 16) lg++;
  h->child_slots_log2 = lg;
  int64_t ccap = (int64_t)((1 << lg) * 0.7);

  if (c.budget_groups > 0) {
    h->budget = c.budget_groups;
    h->unlimited = false;
  } else if (c.budget_groups < 0) {
    h->unlimited = true;
    h->budget = (int64_t)std::max(1024.0, G_t * 1.25 + 1024);
  } else {
    // frame-derived capacity (InvalidBudget floors: test_operators.py:181-192)
    if (M < 2) return fail(AGGB_INVALID_BUDGET, "need at least 2 frames, got %d", M);
    int floor_m = (algo == AGGB_SORT_BASED || algo == AGGB_HASH_SORT) ? 3 : (algo == AGGB_DYNAMIC_DESTAGING ? 5 : 4);
    if (M < floor_m) return fail(AGGB_INVALID_BUDGET, "algorithm %d needs M >= %d, got %d", algo, floor_m, M);
    double bg = ref_group_bytes(c, h->cs.ref_width, G, G_t);
    int p = c.frame_size;
    int frames = M - 1;
    bool bloom = false;
    if (algo != AGGB_SORT_BASED && algo != AGGB_HASH_SORT) {
      bool pp = algo == AGGB_PRE_PARTITIONING;
      double F = fudge_factor(bg, c.fudge, c.slot_ratio, pp);
      int Pref = plan_partitions(G * F, M);
      if (Pref >= 1) {
        frames = M - Pref;
        bloom = pp && Pref > 1;
      }
    }
    h->budget = std::max<int64_t>(1, plan_table_cap(frames, p, bg, c.slot_ratio, bloom));
    h->unlimited = false;
  }
  // An in-memory pre-partitioning plan whose table would not fit in L2 (C3:
  // ~9M groups) aggregates with random HBM accesses per record (ncu: 17.7 GB
  // of DRAM reads for 3.2 GB of input).  The budget is an upper bound, not a
  // target: such a plan runs budgeted at an L2-sized table (~40% of L2), the
  // first-seen (for skewed data: hot) keys resident, the PROBE pass keeping
  // its SMEM tier for them, the rest through the spill path.  C3 (Zipf s=1,
  // 200M): 15.2 -> 11.1 ms.  hash_sort keeps its in-memory table (capped it
  // cuts a run per chunk: 62 ms).
  h->l2_capped = false;
  h->skew_cap = 0;
  if (h->unlimited && algo == AGGB_PRE_PARTITIONING && !getenv("AGGB_NO_L2_CAP")) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cudaGetLastError();
    const double per_group = 2.0 * 8.0 * (h->kw + std::max(1, ns));  // 2 slots per group, key + states
    int64_t l2cap = (int64_t)(0.4 * std::max(l2, 32 << 20) / per_group);
    // one-word keys with one value column PROBE through k_probe: its SMEM bloom
    // (8 bits per resident key in 64 KB) rejects the records to spill, and the
    // heavy-hitter columns fit beside it.  C3 s = 0.5: generic PROBE of a 1M-group
    // table 12.9 ms -> k_probe 4.3 ms (profiles/r01_notes.md, session 3)
    const int64_t l2full = l2cap;
    if (algo == AGGB_PRE_PARTITIONING && h->kw == 1 && h->cs.nv == 1 && !getenv("AGGB_L2CAP_WIDE"))
      l2cap = std::min<int64_t>(l2cap, 65536);
    // heavily skewed pushes (most records on a few hot keys: C3 s = 1.5, 434K
    // groups) keep the full L2-sized table: they fit it and never reach PROBE
    h->skew_cap = l2full > l2cap ? l2full : 0;
    if (getenv("AGGB_L2_CAP_GROUPS")) {  // test hook: this cap, no skew exception
      l2cap = std::max(8, atoi(getenv("AGGB_L2_CAP_GROUPS")));
      h->skew_cap = 0;
    }
    if (h->budget > 2 * l2cap) {
      h->budget = l2cap;
      h->unlimited = false;
      h->l2_capped = true;
    } else {
      h->skew_cap = 0;
    }
  }
  h->child_cap = (int)std::max<int64_t>(1, std::min<int64_t>(ccap, h->budget));
  // spill fan-out: every child partition should fill ~40% of a child table
  // (C2, profiles/r01_notes.md: child 1.08 -> 0.94 ms from 0.5 to 0.4 of the
  // table — lower load, shorter probes, a finer tail — for +0.04 ms of PROBE)
  double spill_groups = std::max(0.0, std::max(G_t, 1.0) - (double)h->budget);
  // (C5 at 100M: 0.55 cut the child 6.33 -> 5.46 ms, but at 500M records per
  // item the gain is gone: 16.5 vs 16.9 ms; 0.4 stays)
  const double load = getenv("AGGB_CHILD_LOAD") ? atof(getenv("AGGB_CHILD_LOAD")) : 0.4;  // experiment knob
  int P = (int)std::ceil(spill_groups / std::max(1.0, load * h->child_cap));
  P = std::max(P, 1);
  if (c.budget_groups == 0 && M >= 3) {
    double bg = ref_group_bytes(c, h->cs.ref_width, G, G_t);
    double F = fudge_factor(bg, c.fudge, c.slot_ratio, algo == AGGB_PRE_PARTITIONING);
    P = std::max(P, plan_partitions(G * F, M));  // Formula 1 as the floor
  }
  int rw0 = h->kw + h->cs.nv;
  int cap_parts = std::min(MAX_PARTS, max_parts_for(rw0));
  // k_probe (one-word keys, one value) keeps its 128 KB bloom only up to ~2.3K
  // partitions of shared-memory state (probe_smem); beyond, PROBE runs 2x slower
  if (h->kw == 1 && h->cs.nv == 1) cap_parts = std::min(cap_parts, h->l2_capped ? 1536 : 2200);  // + hot columns
  if (getenv("AGGB_MAX_P0")) cap_parts = std::max(2, std::min(cap_parts, atoi(getenv("AGGB_MAX_P0"))));  // test hook
  // Shared-memory children hold child_cap groups; when the fan-out that needs is
  // more than one spill pass can write, every level would retire only
  // cap_parts * child_cap groups (C5: ~20 levels).  Then each child CTA takes
  // its partition in nsub sub-passes: sub-pass s aggregates only the records
  // whose sub-hash (an independent seed) falls in range s, in a fresh table,
  // and flushes — the fan-out is P0 x nsub with one spill pass, at the price of
  // re-reading a partition nsub times (C5 100M: 1,211 L2-table children,
  // 134 ms -> SMEM sub-passes).  The L2-table child (the reference's child
  // operator with the full budget) stays behind a test hook.
  h->l2_children = false;
  h->nsub0 = 1;
  const bool force_l2 = getenv("AGGB_FORCE_L2_CHILDREN") != nullptr;  // test hook
  if (force_l2 && !h->unlimited) {
    h->l2_children = true;
    P = std::max(2, (int)std::ceil(spill_groups / std::max(1.0, 0.5 * (double)h->budget)));
  } else if (P > cap_parts) {
    h->nsub0 = (P + cap_parts - 1) / cap_parts;
    P = (P + h->nsub0 - 1) / h->nsub0;
  }
  // whole waves of children: with several partitions per resident child CTA,
  // round the fan-out down to a multiple of the resident child grid (the load
  // per partition grows by at most 1/3: <= ~0.53 of a table)
  if (!h->l2_children && P > 0) {
    const int nwt = nwt_for(std::max(1, h->cs.nv));
    child_fn cf = h->kw == 1 ? child_kernel<1>(nwt, h->prog) : child_kernel<2>(nwt, h->prog);
    const size_t csm = ((size_t)(1 << h->child_slots_log2) + 1) * (h->kw + h->cs.ds.ns) * 8;
    int occ = 0;
    if (cudaFuncSetAttribute((const void*)cf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cf, BLOCK, csm) == cudaSuccess && occ > 0) {
      const int cg = occ * h->sms;
      if (P >= 3 * cg) P = P / cg * cg;
    }
    cudaGetLastError();
  }
  h->P0 = std::min(P, cap_parts);
  if (getenv("AGGB_P0")) h->P0 = atoi(getenv("AGGB_P0"));  // experiment override
  h->fanout_need = (int64_t)h->P0 * h->nsub0;
  wc_plan(h, spill_groups);
  return AGGB_OK;
}

// The write-combined level-0 path (wc2.cuh) for budgeted pre-partitioning of
// one-word keys and one int64 value column with an integer COUNT/SUM/MIN/MAX
// spec.  After the table froze, level 0 routes every record into the run of its
// hash range; every run is aggregated by one child CTA with a compact table
// (u32 states) in shared memory, seeded with the resident keys of its range, in
// whole waves: the number of runs is the smallest multiple of the SM count that
// leaves every child table at most half full, and the runs' write-combining
// rings must fit the scan's shared memory beside its input stages.
constexpr int WC_CBLK = 1024, WC_CRL = 4;
// scan shapes (records per thread and tile x input stages): the tile bounds what one
// run receives between two window moves (a run's window holds 9-16 records)
struct WcShape {
  int blk, R, NS;
  void (*fn)(Wc2Args);
  size_t (*bytes)(int);
};
static const WcShape WC_SHAPES[] = {
    {512, 4, 3, k_scan_wc<512, 4, 3>, Wc2Layout<512, 4, 3>::bytes},
    {512, 4, 2, k_scan_wc<512, 4, 2>, Wc2Layout<512, 4, 2>::bytes},
    {512, 2, 4, k_scan_wc<512, 2, 4>, Wc2Layout<512, 2, 4>::bytes},
};
const WcShape& wc_shape() {
  const int i = getenv("AGGB_WC_SHAPE") ? atoi(getenv("AGGB_WC_SHAPE")) : 0;
  return WC_SHAPES[std::max(0, std::min(2, i))];
}
void wc_plan(Handle* h, double spill_groups) {
  h->wc = false;
  const aggb_config& c = h->cfg;
  if (c.algo != AGGB_PRE_PARTITIONING || h->kw != 1 || h->cs.nv != 1 || (h->prog != 1 && h->prog != 2) ||
      h->unlimited || h->l2_capped || c.level != 0 || h->cs.ds.vty[0] != TY_I64 || getenv("AGGB_NO_WC") ||
      getenv("AGGB_FORCE_L2_CHILDREN"))
    return;
  // slots of a child table: 8-byte key + the extended state words (the level-0 slot of a seeded key)
  const int we = h->prog == 2 ? CwWords<CpC2>::W_EXT : CwWords<CpC1>::W_EXT;
  const int tbytes = 220 * 1024;
  const int nslots = (tbytes / (8 + 4 * we) - 1) / 4 * 4;
  const int sms = std::max(1, h->sms);
  const double groups = (double)std::max<int64_t>(1, h->budget) + std::max(1.0, spill_groups);
  int I = (int)std::ceil(groups / (0.5 * nslots));
  I = std::max(1, (I + sms - 1) / sms * sms);
  if (getenv("AGGB_WC_RUNS")) I = std::max(1, atoi(getenv("AGGB_WC_RUNS")));  // experiment override
  if (wc_shape().bytes(I) + 1024 >= 227 * 1024) return;
  h->wc = true;
  h->wc_table_bytes = tbytes;
  h->P0 = I;
  h->nsub0 = 1;
  h->fanout_need = h->P0;
  h->l2_children = false;
}

int setup_table(Handle* h) {
  const int64_t sx = 2;
  int64_t slots = next_pow2(std::max<int64_t>(64, sx * std::max<int64_t>(h->budget, h->skew_cap)));
  GTable& t = h->tab;
  t.stride = (uint64_t)slots + 1;
  t.mask = (uint64_t)slots - 1;
  // in-memory tables beyond L2 take the slot-major state layout: a record's
  // updates touch one sector of states instead of one per field (C4 / C3
  // hash_sort: random HBM sectors per record 3 -> 2)
  const int ns_t = std::max(1, h->cs.ds.ns);
  const bool aos = ((h->unlimited && (double)slots * (8.0 * h->kw + 8.0 * ns_t) > 0.5 * 126e6) ||
                    getenv("AGGB_AOS_ALL")) &&
                   ns_t <= 4 && !getenv("AGGB_SOA_STATES");
  t.fstride = aos ? 1 : (uint64_t)slots + 1;
  t.sstride = aos ? (uint64_t)ns_t : 1;
  h->aos_planned = aos;
  t.bmask = (uint64_t)(slots / (h->kw == 1 ? 4 : 2)) - 1;
  // Budgeted tables grant exactly the budget.  An unlimited (in-memory) table's
  // "budget" is only a size estimate: grant up to 3/4 of its slots, so the
  // reservations stranded by racing duplicate inserts (returned to per-CTA
  // caches) cannot freeze a table that still has room.
  t.cap = h->unlimited ? (uint64_t)slots * 3 / 4 : (uint64_t)h->budget;
  t.seed = level_seed(h->cfg.seed, SALT_SLOT, h->cfg.level);
  TRY(h->tkeys.ensure((size_t)(t.stride + 1) * h->kw * 8, &h->hw));
  TRY(h->tstates.ensure((size_t)t.stride * std::max(1, h->cs.ds.ns) * 8, &h->hw));
  TRY(h->thdr.ensure(sizeof(TableHdr), &h->hw));
  t.keys = h->tkeys.as<uint64_t>();
  t.states = h->tstates.as<uint64_t>();
  t.hdr = h->thdr.as<TableHdr>();
  h->has_table = true;
  // bloom: ~8 bits per resident key, at most 128 KB (it lives in SMEM), off when too sparse
  if (h->cfg.algo == AGGB_PRE_PARTITIONING && !getenv("AGGB_NO_BLOOM")) {
    int64_t words = next_pow2(std::max<int64_t>(1, (int64_t)(8 * t.cap) / 64));
    words = std::min<int64_t>(words, 16384);
    if (words * 64 >= 4 * (int64_t)t.cap) {
      h->bloom_words = words;
      h->bloom_seed = level_seed(h->cfg.seed, 0x66, h->cfg.level);
      TRY(h->bloom.ensure((size_t)words * 8, &h->hw));
    }
  }
  return table_reset(h);
}

int begin_run(Handle* h) {
  CU(cudaMemsetAsync(h->scratch.p, 0, h->scratch.bytes, h->st));
  CU(cudaMemsetAsync(h->pool_ctr.p, 0, h->pool_ctr.bytes, h->st));
  h->pool_bound = 0;
  h->next_set_id = 1;
  h->records = 0;
  h->launches = 0;
  h->finished = false;
  h->first_push = true;
  if (h->has_table && h->skew_cap) h->tab.cap = (uint64_t)h->budget;
  if (h->has_table && h->aos_planned) {  // restore the planned layout (table_reset below re-inits)
    h->tab.fstride = 1;
    h->tab.sstride = (uint64_t)std::max(1, h->cs.ds.ns);
  }
  h->hash_sort_runs = 0;
  h->sort_n = 0;
  memset(&h->met, 0, sizeof(h->met));
  memset(&h->result, 0, sizeof(h->result));
  int algo = h->cfg.algo;
  uint64_t seed = h->cfg.seed;
  int lv = h->cfg.level;
  if (algo == AGGB_ORIGINAL_HH) {
    h->raw0 = {make_set(h, h->P0 + 1, h->cs.nv, 0, level_seed(seed, SALT_SPILL, lv)), 0};
    h->part0 = {make_set(h, h->P0 + 1, h->cs.ds.ns, 1, level_seed(seed, SALT_SPILL, lv)), 0};
  } else {
    int pp = std::min(h->P0, max_parts_for(h->kw + h->cs.ds.ns));
    // dynamic destaging: a destaged partition's raw records and its evicted
    // groups must land in the same partition of both sets
    const bool dd = algo == AGGB_DYNAMIC_DESTAGING || algo == AGGB_SHARED_HASH;
    h->raw0 = {make_set(h, dd ? pp : h->P0, h->cs.nv, 0,
                        level_seed(seed, SALT_SPILL, lv)), 0};
    h->part0 = {make_set(h, pp, h->cs.ds.ns, 1, level_seed(seed, SALT_SPILL, lv)), 0};
  }
  h->raw0_live = h->part0_live = false;
  if (algo == AGGB_DYNAMIC_DESTAGING || algo == AGGB_SHARED_HASH) {
    const int P = h->part0.ss.nparts;
    h->sh_stage = 0;
    TRY(h->dd_spilled.ensure((size_t)P + 16, &h->hw));
    CU(cudaMemsetAsync(h->dd_spilled.p, 0, (size_t)P + 16, h->st));
    h->dd_host.assign((size_t)P, 0);
    h->dd_evictions = 0;
  }
  if (h->has_table) TRY(table_reset(h));
  h->wc_used = false;
  h->wc_launches = 0;
  h->wc_entries = 0;
  if (h->wc) {
    const size_t NP = (size_t)h->P0;
    TRY(h->wc_meta.ensure(wc_meta_bytes((int)NP), &h->hw));
    CU(cudaMemsetAsync(h->wc_meta.p, 0, wc_meta_bytes((int)NP), h->st));
    if (h->wc_ovf.p) CU(cudaMemsetAsync(h->wc_ovf.p, 0, 8, h->st));
  }
  return AGGB_OK;
}

// ---------------------------------------------------------------------------
// push
// ---------------------------------------------------------------------------

struct Staged {
  const void* k[AGGB_MAX_KEYS];
  const void* v[AGGB_MAX_VALS];
  std::vector<DBuf> owned;
};

int stage_input(Handle* h, const aggb_input* in, Staged& sg) {
  for (int w = 0; w < h->kw; w++) sg.k[w] = in->key[w];
  for (int w = 0; w < h->spec.n_vals; w++) sg.v[w] = in->val[w];
  if (!in->on_host) return AGGB_OK;
  // host pointers: copy each column (strided rows whole) into the handle's
  // grow-only staging buffer; the caller's memory should be pinned for speed
  size_t total = 0;
  std::vector<size_t> off;
  auto span = [&](int64_t stride, int elem) {
    int64_t sb = stride ? stride : elem;
    return (size_t)((in->n_rows - 1) * sb + elem);
  };
  for (int w = 0; w < h->kw; w++) {
    off.push_back(total);
    total += (span(in->key_stride[w], h->spec.key_type[w] == AGGB_I32 ? 4 : 8) + 255) & ~(size_t)255;
  }
  for (int w = 0; w < h->spec.n_vals; w++) {
    off.push_back(total);
    total += (span(in->val_stride[w], h->spec.val_type[w] == AGGB_I32 ? 4 : 8) + 255) & ~(size_t)255;
  }
  TRY(h->stage.ensure(total, &h->hw));
  int q = 0;
  for (int w = 0; w < h->kw; w++, q++) {
    size_t b = span(in->key_stride[w], h->spec.key_type[w] == AGGB_I32 ? 4 : 8);
    CU(cudaMemcpyAsync(h->stage.as<uint8_t>() + off[q], in->key[w], b, cudaMemcpyHostToDevice, h->st));
    sg.k[w] = h->stage.as<uint8_t>() + off[q];
  }
  for (int w = 0; w < h->spec.n_vals; w++, q++) {
    size_t b = span(in->val_stride[w], h->spec.val_type[w] == AGGB_I32 ? 4 : 8);
    CU(cudaMemcpyAsync(h->stage.as<uint8_t>() + off[q], in->val[w], b, cudaMemcpyHostToDevice, h->st));
    sg.v[w] = h->stage.as<uint8_t>() + off[q];
  }
  return AGGB_OK;
}

int ensure_defer(Handle* h, int64_t T, int payload_words) {
  // in flight at a freeze: every CTA's current and prefetched tile (x2 headroom);
  // records of payload_words words (raw values, or partial states in L2 children)
  int64_t need = (int64_t)h->sms * 8 * T + 4096;
  const int words = h->kw + std::max(1, payload_words);
  if (need <= h->defer_cap && words <= h->defer_words) return AGGB_OK;
  need = std::max(need, h->defer_cap);
  TRY(h->defer.ensure((size_t)need * std::max(words, h->defer_words) * 8, &h->hw));
  h->defer_cap = need;
  h->defer_words = std::max(words, h->defer_words);
  return AGGB_OK;
}

int fill_probe(Handle* h, const ColSrc& col, int col_kind, const SpillSet& ss);

// k_scan_wc reads the key and value columns with 16-byte bulk copies
bool wc_eligible(Handle* h, const ColSrc& col) {
  // (a run's claim counter has 23 bits: at most ~8M records per CTA and launch)
  return col.nv == 1 && dense8(col, 1) && col.kty[0] == TY_I64 && col.vty[0] == TY_I64 &&
         col.n + h->defer_cap <= (int64_t)1200000000 &&
         ((uintptr_t)col.key[0] & 15) == 0 && ((uintptr_t)col.val[0] & 15) == 0 && !h->hot_ready &&
         h->pool_bound + (uint64_t)(col.n + h->defer_cap) / 256 +
                 (uint64_t)h->sms * (4ull * h->P0 + 128) < 0xFFFFF0ull;
}

// the runs' lists of resident slots (the frozen table's keys by routing hash)
int wc_build(Handle* h) {
  const uint64_t seed64 = level_seed(h->cfg.seed, SALT_PART, h->cfg.level);
  const uint32_t seed = (uint32_t)seed64 ^ (uint32_t)(seed64 >> 32);
  // a list holds twice a run's share of the budget (small budgets: all of it)
  const uint64_t cap = h->tab.cap;
  h->wc_ocap = (uint32_t)std::min<uint64_t>(cap + 1, 2 * cap / (uint64_t)h->P0 + 1024);
  TRY(h->wc_olist.ensure((size_t)h->P0 * h->wc_ocap * 4, &h->hw));
  TRY(h->wc_olist_n.ensure((size_t)h->P0 * 4, &h->hw));
  CU(cudaMemsetAsync(h->wc_olist_n.p, 0, (size_t)h->P0 * 4, h->st));
  int pe = prof_begin(h, 16);
  k_wc2_build<<<h->sms * 4, 256, 0, h->st>>>(h->tab, seed, h->wc_olist.as<uint32_t>(), h->wc_olist_n.as<uint32_t>(),
                                             h->wc_ocap, (uint32_t)h->P0);
  prof_end(h, pe);
  CU(cudaGetLastError());
  h->launches++;
  return AGGB_OK;
}

// PROBE through k_scan_wc: every record of the batch (and FILL's deferral list) into its run
int wc_probe(Handle* h, const ColSrc& col, const SpillSet& ss) {
  const int NP = h->P0;
  const int grid = h->sms;
  const WcShape& shp = wc_shape();
  const int64_t nlin_cap = h->defer_cap;
  // page lists: every CTA reserves a block of entries per run and launch (twice
  // the pages it expects to open, at least 2); a run that outgrows its block
  // takes single entries
  h->wc_launches++;
  const int64_t exp_pages = (col.n + nlin_cap) / 512 / ((int64_t)grid * std::max(1, NP)) + 1;
  const uint32_t blk = (uint32_t)std::min<int64_t>(64, 2 * exp_pages);
  h->wc_entries += (int64_t)grid * blk + (col.n + nlin_cap) / 512 / std::max(1, NP);  // per run, this launch
  const uint32_t need_cap = (uint32_t)std::min<int64_t>(0x7FFFFFFF, h->wc_entries + 2 * (int64_t)grid + 64);
  if (need_cap > h->wc_plist_cap) {
    DBuf nb;
    const uint32_t new_cap = std::max(need_cap, h->wc_used ? 2 * h->wc_plist_cap : 0u);
    TRY(nb.ensure((size_t)NP * new_cap * 4, &h->hw));
    CU(cudaMemsetAsync(nb.p, 0xFF, (size_t)NP * new_cap * 4, h->st));
    if (h->wc_used && h->wc_plist_cap)
      CU(cudaMemcpy2DAsync(nb.p, (size_t)new_cap * 4, h->wc_plist.p, (size_t)h->wc_plist_cap * 4,
                           (size_t)h->wc_plist_cap * 4, (size_t)NP, cudaMemcpyDeviceToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
    h->wc_plist.release();
    h->wc_plist = nb;
    nb.p = nullptr;
    h->wc_plist_cap = new_cap;
  }
  // the overflow list of pages past a run's list: every page the run's launches can open
  {
    const uint64_t need = (uint64_t)((h->records + col.n + nlin_cap) / 512) + (uint64_t)h->wc_launches * grid * NP + 1024;
    if (need > h->wc_ovf_cap) {
      DBuf nb;
      const uint64_t cap2 = std::min<uint64_t>(0xFFFFFFF0ull, need + need / 2);
      TRY(nb.ensure((size_t)(cap2 + 1) * 8, &h->hw));
      if (h->wc_ovf.p && h->wc_used) {
        CU(cudaMemcpyAsync(nb.p, h->wc_ovf.p, (size_t)(h->wc_ovf_cap + 1) * 8, cudaMemcpyDeviceToDevice, h->st));
      } else {
        CU(cudaMemsetAsync(nb.p, 0, 8, h->st));
      }
      CU(cudaStreamSynchronize(h->st));
      h->wc_ovf.release();
      h->wc_ovf = nb;
      nb.p = nullptr;
      h->wc_ovf_cap = (uint32_t)cap2;
    }
  }
  // pages: the records, plus each (CTA, run) chain's last page, plus stashes
  const int stash = 32;
  const uint64_t pages = (uint64_t)((col.n + nlin_cap) / 512) + 2ull * grid * NP + 4ull * grid * stash + 64;
  TRY(pool_ensure(h, pages));
  Wc2Args a;
  memset(&a, 0, sizeof(a));
  a.t = h->tab;
  {
    const uint64_t seed64 = level_seed(h->cfg.seed, SALT_PART, h->cfg.level);
    a.seed = (uint32_t)seed64 ^ (uint32_t)(seed64 >> 32);
  }
  a.key = (const unsigned long long*)col.key[0];
  a.val = (const unsigned long long*)col.val[0];
  a.n = col.n;
  a.start_tiles = SC(h) + 8;
  a.start_T = 0;
  {
    int nwt = nwt_for(std::max(1, col.nv));
    PassCfg pcfg = pass_kernel<1>(nwt, h->prog);
    a.start_T = (int64_t)pcfg.R * pcfg.blk;  // FILL's tile
  }
  a.lkey = (const unsigned long long*)h->defer.as<uint64_t>();
  a.lval = (const unsigned long long*)(h->defer.as<uint64_t>() + h->defer_cap);
  a.lcount = SC(h) + 10;
  a.pool = pool_of(h);
  a.set_id = ss.id;
  a.NP = NP;
  a.plist = h->wc_plist.as<uint32_t>();
  a.plist_n = wc_pn(h);
  a.plist_cap = h->wc_plist_cap;
  a.plist_blk = blk;
  a.ovf = h->wc_ovf.as<unsigned long long>() + 1;
  a.ovf_n = h->wc_ovf.as<unsigned long long>();
  a.ovf_cap = h->wc_ovf_cap;
  a.part_recs = wc_recs(h);
  a.stats = SC(h);
  a.vinfo = wc_vinfo(h);
  a.fail = wc_fail(h);
  a.stash = stash;
  a.nohot = getenv("AGGB_NO_HOT") ? 1 : 0;
  a.prog = h->prog;
  a.nosend = getenv("AGGB_WC_NOSEND") ? 1 : 0;  // (experiment: lines are not written; results are wrong)
  auto fs = shp.fn;
  const size_t smem = shp.bytes(NP);
  if (h->wc_scan_smem != smem) {  // (once per handle: the call costs host time on every step)
    CU(cudaFuncSetAttribute((const void*)fs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    h->wc_scan_smem = smem;
  }
  int pe = prof_begin(h, 15);
  fs<<<grid, shp.blk + 32, smem, h->st>>>(a);  // + the producer warp
  prof_end(h, pe);
  CU(cudaGetLastError());
  h->launches++;
  h->wc_used = true;
  return AGGB_OK;
}

int push_hybrid(Handle* h, const ColSrc& col) {
  int algo = h->cfg.algo;
  unsigned long long* ctrA = SC(h) + 8;
  unsigned long long* ctrB = SC(h) + 9;
  if (algo == AGGB_ORIGINAL_HH) {
    PassPlan pp;
    pp.mode = MODE_ROUTE;
    pp.col = col;
    pp.ss = h->raw0.ss;
    // partition-0 share: the resident table should end ~90% full (the reference leaves the
    // same slack through the fudge factor, hybrid.py:89-99, :123-131)
    double G_t = std::max(1.0, h->cfg.stats_G_t);
    double r_res = h->cfg.stats_G_t > 0 ? std::min(1.0, 0.9 * (double)h->budget / G_t) : 1.0;
    double c0 = std::floor(r_res * 4294967296.0);
    pp.cut0 = (uint32_t)std::min(4294967295.0, std::max(1.0, c0));
    if (r_res >= 1.0) pp.cut0 = 0xFFFFFFFFu;
    pp.part_seed = level_seed(h->cfg.seed, SALT_PART, h->cfg.level);
    pp.counter = ctrB;
    TRY(launch_pass(h, pp));
    h->raw0_live = true;
    return AGGB_OK;
  }
  if (algo == AGGB_HASH_SORT) {  // FILL only: push_hash_sort handles freezes (cuts)
    int nwt = nwt_for(std::max(1, col.nv));
    PassCfg pcfg = h->kw == 1 ? pass_kernel<1>(nwt, h->prog) : pass_kernel<2>(nwt, h->prog);
    TRY(ensure_defer(h, (int64_t)pcfg.R * pcfg.blk, col.nv));
    CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
    PassPlan f;
    f.mode = MODE_FILL;
    f.col = col;
    f.counter = ctrA;
    return launch_pass(h, f);
  }
  TRY(fill_probe(h, col, 0, h->raw0.ss));
  h->raw0_live = true;
  return AGGB_OK;
}

// FILL then PROBE (kernel boundary = freeze point) of a column source whose
// records are of kind col_kind; misses spill to set ss.  pre_partitioning's
// push, and the body of an L2-table child (drain).
int fill_probe(Handle* h, const ColSrc& col, int col_kind, const SpillSet& ss) {
  unsigned long long* ctrA = SC(h) + 8;
  unsigned long long* ctrB = SC(h) + 9;
  int nwt = nwt_for(std::max(1, col.nv));
  PassCfg pcfg = h->kw == 1 ? pass_kernel<1>(nwt, h->prog) : pass_kernel<2>(nwt, h->prog);
  TRY(ensure_defer(h, (int64_t)pcfg.R * pcfg.blk, col.nv));
  CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
  const bool use_wc = h->wc && col_kind == 0 && ss.id == h->raw0.ss.id && wc_eligible(h, col);
  PassPlan f;
  f.mode = MODE_FILL;
  f.col = col;
  f.col_kind = col_kind;
  f.counter = ctrA;
  TRY(launch_pass(h, f));
  // PROBE the remainder and the deferred records against the frozen table.
  if (use_wc) return wc_probe(h, col, ss);
  // PROBE the remainder and the deferred records against the frozen table.
  // The filter is rebuilt from the table as it stands after FILL (a kernel boundary, so
  // the key set is final once frozen); while the table is not frozen PROBE has no work.
  if (h->bloom_words) {
    CU(cudaMemsetAsync(h->bloom.p, 0, (size_t)h->bloom_words * 8, h->st));
    int pe = prof_begin(h, 12);
    if (h->kw == 1)
      k_bloom_build<1><<<h->sms * 4, 256, 0, h->st>>>(h->tab, h->bloom.as<uint64_t>(), (uint32_t)h->bloom_words - 1);
    else
      k_bloom_build<2><<<h->sms * 4, 256, 0, h->st>>>(h->tab, h->bloom.as<uint64_t>(), (uint32_t)h->bloom_words - 1);
    prof_end(h, pe);
    h->launches++;
  }
  PassPlan p;
  p.mode = MODE_PROBE;
  p.col = col;
  p.col_kind = col_kind;
  p.use_start = true;
  p.lin = h->defer.as<uint64_t>();
  p.lin_stride = h->defer_cap;
  p.lin_count = SC(h) + 10;
  p.lin_kind = col_kind;
  p.lin_words = col.nv;
  p.ss = ss;
  p.counter = ctrB;
  return launch_pass(h, p);
}


// hash_sort (hash_sort.py:40-78): aggregate; when the table is full, cut it to a
// run of partial states (hash-partitioned so the final merge-with-fold runs as
// shared-memory children), reset, and continue with the deferred records and
// the rest of the batch.
int cut_run(Handle* h) {
  // the run holds at most the table's capacity (+ the escape group): a persistent
  // buffer of that size, no read-back of the group count
  int words = h->kw + h->cs.ds.ns;
  int64_t n = (int64_t)h->tab.cap + 2;
  DBuf& tmp = h->cut_tmp;
  TRY(tmp.ensure((size_t)n * words * 8, &h->hw));
  OutBuf o;
  o.keys = tmp.as<uint64_t>();
  o.vals = tmp.as<uint64_t>() + (size_t)h->kw * n;
  o.cap = n;
  o.count = SC(h) + 11;
  o.partial = 1;
  CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
  TRY(flush_table(h, true, &o));
  PassPlan g;
  g.mode = MODE_GRACE;
  g.lin = tmp.as<uint64_t>();
  g.lin_stride = n;
  g.lin_count = SC(h) + 11;
  g.lin_kind = 1;
  g.lin_words = h->cs.ds.ns;
  g.ss = h->part0.ss;
  g.counter = SC(h) + 9;
  TRY(launch_pass(h, g));
  h->part0_live = true;
  h->hash_sort_runs++;
  return table_reset(h);
}

// hash_sort when the table fills about as fast as records arrive (little
// aggregation per run: C5 cuts every ~84K records): instead of a host round
// trip per cut, the rest of the batch is cut blind — chunks of `cap` records
// (at most cap distinct keys, so the table never refuses: its capacity check is
// lifted to the physical limit while the chunk bounds the groups it can hold),
// each aggregated, flushed as a partial run into an accumulation buffer and
// cleared on the way (k_flush_table<CLEAR>); every K runs the buffer is
// hash-partitioned into part0 (GRACE) like cut_run does.  Results are those of
// cutting when full; the runs are only cut earlier than full.
int hash_sort_blind(Handle* h, const ColSrc& rest) {
  const int64_t c = std::max<int64_t>(1, (int64_t)h->tab.cap);
  const int words = h->kw + h->cs.ds.ns;
  // runs accumulate to ~1/8 of the batch (8M to 64M records) per GRACE pass:
  // every pass leaves a partly filled page per (CTA, partition), so fewer passes
  // fragment the pool less (C5 at 500M records: 60 passes left ~16 GB of slack)
  const int64_t acc_recs = std::max<int64_t>(8 << 20, std::min<int64_t>(64 << 20, rest.n / 8));
  const int64_t K = std::max<int64_t>(1, std::min<int64_t>((rest.n + c - 1) / c, acc_recs / (c + 2)));
  const int64_t acc_cap = K * (c + 2);
  TRY(h->cut_tmp.ensure((size_t)acc_cap * words * 8, &h->hw));
  OutBuf o;
  o.keys = h->cut_tmp.as<uint64_t>();
  o.vals = h->cut_tmp.as<uint64_t>() + (size_t)h->kw * acc_cap;
  o.cap = acc_cap;
  o.count = SC(h) + 11;
  o.partial = 1;
  CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
  CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
  const uint64_t cap0 = h->tab.cap;
  // the cut loop on the device (cuts.cuh): one persistent launch per K chunks, then their GRACE pass
  typedef void (*cut_fn)(CutArgs);
  cut_fn cf = nullptr;
  {
    const int nwt = nwt_for(std::max(1, rest.nv));
    if (h->kw == 1 && nwt == 1) cf = k_blind_cuts<1, 1, PD>;
    else if (h->kw == 1 && nwt == 2) cf = k_blind_cuts<1, 2, PD>;
    else if (h->kw == 1 && nwt == 4) cf = k_blind_cuts<1, 4, PD>;
    else if (h->kw == 2 && nwt == 1) cf = k_blind_cuts<2, 1, PD>;
    else if (h->kw == 2 && nwt == 2) cf = k_blind_cuts<2, 2, PD>;
    else if (h->kw == 2 && nwt == 4) cf = h->prog == 5 ? k_blind_cuts<2, 4, ProgC5> : k_blind_cuts<2, 4, PD>;
    if (getenv("AGGB_NO_FUSED_CUTS")) cf = nullptr;
  }
  int occ = 0, coop = 0;
  if (cf) {
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
    if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cf, CUT_BLK, 0) != cudaSuccess || occ < 1) cf = nullptr;
  }
  if (cf) {
    TRY(h->cut_bar.ensure(64, &h->hw));
    CU(cudaMemsetAsync(h->cut_bar.p, 0, 64, h->st));
    const int grid = h->sms;  // (more CTAs only make the grid barrier dearer: 4 x 256 threads per SM 382 ms, 1 x 256 287 ms on C5)
    const int64_t nch = (rest.n + c - 1) / c;
    int rc = AGGB_OK;
    for (int64_t k0 = 0; k0 < nch && rc == AGGB_OK; k0 += K) {
      CutArgs ca;
      memset(&ca, 0, sizeof(ca));
      ca.t = h->tab;
      ca.sp = h->cs.ds;
      ca.col = rest;
      ca.first = k0 * c;
      ca.chunk = c;
      ca.nchunks = std::min<int64_t>(K, nch - k0);
      ca.o = o;
      ca.bar = h->cut_bar.as<unsigned>();
      ca.stats = SC(h);
      void* args[] = {&ca};
      int pe = prof_begin(h, 18);
      CU(cudaLaunchCooperativeKernel((const void*)cf, dim3(grid), dim3(CUT_BLK), args, 0, h->st));
      prof_end(h, pe);
      h->launches++;
      h->hash_sort_runs += ca.nchunks;
      PassPlan g;
      g.mode = MODE_GRACE;
      g.lin = h->cut_tmp.as<uint64_t>();
      g.lin_stride = acc_cap;
      g.lin_count = SC(h) + 11;
      g.lin_kind = 1;
      g.lin_words = h->cs.ds.ns;
      g.ss = h->part0.ss;
      g.counter = SC(h) + 9;
      if ((rc = launch_pass(h, g))) break;
      CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
      h->part0_live = true;
    }
    CU(cudaMemsetAsync(h->tab.hdr, 0, sizeof(TableHdr), h->st));
    return rc;
  }
  h->tab.cap = (h->tab.mask + 1) * 3 / 4;  // no refusals: the chunk bounds the keys
  int rc = AGGB_OK;
  int64_t in_acc = 0;
  for (int64_t off = 0; off < rest.n && rc == AGGB_OK; off += c) {
    ColSrc ch = rest;
    ch.n = std::min<int64_t>(c, rest.n - off);
    for (int w = 0; w < h->kw; w++) ch.key[w] = rest.key[w] + off * rest.kstride[w];
    for (int w = 0; w < rest.nv; w++) ch.val[w] = rest.val[w] + off * rest.vstride[w];
    PassPlan f;
    f.mode = MODE_FILL;
    f.col = ch;
    f.counter = SC(h) + 8;
    if ((rc = launch_pass(h, f))) break;
    if ((rc = flush_table(h, true, &o, true))) break;
    h->hash_sort_runs++;
    if (++in_acc == K || off + c >= rest.n) {
      PassPlan g;
      g.mode = MODE_GRACE;
      g.lin = h->cut_tmp.as<uint64_t>();
      g.lin_stride = acc_cap;
      g.lin_count = SC(h) + 11;
      g.lin_kind = 1;
      g.lin_words = h->cs.ds.ns;
      g.ss = h->part0.ss;
      g.counter = SC(h) + 9;
      if ((rc = launch_pass(h, g))) break;
      CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
      h->part0_live = true;
      in_acc = 0;
    }
  }
  h->tab.cap = cap0;
  return rc;
}

int push_hash_sort(Handle* h, const ColSrc& col0) {
  int nwt = nwt_for(std::max(1, col0.nv));
  PassCfg pcfg = h->kw == 1 ? pass_kernel<1>(nwt, h->prog) : pass_kernel<2>(nwt, h->prog);
  int64_t T = (int64_t)pcfg.R * pcfg.blk;
  TRY(ensure_defer(h, T, col0.nv));
  std::vector<ColSrc> queue{col0};
  std::vector<DBuf> temps;
  int rc = AGGB_OK;
  unsigned long long last_committed = ~0ull;
  while (!queue.empty() && rc == AGGB_OK) {
    ColSrc cur = queue.back();
    queue.pop_back();
    if (cur.n <= 0) continue;
    CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
    PassPlan f;
    f.mode = MODE_FILL;
    f.col = cur;
    f.counter = SC(h) + 8;
    if ((rc = launch_pass(h, f))) break;
    unsigned long long tiles = 0, nd = 0, committed = 0;
    int frozen = 0;
    CU(cudaMemcpyAsync(&tiles, SC(h) + 8, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(&nd, SC(h) + 10, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(&frozen, &h->tab.hdr->frozen, 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(&committed, &h->tab.hdr->committed, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (getenv("AGGB_TRACE"))
      fprintf(stderr, "[aggb] hash_sort FILL: %lld records, tiles %llu, deferred %llu, frozen %d, keys %llu\n",
              (long long)cur.n, tiles, nd, frozen, committed);
    if (!frozen && !nd) continue;
    // A freeze with room left is premature: racing inserts of one key each took a
    // reservation before their CAS, and the losers' reservations stayed in their
    // CTAs.  The reference cuts a run only when the table is full, so reopen the
    // table (grants = keys held) and feed the rest again instead of cutting.
    if (frozen && committed + std::max<uint64_t>(64, h->tab.cap / 64) < h->tab.cap &&
        (committed != last_committed || tiles > 0)) {
      // the keys held count against the chunk region first (kernels.cuh CapCache)
      const unsigned long long cc = h->last_cap_chunked;
      h->reopen[0] = committed <= cc ? 0ull : committed - cc;  // exact-region grants
      h->reopen[1] = committed <= cc ? committed : cc;          // chunk-region grants
      CU(cudaMemcpyAsync(&h->tab.hdr->groups, &h->reopen[0], 8, cudaMemcpyHostToDevice, h->st));
      CU(cudaMemcpyAsync(&h->tab.hdr->chunked, &h->reopen[1], 8, cudaMemcpyHostToDevice, h->st));
      CU(cudaMemsetAsync(&h->tab.hdr->frozen, 0, 4, h->st));
      frozen = 0;
    }
    last_committed = committed;
    int64_t start = std::min<int64_t>(cur.n, (int64_t)tiles * T);
    // keep the deferred records (the deferral buffer is reused by the next FILL)
    ColSrc dc;
    memset(&dc, 0, sizeof(dc));
    if (nd) {
      DBuf tmp;
      int words = h->kw + cur.nv;
      if ((rc = tmp.ensure((size_t)nd * words * 8, nullptr))) break;
      for (int w = 0; w < words; w++)
        CU(cudaMemcpyAsync(tmp.as<uint64_t>() + w * nd, h->defer.as<uint64_t>() + w * h->defer_cap, nd * 8,
                           cudaMemcpyDeviceToDevice, h->st));
      dc.n = (int64_t)nd;
      for (int w = 0; w < h->kw; w++) {
        dc.key[w] = (const uint8_t*)(tmp.as<uint64_t>() + w * nd);
        dc.kstride[w] = 8;
        dc.kty[w] = TY_I64;
      }
      dc.nv = cur.nv;
      for (int w = 0; w < cur.nv; w++) {
        dc.val[w] = (const uint8_t*)(tmp.as<uint64_t>() + (h->kw + w) * nd);
        dc.vstride[w] = 8;
        dc.vty[w] = (h->cs.ds.vty[w] == TY_F64) ? TY_F64 : TY_I64;
      }
      temps.push_back(tmp);
    }
    if (frozen && (rc = cut_run(h))) break;
    if (start < cur.n) {
      ColSrc rest = cur;
      rest.n = cur.n - start;
      for (int w = 0; w < h->kw; w++) rest.key[w] = cur.key[w] + start * cur.kstride[w];
      for (int w = 0; w < cur.nv; w++) rest.val[w] = cur.val[w] + start * cur.vstride[w];
      // the table filled early in the batch (at least 8 more cuts ahead, each a
      // host round trip and a GRACE pass of its own): cut the rest blind
      if (frozen && rest.n > 8 * std::max<int64_t>(start, (int64_t)h->tab.cap) && !getenv("AGGB_HS_NO_BLIND")) {
        if ((rc = hash_sort_blind(h, rest))) break;
      } else {
        queue.push_back(rest);
      }
    }
    if (nd) queue.push_back(dc);  // deferred records first
  }
  cudaStreamSynchronize(h->st);
  for (auto& t : temps) t.release();
  return rc;
}

// ---------------------------------------------------------------------------
// recursion over spilled partitions (hybrid.py:244-277)
// ---------------------------------------------------------------------------

int drain(Handle* h, SetInfo a, bool a_live, SetInfo b, bool b_live, int level) {
  int depth = level;
  int nsub = h->nsub0;  // sub-passes per child at this level (plan)
  bool split_done = false;
  Trace tr;
  for (int guard = 0; guard < 24; guard++) {
    if (!a_live && !b_live) return AGGB_OK;
    if (!a_live) {  // normalize: the live set first
      std::swap(a, b);
      std::swap(a_live, b_live);
    }
    int nparts = std::max(a.ss.nparts, b_live ? b.ss.nparts : 0);
    int nsets = b_live ? 2 : 1;
    if (depth == level && !split_done) {  // level-0 sets: a set with fewer partitions (wide partial states) needs more sub-passes
      const int pmin = b_live ? std::min(a.ss.nparts, b.ss.nparts) : a.ss.nparts;
      nsub = (int)std::max<int64_t>(h->nsub0, (h->fanout_need + pmin - 1) / std::max(1, pmin));
    }
    TRY(h->part_records.ensure((size_t)nparts * 8, &h->hw));
    TRY(h->part_pages.ensure((size_t)nparts * 8, &h->hw));
    TRY(h->cursor.ensure((size_t)nparts * 8, &h->hw));
    CU(cudaMemsetAsync(h->part_records.p, 0, (size_t)nparts * 8, h->st));
    CU(cudaMemsetAsync(h->part_pages.p, 0, (size_t)nparts * 8, h->st));
    PagePool pp = pool_of(h);
    uint32_t first = 0;
    const uint32_t* last = h->pool_ctr.as<uint32_t>();
    int hg = h->sms * 4;
    SetInfo sets[2] = {a, b};
    for (int q = 0; q < nsets; q++) {
      int pe = prof_begin(h, 7);
      k_page_hist<<<hg, 256, 0, h->st>>>(pp, first, last, sets[q].ss.id, nparts, h->part_records.as<unsigned long long>(),
                                          h->part_pages.as<uint32_t>() + (size_t)q * nparts);
      prof_end(h, pe);
      h->launches++;
    }
    std::vector<unsigned long long> recs(nparts);
    std::vector<uint32_t> pages(2 * (size_t)nparts, 0);
    uint32_t ovfl = 0;
    unsigned long long cnt_now = 0;  // output rows so far (the page scatter does not change it)
    {
      const size_t o_pages = (size_t)nparts * 8, o_cnt = o_pages + (size_t)nparts * 8, o_ovfl = o_cnt + 8;
      TRY(h->hpin.ensure(o_ovfl + 8 + (size_t)nparts * 8 + ((size_t)2 * nparts + 1) * 8));  // + the plan's H2D
      uint8_t* hp = h->hpin.as<uint8_t>();
      CU(cudaMemcpyAsync(hp, h->part_records.p, (size_t)nparts * 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(hp + o_pages, h->part_pages.p, (size_t)nparts * 4 * nsets, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(hp + o_cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(hp + o_ovfl, h->pool_ctr.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      memcpy(recs.data(), hp, (size_t)nparts * 8);
      memcpy(pages.data(), hp + o_pages, (size_t)nparts * 4 * nsets);
      memcpy(&cnt_now, hp + o_cnt, 8);
      memcpy(&ovfl, hp + o_ovfl, 4);
    }
    if (ovfl) return fail(AGGB_CAPACITY_EXCEEDED, "spill page pool overflowed");
    std::vector<uint32_t> offs(2 * (size_t)nparts);
    std::vector<int64_t> item_off;
    uint32_t tot = 0;
    int nonempty = 0;
    int64_t max_items_out = 0;
    for (int p = 0; p < nparts; p++) {
      uint32_t na = pages[p], nb = nsets > 1 ? pages[nparts + p] : 0;
      offs[p] = tot;
      offs[nparts + p] = tot + na;
      if (na + nb) {
        item_off.push_back(tot);
        item_off.push_back(tot + na);
        nonempty++;
      }
      tot += na + nb;
    }
    item_off.push_back(tot);
    h->met.spilled_partitions += nonempty;
    if (!nonempty) return AGGB_OK;
    h->met.recursion_depth = std::max<int64_t>(h->met.recursion_depth, depth + 1);
    TRY(h->plist.ensure((size_t)tot * 8, &h->hw));
    TRY(h->item_off.ensure(item_off.size() * 8, &h->hw));
    {
      // staged behind the planning reads in the pinned buffer; its next host
      // write comes after the child's synchronize, its next device write is
      // stream-ordered after these copies
      uint8_t* hp = h->hpin.as<uint8_t>() + (size_t)nparts * 16 + 16;
      memcpy(hp, offs.data(), (size_t)nparts * 4 * nsets);
      memcpy(hp + (size_t)nparts * 8, item_off.data(), item_off.size() * 8);
      CU(cudaMemcpyAsync(h->cursor.p, hp, (size_t)nparts * 4 * nsets, cudaMemcpyHostToDevice, h->st));
      CU(cudaMemcpyAsync(h->item_off.p, hp + (size_t)nparts * 8, item_off.size() * 8, cudaMemcpyHostToDevice, h->st));
    }
    tr.mark(h->st, "drain: page hist + D2H");
    for (int q = 0; q < nsets; q++) {
      int pe = prof_begin(h, 7);
      k_page_scatter<<<hg, 256, 0, h->st>>>(pp, first, last, sets[q].ss.id, nparts,
                                             h->cursor.as<uint32_t>() + (size_t)q * nparts, h->plist.as<uint2>());
      prof_end(h, pe);
      h->launches++;
    }
    if (h->l2_children && nsets == 1) {
      // Children on the L2-resident table, one partition at a time, each the
      // reference's child operator (hybrid.py:244-277): fresh seeds, the full
      // budget, FILL then PROBE; what a child cannot hold spills to one shared
      // next-level set.  This level's pages stay untouched until the next
      // level starts (its spill is appended to the pool).
      const int ikind = a.ss.kind, inw = a.ss.rw - h->kw;
      std::vector<int64_t> irecs;
      for (int p = 0; p < nparts; p++)
        if (pages[p]) irecs.push_back((int64_t)recs[p]);
      int64_t maxr = 0, out_need = 0;
      for (int64_t r : irecs) {
        maxr = std::max(maxr, r);
        out_need += std::min<int64_t>(r, h->budget) + 2;
      }
      unsigned long long cnt = 0;
      CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      TRY(ensure_out(h, (int64_t)cnt + out_need + 16));
      TRY(h->l2stage.ensure((size_t)std::max<int64_t>(maxr, 1) * a.ss.rw * 8, &h->hw));
      const int64_t total = std::accumulate(irecs.begin(), irecs.end(), (int64_t)0);
      const int Pn = std::max(2, std::min(std::min(MAX_PARTS, max_parts_for(a.ss.rw)),
                                          (int)std::ceil((double)total / std::max<int64_t>(1, h->budget))));
      SetInfo nxt{make_set(h, Pn, inw, ikind, level_seed(h->cfg.seed, SALT_SPILL, depth + 1)), 0};
      OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
      const uint64_t seed0 = h->tab.seed;
      h->tab.seed = level_seed(h->cfg.seed, SALT_SLOT, depth + 1);
      tr.mark(h->st, "drain: l2 children setup");
      for (size_t i = 0; i < irecs.size(); i++) {
        const int64_t qa = item_off[2 * i], qb = item_off[2 * i + 2];
        TRY(table_reset(h));
        CU(cudaMemsetAsync(SC(h) + 16, 0, 8, h->st));
        const int gg = (int)std::min<int64_t>(qb - qa, (int64_t)h->sms * 8);
        k_gather_pages<<<std::max(gg, 1), 256, 0, h->st>>>(pool_of(h), h->plist.as<uint2>() + qa, qb - qa, a.ss.rw,
                                                          h->l2stage.as<uint64_t>(), irecs[i], SC(h) + 16);
        h->launches++;
        ColSrc c;
        memset(&c, 0, sizeof(c));
        c.n = irecs[i];
        for (int w = 0; w < h->kw; w++) {
          c.key[w] = (const uint8_t*)(h->l2stage.as<uint64_t>() + (size_t)w * irecs[i]);
          c.kstride[w] = 8;
          c.kty[w] = TY_I64;
        }
        c.nv = inw;
        for (int w = 0; w < inw; w++) {
          c.val[w] = (const uint8_t*)(h->l2stage.as<uint64_t>() + (size_t)(h->kw + w) * irecs[i]);
          c.vstride[w] = 8;
          c.vty[w] = (ikind == 0 && w < h->cs.ds.nv) ? h->cs.ds.vty[w] : TY_I64;
        }
        TRY(fill_probe(h, c, ikind, nxt.ss));
        TRY(flush_table(h, h->cfg.emit_partials != 0, &o));
      }
      h->tab.seed = seed0;
      CU(cudaStreamSynchronize(h->st));
      tr.mark(h->st, "drain: l2 children");
      a = nxt;
      a_live = true;
      b_live = false;
      depth++;
      continue;
    }
    // Partitions that would need >= 3 child sub-passes get one more grace level
    // instead (k_split: the partition is read twice and written once, where
    // sub-passes would read it nsub times); the children then take the
    // page-aligned sub-partitions in one pass each.
    // The split writes the whole set once more while its input stays live: when
    // the pages it needs cannot be mapped from free memory (C5 hash_sort at 500M
    // records: ~60 GB of partial-state runs), the children take sub-passes.
    bool split_fits = true;
    if (nsub >= 3 && nsets == 1) {
      int64_t tin = 0;
      for (int p = 0; p < nparts; p++) tin += (int64_t)recs[p];
      const int per = std::max(1, make_set(h, 1, a.ss.rw - h->kw, a.ss.kind, 0).per_page);
      uint32_t used = 0;
      CU(cudaMemcpyAsync(&used, h->pool_ctr.p, 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      const uint64_t pages = (uint64_t)std::min<uint32_t>(used, h->pool_cap) + (uint64_t)(tin / per) +
                             (uint64_t)nonempty * std::min(nsub, 1024) + 16;
      const size_t bytes = (size_t)pages * PAGE_BYTES;
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      if (bytes > h->pool_base.mapped && bytes - h->pool_base.mapped > (size_t)(0.9 * (double)fr) && h->cut_tmp.p) {
        h->cut_tmp.release();  // hash_sort's run accumulation buffer is idle until the next push
        cudaMemGetInfo(&fr, &tot);
      }
      if (bytes > h->pool_base.mapped && bytes - h->pool_base.mapped > (size_t)(0.9 * (double)fr)) split_fits = false;
      if (getenv("AGGB_TRACE"))
        fprintf(stderr, "[aggb] split level: %llu pages (%.1f GB), mapped %.1f GB, free %.1f GB -> %s\n",
                (unsigned long long)pages, bytes / 1e9, h->pool_base.mapped / 1e9, fr / 1e9,
                split_fits ? "split" : "sub-passes");
    }
    if (nsub >= 3 && nsets == 1 && split_fits && !getenv("AGGB_NO_SPLIT_LEVEL")) {
      const int S = std::min(nsub, 1024);
      int64_t total_in = 0;
      for (int p = 0; p < nparts; p++) total_in += (int64_t)recs[p];
      SetInfo sp{make_set(h, nonempty * S, a.ss.rw - h->kw, a.ss.kind, level_seed(h->cfg.seed, SALT_SPILL, depth + 17)),
                 0};
      TRY(pool_ensure(h, (uint64_t)(total_in / std::max(1, sp.ss.per_page)) + (uint64_t)nonempty * S + 16));
      CU(cudaMemsetAsync(SC(h) + 12, 0, 8, h->st));
      SplitArgs sa;
      memset(&sa, 0, sizeof(sa));
      sa.pool = pool_of(h);
      sa.in = a.ss;
      sa.plist = h->plist.as<uint2>();
      sa.item_off = h->item_off.as<int64_t>();
      sa.nitems = nonempty;
      sa.S = S;
      sa.sub_seed = level_seed(h->cfg.seed, SALT_SUB, depth + 1);
      sa.out = sp.ss;
      sa.item_counter = SC(h) + 12;
      int pe = prof_begin(h, 14);
      void (*sf)(SplitArgs) = h->kw == 1 ? k_split<1, 0> : k_split<2, 0>;
      const int rwi = a.ss.rw;
      if (h->kw == 1 && rwi == 2) sf = k_split<1, 2>;
      if (h->kw == 1 && rwi == 3) sf = k_split<1, 3>;
      if (h->kw == 1 && rwi == 5) sf = k_split<1, 5>;
      if (h->kw == 2 && rwi == 6) sf = k_split<2, 6>;
      if (h->kw == 2 && rwi == 15) sf = k_split<2, 15>;
      sf<<<h->sms * 4, 512, 0, h->st>>>(sa);
      prof_end(h, pe);
      h->launches++;
      CU(cudaGetLastError());
      h->met.grace_levels++;
      h->met.spilled_partitions -= nonempty;  // the sub-partitions are counted next
      tr.mark(h->st, "drain: split level");
      a = sp;
      a_live = true;
      b_live = false;
      nsub = 1;
      split_done = true;
      continue;
    }
    // child pass: output room + overflow room
    max_items_out = (int64_t)nonempty * nsub * (h->child_cap + 1);
    TRY(ensure_out(h, (int64_t)cnt_now + max_items_out + 16));
    int64_t total_recs = 0;
    for (int p = 0; p < nparts; p++) total_recs += (int64_t)recs[p];
    int ovw = h->kw + h->cs.ds.ns;
    // the overflow list holds every record in the worst case, or what half of
    // the free memory holds when that is less (C5 hash_sort at 500M records:
    // 59 GB worst case, ~0 in fact); a longer list fails loudly below
    int64_t ovf_want = total_recs + 16;
    if (ovf_want > h->ovf_cap) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      const int64_t fit = (int64_t)(0.5 * (double)(fr + h->ovf.bytes) / (ovw * 8 * 1.25));
      ovf_want = std::max<int64_t>(std::min<int64_t>(ovf_want, fit), std::min<int64_t>(ovf_want, 1 << 20));
    }
    if (ovf_want > h->ovf_cap) {
      if ((size_t)ovf_want * ovw * 8 > h->ovf.bytes) h->ovf.release();  // no copy needed: reallocate
      h->ovf_cap = 0;
      TRY(h->ovf.ensure((size_t)ovf_want * ovw * 8, &h->hw));
      h->ovf_cap = (int64_t)(h->ovf.bytes / ((size_t)ovw * 8));  // the buffer's headroom counts
    }
    CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
    CU(cudaMemsetAsync(SC(h) + 12, 0, 8, h->st));
    int payload = std::max(a.ss.rw, b_live ? b.ss.rw : 0) - h->kw;
    int nwt = nwt_for(std::max(1, payload));
    child_fn fn = h->kw == 1 ? child_kernel<1>(nwt, h->prog) : child_kernel<2>(nwt, h->prog);
    size_t smem = ((size_t)(1 << h->child_slots_log2) + 1) * (h->kw + h->cs.ds.ns) * 8;
    CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int grid = std::min(grid_for((const void*)fn, smem, h->sms), nonempty);
    ChildArgs ca;
    memset(&ca, 0, sizeof(ca));
    ca.sp = h->cs.ds;
    ca.pool = pp;
    ca.sets[0] = a.ss;
    ca.sets[1] = b_live ? b.ss : a.ss;
    ca.plist = h->plist.as<uint2>();
    ca.item_off = h->item_off.as<int64_t>();
    ca.nitems = nonempty;
    ca.slots_log2 = h->child_slots_log2;
    ca.cap = h->child_cap;
    ca.seed = level_seed(h->cfg.seed, SALT_SLOT, depth + 1);
    ca.nsub = nsub;
    ca.sub_seed = level_seed(h->cfg.seed, SALT_SUB, depth + 1);
    h->met.child_subpasses = std::max<int64_t>(h->met.child_subpasses, nsub);
    ca.out = outbuf(h, h->cfg.emit_partials ? 1 : 0);
    ca.ovf = h->ovf.as<uint64_t>();
    ca.ovf_stride = h->ovf_cap;
    ca.ovf_count = SC(h) + 11;
    ca.item_counter = SC(h) + 12;
    ca.stats = SC(h);
    tr.mark(h->st, "drain: scatter + buffers");
    int pe = prof_begin(h, 4);
    fn<<<grid, BLOCK, smem, h->st>>>(ca);
    prof_end(h, pe);
    h->launches++;
    CU(cudaGetLastError());
    // one round trip: the overflow count, and (if this was the last level) the
    // counters aggb_finish reads next
    TRY(h->hpin.ensure(sizeof(h->tail_sc) + 8));
    CU(cudaMemcpyAsync(h->hpin.p, SC(h), sizeof(h->tail_sc), cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(h->hpin.as<uint8_t>() + sizeof(h->tail_sc), h->pool_ctr.as<uint32_t>() + 1, 4,
                       cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    memcpy(h->tail_sc, h->hpin.p, sizeof(h->tail_sc));
    memcpy(&h->tail_ovfl, h->hpin.as<uint8_t>() + sizeof(h->tail_sc), 4);
    const unsigned long long novf = h->tail_sc[11];
    tr.mark(h->st, "drain: child");
    if (novf > (unsigned long long)h->ovf_cap)
      return fail(AGGB_CAPACITY_EXCEEDED, "child overflow of %llu records exceeds its %lld-record list", novf,
                  (long long)h->ovf_cap);
    if (!novf) {
      h->tail_valid = true;
      return AGGB_OK;
    }
    // next level: grace-partition the overflow with fresh seeds (fresh per level, hybrid.py:181-184).
    // Every page of this level has been consumed by the children, so the pool
    // is recycled: the next level writes its pages from page 0 again.
    CU(cudaMemsetAsync(h->pool_ctr.p, 0, 8, h->st));
    h->pool_bound = 0;
    depth++;
    // novf records bound the groups from above; beyond one pass's fan-out the
    // children take sub-passes (at most 4: the bound is loose)
    const int64_t need = std::max<int64_t>(2, (int64_t)std::ceil(novf / std::max(1.0, 0.5 * h->child_cap)));
    const int pmax = max_parts_for(h->kw + h->cs.ds.ns);
    int P = (int)std::min<int64_t>(pmax, need);
    nsub = (int)std::min<int64_t>(4, (need + pmax - 1) / pmax);
    SetInfo nxt{make_set(h, P, h->cs.ds.ns, 1, level_seed(h->cfg.seed, SALT_SPILL, depth)), 0};
    // move the overflow list into a staging copy (ovf is reused by the next child pass)
    DBuf tmp;
    TRY(tmp.ensure((size_t)novf * ovw * 8, nullptr));
    for (int w = 0; w < ovw; w++)
      CU(cudaMemcpyAsync(tmp.as<uint64_t>() + w * novf, h->ovf.as<uint64_t>() + w * h->ovf_cap, novf * 8,
                         cudaMemcpyDeviceToDevice, h->st));
    CU(cudaMemcpyAsync(SC(h) + 11, &novf, 8, cudaMemcpyHostToDevice, h->st));
    PassPlan g;
    g.mode = MODE_GRACE;
    g.lin = tmp.as<uint64_t>();
    g.lin_stride = (int64_t)novf;
    g.lin_count = SC(h) + 11;
    g.lin_kind = 1;
    g.lin_words = h->cs.ds.ns;
    g.ss = nxt.ss;
    g.counter = SC(h) + 9;
    TRY(launch_pass(h, g));
    CU(cudaStreamSynchronize(h->st));
    tmp.release();
    a = nxt;
    a_live = true;
    b_live = false;
  }
  return fail(AGGB_CAPACITY_EXCEEDED, "recursion did not converge");
}

int aggb_sort_push(Handle* h, const ColSrc& col);
int aggb_sort_finish(Handle* h);

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

const char* aggb_last_error(void) { return g_err.c_str(); }

const char* aggb_version(void) { return "aggb200 0.1 sm_100a"; }

int aggb_create(int device, const aggb_config* cfg, const aggb_spec* spec, void* stream, void** handle) {
  if (!cfg || !spec || !handle) return fail(AGGB_INVALID_ARG, "null argument");
  *handle = nullptr;
  Handle* h = new Handle();
  h->device = device;
  h->cfg = *cfg;
  h->spec = *spec;
  int s = compile_spec(*spec, h->cs);
  if (s) {
    delete h;
    return s;
  }
  h->kw = h->cs.kw;
  h->prog = detect_prog(h->cs.ds, h->kw);
  if (getenv("AGGB_NO_SPECIALIZE")) h->prog = 0;
  // dynamic_destaging and shared_hash share push_dd (MODE_DD passes); they differ
  // in what an overflow destages (dd_evict)
  s = plan(h);
  if (s) {
    delete h;
    return s;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete h;
    return fail(AGGB_CUDA_ERROR, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
  if (stream) {
    h->st = (cudaStream_t)stream;
  } else {
    e = cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete h;
      return fail(AGGB_CUDA_ERROR, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    h->own_stream = true;
  }
  if ((s = h->scratch.ensure(64 * 8, &h->hw)) || (s = h->pool_ctr.ensure(64, &h->hw))) {
    aggb_destroy(h);
    return s;
  }
  if (h->cfg.algo != AGGB_SORT_BASED) {
    if ((s = setup_table(h))) {
      aggb_destroy(h);
      return s;
    }
  }
  if ((s = begin_run(h))) {
    aggb_destroy(h);
    return s;
  }
  *handle = h;
  return AGGB_OK;
}

int aggb_reset(void* handle) {
  Handle* h = (Handle*)handle;
  if (!h) return fail(AGGB_INVALID_ARG, "null handle");
  prof_collect(h);
  return begin_run(h);
}

int aggb_profile(void* handle, int enable) {
  Handle* h = (Handle*)handle;
  if (!h) return fail(AGGB_INVALID_ARG, "null handle");
  prof_collect(h);
  h->prof = enable != 0;
  for (int i = 0; i < 24; i++) {
    h->kms[i] = 0;
    h->kcount[i] = 0;
  }
  return AGGB_OK;
}

int aggb_kernel_stats(void* handle, int i, const char** name, int64_t* launches, double* total_ms) {
  Handle* h = (Handle*)handle;
  if (!h) return fail(AGGB_INVALID_ARG, "null handle");
  if (i < 0 || i >= NKINDS) return fail(AGGB_INVALID_ARG, "kernel index out of range");
  prof_collect(h);
  if (name) *name = KNAMES[i];
  if (launches) *launches = h->kcount[i];
  if (total_ms) *total_ms = h->kms[i];
  return AGGB_OK;
}

void aggb_destroy(void* handle) {
  Handle* h = (Handle*)handle;
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->cst) cudaStreamSynchronize(h->cst);
  DBuf* bufs[] = {&h->tkeys, &h->tstates, &h->thdr, &h->page_part, &h->page_fill, &h->page_set,
                  &h->pool_ctr, &h->defer, &h->scratch, &h->hscratch_dev, &h->out_keys, &h->out_vals,
                  &h->out_i32[0], &h->out_i32[1], &h->part_records, &h->part_pages, &h->cursor, &h->plist,
                  &h->item_off, &h->ovf, &h->pend, &h->l2stage, &h->cut_tmp, &h->bloom, &h->sort_keys, &h->sort_vals,
                  &h->hot, &h->sort_hist, &h->dd_spilled, &h->dd_tmp, &h->cand, &h->chains,
                  &h->cut_bar, &h->wc_ovf, &h->wc_plist, &h->wc_meta, &h->wc_olist,
                  &h->wc_olist_n, &h->wc_gather, &h->partials_soa};
  for (DBuf* b : bufs) b->release();
  h->pool_base.release();
  h->stage.release();
  h->pstage[0].release();
  h->pstage[1].release();
  for (auto& e : h->evs) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : h->free_events) cudaEventDestroy(e);
  if (h->own_stream && h->st) cudaStreamDestroy(h->st);
  if (h->cst) {
    cudaStreamDestroy(h->cst);
    for (int b = 0; b < 2; b++) {
      cudaEventDestroy(h->ev_copied[b]);
      cudaEventDestroy(h->ev_used[b]);
    }
  }
  if (h->ev_staged) cudaEventDestroy(h->ev_staged);
  delete h;
}


// ---------------------------------------------------------------------------
// dynamic destaging (hybrid.py:974-1149, DynamicDestaging): every partition
// aggregates in the shared table until it runs dry; then the largest resident
// partitions are destaged — their groups cut to a partial run (part0) and their
// later records spilled raw (raw0) — and the pass resumes.  The partitions are
// the spill sets' fine partitions (children fit them); one destaging round
// evicts largest-first until 1/dd_rounds() of the table is free, the share one of
// the reference's coarse partitions holds.
// ---------------------------------------------------------------------------
int dd_rounds() {  // share of the table one destaging round frees: 1/DD_ROUNDS
  const char* e = getenv("AGGB_DD_ROUNDS");
  return e ? std::max(1, atoi(e)) : 4;  // C2 100M: 16 -> 34.5 ms, 8 -> 22.0, 4 -> 15.7 (same spill), 2 -> 13.5 (+5% spill)
}

int dd_evict(Handle* h) {
  const int P = h->part0.ss.nparts;
  const int words = h->kw + h->cs.ds.ns;
  const int64_t n = (int64_t)h->tab.cap + 2;
  TRY(h->dd_tmp.ensure((size_t)3 * n * words * 8 + 64 + (size_t)P * 8, &h->hw));
  uint64_t* all = h->dd_tmp.as<uint64_t>();
  uint64_t* ev = all + (size_t)n * words;
  uint64_t* kept = ev + (size_t)n * words;
  unsigned long long* hist = (unsigned long long*)(kept + (size_t)n * words);
  unsigned long long* cnts = SC(h) + 40;  // [40] all, [41] evicted, [42] kept
  OutBuf o;
  o.keys = all;
  o.vals = all + (size_t)h->kw * n;
  o.cap = n;
  o.count = cnts;
  o.partial = 1;
  CU(cudaMemsetAsync(cnts, 0, 24, h->st));
  CU(cudaMemsetAsync(hist, 0, (size_t)P * 8, h->st));
  TRY(flush_table(h, true, &o));
  const uint64_t seed = h->part0.ss.seed;
  const int grid = h->sms * 4;
  if (h->kw == 1) k_dd_hist<1><<<grid, 256, 0, h->st>>>(all, n, cnts, seed, P, hist);
  else k_dd_hist<2><<<grid, 256, 0, h->st>>>(all, n, cnts, seed, P, hist);
  std::vector<unsigned long long> hh(P);
  unsigned long long total = 0;
  CU(cudaMemcpyAsync(hh.data(), hist, (size_t)P * 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaMemcpyAsync(&total, cnts, 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  // largest resident partitions first, until a round's share of the table is free
  std::vector<int> order;
  for (int p = 0; p < P; p++)
    if (!h->dd_host[p] && hh[p]) order.push_back(p);
  std::sort(order.begin(), order.end(), [&](int x, int y) { return hh[x] > hh[y] || (hh[x] == hh[y] && x < y); });
  std::vector<uint8_t> evict(P, 0);
  if (h->cfg.algo == AGGB_SHARED_HASH) {
    // shared_hash (hybrid.py:579-915): the first overflow cuts every partition but
    // partition 0 (the resident share r_res of the hash range, as original_hh
    // plans it) to runs; a second overflow cuts partition 0 too: pure routing
    const double G_t = std::max(1.0, h->cfg.stats_G_t);
    const double r_res = h->cfg.stats_G_t > 0 ? std::min(1.0, 0.9 * (double)h->budget / G_t) : 0.5;
    const int k0 = h->sh_stage == 0 ? std::max(1, std::min(P - 1, (int)std::lround(r_res * P))) : 0;
    for (int p = k0; p < P; p++)
      if (!h->dd_host[p]) {
        evict[p] = 1;
        h->dd_host[p] = 1;
        h->dd_evictions++;
      }
    h->sh_stage++;
  } else {
    const unsigned long long want = std::max<unsigned long long>(1, (unsigned long long)h->tab.cap / dd_rounds());
    unsigned long long freed = 0;
    for (int p : order) {
      if (freed >= want) break;
      evict[p] = 1;
      h->dd_host[p] = 1;
      freed += hh[p];
      h->dd_evictions++;
    }
  }
  if (order.empty()) {  // nothing resident left to destage: every later record spills raw
    for (int p = 0; p < P; p++) h->dd_host[p] = 1;
  }
  uint8_t* flags = h->dd_spilled.as<uint8_t>();
  CU(cudaMemcpyAsync(flags, h->dd_host.data(), (size_t)P, cudaMemcpyHostToDevice, h->st));
  // split the flushed groups: evicted -> the partial set, kept -> back into the table
  if (h->kw == 1) k_dd_split<1><<<grid, 256, 0, h->st>>>(all, n, cnts, words, seed, P, flags, ev, kept, cnts + 1);
  else k_dd_split<2><<<grid, 256, 0, h->st>>>(all, n, cnts, words, seed, P, flags, ev, kept, cnts + 1);
  h->launches += 3;
  CU(cudaGetLastError());
  PassPlan g;
  g.mode = MODE_GRACE;
  g.lin = ev;
  g.lin_stride = n;
  g.lin_count = cnts + 1;
  g.lin_kind = 1;
  g.lin_words = h->cs.ds.ns;
  g.ss = h->part0.ss;
  g.counter = SC(h) + 9;
  TRY(launch_pass(h, g));
  h->part0_live = true;
  TRY(table_reset(h));
  PassPlan f;  // the kept groups: merge ops into the fresh table (they fit: fewer than before)
  f.mode = MODE_FILL;
  f.lin = kept;
  f.lin_stride = n;
  f.lin_count = cnts + 2;
  f.lin_kind = 1;
  f.lin_words = h->cs.ds.ns;
  f.counter = SC(h) + 8;
  CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
  TRY(launch_pass(h, f));
  return AGGB_OK;
}

int push_dd(Handle* h, const ColSrc& col0) {
  const int nwt = nwt_for(std::max(1, col0.nv));
  PassCfg pcfg = h->kw == 1 ? pass_kernel<1>(nwt, h->prog) : pass_kernel<2>(nwt, h->prog);
  const int64_t T = (int64_t)pcfg.R * pcfg.blk;
  TRY(ensure_defer(h, T, col0.nv));
  std::vector<ColSrc> queue{col0};
  std::vector<DBuf> temps;
  int rc = AGGB_OK;
  int guard = 0;
  while (!queue.empty() && rc == AGGB_OK) {
    ColSrc cur = queue.back();
    queue.pop_back();
    if (cur.n <= 0) continue;
    CU(cudaMemsetAsync(SC(h) + 10, 0, 8, h->st));
    PassPlan f;
    f.mode = MODE_DD;
    f.col = cur;
    f.ss = h->raw0.ss;
    f.counter = SC(h) + 8;
    if ((rc = launch_pass(h, f))) break;
    h->raw0_live = true;
    unsigned long long tiles = 0, nd = 0;
    int frozen = 0;
    CU(cudaMemcpyAsync(&tiles, SC(h) + 8, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(&nd, SC(h) + 10, 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(&frozen, &h->tab.hdr->frozen, 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (!frozen && !nd) continue;
    if (++guard > h->part0.ss.nparts + 64) {  // every round destages at least one partition
      rc = fail(AGGB_CAPACITY_EXCEEDED, "dynamic destaging made no progress");
      break;
    }
    const int64_t start = std::min<int64_t>(cur.n, (int64_t)tiles * T);
    ColSrc dc;
    memset(&dc, 0, sizeof(dc));
    if (nd) {  // keep the refused records (the deferral buffer is reused)
      DBuf tmp;
      const int words = h->kw + cur.nv;
      if ((rc = tmp.ensure((size_t)nd * words * 8, nullptr))) break;
      for (int w = 0; w < words; w++)
        CU(cudaMemcpyAsync(tmp.as<uint64_t>() + w * nd, h->defer.as<uint64_t>() + w * h->defer_cap, nd * 8,
                           cudaMemcpyDeviceToDevice, h->st));
      dc.n = (int64_t)nd;
      for (int w = 0; w < h->kw; w++) {
        dc.key[w] = (const uint8_t*)(tmp.as<uint64_t>() + w * nd);
        dc.kstride[w] = 8;
        dc.kty[w] = TY_I64;
      }
      dc.nv = cur.nv;
      for (int w = 0; w < cur.nv; w++) {
        dc.val[w] = (const uint8_t*)(tmp.as<uint64_t>() + (h->kw + w) * nd);
        dc.vstride[w] = 8;
        dc.vty[w] = (h->cs.ds.vty[w] == TY_F64) ? TY_F64 : TY_I64;
      }
      temps.push_back(tmp);
    }
    if ((rc = dd_evict(h))) break;  // the pool ran dry: destage the largest partitions
    if (start < cur.n) {
      ColSrc rest = cur;
      rest.n = cur.n - start;
      for (int w = 0; w < h->kw; w++) rest.key[w] = cur.key[w] + start * cur.kstride[w];
      for (int w = 0; w < cur.nv; w++) rest.val[w] = cur.val[w] + start * cur.vstride[w];
      queue.push_back(rest);
    }
    if (nd) queue.push_back(dc);  // refused records first
  }
  cudaStreamSynchronize(h->st);
  for (auto& t : temps) t.release();
  h->met.spilled_partitions = 0;
  for (uint8_t x : h->dd_host) h->met.spilled_partitions += x;
  return rc;
}

// Heavy hitters of this push (pass.cuh k_hot_sample): in-memory and L2-capped
// plans of one-word keys with the COUNT/SUM programs (C1, C3, C4).  Budgeted
// plans keep the reference's arrival-order residency untouched (the tier only
// takes keys already resolved resident, but its sample is not needed there).
int hot_sample(Handle* h, const ColSrc& col) {
  h->hot_ready = false;
  const bool eligible = h->kw == 1 && col.nv == 1 && (h->prog == 1 || h->prog == 3) &&
                        (h->unlimited || h->l2_capped) && (h->cfg.algo == AGGB_PRE_PARTITIONING ||
                                                           h->cfg.algo == AGGB_HASH_SORT) &&
                        col.n >= (1 << 16) && !getenv("AGGB_NO_HOT");
  if (!eligible) return AGGB_OK;
  TRY(h->hot.ensure((HOT_MAX + 2) * 8, &h->hw));
  const int64_t sample = std::min<int64_t>(col.n, 1 << 17);
  const uint32_t min_count = (uint32_t)std::max<int64_t>(8, sample / 256);  // >= 0.4% of the records
  k_hot_sample<<<1, 1024, 0, h->st>>>(col, col.n, sample, min_count, h->hot.as<uint64_t>());
  h->launches++;
  CU(cudaGetLastError());
  uint64_t nh[2] = {0, 0};  // no heavy hitters (uniform keys): the plain pass, no tier cost
  CU(cudaMemcpyAsync(nh, h->hot.as<uint64_t>() + HOT_MAX, 16, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  h->hot_ready = nh[0] > 0;
  // When the hot keys carry most of the records (Zipf s = 1.5: ~74%), the keys
  // just below them are still hot enough to serialise the SMEM tier's CAS loops
  // (f64 ADD), while L2 REDs do not stall the issuing warp: the pass runs
  // without the SMEM tier (C3 s = 1.5 FILL 14.0 -> 5.2 ms; at s = 1.0, 16%
  // covered, the tier stays: 9.06 vs 9.63 ms without it).
  h->hot_no_tier = h->hot_ready && nh[1] * 10 >= (uint64_t)sample * 4;
  if (h->skew_cap && h->first_push) {  // the table was sized for skew_cap; grant it to skewed runs
    h->tab.cap = h->hot_no_tier ? (uint64_t)h->skew_cap : (uint64_t)h->budget;
  }
  if (h->aos_planned && h->first_push && h->hot_no_tier) {
    // heavily skewed: the warm keys' REDs to one sector per slot serialise in L2
    // (C3 s = 1.5 hash_sort FILL 7.40 ms field-major vs 8.05 slot-major); the
    // table is still empty: switch it to field-major
    h->tab.fstride = h->tab.stride;
    h->tab.sstride = 1;
    TRY(table_reset(h));
  }
  h->first_push = false;
  return AGGB_OK;
}

int push_col(Handle* h, const ColSrc& col) {
  if (h->cfg.algo == AGGB_SORT_BASED) return aggb_sort_push(h, col);
  if (h->cfg.algo == AGGB_DYNAMIC_DESTAGING || h->cfg.algo == AGGB_SHARED_HASH) return push_dd(h, col);
  TRY(hot_sample(h, col));
  if (h->cfg.algo == AGGB_HASH_SORT) return push_hash_sort(h, col);
  return push_hybrid(h, col);
}

// Host input larger than two chunks: chunk c+2's host-to-device copy (copy
// stream) overlaps chunk c's aggregation; two staging buffers alternate, each
// refilled only after the aggregation that read it.  Each chunk is a push of
// its own (the operators accept any number of pushes).
int64_t pipe_chunk() {
  const char* e = getenv("AGGB_PIPE_CHUNK");  // tests exercise the pipeline on small inputs
  return e ? std::max<int64_t>(1, atoll(e)) : 25000000;
}

int push_pipelined(Handle* h, const aggb_input* in) {
  const int64_t PIPE_CHUNK = pipe_chunk();
  if (!h->cst) {
    CU(cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
      CU(cudaEventCreateWithFlags(&h->ev_copied[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&h->ev_used[b], cudaEventDisableTiming));
    }
  }
  const int nk = h->kw, nv = h->spec.n_vals;
  auto esz = [&](bool key, int w) { return (key ? h->spec.key_type[w] : h->spec.val_type[w]) == AGGB_I32 ? 4 : 8; };
  auto strd = [&](bool key, int w) {
    const int64_t st = key ? in->key_stride[w] : in->val_stride[w];
    return st ? st : (int64_t)esz(key, w);
  };
  auto span = [&](bool key, int w, int64_t rows) { return (size_t)((rows - 1) * strd(key, w) + esz(key, w)); };
  size_t per = 0;
  for (int w = 0; w < nk; w++) per += (span(true, w, PIPE_CHUNK) + 255) & ~(size_t)255;
  for (int w = 0; w < nv; w++) per += (span(false, w, PIPE_CHUNK) + 255) & ~(size_t)255;
  for (int b = 0; b < 2; b++) TRY(h->pstage[b].ensure(per, &h->hw));
  const int64_t n = in->n_rows, nch = (n + PIPE_CHUNK - 1) / PIPE_CHUNK;
  std::vector<std::vector<const uint8_t*>> ptrs(nch);
  auto copy = [&](int64_t c) -> int {
    const int b = (int)(c & 1);
    const int64_t r0 = c * PIPE_CHUNK, rows = std::min<int64_t>(PIPE_CHUNK, n - r0);
    if (h->pstage_busy[b]) CU(cudaStreamWaitEvent(h->cst, h->ev_used[b], 0));  // also across pushes
    size_t off = 0;
    ptrs[c].clear();
    for (int q = 0; q < nk + nv; q++) {
      const bool key = q < nk;
      const int w = key ? q : q - nk;
      const uint8_t* src = (const uint8_t*)(key ? in->key[w] : in->val[w]) + r0 * strd(key, w);
      uint8_t* dst = h->pstage[b].as<uint8_t>() + off;
      CU(cudaMemcpyAsync(dst, src, span(key, w, rows), cudaMemcpyHostToDevice, h->cst));
      ptrs[c].push_back(dst);
      off += (span(key, w, PIPE_CHUNK) + 255) & ~(size_t)255;
    }
    CU(cudaEventRecord(h->ev_copied[b], h->cst));
    return AGGB_OK;
  };
  TRY(copy(0));
  if (nch > 1) TRY(copy(1));
  for (int64_t c = 0; c < nch; c++) {
    const int b = (int)(c & 1);
    const int64_t rows = std::min<int64_t>(PIPE_CHUNK, n - c * PIPE_CHUNK);
    CU(cudaStreamWaitEvent(h->st, h->ev_copied[b], 0));
    aggb_input part = *in;
    part.n_rows = rows;
    part.on_host = 0;
    const void* kp[AGGB_MAX_KEYS];
    const void* vp[AGGB_MAX_VALS];
    for (int w = 0; w < nk; w++) kp[w] = ptrs[c][w];
    for (int w = 0; w < nv; w++) vp[w] = ptrs[c][nk + w];
    ColSrc col = col_of(h, &part, kp, vp);
    h->records += rows;
    TRY(push_col(h, col));
    CU(cudaEventRecord(h->ev_used[b], h->st));
    h->pstage_busy[b] = true;
    if (c + 2 < nch) TRY(copy(c + 2));
  }
  // the caller may reuse its host buffers once push returns: wait for the last
  // copy out of them (in order on the copy stream), not for the aggregation
  CU(cudaEventSynchronize(h->ev_copied[(int)((nch - 1) & 1)]));
  return AGGB_OK;
}

int aggb_push(void* handle, const aggb_input* in) {
  Handle* h = (Handle*)handle;
  if (!h || !in) return fail(AGGB_INVALID_ARG, "null argument");
  if (h->finished) return fail(AGGB_INVALID_ARG, "push after finish; call aggb_reset");
  if (in->n_rows < 0) return fail(AGGB_INVALID_ARG, "negative row count");
  if (in->n_rows == 0) return AGGB_OK;
  cudaSetDevice(h->device);
  if (in->on_host && in->n_rows > 2 * pipe_chunk() && !getenv("AGGB_NO_PIPELINE")) {
    Trace tr;
    const int s = push_pipelined(h, in);
    tr.mark(h->st, "push (pipelined)");
    return s;
  }
  Staged sg;
  TRY(stage_input(h, in, sg));
  if (in->on_host) {  // the copies out of the caller's memory (waited for before returning)
    if (!h->ev_staged) CU(cudaEventCreateWithFlags(&h->ev_staged, cudaEventDisableTiming));
    CU(cudaEventRecord(h->ev_staged, h->st));
  }
  ColSrc col = col_of(h, in, sg.k, sg.v);
  h->records += in->n_rows;
  int s;
  Trace tr;
  s = push_col(h, col);
  tr.mark(h->st, "push");
  if (!sg.owned.empty()) {
    cudaStreamSynchronize(h->st);
    for (auto& b : sg.owned) b.release();
  }
  if (in->on_host) CU(cudaEventSynchronize(h->ev_staged));  // host buffers reusable on return
  return s;
}

int aggb_push_partials(void* handle, const void* recv, int64_t n_records) {
  Handle* h = (Handle*)handle;
  if (!h) return fail(AGGB_INVALID_ARG, "null handle");
  if (h->finished) return fail(AGGB_INVALID_ARG, "push after finish; call aggb_reset");
  if (n_records <= 0) return AGGB_OK;
  if (h->cfg.algo == AGGB_SORT_BASED) return fail(AGGB_SPEC_ERROR, "partials merge through a hash algorithm");
  cudaSetDevice(h->device);
  // partial records (AoS: kw key words then ns state words) are transposed to
  // the list layout and partitioned into the partial spill set; the children
  // of aggb_finish merge them (merge ops only, like the reference's runs).
  // The list buffer belongs to the handle (grow-only, stream-ordered reuse): no
  // allocation and no synchronization per call.
  int rw = h->kw + h->cs.ds.ns;
  DBuf& soa = h->partials_soa;
  TRY(soa.ensure((size_t)n_records * rw * 8, &h->hw));
  k_aos_to_soa<<<h->sms * 8, 256, 0, h->st>>>((const uint64_t*)recv, n_records, rw, soa.as<uint64_t>());
  h->launches++;
  k_set_u64<<<1, 1, 0, h->st>>>(SC(h) + 11, (unsigned long long)n_records);  // (by value: no host buffer to keep alive)
  h->launches++;
  PassPlan g;
  g.mode = MODE_GRACE;
  g.lin = soa.as<uint64_t>();
  g.lin_stride = n_records;
  g.lin_count = SC(h) + 11;
  g.lin_kind = 1;
  g.lin_words = h->cs.ds.ns;
  g.ss = h->part0.ss;
  g.counter = SC(h) + 9;
  TRY(launch_pass(h, g));
  h->part0_live = true;
  h->records += n_records;
  return AGGB_OK;
}

// the children of the write-combined level 0 (k_child2_wc): one CTA per run,
// whole waves; owner runs are seeded from the owners' lists of resident slots
int wc_children(Handle* h) {
  TRY(wc_build(h));
  Cw2Args ca;
  memset(&ca, 0, sizeof(ca));
  ca.sp = h->cs.ds;
  ca.pool = pool_of(h);
  ca.plist = h->wc_plist.as<uint32_t>();
  ca.plist_n = wc_pn(h);
  ca.plist_cap = h->wc_plist_cap;
  ca.ovf = h->wc_ovf.as<unsigned long long>() + 1;
  ca.ovf_n = h->wc_ovf.as<unsigned long long>();
  ca.ovf_cap = h->wc_ovf_cap;
  ca.part_recs = wc_recs(h);
  ca.vinfo = wc_vinfo(h);
  ca.NP = h->P0;
  ca.table_bytes = h->wc_table_bytes;
  if (getenv("AGGB_WC_CHILD_KB"))  // test hook: small child tables send runs to the fallback
    ca.table_bytes = std::max(1, std::min(h->wc_table_bytes / 1024, atoi(getenv("AGGB_WC_CHILD_KB")))) * 1024;
  ca.seed = level_seed(h->cfg.seed, SALT_SLOT, h->cfg.level + 1);
  ca.out = outbuf(h, h->cfg.emit_partials ? 1 : 0);
  ca.failed = wc_failed(h);
  ca.fail = wc_fail(h);
  ca.stats = SC(h);
  ca.t = h->tab;
  ca.olist = h->wc_olist.as<uint32_t>();
  ca.olist_n = h->wc_olist_n.as<uint32_t>();
  ca.ocap = h->wc_ocap;
  auto fc = h->prog == 2 ? k_child2_wc<CpC2, WC_CBLK, WC_CRL> : k_child2_wc<CpC1, WC_CBLK, WC_CRL>;
  if (!h->wc_child_attr) {
    CU(cudaFuncSetAttribute((const void*)fc, cudaFuncAttributeMaxDynamicSharedMemorySize, h->wc_table_bytes));
    h->wc_child_attr = true;
  }
  int pe = prof_begin(h, 17);
  fc<<<std::min(h->sms, ca.NP), WC_CBLK, h->wc_table_bytes, h->st>>>(ca);
  prof_end(h, pe);
  CU(cudaGetLastError());
  h->launches++;
  return AGGB_OK;
}

__global__ void k_stat_sub(unsigned long long* stats, unsigned long long n) {
  stats[ST_SPILLED] -= n;
  stats[ST_RECORDS] -= n;
}

// Runs k_child2_wc could not hold (more groups than its table, rows past the
// output estimate, an overflowed page list, values beyond int32).  A run holds
// records of resident keys, so it cannot go to the generic recursion as it is:
// it is gathered into dense columns and probed against the frozen table by the
// generic PROBE (hits aggregate in place, the rest spills into the generic
// partitions), the table is flushed again over its first flush, every run's
// pages are retired and the generic recursion takes the new spill.
int wc_fallback(Handle* h) {
  const int NP = h->P0;
  std::vector<uint32_t> failed((size_t)NP), pn((size_t)NP);
  std::vector<unsigned long long> recs((size_t)NP);
  CU(cudaMemcpyAsync(failed.data(), wc_failed(h), (size_t)NP * 4, cudaMemcpyDeviceToHost, h->st));
  CU(cudaMemcpyAsync(pn.data(), wc_pn(h), (size_t)NP * 4, cudaMemcpyDeviceToHost, h->st));
  CU(cudaMemcpyAsync(recs.data(), wc_recs(h), (size_t)NP * 8, cudaMemcpyDeviceToHost, h->st));
  unsigned long long novf = 0;
  CU(cudaMemcpyAsync(&novf, h->wc_ovf.p, 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  if (novf > h->wc_ovf_cap) return fail(AGGB_CAPACITY_EXCEEDED, "overflow page list overflowed (internal error)");
  // the table's rows are rewritten below: back to the row count before its flush
  CU(cudaMemcpyAsync(SC(h) + 13, SC(h) + 30, 8, cudaMemcpyDeviceToDevice, h->st));
  if (h->bloom_words) {
    CU(cudaMemsetAsync(h->bloom.p, 0, (size_t)h->bloom_words * 8, h->st));
    k_bloom_build<1><<<h->sms * 4, 256, 0, h->st>>>(h->tab, h->bloom.as<uint64_t>(), (uint32_t)h->bloom_words - 1);
    h->launches++;
  }
  int64_t nmax = 0;
  for (int p = 0; p < NP; p++)
    if (failed[(size_t)p]) nmax = std::max<int64_t>(nmax, (int64_t)recs[(size_t)p]);
  TRY(h->wc_gather.ensure((size_t)std::max<int64_t>(nmax, 1) * 16, &h->hw));
  for (int p = 0; p < NP; p++) {
    if (!failed[(size_t)p]) continue;
    const int64_t n = (int64_t)recs[(size_t)p];
    if (n == 0) continue;
    unsigned long long* gk = h->wc_gather.as<unsigned long long>();
    unsigned long long* gv = gk + nmax;
    CU(cudaMemsetAsync(SC(h) + 31, 0, 8, h->st));
    const uint32_t nown = std::min(pn[(size_t)p], h->wc_plist_cap);
    const uint32_t nov = pn[(size_t)p] > h->wc_plist_cap ? (uint32_t)novf : 0u;
    k_wc2_gather<<<std::max(1, std::min<int>((int)std::min<uint64_t>((uint64_t)nown + nov, 1u << 20), h->sms * 4)), 256, 0, h->st>>>(
        pool_of(h), h->wc_plist.as<uint32_t>() + (size_t)p * h->wc_plist_cap, nown, h->wc_ovf.as<unsigned long long>() + 1,
        nov, (uint32_t)p, gk, gv, SC(h) + 31);
    k_stat_sub<<<1, 1, 0, h->st>>>(SC(h), (unsigned long long)n);  // (the PROBE below counts them again)
    CU(cudaGetLastError());
    h->launches += 2;
    ColSrc col;
    memset(&col, 0, sizeof(col));
    col.n = n;
    col.key[0] = (const uint8_t*)gk;
    col.kstride[0] = 8;
    col.kty[0] = TY_I64;
    col.nv = 1;
    col.val[0] = (const uint8_t*)gv;
    col.vstride[0] = 8;
    col.vty[0] = TY_I64;
    PassPlan pr;
    pr.mode = MODE_PROBE;
    pr.col = col;
    pr.ss = h->raw0.ss;
    pr.counter = SC(h) + 9;
    TRY(launch_pass(h, pr));
  }
  OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
  TRY(flush_table(h, h->cfg.emit_partials != 0, &o));
  k_wc2_retire<<<std::max(1, std::min(NP, h->sms * 4)), 256, 0, h->st>>>(
      h->wc_plist.as<uint32_t>(), wc_pn(h), h->wc_plist_cap, NP, h->wc_ovf.as<unsigned long long>() + 1,
      h->wc_ovf.as<unsigned long long>(), h->wc_ovf_cap, h->page_set.as<int32_t>());
  CU(cudaGetLastError());
  h->launches++;
  h->tail_valid = false;
  return drain(h, h->raw0, true, h->part0, h->part0_live, h->cfg.level);
}

int aggb_finish(void* handle, aggb_result* out) {
  Handle* h = (Handle*)handle;
  if (!h || !out) return fail(AGGB_INVALID_ARG, "null argument");
  cudaSetDevice(h->device);
  Trace tr;
  h->tail_valid = false;
  if (!h->finished) {
    if (h->cfg.algo == AGGB_SORT_BASED) {
      TRY(aggb_sort_finish(h));
    } else {
      const int algo0 = h->cfg.algo;
      // No level-0 decision of these schedules depends on the device counters:
      // flush without a round trip (the table holds at most tab.cap groups + the
      // escape group, and nothing has been emitted yet); the two metrics the
      // close reports travel to scratch slots 14/15 and come back with the
      // tail's read (C2: one host round trip less per step)
      const bool no_rt = (algo0 == AGGB_PRE_PARTITIONING || algo0 == AGGB_SHARED_HASH ||
                          algo0 == AGGB_DYNAMIC_DESTAGING) && !getenv("AGGB_L0_ROUNDTRIP");
      if (no_rt) {
        // (k_child2_wc: rows for the expected groups; a run past them falls back to drain)
        const int64_t wc_rows =
            h->wc_used ? (int64_t)std::min<double>((double)h->records, std::max(2.0 * h->cfg.stats_G_t, 1.0e6)) : 0;
        TRY(ensure_out(h, (int64_t)h->tab.cap + 4 + wc_rows));
        if (h->wc_used) {
          // the children first: owner runs merge their resident groups into the
          // table (and take their records out of the spill count) before it is flushed
          TRY(wc_children(h));
          tr.mark(h->st, "finish: wc children");
          CU(cudaMemcpyAsync(SC(h) + 30, SC(h) + 13, 8, cudaMemcpyDeviceToDevice, h->st));  // rows before the flush
        }
        CU(cudaMemcpyAsync(SC(h) + 14, &h->tab.hdr->committed, 8, cudaMemcpyDeviceToDevice, h->st));
        CU(cudaMemcpyAsync(SC(h) + 15, SC(h) + ST_SPILLED, 8, cudaMemcpyDeviceToDevice, h->st));
        OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
        TRY(flush_table(h, h->cfg.emit_partials != 0, &o));
        tr.mark(h->st, "finish: level-0 flush");
        h->l0_deferred = true;
        if (!h->wc_used) TRY(drain(h, h->raw0, h->raw0_live, h->part0, h->part0_live, h->cfg.level));
      }
      int frozen = 0, refused = 0;
      unsigned long long groups = 0, cnt0 = 0, sp0 = 0;
      // one round trip for everything the level-0 close needs
      if (!no_rt) {
      CU(cudaMemcpyAsync(&frozen, &h->tab.hdr->frozen, 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(&refused, &h->tab.hdr->pad, 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(&groups, &h->tab.hdr->committed, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(&cnt0, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(&sp0, SC(h) + ST_SPILLED, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      if (h->cfg.algo == AGGB_ORIGINAL_HH && refused) frozen = 1;  // partition 0 spilled: cut the table
      h->met.resident_groups = (int64_t)groups;
      if (h->cfg.algo == AGGB_ORIGINAL_HH && frozen) {
        // overflow: cut the table into partition 0 as partial states (hybrid.py:431-451)
        unsigned long long cnt = 0;
        CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
        CU(cudaStreamSynchronize(h->st));
        int words = h->kw + h->cs.ds.ns;
        DBuf tmp;
        int64_t n = (int64_t)groups + 2;
        TRY(tmp.ensure((size_t)n * words * 8, nullptr));
        OutBuf o;
        o.keys = tmp.as<uint64_t>();
        o.vals = tmp.as<uint64_t>() + (size_t)h->kw * n;
        o.cap = n;
        o.count = SC(h) + 11;
        o.partial = 1;
        CU(cudaMemsetAsync(SC(h) + 11, 0, 8, h->st));
        TRY(flush_table(h, true, &o));
        PassPlan g;
        g.mode = MODE_GRACE;
        g.lin = tmp.as<uint64_t>();
        g.lin_stride = n;
        g.lin_count = SC(h) + 11;
        g.lin_kind = 1;
        g.lin_words = h->cs.ds.ns;
        // partition 0 of the raw set: all records to partition 0 of the partial set
        SpillSet s0 = h->part0.ss;
        s0.nparts = 1;
        g.ss = s0;
        g.counter = SC(h) + 9;
        TRY(launch_pass(h, g));
        CU(cudaStreamSynchronize(h->st));
        tmp.release();
        h->part0_live = true;
        h->part0.ss.nparts = h->raw0.ss.nparts;
      } else if (h->cfg.algo == AGGB_HASH_SORT && h->hash_sort_runs > 0) {
        TRY(cut_run(h));  // last run; the merge-with-fold is the drain below
      } else {
        // the table holds at most `groups` keys (+ the escape group): size the
        // output from the counts read above, flush without another round trip
        TRY(ensure_out(h, (int64_t)cnt0 + (int64_t)groups + 2));
        OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
        TRY(flush_table(h, h->cfg.emit_partials != 0, &o));
      }
      tr.mark(h->st, "finish: level-0 flush");
      h->met.level0_spilled_records = (int64_t)sp0;
      TRY(drain(h, h->raw0, h->raw0_live, h->part0, h->part0_live, h->cfg.level));
      }
    }
    unsigned long long cnt = 0, st[ST_NSTATS];
    uint32_t ovfl = 0;
    unsigned long long l0[2] = {0, 0};  // deferred level-0 metrics (scratch 14, 15)
    if (h->tail_valid) {  // read by drain right after the last child pass
      cnt = h->tail_sc[13];
      memcpy(st, h->tail_sc, sizeof(st));
      ovfl = h->tail_ovfl;
      l0[0] = h->tail_sc[14];
      l0[1] = h->tail_sc[15];
    } else {
      uint32_t wcf = 0;
      CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(st, SC(h), sizeof(st), cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(&ovfl, h->pool_ctr.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(l0, SC(h) + 14, 16, cudaMemcpyDeviceToHost, h->st));
      if (h->wc_used) CU(cudaMemcpyAsync(&wcf, wc_fail(h), 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      if (wcf & 2u) return fail(AGGB_CUDA_ERROR, "k_scan_wc: page map inconsistency (internal error)");
      if (h->wc_used) {
        h->met.recursion_depth = std::max<int64_t>(h->met.recursion_depth, st[ST_SPILLED] ? 1 : 0);
        h->met.spilled_partitions += st[ST_SPILLED] ? h->raw0.ss.nparts : 0;
      }
      if (wcf) {  // some run did not fit k_child2_wc: re-probed (owner runs) / left to the generic recursion
        TRY(wc_fallback(h));
        h->wc_fallbacks++;
        CU(cudaMemcpyAsync(&cnt, SC(h) + 13, 8, cudaMemcpyDeviceToHost, h->st));
        CU(cudaMemcpyAsync(st, SC(h), sizeof(st), cudaMemcpyDeviceToHost, h->st));
        CU(cudaMemcpyAsync(&ovfl, h->pool_ctr.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToHost, h->st));
        CU(cudaMemcpyAsync(l0 + 1, SC(h) + ST_SPILLED, 8, cudaMemcpyDeviceToHost, h->st));
        CU(cudaStreamSynchronize(h->st));
      }
    }
    if (h->l0_deferred) {
      h->met.resident_groups = (int64_t)l0[0];
      h->met.level0_spilled_records = (int64_t)l0[1];
      h->l0_deferred = false;
    }
    if (ovfl) return fail(AGGB_CAPACITY_EXCEEDED, "spill page pool overflowed");
    if ((int64_t)cnt > h->out_cap) return fail(AGGB_CAPACITY_EXCEEDED, "output buffer overflow (%llu > %lld)", cnt, (long long)h->out_cap);
    // typed key columns
    aggb_result& r = h->result;
    memset(&r, 0, sizeof(r));
    r.n_groups = (int64_t)cnt;
    for (int w = 0; w < h->kw; w++) {
      uint64_t* col = h->out_keys.as<uint64_t>() + (size_t)w * h->out_cap;
      if (h->spec.key_type[w] == AGGB_I32) {
        TRY(h->out_i32[w].ensure(std::max<size_t>(cnt, 1) * 4, &h->hw));
        if (cnt) {
          k_key_to_i32<<<h->sms * 4, 256, 0, h->st>>>(col, h->out_i32[w].as<int32_t>(), (int64_t)cnt);
          h->launches++;
        }
        r.key[w] = h->out_i32[w].p;
      } else {
        r.key[w] = col;
      }
    }
    int ncols = h->cfg.emit_partials ? h->cs.ds.ns : h->cs.ds.nout;
    for (int j = 0; j < ncols; j++) {
      r.out[j] = h->out_vals.as<uint64_t>() + (size_t)j * h->out_cap;
      r.out_type[j] = h->cfg.emit_partials ? (h->cs.ds.ty[j] == TY_F64 && h->cs.ds.op[j] == OP_ADD ? AGGB_F64 : AGGB_I64)
                                           : h->cs.out_type[j];
    }
    r.sorted = h->cfg.algo == AGGB_SORT_BASED ? 1 : 0;
    CU(cudaStreamSynchronize(h->st));
    h->met.records = h->records;
    h->met.output_groups = (int64_t)cnt;
    h->met.spilled_records = (int64_t)st[ST_SPILLED];
    h->met.spilled_bytes = (int64_t)st[ST_SPILLED] * 8 * (h->kw + h->cs.nv);
    h->met.budget_groups = h->budget;
    h->met.partitions_level0 = h->P0;
    h->finished = true;
    prof_collect(h);
    tr.mark(h->st, "finish: tail");
  }
  h->met.kernel_launches = h->launches;
  h->met.high_water_bytes = (int64_t)h->hw;
  *out = h->result;
  return AGGB_OK;
}

int aggb_copy_result(void* handle, void* const* host_keys, void* const* host_out) {
  Handle* h = (Handle*)handle;
  if (!h || !h->finished) return fail(AGGB_INVALID_ARG, "no finished result");
  int64_t n = h->result.n_groups;
  if (n == 0) return AGGB_OK;
  for (int w = 0; w < h->kw; w++)
    if (host_keys && host_keys[w])
      CU(cudaMemcpyAsync(host_keys[w], h->result.key[w], (size_t)n * (h->spec.key_type[w] == AGGB_I32 ? 4 : 8),
                         cudaMemcpyDefault, h->st));
  for (int j = 0; j < h->cs.ds.nout; j++)
    if (host_out && host_out[j])
      CU(cudaMemcpyAsync(host_out[j], h->result.out[j], (size_t)n * 8, cudaMemcpyDefault, h->st));
  CU(cudaStreamSynchronize(h->st));
  return AGGB_OK;
}

int aggb_metrics_get(void* handle, aggb_metrics* out) {
  Handle* h = (Handle*)handle;
  if (!h || !out) return fail(AGGB_INVALID_ARG, "null argument");
  h->met.kernel_launches = h->launches;
  h->met.high_water_bytes = (int64_t)h->hw;
  h->met.budget_groups = h->budget;
  h->met.partitions_level0 = h->P0;
  *out = h->met;
  return AGGB_OK;
}

int aggb_generate(void* stream, int kind, uint64_t seed, uint64_t stream_id, int64_t start, int64_t n, int64_t lo,
                  int64_t range, const double* cdf, int64_t K, uint64_t a, uint64_t b, void* out, int64_t out_stride) {
  if (n <= 0) return AGGB_OK;
  if ((kind == 0 || kind == 4) && range <= 0) return fail(AGGB_INVALID_ARG, "range must be positive");
  auto base_of = [](uint64_t s, uint64_t sid) {
    uint64_t z = s * 0x9E3779B97F4A7C15ull + sid * 0xD1B54A32D192ED03ull;
    return mix64_sm(z);
  };
  uint64_t base = base_of(seed, stream_id);
  uint64_t base2 = base_of(seed, stream_id + 100);
  int elem = (kind == 4) ? 4 : 8;
  k_gen<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(kind, base, base2, start, n, lo, range, cdf, K, a, b, (uint8_t*)out,
                                                   out_stride ? out_stride : elem);
  CU(cudaGetLastError());
  return AGGB_OK;
}

int aggb_l2_flush(void* stream, void* scratch, int64_t bytes) {
  static uint32_t salt = 1;
  k_l2flush<<<148 * 4, 256, 0, (cudaStream_t)stream>>>((uint4*)scratch, bytes / 16, salt++);
  CU(cudaGetLastError());
  return AGGB_OK;
}

}  // extern "C"

namespace {

int sort_words(Handle* h) { return h->kw + h->cs.nv; }

SortBuf sortbuf(Handle* h, DBuf& b, int64_t cap) {
  SortBuf s;
  memset(&s, 0, sizeof(s));
  s.nw = sort_words(h);
  for (int w = 0; w < s.nw; w++) s.w[w] = b.as<uint64_t>() + (size_t)w * cap;
  return s;
}

// sort_based push: append the batch to the load (k_sort_load, _kernels.py:544-581)
int aggb_sort_push(Handle* h, const ColSrc& col) {
  int64_t need = h->sort_n + col.n;
  int nw = sort_words(h);
  if (need > h->sort_cap) {
    int64_t cap = std::max<int64_t>(need + need / 4, 1 << 16);
    DBuf nb;
    TRY(nb.ensure((size_t)cap * nw * 8, &h->hw));
    for (int w = 0; w < nw && h->sort_n; w++)
      CU(cudaMemcpyAsync(nb.as<uint64_t>() + (size_t)w * cap, h->sort_keys.as<uint64_t>() + (size_t)w * h->sort_cap,
                         (size_t)h->sort_n * 8, cudaMemcpyDeviceToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
    h->sort_keys.release();
    h->sort_keys = nb;
    h->sort_vals.release();
    TRY(h->sort_vals.ensure((size_t)cap * nw * 8, &h->hw));
    h->sort_cap = cap;
  }
  SortBuf a = sortbuf(h, h->sort_keys, h->sort_cap);
  TRY(h->sort_hist.ensure(16 * 256 * 8, &h->hw));
  if (h->sort_n == 0) CU(cudaMemsetAsync(h->sort_hist.p, 0, 16 * 256 * 8, h->st));
  int pe = prof_begin(h, 9);
  unsigned long long* hist = h->sort_hist.as<unsigned long long>();
  if (h->kw == 1) k_sort_append<1, 1><<<h->sms * 8, 256, 0, h->st>>>(col, col.nv, a, h->sort_n, hist);
  else k_sort_append<2, 1><<<h->sms * 8, 256, 0, h->st>>>(col, col.nv, a, h->sort_n, hist);
  prof_end(h, pe);
  h->launches++;
  CU(cudaGetLastError());
  h->sort_n = need;
  return AGGB_OK;
}

int scan_u32(Handle* h, const uint32_t* in, int64_t n, unsigned long long* out, DBuf& tmp) {
  int64_t nb = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
  TRY(tmp.ensure((size_t)(nb + 1) * 8, &h->hw));
  unsigned long long* bs = tmp.as<unsigned long long>();
  k_scan_reduce<<<(unsigned)std::max<int64_t>(nb, 1), 256, 0, h->st>>>(in, n, bs);
  k_scan_top<<<1, 1024, 0, h->st>>>(bs, nb);
  k_scan_down<<<(unsigned)std::max<int64_t>(nb, 1), 256, 0, h->st>>>(in, n, bs, out);
  h->launches += 3;
  CU(cudaGetLastError());
  return AGGB_OK;
}

template <int KW>
int seg_reduce(Handle* h, SortBuf cur, int64_t n) {
  int64_t ntiles = (n + SORT_TILE - 1) / SORT_TILE;
  DBuf th, toff, tmp, heads, longl;
  TRY(th.ensure((size_t)ntiles * 4, nullptr));
  TRY(toff.ensure((size_t)(ntiles + 1) * 8, nullptr));
  int grid = (int)std::min<int64_t>(ntiles, (int64_t)h->sms * 8);
  int pe = prof_begin(h, 11);
  k_head_count<KW><<<grid, SORT_BLOCK, 0, h->st>>>(cur, n, th.as<uint32_t>(), ntiles);
  TRY(scan_u32(h, th.as<uint32_t>(), ntiles, toff.as<unsigned long long>(), tmp));
  unsigned long long last_off = 0;
  uint32_t last_cnt = 0;
  CU(cudaMemcpyAsync(&last_off, toff.as<unsigned long long>() + ntiles - 1, 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaMemcpyAsync(&last_cnt, th.as<uint32_t>() + ntiles - 1, 4, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  int64_t G = (int64_t)last_off + last_cnt;
  // one-word keys, one int64 value, COUNT/SUM(/MIN/MAX): the fused pass (sort.cuh k_seg_emit2)
  if (KW == 1 && cur.nw == 2 && (h->prog == 1 || h->prog == 2) && h->cs.ds.vty[0] == TY_I64 && !getenv("AGGB_NO_SEGFUSE")) {
    TRY(ensure_out(h, G + 16));
    TRY(longl.ensure((size_t)(n / SEG_WALK + 2) * 16, nullptr));
    CU(cudaMemsetAsync(SC(h) + 14, 0, 8, h->st));
    OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
    const int g2 = (int)std::min<int64_t>(ntiles, (int64_t)h->sms * 16);
    if (h->prog == 2) {
      k_seg_emit2<CpC2><<<g2, SEG_BLOCK, 0, h->st>>>(cur.w[0], cur.w[1], n, toff.as<unsigned long long>(), ntiles,
                                                    h->cs.ds, o, longl.as<long long>(), SC(h) + 14);
      k_seg_long2<CpC2><<<h->sms * 2, 256, 0, h->st>>>(cur.w[0], cur.w[1], n, h->cs.ds, o, longl.as<long long>(), SC(h) + 14);
    } else {
      k_seg_emit2<CpC1><<<g2, SEG_BLOCK, 0, h->st>>>(cur.w[0], cur.w[1], n, toff.as<unsigned long long>(), ntiles,
                                                    h->cs.ds, o, longl.as<long long>(), SC(h) + 14);
      k_seg_long2<CpC1><<<h->sms * 2, 256, 0, h->st>>>(cur.w[0], cur.w[1], n, h->cs.ds, o, longl.as<long long>(), SC(h) + 14);
    }
    prof_end(h, pe);
    h->launches += 4;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(SC(h) + 13, &G, 8, cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
    th.release();
    toff.release();
    tmp.release();
    longl.release();
    return AGGB_OK;
  }
  TRY(heads.ensure((size_t)std::max<int64_t>(G, 1) * 8, nullptr));
  TRY(longl.ensure((size_t)std::max<int64_t>(G, 1) * 8, nullptr));
  k_head_compact<KW><<<grid, SORT_BLOCK, 0, h->st>>>(cur, n, toff.as<unsigned long long>(), ntiles,
                                                     heads.as<int64_t>());
  TRY(ensure_out(h, G + 16));
  CU(cudaMemsetAsync(SC(h) + 14, 0, 8, h->st));
  OutBuf o = outbuf(h, h->cfg.emit_partials ? 1 : 0);
  int nwt = nwt_for(std::max(1, cur.nw - KW));
  int sg = (int)std::min<int64_t>((G + 255) / 256, (int64_t)h->sms * 16);
  sg = std::max(sg, 1);
  switch (nwt) {
#define SEG_CASE(NW)                                                                                          \
  case NW:                                                                                                    \
    k_seg_reduce<KW, NW><<<sg, 256, 0, h->st>>>(cur, h->cs.ds, 0, n, heads.as<int64_t>(), G, o,               \
                                                longl.as<int64_t>(), SC(h) + 14);                             \
    k_seg_reduce_long<KW, NW><<<h->sms, SORT_BLOCK, 0, h->st>>>(cur, h->cs.ds, 0, n, heads.as<int64_t>(), G, o, \
                                                                longl.as<int64_t>(), SC(h) + 14);             \
    break;
    SEG_CASE(1) SEG_CASE(2) SEG_CASE(4) SEG_CASE(8) SEG_CASE(16)
    default: SEG_CASE(32)
#undef SEG_CASE
  }
  prof_end(h, pe);
  h->launches += 4;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(SC(h) + 13, &G, 8, cudaMemcpyHostToDevice, h->st));
  CU(cudaStreamSynchronize(h->st));
  th.release();
  toff.release();
  tmp.release();
  heads.release();
  longl.release();
  return AGGB_OK;
}

// sort_based close: radix sort + fold (sort_based.py:135-211, k_fold_sorted :601-638)
int aggb_sort_finish(Handle* h) {
  int64_t n = h->sort_n;
  if (n == 0) return AGGB_OK;
  SortBuf a = sortbuf(h, h->sort_keys, h->sort_cap);
  SortBuf b = sortbuf(h, h->sort_vals, h->sort_cap);
  if (h->cfg.input_sorted) {  // streamed fold with the order contract
    int bad = 0;
    CU(cudaMemsetAsync(SC(h) + 15, 0, 8, h->st));
    if (h->kw == 1) k_check_sorted<1><<<h->sms * 4, 256, 0, h->st>>>(a, n, (int*)(SC(h) + 15));
    else k_check_sorted<2><<<h->sms * 4, 256, 0, h->st>>>(a, n, (int*)(SC(h) + 15));
    CU(cudaMemcpyAsync(&bad, SC(h) + 15, 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    if (bad) return fail(AGGB_ORDER_ERROR, "input declared sorted but a key decreased");
  } else {
    // byte histograms of every key, gathered by k_sort_append as the keys came in
    std::vector<unsigned long long> hh(16 * 256);
    CU(cudaMemcpyAsync(hh.data(), h->sort_hist.p, 16 * 256 * 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    // LSD order: least significant word last in the key, lowest byte first
    std::vector<std::pair<int, int>> passes;
    for (int w = h->kw - 1; w >= 0; w--)
      for (int by = 0; by < 8; by++) {
        const unsigned long long* row = &hh[(size_t)(w * 8 + by) * 256];
        int nz = 0;
        for (int d = 0; d < 256; d++) nz += row[d] != 0;
        if (nz > 1) passes.push_back({w, by});
      }
    int64_t ntiles = (n + SORT_TILE - 1) / SORT_TILE;
    DBuf counts, offs, tmp;
    // two-word records below 2^30: one-sweep passes (chained scan with decoupled
    // look-back inside the scatter; the digits' global bases from the byte histograms)
    const bool onesweep = a.nw == 2 && n < (1ll << 30) && !getenv("AGGB_NO_ONESWEEP");
    if (onesweep && !passes.empty()) {
      DBuf status, gb;
      TRY(status.ensure((size_t)ntiles * 256 * 4, nullptr));
      TRY(gb.ensure(passes.size() * 256 * 8 + 8, nullptr));
      std::vector<unsigned long long> bases(passes.size() * 256);
      for (size_t q = 0; q < passes.size(); q++) {
        const unsigned long long* row = &hh[(size_t)(passes[q].first * 8 + passes[q].second) * 256];
        unsigned long long acc = 0;
        for (int d = 0; d < 256; d++) {
          bases[q * 256 + d] = acc;
          acc += row[d];
        }
      }
      CU(cudaMemcpyAsync(gb.p, bases.data(), bases.size() * 8, cudaMemcpyHostToDevice, h->st));
      const int smem2 = SORT_TILE * 16;
      CU(cudaFuncSetAttribute((const void*)k_onesweep2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      int occ2 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_onesweep2, S2_BLOCK, smem2);
      const int grid2 = (int)ntiles;  // one tile per CTA, taken in ticket order
      unsigned long long* ticket = gb.as<unsigned long long>() + passes.size() * 256;
      for (size_t q = 0; q < passes.size(); q++) {
        int pe2 = prof_begin(h, 9);
        CU(cudaMemsetAsync(status.p, 0, (size_t)ntiles * 256 * 4, h->st));
        CU(cudaMemsetAsync(ticket, 0, 8, h->st));
        k_onesweep2<<<grid2, S2_BLOCK, smem2, h->st>>>(a, b, passes[q].first, 8 * passes[q].second, n,
                                                         gb.as<unsigned long long>() + q * 256, status.as<uint32_t>(),
                                                         ticket, ntiles, getenv("AGGB_OS_NOWRITE") ? 1 : 0);
        prof_end(h, pe2);
        h->launches++;
        CU(cudaGetLastError());
        std::swap(a, b);
      }
      CU(cudaStreamSynchronize(h->st));
      status.release();
      gb.release();
      passes.clear();
    }
    if (!passes.empty()) {
      TRY(counts.ensure((size_t)ntiles * 256 * 4, nullptr));
      TRY(offs.ensure((size_t)ntiles * 256 * 8, nullptr));
    }
    int grid = (int)std::min<int64_t>(ntiles, (int64_t)h->sms * 8);
    for (auto& pw : passes) {
      int pe2 = prof_begin(h, 9);
      k_tile_hist<<<grid, 256, 0, h->st>>>(a.w[pw.first], 8 * pw.second, n, counts.as<uint32_t>(), ntiles);
      TRY(scan_u32(h, counts.as<uint32_t>(), ntiles * 256, offs.as<unsigned long long>(), tmp));
      if (a.nw == 2) {  // key word + one payload word: tile-local rank + SMEM reorder
        const int smem2 = SORT_TILE * 16;
        CU(cudaFuncSetAttribute((const void*)k_scatter2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
        int occ2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_scatter2, S2_BLOCK, smem2);
        const int grid2 = (int)std::min<int64_t>(ntiles, (int64_t)std::max(1, occ2) * h->sms);
        k_scatter2<<<grid2, S2_BLOCK, smem2, h->st>>>(a, b, pw.first, 8 * pw.second, n,
                                                        offs.as<unsigned long long>(), ntiles);
      } else {
        k_scatter<<<grid, SORT_BLOCK, 0, h->st>>>(a, b, pw.first, 8 * pw.second, n, offs.as<unsigned long long>(),
                                                  ntiles);
      }
      prof_end(h, pe2);
      h->launches += 2;
      CU(cudaGetLastError());
      std::swap(a, b);
    }
    CU(cudaStreamSynchronize(h->st));
    counts.release();
    offs.release();
    tmp.release();
  }
  return h->kw == 1 ? seg_reduce<1>(h, a, n) : seg_reduce<2>(h, a, n);
}
}  // namespace

extern "C" {
int64_t aggb_exchange_record_bytes(void* handle) {
  Handle* h = (Handle*)handle;
  return h ? (int64_t)(h->kw + h->cs.ds.ns) * 8 : 0;
}

int64_t aggb_pool_host_bytes(void* handle) {
  Handle* h = (Handle*)handle;
  return h ? (int64_t)h->pool_base.host_mapped : -1;
}

int64_t aggb_exchange_raw_record_bytes(void* handle) {
  Handle* h = (Handle*)handle;
  return h ? (int64_t)(h->spec.n_keys + h->spec.n_vals) * 8 : -1;
}

int aggb_exchange_pack_raw(void* handle, const aggb_input* in, int nranks, void* send, int64_t* counts) {
  Handle* h = (Handle*)handle;
  if (!h || !in || !counts || nranks < 1 || nranks > 256) return fail(AGGB_INVALID_ARG, "bad exchange arguments");
  if (in->on_host) return fail(AGGB_INVALID_ARG, "exchange_pack_raw takes device columns");
  cudaSetDevice(h->device);
  for (int i = 0; i < nranks; i++) counts[i] = 0;
  if (in->n_rows <= 0) return AGGB_OK;
  if (!send) return fail(AGGB_INVALID_ARG, "null send buffer");
  ColSrc col = col_of(h, in, in->key, in->val);
  // the partial exchange's seed: either mode sends a key to the same rank
  const uint64_t seed = level_seed(h->cfg.seed, SALT_EXCH, 0);
  DBuf c;
  TRY(c.ensure(2 * 256 * 8, nullptr));
  unsigned long long* cnt = c.as<unsigned long long>();
  CU(cudaMemsetAsync(cnt, 0, 256 * 8, h->st));
  const int grid = (int)std::min<int64_t>((col.n + 255) / 256, (int64_t)h->sms * 8);
  int pe = prof_begin(h, 10);
  if (h->kw == 1) k_exch_raw_count<1><<<grid, 256, 0, h->st>>>(col, seed, nranks, cnt);
  else k_exch_raw_count<2><<<grid, 256, 0, h->st>>>(col, seed, nranks, cnt);
  std::vector<unsigned long long> hc(nranks), off(nranks);
  CU(cudaMemcpyAsync(hc.data(), cnt, nranks * 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  unsigned long long acc = 0;
  for (int i = 0; i < nranks; i++) {
    off[i] = acc;
    acc += hc[i];
    counts[i] = (int64_t)hc[i];
  }
  CU(cudaMemcpyAsync(cnt + 256, off.data(), nranks * 8, cudaMemcpyHostToDevice, h->st));
  if (h->kw == 1) k_exch_raw_scatter<1><<<grid, 256, 0, h->st>>>(col, seed, nranks, cnt + 256, (uint64_t*)send);
  else k_exch_raw_scatter<2><<<grid, 256, 0, h->st>>>(col, seed, nranks, cnt + 256, (uint64_t*)send);
  prof_end(h, pe);
  h->launches += 2;
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->st));
  return AGGB_OK;
}

int aggb_exchange_pack(void* handle, int nranks, void* send, int64_t* counts) {
  Handle* h = (Handle*)handle;
  if (!h || !counts || nranks < 1 || nranks > 256) return fail(AGGB_INVALID_ARG, "bad exchange arguments");
  if (!h->finished) return fail(AGGB_INVALID_ARG, "exchange_pack before finish");
  if (!h->cfg.emit_partials) return fail(AGGB_SPEC_ERROR, "exchange needs a handle created with emit_partials=1");
  cudaSetDevice(h->device);
  int64_t n = h->result.n_groups;
  for (int i = 0; i < nranks; i++) counts[i] = 0;
  if (n == 0) return AGGB_OK;
  if (!send) return fail(AGGB_INVALID_ARG, "null send buffer");
  uint64_t seed = level_seed(h->cfg.seed, SALT_EXCH, 0);
  DBuf c;
  TRY(c.ensure(2 * 256 * 8, nullptr));
  unsigned long long* cnt = c.as<unsigned long long>();
  CU(cudaMemsetAsync(cnt, 0, 256 * 8, h->st));
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)h->sms * 8);
  int pe = prof_begin(h, 10);
  if (h->kw == 1) k_exch_count<1><<<grid, 256, 0, h->st>>>(h->out_keys.as<uint64_t>(), h->out_cap, n, seed, nranks, cnt);
  else k_exch_count<2><<<grid, 256, 0, h->st>>>(h->out_keys.as<uint64_t>(), h->out_cap, n, seed, nranks, cnt);
  std::vector<unsigned long long> hc(nranks), off(nranks);
  CU(cudaMemcpyAsync(hc.data(), cnt, nranks * 8, cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  unsigned long long acc = 0;
  for (int i = 0; i < nranks; i++) {
    off[i] = acc;
    acc += hc[i];
    counts[i] = (int64_t)hc[i];
  }
  CU(cudaMemcpyAsync(cnt + 256, off.data(), nranks * 8, cudaMemcpyHostToDevice, h->st));
  if (h->kw == 1)
    k_exch_scatter<1><<<grid, 256, 0, h->st>>>(h->out_keys.as<uint64_t>(), h->out_vals.as<uint64_t>(), h->out_cap, n,
                                               h->cs.ds.ns, seed, nranks, cnt + 256, (uint64_t*)send);
  else
    k_exch_scatter<2><<<grid, 256, 0, h->st>>>(h->out_keys.as<uint64_t>(), h->out_vals.as<uint64_t>(), h->out_cap, n,
                                               h->cs.ds.ns, seed, nranks, cnt + 256, (uint64_t*)send);
  prof_end(h, pe);
  h->launches += 2;
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->st));
  return AGGB_OK;
}
}
