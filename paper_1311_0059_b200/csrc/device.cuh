// device.cuh — device building blocks of the group-by hot path (sm_100a).
//
// Restates, for the GPU, the per-record arithmetic of the reference kernels
// (/root/reference/pkg/src/aggbench/_kernels.py):
//   hash_bytes/mix_seed (:102-118)  -> seeded 64-bit fmix hash per role/level
//   _key_cmp (:121-131)             -> 1-2 word key compare (BE key bytes ==
//                                      unsigned word order)
//   _merge_fields (:148-159)        -> typed atomic ADD / MIN / MAX updates
//   init ops (k_expand :237-264)    -> contribution words built on load
//   finish ops (_emit_record :199-229) -> finalize in the flush kernels
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aggb {

constexpr int MAX_STATES = 32;
constexpr int MAX_VALS = 32;
constexpr int MAX_OUT = 32;
constexpr uint64_t EMPTY = 0x8000000000000000ull;  // key word of an empty slot

enum : uint8_t { OP_ADD = 0, OP_MIN = 1, OP_MAX = 2 };
enum : uint8_t { TY_I64 = 0, TY_F64 = 1, TY_I32 = 2 };
// how a state field's contribution is formed from a loaded record
enum : uint8_t {
  SRC_ONE = 0,        // COUNT: constant 1 (INIT_ONE, core.py:71-72)
  SRC_VAL = 1,        // raw value column (INIT_COPY)
  SRC_STATE_F64 = 2,  // external state column stored as f64 (reference frames)
  SRC_NATIVE = 3      // our own partial-state word (already in state form)
};

// Compiled AggSpec (core.py:126-185) with duplicate state fields removed:
// AVG's (sum, count) share SUM / COUNT fields of the same column.
struct DevSpec {
  int32_t ns;                    // state fields
  int32_t nv;                    // payload words per raw record
  uint8_t op[MAX_STATES];        // OP_*
  uint8_t ty[MAX_STATES];        // TY_I64 / TY_F64 (state representation)
  uint8_t srck[MAX_STATES];      // SRC_*
  int8_t src[MAX_STATES];        // payload word index for SRC_VAL / SRC_STATE_F64
  uint8_t vty[MAX_VALS];         // payload word type (TY_I64 / TY_F64)
  int32_t nout;
  uint8_t fin_div[MAX_OUT];      // 0 FINISH_FIRST, 1 FINISH_DIV
  uint8_t fin_a[MAX_OUT];        // state field (numerator)
  uint8_t fin_b[MAX_OUT];        // state field (denominator, DIV)
  uint8_t out_ty[MAX_OUT];       // TY_I64 / TY_F64
};

// ---------------------------------------------------------------------------
// hashing
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

template <int KW>
__device__ __forceinline__ uint64_t hash_key(const uint64_t (&k)[KW], uint64_t seed) {
  uint64_t h = fmix64(k[0] ^ seed);
  if (KW == 2) h = fmix64(h ^ k[1] ^ 0x9E3779B97F4A7C15ull);
  return h;
}

// range-reduce the top 32 bits of a hash onto [0, n).  Written with __umulhi:
// nvcc 12.9 lowered the equivalent (uint32_t)(((h >> 32) * (uint64_t)n) >> 32)
// into a wrong shared-memory address computation when the result indexed a
// __shared__ array directly (k_exch_count counted every record into bin 0;
// profiles/r01_notes.md).
__device__ __forceinline__ uint32_t reduce32(uint64_t h, uint32_t n) {
  return __umulhi((uint32_t)(h >> 32), n);
}

template <int KW>
__device__ __forceinline__ bool is_sentinel(const uint64_t (&k)[KW]) {
  bool s = k[0] == EMPTY;
  if (KW == 2) s = s && (k[1] == EMPTY);
  return s;
}

template <int KW>
__device__ __forceinline__ bool key_eq(const uint64_t (&a)[KW], const uint64_t (&b)[KW]) {
  bool e = a[0] == b[0];
  if (KW == 2) e = e && (a[1] == b[1]);
  return e;
}

// ---------------------------------------------------------------------------
// state representation
// ---------------------------------------------------------------------------

// order-preserving f64 -> u64 (MIN/MAX on doubles through integer atomics)
__device__ __forceinline__ uint64_t f64_ord(uint64_t b) {
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ uint64_t ord_f64(uint64_t o) {
  return (o & 0x8000000000000000ull) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
}

__host__ __device__ __forceinline__ uint64_t state_identity(uint8_t op, uint8_t ty) {
  if (op == OP_ADD) return 0ull;  // 0 and +0.0
  if (op == OP_MIN) return ty == TY_I64 ? 0x7FFFFFFFFFFFFFFFull : 0xFFFFFFFFFFFFFFFFull;
  return ty == TY_I64 ? 0x8000000000000000ull : 0ull;
}

// contribution word of state field j for a record whose payload words are v[]
__device__ __forceinline__ uint64_t contribution(const DevSpec& sp, int j, const uint64_t* v) {
  uint8_t k = sp.srck[j];
  if (k == SRC_ONE) return 1ull;
  uint64_t w = v[sp.src[j]];
  if (k == SRC_NATIVE) return w;
  if (k == SRC_STATE_F64) {
    double d = __longlong_as_double((long long)w);
    if (sp.ty[j] == TY_I64) return (uint64_t)(long long)d;  // counts are integral
    w = (uint64_t)__double_as_longlong(d);
  } else if (sp.ty[j] == TY_F64 && sp.vty[sp.src[j]] == TY_I64) {
    w = (uint64_t)__double_as_longlong((double)(long long)w);
  }
  if (sp.ty[j] == TY_F64 && sp.op[j] != OP_ADD) return f64_ord(w);
  return w;
}

// global-memory (L2) update: RED.ADD.64 / RED.ADD.F64 / RED.MIN / RED.MAX.
// Written as red.global PTX: through a generic pointer the compiler emits an
// address-space test and both a shared and a global path for every atomic
// (ncu, k_probe_wc<resolve>: ~135 instructions per hit for four REDs).
__device__ __forceinline__ void gupdate(uint64_t* p, uint8_t op, uint8_t ty, uint64_t c) {
  if (op == OP_ADD) {
    if (ty == TY_F64) asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(__longlong_as_double((long long)c)) : "memory");
    else asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(c) : "memory");
  } else if (op == OP_MIN) {
    if (ty == TY_I64) asm volatile("red.global.min.s64 [%0], %1;" ::"l"(p), "l"(c) : "memory");
    else asm volatile("red.global.min.u64 [%0], %1;" ::"l"(p), "l"(c) : "memory");
  } else {
    if (ty == TY_I64) asm volatile("red.global.max.s64 [%0], %1;" ::"l"(p), "l"(c) : "memory");
    else asm volatile("red.global.max.u64 [%0], %1;" ::"l"(p), "l"(c) : "memory");
  }
}

// shared-memory update.  64-bit ATOMS.ADD does not exist on sm_100a (it is a
// CAS loop, 3x slower than 32-bit ATOMS.ADD, profiles/r01_ubench_calibration.txt),
// so integer ADD is two 32-bit adds with an explicit carry.  MIN/MAX read first
// and only CAS when the value improves (most records do not).
__device__ __forceinline__ void supdate(uint64_t* p, uint8_t op, uint8_t ty, uint64_t c) {
  if (op == OP_ADD) {
    if (ty == TY_F64) {
      atomicAdd((double*)p, __longlong_as_double((long long)c));
    } else {
      uint32_t* w = (uint32_t*)p;
      uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
      uint32_t old = atomicAdd(w, lo);
      hi += (uint32_t)((uint32_t)(old + lo) < old);
      if (hi) atomicAdd(w + 1, hi);
    }
    return;
  }
  // native 64-bit shared-memory MIN / MAX (ATOMS.MIN/MAX.64), fire-and-forget: no read
  // of the state before the update (the read-then-CAS loop made every record wait for
  // a shared-memory round trip per MIN/MAX field)
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  if (op == OP_MIN) {
    if (ty == TY_I64) asm volatile("red.shared.min.s64 [%0], %1;" ::"r"(a), "l"((long long)c) : "memory");
    else asm volatile("red.shared.min.u64 [%0], %1;" ::"r"(a), "l"(c) : "memory");
  } else {
    if (ty == TY_I64) asm volatile("red.shared.max.s64 [%0], %1;" ::"r"(a), "l"((long long)c) : "memory");
    else asm volatile("red.shared.max.u64 [%0], %1;" ::"r"(a), "l"(c) : "memory");
  }
}

// plain (single-owner) merge of two state words, used where one thread owns a group
__device__ __forceinline__ uint64_t merge_word(uint64_t a, uint64_t b, uint8_t op, uint8_t ty) {
  if (op == OP_ADD) {
    if (ty == TY_F64)
      return (uint64_t)__double_as_longlong(__longlong_as_double((long long)a) + __longlong_as_double((long long)b));
    return a + b;
  }
  bool smaller = (ty == TY_I64) ? ((long long)b < (long long)a) : (b < a);
  if (op == OP_MIN) return smaller ? b : a;
  bool larger = (ty == TY_I64) ? ((long long)b > (long long)a) : (b > a);
  return larger ? b : a;
}

// ---------------------------------------------------------------------------
// compact per-field descriptors (kept in shared memory by the kernels so that
// the per-record update loop indexes SMEM instead of a local copy of DevSpec)
//   bits 0-1 op, 2-3 state type, 4-5 source kind, 6-7 source value type,
//   8-15 source word index
// ---------------------------------------------------------------------------

__host__ __device__ __forceinline__ uint32_t field_desc(const DevSpec& sp, int j) {
  int src = sp.src[j] < 0 ? 0 : sp.src[j];
  uint32_t vty = sp.srck[j] == SRC_VAL ? sp.vty[src] : TY_I64;
  return (uint32_t)sp.op[j] | ((uint32_t)sp.ty[j] << 2) | ((uint32_t)sp.srck[j] << 4) | (vty << 6) |
         ((uint32_t)src << 8);
}

template <int NWT>
__device__ __forceinline__ uint64_t pick(const uint64_t (&v)[NWT], int i) {
  uint64_t w = v[0];
#pragma unroll
  for (int q = 1; q < NWT; q++)
    if (q == i) w = v[q];
  return w;
}

// contribution of field j (descriptor fd) for a record with payload v[]:
// kind 0 = raw payload (init ops applied), kind 1 = native partial states
template <int NWT>
__device__ __forceinline__ uint64_t contrib_fd(uint32_t fd, int kind, int j, const uint64_t (&v)[NWT]) {
  if (kind) return pick<NWT>(v, j);
  uint32_t sk = (fd >> 4) & 3;
  if (sk == SRC_ONE) return 1ull;
  uint64_t w = pick<NWT>(v, (int)(fd >> 8));
  uint32_t ty = (fd >> 2) & 3, op = fd & 3;
  if (sk == SRC_STATE_F64) {
    double d = __longlong_as_double((long long)w);
    if (ty == TY_I64) return (uint64_t)(long long)d;
  } else if (ty == TY_F64 && ((fd >> 6) & 3) == TY_I64) {
    w = (uint64_t)__double_as_longlong((double)(long long)w);
  }
  if (ty == TY_F64 && op != OP_ADD) return f64_ord(w);
  return w;
}

// ---------------------------------------------------------------------------
// field programs: the per-record update sequence of a compiled AggSpec.
//   PD           runtime program (descriptors in shared memory, any spec)
//   PS<F...>     compile-time program: the benchmark specs get straight-line
//                update code with every op/type/source branch folded away
// ---------------------------------------------------------------------------

struct PD {
  static constexpr int N = 0;
};
template <uint32_t... F>
struct PS {
  static constexpr int N = sizeof...(F);
};

// global (L2) updates
template <int NWT, uint32_t F, uint32_t... Fs>
__device__ __forceinline__ void gupd_s(uint64_t* st, uint64_t stride, uint64_t s, int kind, int j,
                                       const uint64_t (&v)[NWT]) {
  gupdate(st + (uint64_t)j * stride + s, F & 3, (F >> 2) & 3, contrib_fd<NWT>(F, kind, j, v));
  if constexpr (sizeof...(Fs) > 0) gupd_s<NWT, Fs...>(st, stride, s, kind, j + 1, v);
}
template <class PG>
struct Upd;
template <>
struct Upd<PD> {
  template <int NWT>
  static __device__ __forceinline__ void g(uint64_t* st, uint64_t stride, uint64_t s, int kind, const uint32_t* fd,
                                           int ns, const uint64_t (&v)[NWT]) {
    for (int j = 0; j < ns; j++) {
      uint32_t f = fd[j];
      gupdate(st + (uint64_t)j * stride + s, f & 3, (f >> 2) & 3, contrib_fd<NWT>(f, kind, j, v));
    }
  }
  template <int NWT>
  static __device__ __forceinline__ void sm(uint64_t* st, int stride, int s, int kind, const uint32_t* fd, int ns,
                                            const uint64_t (&v)[NWT]) {
    for (int j = 0; j < ns; j++) {
      uint32_t f = fd[j];
      supdate(st + (size_t)j * stride + s, f & 3, (f >> 2) & 3, contrib_fd<NWT>(f, kind, j, v));
    }
  }
};

template <int NWT, uint32_t F, uint32_t... Fs>
__device__ __forceinline__ void supd_s(uint64_t* st, int stride, int s, int kind, int j, const uint64_t (&v)[NWT]) {
  supdate(st + (size_t)j * stride + s, F & 3, (F >> 2) & 3, contrib_fd<NWT>(F, kind, j, v));
  if constexpr (sizeof...(Fs) > 0) supd_s<NWT, Fs...>(st, stride, s, kind, j + 1, v);
}

template <uint32_t... F>
struct Upd<PS<F...>> {
  template <int NWT>
  static __device__ __forceinline__ void g(uint64_t* st, uint64_t stride, uint64_t s, int kind, const uint32_t*, int,
                                           const uint64_t (&v)[NWT]) {
    gupd_s<NWT, F...>(st, stride, s, kind, 0, v);
  }
  template <int NWT>
  static __device__ __forceinline__ void sm(uint64_t* st, int stride, int s, int kind, const uint32_t*, int,
                                            const uint64_t (&v)[NWT]) {
    supd_s<NWT, F...>(st, stride, s, kind, 0, v);
  }
};

// the benchmark specs (descriptor = op | ty<<2 | srck<<4 | vty<<6 | src<<8)
using ProgC1 = PS<0x000, 0x010>;                           // COUNT, SUM(i64)        C1, C4
using ProgC2 = PS<0x000, 0x010, 0x011, 0x012>;             // COUNT, SUM, MIN, MAX   C2
using ProgC3 = PS<0x000, 0x054>;                           // COUNT, SUM(f64) (+AVG) C3
using ProgC5 = PS<0x000, 0x010, 0x011, 0x012, 0x110, 0x111, 0x112,
                  0x254, 0x255, 0x256, 0x354, 0x355, 0x356>;  // C5: 13 fields

// ---------------------------------------------------------------------------
// 128-bit CAS (two-word keys, e.g. C5's int64 || int32)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cas128(uint64_t* p, uint64_t clo, uint64_t chi, uint64_t nlo,
                                       uint64_t nhi, uint64_t& olo, uint64_t& ohi) {
  asm volatile(
      "{\n .reg .b128 d, c, n;\n mov.b128 c, {%2,%3};\n mov.b128 n, {%4,%5};\n"
      " atom.cas.b128 d, [%6], c, n;\n mov.b128 {%0,%1}, d;\n}"
      : "=l"(olo), "=l"(ohi)
      : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "l"(p)
      : "memory");
}

// ---------------------------------------------------------------------------
// spill page pool: CTA-private pages (no spin waits, one atomic per page)
// ---------------------------------------------------------------------------

struct PagePool {
  uint8_t* base;            // one contiguous allocation of capacity pages
  uint32_t page_bytes;
  uint32_t* next_page;      // allocation counter
  uint32_t capacity;        // pages available
  int32_t* page_part;       // partition of each page
  int32_t* page_fill;       // records in each page
  int32_t* page_set;        // spill set id of each page
  uint32_t* overflow;       // set when a pass ran out of pages
};

__device__ __forceinline__ uint8_t* page_ptr(const PagePool& pp, uint32_t pg) {
  return pp.base + (size_t)pg * pp.page_bytes;
}

__device__ __forceinline__ int32_t page_alloc(const PagePool& pp, int32_t part, int32_t set) {
  uint32_t pg = atomicAdd(pp.next_page, 1u);
  if (pg >= pp.capacity) {
    atomicExch(pp.overflow, 1u);
    return -1;
  }
  pp.page_part[pg] = part;
  pp.page_set[pg] = set;
  pp.page_fill[pg] = 0;
  return (int32_t)pg;
}

// a spill set: records of `rw` 8-byte words (key words first), stored record
// after record (AoS) inside a page, so a 32-byte sector holds whole records
struct SpillSet {
  int32_t id;
  int32_t nparts;
  int32_t rw;               // words per record
  int32_t per_page;         // records per page
  uint64_t seed;            // partition hash seed of this set (level / role specific)
  int32_t kind;             // 0 raw payload, 1 native partial states
};

__device__ __forceinline__ uint64_t* page_rec(const PagePool& pp, uint32_t pg, int rw, int slot) {
  return (uint64_t*)page_ptr(pp, pg) + (size_t)slot * rw;
}

}  // namespace aggb
