/*
 * aggoracle.c — CPU ORACLE (test infrastructure only; never on the product path).
 *
 * Plain-C restatement of the reference's memory-bounded GROUP-BY operators
 * (arXiv 1311.0059, package `aggbench` under /root/reference/pkg/src/aggbench).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library, and only as the checker or as the timed
 * CPU baseline ("kind": "port").
 *
 * What is restated (each function cites the reference file:line it follows):
 *   - the wire format: record = u16 LE klen | key bytes | f64 x nf, records never
 *     straddle a frame, klen 0 ends a frame            (core.py:1-10, :193-265)
 *   - hash_bytes / mix_seed, bit-exact                 (_kernels.py:102-118)
 *   - byte-lexicographic key order                     (_kernels.py:121-131)
 *   - per-field merge ADD/MIN/MAX on f64, finish FIRST/DIV (_kernels.py:148-229)
 *   - the frame budget (FrameAllocator) and its high-water mark (core.py:273-331)
 *   - plan_table / ChainedHashTable with slot + bloom overhead frames,
 *     first-fit chain append, TABLE_FULL on physical fullness
 *                                                      (hash_table.py:31-171,
 *                                                       _kernels.py:298-392)
 *   - planning: fudge_factor, plan_partitions (Formula 1), plan_hybrid (grace
 *     trigger G*F >= M^2), sort_merge_levels, fallback_controller, make_cuts
 *                                                      (hybrid.py:89-163,
 *                                                       run_store.py:222-246)
 *   - operators pre_partitioning (fill / freeze / bloom-probe / spill,
 *     hybrid.py:481-576, _kernels.py:917-962), original_hh (partition-0 table,
 *     overflow cut, hybrid.py:356-478, _kernels.py:865-914), grace partitioning
 *     (hybrid.py:281-318), recursion with fresh per-level seeds and hash_sort
 *     fallback (hybrid.py:244-277), hash_sort (hash_sort.py:20-115) and
 *     sort_based (sort_based.py:24-211).
 *
 * Deliberate simplifications (results are unaffected; documented in DESIGN.md):
 *   - spill runs are in-memory frame lists instead of files (run_store.py:36-110);
 *   - the multi-round loser-tree merge (run_store.py:249-386, _kernels.py:702-857)
 *     is one k-way heap merge per operator close: the fold result is identical,
 *     only the number of intermediate rounds differs;
 *   - sort_based sorts record indices with qsort + a key tie-break on arrival
 *     order instead of the seeded 3-way quicksort (_kernels.py:414-470);
 *   - counters (comparisons etc.) are not modelled, only groups/spills/levels.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORA_OK 0
#define ORA_INVALID_BUDGET 1
#define ORA_CAPACITY_EXCEEDED 3
#define ORA_SPEC_ERROR 4
#define ORA_ORDER_ERROR 5
#define ORA_NOMEM 8

#define KLEN_SIZE 2
#define FIELD_SIZE 8
#define LINK_SIZE 8
#define SLOT_SIZE 8
#define HASH_SPACE 4294967296LL

enum { ALGO_SORT_BASED = 0, ALGO_HASH_SORT = 1, ALGO_ORIGINAL_HH = 2,
       ALGO_PRE_PARTITIONING = 5 };
enum { MERGE_ADD = 0, MERGE_MIN = 1, MERGE_MAX = 2 };
enum { FINISH_FIRST = 0, FINISH_DIV = 1 };

/* ------------------------------------------------------------------------ */
/* hashing (_kernels.py:102-118)                                             */
/* ------------------------------------------------------------------------ */

uint32_t ora_hash_bytes(const uint8_t* b, int64_t len, uint32_t seed) {
  uint32_t h = 0x811C9DC5u ^ seed;
  for (int64_t i = 0; i < len; i++) h = (h ^ b[i]) * 0x01000193u;
  h = (h ^ (h >> 16)) * 0x045D9F3Bu;
  h = (h ^ (h >> 16)) * 0x045D9F3Bu;
  return h ^ (h >> 16);
}

uint32_t ora_mix_seed(uint64_t seed, uint64_t salt) {
  uint32_t h = (uint32_t)(seed * 2654435761ull + salt * 40503ull + 0x9E37ull);
  h = (h ^ (h >> 15)) * 2246822519u;
  h = (h ^ (h >> 13)) * 3266489917u;
  return h ^ (h >> 16);
}

/* _kernels.py:121-131 */
static int key_cmp(const uint8_t* a, int alen, const uint8_t* b, int blen) {
  int n = alen < blen ? alen : blen;
  int c = memcmp(a, b, (size_t)n);
  if (c) return c < 0 ? -1 : 1;
  if (alen == blen) return 0;
  return alen < blen ? -1 : 1;
}

static inline uint16_t rd16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static inline void wr16(uint8_t* p, uint16_t v) { p[0] = v & 0xFF; p[1] = v >> 8; }
static inline double rdf(const uint8_t* p) { double d; memcpy(&d, p, 8); return d; }
static inline void wrf(uint8_t* p, double d) { memcpy(p, &d, 8); }
static inline int64_t rdi(const uint8_t* p) { int64_t d; memcpy(&d, p, 8); return d; }
static inline void wri(uint8_t* p, int64_t d) { memcpy(p, &d, 8); }

/* ------------------------------------------------------------------------ */
/* spec + config                                                             */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t nf;              /* state width                                   */
  int8_t merge_ops[64];
  int32_t nout;            /* out width                                     */
  int8_t finish_ops[64];
  int8_t finish_src[64];
} ora_spec;

typedef struct {
  int32_t algo;
  int32_t memory_frames;
  int32_t frame_size;
  int32_t input_sorted;
  double fudge;
  double slot_ratio;
  uint64_t seed;
  double group_estimate;   /* < 0 : None                                    */
  /* DatasetStats (core.py:383-404) */
  double R, R_t, G, G_t;
} ora_cfg;

typedef struct {
  int64_t output_groups;
  int64_t frames_written;
  int64_t frames_read;
  int64_t spilled_partitions;
  int64_t fallbacks;
  int64_t grace_levels;
  int64_t recursion_depth;
  int64_t high_water;
  int64_t spilled_records;
} ora_metrics;

/* ------------------------------------------------------------------------ */
/* frame budget (core.py:273-331)                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
  int32_t budget, p;
  uint8_t* pool;           /* budget * p bytes                              */
  int64_t* used;
  int32_t* free_list;
  int32_t nfree;
  int32_t high_water;
} Alloc;

static int alloc_init(Alloc* a, int32_t budget, int32_t p) {
  a->budget = budget; a->p = p;
  a->pool = (uint8_t*)calloc((size_t)budget, (size_t)p);
  a->used = (int64_t*)calloc((size_t)budget, sizeof(int64_t));
  a->free_list = (int32_t*)malloc(sizeof(int32_t) * (size_t)budget);
  if (!a->pool || !a->used || !a->free_list) return ORA_NOMEM;
  for (int32_t i = 0; i < budget; i++) a->free_list[i] = budget - 1 - i;
  a->nfree = budget; a->high_water = 0;
  return ORA_OK;
}
static void alloc_free(Alloc* a) { free(a->pool); free(a->used); free(a->free_list); }
static int32_t outstanding(const Alloc* a) { return a->budget - a->nfree; }
static uint8_t* fview(Alloc* a, int32_t fid) { return a->pool + (size_t)fid * a->p; }
static void clear_frame(Alloc* a, int32_t fid) { memset(fview(a, fid), 0, (size_t)a->p); a->used[fid] = 0; }
static int32_t frame_alloc(Alloc* a) {
  if (a->nfree == 0) return -1;
  int32_t fid = a->free_list[--a->nfree];
  clear_frame(a, fid);
  if (outstanding(a) > a->high_water) a->high_water = outstanding(a);
  return fid;
}
static void frame_release(Alloc* a, int32_t fid) { a->free_list[a->nfree++] = fid; }

/* ------------------------------------------------------------------------ */
/* in-memory runs (replaces run files, run_store.py:36-131)                  */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* data;           /* frames back to back                           */
  int64_t frames, cap;
  int64_t records;
  int32_t p;
} Run;

static int run_append(Run* r, const uint8_t* frame, int32_t p) {
  if (r->frames == r->cap) {
    int64_t nc = r->cap ? r->cap * 2 : 8;
    uint8_t* nd = (uint8_t*)realloc(r->data, (size_t)nc * p);
    if (!nd) return ORA_NOMEM;
    r->data = nd; r->cap = nc;
  }
  memcpy(r->data + (size_t)r->frames * p, frame, (size_t)p);
  r->frames++; r->p = p;
  return ORA_OK;
}
static void run_free(Run* r) { free(r->data); memset(r, 0, sizeof(*r)); }

static int64_t count_records(const uint8_t* f, int32_t p, int nf) {  /* _kernels.py:1129-1140 */
  int64_t off = 0, n = 0;
  while (off <= p - KLEN_SIZE) {
    int kl = rd16(f + off);
    if (!kl) break;
    n++; off += KLEN_SIZE + kl + FIELD_SIZE * nf;
  }
  return n;
}

/* ------------------------------------------------------------------------ */
/* output sink: collects finalized groups (decoded)                          */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* keys;           /* n * klen_max, zero padded                     */
  int32_t* klens;
  double* vals;            /* n * nout                                      */
  int64_t n, cap;
  int32_t kmax, nout;
} Sink;

static int sink_push(Sink* s, const uint8_t* key, int klen, const double* v) {
  if (klen > s->kmax) return ORA_SPEC_ERROR;
  if (s->n == s->cap) {
    int64_t nc = s->cap ? s->cap * 2 : 1024;
    uint8_t* k = (uint8_t*)realloc(s->keys, (size_t)nc * s->kmax);
    int32_t* kl = (int32_t*)realloc(s->klens, (size_t)nc * sizeof(int32_t));
    double* vv = (double*)realloc(s->vals, (size_t)nc * s->nout * sizeof(double));
    if (!k || !kl || !vv) return ORA_NOMEM;
    s->keys = k; s->klens = kl; s->vals = vv; s->cap = nc;
  }
  memset(s->keys + (size_t)s->n * s->kmax, 0, (size_t)s->kmax);
  memcpy(s->keys + (size_t)s->n * s->kmax, key, (size_t)klen);
  s->klens[s->n] = klen;
  memcpy(s->vals + (size_t)s->n * s->nout, v, sizeof(double) * s->nout);
  s->n++;
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* engine context                                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
  ora_cfg cfg;
  ora_spec spec;
  Alloc alloc;
  ora_metrics m;
  Sink sink;
  int err;
} Ctx;

static void merge_fields(uint8_t* dst, const uint8_t* src, const ora_spec* sp) {  /* _kernels.py:148-159 */
  for (int j = 0; j < sp->nf; j++) {
    double a = rdf(dst + 8 * j), b = rdf(src + 8 * j);
    double r;
    if (sp->merge_ops[j] == MERGE_ADD) r = a + b;
    else if (sp->merge_ops[j] == MERGE_MIN) r = (a < b) ? a : b;
    else r = (a > b) ? a : b;
    wrf(dst + 8 * j, r);
  }
}

static int emit_final(Ctx* c, const uint8_t* key, int klen, const uint8_t* st) {  /* _kernels.py:175-229 */
  double v[64];
  for (int j = 0; j < c->spec.nout; j++) {
    int s = c->spec.finish_src[j];
    double x = rdf(st + 8 * s);
    if (c->spec.finish_ops[j] == FINISH_DIV) x = x / rdf(st + 8 * (s + 1));
    v[j] = x;
  }
  c->m.output_groups++;
  return sink_push(&c->sink, key, klen, v);
}

/* ------------------------------------------------------------------------ */
/* frame writer helper: append a state record into a buffer frame; when the */
/* frame is full it is flushed to the run (spill_frame, base.py:155-163)     */
/* ------------------------------------------------------------------------ */

static int spill_frame(Ctx* c, Run* r, int32_t fid) {
  Alloc* a = &c->alloc;
  r->records += count_records(fview(a, fid), a->p, c->spec.nf);
  int e = run_append(r, fview(a, fid), a->p);
  c->m.frames_written++;
  clear_frame(a, fid);
  return e;
}

static int buf_append(Ctx* c, int32_t fid, Run* r, const uint8_t* rec, int64_t need) {
  Alloc* a = &c->alloc;
  if (a->used[fid] + need > a->p) {
    int e = spill_frame(c, r, fid);
    if (e) return e;
  }
  memcpy(fview(a, fid) + a->used[fid], rec, (size_t)need);
  a->used[fid] += need;
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* chained hash table (hash_table.py:31-171, _kernels.py:298-392)            */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n_slots;
  uint32_t seed;
  int bloom_on;
  int64_t* slots;          /* absolute pool offsets, -1 empty              */
  uint8_t* bloom;
  int32_t* tfids; int32_t ntf; int32_t tcur;
  int32_t* ohfids; int32_t noh;
  int64_t stored_groups;
} Table;

/* plan_table (hash_table.py:31-45) */
static int plan_table(int32_t n_frames, int32_t p, double group_bytes, double slot_ratio,
                      int bloom, int64_t* cap, int64_t* n_slots) {
  if (n_frames < 2) return ORA_CAPACITY_EXCEEDED;
  double per_group = group_bytes + LINK_SIZE + slot_ratio * (SLOT_SIZE + (bloom ? 1 : 0));
  *cap = (int64_t)(n_frames * (double)p / per_group);
  int64_t ns = (int64_t)ceil(slot_ratio * (double)*cap);
  *n_slots = ns < 1 ? 1 : ns;
  return ORA_OK;
}

static int table_open(Ctx* c, Table* t, int32_t n_frames, int64_t n_slots, uint32_t seed, int bloom) {
  Alloc* a = &c->alloc;
  int64_t oh = (int64_t)ceil((double)(SLOT_SIZE * n_slots + (bloom ? n_slots : 0)) / a->p);
  memset(t, 0, sizeof(*t));
  if (n_frames - oh < 1) return ORA_CAPACITY_EXCEEDED;
  if (oh > a->nfree || n_frames - oh > a->nfree - oh) return ORA_INVALID_BUDGET;
  t->n_slots = n_slots; t->seed = seed; t->bloom_on = bloom;
  t->ohfids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(oh + 1));
  t->tfids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_frames - oh + 1));
  t->slots = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_slots);
  t->bloom = (uint8_t*)calloc((size_t)(bloom ? n_slots : 1), 1);
  if (!t->ohfids || !t->tfids || !t->slots || !t->bloom) return ORA_NOMEM;
  for (int64_t i = 0; i < oh; i++) t->ohfids[t->noh++] = frame_alloc(a);
  for (int64_t i = 0; i < n_frames - oh; i++) t->tfids[t->ntf++] = frame_alloc(a);
  for (int64_t i = 0; i < n_slots; i++) t->slots[i] = -1;
  return ORA_OK;
}

static void table_close(Ctx* c, Table* t) {
  for (int i = 0; i < t->noh; i++) frame_release(&c->alloc, t->ohfids[i]);
  for (int i = 0; i < t->ntf; i++) frame_release(&c->alloc, t->tfids[i]);
  free(t->ohfids); free(t->tfids); free(t->slots); free(t->bloom);
  memset(t, 0, sizeof(*t));
}

static void table_clear(Ctx* c, Table* t) {
  for (int64_t i = 0; i < t->n_slots; i++) t->slots[i] = -1;
  if (t->bloom_on) memset(t->bloom, 0, (size_t)t->n_slots);
  t->tcur = 0; t->stored_groups = 0;
  for (int i = 0; i < t->ntf; i++) clear_frame(&c->alloc, t->tfids[i]);
}

static inline uint8_t bloom_mask(uint32_t u) {  /* _kernels.py:388-390 */
  uint32_t hb = (u ^ (u >> 7)) * 0x2545F491u;
  return (uint8_t)((1u << (hb & 7)) | (1u << ((hb >> 13) & 7)));
}

static int64_t chain_find(Ctx* c, Table* t, int64_t s, const uint8_t* key, int klen) {  /* _kernels.py:298-309 */
  uint8_t* pool = c->alloc.pool;
  int64_t addr = t->slots[s];
  while (addr != -1) {
    const uint8_t* rec = pool + addr + LINK_SIZE;
    if (key_cmp(rec + KLEN_SIZE, rd16(rec), key, klen) == 0) return addr;
    addr = rdi(pool + addr);
  }
  return -1;
}

/* _table_append (_kernels.py:312-350): 0 ok, 1 full */
static int table_append(Ctx* c, Table* t, int64_t s, const uint8_t* key, int klen, const uint8_t* st) {
  Alloc* a = &c->alloc;
  int64_t need = LINK_SIZE + KLEN_SIZE + klen + FIELD_SIZE * c->spec.nf;
  int32_t cur = t->tcur, fid = t->tfids[cur];
  if (a->used[fid] + need > a->p) {
    int placed = 0;
    while (cur + 1 < t->ntf) {
      cur++; fid = t->tfids[cur];
      if (a->used[fid] + need <= a->p) { t->tcur = cur; placed = 1; break; }
    }
    if (!placed) {
      fid = -1;
      for (int i = 0; i < t->ntf; i++)
        if (a->used[t->tfids[i]] + need <= a->p) { fid = t->tfids[i]; break; }
      if (fid == -1) return 1;
    }
  }
  int64_t base = (int64_t)fid * a->p + a->used[fid];
  uint8_t* b = a->pool + base;
  wri(b, t->slots[s]);
  wr16(b + LINK_SIZE, (uint16_t)klen);
  memcpy(b + LINK_SIZE + KLEN_SIZE, key, (size_t)klen);
  memcpy(b + LINK_SIZE + KLEN_SIZE + klen, st, (size_t)FIELD_SIZE * c->spec.nf);
  a->used[fid] += need;
  t->slots[s] = base;
  return 0;
}

/* insert-or-aggregate one record (_kernels.py:353-392): 0 ok, 1 TABLE_FULL */
static int table_insert(Ctx* c, Table* t, const uint8_t* key, int klen, const uint8_t* st) {
  uint32_t u = ora_hash_bytes(key, klen, t->seed);
  int64_t s = (int64_t)(u % (uint64_t)t->n_slots);
  int64_t addr = chain_find(c, t, s, key, klen);
  if (addr != -1) {
    merge_fields(c->alloc.pool + addr + LINK_SIZE + KLEN_SIZE + klen, st, &c->spec);
    return 0;
  }
  if (table_append(c, t, s, key, klen, st)) return 1;
  t->stored_groups++;
  if (t->bloom_on) t->bloom[s] |= bloom_mask(u);
  return 0;
}

/* visit groups in slot-chain order (k_flush_slots, _kernels.py:473-519) */
typedef int (*group_fn)(Ctx*, void*, const uint8_t* key, int klen, const uint8_t* st);
static int table_visit(Ctx* c, Table* t, group_fn fn, void* arg) {
  uint8_t* pool = c->alloc.pool;
  for (int64_t s = 0; s < t->n_slots; s++) {
    int64_t addr = t->slots[s];
    while (addr != -1) {
      const uint8_t* rec = pool + addr + LINK_SIZE;
      int kl = rd16(rec);
      int e = fn(c, arg, rec + KLEN_SIZE, kl, rec + KLEN_SIZE + kl);
      if (e) return e;
      addr = rdi(pool + addr);
    }
  }
  return ORA_OK;
}
static int visit_emit_final(Ctx* c, void* arg, const uint8_t* key, int klen, const uint8_t* st) {
  (void)arg; return emit_final(c, key, klen, st);
}
typedef struct { int32_t stage; Run* run; } SpillArg;
static int visit_spill_state(Ctx* c, void* arg, const uint8_t* key, int klen, const uint8_t* st) {
  SpillArg* sa = (SpillArg*)arg;
  uint8_t rec[KLEN_SIZE + 65536 + 8 * 64];
  wr16(rec, (uint16_t)klen);
  memcpy(rec + KLEN_SIZE, key, (size_t)klen);
  memcpy(rec + KLEN_SIZE + klen, st, (size_t)FIELD_SIZE * c->spec.nf);
  return buf_append(c, sa->stage, sa->run, rec, KLEN_SIZE + klen + FIELD_SIZE * c->spec.nf);
}

/* ------------------------------------------------------------------------ */
/* planning (hybrid.py:89-163, run_store.py:222-246)                         */
/* ------------------------------------------------------------------------ */

double ora_fudge_factor(double group_bytes, double extra, double slot_ratio, int bloom) {
  double per_group = group_bytes + LINK_SIZE + slot_ratio * (SLOT_SIZE + (bloom ? 1 : 0));
  return per_group * extra / (group_bytes > 1e-300 ? group_bytes : 1e-300);
}

int ora_plan_partitions(double gf, int32_t M, int32_t* P) {
  if (M < 3) return ORA_INVALID_BUDGET;
  if (gf <= M) { *P = 0; return ORA_OK; }
  double p = ceil((gf - M) / (M - 2));
  if (p > M - 2) p = M - 2;
  if (p < 1) p = 1;
  *P = (int32_t)p;
  return ORA_OK;
}

typedef struct { int32_t M, P, grace_levels; double F, r_res, r_spill, gf; } Plan;

int ora_plan_hybrid(double G, int32_t M, double F, Plan* pl) {
  if (M < 4) return ORA_INVALID_BUDGET;
  double gf = G * F;
  int levels = 0;
  if (gf >= (double)M * M) {
    double need = gf;
    while (need >= (double)M * M) { levels++; need = gf / pow((double)(M - 1), levels); }
  }
  int32_t P;
  int e = ora_plan_partitions(gf, M, &P);
  if (e) return e;
  pl->M = M; pl->P = P; pl->F = F; pl->gf = gf; pl->grace_levels = levels;
  if (P == 0) { pl->r_res = 1.0; pl->r_spill = 0.0; }
  else { pl->r_res = (double)(M - P) / ((double)(M - P) + (double)M * P); pl->r_spill = (1.0 - pl->r_res) / P; }
  return ORA_OK;
}

int ora_merge_rounds(int64_t n_runs, int64_t fan_in) {  /* len(plan_merge_rounds(...)) */
  if (n_runs <= 1) return n_runs == 1 ? 1 : 0;
  int64_t q = n_runs; int rounds = 0;
  while (q > fan_in) {
    int64_t z = q > 2 * fan_in - 1 ? fan_in : q - fan_in + 1;
    q = q - z + 1; rounds++;
  }
  return rounds + 1;
}

int ora_sort_merge_levels(double input_frames, int32_t M) {
  int64_t fan = M - 1 > 2 ? M - 1 : 2;
  int64_t runs = (int64_t)ceil(input_frames / (double)fan);
  if (runs < 1) runs = 1;
  return ora_merge_rounds(runs, fan);
}

/* 1 = fallback to hash_sort, 0 = recurse */
int ora_fallback(double run_frames, double parent_frames, int level, int sort_levels) {
  if (parent_frames > 0 && run_frames > 0 && run_frames > 0.8 * parent_frames) return 1;
  if (level > sort_levels) return 1;
  return 0;
}

void ora_make_cuts(double r_res, int32_t P, int64_t* cuts) {
  if (P == 0) { cuts[0] = HASH_SPACE; return; }
  int64_t c0 = (int64_t)(r_res * (double)HASH_SPACE);
  if (c0 < 1) c0 = 1;
  int64_t rest = HASH_SPACE - c0;
  for (int i = 0; i < P; i++) cuts[i + 1] = c0 + (rest * (i + 1)) / P;
  cuts[0] = c0; cuts[P] = HASH_SPACE;
}

static int part_of(uint32_t u, const int64_t* cuts, int n) {  /* _kernels.py:134-145 */
  int lo = 0, hi = n;
  while (lo < hi) { int mid = (lo + hi) >> 1; if ((int64_t)u < cuts[mid]) hi = mid; else lo = mid + 1; }
  return lo;
}

/* ------------------------------------------------------------------------ */
/* record sources: a list of runs, or the caller's frames                    */
/* ------------------------------------------------------------------------ */

typedef struct {
  const uint8_t* frames;   /* contiguous frames                             */
  int64_t nframes;
  int32_t p;
} Src;

typedef struct {
  double R, R_t, G, G_t;
} Stats;

typedef int (*rec_fn)(Ctx*, void*, const uint8_t* rec, int klen, int64_t need);

static int src_foreach(Ctx* c, const Src* s, rec_fn fn, void* arg) {
  for (int64_t f = 0; f < s->nframes; f++) {
    const uint8_t* fr = s->frames + (size_t)f * s->p;
    int64_t off = 0;
    while (off <= s->p - KLEN_SIZE) {
      int kl = rd16(fr + off);
      if (!kl) break;
      int64_t need = KLEN_SIZE + kl + FIELD_SIZE * c->spec.nf;
      int e = fn(c, arg, fr + off, kl, need);
      if (e) return e;
      off += need;
    }
  }
  return ORA_OK;
}

static double group_bytes_of(const Ctx* c, const Stats* st) {  /* base.py:141-147 */
  double floor_b = KLEN_SIZE + 1 + FIELD_SIZE * c->spec.nf;
  if (st->G_t > 0 && st->G > 0) {
    double g = st->G * c->cfg.frame_size / st->G_t;
    return g > floor_b ? g : floor_b;
  }
  return KLEN_SIZE + 16 + FIELD_SIZE * c->spec.nf;
}

static int run_operator_level(Ctx* c, int algo, const Stats* st, int level, int sort_levels,
                              int grace_depth, const Src* src);

/* ------------------------------------------------------------------------ */
/* hash_sort (hash_sort.py:20-115)                                           */
/* ------------------------------------------------------------------------ */

typedef struct { const uint8_t* rec; uint32_t slot; int klen; int run; int64_t seq; } MRec;

static int mrec_cmp(const void* A, const void* B) {
  const MRec* a = (const MRec*)A; const MRec* b = (const MRec*)B;
  if (a->slot != b->slot) return a->slot < b->slot ? -1 : 1;
  int k = key_cmp(a->rec + KLEN_SIZE, a->klen, b->rec + KLEN_SIZE, b->klen);
  if (k) return k;
  if (a->seq != b->seq) return a->seq < b->seq ? -1 : 1;
  return 0;
}

/* gather every record of a set of runs into an index array */
static int gather_runs(Ctx* c, Run* runs, int nruns, MRec** out, int64_t* n_out,
                       int slot_mode, uint32_t seed, int64_t H) {
  int64_t total = 0;
  for (int r = 0; r < nruns; r++) total += runs[r].records;
  MRec* m = (MRec*)malloc(sizeof(MRec) * (size_t)(total + 1));
  if (!m) return ORA_NOMEM;
  int64_t n = 0;
  for (int r = 0; r < nruns; r++) {
    for (int64_t f = 0; f < runs[r].frames; f++) {
      const uint8_t* fr = runs[r].data + (size_t)f * runs[r].p;
      int64_t off = 0;
      while (off <= runs[r].p - KLEN_SIZE) {
        int kl = rd16(fr + off);
        if (!kl) break;
        m[n].rec = fr + off; m[n].klen = kl; m[n].run = r; m[n].seq = n;
        m[n].slot = slot_mode ? (uint32_t)(ora_hash_bytes(fr + off + KLEN_SIZE, kl, seed) % (uint64_t)H) : 0;
        n++;
        off += KLEN_SIZE + kl + FIELD_SIZE * c->spec.nf;
      }
    }
    c->m.frames_read += runs[r].frames;
  }
  *out = m; *n_out = n;
  return ORA_OK;
}

/* fold an ordered record array and emit finalized groups (k_fold_sorted + k_fold_finish) */
static int fold_emit(Ctx* c, MRec* m, int64_t n) {
  uint8_t st[8 * 64];
  int64_t i = 0;
  while (i < n) {
    memcpy(st, m[i].rec + KLEN_SIZE + m[i].klen, (size_t)8 * c->spec.nf);
    int64_t j = i + 1;
    while (j < n && key_cmp(m[j].rec + KLEN_SIZE, m[j].klen, m[i].rec + KLEN_SIZE, m[i].klen) == 0) {
      merge_fields(st, m[j].rec + KLEN_SIZE + m[j].klen, &c->spec);
      j++;
    }
    int e = emit_final(c, m[i].rec + KLEN_SIZE, m[i].klen, st);
    if (e) return e;
    i = j;
  }
  return ORA_OK;
}

typedef struct { Table t; Run* runs; int nruns, caprun; } HS;

static int hs_flush_to_run(Ctx* c, HS* h) {  /* hash_sort.py:51-78 */
  if (h->nruns == h->caprun) {
    int nc = h->caprun ? h->caprun * 2 : 4;
    Run* nr = (Run*)realloc(h->runs, sizeof(Run) * (size_t)nc);
    if (!nr) return ORA_NOMEM;
    memset(nr + h->caprun, 0, sizeof(Run) * (size_t)(nc - h->caprun));
    h->runs = nr; h->caprun = nc;
  }
  Run* r = &h->runs[h->nruns++];
  int32_t out = frame_alloc(&c->alloc);
  if (out < 0) return ORA_INVALID_BUDGET;
  /* per-slot key-sorted order: collect the table records and sort by (slot, key) */
  int64_t n = h->t.stored_groups, k = 0;
  MRec* m = (MRec*)malloc(sizeof(MRec) * (size_t)(n + 1));
  if (!m) return ORA_NOMEM;
  uint8_t* pool = c->alloc.pool;
  for (int64_t s = 0; s < h->t.n_slots; s++) {
    int64_t addr = h->t.slots[s];
    while (addr != -1) {
      m[k].rec = pool + addr + LINK_SIZE; m[k].klen = rd16(m[k].rec);
      m[k].slot = (uint32_t)s; m[k].seq = k; k++;
      addr = rdi(pool + addr);
    }
  }
  qsort(m, (size_t)k, sizeof(MRec), mrec_cmp);
  SpillArg sa = {out, r};
  int e = 0;
  for (int64_t i = 0; i < k && !e; i++)
    e = visit_spill_state(c, &sa, m[i].rec + KLEN_SIZE, m[i].klen, m[i].rec + KLEN_SIZE + m[i].klen);
  free(m);
  if (!e && c->alloc.used[out] > 0) e = spill_frame(c, r, out);
  frame_release(&c->alloc, out);
  r->records = k;
  table_clear(c, &h->t);
  return e;
}

static int hs_push(Ctx* c, void* arg, const uint8_t* rec, int klen, int64_t need) {
  (void)need;
  HS* h = (HS*)arg;
  for (;;) {
    if (!table_insert(c, &h->t, rec + KLEN_SIZE, klen, rec + KLEN_SIZE + klen)) return ORA_OK;
    int e = hs_flush_to_run(c, h);
    if (e) return e;
  }
}

static int op_hash_sort(Ctx* c, const Stats* st, int level, const Src* src) {
  int32_t M = c->cfg.memory_frames;
  if (M < 3) return ORA_INVALID_BUDGET;
  HS h; memset(&h, 0, sizeof(h));
  uint32_t slot_seed = ora_mix_seed(c->cfg.seed, 0x45 + ((uint64_t)level << 8));
  int64_t cap, ns;
  int e = plan_table(M - 1, c->cfg.frame_size, group_bytes_of(c, st), c->cfg.slot_ratio, 0, &cap, &ns);
  if (e) return e;
  e = table_open(c, &h.t, M - 1, ns, slot_seed, 0);
  if (e) return e;
  e = src_foreach(c, src, hs_push, &h);
  if (e) return e;
  if (h.nruns == 0) {
    e = table_visit(c, &h.t, visit_emit_final, NULL);
    table_close(c, &h.t);
    return e;
  }
  if (h.t.stored_groups > 0) { e = hs_flush_to_run(c, &h); if (e) return e; }
  int64_t H = h.t.n_slots;
  table_close(c, &h.t);
  /* MergeDriver(ORDER_SLOT_KEY, fold) — one k-way pass (see header) */
  MRec* m; int64_t n;
  e = gather_runs(c, h.runs, h.nruns, &m, &n, 1, slot_seed, H);
  if (e) return e;
  qsort(m, (size_t)n, sizeof(MRec), mrec_cmp);
  e = fold_emit(c, m, n);
  free(m);
  for (int r = 0; r < h.nruns; r++) run_free(&h.runs[r]);
  free(h.runs);
  return e;
}

/* ------------------------------------------------------------------------ */
/* sort_based (sort_based.py:24-211)                                         */
/* ------------------------------------------------------------------------ */

static int op_sort_based(Ctx* c, const Src* src) {
  int32_t M = c->cfg.memory_frames;
  if (M < 3) return ORA_INVALID_BUDGET;
  Run all; memset(&all, 0, sizeof(all));
  all.data = (uint8_t*)src->frames; all.frames = src->nframes; all.p = src->p;
  int64_t tot = 0;
  for (int64_t f = 0; f < src->nframes; f++) tot += count_records(src->frames + (size_t)f * src->p, src->p, c->spec.nf);
  all.records = tot;
  MRec* m; int64_t n;
  int e = gather_runs(c, &all, 1, &m, &n, 0, 0, 1);
  c->m.frames_read -= src->nframes;  /* input scan is not run traffic */
  if (e) return e;
  if (c->cfg.input_sorted) {  /* k_stream_fold order contract (_kernels.py:655-694) */
    for (int64_t i = 1; i < n; i++)
      if (key_cmp(m[i].rec + KLEN_SIZE, m[i].klen, m[i - 1].rec + KLEN_SIZE, m[i - 1].klen) < 0) {
        free(m); return ORA_ORDER_ERROR;
      }
  } else {
    qsort(m, (size_t)n, sizeof(MRec), mrec_cmp);  /* slot == 0: key then arrival order */
  }
  e = fold_emit(c, m, n);
  free(m);
  return e;
}

/* ------------------------------------------------------------------------ */
/* hybrid operators: pre_partitioning, original_hh, grace                    */
/* ------------------------------------------------------------------------ */

typedef struct {
  int level, sort_levels, grace_depth, algo;
  Stats st;
  uint32_t part_seed, slot_seed, spill_seed;
  Plan plan;
  /* table state */
  Table t; int table_live;
  int mode;                /* 0 fill/table 1 probe/route 2 grace           */
  int32_t P, nspill, reserved;
  int32_t* out;            /* buffer frame per spill partition, -1 none    */
  int32_t nout;
  Run* runs;               /* one run per partition id                    */
  int64_t* cuts; int32_t ncuts;
  int64_t stored_at_cut;
} HY;

static int hy_child(Ctx* c, HY* h, Run* run, double gest);

static Stats effective_stats(Ctx* c, const Stats* st, int level) {  /* hybrid.py:193-203 */
  Stats s = *st;
  if (level == 0 && c->cfg.group_estimate >= 0) {
    double b_g = group_bytes_of(c, st);
    double gt = c->cfg.group_estimate > 1.0 ? c->cfg.group_estimate : 1.0;
    s.R_t = st->R_t > gt ? st->R_t : gt;
    s.G = gt * b_g / c->cfg.frame_size;
    s.G_t = gt;
  }
  return s;
}

static int hy_pp_push(Ctx* c, void* arg, const uint8_t* rec, int klen, int64_t need) {
  HY* h = (HY*)arg;
  const uint8_t* key = rec + KLEN_SIZE;
  const uint8_t* st = key + klen;
  if (h->mode == 0) {                                   /* fill */
    if (!table_insert(c, &h->t, key, klen, st)) return ORA_OK;
    /* _freeze (hybrid.py:545-552) */
    if (h->P == 0) { h->out[0] = h->reserved; h->nspill = 1; }
    h->mode = 1;
  }
  /* k_pp_probe (_kernels.py:917-962) */
  uint32_t u = ora_hash_bytes(key, klen, h->t.seed);
  int64_t s = (int64_t)(u % (uint64_t)h->t.n_slots);
  int passed = 1;
  if (h->t.bloom_on) { uint8_t mk = bloom_mask(u); if ((h->t.bloom[s] & mk) != mk) passed = 0; }
  int64_t addr = passed ? chain_find(c, &h->t, s, key, klen) : -1;
  if (addr != -1) { merge_fields(c->alloc.pool + addr + LINK_SIZE + KLEN_SIZE + klen, st, &c->spec); return ORA_OK; }
  int pidx = (int)(ora_hash_bytes(key, klen, h->spill_seed) % (uint32_t)h->nspill);
  c->m.spilled_records++;
  return buf_append(c, h->out[pidx], &h->runs[pidx], rec, need);
}

static int hy_hh_push(Ctx* c, void* arg, const uint8_t* rec, int klen, int64_t need) {
  HY* h = (HY*)arg;
  const uint8_t* key = rec + KLEN_SIZE;
  uint32_t up = ora_hash_bytes(key, klen, h->part_seed);
  int pidx = part_of(up, h->cuts, h->ncuts);
  if (pidx == 0 && h->mode == 0 && h->table_live) {
    if (!table_insert(c, &h->t, key, klen, key + klen)) return ORA_OK;
    /* _overflow (hybrid.py:431-451) */
    int32_t stage;
    if (h->P >= 1) {
      stage = h->out[1];
      if (c->alloc.used[stage] > 0) { int e = spill_frame(c, &h->runs[1], stage); if (e) return e; }
    } else stage = h->reserved;
    SpillArg sa = {stage, &h->runs[0]};
    int e = table_visit(c, &h->t, visit_spill_state, &sa);
    if (e) return e;
    if (c->alloc.used[stage] > 0) { e = spill_frame(c, &h->runs[0], stage); if (e) return e; }
    h->stored_at_cut = h->t.stored_groups;
    table_close(c, &h->t); h->table_live = 0;
    if (h->P >= 1) { int32_t b0 = frame_alloc(&c->alloc); if (b0 < 0) return ORA_INVALID_BUDGET; h->out[0] = b0; }
    else { h->out[0] = stage; h->reserved = -1; }
    h->mode = 1;
  }
  c->m.spilled_records++;
  return buf_append(c, h->out[pidx], &h->runs[pidx], rec, need);
}

static int hy_free(HY* h) {
  if (h->runs) for (int i = 0; i < h->nout; i++) run_free(&h->runs[i]);
  free(h->runs); free(h->out); free(h->cuts);
  return 0;
}

/* _drain_runs for one (run, estimate) item (hybrid.py:244-277) */
static int hy_child(Ctx* c, HY* h, Run* run, double gest) {
  double frames = (double)run->frames, records = (double)run->records;
  if (records <= 0) gest = 0.0;
  else gest = gest < records ? (gest > 1.0 ? gest : 1.0) : (records > 1.0 ? records : 1.0);
  int fb = ora_fallback(frames, h->st.R, h->level + 1, h->sort_levels);
  Stats cs = {frames, records, gest * group_bytes_of(c, &h->st) / c->cfg.frame_size, gest};
  Src s = {run->data, run->frames, c->cfg.frame_size};
  c->m.frames_read += run->frames;
  int e;
  if (fb) { c->m.fallbacks++; e = run_operator_level(c, ALGO_HASH_SORT, &cs, h->level + 1, h->sort_levels, 0, &s); }
  else e = run_operator_level(c, h->algo, &cs, h->level + 1, h->sort_levels,
                              h->grace_depth + (h->mode == 2 ? 1 : 0), &s);
  run_free(run);
  return e;
}

static int op_hybrid(Ctx* c, int algo, const Stats* st_in, int level, int sort_levels, int grace_depth,
                     const Src* src) {
  HY h; memset(&h, 0, sizeof(h));
  h.algo = algo; h.level = level; h.grace_depth = grace_depth; h.reserved = -1;
  uint64_t lv = (uint64_t)level << 8;
  h.part_seed = ora_mix_seed(c->cfg.seed, 0x11 + lv);
  h.slot_seed = ora_mix_seed(c->cfg.seed, 0x22 + lv);
  h.spill_seed = ora_mix_seed(c->cfg.seed, 0x33 + lv);
  int32_t M = c->cfg.memory_frames, p = c->cfg.frame_size;
  h.st = effective_stats(c, st_in, level);
  h.sort_levels = sort_levels >= 0 ? sort_levels : ora_sort_merge_levels(h.st.R, M);
  double b_g = group_bytes_of(c, &h.st);
  int pp = algo == ALGO_PRE_PARTITIONING;
  double F = ora_fudge_factor(b_g, c->cfg.fudge, c->cfg.slot_ratio, pp);
  int e = ora_plan_hybrid(h.st.G, M, F, &h.plan);
  if (e) return e;
  if (level > c->m.recursion_depth) c->m.recursion_depth = level;
  Src* s = (Src*)src;
  if (h.plan.grace_levels) {                           /* _grace_open (hybrid.py:281-293) */
    int32_t n = M - 1;
    h.mode = 2; h.nout = n;
    h.out = (int32_t*)malloc(sizeof(int32_t) * n);
    h.runs = (Run*)calloc((size_t)n, sizeof(Run));
    h.cuts = (int64_t*)malloc(sizeof(int64_t) * n); h.ncuts = n;
    for (int i = 0; i < n; i++) { h.cuts[i] = (HASH_SPACE * (i + 1)) / n; h.out[i] = frame_alloc(&c->alloc); if (h.out[i] < 0) return ORA_INVALID_BUDGET; }
    h.cuts[n - 1] = HASH_SPACE;
    if (grace_depth + 1 > c->m.grace_levels) c->m.grace_levels = grace_depth + 1;
    h.P = n;
    /* k_hh_push with table_on = 0 */
    e = src_foreach(c, s, hy_hh_push, &h);
    if (e) return e;
    for (int i = 0; i < n; i++) {
      if (c->alloc.used[h.out[i]] > 0) { e = spill_frame(c, &h.runs[i], h.out[i]); if (e) return e; }
      frame_release(&c->alloc, h.out[i]);
    }
    double gest = h.st.G_t / n;
    for (int i = 0; i < n; i++) if (h.runs[i].frames) c->m.spilled_partitions++;
    for (int i = 0; i < n && !e; i++) if (h.runs[i].frames) e = hy_child(c, &h, &h.runs[i], gest);
    hy_free(&h);
    return e;
  }
  h.P = h.plan.P;
  int64_t cap, ns;
  if (pp) {                                            /* PrePartitioning.open (hybrid.py:488-516) */
    if (h.P >= 1) {
      int bloom = h.P > 1;
      e = plan_table(M - h.P, p, b_g, c->cfg.slot_ratio, bloom, &cap, &ns); if (e) return e;
      e = table_open(c, &h.t, M - h.P, ns, h.slot_seed, bloom); if (e) return e;
      h.nout = h.P; h.nspill = h.P;
      h.out = (int32_t*)malloc(sizeof(int32_t) * h.nout);
      for (int i = 0; i < h.P; i++) { h.out[i] = frame_alloc(&c->alloc); if (h.out[i] < 0) return ORA_INVALID_BUDGET; }
    } else {
      e = plan_table(M - 1, p, b_g, c->cfg.slot_ratio, 0, &cap, &ns); if (e) return e;
      e = table_open(c, &h.t, M - 1, ns, h.slot_seed, 0); if (e) return e;
      h.reserved = frame_alloc(&c->alloc); if (h.reserved < 0) return ORA_INVALID_BUDGET;
      h.nout = 1; h.nspill = 0;
      h.out = (int32_t*)malloc(sizeof(int32_t)); h.out[0] = -1;
    }
    h.table_live = 1;
    h.runs = (Run*)calloc((size_t)h.nout, sizeof(Run));
    e = src_foreach(c, s, hy_pp_push, &h);
    if (e) return e;
    /* close (hybrid.py:554-576) */
    for (int i = 0; i < h.nspill; i++)
      if (c->alloc.used[h.out[i]] > 0) { e = spill_frame(c, &h.runs[i], h.out[i]); if (e) return e; }
    e = table_visit(c, &h.t, visit_emit_final, NULL); if (e) return e;
    int64_t resident = h.t.stored_groups;
    table_close(c, &h.t);
    if (h.P >= 1) for (int i = 0; i < h.P; i++) frame_release(&c->alloc, h.out[i]);
    else frame_release(&c->alloc, h.reserved);
    int nr = 0;
    for (int i = 0; i < h.nout; i++) if (h.runs[i].frames) nr++;
    c->m.spilled_partitions += nr;
    double remaining = h.st.G_t - (double)resident;
    if (remaining < nr) remaining = nr;
    double gest = remaining / (h.nspill > 1 ? h.nspill : 1);
    for (int i = 0; i < h.nout && !e; i++) if (h.runs[i].frames) e = hy_child(c, &h, &h.runs[i], gest);
    hy_free(&h);
    return e;
  }
  /* OriginalHybridHash.open (hybrid.py:363-390) */
  if (h.P >= 1) {
    e = plan_table(M - h.P, p, b_g, c->cfg.slot_ratio, 0, &cap, &ns); if (e) return e;
    e = table_open(c, &h.t, M - h.P, ns, h.slot_seed, 0); if (e) return e;
    h.nout = h.P + 1;
    h.out = (int32_t*)malloc(sizeof(int32_t) * h.nout); h.out[0] = -1;
    for (int i = 0; i < h.P; i++) { h.out[i + 1] = frame_alloc(&c->alloc); if (h.out[i + 1] < 0) return ORA_INVALID_BUDGET; }
    h.cuts = (int64_t*)malloc(sizeof(int64_t) * (h.P + 1)); h.ncuts = h.P + 1;
    ora_make_cuts(h.plan.r_res, h.P, h.cuts);
  } else {
    e = plan_table(M - 1, p, b_g, c->cfg.slot_ratio, 0, &cap, &ns); if (e) return e;
    e = table_open(c, &h.t, M - 1, ns, h.slot_seed, 0); if (e) return e;
    h.reserved = frame_alloc(&c->alloc); if (h.reserved < 0) return ORA_INVALID_BUDGET;
    h.nout = 1; h.out = (int32_t*)malloc(sizeof(int32_t)); h.out[0] = -1;
    h.cuts = (int64_t*)malloc(sizeof(int64_t)); h.ncuts = 1; h.cuts[0] = HASH_SPACE;
  }
  h.table_live = 1;
  h.runs = (Run*)calloc((size_t)h.nout, sizeof(Run));
  e = src_foreach(c, s, hy_hh_push, &h);
  if (e) return e;
  /* close (hybrid.py:453-478) */
  for (int i = 0; i < h.nout; i++)
    if (h.out[i] >= 0 && c->alloc.used[h.out[i]] > 0) { e = spill_frame(c, &h.runs[i], h.out[i]); if (e) return e; }
  if (h.table_live) {
    e = table_visit(c, &h.t, visit_emit_final, NULL); if (e) return e;
    table_close(c, &h.t); h.table_live = 0;
  }
  for (int i = 0; i < h.nout; i++) if (h.out[i] >= 0) frame_release(&c->alloc, h.out[i]);
  if (h.P == 0 && h.mode == 0) frame_release(&c->alloc, h.reserved);
  int nr = 0;
  for (int i = 0; i < h.nout; i++) if (h.runs[i].frames) nr++;
  c->m.spilled_partitions += nr;
  for (int i = 0; i < h.nout && !e; i++) {
    if (!h.runs[i].frames) continue;
    double est;
    if (i == 0) {
      double suffix = (double)h.runs[0].records - (double)h.stored_at_cut;
      if (suffix < 0) suffix = 0;
      double ratio = h.st.G_t / (h.st.R_t > 1.0 ? h.st.R_t : 1.0);
      est = (double)h.stored_at_cut + suffix * ratio;
    } else est = h.plan.r_spill * h.st.G_t;
    e = hy_child(c, &h, &h.runs[i], est);
  }
  hy_free(&h);
  return e;
}

static int run_operator_level(Ctx* c, int algo, const Stats* st, int level, int sort_levels,
                              int grace_depth, const Src* src) {
  if (level > c->m.recursion_depth) c->m.recursion_depth = level;
  switch (algo) {
    case ALGO_HASH_SORT: return op_hash_sort(c, st, level, src);
    case ALGO_SORT_BASED: return op_sort_based(c, src);
    case ALGO_ORIGINAL_HH:
    case ALGO_PRE_PARTITIONING: return op_hybrid(c, algo, st, level, sort_levels, grace_depth, src);
    default: return ORA_SPEC_ERROR;
  }
}

/* ------------------------------------------------------------------------ */
/* public entry                                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n;               /* groups                                        */
  int32_t kmax, nout;
  uint8_t* keys;           /* n * kmax zero padded                          */
  int32_t* klens;
  double* vals;            /* n * nout                                      */
} ora_result;

/*
 * Run one operator over caller frames (state records, fixed frame size).
 * Mirrors run_operator(OPERATORS[algo](ctx, stats), FrameSource.from_frames)
 * (base.py:185-217, conftest.py:117-139) including the leak check.
 */
int ora_run(const ora_cfg* cfg, const ora_spec* spec, const uint8_t* frames, int64_t nframes,
            int32_t kmax, ora_result* res, ora_metrics* met) {
  Ctx c; memset(&c, 0, sizeof(c));
  c.cfg = *cfg; c.spec = *spec;
  if (spec->nf < 1 || spec->nf > 64 || spec->nout < 1 || spec->nout > 64) return ORA_SPEC_ERROR;
  if (cfg->memory_frames < 2) return ORA_INVALID_BUDGET;  /* OpContext (base.py:77-79) */
  int e = alloc_init(&c.alloc, cfg->memory_frames, cfg->frame_size);
  if (e) return e;
  c.sink.kmax = kmax; c.sink.nout = spec->nout;
  Src src = {frames, nframes, cfg->frame_size};
  Stats st = {cfg->R, cfg->R_t, cfg->G, cfg->G_t};
  e = run_operator_level(&c, cfg->algo, &st, 0, -1, 0, &src);
  c.m.high_water = c.alloc.high_water;
  if (!e && outstanding(&c.alloc) != 0) e = 9;  /* AggregationError: leaked frames */
  alloc_free(&c.alloc);
  if (met) *met = c.m;
  res->n = c.sink.n; res->kmax = kmax; res->nout = spec->nout;
  res->keys = c.sink.keys; res->klens = c.sink.klens; res->vals = c.sink.vals;
  return e;
}

void ora_result_free(ora_result* r) {
  free(r->keys); free(r->klens); free(r->vals);
  memset(r, 0, sizeof(*r));
}
