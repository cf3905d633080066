/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Numeric CPU restatement of the reference executor
 *   hiercoll::run_transfers / execute_plan   (proj/src/engine.cpp:285-347)
 * used as the parity oracle for the device executor and, multithreaded,
 * as the CPU baseline timed by bench.py. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may call it.
 *
 * What it restates, line by line:
 *   engine.cpp:288-293  transfers run in (slot, id) order (stable sort);
 *   engine.cpp:309-326  per element: read src (reading a never-written
 *                       element is UninitializedRead), then either
 *                       dst = v (copy) or dst = fold(op, dst, v) (reduce;
 *                       the accumulator must already be written).
 * The reference folds *symbols*; here the symbols are numbers, so the
 * arithmetic of one fold is fixed explicitly (same rules as the device):
 *   f32 / f64 sum   one IEEE add, no contraction (-ffp-contract=off)
 *   bf16 / f16 sum  widen to f32, add, round-to-nearest-even to the type
 *   integer sum     wrapping add
 *   max             (acc < v) ? v : acc
 * Input generator (shared with the device fill kernel):
 *   h = splitmix64(seed ^ (rank << 40) ^ index)
 *   f32 = ((h >> 40) * 2^-24) * 2 - 1;  bf16/f16 = RNE(f32);  f64 = f32
 *   i32/i64 = (h >> 33) & 0xFFFF;        u8 = h >> 56
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_F32 = 0, OR_BF16 = 1, OR_F16 = 2, OR_I32 = 3, OR_I64 = 4, OR_F64 = 5, OR_U8 = 6 };

/* Same field layout as hc_transfer in include/hiccl.h, declared
 * independently so the oracle shares no code with the product. */
typedef struct {
  int32_t id, src, dst, src_buf, dst_buf;
  int32_t reduce, op, stage, slot, channel, stripe, level, step, n_deps;
  int64_t src_off, dst_off, count;
} or_transfer;

static int esize_of(int dt) {
  switch (dt) {
    case OR_F32: case OR_I32: return 4;
    case OR_BF16: case OR_F16: return 2;
    case OR_I64: case OR_F64: return 8;
    case OR_U8: return 1;
  }
  return 0;
}

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static float f16_to_f32(uint16_t h) {
  _Float16 x;
  memcpy(&x, &h, 2);
  return (float)x;
}

static uint16_t f32_to_f16_rne(float f) {
  _Float16 x = (_Float16)f; /* IEEE conversion, round-to-nearest-even */
  uint16_t h;
  memcpy(&h, &x, 2);
  return h;
}

void oracle_fill(void* out, int64_t n, int dtype, uint64_t seed, int rank, int64_t index_base) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t h = splitmix64(seed ^ ((uint64_t)rank << 40) ^ (uint64_t)(index_base + i));
    const float f = ((float)(h >> 40) * 5.9604644775390625e-08f) * 2.0f - 1.0f;
    switch (dtype) {
      case OR_F32: ((float*)out)[i] = f; break;
      case OR_BF16: ((uint16_t*)out)[i] = f32_to_bf16_rne(f); break;
      case OR_F16: ((uint16_t*)out)[i] = f32_to_f16_rne(f); break;
      case OR_I32: ((int32_t*)out)[i] = (int32_t)((h >> 33) & 0xFFFF); break;
      case OR_I64: ((int64_t*)out)[i] = (int64_t)((h >> 33) & 0xFFFF); break;
      case OR_F64: ((double*)out)[i] = (double)f; break;
      case OR_U8: ((uint8_t*)out)[i] = (uint8_t)(h >> 56); break;
    }
  }
}

/* One fold of the reference's reduce-into (engine.cpp:316-322), numeric. */
static void fold_range(int dt, int op, void* dst, const void* src, int64_t n) {
  int64_t i;
  switch (dt) {
    case OR_F32: {
      float* d = dst; const float* s = src;
      if (op == 0) for (i = 0; i < n; ++i) d[i] = d[i] + s[i];
      else for (i = 0; i < n; ++i) d[i] = (d[i] < s[i]) ? s[i] : d[i];
      break;
    }
    case OR_F64: {
      double* d = dst; const double* s = src;
      if (op == 0) for (i = 0; i < n; ++i) d[i] = d[i] + s[i];
      else for (i = 0; i < n; ++i) d[i] = (d[i] < s[i]) ? s[i] : d[i];
      break;
    }
    case OR_BF16: {
      uint16_t* d = dst; const uint16_t* s = src;
      for (i = 0; i < n; ++i) {
        const float a = bf16_to_f32(d[i]), b = bf16_to_f32(s[i]);
        if (op == 0) d[i] = f32_to_bf16_rne(a + b);
        else d[i] = (a < b) ? s[i] : d[i];
      }
      break;
    }
    case OR_F16: {
      uint16_t* d = dst; const uint16_t* s = src;
      for (i = 0; i < n; ++i) {
        const float a = f16_to_f32(d[i]), b = f16_to_f32(s[i]);
        if (op == 0) d[i] = f32_to_f16_rne(a + b);
        else d[i] = (a < b) ? s[i] : d[i];
      }
      break;
    }
    case OR_I32: {
      int32_t* d = dst; const int32_t* s = src;
      if (op == 0) for (i = 0; i < n; ++i) d[i] = (int32_t)((uint32_t)d[i] + (uint32_t)s[i]);
      else for (i = 0; i < n; ++i) d[i] = (d[i] < s[i]) ? s[i] : d[i];
      break;
    }
    case OR_I64: {
      int64_t* d = dst; const int64_t* s = src;
      if (op == 0) for (i = 0; i < n; ++i) d[i] = (int64_t)((uint64_t)d[i] + (uint64_t)s[i]);
      else for (i = 0; i < n; ++i) d[i] = (d[i] < s[i]) ? s[i] : d[i];
      break;
    }
    case OR_U8: {
      uint8_t* d = dst; const uint8_t* s = src;
      if (op == 0) for (i = 0; i < n; ++i) d[i] = (uint8_t)(d[i] + s[i]);
      else for (i = 0; i < n; ++i) d[i] = (d[i] < s[i]) ? s[i] : d[i];
      break;
    }
  }
}

/* ---- worker pool: one transfer at a time, its element range split ---- */

typedef struct {
  pthread_t* th;
  int n;
  pthread_barrier_t start, done;
  volatile int quit;
  /* current job */
  int dt, op, reduce;
  char* dst;
  const char* src;
  int64_t count;
} pool_t;

typedef struct {
  pool_t* pool;
  int index;
} worker_arg;

static void run_slice(pool_t* P, int index) {
  const int es = esize_of(P->dt);
  const int64_t per = (P->count + P->n - 1) / P->n;
  const int64_t lo = per * index;
  int64_t hi = lo + per;
  if (hi > P->count) hi = P->count;
  if (lo >= hi) return;
  if (P->reduce) fold_range(P->dt, P->op, P->dst + lo * es, P->src + lo * es, hi - lo);
  else memmove(P->dst + lo * es, P->src + lo * es, (size_t)(hi - lo) * es);
}

static void* worker(void* a) {
  worker_arg* w = a;
  pool_t* P = w->pool;
  for (;;) {
    pthread_barrier_wait(&P->start);
    if (P->quit) break;
    run_slice(P, w->index);
    pthread_barrier_wait(&P->done);
  }
  free(w);
  return NULL;
}

static int cmp_slot_id(const void* a, const void* b) {
  const or_transfer* x = *(const or_transfer* const*)a;
  const or_transfer* y = *(const or_transfer* const*)b;
  if (x->slot != y->slot) return x->slot < y->slot ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* Executes `n` transfers over host buffers bufs[buf * world + rank]
 * (element counts lengths[buf]). `defined` (optional, same indexing, one
 * byte per element) tracks written elements so reads of never-written
 * data fail like the reference (returns 10 = 1 + UninitializedRead);
 * pass NULL to skip tracking. threads <= 1 runs single-threaded.
 * Returns 0 on success, 6 (BadBufferRef) on out-of-range access. */
int oracle_run_transfers(const or_transfer* ts, int n, void* const* bufs,
                         const int64_t* lengths, int world, int nbuf, int dtype,
                         unsigned char* const* defined, int threads) {
  const int es = esize_of(dtype);
  if (!es) return 99;
  const or_transfer** order = malloc(sizeof(*order) * (n ? n : 1));
  for (int i = 0; i < n; ++i) order[i] = &ts[i];
  qsort(order, n, sizeof(*order), cmp_slot_id); /* ids unique: stable by construction */

  pool_t P;
  memset(&P, 0, sizeof P);
  P.n = threads > 1 ? threads : 1;
  P.dt = dtype;
  if (P.n > 1) {
    P.th = malloc(sizeof(pthread_t) * P.n);
    pthread_barrier_init(&P.start, NULL, P.n);
    pthread_barrier_init(&P.done, NULL, P.n);
    for (int i = 1; i < P.n; ++i) {
      worker_arg* w = malloc(sizeof *w);
      w->pool = &P;
      w->index = i;
      pthread_create(&P.th[i], NULL, worker, w);
    }
  }
  int rc = 0;
  for (int k = 0; k < n && !rc; ++k) {
    const or_transfer* t = order[k];
    if (t->src < 0 || t->src >= world || t->dst < 0 || t->dst >= world || t->src_buf < 0 ||
        t->src_buf >= nbuf || t->dst_buf < 0 || t->dst_buf >= nbuf) { rc = 6; break; }
    if (t->src_off < 0 || t->dst_off < 0 || t->src_off + t->count > lengths[t->src_buf] ||
        t->dst_off + t->count > lengths[t->dst_buf]) { rc = 6; break; }
    char* dst = (char*)bufs[t->dst_buf * world + t->dst] + t->dst_off * es;
    const char* src = (const char*)bufs[t->src_buf * world + t->src] + t->src_off * es;
    if (defined) {
      const unsigned char* ds = defined[t->src_buf * world + t->src] + t->src_off;
      unsigned char* dd = defined[t->dst_buf * world + t->dst] + t->dst_off;
      for (int64_t i = 0; i < t->count; ++i) {
        if (!ds[i] || (t->reduce && !dd[i])) { rc = 10; break; }
      }
      if (rc) break;
      memset(dd, 1, (size_t)t->count);
    }
    /* Aliasing ranges of one rank's buffer are applied element by element
     * in ascending order, exactly like the reference loop. */
    const int alias = (t->src == t->dst && t->src_buf == t->dst_buf &&
                       t->src_off < t->dst_off + t->count && t->dst_off < t->src_off + t->count);
    if (alias) {
      if (t->src_off == t->dst_off && !t->reduce) continue; /* self copy */
      for (int64_t i = 0; i < t->count; ++i) {
        if (t->reduce) fold_range(dtype, t->op, dst + i * es, src + i * es, 1);
        else memcpy(dst + i * es, src + i * es, es);
      }
      continue;
    }
    if (P.n == 1 || t->count < 65536) {
      if (t->reduce) fold_range(dtype, t->op, dst, src, t->count);
      else memcpy(dst, src, (size_t)t->count * es);
      continue;
    }
    P.op = t->op;
    P.reduce = t->reduce;
    P.dst = dst;
    P.src = src;
    P.count = t->count;
    pthread_barrier_wait(&P.start);
    run_slice(&P, 0);
    pthread_barrier_wait(&P.done);
  }
  if (P.n > 1) {
    P.quit = 1;
    pthread_barrier_wait(&P.start);
    for (int i = 1; i < P.n; ++i) pthread_join(P.th[i], NULL);
    pthread_barrier_destroy(&P.start);
    pthread_barrier_destroy(&P.done);
    free(P.th);
  }
  free(order);
  return rc;
}
