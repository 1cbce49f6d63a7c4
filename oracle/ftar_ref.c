/*
 * ftar_ref.c — C port of the reference CPU FTAR data path — TEST / BASELINE
 * INFRASTRUCTURE ONLY (never linked into the product library).
 *
 * Restates, per member and per partition, what pkg/src/ftdp/ftar.py does:
 *   _reduce_partition  ftar.py:329-353  staging copy `work = buf[p].copy()`,
 *                                       N-1 reduce-scatter ring steps
 *                                       (send (me-t)%n, recv (me-t-1)%n,
 *                                       accumulate), N-1 all-gather steps
 *                                       (send (me-t+1)%n, recv (me-t)%n, copy),
 *                                       isfinite check, commit buf[p] = work
 *   accumulate         _ckernels.pyx:9-18   dst[i] += src[i] (fp32, in order)
 *   copy_into          _ckernels.pyx:21-27  memcpy
 * with the TCP hop replaced by reading the left neighbour's staging buffer
 * after a barrier (each ring step is a barrier epoch, so the neighbour's
 * segment is exactly the bytes the reference would have put on the wire).
 * Members run as threads (as the reference's rank threads do); every member
 * may split each step's segment across `tpm` worker threads.
 *
 * oracle_reduce_f32 is the closed form of tests/test_ftar.py:20-40.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t off, len;
} span_t;

static void balanced(uint64_t total, uint64_t parts, uint64_t i, span_t* s) {
  uint64_t q = total / parts, r = total % parts;
  s->off = i * q + (i < r ? i : r);
  s->len = q + (i < r ? 1 : 0);
}

static uint64_t n_partitions(uint64_t total, uint64_t chunk_bytes, int C, int n) {
  if (total == 0) return 1;
  uint64_t cap = (chunk_bytes * (uint64_t)C * (uint64_t)n) / 4;
  if (cap < 1) cap = 1;
  return (total + cap - 1) / cap;
}

/* closed form: per segment, fp32 left fold from the owner in ring order */
void oracle_reduce_f32(const float* const* arrays, int n, uint64_t total, uint64_t chunk_bytes, int C,
                       float* out) {
  const uint64_t np = n_partitions(total, chunk_bytes, C, n);
  for (uint64_t p = 0; p < np; ++p) {
    span_t ps;
    if (total == 0) break;
    balanced(total, np, p, &ps);
    for (int j = 0; j < n; ++j) {
      span_t ss;
      balanced(ps.len, (uint64_t)n, (uint64_t)j, &ss);
      const uint64_t lo = ps.off + ss.off;
      for (uint64_t e = lo; e < lo + ss.len; ++e) {
        float acc = arrays[j][e];
        for (int k = 1; k < n; ++k) {
          volatile float x = arrays[(j + k) % n][e];
          acc = acc + x;
        }
        out[e] = acc;
      }
    }
  }
}

typedef struct {
  float** bufs;    /* member buffers (in place) */
  float** work;    /* member staging buffers (partition-sized) */
  int n, tpm;
  uint64_t total, chunk_bytes;
  int C;
  pthread_barrier_t bar;
  volatile int nonfinite[8];
  int status;
} ring_t;

typedef struct {
  ring_t* r;
  int member, worker;
} arg_t;

static void part_of(uint64_t len, int tpm, int w, uint64_t* lo, uint64_t* hi) {
  span_t s;
  balanced(len, (uint64_t)tpm, (uint64_t)w, &s);
  *lo = s.off;
  *hi = s.off + s.len;
}

static void* member_main(void* vp) {
  arg_t* a = (arg_t*)vp;
  ring_t* r = a->r;
  const int n = r->n, me = a->member, w = a->worker;
  const int left = (me - 1 + n) % n;
  const uint64_t np = n_partitions(r->total, r->chunk_bytes, r->C, n);
  for (uint64_t p = 0; p < np && r->total; ++p) {
    span_t ps;
    balanced(r->total, np, p, &ps);
    float* work = r->work[me];
    const float* lwork = r->work[left];
    uint64_t lo, hi;
    /* staging copy (ftar.py:335) */
    part_of(ps.len, r->tpm, w, &lo, &hi);
    memcpy(work + lo, r->bufs[me] + ps.off + lo, (hi - lo) * sizeof(float));
    pthread_barrier_wait(&r->bar);
    /* reduce-scatter (ftar.py:339-342) */
    for (int t = 0; t < n - 1; ++t) {
      span_t seg;
      balanced(ps.len, (uint64_t)n, (uint64_t)(((me - t - 1) % n + n) % n), &seg);
      part_of(seg.len, r->tpm, w, &lo, &hi);
      for (uint64_t e = seg.off + lo; e < seg.off + hi; ++e) work[e] += lwork[e];
      pthread_barrier_wait(&r->bar);
    }
    /* all-gather (ftar.py:343-346) */
    for (int t = 0; t < n - 1; ++t) {
      span_t seg;
      balanced(ps.len, (uint64_t)n, (uint64_t)(((me - t) % n + n) % n), &seg);
      part_of(seg.len, r->tpm, w, &lo, &hi);
      memcpy(work + seg.off + lo, lwork + seg.off + lo, (hi - lo) * sizeof(float));
      pthread_barrier_wait(&r->bar);
    }
    /* isfinite + commit (ftar.py:351-353) */
    part_of(ps.len, r->tpm, w, &lo, &hi);
    int bad = 0;
    for (uint64_t e = lo; e < hi; ++e)
      if (!isfinite(work[e])) bad = 1;
    if (bad) r->nonfinite[me] = 1;
    pthread_barrier_wait(&r->bar);
    if (r->nonfinite[me]) break; /* Fatal(NUMERICAL): nothing more committed */
    memcpy(r->bufs[me] + ps.off + lo, work + lo, (hi - lo) * sizeof(float));
    pthread_barrier_wait(&r->bar);
  }
  return NULL;
}

/* In-place ring all-reduce of n member buffers; returns 0, or 5 (NUMERICAL)
 * when any member's partition was non-finite. */
int oracle_ring_allreduce(float** bufs, int n, uint64_t total, uint64_t chunk_bytes, int C, int tpm) {
  if (n < 1 || n > 8 || tpm < 1) return 6;
  ring_t r;
  memset(&r, 0, sizeof(r));
  r.bufs = bufs;
  r.n = n;
  r.tpm = tpm;
  r.total = total;
  r.chunk_bytes = chunk_bytes;
  r.C = C;
  const uint64_t np = n_partitions(total, chunk_bytes, C, n);
  const uint64_t plen = total ? (total + np - 1) / np : 1;
  float* work_store[8];
  for (int m = 0; m < n; ++m) work_store[m] = (float*)malloc(plen * sizeof(float) + 16);
  r.work = work_store;
  pthread_barrier_init(&r.bar, NULL, (unsigned)(n * tpm));
  pthread_t th[64];
  arg_t args[64];
  int k = 0;
  for (int m = 0; m < n; ++m)
    for (int w = 0; w < tpm; ++w, ++k) {
      args[k].r = &r;
      args[k].member = m;
      args[k].worker = w;
      pthread_create(&th[k], NULL, member_main, &args[k]);
    }
  for (int i = 0; i < k; ++i) pthread_join(th[i], NULL);
  pthread_barrier_destroy(&r.bar);
  int st = 0;
  for (int m = 0; m < n; ++m) {
    if (r.nonfinite[m]) st = 5;
    free(work_store[m]);
  }
  return st;
}

/* model.py:146-155, separately rounded fp32 ops */
void oracle_sgd_momentum(float* p, float* m, const float* g, uint64_t len, float beta, float lr) {
  for (uint64_t i = 0; i < len; ++i) {
    volatile float mb = m[i] * beta;
    volatile float mg = mb + g[i];
    m[i] = mg;
    volatile float step = lr * mg;
    p[i] = p[i] - step;
  }
}
