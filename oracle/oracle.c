/* TEST INFRASTRUCTURE -- C restatement of halftile's exact oracle.
 *
 * Restates pkg/src/halftile/oracle.py:47-75 (binary64 segmented sums and
 * prefix sums of binary16 inputs) with the ragged-last-segment semantics of
 * pad_segmented (segmented.py:57-89), multi-threaded with pthreads so it can
 * serve as the CPU baseline that bench.py times next to the GPU.  Never
 * linked into the product; tests/ and bench.py load it via ctypes from
 * oracle/build/liboracle.so (built by oracle/Makefile).
 *
 * binary16 decoding is a bit-level table (no compiler __fp16 support
 * needed); every binary16 value is exact in binary64.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double g_f16[65536];
static int g_init = 0;

static double f16_to_f64(uint16_t h) {
  const int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0)
    v = (double)m / 16777216.0; /* subnormal: m * 2^-24 */
  else if (e == 31)
    v = m ? (0.0 / 0.0) : (1.0 / 0.0);
  else {
    v = (double)(1024 + m);
    int ex = e - 25; /* (1024+m) * 2^(e-15-10) */
    while (ex > 0) { v *= 2.0; --ex; }
    while (ex < 0) { v *= 0.5; ++ex; }
  }
  return s ? -v : v;
}

void or_init(void) {
  if (g_init) return;
  for (int i = 0; i < 65536; ++i) g_f16[i] = f16_to_f64((uint16_t)i);
  g_init = 1;
}

double or_f16_to_f64(uint16_t h) {
  or_init();
  return g_f16[h];
}

/* ------------------------------------------------------------ reduce */
typedef struct {
  const uint16_t* x;
  int64_t n, s, k0, k1;
  double* out;
} red_job;

static void* red_worker(void* arg) {
  red_job* j = (red_job*)arg;
  for (int64_t k = j->k0; k < j->k1; ++k) {
    int64_t lo = k * j->s, hi = lo + j->s;
    if (hi > j->n) hi = j->n;
    double acc = 0.0;
    for (int64_t e = lo; e < hi; ++e) acc += g_f16[j->x[e]];
    j->out[k] = acc;
  }
  return NULL;
}

/* huge segments: per-thread partial over an element range */
typedef struct {
  const uint16_t* x;
  int64_t lo, hi;
  double sum;
} sum_job;

static void* sum_worker(void* arg) {
  sum_job* j = (sum_job*)arg;
  double acc = 0.0;
  for (int64_t e = j->lo; e < j->hi; ++e) acc += g_f16[j->x[e]];
  j->sum = acc;
  return NULL;
}

/* out[k] = sum of segment k (ceil(n/s) outputs), threads >= 1 */
void or_seg_reduce(const uint16_t* x, int64_t n, int64_t s, double* out, int threads) {
  or_init();
  if (threads < 1) threads = 1;
  const int64_t nseg = (n + s - 1) / s;
  if (nseg >= threads) {
    pthread_t th[256];
    red_job jobs[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; ++t) {
      jobs[t].x = x;
      jobs[t].n = n;
      jobs[t].s = s;
      jobs[t].k0 = nseg * t / threads;
      jobs[t].k1 = nseg * (t + 1) / threads;
      jobs[t].out = out;
      pthread_create(&th[t], NULL, red_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return;
  }
  /* few large segments: split each segment across the threads, combine in order */
  for (int64_t k = 0; k < nseg; ++k) {
    int64_t lo = k * s, hi = lo + s;
    if (hi > n) hi = n;
    pthread_t th[256];
    sum_job jobs[256];
    int nt = threads > 256 ? 256 : threads;
    for (int t = 0; t < nt; ++t) {
      jobs[t].x = x;
      jobs[t].lo = lo + (hi - lo) * t / nt;
      jobs[t].hi = lo + (hi - lo) * (t + 1) / nt;
      pthread_create(&th[t], NULL, sum_worker, &jobs[t]);
    }
    double acc = 0.0;
    for (int t = 0; t < nt; ++t) {
      pthread_join(th[t], NULL);
      acc += jobs[t].sum;
    }
    out[k] = acc;
  }
}

/* -------------------------------------------------------------- scan */
typedef struct {
  const uint16_t* x;
  int64_t n, s, lo, hi;
  int inclusive;
  int cont0;    /* element 0 continues a segment (carry given): not a start */
  double entry; /* value of the open segment entering lo */
  double tail;  /* pass 1: sum since the chunk's last segment start */
  int started;  /* pass 1: chunk contains a segment start */
  double* out;
} scan_job;

static inline int is_start(const scan_job* j, int64_t e) {
  return (e % j->s == 0) && !(e == 0 && j->cont0);
}

static void* scan_worker(void* arg) {
  scan_job* j = (scan_job*)arg;
  double run = j->entry;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    if (is_start(j, e)) run = 0.0;
    const double v = g_f16[j->x[e]];
    if (j->inclusive) {
      run += v;
      j->out[e] = run;
    } else {
      j->out[e] = run;
      run += v;
    }
  }
  return NULL;
}

static void* tail_worker(void* arg) {
  scan_job* j = (scan_job*)arg;
  double run = 0.0;
  int started = 0;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    if (is_start(j, e)) {
      run = 0.0;
      started = 1;
    }
    run += g_f16[j->x[e]];
  }
  j->tail = run;
  j->started = started;
  return NULL;
}

/* Segmented prefix sums, n outputs.  has_carry: segment 0 continues with
 * running value `carry`.  With threads > 1: pass 1 computes each chunk's
 * open-segment tail, a sequential pass chains them into chunk entries, pass
 * 2 scans every chunk from its entry (left-to-right order inside chunks). */
void or_seg_scan(const uint16_t* x, int64_t n, int64_t s, int inclusive, double carry,
                 int has_carry, double* out, int threads) {
  or_init();
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (n < (int64_t)threads * 4096) threads = 1;
  pthread_t th[256];
  scan_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].x = x;
    jobs[t].n = n;
    jobs[t].s = s;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    jobs[t].inclusive = inclusive;
    jobs[t].cont0 = has_carry ? 1 : 0;
    jobs[t].out = out;
  }
  if (threads > 1) {
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, tail_worker, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  }
  double run = has_carry ? carry : 0.0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].entry = run;
    if (threads > 1) run = jobs[t].started ? jobs[t].tail : run + jobs[t].tail;
  }
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, scan_worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}
