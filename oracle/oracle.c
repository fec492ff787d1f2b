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

/* ------------------------------------------------------ tolerance checkers
 * Compare a GPU result with the exact oracle without materialising the
 * binary64 reference (needed at 2^30 / 2^33 elements).  For every output:
 * v = the exact value (binary64), A = the absolute mass it sums (sum of |x|
 * over the elements of v), bound = ulps * ulp_out(v) + gamma * A.  An output
 * violates when |got - v| > bound or got is not finite.  stats[0] = the
 * largest |got - v| / bound, stats[1] = the largest |got - v|, stats[2] = the
 * first violating index (-1 if none), stats[3] = the largest relative error
 * |got - v| / |v| over outputs with |v| >= 1; returns the violation count.
 * dt: 0 = binary16 bits, 1 = binary32, 2 = binary64. */
#include <math.h>

static double ulp_of(double v, int dt) {
  int e;
  v = fabs(v);
  if (v == 0.0) return dt == 0 ? ldexp(1.0, -24) : dt == 1 ? ldexp(1.0, -149) : ldexp(1.0, -1074);
  frexp(v, &e); /* v = m * 2^e, m in [0.5, 1) */
  if (dt == 0) return (e - 1 < -14) ? ldexp(1.0, -24) : ldexp(1.0, e - 1 - 10);
  if (dt == 1) return (e - 1 < -126) ? ldexp(1.0, -149) : ldexp(1.0, e - 1 - 23);
  return ldexp(1.0, e - 1 - 52);
}

static double got_at(const void* g, int dt, int64_t i) {
  if (dt == 0) return g_f16[((const uint16_t*)g)[i]];
  if (dt == 1) return (double)((const float*)g)[i];
  return ((const double*)g)[i];
}

typedef struct {
  double max_ratio, max_abs, max_rel;
  int64_t bad, first_bad;
} chk_acc;

static void chk_one(chk_acc* a, int64_t i, double got, double v, double A, int dt, double ulps,
                    double gamma) {
  const double err = fabs(got - v);
  const double bound = ulps * ulp_of(v, dt) + gamma * A;
  const int ok = isfinite(got) && err <= bound;
  if (!ok) {
    if (a->bad == 0 || i < a->first_bad) a->first_bad = i;
    a->bad++;
  }
  if (isfinite(got)) {
    const double r = bound > 0 ? err / bound : (err > 0 ? INFINITY : 0.0);
    if (r > a->max_ratio) a->max_ratio = r;
    if (err > a->max_abs) a->max_abs = err;
    if (fabs(v) >= 1.0 && err / fabs(v) > a->max_rel) a->max_rel = err / fabs(v);
  } else {
    a->max_ratio = INFINITY;
  }
}

static void chk_merge(chk_acc* d, const chk_acc* s) {
  if (s->max_ratio > d->max_ratio) d->max_ratio = s->max_ratio;
  if (s->max_abs > d->max_abs) d->max_abs = s->max_abs;
  if (s->max_rel > d->max_rel) d->max_rel = s->max_rel;
  if (s->bad && (d->bad == 0 || s->first_bad < d->first_bad)) d->first_bad = s->first_bad;
  d->bad += s->bad;
}

static void chk_stats(const chk_acc* a, double* stats) {
  stats[0] = a->max_ratio;
  stats[1] = a->max_abs;
  stats[2] = a->bad ? (double)a->first_bad : -1.0;
  stats[3] = a->max_rel;
}

typedef struct {
  const uint16_t* x;
  int64_t n, s, k0, k1;
  const void* got;
  int dt;
  double ulps, gamma;
  chk_acc acc;
} chk_red_job;

static void* chk_red_worker(void* arg) {
  chk_red_job* j = (chk_red_job*)arg;
  for (int64_t k = j->k0; k < j->k1; ++k) {
    int64_t lo = k * j->s, hi = lo + j->s;
    if (hi > j->n) hi = j->n;
    double v = 0.0, A = 0.0;
    for (int64_t e = lo; e < hi; ++e) {
      const double y = g_f16[j->x[e]];
      v += y;
      A += fabs(y);
    }
    chk_one(&j->acc, k, got_at(j->got, j->dt, k), v, A, j->dt, j->ulps, j->gamma);
  }
  return NULL;
}

typedef struct {
  const uint16_t* x;
  int64_t lo, hi;
  double sum, asum;
} chk_sum_job;

static void* chk_sum_worker(void* arg) {
  chk_sum_job* j = (chk_sum_job*)arg;
  double v = 0.0, a = 0.0;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    const double y = g_f16[j->x[e]];
    v += y;
    a += fabs(y);
  }
  j->sum = v;
  j->asum = a;
  return NULL;
}

/* segmented reduce: got[k], k < ceil(n/s) */
int64_t or_check_seg_reduce(const uint16_t* x, int64_t n, int64_t s, const void* got, int dt,
                            double ulps, double gamma, int threads, double* stats) {
  or_init();
  const int64_t nseg = (n + s - 1) / s;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  chk_acc tot = {0, 0, 0, 0, 0};
  if (nseg < threads) {
    /* few huge segments: exact sums by element ranges, one check per segment */
    for (int64_t k = 0; k < nseg; ++k) {
      int64_t lo = k * s, hi = lo + s;
      if (hi > n) hi = n;
      double v = 0.0, A = 0.0;
      pthread_t th[256];
      chk_sum_job jobs[256];
      for (int t = 0; t < threads; ++t) {
        jobs[t].x = x;
        jobs[t].lo = lo + (hi - lo) * t / threads;
        jobs[t].hi = lo + (hi - lo) * (t + 1) / threads;
        pthread_create(&th[t], NULL, chk_sum_worker, &jobs[t]);
      }
      for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        v += jobs[t].sum;
        A += jobs[t].asum;
      }
      chk_one(&tot, k, got_at(got, dt, k), v, A, dt, ulps, gamma);
    }
    chk_stats(&tot, stats);
    return tot.bad;
  }
  pthread_t th[256];
  chk_red_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    chk_red_job* j = &jobs[t];
    j->x = x;
    j->n = n;
    j->s = s;
    j->k0 = nseg * t / threads;
    j->k1 = nseg * (t + 1) / threads;
    j->got = got;
    j->dt = dt;
    j->ulps = ulps;
    j->gamma = gamma;
    memset(&j->acc, 0, sizeof(j->acc));
    pthread_create(&th[t], NULL, chk_red_worker, j);
  }
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    chk_merge(&tot, &jobs[t].acc);
  }
  chk_stats(&tot, stats);
  return tot.bad;
}

typedef struct {
  const uint16_t* x;
  int64_t lo, hi, s, base;
  int inclusive, cont0;
  double run, arun;   /* state entering lo */
  double trun, tarun; /* pass 1: state after hi starting from (0, 0) */
  int started;
  const void* got;
  int dt;
  double ulps, gamma;
  chk_acc acc;
} chk_scan_job;

static inline int chk_is_start(const chk_scan_job* j, int64_t e) {
  return (e % j->s == 0) && !(e == 0 && j->cont0);
}

static void* chk_tail_worker(void* arg) {
  chk_scan_job* j = (chk_scan_job*)arg;
  double r = 0.0, a = 0.0;
  int st = 0;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    if (chk_is_start(j, e)) {
      r = 0.0;
      a = 0.0;
      st = 1;
    }
    const double y = g_f16[j->x[e]];
    r += y;
    a += fabs(y);
  }
  j->trun = r;
  j->tarun = a;
  j->started = st;
  return NULL;
}

static void* chk_scan_worker(void* arg) {
  chk_scan_job* j = (chk_scan_job*)arg;
  double r = j->run, a = j->arun;
  for (int64_t e = j->lo; e < j->hi; ++e) {
    if (chk_is_start(j, e)) {
      r = 0.0;
      a = 0.0;
    }
    const double y = g_f16[j->x[e]];
    const double g = got_at(j->got, j->dt, e - j->base);
    if (j->inclusive) {
      r += y;
      a += fabs(y);
      chk_one(&j->acc, e, g, r, a, j->dt, j->ulps, j->gamma);
    } else {
      chk_one(&j->acc, e, g, r, a, j->dt, j->ulps, j->gamma);
      r += y;
      a += fabs(y);
    }
  }
  return NULL;
}

/* segmented scan outputs got[0 .. hi-lo) for elements [lo, hi) of x (global
 * indices: segment k starts at k*s; cont0: element 0 continues the caller's
 * carry).  *run / *arun: exact running sum and running |x| sum entering lo
 * (in), leaving hi (out), so a huge result can be checked chunk by chunk. */
int64_t or_check_seg_scan(const uint16_t* x, int64_t lo, int64_t hi, int64_t s, int inclusive,
                          int cont0, double* run, double* arun, const void* got, int dt,
                          double ulps, double gamma, int threads, double* stats) {
  or_init();
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (hi - lo < (int64_t)threads * 4096) threads = 1;
  pthread_t th[256];
  chk_scan_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    chk_scan_job* j = &jobs[t];
    memset(j, 0, sizeof(*j));
    j->x = x;
    j->lo = lo + (hi - lo) * t / threads;
    j->hi = lo + (hi - lo) * (t + 1) / threads;
    j->s = s;
    j->base = lo;
    j->inclusive = inclusive;
    j->cont0 = cont0;
    j->got = got;
    j->dt = dt;
    j->ulps = ulps;
    j->gamma = gamma;
  }
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, chk_tail_worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  double r = *run, a = *arun;
  for (int t = 0; t < threads; ++t) {
    jobs[t].run = r;
    jobs[t].arun = a;
    if (jobs[t].started) {
      r = jobs[t].trun;
      a = jobs[t].tarun;
    } else {
      r += jobs[t].trun;
      a += jobs[t].tarun;
    }
  }
  *run = r;
  *arun = a;
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, chk_scan_worker, &jobs[t]);
  chk_acc tot = {0, 0, 0, 0, 0};
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    chk_merge(&tot, &jobs[t].acc);
  }
  chk_stats(&tot, stats);
  return tot.bad;
}
