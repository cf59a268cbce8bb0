/*
 * fmafft_oracle.c -- TEST INFRASTRUCTURE ONLY (see fmafft_oracle.h).
 *
 * CPU restatement of the reference's forward-FFT hot path.  Each function
 * cites the reference file:line (under /root/reference/proj/core/) it
 * follows.  Compiled with -ffp-contract=off like the reference
 * (proj/CMakeLists.txt:11-13) so no mul+add is fused behind our back.
 */
#define _GNU_SOURCE
#include "fmafft_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

const char* orc_last_error(void) { return g_err; }

/* ---- precision.cpp ------------------------------------------------------ */

/* precision.cpp:36-43 */
double orc_machine_epsilon(int p) {
  switch (p) {
    case ORC_FP16: return 0x1p-11;
    case ORC_FP32: return 0x1p-24;
    default: return 0x1p-53;
  }
}

/* precision.cpp:24-32 round_mag_to_binary16 */
static double round_mag_to_binary16(double ax) {
  if (ax < 0x1p-14) {
    if (ax <= 0x1p-25) return 0.0;
    return nearbyint(ax * 0x1p24) * 0x1p-24;
  }
  int e;
  double m = frexp(ax, &e);
  return ldexp(nearbyint(m * 0x1p11), e - 11);
}

/* precision.cpp:61-75 round_to */
double orc_round_to(double x, int p) {
  if (p == ORC_FP64 || x == 0.0 || isnan(x)) return x;
  const double ax = fabs(x);
  if (p == ORC_FP16) {
    if (ax >= 65520.0) return copysign(INFINITY, x);
    return copysign(round_mag_to_binary16(ax), x);
  }
  if (ax >= 0x1.ffffffp+127) return copysign(INFINITY, x);
  return (double)(float)x;
}

void orc_round_array(const double* x, double* out, size_t count, int p) {
  for (size_t i = 0; i < count; ++i) out[i] = orc_round_to(x[i], p);
}

/* ArithmeticContext (precision.hpp:50-62, precision.cpp:77-111). */
typedef struct {
  int p;
  orc_counters c;
} ctx_t;

static double ctx_add(ctx_t* cx, double a, double b) { /* precision.cpp:77-82 */
  ++cx->c.add_count;
  if (cx->p == ORC_FP32) return (double)((float)a + (float)b);
  return orc_round_to(a + b, cx->p);
}
static double ctx_sub(ctx_t* cx, double a, double b) { /* precision.cpp:84-89 */
  ++cx->c.add_count;
  if (cx->p == ORC_FP32) return (double)((float)a - (float)b);
  return orc_round_to(a - b, cx->p);
}
static double ctx_mul(ctx_t* cx, double a, double b) { /* precision.cpp:91-96 */
  ++cx->c.mul_count;
  if (cx->p == ORC_FP32) return (double)((float)a * (float)b);
  return orc_round_to(a * b, cx->p);
}
static double ctx_fma(ctx_t* cx, double a, double b, double c) { /* precision.cpp:98-111 */
  ++cx->c.fma_count;
  switch (cx->p) {
    case ORC_FP16: return orc_round_to(fma(a, b, c), ORC_FP16);
    case ORC_FP32: return (double)fmaf((float)a, (float)b, (float)c);
    default: return fma(a, b, c);
  }
}

/* ---- twiddle.cpp -------------------------------------------------------- */

/* the context operations elementwise (op 0 add, 1 sub, 2 mul, 3 fma) */
void orc_ctx_op(int p, int op, const double* a, const double* b, const double* c, double* out,
                size_t count) {
  ctx_t cx;
  memset(&cx, 0, sizeof cx);
  cx.p = p;
  for (size_t i = 0; i < count; ++i)
    out[i] = op == 0 ? ctx_add(&cx, a[i], b[i])
           : op == 1 ? ctx_sub(&cx, a[i], b[i])
           : op == 2 ? ctx_mul(&cx, a[i], b[i])
                     : ctx_fma(&cx, a[i], b[i], c[i]);
}

static int check_size(size_t n) { /* twiddle.cpp:14-18 */
  if (n < 2 || (n & (n - 1)) != 0) {
    snprintf(g_err, sizeof g_err, "FFT size must be a power of two >= 2, got %zu", n);
    return -1;
  }
  return 0;
}

/* twiddle.cpp:55-57 -- pi is std::numbers::pi == M_PI as a double. */
double orc_twiddle_angle(size_t k, size_t n) {
  return -(2.0 * 3.141592653589793) * ((double)k / (double)n);
}

int orc_build_table(size_t n, int s, double clamp_eps, orc_entry* out) {
  if (s == ORC_LINZER_FEIG && !(clamp_eps > 0.0)) /* twiddle.cpp:75-76 */
    return fail("clamp_eps must be positive");
  if (check_size(n)) return -1;
  if (s < 0 || s > 3) return fail("unknown strategy");
  for (size_t k = 0; k < n / 2; ++k) {
    const double theta = orc_twiddle_angle(k, n);
    orc_entry* e = &out[k];
    e->omega_r = cos(theta);
    e->omega_i = sin(theta);
    e->clamped = 0;
    switch (s) {
      case ORC_STANDARD: /* twiddle.cpp:59-72 */
        e->multiplier = e->omega_r;
        e->ratio = 0.0;
        e->path = ORC_PATH_COS;
        break;
      case ORC_LINZER_FEIG: /* twiddle.cpp:74-95 */
        e->path = ORC_PATH_SIN;
        if (e->omega_i == 0.0) {
          e->multiplier = -clamp_eps;
          e->ratio = e->omega_r / -clamp_eps;
          e->clamped = 1;
        } else {
          e->multiplier = e->omega_i;
          e->ratio = e->omega_r / e->omega_i;
        }
        break;
      case ORC_COSINE: /* twiddle.cpp:97-110 */
        e->path = ORC_PATH_COS;
        e->multiplier = e->omega_r;
        e->ratio = e->omega_i / e->omega_r;
        break;
      case ORC_DUAL: /* twiddle.cpp:112-131: Algorithm 1, tie -> COS */
        if (fabs(e->omega_r) >= fabs(e->omega_i)) {
          e->path = ORC_PATH_COS;
          e->multiplier = e->omega_r;
          e->ratio = e->omega_i / e->omega_r;
        } else {
          e->path = ORC_PATH_SIN;
          e->multiplier = e->omega_i;
          e->ratio = e->omega_r / e->omega_i;
        }
        break;
    }
  }
  return 0;
}

/* fft.cpp:56-72 make_plan: n <= 2^24, table rounded once. */
int orc_plan_table(size_t n, int s, int p, orc_entry* out) {
  if (n > ((size_t)1 << 24)) return fail("FFT size exceeds 2^24");
  if (orc_build_table(n, s, 1e-7, out)) return -1;
  for (size_t k = 0; k < n / 2; ++k) {
    out[k].multiplier = orc_round_to(out[k].multiplier, p);
    out[k].ratio = orc_round_to(out[k].ratio, p);
    out[k].omega_r = orc_round_to(out[k].omega_r, p);
    out[k].omega_i = orc_round_to(out[k].omega_i, p);
  }
  return 0;
}

/* twiddle.cpp:143-162 */
int orc_table_stats(size_t n, int s, double* t_max, uint64_t* argmax_k,
                    uint64_t* singular, uint64_t* cos_count, uint64_t* sin_count) {
  orc_entry* t = (orc_entry*)malloc(sizeof(orc_entry) * (n / 2 ? n / 2 : 1));
  if (orc_build_table(n, s, 1e-7, t)) { free(t); return -1; }
  double tm = 0.0;
  uint64_t am = 0, sg = 0, cc = 0, sc = 0;
  for (size_t k = 0; k < n / 2; ++k) {
    if (t[k].path == ORC_PATH_COS) ++cc; else ++sc;
    if (t[k].clamped) { ++sg; continue; }
    const double r = fabs(t[k].ratio);
    if (r > tm) { tm = r; am = k; }
  }
  free(t);
  *t_max = tm; *argmax_k = am; *singular = sg; *cos_count = cc; *sin_count = sc;
  return 0;
}

/* ---- butterfly.cpp ------------------------------------------------------ */

/* butterfly.cpp:10-20 cosine_core */
static void cosine_core(ctx_t* cx, const double* a, const double* b, double t,
                        double w, double* o) {
  const double s1 = ctx_fma(cx, -t, b[1], b[0]);
  const double s2 = ctx_fma(cx, t, b[0], b[1]);
  o[0] = ctx_fma(cx, s1, w, a[0]);
  o[1] = ctx_fma(cx, s2, w, a[1]);
  o[2] = ctx_fma(cx, -s1, w, a[0]);
  o[3] = ctx_fma(cx, -s2, w, a[1]);
}

/* butterfly.cpp:23-33 sine_core */
static void sine_core(ctx_t* cx, const double* a, const double* b, double t,
                      double w, double* o) {
  const double s1 = ctx_fma(cx, -t, b[0], b[1]);
  const double s2 = ctx_fma(cx, t, b[1], b[0]);
  o[0] = ctx_fma(cx, -s1, w, a[0]);
  o[1] = ctx_fma(cx, s2, w, a[1]);
  o[2] = ctx_fma(cx, s1, w, a[0]);
  o[3] = ctx_fma(cx, -s2, w, a[1]);
}

/* butterfly.cpp:37-90: the four kernels behind kernel_for(strategy). */
static void butterfly(ctx_t* cx, int s, const double* a, const double* b,
                      const orc_entry* e, double* o) {
  switch (s) {
    case ORC_STANDARD: { /* butterfly.cpp:37-53 */
      const double rr = ctx_mul(cx, e->omega_r, b[0]);
      const double ii = ctx_mul(cx, e->omega_i, b[1]);
      const double ir = ctx_mul(cx, e->omega_i, b[0]);
      const double ri = ctx_mul(cx, e->omega_r, b[1]);
      const double tr = ctx_sub(cx, rr, ii);
      const double ti = ctx_add(cx, ir, ri);
      o[0] = ctx_add(cx, a[0], tr);
      o[1] = ctx_add(cx, a[1], ti);
      o[2] = ctx_sub(cx, a[0], tr);
      o[3] = ctx_sub(cx, a[1], ti);
      return;
    }
    case ORC_LINZER_FEIG: /* butterfly.cpp:55-65 */
      if (e->clamped) cosine_core(cx, a, b, e->omega_i, e->omega_r, o);
      else sine_core(cx, a, b, e->ratio, e->multiplier, o);
      return;
    case ORC_COSINE: /* butterfly.cpp:67-72 */
      cosine_core(cx, a, b, e->ratio, e->multiplier, o);
      return;
    default: /* butterfly.cpp:74-80 butterfly_dual */
      if (e->path == ORC_PATH_COS) cosine_core(cx, a, b, e->ratio, e->multiplier, o);
      else sine_core(cx, a, b, e->ratio, e->multiplier, o);
      return;
  }
}

int orc_butterfly(int s, int p, const double a[2], const double b[2],
                  const orc_entry* e, double out[4], orc_counters* counters) {
  ctx_t cx = {p, {0, 0, 0}};
  butterfly(&cx, s, a, b, e, out);
  if (counters) *counters = cx.c;
  return 0;
}

/* ---- fft.cpp ------------------------------------------------------------ */

/* fft.cpp:32-52 run_passes: Stockham DIT, ping-pong, natural order.
 * buf/other hold 2n doubles; the result ends in *res. */
static double* run_passes(ctx_t* cx, size_t n, int s, const orc_entry* tab,
                          double* buf, double* other) {
  const size_t half_n = n / 2;
  unsigned m = 0;
  while (((size_t)1 << m) < n) ++m;
  size_t block = 1;
  for (unsigned pass = 0; pass < m; ++pass, block <<= 1) {
    const size_t stride = n / (2 * block);
    for (size_t j = 0; j < half_n; ++j) {
      const size_t jq = j & (block - 1);
      const orc_entry* e = &tab[jq * stride];
      double r[4];
      butterfly(cx, s, &buf[2 * j], &buf[2 * (j + half_n)], e, r);
      const size_t base = ((j >> pass) * 2) * block + jq;
      other[2 * base] = r[0];
      other[2 * base + 1] = r[1];
      other[2 * (base + block)] = r[2];
      other[2 * (base + block) + 1] = r[3];
    }
    double* t = buf; buf = other; other = t;
  }
  return buf;
}

/* fft.cpp:74-84 forward (ingest rounding, then the passes). */
static void forward_one(ctx_t* cx, size_t n, int s, const orc_entry* tab,
                        const double* in, double* out, double* w0, double* w1) {
  for (size_t i = 0; i < 2 * n; ++i) w0[i] = orc_round_to(in[i], cx->p);
  const double* r = run_passes(cx, n, s, tab, w0, w1);
  memcpy(out, r, sizeof(double) * 2 * n);
}

/* fft.cpp:86-101 inverse: conj -> forward -> conj * round_to(1/n). */
static void inverse_one(ctx_t* cx, size_t n, int s, const orc_entry* tab,
                        const double* in, double* out, double* w0, double* w1) {
  for (size_t i = 0; i < n; ++i) {
    w0[2 * i] = orc_round_to(in[2 * i], cx->p);
    w0[2 * i + 1] = orc_round_to(-in[2 * i + 1], cx->p);
  }
  const double* r = run_passes(cx, n, s, tab, w0, w1);
  const double scale = orc_round_to(1.0 / (double)n, cx->p);
  for (size_t i = 0; i < n; ++i) {
    out[2 * i] = ctx_mul(cx, r[2 * i], scale);
    out[2 * i + 1] = ctx_mul(cx, -r[2 * i + 1], scale);
  }
}

typedef struct {
  size_t n, b0, b1;
  int s, p, inverse;
  const orc_entry* tab;
  const double* in;
  double* out;
  orc_counters c;
} fwd_job;

static void* fwd_worker(void* arg) {
  fwd_job* j = (fwd_job*)arg;
  ctx_t cx = {j->p, {0, 0, 0}};
  double* w0 = (double*)malloc(sizeof(double) * 2 * j->n);
  double* w1 = (double*)malloc(sizeof(double) * 2 * j->n);
  for (size_t b = j->b0; b < j->b1; ++b) {
    const double* in = j->in + 2 * j->n * b;
    double* out = j->out + 2 * j->n * b;
    if (j->inverse) inverse_one(&cx, j->n, j->s, j->tab, in, out, w0, w1);
    else forward_one(&cx, j->n, j->s, j->tab, in, out, w0, w1);
  }
  free(w0);
  free(w1);
  j->c = cx.c;
  return NULL;
}

static int resolve_threads(int threads, size_t batch) {
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads < 1) threads = 1;
  if ((size_t)threads > batch) threads = (int)(batch ? batch : 1);
  return threads;
}

static int run_batch(size_t n, int s, int p, const double* in, double* out,
                     size_t batch, int threads, orc_counters* counters, int inv) {
  if (p < 0 || p > 2) return fail("unknown precision");
  orc_entry* tab = (orc_entry*)malloc(sizeof(orc_entry) * (n / 2 ? n / 2 : 1));
  if (orc_plan_table(n, s, p, tab)) { free(tab); return -1; }
  threads = resolve_threads(threads, batch);
  fwd_job* jobs = (fwd_job*)calloc((size_t)threads, sizeof(fwd_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    fwd_job* j = &jobs[t];
    j->n = n; j->s = s; j->p = p; j->inverse = inv; j->tab = tab;
    j->in = in; j->out = out;
    j->b0 = batch * (size_t)t / (size_t)threads;
    j->b1 = batch * (size_t)(t + 1) / (size_t)threads;
    if (threads == 1) fwd_worker(j);
    else pthread_create(&th[t], NULL, fwd_worker, j);
  }
  orc_counters tot = {0, 0, 0};
  for (int t = 0; t < threads; ++t) {
    if (threads > 1) pthread_join(th[t], NULL);
    tot.fma_count += jobs[t].c.fma_count;
    tot.add_count += jobs[t].c.add_count;
    tot.mul_count += jobs[t].c.mul_count;
  }
  if (counters) *counters = tot;
  free(jobs); free(th); free(tab);
  return 0;
}

int orc_forward(size_t n, int s, int p, const double* in, double* out,
                size_t batch, int threads, orc_counters* counters) {
  return run_batch(n, s, p, in, out, batch, threads, counters, 0);
}

int orc_inverse(size_t n, int s, int p, const double* in, double* out,
                size_t batch, int threads, orc_counters* counters) {
  return run_batch(n, s, p, in, out, batch, threads, counters, 1);
}

/* fft.cpp:103-121 dft_oracle: FP64 O(n^2), angles reduced through jk mod n. */
static void dft_one(size_t n, const double* in, double* out) {
  const double two_pi_over_n = (2.0 * 3.141592653589793) / (double)n;
  for (size_t j = 0; j < n; ++j) {
    double acc_re = 0.0, acc_im = 0.0;
    for (size_t k = 0; k < n; ++k) {
      const double theta = -two_pi_over_n * (double)((j * k) % n);
      const double c = cos(theta);
      const double s = sin(theta);
      acc_re += in[2 * k] * c - in[2 * k + 1] * s;
      acc_im += in[2 * k] * s + in[2 * k + 1] * c;
    }
    out[2 * j] = acc_re;
    out[2 * j + 1] = acc_im;
  }
}

typedef struct { size_t n, b0, b1; const double* in; double* out; } dft_job;

static void* dft_worker(void* arg) {
  dft_job* j = (dft_job*)arg;
  for (size_t b = j->b0; b < j->b1; ++b)
    dft_one(j->n, j->in + 2 * j->n * b, j->out + 2 * j->n * b);
  return NULL;
}

void orc_dft(size_t n, const double* in, double* out, size_t batch, int threads) {
  threads = resolve_threads(threads, batch);
  dft_job* jobs = (dft_job*)calloc((size_t)threads, sizeof(dft_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (dft_job){n, batch * (size_t)t / (size_t)threads,
                        batch * (size_t)(t + 1) / (size_t)threads, in, out};
    if (threads == 1) dft_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, dft_worker, &jobs[t]);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th);
}

/* ---- analysis.cpp ------------------------------------------------------- */

/* analysis.cpp:41-57 relative_l2_error (throws -> NaN here). */
double orc_rel_l2(const double* x, const double* y, size_t n) {
  double num = 0.0, den = 0.0;
  int finite = 1;
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(x[2 * i]) || !isfinite(x[2 * i + 1])) finite = 0;
    const double dr = x[2 * i] - y[2 * i];
    const double di = x[2 * i + 1] - y[2 * i + 1];
    num += dr * dr + di * di;
    den += y[2 * i] * y[2 * i] + y[2 * i + 1] * y[2 * i + 1];
  }
  if (den == 0.0) { fail("relative_l2_error: all-zero reference"); return NAN; }
  if (!finite) return INFINITY;
  return sqrt(num / den);
}

/* analysis.cpp:61-63 */
double orc_cumulative_bound(double t_max, double eps, unsigned m) {
  return pow(1.0 + t_max * eps, (double)m) - 1.0;
}

/* analysis.hpp:77-87 SplitMix64::next / uniform_pm1 */
uint64_t orc_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_splitmix_uniform(uint64_t seed, double* out, size_t count) {
  uint64_t st = seed;
  for (size_t i = 0; i < count; ++i)
    out[i] = 2.0 * ((double)(orc_splitmix_next(&st) >> 11) * 0x1p-53) - 1.0;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* analysis.cpp:101-154 measure_error (median: analysis.cpp:16-22). */
int orc_measure_error(size_t n, int s, int p, int metric, size_t trials,
                      uint64_t seed, orc_error_report* rep) {
  if (trials < 1) return fail("trials must be >= 1");
  if (n > ((size_t)1 << 24)) return fail("FFT size exceeds 2^24");
  orc_entry* tab = (orc_entry*)malloc(sizeof(orc_entry) * (n / 2 ? n / 2 : 1));
  if (orc_plan_table(n, s, p, tab)) { free(tab); return -1; }
  memset(rep, 0, sizeof *rep);
  rep->n = n; rep->strategy = s; rep->precision = p; rep->metric = metric;
  rep->trials = trials; rep->seed = seed;
  double* x = (double*)malloc(sizeof(double) * 2 * n);
  double* ing = (double*)malloc(sizeof(double) * 2 * n);
  double* y = (double*)malloc(sizeof(double) * 2 * n);
  double* z = (double*)malloc(sizeof(double) * 2 * n);
  double* w0 = (double*)malloc(sizeof(double) * 2 * n);
  double* w1 = (double*)malloc(sizeof(double) * 2 * n);
  double* errs = (double*)malloc(sizeof(double) * trials);
  size_t nfin = 0;
  double max_err = 0.0;
  uint64_t st = seed;
  for (size_t t = 0; t < trials; ++t) {
    for (size_t i = 0; i < 2 * n; ++i)
      x[i] = 2.0 * ((double)(orc_splitmix_next(&st) >> 11) * 0x1p-53) - 1.0;
    for (size_t i = 0; i < 2 * n; ++i) ing[i] = orc_round_to(x[i], p);
    ctx_t cx = {p, {0, 0, 0}};
    double err;
    forward_one(&cx, n, s, tab, x, y, w0, w1);
    if (metric == ORC_ROUNDTRIP) {
      inverse_one(&cx, n, s, tab, y, z, w0, w1);
      err = orc_rel_l2(z, ing, n);
    } else {
      dft_one(n, ing, z);
      err = orc_rel_l2(y, z, n);
    }
    if (isfinite(err)) {
      errs[nfin++] = err;
      if (err > max_err) max_err = err;
    } else {
      ++rep->nonfinite_trials;
      max_err = INFINITY;
    }
  }
  if (nfin == 0) {
    rep->rel_l2_median = INFINITY;
  } else {
    qsort(errs, nfin, sizeof(double), cmp_double);
    rep->rel_l2_median = (nfin % 2) ? errs[nfin / 2]
                                    : (errs[nfin / 2 - 1] + errs[nfin / 2]) / 2.0;
  }
  rep->rel_l2_max = rep->nonfinite_trials > 0 ? INFINITY : max_err;
  free(x); free(ing); free(y); free(z); free(w0); free(w1); free(errs); free(tab);
  return 0;
}
