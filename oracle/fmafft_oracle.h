/*
 * fmafft_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm (arxiv/paper_2604_00567,
 * "fmafft") for the batched forward FFT hot path.  It is the parity checker for
 * the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2604_00567_b200/libdsfft.so) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference itself, compiled from /root/reference sources into
 * oracle/_ref/libfmafft_ref.so (oracle/Makefile), and against the golden
 * vectors that library generated (tests/golden/, tests/golden/make_golden.py).
 *
 * Enumerations follow the reference declaration order:
 *   Precision { fp16, fp32, fp64 }                precision.hpp:12
 *   Strategy  { standard, linzer_feig, cosine, dual_select }   twiddle.hpp:14
 *   TwiddlePath { cos, sin }                      twiddle.hpp:12
 */
#ifndef FMAFFT_ORACLE_H
#define FMAFFT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FP16 = 0, ORC_FP32 = 1, ORC_FP64 = 2 };
enum { ORC_STANDARD = 0, ORC_LINZER_FEIG = 1, ORC_COSINE = 2, ORC_DUAL = 3 };
enum { ORC_PATH_COS = 0, ORC_PATH_SIN = 1 };
enum { ORC_ROUNDTRIP = 0, ORC_FORWARD_VS_ORACLE = 1 };

/* Mirrors fmafft::TwiddleEntry (twiddle.hpp:26-41), fixed-width for ctypes. */
typedef struct {
  double multiplier;
  double ratio;
  int32_t path;
  int32_t clamped;
  double omega_r;
  double omega_i;
} orc_entry;

/* Mirrors fmafft::OpCounter (precision.hpp:25-31). */
typedef struct {
  uint64_t fma_count;
  uint64_t add_count;
  uint64_t mul_count;
} orc_counters;

/* Mirrors fmafft::ErrorReport (analysis.hpp:58-68). */
typedef struct {
  uint64_t n;
  int32_t strategy;
  int32_t precision;
  int32_t metric;
  int32_t pad_;
  uint64_t trials;
  uint64_t seed;
  double rel_l2_median;
  double rel_l2_max;
  uint64_t nonfinite_trials;
} orc_error_report;

/* Every int-returning entry point: 0 ok, -1 invalid argument (the reference
 * would throw std::invalid_argument); the message is in orc_last_error(). */
const char* orc_last_error(void);

double orc_machine_epsilon(int precision);
double orc_round_to(double x, int precision);
void orc_round_array(const double* x, double* out, size_t count, int precision);

double orc_twiddle_angle(size_t k, size_t n);
int orc_build_table(size_t n, int strategy, double clamp_eps, orc_entry* out);
/* make_plan's table: FP64 table rounded once into the precision. */
int orc_plan_table(size_t n, int strategy, int precision, orc_entry* out);

/* Batched forward / inverse over `batch` transforms of n interleaved
 * (re, im) doubles each; `threads` host threads (<=0: all cores).  counters
 * (optional) receives the summed op counts. */
int orc_forward(size_t n, int strategy, int precision, const double* in,
                double* out, size_t batch, int threads, orc_counters* counters);
int orc_inverse(size_t n, int strategy, int precision, const double* in,
                double* out, size_t batch, int threads, orc_counters* counters);

/* Single butterfly through kernel_for(strategy) (butterfly.cpp:82-90). */
int orc_butterfly(int strategy, int precision, const double a[2],
                  const double b[2], const orc_entry* e, double out[4],
                  orc_counters* counters);
/* ArithmeticContext::add / sub / mul / fma (op 0..3, precision.cpp:77-111), elementwise */
void orc_ctx_op(int p, int op, const double* a, const double* b, const double* c, double* out,
                size_t count);

void orc_dft(size_t n, const double* in, double* out, size_t batch, int threads);
/* +inf when x holds a non-finite component; NaN on length/zero-ref error. */
double orc_rel_l2(const double* x, const double* y, size_t n);
double orc_cumulative_bound(double t_max, double eps, unsigned m);

/* SplitMix64 uniform_pm1 stream (analysis.hpp:73-91). */
void orc_splitmix_uniform(uint64_t seed, double* out, size_t count);
uint64_t orc_splitmix_next(uint64_t* state);

int orc_measure_error(size_t n, int strategy, int precision, int metric,
                      size_t trials, uint64_t seed, orc_error_report* out);

/* table_stats (twiddle.cpp:143-162): t_max, argmax, singular, cos, sin. */
int orc_table_stats(size_t n, int strategy, double* t_max, uint64_t* argmax_k,
                    uint64_t* singular, uint64_t* cos_count, uint64_t* sin_count);

#ifdef __cplusplus
}
#endif

#endif
