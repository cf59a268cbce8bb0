/*
 * dsfft.h -- C ABI of the B200-native batched dual-select FFT (libdsfft.so).
 *
 * This is the drop-in boundary for the reference's plan/execute hot path
 * (arxiv/paper_2604_00567 "fmafft", /root/reference/proj/core).  Plain
 * pointers and sizes only; no C++ or torch types cross it.  Each entry point
 * names the reference interface it replaces (file:line under
 * /root/reference/proj/core/).  The C++ mirror of the reference API lives in
 * include/fmafft_b200.hpp; INTEGRATION.md shows the bindings.
 *
 * Enumerations keep the reference's declaration order so values cast 1:1:
 *   dsfft_strategy  == fmafft::Strategy     (include/fmafft/twiddle.hpp:14)
 *   dsfft_precision == fmafft::Precision    (include/fmafft/precision.hpp:12)
 *
 * Sample layout on device and in the *_host working-precision calls:
 * interleaved complex in the working precision, transform-major:
 *   fp16: binary16 pairs (re, im) = 4 bytes per sample
 *   fp32: binary32 pairs (re, im) = 8 bytes per sample
 * Buffers must be 16-byte aligned.  in == out (in place) is allowed.
 *
 * Errors: every int-returning call returns a dsfft_status; on failure
 * dsfft_last_error() holds the reference's exception text where one exists
 * (e.g. "FFT size must be a power of two >= 2, got 1023").  NaN/inf data is
 * never an error: it propagates exactly as in the reference.
 */
#ifndef DSFFT_H
#define DSFFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSFFT_VERSION 2

typedef enum {
  DSFFT_STANDARD = 0,
  DSFFT_LINZER_FEIG = 1,
  DSFFT_COSINE = 2,
  DSFFT_DUAL_SELECT = 3
} dsfft_strategy;

typedef enum { DSFFT_FP16 = 0, DSFFT_FP32 = 1, DSFFT_FP64 = 2 } dsfft_precision;

typedef enum { DSFFT_FORWARD = 0, DSFFT_INVERSE = 1 } dsfft_direction;

typedef enum {
  DSFFT_OK = 0,
  DSFFT_ERR_INVALID = 1,     /* reference: std::invalid_argument */
  DSFFT_ERR_UNSUPPORTED = 2, /* reserved: every reference configuration runs on the device */
  DSFFT_ERR_CUDA = 3,        /* CUDA runtime / launch failure */
  DSFFT_ERR_NO_DEVICE = 4    /* no sm_100 device: the product never falls back to CPU */
} dsfft_status;

typedef struct dsfft_plan_s* dsfft_plan;

/* One rounded table record == fmafft::TwiddleEntry (twiddle.hpp:26-41). */
typedef struct {
  double multiplier;
  double ratio;
  int32_t path; /* 0 COS, 1 SIN */
  int32_t clamped;
  double omega_r;
  double omega_i;
} dsfft_entry;

/* Replaces fmafft::make_plan(n, strategy, precision)        (fft.hpp:26, fft.cpp:56-72)
 * and build_table(n, s, clamp_eps)                          (twiddle.hpp:65).
 * Builds the FP64 table on the host with the reference algorithm (libm
 * cos/sin, Algorithm 1 with the >= tie to COS), rounds it once into the working
 * precision, packs the per-stage device records and uploads them to `device`.
 * n: power of two in [2, 2^24]; clamp_eps > 0 (used by linzer_feig only). */
int dsfft_plan_create(size_t n, int strategy, int precision, double clamp_eps, int device,
                      dsfft_plan* out);

/* A plan over a caller-supplied table: `table` holds the n/2 records of
 * FftPlan::table.entries exactly as the reference's forward would read them
 * (already rounded into `precision`, possibly edited by the caller -- the
 * reference's FftPlan is a plain struct with a public table, see the
 * "negative control" case of test_fft.cpp).  Records are packed and uploaded
 * as given; nothing is recomputed.  strategy selects the butterfly
 * (butterfly.cpp:82-90 kernel_for). */
int dsfft_plan_create_with_table(size_t n, int strategy, int precision, const dsfft_entry* table,
                                 size_t count, int device, dsfft_plan* out);

int dsfft_plan_destroy(dsfft_plan plan);

/* FftPlan fields (fft.hpp:17-23). */
int dsfft_plan_info(dsfft_plan plan, size_t* n, unsigned* m, int* strategy, int* precision);

/* Host-only table builder (no device needed): make_plan's table, i.e.
 * build_table(n, strategy, clamp_eps) (twiddle.cpp:133-141) rounded once into
 * `precision` (fft.cpp:65-70); precision fp64 returns the raw FP64 table.
 * `out` receives n/2 records. */
int dsfft_build_table(size_t n, int strategy, int precision, double clamp_eps, dsfft_entry* out,
                      size_t count);

/* The table dump in the reference's CSV schema, write_table_csv
 * (serialize.cpp:48-57: "k,theta,omega_r,omega_i,path,multiplier,ratio,clamped",
 * %.17g): precision fp64 gives the CLI `twiddles` dump of build_table
 * (main.cpp:34-42); fp16/fp32 give the plan's rounded table, i.e. exactly the
 * values the device records are packed from.  Returns the bytes needed
 * including the terminating NUL (0 on error); copies when `cap` suffices. */
size_t dsfft_table_csv(size_t n, int strategy, int precision, double clamp_eps, char* out,
                       size_t cap);

/* Ratio statistics and error bounds in the reference's CSV schema,
 * write_bounds_csv (serialize.cpp:79-91: "strategy,t_max,argmax_k,
 * singular_count,cos_path_count,sin_path_count,per_butterfly_bound,
 * cumulative_bound,improvement_vs_baseline,divergent"):
 *   kind DSFFT_STATS_RATIO      reproduce_ratio_table(n) (analysis.cpp:65-76),
 *                               the CLI `stats` command (main.cpp:45-52):
 *                               LF, cosine, dual at binary16 epsilon;
 *   kind DSFFT_STATS_CUMULATIVE reproduce_cumulative_table(n, precision)
 *                               (analysis.cpp:78-88), the CLI `bounds`: LF, dual.
 * Statistics come from the FP64 tables (table_stats, twiddle.cpp:143-162).
 * Returns the bytes needed including the NUL (0 on error); copies when `cap`
 * suffices. */
enum { DSFFT_STATS_RATIO = 0, DSFFT_STATS_CUMULATIVE = 1 };
size_t dsfft_bounds_csv(size_t n, int kind, int precision, char* out, size_t cap);

/* Copy of the plan's rounded table: FftPlan::table.entries (n/2 records). */
int dsfft_plan_table(dsfft_plan plan, dsfft_entry* out, size_t count);

/* Batched forward / inverse on device buffers, enqueued on `stream`
 * (cudaStream_t; NULL = legacy default stream).  Replaces
 *   SampleBuffer forward(const FftPlan&, const SampleBuffer&, ArithmeticContext&)  (fft.hpp:33-34)
 *   SampleBuffer inverse(const FftPlan&, const SampleBuffer&, ArithmeticContext&)  (fft.hpp:38-39)
 * for `batch` independent transforms.  Input must already be in the working
 * precision (the reference's ingest rounding, fft.cpp:79-82, is dsfft_round_to).
 * Bit-identical to the reference in fp32 and fp16. */
int dsfft_execute(dsfft_plan plan, int direction, const void* d_in, void* d_out, size_t batch,
                  void* stream);

/* Same, from and to HOST buffers in the working precision (pinned memory
 * gives full PCIe overlap).  Copies are chunked and pipelined against the
 * kernels on internal streams ordered after / before `stream`; returns after
 * the results are in h_out. */
int dsfft_execute_host(dsfft_plan plan, int direction, const void* h_in, void* h_out,
                       size_t batch, void* stream);

/* Batch partitioner over the GPUs of one box: plans[i] is a
 * plan for device i (same n / strategy / precision); transforms
 * [i*batch/nplans, (i+1)*batch/nplans) of the host buffers run on device i
 * through its own dsfft_execute_host pipeline, one host thread per device.
 * No data crosses devices (no collectives).  The reference has no parallel
 * path; this extends forward/inverse (fft.hpp:33-39) over devices. */
int dsfft_execute_multi(const dsfft_plan* plans, int nplans, int direction, const void* h_in,
                        void* h_out, size_t batch);

/* The reference's exact calling convention: double-carrier SampleBuffers
 * (interleaved re, im doubles, fft.hpp:12).  Rounds on ingest with round_to
 * semantics, runs on the device, widens the result back to double. */
int dsfft_execute_f64(dsfft_plan plan, int direction, const double* in, double* out,
                      size_t batch);

/* == fmafft::ErrorReport (analysis.hpp:58-68). metric: 0 roundtrip,
 * 1 forward_vs_oracle (ErrorMetric, analysis.hpp:49). */
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
} dsfft_error_report;

/* FP64 reference of the forward_vs_oracle metric:
 *   DSFFT_REF_DFT    the device dft_oracle (bit-identical to fft.cpp:103-121;
 *                    O(n^2) per transform);
 *   DSFFT_REF_FFT64  this library's fp64 FFT (bit-identical to the
 *                    reference's fp64 forward; within 1e-11 of the DFT);
 *   DSFFT_REF_AUTO   the DFT for n <= 4096, the fp64 FFT above. */
enum { DSFFT_REF_AUTO = 0, DSFFT_REF_DFT = 1, DSFFT_REF_FFT64 = 2 };

/* Device error harness over a whole batch already on the device (working
 * precision, 16-byte aligned): per-transform relative_l2_error
 * (analysis.cpp:41-57, the same sequential sums, bit-identical) of the
 * forward against the FP64 reference of the ingested input, or of
 * inverse(forward(x)) against x; median over finite transforms, max (+inf if
 * any non-finite) and the non-finite count (analysis.cpp:16-22,142-152).
 * `errs` (optional, `batch` doubles, host) receives the per-transform errors.
 * dsfft_error_device == dsfft_error_device_ex(..., DSFFT_REF_AUTO, ...). */
int dsfft_error_device(dsfft_plan plan, int metric, const void* d_x, size_t batch, void* stream,
                       dsfft_error_report* out, double* errs);
int dsfft_error_device_ex(dsfft_plan plan, int metric, int reference, const void* d_x,
                          size_t batch, void* stream, dsfft_error_report* out, double* errs);

/* dft_oracle (fft.hpp:44, fft.cpp:103-121) on the device, bit-identical:
 * the reference's cos/sin per residue (j k) mod n, sequential k-order
 * accumulation with separately rounded FP64 mul / add / sub.  Any n in
 * [1, 2^24] (not only powers of two).  Interleaved (re, im) doubles.
 *   dsfft_dft_device  device buffers (16-byte aligned, out of place), stream-ordered,
 *                     returns after the kernel completes;
 *   dsfft_dft_oracle  host buffers (the SampleBuffer carrier), synchronous. */
int dsfft_dft_device(const void* d_in, void* d_out, size_t n, size_t batch, int device,
                     void* stream);
int dsfft_dft_oracle(const double* in, double* out, size_t n, size_t batch, int device);

/* measure_error(n, strategy, precision, metric, trials, seed)
 * (analysis.cpp:101-154): the reference's protocol (one SplitMix64 stream,
 * re then im, ingest round_to) with every transform on `device`.  For
 * n <= 2^16 the FP64 reference is the device dft_oracle and the report is
 * bit-identical to the reference's; beyond, the fp64 FFT (O(n^2) DFTs of 2^20
 * points take seconds each). */
int dsfft_measure_error(size_t n, int strategy, int precision, int metric, size_t trials,
                        uint64_t seed, int device, dsfft_error_report* out);

/* Synthetic batch on the device, keyed by the GLOBAL transform index: fills
 * `count` transforms of n samples (working precision) with transforms
 * [first_transform, first_transform + count) of the batch defined by `seed`.
 * Component c of sample s of transform b is uniform [-1, 1) (the
 * reference's 53-bit construction, analysis.hpp:84-87) from a splitmix64 hash
 * of (seed, 2(b n + s) + c), rounded once into `precision`.  A shard generated
 * on any device equals the same rows of the whole batch generated on one
 * (the multi-GPU bench checks its shards this way).  Stream-ordered. */
int dsfft_fill_uniform(void* d_out, size_t n, uint64_t first_transform, size_t count,
                       uint64_t seed, int precision, int device, void* stream);

/* round_to (precision.cpp:61-75) of `count` doubles into the working format
 * (binary16 / binary32 words), and the exact widening back. */
int dsfft_round_to(const double* in, void* out, size_t count, int precision);
int dsfft_widen(const void* in, double* out, size_t count, int precision);

/* The reference's scalar precision model, ArithmeticContext::add / sub / mul
 * / fma (precision.cpp:77-111), evaluated on `device` elementwise over host
 * arrays: out[i] = op(a[i], b[i] [, c[i]]) with op DSFFT_OP_*, rounded exactly
 * as the context rounds (fp16: the double result rounded to binary16 with
 * round_to's overflow rule; fp32: the operation on the float-cast operands;
 * fp64: the double operation), for any double inputs.  `c` is read for FMA
 * only. */
enum { DSFFT_OP_ADD = 0, DSFFT_OP_SUB = 1, DSFFT_OP_MUL = 2, DSFFT_OP_FMA = 3 };
int dsfft_context_ops(int precision, int op, const double* a, const double* b, const double* c,
                      double* out, size_t count, int device);

/* The butterfly-variant API (butterfly.hpp:22-61: butterfly_standard /
 * _linzer_feig / _cosine / _dual, selected like kernel_for(strategy)) on
 * `device`, batched: for each i, the variant's butterfly of a[2i..2i+1],
 * b[2i..2i+1] (re, im) with table entry entries[i] under `precision`'s
 * rounding; out[4i..4i+3] = sum.re, sum.im, diff.re, diff.im.  Bit-identical
 * to the reference for any double inputs. */
int dsfft_butterflies(int strategy, int precision, const double* a, const double* b,
                      const dsfft_entry* entries, double* out, size_t count, int device);

/* Bytes of one complex sample in the working precision (4, 8), 0 if invalid. */
size_t dsfft_sample_bytes(int precision);

/* Number of device kernel launches the last execute on this thread issued. */
uint64_t dsfft_last_launch_count(void);

/* Thread-local text of the last failure ("" when none). */
const char* dsfft_last_error(void);

int dsfft_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DSFFT_H */
