// error_harness.cuh -- device error measurement helpers (see error_harness.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace dsfft {

// Largest n whose DFT runs with the transform and its twiddles in shared
// memory (2 n double2 = 128 KiB at 4096).
constexpr long long kDftSmemN = 4096;
// Default cut-over of the error harness: DFT reference (bit-identical to
// measure_error) up to here, the fp64 FFT beyond.
constexpr long long kDftMaxN = 4096;
// Per-transform error value of an all-zero reference (relative_l2_error throws).
constexpr double kZeroReference = -1.0;

struct ErrorStats {
  double median = 0.0, max = 0.0;
  size_t nonfinite = 0;
  bool invalid = false;  // an all-zero reference transform (the reference throws)
};

int launch_widen(const void* in, double2* out, long long count, int precision,
                 cudaStream_t stream);
// relative_l2_error(y_b, r_b) for every transform b (sequential sums).
int launch_rel_l2(const double2* y, const double2* r, double* err, long long n, long long batch,
                  cudaStream_t stream);
// dft_oracle of every transform; tw = dft_table(n) on the device.
int launch_dft(const double2* x, double2* y, const double2* tw, long long n, long long batch,
               int sm_count, cudaStream_t stream);
ErrorStats aggregate_errors(const std::vector<double>& errs);

}  // namespace dsfft
