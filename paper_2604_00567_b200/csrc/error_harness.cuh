// error_harness.cuh -- device error measurement helpers (see error_harness.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace dsfft {

struct ErrorStats {
  double median = 0.0, max = 0.0;
  size_t nonfinite = 0;
  bool invalid = false;  // an all-zero reference transform (the reference throws)
};

int launch_widen(const void* in, double2* out, long long count, int precision,
                 cudaStream_t stream);
int launch_rel_l2(const double2* y, const double2* r, double* err, long long n, long long batch,
                  cudaStream_t stream);
ErrorStats aggregate_errors(const std::vector<double>& errs);

}  // namespace dsfft
