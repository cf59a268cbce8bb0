// error_harness.cu -- device error measurement.
//
// Mirrors measure_error (analysis.cpp:101-154) over a whole device batch:
//   forward_vs_oracle: rel-L2 of the working-precision forward against an
//     FP64 reference transform of the same (ingested) input;
//   roundtrip: rel-L2 of inverse(forward(x)) against x;
// per transform (relative_l2_error, analysis.cpp:41-57: +inf when the result
// has a non-finite component), then median over finite transforms, max (+inf
// if any is non-finite) and the non-finite count (analysis.cpp:16-22,142-152).
//
// The FP64 reference is this library's own fp64 transform (DFMA passes,
// bit-identical to the reference's fp64 forward) instead of the O(n^2)
// dft_oracle: both are FP64-accurate (test_fft.cpp:110-128 bound them within
// 1e-11 of each other), so the measured fp16/fp32 errors agree with the
// reference's to about 1e-9 relative while the harness runs at device speed.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "error_harness.cuh"

namespace dsfft {

namespace {

// working precision -> double2 (exact widening)
__global__ void widen_kernel(const void* in, double2* out, long long count, int precision) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double2 v;
    if (precision == 0) {
      const __half2 h = reinterpret_cast<const __half2*>(in)[i];
      v = make_double2(double(__low2float(h)), double(__high2float(h)));
    } else if (precision == 1) {
      const float2 f = reinterpret_cast<const float2*>(in)[i];
      v = make_double2(double(f.x), double(f.y));
    } else {
      v = reinterpret_cast<const double2*>(in)[i];
    }
    out[i] = v;
  }
}

// one block per transform: err[b] = ||y_b - r_b|| / ||r_b||, +inf if y_b has a
// non-finite component, NaN for an all-zero reference (the reference throws)
__global__ void __launch_bounds__(256) rel_l2_kernel(const double2* y, const double2* r,
                                                     double* err, long long n) {
  __shared__ double s_num[256], s_den[256];
  __shared__ int s_fin[256];
  const long long b = blockIdx.x;
  const double2* yb = y + b * n;
  const double2* rb = r + b * n;
  double num = 0.0, den = 0.0;
  int fin = 1;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 a = yb[i], c = rb[i];
    if (!isfinite(a.x) || !isfinite(a.y)) fin = 0;
    const double dr = a.x - c.x, di = a.y - c.y;
    num += dr * dr + di * di;
    den += c.x * c.x + c.y * c.y;
  }
  s_num[threadIdx.x] = num;
  s_den[threadIdx.x] = den;
  s_fin[threadIdx.x] = fin;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_num[threadIdx.x] += s_num[threadIdx.x + s];
      s_den[threadIdx.x] += s_den[threadIdx.x + s];
      s_fin[threadIdx.x] &= s_fin[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double e;
    if (s_den[0] == 0.0) e = NAN;
    else if (!s_fin[0]) e = INFINITY;
    else e = sqrt(s_num[0] / s_den[0]);
    err[b] = e;
  }
}

}  // namespace

int launch_widen(const void* in, double2* out, long long count, int precision,
                 cudaStream_t st) {
  const int grid = int(std::min<long long>((count + 255) / 256, 148LL * 16));
  widen_kernel<<<grid, 256, 0, st>>>(in, out, count, precision);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_rel_l2(const double2* y, const double2* r, double* err, long long n, long long batch,
                  cudaStream_t st) {
  rel_l2_kernel<<<unsigned(batch), 256, 0, st>>>(y, r, err, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

ErrorStats aggregate_errors(const std::vector<double>& errs) {
  ErrorStats s;
  std::vector<double> finite;
  finite.reserve(errs.size());
  for (double e : errs) {
    if (std::isnan(e)) {
      s.invalid = true;
    } else if (std::isfinite(e)) {
      finite.push_back(e);
      s.max = std::max(s.max, e);
    } else {
      ++s.nonfinite;
    }
  }
  if (finite.empty()) {
    s.median = INFINITY;
  } else {
    std::sort(finite.begin(), finite.end());
    const size_t mid = finite.size() / 2;
    s.median = finite.size() % 2 ? finite[mid] : (finite[mid - 1] + finite[mid]) / 2.0;
  }
  if (s.nonfinite) s.max = INFINITY;
  return s;
}

}  // namespace dsfft
