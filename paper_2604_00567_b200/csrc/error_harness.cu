// error_harness.cu -- device error measurement.
//
// Mirrors measure_error (analysis.cpp:101-154) over a whole device batch:
//   forward_vs_oracle: rel-L2 of the working-precision forward against the
//     FP64 DFT of the same (ingested) input;
//   roundtrip: rel-L2 of inverse(forward(x)) against x;
// per transform (relative_l2_error, analysis.cpp:41-57: +inf when the result
// has a non-finite component), then median over finite transforms, max (+inf
// if any is non-finite) and the non-finite count (analysis.cpp:16-22,142-152).
//
// Both pieces are bit-identical to the reference, not just close:
//   dft_kernel      == dft_oracle (fft.cpp:103-121): the cos/sin of every
//                      residue r = (j k) mod n is tabulated on the host with
//                      the reference's own expression and libm; each output j
//                      accumulates k = 0, 1, ..., n-1 in order with separately
//                      rounded __dmul_rn / __dsub_rn / __dadd_rn (the
//                      reference builds with -ffp-contract=off);
//   rel_l2_seq      == relative_l2_error: one thread per transform, the same
//                      sequential sums, __ddiv_rn / __dsqrt_rn.
// So dsfft_measure_error reports equal the reference's bit for bit
// ("Equal arguments give bit-identical reports", analysis.hpp:96-97).  For
// n > kDftMaxN the O(n^2) DFT is replaced by this library's fp64 FFT (DFMA
// passes, bit-identical to the reference's fp64 forward, within 1e-11 of the
// DFT: test_fft.cpp:110-128) unless the caller asks for the DFT explicitly.
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

// relative_l2_error(y, r) per transform, the reference's sequential sums:
//   num += dr*dr + di*di; den += r.re*r.re + r.im*r.im   (analysis.cpp:46-53)
// err = sqrt(num / den); +inf if y has a non-finite component; kZeroRef when
// den == 0 (the reference throws "all-zero reference" -- checked first).
__global__ void rel_l2_seq_kernel(const double2* __restrict__ y, const double2* __restrict__ r,
                                  double* __restrict__ err, long long n, long long batch) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double2* yb = y + b * n;
  const double2* rb = r + b * n;
  double num = 0.0, den = 0.0;
  bool fin = true;
#pragma unroll 4
  for (long long i = 0; i < n; ++i) {
    const double2 a = yb[i], c = rb[i];
    if (!isfinite(a.x) || !isfinite(a.y)) fin = false;
    const double dr = __dsub_rn(a.x, c.x);
    const double di = __dsub_rn(a.y, c.y);
    num = __dadd_rn(num, __dadd_rn(__dmul_rn(dr, dr), __dmul_rn(di, di)));
    den = __dadd_rn(den, __dadd_rn(__dmul_rn(c.x, c.x), __dmul_rn(c.y, c.y)));
  }
  double e;
  if (den == 0.0) e = kZeroReference;
  else if (!fin) e = INFINITY;
  else e = __dsqrt_rn(__ddiv_rn(num, den));
  err[b] = e;
}

// dft_oracle (fft.cpp:103-121) for `batch` transforms of length n (any n).
// One CTA per transform (grid-stride over the batch); thread t owns outputs
// j = t + blockDim*i (JT of them in registers, sharing each x[k] load).
// r_j = (j k) mod n advances by j per k.  With SMEM the transform and the
// twiddle table sit in shared memory (n <= kDftSmemN), else both are read
// through L1 / L2.
template <int JT, bool SMEM>
__global__ void __launch_bounds__(256) dft_kernel(const double2* __restrict__ x,
                                                  double2* __restrict__ y,
                                                  const double2* __restrict__ tw, int n,
                                                  long long batch) {
  extern __shared__ double2 sm[];
  const double2* ts = tw;
  if constexpr (SMEM) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[n + i] = tw[i];
    ts = sm + n;
  }
  for (long long b = blockIdx.x; b < batch; b += gridDim.x) {
    const double2* xs = x + b * n;
    if constexpr (SMEM) {
      __syncthreads();  // previous transform's reads are done
      for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = xs[i];
      __syncthreads();
      xs = sm;
    }
    for (int j0 = threadIdx.x; j0 < n; j0 += blockDim.x * JT) {
      double ar[JT], ai[JT];
      int jj[JT], js[JT], r[JT];
#pragma unroll
      for (int t = 0; t < JT; ++t) {
        jj[t] = j0 + t * int(blockDim.x);
        js[t] = jj[t] < n ? jj[t] : 0;  // outputs past n: keep r in range, never stored
        ar[t] = 0.0;
        ai[t] = 0.0;
        r[t] = 0;
      }
      for (int k = 0; k < n; ++k) {
        const double2 v = xs[k];
#pragma unroll
        for (int t = 0; t < JT; ++t) {
          const double2 w = ts[r[t]];  // (cos, sin) of theta_{(j k) mod n}
          // acc_re += re*c - im*s; acc_im += re*s + im*c, each op rounded
          ar[t] = __dadd_rn(ar[t], __dsub_rn(__dmul_rn(v.x, w.x), __dmul_rn(v.y, w.y)));
          ai[t] = __dadd_rn(ai[t], __dadd_rn(__dmul_rn(v.x, w.y), __dmul_rn(v.y, w.x)));
          r[t] += js[t];
          if (r[t] >= n) r[t] -= n;
        }
      }
#pragma unroll
      for (int t = 0; t < JT; ++t)
        if (jj[t] < n) y[b * n + jj[t]] = make_double2(ar[t], ai[t]);
    }
  }
}

template <int JT>
cudaError_t dft_go(const double2* x, double2* y, const double2* tw, int n, long long batch,
                   int threads, int grid, cudaStream_t st) {
  if (n <= kDftSmemN) {
    const size_t smem = size_t(2) * n * sizeof(double2);
    auto kern = dft_kernel<JT, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(x, y, tw, n, batch);
  } else {
    dft_kernel<JT, false><<<grid, threads, 0, st>>>(x, y, tw, n, batch);
  }
  return cudaGetLastError();
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
  const unsigned grid = unsigned((batch + 127) / 128);
  rel_l2_seq_kernel<<<grid, 128, 0, st>>>(y, r, err, n, batch);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_dft(const double2* x, double2* y, const double2* tw, long long n, long long batch,
               int sm_count, cudaStream_t st) {
  if (n < 1 || n > (1LL << 24)) return 1;
  if (batch == 0) return 0;
  const int threads = int(std::min<long long>(256, (n + 31) / 32 * 32));
  const long long per_thread = (n + threads - 1) / threads;
  const int grid = int(std::min<long long>(batch, (long long)sm_count * 8));
  cudaError_t e;
  if (per_thread >= 8) e = dft_go<8>(x, y, tw, int(n), batch, threads, grid, st);
  else if (per_thread >= 4) e = dft_go<4>(x, y, tw, int(n), batch, threads, grid, st);
  else if (per_thread >= 2) e = dft_go<2>(x, y, tw, int(n), batch, threads, grid, st);
  else e = dft_go<1>(x, y, tw, int(n), batch, threads, grid, st);
  return e == cudaSuccess ? 0 : 1;
}

ErrorStats aggregate_errors(const std::vector<double>& errs) {
  // measure_error's aggregation (analysis.cpp:142-152): finite errors feed the
  // median and max; any non-finite error counts and makes the max +inf
  ErrorStats s;
  std::vector<double> finite;
  finite.reserve(errs.size());
  for (double e : errs) {
    if (e == kZeroReference) {
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
