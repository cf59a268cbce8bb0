// synth.cu -- synthetic batches generated on the device from the GLOBAL
// transform index: sample s of transform b is a pure
// function of (seed, b, s), so a shard [b0, b0+count) generated on any GPU is
// bit-identical to the same rows of a 1-GPU batch -- the multi-GPU runs can be
// checked against the single-GPU one without moving data.
//
// Values follow the reference's distribution (uniform [-1, 1) from the top 53
// bits of a splitmix64 output, analysis.hpp:84-87), but each component is a
// counter-based hash instead of one sequential stream:
//   u = splitmix64_finalize(seed + golden * (2 (b n + s) + c + 1))
//   x = 2 (u >> 11) 2^-53 - 1, then rounded once into the working precision
// (binary16 / binary32 round-to-nearest-even from the double, as round_to).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "synth.cuh"

namespace dsfft {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform_pm1(uint64_t seed, uint64_t counter) {
  const uint64_t u = mix64(seed + 0x9E3779B97F4A7C15ull * (counter + 1));
  return 2.0 * (double(u >> 11) * 0x1p-53) - 1.0;
}

// one thread per complex sample; `first` = global index of the shard's first
// component (2 * first_transform * n)
__global__ void fill_uniform_kernel(void* out, long long count, uint64_t first, uint64_t seed,
                                    int precision) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t c = first + 2ull * uint64_t(i);
    const double re = uniform_pm1(seed, c), im = uniform_pm1(seed, c + 1);
    if (precision == 0) {
      reinterpret_cast<__half2*>(out)[i] = __halves2half2(__double2half(re), __double2half(im));
    } else if (precision == 1) {
      reinterpret_cast<float2*>(out)[i] = make_float2(__double2float_rn(re), __double2float_rn(im));
    } else {
      reinterpret_cast<double2*>(out)[i] = make_double2(re, im);
    }
  }
}

}  // namespace

int launch_fill_uniform(void* out, size_t n, uint64_t first_transform, size_t count,
                        uint64_t seed, int precision, int sm_count, cudaStream_t st) {
  const long long samples = (long long)(n * count);
  if (samples == 0) return 0;
  const int grid = int(std::min<long long>((samples + 255) / 256, (long long)sm_count * 16));
  fill_uniform_kernel<<<grid, 256, 0, st>>>(out, samples, 2ull * first_transform * n, seed,
                                            precision);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace dsfft
