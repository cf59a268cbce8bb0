// stream_alloc.cuh -- stream-ordered scratch for executes that need
// intermediates (multipass, fp64, the N=2 fp16 tail).
//
// Plans are shareable across threads (fft.hpp:14-16); a per-plan scratch
// buffer would race when one plan runs on two streams at once.  Scratch is
// therefore allocated per call with cudaMallocAsync on the caller's stream and
// freed with cudaFreeAsync behind the last kernel that uses it.  The device's
// default pool is told to keep freed memory (release threshold = max), so a
// repeated execute reuses the same allocation without touching the driver.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>

namespace dsfft {

inline cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static std::set<int> configured;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!configured.count(dev)) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      configured.insert(dev);
    }
  }
  return cudaMallocAsync(ptr, bytes, stream);
}

inline void scratch_free(void* ptr, cudaStream_t stream) {
  if (ptr) cudaFreeAsync(ptr, stream);
}

}  // namespace dsfft
