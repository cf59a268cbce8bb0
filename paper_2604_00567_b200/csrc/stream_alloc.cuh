// stream_alloc.cuh -- stream-ordered scratch for executes that need
// intermediates (multipass, fp64, the N=2 fp16 tail, the DFT table).
//
// Plans are shareable across threads (fft.hpp:14-16); a per-plan scratch
// buffer would race when one plan runs on two streams at once.  Scratch is
// therefore allocated per call on the caller's stream and freed behind the
// last kernel that uses it.  It comes from a memory pool the library owns
// (one per device, created on first use): the pool keeps freed blocks, so a
// repeated execute reuses the same memory without touching the driver, and
// the device's default pool -- shared with the rest of the process -- is left
// alone.  dsfft_plan_destroy trims the library pool (scratch_trim), returning
// every block that no call still holds.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>

namespace dsfft {

inline std::mutex& scratch_mutex() {
  static std::mutex mu;
  return mu;
}
inline std::map<int, cudaMemPool_t>& scratch_pools() {
  static std::map<int, cudaMemPool_t> pools;
  return pools;
}

inline cudaError_t scratch_pool(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lock(scratch_mutex());
  auto& pools = scratch_pools();
  auto it = pools.find(dev);
  if (it != pools.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  cudaError_t e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;  // keep freed blocks for the next call (trimmed on destroy)
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  pools[dev] = pool;
  *out = pool;
  return cudaSuccess;
}

inline cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = scratch_pool(dev, &pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
}

inline void scratch_free(void* ptr, cudaStream_t stream) {
  if (ptr) cudaFreeAsync(ptr, stream);
}

// Release the library pool's unused blocks on `dev` (blocks whose
// stream-ordered free has not executed yet are released by the next trim).
inline void scratch_trim(int dev) {
  std::lock_guard<std::mutex> lock(scratch_mutex());
  auto& pools = scratch_pools();
  auto it = pools.find(dev);
  if (it != pools.end()) cudaMemPoolTrimTo(it->second, 0);
}

}  // namespace dsfft
