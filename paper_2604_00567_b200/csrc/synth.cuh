// synth.cuh -- device synthetic batches keyed by the global transform index (see synth.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace dsfft {

int launch_fill_uniform(void* out, size_t n, uint64_t first_transform, size_t count,
                        uint64_t seed, int precision, int sm_count, cudaStream_t stream);

}  // namespace dsfft
