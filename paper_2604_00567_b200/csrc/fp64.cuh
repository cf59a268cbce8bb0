// fp64.cuh -- Precision::fp64 device path (see fp64.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host_table.hpp"

namespace dsfft {

struct F64Plan;

F64Plan* fp64_create(const std::vector<TableEntry>& table, int m, int strategy);
void fp64_destroy(F64Plan* fp);
int fp64_execute(F64Plan& fp, bool inverse, const void* in, void* out, size_t batch,
                 double scale, int sm_count, cudaStream_t stream, uint64_t* launches);
const char* fp64_error();

}  // namespace dsfft
