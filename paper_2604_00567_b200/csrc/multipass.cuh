// multipass.cuh -- large-N (2^13 .. 2^24) path: the transform is split into
// two or three batched "column" / "row" kernels over HBM-resident
// intermediates (see multipass.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host_table.hpp"

namespace dsfft {

struct MultipassPlan;

MultipassPlan* multipass_create(const std::vector<TableEntry>& rounded_table, int m,
                                int strategy, int precision, int sm_count, size_t smem_optin);
void multipass_destroy(MultipassPlan* mp);
int multipass_execute(MultipassPlan& mp, bool inverse, const void* in, void* out, size_t batch,
                      uint32_t scale, cudaStream_t stream, uint64_t* launches);
const char* multipass_error();

}  // namespace dsfft
