// multipass.cu -- placeholder until the large-N kernels land.
#include <string>

#include "multipass.cuh"

namespace dsfft {

namespace {
thread_local std::string g_mp_err;
}

struct MultipassPlan {};

MultipassPlan* multipass_create(const std::vector<TableEntry>&, int, int, int, int, size_t) {
  g_mp_err = "N > 4096 (multi-pass) is not implemented yet";
  return nullptr;
}
void multipass_destroy(MultipassPlan* mp) { delete mp; }
int multipass_execute(MultipassPlan&, bool, const void*, void*, size_t, uint32_t, cudaStream_t,
                      uint64_t*) {
  g_mp_err = "N > 4096 (multi-pass) is not implemented yet";
  return 1;
}
const char* multipass_error() { return g_mp_err.c_str(); }

}  // namespace dsfft
