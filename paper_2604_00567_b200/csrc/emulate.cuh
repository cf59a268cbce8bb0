// emulate.cuh -- the reference's scalar precision model and per-butterfly
// kernels on the device (see emulate.cu).
#pragma once
#include <cuda_runtime.h>

#include "../../include/dsfft.h"

namespace dsfft {

enum : int { kEmuFp16 = 0, kEmuFp32 = 1, kEmuFp64 = 2 };
enum : int { kEmuAdd = 0, kEmuSub = 1, kEmuMul = 2, kEmuFma = 3 };
enum : int { kEmuStandard = 0, kEmuLinzerFeig = 1, kEmuCosine = 2, kEmuDual = 3 };
using EmuEntry = dsfft_entry;

int launch_context_ops(int precision, int op, const double* a, const double* b, const double* c,
                       double* out, long long n, cudaStream_t stream);
int launch_butterflies(int strategy, int precision, const double2* a, const double2* b,
                       const EmuEntry* e, double* out, long long n, cudaStream_t stream);

}  // namespace dsfft
