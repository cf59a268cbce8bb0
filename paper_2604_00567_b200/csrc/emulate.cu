// emulate.cu -- the reference's scalar precision model and its per-butterfly
// kernels, evaluated on the device (batched, one thread per element).
//
// The reference exposes two fine-grained APIs besides plan/execute:
//   * ArithmeticContext::add / sub / mul / fma (precision.cpp:77-111): a
//     double carrier rounded after every operation into the context precision;
//   * the butterfly-variant plugin point: butterfly_standard / _linzer_feig /
//     _cosine / _dual and kernel_for (butterfly.hpp:22-61, butterfly.cpp).
// This library has no CPU arithmetic, so both run here, on arrays of
// arguments, with the reference's exact rounding for ANY double inputs (not
// only representable ones):
//   fp16: round_to(op in double)            -- DADD / DMUL / DFMA, then RNE to
//                                              binary16 with round_to's
//                                              overflow (|x| >= 65520 -> inf),
//                                              zero and NaN pass-through;
//   fp32: op on the float-cast operands     -- FADD / FMUL / FFMA;
//   fp64: the double op                     -- DADD / DMUL / DFMA.
// The FFT kernels never use this path: they work in the native formats,
// where HFMA2 / FFMA lanes equal these roundings.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "emulate.cuh"

namespace dsfft {

namespace {

// round_to (precision.cpp:61-75)
__device__ __forceinline__ double round_to_dev(double x, int p) {
  if (p == kEmuFp64 || x == 0.0 || isnan(x)) return x;
  const double ax = fabs(x);
  if (p == kEmuFp16) {
    if (ax >= 65520.0) return copysign(INFINITY, x);
    return double(__half2float(__double2half(x)));  // RNE, one rounding (cvt.rn.f16.f64)
  }
  if (ax >= 0x1.ffffffp+127) return copysign(INFINITY, x);
  return double(__double2float_rn(x));
}

// ArithmeticContext's rounded operations at precision p
struct Ctx {
  int p;
  __device__ double add(double a, double b) const {
    if (p == kEmuFp32) return double(__fadd_rn(__double2float_rn(a), __double2float_rn(b)));
    return round_to_dev(__dadd_rn(a, b), p);
  }
  __device__ double sub(double a, double b) const {
    if (p == kEmuFp32) return double(__fsub_rn(__double2float_rn(a), __double2float_rn(b)));
    return round_to_dev(__dsub_rn(a, b), p);
  }
  __device__ double mul(double a, double b) const {
    if (p == kEmuFp32) return double(__fmul_rn(__double2float_rn(a), __double2float_rn(b)));
    return round_to_dev(__dmul_rn(a, b), p);
  }
  __device__ double fma(double a, double b, double c) const {
    if (p == kEmuFp32)
      return double(
          __fmaf_rn(__double2float_rn(a), __double2float_rn(b), __double2float_rn(c)));
    return round_to_dev(__fma_rn(a, b, c), p);
  }
};

__global__ void context_ops_kernel(int p, int op, const double* a, const double* b,
                                   const double* c, double* out, long long n) {
  const Ctx ctx{p};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double r;
    switch (op) {
      case kEmuAdd: r = ctx.add(a[i], b[i]); break;
      case kEmuSub: r = ctx.sub(a[i], b[i]); break;
      case kEmuMul: r = ctx.mul(a[i], b[i]); break;
      default: r = ctx.fma(a[i], b[i], c[i]); break;
    }
    out[i] = r;
  }
}

// The 6-FMA cores with the ratio t and outer multiplier w of the entry the
// variant selects: COS form s1 = b.re - t b.im, s2 = b.im + t b.re,
// A = a + w (s1, s2); SIN form s1 = b.im - t b.re, s2 = b.re + t b.im,
// A = a + w (-s1, s2); B mirrors A.  (butterfly.hpp:27-47)
__device__ void fma_core(const Ctx& x, bool cos_form, double t, double w, double2 a, double2 b,
                         double* o) {
  const double p = cos_form ? b.y : b.x, q = cos_form ? b.x : b.y;  // (inner, addend)
  const double s1 = x.fma(-t, p, q);
  const double s2 = x.fma(t, q, p);
  if (cos_form) {
    o[0] = x.fma(s1, w, a.x);
    o[1] = x.fma(s2, w, a.y);
    o[2] = x.fma(-s1, w, a.x);
    o[3] = x.fma(-s2, w, a.y);
  } else {
    o[0] = x.fma(-s1, w, a.x);
    o[1] = x.fma(s2, w, a.y);
    o[2] = x.fma(s1, w, a.x);
    o[3] = x.fma(-s2, w, a.y);
  }
}

__global__ void butterflies_kernel(int strategy, int p, const double2* a, const double2* b,
                                   const EmuEntry* e, double* out, long long n) {
  const Ctx x{p};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const EmuEntry en = e[i];
    double* o = out + 4 * i;
    const double2 ai = a[i], bi = b[i];
    if (strategy == kEmuStandard) {  // 4 rounded mul, 6 rounded add / sub
      const double rr = x.mul(en.omega_r, bi.x), ii = x.mul(en.omega_i, bi.y);
      const double ir = x.mul(en.omega_i, bi.x), ri = x.mul(en.omega_r, bi.y);
      const double tr = x.sub(rr, ii), ti = x.add(ir, ri);
      o[0] = x.add(ai.x, tr);
      o[1] = x.add(ai.y, ti);
      o[2] = x.sub(ai.x, tr);
      o[3] = x.sub(ai.y, ti);
    } else if (strategy == kEmuLinzerFeig && en.clamped) {
      // the clamped k = 0 entry keeps W = 1 exact through the COS form on
      // its true (omega_r, omega_i)
      fma_core(x, true, en.omega_i, en.omega_r, ai, bi, o);
    } else {
      const bool cos_form = strategy == kEmuCosine ||
                            (strategy == kEmuDual && en.path == 0);  // LF: always SIN
      fma_core(x, cos_form, en.ratio, en.multiplier, ai, bi, o);
    }
  }
}

int grid_for(long long n) { return int(std::max(1LL, std::min((n + 127) / 128, 148LL * 8))); }

}  // namespace

int launch_context_ops(int precision, int op, const double* a, const double* b, const double* c,
                       double* out, long long n, cudaStream_t st) {
  context_ops_kernel<<<grid_for(n), 128, 0, st>>>(precision, op, a, b, c, out, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_butterflies(int strategy, int precision, const double2* a, const double2* b,
                       const EmuEntry* e, double* out, long long n, cudaStream_t st) {
  butterflies_kernel<<<grid_for(n), 128, 0, st>>>(strategy, precision, a, b, e, out, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace dsfft
