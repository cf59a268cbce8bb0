// fmafft_b200.hpp -- C++ drop-in for the reference's plan/execute API
// (fmafft: /root/reference/proj/core/include/fmafft/{precision,twiddle,
// butterfly,fft}.hpp), header-only over the C ABI in dsfft.h.
//
// Same type names, fields, signatures, argument meaning and exceptions as the
// reference, so a caller switches with
//     #include "fmafft_b200.hpp"
//     namespace fmafft = fmafft_b200;
// and links libdsfft.so.  Differences a caller can observe:
//   * forward/inverse run on the plan's B200; fp32 and fp16 results are
//     bit-identical to the reference (its ArithmeticContext rounding).
//   * ArithmeticContext counters are advanced analytically by the exact
//     counts the reference's kernels would have issued (6 FMAs per butterfly,
//     4 mul + 6 add for standard, 2n muls for the inverse scaling), since the
//     hardware FMAs are not routed through the context.
//   * fp64 plans build their table but forward/inverse throw
//     std::runtime_error (the device path is fp16/fp32).
//   * Batched overloads (forward_batch / inverse_batch) transform many
//     SampleBuffers in one call; device-buffer execution is dsfft_execute.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dsfft.h"

namespace fmafft_b200 {

// precision.hpp:12-62
enum class Precision { fp16, fp32, fp64 };

inline double machine_epsilon(Precision p) {
  return p == Precision::fp16 ? 0x1p-11 : p == Precision::fp32 ? 0x1p-24 : 0x1p-53;
}
inline std::string_view to_string(Precision p) {
  return p == Precision::fp16 ? "fp16" : p == Precision::fp32 ? "fp32" : "fp64";
}
inline Precision parse_precision(std::string_view name) {
  if (name == "fp16") return Precision::fp16;
  if (name == "fp32") return Precision::fp32;
  if (name == "fp64") return Precision::fp64;
  throw std::invalid_argument("unknown precision: " + std::string(name));
}

struct OpCounter {
  std::uint64_t fma_count = 0;
  std::uint64_t add_count = 0;
  std::uint64_t mul_count = 0;
  void reset() { fma_count = add_count = mul_count = 0; }
};

class ArithmeticContext {
 public:
  explicit ArithmeticContext(Precision p) : precision_(p) {}
  Precision precision() const { return precision_; }
  const OpCounter& counters() const { return counters_; }
  void reset_counters() { counters_.reset(); }
  // analytic accounting used by forward/inverse below
  void account(std::uint64_t fma, std::uint64_t add, std::uint64_t mul) {
    counters_.fma_count += fma;
    counters_.add_count += add;
    counters_.mul_count += mul;
  }

 private:
  Precision precision_;
  OpCounter counters_;
};

// twiddle.hpp:12-75
enum class TwiddlePath { cos, sin };
enum class Strategy { standard, linzer_feig, cosine, dual_select };

inline std::string_view to_string(Strategy s) {
  switch (s) {
    case Strategy::standard: return "standard";
    case Strategy::linzer_feig: return "lf";
    case Strategy::cosine: return "cosine";
    case Strategy::dual_select: return "dual";
  }
  return "standard";
}
inline std::string_view to_string(TwiddlePath p) { return p == TwiddlePath::cos ? "COS" : "SIN"; }
inline Strategy parse_strategy(std::string_view name) {
  if (name == "standard") return Strategy::standard;
  if (name == "lf" || name == "linzer-feig" || name == "linzer_feig") return Strategy::linzer_feig;
  if (name == "cosine") return Strategy::cosine;
  if (name == "dual" || name == "dual-select" || name == "dual_select") return Strategy::dual_select;
  throw std::invalid_argument("unknown strategy: " + std::string(name));
}

struct TwiddleEntry {
  double multiplier = 0.0;
  double ratio = 0.0;
  TwiddlePath path = TwiddlePath::cos;
  double omega_r = 0.0;
  double omega_i = 0.0;
  bool clamped = false;
};

struct TwiddleTable {
  std::size_t n = 0;
  Strategy strategy = Strategy::standard;
  std::vector<TwiddleEntry> entries;
};

// butterfly.hpp:8-17
struct ComplexSample {
  double re = 0.0;
  double im = 0.0;
};
struct ButterflyResult {
  ComplexSample sum;
  ComplexSample diff;
};

// fft.hpp:12-44
using SampleBuffer = std::vector<ComplexSample>;

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string msg = dsfft_last_error();
  if (rc == DSFFT_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void check(int rc) {
  if (rc != DSFFT_OK) raise(rc);
}
inline TwiddleTable to_table(std::size_t n, Strategy s, const std::vector<dsfft_entry>& raw) {
  TwiddleTable t;
  t.n = n;
  t.strategy = s;
  t.entries.resize(raw.size());
  for (std::size_t k = 0; k < raw.size(); ++k) {
    const dsfft_entry& e = raw[k];
    t.entries[k] = TwiddleEntry{e.multiplier, e.ratio, e.path ? TwiddlePath::sin : TwiddlePath::cos,
                                e.omega_r, e.omega_i, e.clamped != 0};
  }
  return t;
}
struct PlanDeleter {
  void operator()(dsfft_plan p) const { dsfft_plan_destroy(p); }
};
}  // namespace detail

// Host-only table builders (twiddle.cpp:59-141): FP64, unrounded.
inline TwiddleTable build_table(std::size_t n, Strategy s, double clamp_eps = 1e-7) {
  std::vector<dsfft_entry> raw(n / 2 ? n / 2 : 1);
  detail::check(dsfft_build_table(n, int(s), DSFFT_FP64, clamp_eps, raw.data(), raw.size()));
  raw.resize(n / 2);
  return detail::to_table(n, s, raw);
}
inline TwiddleTable build_standard_table(std::size_t n) { return build_table(n, Strategy::standard); }
inline TwiddleTable build_linzer_feig_table(std::size_t n, double clamp_eps = 1e-7) {
  return build_table(n, Strategy::linzer_feig, clamp_eps);
}
inline TwiddleTable build_cosine_table(std::size_t n) { return build_table(n, Strategy::cosine); }
inline TwiddleTable build_dual_select_table(std::size_t n) {
  return build_table(n, Strategy::dual_select);
}

// precision.cpp:61-75
inline double round_to(double x, Precision p) {
  if (p == Precision::fp64) return x;
  double out = 0.0;
  if (p == Precision::fp16) {
    std::uint16_t h;
    detail::check(dsfft_round_to(&x, &h, 1, DSFFT_FP16));
    detail::check(dsfft_widen(&h, &out, 1, DSFFT_FP16));
  } else {
    float f;
    detail::check(dsfft_round_to(&x, &f, 1, DSFFT_FP32));
    out = double(f);
  }
  return out;
}

// Immutable execution recipe (fft.hpp:17-23) plus the device plan it owns.
struct FftPlan {
  std::size_t n = 0;
  unsigned m = 0;
  Strategy strategy = Strategy::standard;
  Precision precision = Precision::fp64;
  TwiddleTable table;
  std::shared_ptr<std::remove_pointer_t<dsfft_plan>> device;  // shared, immutable
  dsfft_plan handle() const { return device.get(); }
};

// fft.cpp:56-72: n a power of two in [2, 2^24]; the table is built in FP64
// and every scalar rounded once into the working precision.
inline FftPlan make_plan(std::size_t n, Strategy strategy, Precision precision,
                         int device = 0) {
  dsfft_plan h = nullptr;
  detail::check(dsfft_plan_create(n, int(strategy), int(precision), 1e-7, device, &h));
  FftPlan p;
  p.device.reset(h, detail::PlanDeleter{});
  unsigned m = 0;
  detail::check(dsfft_plan_info(h, &p.n, &m, nullptr, nullptr));
  p.m = m;
  p.strategy = strategy;
  p.precision = precision;
  std::vector<dsfft_entry> raw(n / 2 ? n / 2 : 1);
  detail::check(dsfft_plan_table(h, raw.data(), raw.size()));
  raw.resize(n / 2);
  p.table = detail::to_table(n, strategy, raw);
  return p;
}

namespace detail {
inline void check_call(const FftPlan& plan, std::size_t len, const ArithmeticContext& ctx) {
  if (len != plan.n)  // fft.cpp:16-21
    throw std::invalid_argument("buffer length " + std::to_string(len) +
                                " does not match plan size " + std::to_string(plan.n));
  if (ctx.precision() != plan.precision)  // fft.cpp:23-26
    throw std::invalid_argument("context precision does not match plan");
}
inline void account(const FftPlan& plan, ArithmeticContext& ctx, std::size_t batch, bool inv) {
  const std::uint64_t bf = std::uint64_t(plan.n / 2) * plan.m * batch;
  if (plan.strategy == Strategy::standard)
    ctx.account(0, 6 * bf, 4 * bf);
  else
    ctx.account(6 * bf, 0, 0);
  if (inv) ctx.account(0, 0, 2 * std::uint64_t(plan.n) * batch);
}
inline std::vector<SampleBuffer> run(const FftPlan& plan, const std::vector<SampleBuffer>& xs,
                                     ArithmeticContext& ctx, int dir) {
  for (const auto& x : xs) check_call(plan, x.size(), ctx);
  std::vector<double> in(2 * plan.n * xs.size()), out(in.size());
  for (std::size_t b = 0; b < xs.size(); ++b)
    for (std::size_t i = 0; i < plan.n; ++i) {
      in[2 * (b * plan.n + i)] = xs[b][i].re;
      in[2 * (b * plan.n + i) + 1] = xs[b][i].im;
    }
  check(dsfft_execute_f64(plan.handle(), dir, in.data(), out.data(), xs.size()));
  std::vector<SampleBuffer> ys(xs.size(), SampleBuffer(plan.n));
  for (std::size_t b = 0; b < xs.size(); ++b)
    for (std::size_t i = 0; i < plan.n; ++i)
      ys[b][i] = ComplexSample{out[2 * (b * plan.n + i)], out[2 * (b * plan.n + i) + 1]};
  account(plan, ctx, xs.size(), dir == DSFFT_INVERSE);
  return ys;
}
}  // namespace detail

// fft.hpp:33-34: out-of-place Stockham DIT forward, ingest-rounded input.
inline SampleBuffer forward(const FftPlan& plan, const SampleBuffer& input,
                            ArithmeticContext& ctx) {
  return detail::run(plan, {input}, ctx, DSFFT_FORWARD)[0];
}

// fft.hpp:38-39: conj -> forward -> conj * round_to(1/n).
inline SampleBuffer inverse(const FftPlan& plan, const SampleBuffer& spectrum,
                            ArithmeticContext& ctx) {
  return detail::run(plan, {spectrum}, ctx, DSFFT_INVERSE)[0];
}

// Batched extensions: one device call for many transforms.
inline std::vector<SampleBuffer> forward_batch(const FftPlan& plan,
                                               const std::vector<SampleBuffer>& inputs,
                                               ArithmeticContext& ctx) {
  return detail::run(plan, inputs, ctx, DSFFT_FORWARD);
}
inline std::vector<SampleBuffer> inverse_batch(const FftPlan& plan,
                                               const std::vector<SampleBuffer>& spectra,
                                               ArithmeticContext& ctx) {
  return detail::run(plan, spectra, ctx, DSFFT_INVERSE);
}

}  // namespace fmafft_b200
