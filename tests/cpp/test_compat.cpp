// test_compat.cpp -- the C++ drop-in (include/fmafft_b200.hpp) exercised the
// way the reference's own doctest suites exercise fmafft (tests/test_fft.cpp,
// test_twiddle.cpp), via `namespace fmafft = fmafft_b200`.
//   ./test_compat host     table/precision/error checks (no GPU needed)
//   ./test_compat          everything (needs a B200)
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <stdexcept>

#include "fmafft_b200.hpp"

namespace fmafft = fmafft_b200;
using namespace fmafft;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    ++g_checks;                                                   \
    if (!(c)) {                                                   \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
    }                                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, T)        \
  do {                                  \
    bool caught_ = false;               \
    try {                               \
      (void)(expr);                     \
    } catch (const T&) {                \
      caught_ = true;                   \
    } catch (...) {                     \
    }                                   \
    CHECK(caught_);                     \
  } while (0)

// SplitMix64 uniform_pm1 stream (analysis.hpp:73-91)
static SampleBuffer random_buffer(std::size_t n, std::uint64_t seed) {
  std::uint64_t s = seed;
  auto next = [&] {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  SampleBuffer x(n);
  for (auto& c : x) {
    c.re = 2.0 * (double(next() >> 11) * 0x1p-53) - 1.0;
    c.im = 2.0 * (double(next() >> 11) * 0x1p-53) - 1.0;
  }
  return x;
}

static double rel_l2(const SampleBuffer& x, const SampleBuffer& y) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    if (!std::isfinite(x[i].re) || !std::isfinite(x[i].im)) return INFINITY;
    num += (x[i].re - y[i].re) * (x[i].re - y[i].re) + (x[i].im - y[i].im) * (x[i].im - y[i].im);
    den += y[i].re * y[i].re + y[i].im * y[i].im;
  }
  return std::sqrt(num / den);
}

static SampleBuffer dft(const SampleBuffer& x) {  // FP64 O(n^2) (fft.cpp:103-121)
  const std::size_t n = x.size();
  SampleBuffer out(n);
  for (std::size_t j = 0; j < n; ++j) {
    double ar = 0, ai = 0;
    for (std::size_t k = 0; k < n; ++k) {
      const double th = -(2.0 * 3.141592653589793 / double(n)) * double((j * k) % n);
      ar += x[k].re * std::cos(th) - x[k].im * std::sin(th);
      ai += x[k].re * std::sin(th) + x[k].im * std::cos(th);
    }
    out[j] = {ar, ai};
  }
  return out;
}

static void host_checks() {
  // test_twiddle.cpp:26-33 size validation
  CHECK_THROWS_AS(build_standard_table(0), std::invalid_argument);
  CHECK_THROWS_AS(build_dual_select_table(1023), std::invalid_argument);
  CHECK_THROWS_AS(build_linzer_feig_table(8, 0.0), std::invalid_argument);
  // test_twiddle.cpp:54-108
  const TwiddleTable lf = build_linzer_feig_table(1024);
  CHECK(lf.entries[0].clamped && lf.entries[0].multiplier == -1e-7);
  CHECK(std::signbit(lf.entries[0].omega_i));
  CHECK(std::fabs(std::fabs(lf.entries[1].ratio) - 163.0) < 0.1);
  const TwiddleTable du = build_dual_select_table(1024);
  CHECK(du.entries[0].path == TwiddlePath::cos && du.entries[0].ratio == 0.0);
  CHECK(du.entries[128].path == TwiddlePath::cos);
  CHECK(du.entries[256].path == TwiddlePath::sin && du.entries[256].multiplier == -1.0);
  for (const auto& e : du.entries) CHECK(std::fabs(e.ratio) <= 1.0);
  // precision KATs (acceptance.cpp:296-305)
  CHECK(round_to(65519.999, Precision::fp16) == 65504.0);
  CHECK(std::isinf(round_to(65520.0, Precision::fp16)));
  CHECK(round_to(0x1p-25, Precision::fp16) == 0.0);
  CHECK(round_to(0x1.8p-24, Precision::fp16) == 0x1p-23);
  CHECK(parse_strategy("dual-select") == Strategy::dual_select);
  CHECK_THROWS_AS(parse_strategy("radix4"), std::invalid_argument);
  CHECK_THROWS_AS(parse_precision("bf16"), std::invalid_argument);
  CHECK_THROWS_AS(make_plan(1023, Strategy::standard, Precision::fp32), std::invalid_argument);
  CHECK_THROWS_AS(make_plan(std::size_t{1} << 25, Strategy::standard, Precision::fp32),
                  std::invalid_argument);
}

static void device_checks() {
  // acceptance.cpp:209-242 / test_analysis.cpp:144-172 through measure_error:
  // fp16 dual beats LF with the clamp, within the paper's cumulative bound
  {
    const ErrorReport d =
        measure_error(1024, Strategy::dual_select, Precision::fp16, ErrorMetric::forward_vs_oracle,
                      10, 42);
    const ErrorReport lf =
        measure_error(1024, Strategy::linzer_feig, Precision::fp16, ErrorMetric::forward_vs_oracle,
                      10, 42);
    CHECK(d.trials == 10 && d.nonfinite_trials == 0 && lf.nonfinite_trials == 0);
    CHECK(d.rel_l2_median < lf.rel_l2_median);
    CHECK(d.rel_l2_max <= reproduce_cumulative_table(1024)[1].cumulative_bound);
    const ErrorReport rt = measure_error(1024, Strategy::dual_select, Precision::fp32,
                                         ErrorMetric::roundtrip, 20, 42);
    CHECK(rt.rel_l2_median > 1e-8 && rt.rel_l2_median < 1e-6);  // acceptance.cpp:185-205
    std::ostringstream os;
    write_error_csv(os, rt);
    CHECK(os.str().rfind("n,strategy,precision,metric,trials,seed,", 0) == 0);
    CHECK(os.str().find("\n1024,dual,fp32,roundtrip,20,42,") != std::string::npos);
    CHECK_THROWS_AS(measure_error(64, Strategy::dual_select, Precision::fp16,
                                  ErrorMetric::roundtrip, 0, 1),
                    std::invalid_argument);
  }
  // test_fft.cpp:33-61 plan construction and table rounding
  const FftPlan p = make_plan(1024, Strategy::dual_select, Precision::fp16);
  CHECK(p.n == 1024 && p.m == 10 && p.table.entries.size() == 512);
  for (const auto& e : p.table.entries) CHECK(std::fabs(e.ratio) <= 1.0);
  const FftPlan p16 = make_plan(64, Strategy::cosine, Precision::fp16);
  const TwiddleTable t64 = build_cosine_table(64);
  for (std::size_t k = 0; k < 32; ++k)
    CHECK(p16.table.entries[k].ratio == round_to(t64.entries[k].ratio, Precision::fp16));

  // forward basics (test_fft.cpp:63-86), fp32 on the device
  const FftPlan p4 = make_plan(4, Strategy::standard, Precision::fp32);
  ArithmeticContext ctx(Precision::fp32);
  SampleBuffer dc{{1, 0}, {1, 0}, {1, 0}, {1, 0}};
  SampleBuffer spec = forward(p4, dc, ctx);
  CHECK(spec[0].re == 4.0);
  for (int j = 1; j < 4; ++j) CHECK(std::fabs(spec[j].re) < 1e-6 && std::fabs(spec[j].im) < 1e-6);
  SampleBuffer wrong(3);
  CHECK_THROWS_AS(forward(p4, wrong, ctx), std::invalid_argument);
  ArithmeticContext ctx16(Precision::fp16);
  CHECK_THROWS_AS(forward(p4, dc, ctx16), std::invalid_argument);

  // oracle agreement at fp32 for every strategy (test_fft.cpp:110-128 at fp32)
  for (std::size_t n = 2; n <= 512; n <<= 1) {
    const SampleBuffer x = random_buffer(n, 1000 + n);
    const SampleBuffer ref = dft(x);
    for (Strategy s : {Strategy::standard, Strategy::linzer_feig, Strategy::cosine,
                       Strategy::dual_select}) {
      ArithmeticContext c(Precision::fp32);
      CHECK(rel_l2(forward(make_plan(n, s, Precision::fp32), x, c), ref) < 1e-6);
    }
  }

  // op accounting (test_fft.cpp:130-149) and inverse scaling (180-189)
  for (std::size_t n : {2ul, 64ul, 1024ul}) {
    const std::uint64_t bf = std::uint64_t(n / 2) * std::uint64_t(std::countr_zero(n));
    const SampleBuffer x = random_buffer(n, n);
    for (Strategy s : {Strategy::linzer_feig, Strategy::cosine, Strategy::dual_select}) {
      ArithmeticContext c(Precision::fp32);
      forward(make_plan(n, s, Precision::fp32), x, c);
      CHECK(c.counters().fma_count == 6 * bf && c.counters().mul_count == 0 &&
            c.counters().add_count == 0);
    }
    ArithmeticContext c(Precision::fp32);
    forward(make_plan(n, Strategy::standard, Precision::fp32), x, c);
    CHECK(c.counters().mul_count == 4 * bf && c.counters().add_count == 6 * bf);
  }
  {
    ArithmeticContext c(Precision::fp32);
    inverse(make_plan(64, Strategy::dual_select, Precision::fp32), random_buffer(64, 5), c);
    CHECK(c.counters().fma_count == 6 * 32 * 6 && c.counters().mul_count == 2 * 64);
  }

  // roundtrip (test_fft.cpp:151-178 at fp32) and the batched extension
  for (std::size_t n = 2; n <= 4096; n <<= 2) {
    const FftPlan pl = make_plan(n, Strategy::dual_select, Precision::fp32);
    ArithmeticContext c(Precision::fp32);
    const SampleBuffer in = random_buffer(n, 31 * n);
    SampleBuffer ing(in.size());
    for (std::size_t i = 0; i < n; ++i)
      ing[i] = {round_to(in[i].re, Precision::fp32), round_to(in[i].im, Precision::fp32)};
    CHECK(rel_l2(inverse(pl, forward(pl, in, c), c), ing) < 1e-5);
    const auto ys = forward_batch(pl, {in, in, in}, c);
    const SampleBuffer y0 = forward(pl, in, c);
    CHECK(ys.size() == 3 && std::memcmp(ys[2].data(), y0.data(), n * sizeof(ComplexSample)) == 0);
  }

  // fp16 dual beats LF against the FP64 DFT at N=1024 (acceptance criterion 7 shape)
  {
    const SampleBuffer x = random_buffer(1024, 42);
    SampleBuffer ing(1024);
    for (std::size_t i = 0; i < 1024; ++i)
      ing[i] = {round_to(x[i].re, Precision::fp16), round_to(x[i].im, Precision::fp16)};
    const SampleBuffer ref = dft(ing);
    ArithmeticContext c(Precision::fp16);
    const double e_du = rel_l2(forward(make_plan(1024, Strategy::dual_select, Precision::fp16), x, c), ref);
    const double e_lf = rel_l2(forward(make_plan(1024, Strategy::linzer_feig, Precision::fp16), x, c), ref);
    CHECK(e_du < e_lf && e_du < 4.89e-3);
  }

  // non-finite propagation (test_fft.cpp:252-262)
  {
    const FftPlan p8 = make_plan(8, Strategy::dual_select, Precision::fp16);
    SampleBuffer x(8, ComplexSample{1.0, 0.0});
    x[3].re = std::nan("");
    ArithmeticContext c(Precision::fp16);
    bool any_nan = false;
    for (const auto& v : forward(p8, x, c)) any_nan = any_nan || std::isnan(v.re) || std::isnan(v.im);
    CHECK(any_nan);
  }
  // fp64 on the device: the reference's own fp64 tests verbatim
  // (test_fft.cpp:110-128 oracle equivalence < 1e-11, 130-149 op accounting)
  for (std::size_t n = 2; n <= 512; n <<= 1) {
    const SampleBuffer x = random_buffer(n, 1000 + n);
    const SampleBuffer ref = dft(x);
    for (Strategy s : {Strategy::standard, Strategy::linzer_feig, Strategy::cosine,
                       Strategy::dual_select}) {
      ArithmeticContext c(Precision::fp64);
      CHECK(rel_l2(forward(make_plan(n, s, Precision::fp64), x, c), ref) < 1e-11);
    }
  }
  {
    const FftPlan p1024 = make_plan(1024, Strategy::dual_select, Precision::fp64);
    ArithmeticContext c(Precision::fp64);
    const SampleBuffer x = random_buffer(1024, 8);
    forward(p1024, x, c);
    CHECK(c.counters().fma_count == 6 * 512 * 10);
    const SampleBuffer back = inverse(p1024, forward(p1024, x, c), c);
    CHECK(rel_l2(back, x) < 1e-13);
  }
}

// `test_compat csv`: the CLI's table and statistics dumps through the C++
// mirror (write_table_csv of build_table, write_bounds_csv of the bound
// tables), compared byte for byte with the reference's own dumps by
// tests/test_cpp_compat.py.
static int csv_dump() {
  std::ostringstream os;
  const struct {
    std::size_t n;
    Strategy s;
    const char* name;
  } tables[] = {{64, Strategy::dual_select, "dual"},
                {64, Strategy::linzer_feig, "lf"},
                {8, Strategy::standard, "standard"}};
  for (const auto& t : tables) {
    os << "== csv/" << t.n << "/" << t.name << "/fp64\n";
    write_table_csv(os, build_table(t.n, t.s));
  }
  for (std::size_t n : {std::size_t(1024), std::size_t(64), std::size_t(1) << 20, std::size_t(2)}) {
    os << "== bounds/" << n << "/stats/fp16\n";
    write_bounds_csv(os, reproduce_ratio_table(n));
  }
  const struct {
    std::size_t n;
    Precision p;
    const char* name;
  } cum[] = {{1024, Precision::fp16, "fp16"},
             {1024, Precision::fp32, "fp32"},
             {4096, Precision::fp64, "fp64"},
             {8, Precision::fp16, "fp16"}};
  for (const auto& c : cum) {
    os << "== bounds/" << c.n << "/bounds/" << c.name << "\n";
    write_bounds_csv(os, reproduce_cumulative_table(c.n, c.p));
  }
  std::fputs(os.str().c_str(), stdout);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "csv") == 0) return csv_dump();
  host_checks();
  if (!(argc > 1 && std::strcmp(argv[1], "host") == 0)) device_checks();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
