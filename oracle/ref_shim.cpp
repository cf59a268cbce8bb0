// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" face over the UNMODIFIED reference library (fmafft core compiled
// from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libfmafft_ref.so).  Used to (1) pin oracle/fmafft_oracle.c,
// (2) generate tests/golden/ vectors and (3) time the reference's own CPU path
// for bench.py's cpu_baseline / --impl reference legs.  Never linked into the
// product.  Signatures mirror fmafft_oracle.h with a ref_ prefix.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fmafft/analysis.hpp"
#include "fmafft/butterfly.hpp"
#include "fmafft/fft.hpp"
#include "fmafft/precision.hpp"
#include "fmafft/twiddle.hpp"

namespace {

thread_local std::string g_err;

struct ref_entry {
  double multiplier;
  double ratio;
  int32_t path;
  int32_t clamped;
  double omega_r;
  double omega_i;
};

struct ref_counters {
  uint64_t fma_count, add_count, mul_count;
};

struct ref_error_report {
  uint64_t n;
  int32_t strategy, precision, metric, pad_;
  uint64_t trials, seed;
  double rel_l2_median, rel_l2_max;
  uint64_t nonfinite_trials;
};

fmafft::Precision P(int p) { return static_cast<fmafft::Precision>(p); }
fmafft::Strategy S(int s) { return static_cast<fmafft::Strategy>(s); }

void put(const fmafft::TwiddleTable& t, ref_entry* out) {
  for (std::size_t k = 0; k < t.entries.size(); ++k) {
    const auto& e = t.entries[k];
    out[k] = ref_entry{e.multiplier, e.ratio, e.path == fmafft::TwiddlePath::sin,
                       e.clamped ? 1 : 0, e.omega_r, e.omega_i};
  }
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int batch_run(std::size_t n, int s, int p, const double* in, double* out,
              std::size_t batch, int threads, ref_counters* counters, bool inv) {
  return guard([&] {
    const fmafft::FftPlan plan = fmafft::make_plan(n, S(s), P(p));
    unsigned nt = threads > 0 ? unsigned(threads) : std::thread::hardware_concurrency();
    nt = std::max(1u, std::min<unsigned>(nt, unsigned(std::max<std::size_t>(batch, 1))));
    std::vector<ref_counters> cs(nt, ref_counters{0, 0, 0});
    std::vector<std::string> errs(nt);
    auto work = [&](unsigned t) {
      try {
        fmafft::ArithmeticContext ctx(P(p));
        fmafft::SampleBuffer x(n);
        const std::size_t b0 = batch * t / nt, b1 = batch * (t + 1) / nt;
        for (std::size_t b = b0; b < b1; ++b) {
          const double* src = in + 2 * n * b;
          for (std::size_t i = 0; i < n; ++i) x[i] = {src[2 * i], src[2 * i + 1]};
          const fmafft::SampleBuffer y =
              inv ? fmafft::inverse(plan, x, ctx) : fmafft::forward(plan, x, ctx);
          double* dst = out + 2 * n * b;
          for (std::size_t i = 0; i < n; ++i) {
            dst[2 * i] = y[i].re;
            dst[2 * i + 1] = y[i].im;
          }
        }
        const auto& c = ctx.counters();
        cs[t] = ref_counters{c.fma_count, c.add_count, c.mul_count};
      } catch (const std::exception& e) {
        errs[t] = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
    if (counters) {
      *counters = ref_counters{0, 0, 0};
      for (auto& c : cs) {
        counters->fma_count += c.fma_count;
        counters->add_count += c.add_count;
        counters->mul_count += c.mul_count;
      }
    }
  });
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

double ref_round_to(double x, int p) { return fmafft::round_to(x, P(p)); }

void ref_round_array(const double* x, double* out, std::size_t count, int p) {
  for (std::size_t i = 0; i < count; ++i) out[i] = fmafft::round_to(x[i], P(p));
}

double ref_machine_epsilon(int p) { return fmafft::machine_epsilon(P(p)); }

int ref_build_table(std::size_t n, int s, double clamp_eps, ref_entry* out) {
  return guard([&] { put(fmafft::build_table(n, S(s), clamp_eps), out); });
}

int ref_plan_table(std::size_t n, int s, int p, ref_entry* out) {
  return guard([&] { put(fmafft::make_plan(n, S(s), P(p)).table, out); });
}

int ref_forward(std::size_t n, int s, int p, const double* in, double* out,
                std::size_t batch, int threads, ref_counters* counters) {
  return batch_run(n, s, p, in, out, batch, threads, counters, false);
}

int ref_inverse(std::size_t n, int s, int p, const double* in, double* out,
                std::size_t batch, int threads, ref_counters* counters) {
  return batch_run(n, s, p, in, out, batch, threads, counters, true);
}

int ref_butterfly(int s, int p, const double a[2], const double b[2],
                  const ref_entry* e, double out[4], ref_counters* counters) {
  return guard([&] {
    fmafft::TwiddleEntry te;
    te.multiplier = e->multiplier;
    te.ratio = e->ratio;
    te.path = e->path ? fmafft::TwiddlePath::sin : fmafft::TwiddlePath::cos;
    te.clamped = e->clamped != 0;
    te.omega_r = e->omega_r;
    te.omega_i = e->omega_i;
    fmafft::ArithmeticContext ctx(P(p));
    const auto r = fmafft::kernel_for(S(s))({a[0], a[1]}, {b[0], b[1]}, te, ctx);
    out[0] = r.sum.re;
    out[1] = r.sum.im;
    out[2] = r.diff.re;
    out[3] = r.diff.im;
    if (counters)
      *counters = ref_counters{ctx.counters().fma_count, ctx.counters().add_count,
                               ctx.counters().mul_count};
  });
}

// ArithmeticContext::add/sub/mul/fma (op 0..3) of a fresh context, elementwise
void ref_ctx_op(int p, int op, const double* a, const double* b, const double* c, double* out,
                std::size_t count) {
  fmafft::ArithmeticContext ctx(P(p));
  for (std::size_t i = 0; i < count; ++i)
    out[i] = op == 0 ? ctx.add(a[i], b[i])
           : op == 1 ? ctx.sub(a[i], b[i])
           : op == 2 ? ctx.mul(a[i], b[i])
                     : ctx.fma(a[i], b[i], c[i]);
}

void ref_dft(std::size_t n, const double* in, double* out, std::size_t batch) {
  fmafft::SampleBuffer x(n);
  for (std::size_t b = 0; b < batch; ++b) {
    for (std::size_t i = 0; i < n; ++i) x[i] = {in[2 * n * b + 2 * i], in[2 * n * b + 2 * i + 1]};
    const auto y = fmafft::dft_oracle(x);
    for (std::size_t i = 0; i < n; ++i) {
      out[2 * n * b + 2 * i] = y[i].re;
      out[2 * n * b + 2 * i + 1] = y[i].im;
    }
  }
}

double ref_rel_l2(const double* x, const double* y, std::size_t n) {
  fmafft::SampleBuffer a(n), b(n);
  for (std::size_t i = 0; i < n; ++i) {
    a[i] = {x[2 * i], x[2 * i + 1]};
    b[i] = {y[2 * i], y[2 * i + 1]};
  }
  try {
    return fmafft::relative_l2_error(a, b);
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::nan("");
  }
}

double ref_cumulative_bound(double t_max, double eps, unsigned m) {
  return fmafft::cumulative_bound(t_max, eps, m);
}

void ref_splitmix_uniform(uint64_t seed, double* out, std::size_t count) {
  fmafft::SplitMix64 rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.uniform_pm1();
}

int ref_measure_error(std::size_t n, int s, int p, int metric, std::size_t trials,
                      uint64_t seed, ref_error_report* out) {
  return guard([&] {
    const auto r = fmafft::measure_error(n, S(s), P(p),
                                         static_cast<fmafft::ErrorMetric>(metric),
                                         trials, seed);
    *out = ref_error_report{r.n, int32_t(r.strategy), int32_t(r.precision),
                            int32_t(r.metric), 0, r.trials, r.seed,
                            r.rel_l2_median, r.rel_l2_max, r.nonfinite_trials};
  });
}

int ref_table_stats(std::size_t n, int s, double* t_max, uint64_t* argmax_k,
                    uint64_t* singular, uint64_t* cos_count, uint64_t* sin_count) {
  return guard([&] {
    const auto st = fmafft::table_stats(fmafft::build_table(n, S(s)));
    *t_max = st.t_max;
    *argmax_k = st.argmax_k;
    *singular = st.singular_count;
    *cos_count = st.cos_path_count;
    *sin_count = st.sin_path_count;
  });
}

}  // extern "C"

#ifdef REF_HAVE_SERIALIZE
#include <sstream>

#include "fmafft/serialize.hpp"

extern "C" {
// write_table_csv (serialize.cpp:48-57) of build_table (the CLI `twiddles`
// dump, main.cpp:34-42) or, for precision fp16/fp32, of make_plan's rounded
// table.  Returns the bytes needed (incl. NUL); copies when cap suffices.
size_t ref_table_csv(std::size_t n, int s, int p, double clamp_eps, char* out, size_t cap) {
  std::ostringstream os;
  try {
    if (p == 2)
      fmafft::write_table_csv(os, fmafft::build_table(n, S(s), clamp_eps));
    else
      fmafft::write_table_csv(os, fmafft::make_plan(n, S(s), P(p)).table);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
  const std::string str = os.str();
  if (out && cap > str.size()) std::memcpy(out, str.c_str(), str.size() + 1);
  return str.size() + 1;
}

// write_bounds_csv (serialize.cpp:79-91) of reproduce_ratio_table(n) (kind 0,
// the CLI `stats` command) or reproduce_cumulative_table(n, p) (kind 1, `bounds`).
size_t ref_bounds_csv(std::size_t n, int kind, int p, char* out, size_t cap) {
  std::ostringstream os;
  try {
    if (kind == 0)
      fmafft::write_bounds_csv(os, fmafft::reproduce_ratio_table(n));
    else
      fmafft::write_bounds_csv(os, fmafft::reproduce_cumulative_table(n, P(p)));
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
  const std::string str = os.str();
  if (out && cap > str.size()) std::memcpy(out, str.c_str(), str.size() + 1);
  return str.size() + 1;
}
}
#endif
