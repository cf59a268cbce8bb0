// dsfft_capi.cu -- C ABI (include/dsfft.h): plans, device upload, dispatch,
// host-buffer pipelines.  The only compute path is the sm_100a kernels; there
// is no CPU fallback: without an sm_100 device every execute fails loudly.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dsfft.h"
#include "host_table.hpp"
#include "emulate.cuh"
#include "error_harness.cuh"
#include "fp64.cuh"
#include "multipass.cuh"
#include "small_launch.cuh"
#include "stream_alloc.cuh"
#include "synth.cuh"

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(DSFFT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define DSFFT_CUDA(call)                                 \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

// Makes `dev`'s primary context current on this thread (always: a fresh host
// thread has no current context, which the driver-API tensor-map encoder
// needs) and restores the caller's device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

const dsfft::SmallEntry& small_entry(int m) {
  static const dsfft::SmallEntry table[14] = {
      {},
      dsfft::small_entry_m1(),  dsfft::small_entry_m2(),  dsfft::small_entry_m3(),
      dsfft::small_entry_m4(),  dsfft::small_entry_m5(),  dsfft::small_entry_m6(),
      dsfft::small_entry_m7(),  dsfft::small_entry_m8(),  dsfft::small_entry_m9(),
      dsfft::small_entry_m10(), dsfft::small_entry_m11(), dsfft::small_entry_m12(),
      dsfft::small_entry_m13()};
  return table[m];
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Host-buffer pipeline: NSLOT chunk slots, each with its own stream and
// device in/out buffers, so H2D(i+1) / kernel(i) / D2H(i-1) overlap.
struct HostPipe {
  static constexpr int kSlots = 3;
  size_t chunk_bytes = 0;
  void* d_in[kSlots] = {};
  void* d_out[kSlots] = {};
  cudaStream_t st[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  cudaEvent_t start = nullptr;
  ~HostPipe() {
    for (int i = 0; i < kSlots; ++i) {
      if (d_in[i]) cudaFree(d_in[i]);
      if (d_out[i]) cudaFree(d_out[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    if (start) cudaEventDestroy(start);
  }
};

}  // namespace

struct dsfft_plan_s {
  size_t n = 0;
  unsigned m = 0;
  int strategy = 0, precision = 0, device = 0;
  double clamp_eps = 1e-7;
  std::vector<dsfft::TableEntry> table;  // rounded (FftPlan::table)
  // single-kernel path (m <= 12)
  const dsfft::SmallVariant* small = nullptr;
  int variant = 0;  // dsfft::SmallVariantId
  uint4* d_tw = nullptr;
  int groups = 0, stages = 0, grid = 0;
  // multi-pass path (m > 12)
  dsfft::MultipassPlan* mp = nullptr;
  // fp64 path (per-pass DFMA kernels)
  dsfft::F64Plan* f64 = nullptr;
  int sm_count = 0;
  size_t smem_optin = 0;
  std::mutex mu;
  HostPipe* pipe = nullptr;
  dsfft::F64Plan* ref64 = nullptr;  // lazily built FP64 reference for the error harness
};

namespace {

size_t sample_bytes(int p) {
  return p == DSFFT_FP16 ? 4 : p == DSFFT_FP32 ? 8 : p == DSFFT_FP64 ? 16 : 0;
}

uint32_t inverse_scale_word(const dsfft_plan_s* p) {
  const double s = dsfft::round_to(1.0 / double(p->n), p->precision);  // fft.cpp:92-93
  if (p->precision == DSFFT_FP16) {
    const uint32_t h = dsfft::half_bits(s);
    return h | (h << 16);
  }
  const float f = float(s);
  uint32_t b;
  std::memcpy(&b, &f, 4);
  return b;
}

// Choose groups per CTA and buffers per group for the single-kernel path.
void choose_small_launch(dsfft_plan_s* p, int default_stages) {
  const dsfft::SmallGeom& g = p->small->geom;
  const int T = 32 * g.warps;
  int stages = env_int("DSFFT_STAGES", default_stages);
  stages = std::max(1, std::min(stages, 8));
  int max_groups = std::max(1, g.max_threads / T);
  int want = env_int("DSFFT_GROUPS", 0);
  int groups = 0;
  for (int ng = max_groups; ng >= 1; --ng) {
    // whole warps per SM sub-partition: 13 one-warp groups leave one SMSP
    // with 4 warps and three with 3 (measured -20% at N=1024 vs 12)
    if (ng * g.warps > 4 && (ng * g.warps) % 4 != 0) continue;
    if (p->small->smem_bytes(ng, stages) <= p->smem_optin) {
      groups = ng;
      break;
    }
  }
  while (groups == 0 && stages > 1) {  // shrink the ring if even one group does not fit
    --stages;
    if (p->small->smem_bytes(1, stages) <= p->smem_optin) groups = 1;
  }
  if (want > 0 && want <= max_groups && p->small->smem_bytes(want, stages) <= p->smem_optin)
    groups = want;
  p->groups = std::max(1, groups);
  p->stages = stages;
  p->grid = p->sm_count * std::max(1, env_int("DSFFT_CTAS_PER_SM", 1));
}

int upload_small_tables(dsfft_plan_s* p) {
  const dsfft::SmallGeom& g = p->small->geom;
  std::vector<dsfft::Record> rec(g.tw_records);
  for (int st = 0; st < g.nstage; ++st) {
    const int P = g.P[st], s = g.s[st];
    for (int pl = 0; pl < s; ++pl)
      for (int rl = 0; rl < (1 << pl); ++rl)
        for (int r = 0; r < (1 << P); ++r) {
          const int slot = g.tw_off[st] + dsfft::tw_slot(P, r, pl, rl);
          const int k = dsfft::tw_entry(int(p->m), P, r, pl, rl);
          rec[slot] = dsfft::pack_record(p->table[k], p->strategy, p->precision,
                                         p->variant == dsfft::kVarF16C);
        }
  }
  const std::vector<uint8_t> img = dsfft::serialize_records(
      rec, dsfft::record_bytes(p->precision, p->variant == dsfft::kVarF16C));
  DSFFT_CUDA(cudaMalloc(&p->d_tw, img.size()));
  DSFFT_CUDA(cudaMemcpy(p->d_tw, img.data(), img.size(), cudaMemcpyHostToDevice));
  return DSFFT_OK;
}

// Launch the batched transform on device buffers (no argument checks).
int launch(dsfft_plan_s* p, int dir, const void* in, void* out, size_t batch,
           cudaStream_t stream) {
  if (batch == 0) return DSFFT_OK;
  if (p->f64) {
    const int e = dsfft::fp64_execute(*p->f64, dir == DSFFT_INVERSE, in, out, batch,
                                      1.0 / double(p->n), p->sm_count, stream, &g_launches);
    if (e) return fail(DSFFT_ERR_CUDA, dsfft::fp64_error());
    return DSFFT_OK;
  }
  const uint32_t scale = inverse_scale_word(p);
  if (p->mp) {
    const int e = dsfft::multipass_execute(*p->mp, dir == DSFFT_INVERSE, in, out, batch, scale,
                                           stream, &g_launches);
    if (e) return fail(DSFFT_ERR_CUDA, dsfft::multipass_error());
    return DSFFT_OK;
  }
  const dsfft::SmallGeom& g = p->small->geom;
  const size_t tb = p->n * sample_bytes(p->precision);
  const long long tpi = g.tpi;
  // bulk copies move multiples of 16 bytes: N=2 fp16 with an odd batch
  // stages its last transform through a padded scratch buffer
  size_t main_batch = batch;
  if ((batch * tb) % 16 != 0) main_batch = batch - 1;
  if (main_batch) {
    dsfft::LaunchArgs a{};
    a.standard = p->strategy == DSFFT_STANDARD;
    a.inverse = dir == DSFFT_INVERSE;
    a.kp.in = static_cast<const uint8_t*>(in);
    a.kp.out = static_cast<uint8_t*>(out);
    a.kp.tw = p->d_tw;
    a.kp.batch = (long long)main_batch;
    a.kp.n_items = ((long long)main_batch + tpi - 1) / tpi;
    a.kp.scale = scale;
    a.kp.stages = p->stages;
    a.stream = stream;
    a.groups = p->groups;
    a.grid = int(std::min<long long>(p->grid, (a.kp.n_items + p->groups - 1) / p->groups));
    cudaError_t e = p->small->launch(a);
    if (e != cudaSuccess) return cuda_fail(e, "fft_small_kernel launch");
    ++g_launches;
  }
  if (main_batch != batch) {
    uint8_t* scratch = nullptr;  // stream-ordered: safe when a plan runs on several streams
    DSFFT_CUDA(dsfft::scratch_alloc(reinterpret_cast<void**>(&scratch), 64, stream));
    struct Release {
      uint8_t* s;
      cudaStream_t st;
      ~Release() { dsfft::scratch_free(s, st); }
    } release{scratch, stream};
    const size_t off = main_batch * tb;
    DSFFT_CUDA(cudaMemsetAsync(scratch, 0, 64, stream));
    DSFFT_CUDA(cudaMemcpyAsync(scratch, static_cast<const uint8_t*>(in) + off, tb,
                               cudaMemcpyDeviceToDevice, stream));
    dsfft::LaunchArgs a{};
    a.standard = p->strategy == DSFFT_STANDARD;
    a.inverse = dir == DSFFT_INVERSE;
    a.kp.in = scratch;
    a.kp.out = scratch;
    a.kp.tw = p->d_tw;
    a.kp.batch = 2;  // pad to a 16-byte transfer; the second transform is discarded
    a.kp.n_items = 1;
    a.kp.scale = scale;
    a.kp.stages = p->stages;
    a.stream = stream;
    a.groups = 1;
    a.grid = 1;
    cudaError_t e = p->small->launch(a);
    if (e != cudaSuccess) return cuda_fail(e, "fft_small_kernel launch (tail)");
    ++g_launches;
    DSFFT_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(out) + off, scratch, tb,
                               cudaMemcpyDeviceToDevice, stream));
  }
  return DSFFT_OK;
}

int check_exec_args(dsfft_plan_s* p, int dir, const void* in, void* out, size_t batch) {
  if (!p) return fail(DSFFT_ERR_INVALID, "null plan");
  if (dir != DSFFT_FORWARD && dir != DSFFT_INVERSE)
    return fail(DSFFT_ERR_INVALID, "unknown direction");
  if (!in || !out) return fail(DSFFT_ERR_INVALID, "null buffer");
  // byte counts (and the f64 carrier's 16 B per sample) must fit in size_t
  if (batch > (SIZE_MAX / 16) / p->n)
    return fail(DSFFT_ERR_INVALID, "batch too large: byte count overflows size_t");
  return DSFFT_OK;
}

}  // namespace

extern "C" {

const char* dsfft_last_error(void) { return g_err.c_str(); }

int dsfft_version(void) { return DSFFT_VERSION; }

uint64_t dsfft_last_launch_count(void) { return g_launches; }

size_t dsfft_sample_bytes(int precision) { return sample_bytes(precision); }

}  // extern "C"

namespace {

// Plan over a rounded table (make_plan's, or a caller's edited copy).
int plan_create_from(std::vector<dsfft::TableEntry> table, size_t n, int strategy,
                     int precision, double clamp_eps, int device, dsfft_plan* out) {
  auto* p = new dsfft_plan_s();
  p->table = std::move(table);
  p->n = n;
  while ((size_t(1) << p->m) < n) ++p->m;
  p->strategy = strategy;
  p->precision = precision;
  p->clamp_eps = clamp_eps;
  p->device = device;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete p;
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) {
    delete p;
    return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) {
    delete p;
    return fail(DSFFT_ERR_NO_DEVICE, "device is not sm_100 (B200): dsfft is sm_100a-only");
  }
  p->sm_count = prop.multiProcessorCount;
  p->smem_optin = prop.sharedMemPerBlockOptin;
  DeviceGuard guard(device);
  int rc = DSFFT_OK;
  if (precision == DSFFT_FP64) {
    p->f64 = dsfft::fp64_create(p->table, int(p->m), strategy);
    if (!p->f64) rc = fail(DSFFT_ERR_CUDA, dsfft::fp64_error());
  } else if (p->m <= 12 || (p->m == 13 && env_int("DSFFT_SMALL13", 1) != 0)) {
    const dsfft::SmallEntry& se = small_entry(int(p->m));
    p->variant = dsfft::kVarF32;
    if (precision == DSFFT_FP16) {
      const int want = env_int("DSFFT_F16_LAYOUT", -1);  // 1 pairs, 2 complex
      p->variant = (want == dsfft::kVarF16P || want == dsfft::kVarF16C) ? want : se.f16_default;
    }
    p->small = &se.v[p->variant];
    choose_small_launch(p, se.stages[p->variant]);
    rc = upload_small_tables(p);
  } else {
    p->mp = dsfft::multipass_create(p->table, int(p->m), strategy, precision, p->sm_count,
                                    p->smem_optin);
    if (!p->mp) rc = fail(DSFFT_ERR_CUDA, dsfft::multipass_error());
  }
  if (rc != DSFFT_OK) {
    dsfft_plan_destroy(p);
    return rc;
  }
  *out = p;
  return DSFFT_OK;
}

int check_kinds(int strategy, int precision) {
  if (precision < DSFFT_FP16 || precision > DSFFT_FP64)
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  if (strategy < DSFFT_STANDARD || strategy > DSFFT_DUAL_SELECT)
    return fail(DSFFT_ERR_INVALID, "unknown strategy: " + std::to_string(strategy));
  return DSFFT_OK;
}

}  // namespace

extern "C" {

int dsfft_plan_create(size_t n, int strategy, int precision, double clamp_eps, int device,
                      dsfft_plan* out) {
  g_err.clear();
  if (!out) return fail(DSFFT_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (int rc = check_kinds(strategy, precision)) return rc;
  std::vector<dsfft::TableEntry> table;
  try {
    table = dsfft::plan_table(n, strategy, precision, clamp_eps);
  } catch (const std::exception& e) {
    return fail(DSFFT_ERR_INVALID, e.what());
  }
  return plan_create_from(std::move(table), n, strategy, precision, clamp_eps, device, out);
}

int dsfft_plan_create_with_table(size_t n, int strategy, int precision, const dsfft_entry* table,
                                 size_t count, int device, dsfft_plan* out) {
  g_err.clear();
  if (!out || !table) return fail(DSFFT_ERR_INVALID, "null argument");
  *out = nullptr;
  if (int rc = check_kinds(strategy, precision)) return rc;
  if (n < 2 || (n & (n - 1)) != 0)
    return fail(DSFFT_ERR_INVALID, "FFT size must be a power of two >= 2, got " +
                                       std::to_string(n));
  if (n > (size_t(1) << 24))  // fft.cpp:57-58
    return fail(DSFFT_ERR_INVALID, "FFT size exceeds 2^24");
  if (count != n / 2)
    return fail(DSFFT_ERR_INVALID, "table length mismatch: need n/2 entries");
  std::vector<dsfft::TableEntry> t(count);
  for (size_t k = 0; k < count; ++k) {
    const dsfft_entry& e = table[k];
    t[k].multiplier = e.multiplier;
    t[k].ratio = e.ratio;
    t[k].path = e.path ? dsfft::kSin : dsfft::kCos;
    t[k].clamped = e.clamped != 0;
    t[k].omega_r = e.omega_r;
    t[k].omega_i = e.omega_i;
  }
  return plan_create_from(std::move(t), n, strategy, precision, 1e-7, device, out);
}

int dsfft_plan_destroy(dsfft_plan p) {
  if (!p) return DSFFT_OK;
  {
    DeviceGuard guard(p->device);
    if (p->d_tw) cudaFree(p->d_tw);
    delete p->pipe;
    if (p->mp) dsfft::multipass_destroy(p->mp);
    if (p->f64) dsfft::fp64_destroy(p->f64);
    if (p->ref64) dsfft::fp64_destroy(p->ref64);
    dsfft::scratch_trim(p->device);  // scratch blocks no call still holds
  }
  delete p;
  return DSFFT_OK;
}

int dsfft_plan_info(dsfft_plan p, size_t* n, unsigned* m, int* strategy, int* precision) {
  if (!p) return fail(DSFFT_ERR_INVALID, "null plan");
  if (n) *n = p->n;
  if (m) *m = p->m;
  if (strategy) *strategy = p->strategy;
  if (precision) *precision = p->precision;
  return DSFFT_OK;
}

int dsfft_build_table(size_t n, int strategy, int precision, double clamp_eps, dsfft_entry* out,
                      size_t count) {
  if (!out) return fail(DSFFT_ERR_INVALID, "null argument");
  std::vector<dsfft::TableEntry> t;
  try {
    t = dsfft::plan_table(n, strategy, precision, clamp_eps);
  } catch (const std::exception& e) {
    return fail(DSFFT_ERR_INVALID, e.what());
  }
  if (count < t.size()) return fail(DSFFT_ERR_INVALID, "output too small");
  for (size_t k = 0; k < t.size(); ++k) {
    const auto& e = t[k];
    out[k] = dsfft_entry{e.multiplier, e.ratio, e.path, e.clamped ? 1 : 0, e.omega_r, e.omega_i};
  }
  return DSFFT_OK;
}

size_t dsfft_table_csv(size_t n, int strategy, int precision, double clamp_eps, char* out,
                       size_t cap) {
  std::vector<dsfft::TableEntry> t;
  try {
    t = dsfft::plan_table(n, strategy, precision, clamp_eps);
  } catch (const std::exception& e) {
    fail(DSFFT_ERR_INVALID, e.what());
    return 0;
  }
  std::string s = "k,theta,omega_r,omega_i,path,multiplier,ratio,clamped\n";
  char buf[48];
  auto num = [&](double v) {  // format_double: %.17g (serialize.cpp:42-46)
    std::snprintf(buf, sizeof buf, "%.17g", v);
    s += buf;
  };
  for (size_t k = 0; k < t.size(); ++k) {
    const auto& e = t[k];
    s += std::to_string(k);
    s += ',';
    num(dsfft::twiddle_angle(k, n));
    s += ',';
    num(e.omega_r);
    s += ',';
    num(e.omega_i);
    s += e.path == dsfft::kCos ? ",COS," : ",SIN,";
    num(e.multiplier);
    s += ',';
    num(e.ratio);
    s += e.clamped ? ",true\n" : ",false\n";
  }
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return s.size() + 1;
}

size_t dsfft_bounds_csv(size_t n, int kind, int precision, char* out, size_t cap) {
  if (kind != DSFFT_STATS_RATIO && kind != DSFFT_STATS_CUMULATIVE) {
    fail(DSFFT_ERR_INVALID, "unknown statistics kind");
    return 0;
  }
  if (kind == DSFFT_STATS_CUMULATIVE && (precision < 0 || precision > 2)) {
    fail(DSFFT_ERR_INVALID, "unknown precision");
    return 0;
  }
  // machine_epsilon (precision.cpp:36-43); the ratio table is quoted at fp16
  const double eps = kind == DSFFT_STATS_RATIO || precision == dsfft::kFp16 ? 0x1p-11
                     : precision == dsfft::kFp32                           ? 0x1p-24
                                                                           : 0x1p-53;
  struct Row {
    int strategy;
    double t_max = 0.0, per = 0.0, cum = 0.0, improvement = 1.0;
    size_t argmax = 0, singular = 0, ncos = 0, nsin = 0;
  };
  std::vector<Row> rows;
  const std::vector<int> strategies =
      kind == DSFFT_STATS_RATIO
          ? std::vector<int>{dsfft::kLinzerFeig, dsfft::kCosine, dsfft::kDual}
          : std::vector<int>{dsfft::kLinzerFeig, dsfft::kDual};
  try {
    for (int st : strategies) {
      const std::vector<dsfft::TableEntry> t = dsfft::build_table(n, st, 1e-7);
      Row r;
      r.strategy = st;
      for (size_t k = 0; k < t.size(); ++k) {  // table_stats (twiddle.cpp:143-162)
        (t[k].path == dsfft::kCos ? r.ncos : r.nsin)++;
        if (t[k].clamped) {
          ++r.singular;
          continue;
        }
        const double a = std::fabs(t[k].ratio);
        if (a > r.t_max) {
          r.t_max = a;
          r.argmax = k;
        }
      }
      // per_butterfly_bound / cumulative_bound (analysis.cpp:59-63), m = log2 n
      r.per = r.t_max * eps;
      r.cum = std::pow(1.0 + r.t_max * eps, double(__builtin_ctzll(n))) - 1.0;
      rows.push_back(r);
    }
  } catch (const std::exception& e) {
    fail(DSFFT_ERR_INVALID, e.what());
    return 0;
  }
  for (size_t i = 1; i < rows.size(); ++i) rows[i].improvement = rows[0].cum / rows[i].cum;
  std::string s =
      "strategy,t_max,argmax_k,singular_count,cos_path_count,sin_path_count,"
      "per_butterfly_bound,cumulative_bound,improvement_vs_baseline,divergent\n";
  char buf[48];
  auto num = [&](double v) {  // format_double: %.17g (serialize.cpp:42-46)
    std::snprintf(buf, sizeof buf, "%.17g", v);
    s += buf;
  };
  static const char* kNames[] = {"standard", "lf", "cosine", "dual"};  // twiddle.cpp:31-39
  for (const Row& r : rows) {
    s += kNames[r.strategy];
    s += ',';
    num(r.t_max);
    s += ',' + std::to_string(r.argmax) + ',' + std::to_string(r.singular) + ',' +
         std::to_string(r.ncos) + ',' + std::to_string(r.nsin) + ',';
    num(r.per);
    s += ',';
    num(r.cum);
    s += ',';
    num(r.improvement);
    s += r.per >= 1.0 ? ",true\n" : ",false\n";
  }
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return s.size() + 1;
}

int dsfft_plan_table(dsfft_plan p, dsfft_entry* out, size_t count) {
  if (!p || !out) return fail(DSFFT_ERR_INVALID, "null argument");
  if (count < p->table.size()) return fail(DSFFT_ERR_INVALID, "output too small");
  for (size_t k = 0; k < p->table.size(); ++k) {
    const auto& e = p->table[k];
    out[k] = dsfft_entry{e.multiplier, e.ratio, e.path, e.clamped ? 1 : 0, e.omega_r, e.omega_i};
  }
  return DSFFT_OK;
}

int dsfft_execute(dsfft_plan p, int dir, const void* in, void* out, size_t batch, void* stream) {
  g_launches = 0;
  int rc = check_exec_args(p, dir, in, out, batch);
  if (rc) return rc;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(DSFFT_ERR_INVALID, "device buffers must be 16-byte aligned");
  DeviceGuard guard(p->device);
  return launch(p, dir, in, out, batch, static_cast<cudaStream_t>(stream));
}

int dsfft_execute_host(dsfft_plan p, int dir, const void* h_in, void* h_out, size_t batch,
                       void* stream_) {
  g_launches = 0;
  int rc = check_exec_args(p, dir, h_in, h_out, batch);
  if (rc) return rc;
  if (batch == 0) return DSFFT_OK;
  DeviceGuard guard(p->device);
  std::lock_guard<std::mutex> lock(p->mu);
  cudaStream_t user = static_cast<cudaStream_t>(stream_);
  const size_t tb = p->n * sample_bytes(p->precision);
  // 64 MiB chunks: ~96 GB/s H2D+D2H on PCIe Gen5 x16 (16 MiB: 85, 256 MiB: 93)
  const size_t want_chunk = size_t(env_int("DSFFT_HOST_CHUNK_MB", 64)) << 20;
  size_t per = std::max<size_t>(1, want_chunk / tb);
  if (per % 2) per += (per > 1) ? -1 : 1;  // keep fp16 pairs whole
  const size_t chunk_bytes = per * tb;
  if (!p->pipe || p->pipe->chunk_bytes < chunk_bytes) {
    // build the pipe completely before publishing it: a failed allocation
    // leaves the plan without a pipe rather than with a half-built one
    std::unique_ptr<HostPipe> hp(new HostPipe());
    hp->chunk_bytes = chunk_bytes;
    for (int i = 0; i < HostPipe::kSlots; ++i) {
      DSFFT_CUDA(cudaMalloc(&hp->d_in[i], chunk_bytes));
      DSFFT_CUDA(cudaMalloc(&hp->d_out[i], chunk_bytes));
      DSFFT_CUDA(cudaStreamCreateWithFlags(&hp->st[i], cudaStreamNonBlocking));
      DSFFT_CUDA(cudaEventCreateWithFlags(&hp->ev[i], cudaEventDisableTiming));
    }
    DSFFT_CUDA(cudaEventCreateWithFlags(&hp->start, cudaEventDisableTiming));
    delete p->pipe;
    p->pipe = hp.release();
  }
  HostPipe& hp = *p->pipe;
  // on any failure below, drain the pipe's streams before returning: no copy
  // of the caller's host buffers may still be in flight
  auto drain = [&](int code) {
    for (int i = 0; i < HostPipe::kSlots; ++i) cudaStreamSynchronize(hp.st[i]);
    return code;
  };
  DSFFT_CUDA(cudaEventRecord(hp.start, user));
  for (int i = 0; i < HostPipe::kSlots; ++i) DSFFT_CUDA(cudaStreamWaitEvent(hp.st[i], hp.start, 0));
  uint64_t launches = 0;
  const uint8_t* src = static_cast<const uint8_t*>(h_in);
  uint8_t* dst = static_cast<uint8_t*>(h_out);
  size_t done = 0;
  for (size_t c = 0; done < batch; ++c) {
    const int slot = int(c % HostPipe::kSlots);
    const size_t nb = std::min(per, batch - done);
    cudaStream_t s = hp.st[slot];
    cudaError_t e = cudaMemcpyAsync(hp.d_in[slot], src + done * tb, nb * tb,
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return drain(cuda_fail(e, "execute_host: H2D copy"));
    rc = launch(p, dir, hp.d_in[slot], hp.d_out[slot], nb, s);
    if (rc) return drain(rc);
    launches += g_launches;
    g_launches = 0;
    e = cudaMemcpyAsync(dst + done * tb, hp.d_out[slot], nb * tb, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return drain(cuda_fail(e, "execute_host: D2H copy"));
    done += nb;
  }
  for (int i = 0; i < HostPipe::kSlots; ++i) {
    cudaError_t e = cudaEventRecord(hp.ev[i], hp.st[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, hp.ev[i], 0);
    if (e != cudaSuccess) return drain(cuda_fail(e, "execute_host: join"));
  }
  DSFFT_CUDA(cudaStreamSynchronize(user));
  g_launches = launches;
  return DSFFT_OK;
}

int dsfft_execute_multi(const dsfft_plan* plans, int nplans, int dir, const void* h_in,
                        void* h_out, size_t batch) {
  g_launches = 0;
  if (!plans || nplans < 1) return fail(DSFFT_ERR_INVALID, "no plans");
  for (int i = 0; i < nplans; ++i) {
    int rc = check_exec_args(plans[i], dir, h_in, h_out, batch);
    if (rc) return rc;
    if (plans[i]->n != plans[0]->n || plans[i]->precision != plans[0]->precision ||
        plans[i]->strategy != plans[0]->strategy)
      return fail(DSFFT_ERR_INVALID, "plans differ in size, strategy or precision");
  }
  const size_t tb = plans[0]->n * sample_bytes(plans[0]->precision);
  std::vector<int> rcs(nplans, DSFFT_OK);
  std::vector<std::string> errs(nplans);
  std::vector<uint64_t> launches(nplans, 0);
  std::vector<std::thread> pool;
  for (int i = 0; i < nplans; ++i) {
    const size_t b0 = batch * size_t(i) / size_t(nplans);
    const size_t b1 = batch * size_t(i + 1) / size_t(nplans);
    pool.emplace_back([&, i, b0, b1] {
      if (b1 == b0) return;
      rcs[i] = dsfft_execute_host(plans[i], dir, static_cast<const uint8_t*>(h_in) + b0 * tb,
                                  static_cast<uint8_t*>(h_out) + b0 * tb, b1 - b0, nullptr);
      errs[i] = g_err;
      launches[i] = g_launches;
    });
  }
  for (auto& t : pool) t.join();
  uint64_t total = 0;
  for (int i = 0; i < nplans; ++i) {
    if (rcs[i] != DSFFT_OK) return fail(rcs[i], "device " + std::to_string(i) + ": " + errs[i]);
    total += launches[i];
  }
  g_launches = total;
  return DSFFT_OK;
}

int dsfft_error_device_ex(dsfft_plan p, int metric, int reference, const void* d_x,
                          size_t batch, void* stream_, dsfft_error_report* out,
                          double* errs_out) {
  g_launches = 0;
  int rc = check_exec_args(p, DSFFT_FORWARD, d_x, const_cast<void*>(d_x), batch);
  if (rc) return rc;
  if (reinterpret_cast<uintptr_t>(d_x) & 15)
    return fail(DSFFT_ERR_INVALID, "device buffers must be 16-byte aligned");
  if (metric != 0 && metric != 1) return fail(DSFFT_ERR_INVALID, "unknown metric");
  if (reference < DSFFT_REF_AUTO || reference > DSFFT_REF_FFT64)
    return fail(DSFFT_ERR_INVALID, "unknown error reference");
  if (batch == 0) return fail(DSFFT_ERR_INVALID, "trials must be >= 1");
  DeviceGuard guard(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  const size_t n = p->n, tb = n * sample_bytes(p->precision);
  const bool use_dft = metric == 1 && (reference == DSFFT_REF_DFT ||
                                       (reference == DSFFT_REF_AUTO &&
                                        (long long)n <= dsfft::kDftMaxN));
  if (metric == 1 && !use_dft) {  // FP64 FFT reference (any strategy is FP64-accurate)
    std::lock_guard<std::mutex> lock(p->mu);
    if (!p->ref64)
      p->ref64 = dsfft::fp64_create(
          dsfft::plan_table(p->n, DSFFT_DUAL_SELECT, DSFFT_FP64, 1e-7), int(p->m),
          DSFFT_DUAL_SELECT);
    if (!p->ref64) return fail(DSFFT_ERR_CUDA, dsfft::fp64_error());
  }
  const size_t chunk = std::max<size_t>(1, (size_t(256) << 20) / (n * sizeof(double2)));
  void *y = nullptr, *z = nullptr;
  double2 *ax = nullptr, *bx = nullptr, *dtw = nullptr;
  double* derr = nullptr;
  const size_t cb = std::min(chunk, batch);
  auto cleanup = [&] {
    cudaFree(y);
    cudaFree(z);
    cudaFree(ax);
    cudaFree(bx);
    cudaFree(derr);
    cudaFree(dtw);
  };
  if (cudaMalloc(&y, cb * tb) != cudaSuccess || cudaMalloc(&z, cb * tb) != cudaSuccess ||
      cudaMalloc(&ax, cb * n * sizeof(double2)) != cudaSuccess ||
      cudaMalloc(&bx, cb * n * sizeof(double2)) != cudaSuccess ||
      cudaMalloc(&derr, cb * sizeof(double)) != cudaSuccess ||
      (use_dft && cudaMalloc(&dtw, n * sizeof(double2)) != cudaSuccess)) {
    cleanup();
    cudaGetLastError();
    return fail(DSFFT_ERR_CUDA, "error harness: device allocation failed");
  }
  if (use_dft) {
    const std::vector<double> tw = dsfft::dft_table(n);
    if (cudaMemcpy(dtw, tw.data(), n * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess) {
      cleanup();
      return fail(DSFFT_ERR_CUDA, "error harness: DFT table upload failed");
    }
  }
  std::vector<double> errs(batch);
  uint64_t launches = 0;
  for (size_t b0 = 0; b0 < batch && rc == DSFFT_OK; b0 += chunk) {
    const size_t nb = std::min(chunk, batch - b0);
    const void* x = static_cast<const uint8_t*>(d_x) + b0 * tb;
    rc = launch(p, DSFFT_FORWARD, x, y, nb, st);  // the measured transform
    launches += g_launches;
    g_launches = 0;
    if (rc) break;
    if (metric == 1) {  // forward vs the FP64 reference of the ingested input
      const int e1 = dsfft::launch_widen(x, bx, (long long)(nb * n), p->precision, st);
      const int e2 = use_dft ? dsfft::launch_dft(bx, ax, dtw, (long long)n, (long long)nb,
                                                 p->sm_count, st)
                             : dsfft::fp64_execute(*p->ref64, false, bx, ax, nb, 0.0,
                                                   p->sm_count, st, &launches);
      const int e3 = dsfft::launch_widen(y, bx, (long long)(nb * n), p->precision, st);
      launches += use_dft ? 3 : 2;
      if (e1 || e2 || e3) rc = fail(DSFFT_ERR_CUDA, "error harness: reference transform failed");
    } else {  // roundtrip: inverse(forward(x)) vs x
      rc = launch(p, DSFFT_INVERSE, y, z, nb, st);
      launches += g_launches + 2;
      g_launches = 0;
      if (!rc && (dsfft::launch_widen(z, bx, (long long)(nb * n), p->precision, st) ||
                  dsfft::launch_widen(x, ax, (long long)(nb * n), p->precision, st)))
        rc = fail(DSFFT_ERR_CUDA, "error harness: widening failed");
    }
    if (rc) break;
    ++launches;
    if (dsfft::launch_rel_l2(bx, ax, derr, (long long)n, (long long)nb, st) ||
        cudaMemcpyAsync(errs.data() + b0, derr, nb * sizeof(double), cudaMemcpyDeviceToHost,
                        st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      rc = fail(DSFFT_ERR_CUDA, "error harness: reduction failed");
  }
  cleanup();
  if (rc) return rc;
  const dsfft::ErrorStats s = dsfft::aggregate_errors(errs);
  if (s.invalid) return fail(DSFFT_ERR_INVALID, "relative_l2_error: all-zero reference");
  if (out) {
    *out = dsfft_error_report{};
    out->n = p->n;
    out->strategy = p->strategy;
    out->precision = p->precision;
    out->metric = metric;
    out->trials = batch;
    out->rel_l2_median = s.median;
    out->rel_l2_max = s.max;
    out->nonfinite_trials = s.nonfinite;
  }
  if (errs_out) std::memcpy(errs_out, errs.data(), batch * sizeof(double));
  g_launches = launches;
  return DSFFT_OK;
}

int dsfft_error_device(dsfft_plan p, int metric, const void* d_x, size_t batch, void* stream_,
                       dsfft_error_report* out, double* errs_out) {
  return dsfft_error_device_ex(p, metric, DSFFT_REF_AUTO, d_x, batch, stream_, out, errs_out);
}

int dsfft_dft_device(const void* d_in, void* d_out, size_t n, size_t batch, int device,
                     void* stream_) {
  g_launches = 0;
  if (!d_in || !d_out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (n < 1 || n > (size_t(1) << 24)) return fail(DSFFT_ERR_INVALID, "dft_oracle: n out of range");
  if (d_in == d_out) return fail(DSFFT_ERR_INVALID, "dft_oracle is out of place");
  if ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out)) & 15)
    return fail(DSFFT_ERR_INVALID, "device buffers must be 16-byte aligned");
  if (batch == 0) return DSFFT_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  const std::vector<double> tw = dsfft::dft_table(n);
  double2* dtw = nullptr;
  DSFFT_CUDA(dsfft::scratch_alloc(reinterpret_cast<void**>(&dtw), n * sizeof(double2), st));
  struct Release {
    double2* s;
    cudaStream_t st;
    ~Release() { dsfft::scratch_free(s, st); }
  } release{dtw, st};
  DSFFT_CUDA(cudaMemcpyAsync(dtw, tw.data(), n * sizeof(double2), cudaMemcpyHostToDevice, st));
  if (dsfft::launch_dft(static_cast<const double2*>(d_in), static_cast<double2*>(d_out), dtw,
                        (long long)n, (long long)batch, sms, st))
    return cuda_fail(cudaGetLastError(), "dft kernel launch");
  // the host table must outlive the async upload
  DSFFT_CUDA(cudaStreamSynchronize(st));
  g_launches = 1;
  return DSFFT_OK;
}

int dsfft_fill_uniform(void* d_out, size_t n, uint64_t first_transform, size_t count,
                       uint64_t seed, int precision, int device, void* stream_) {
  g_launches = 0;
  if (!d_out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (precision < DSFFT_FP16 || precision > DSFFT_FP64)
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  if (n && count > (SIZE_MAX / 16) / n)
    return fail(DSFFT_ERR_INVALID, "count too large: byte count overflows size_t");
  if (n == 0 || count == 0) return DSFFT_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (dsfft::launch_fill_uniform(d_out, n, first_transform, count, seed, precision, sms,
                                 static_cast<cudaStream_t>(stream_)))
    return cuda_fail(cudaGetLastError(), "fill_uniform launch");
  g_launches = 1;
  return DSFFT_OK;
}

}  // extern "C"

namespace {

// Host arrays -> device, one emulation kernel, results back (synchronous).
template <class Launch>
int emulate_call(int device, size_t in_bytes, const void* const* ins, int n_in, void* out,
                 size_t out_bytes, Launch&& launch) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(device);
  void* d[4] = {};
  void* d_out = nullptr;
  auto cleanup = [&] {
    for (void* p : d) cudaFree(p);
    cudaFree(d_out);
  };
  int rc = DSFFT_OK;
  for (int i = 0; i < n_in && !rc; ++i)
    if (cudaMalloc(&d[i], in_bytes) != cudaSuccess ||
        cudaMemcpy(d[i], ins[i], in_bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail(DSFFT_ERR_CUDA, "emulation: upload failed");
  if (!rc && cudaMalloc(&d_out, out_bytes) != cudaSuccess)
    rc = fail(DSFFT_ERR_CUDA, "emulation: device allocation failed");
  if (!rc && launch(d, d_out)) rc = cuda_fail(cudaGetLastError(), "emulation kernel launch");
  if (!rc && cudaMemcpy(out, d_out, out_bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(DSFFT_ERR_CUDA, "emulation: download failed");
  cleanup();
  if (!rc) g_launches = 1;
  return rc;
}

}  // namespace

extern "C" {

int dsfft_context_ops(int precision, int op, const double* a, const double* b, const double* c,
                      double* out, size_t count, int device) {
  g_launches = 0;
  if (precision < DSFFT_FP16 || precision > DSFFT_FP64)
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  if (op < DSFFT_OP_ADD || op > DSFFT_OP_FMA) return fail(DSFFT_ERR_INVALID, "unknown operation");
  if (!a || !b || !out || (op == DSFFT_OP_FMA && !c)) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (count == 0) return DSFFT_OK;
  if (count > SIZE_MAX / 8) return fail(DSFFT_ERR_INVALID, "count too large");
  const size_t bytes = count * sizeof(double);
  const void* ins[3] = {a, b, op == DSFFT_OP_FMA ? c : a};
  return emulate_call(device, bytes, ins, 3, out, bytes, [&](void** d, void* o) {
    return dsfft::launch_context_ops(precision, op, static_cast<const double*>(d[0]),
                                     static_cast<const double*>(d[1]),
                                     static_cast<const double*>(d[2]), static_cast<double*>(o),
                                     (long long)count, nullptr);
  });
}

int dsfft_butterflies(int strategy, int precision, const double* a, const double* b,
                      const dsfft_entry* entries, double* out, size_t count, int device) {
  g_launches = 0;
  if (precision < DSFFT_FP16 || precision > DSFFT_FP64)
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  if (strategy < DSFFT_STANDARD || strategy > DSFFT_DUAL_SELECT)
    return fail(DSFFT_ERR_INVALID, "unknown strategy");  // kernel_for (butterfly.cpp:82-90)
  if (!a || !b || !entries || !out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (count == 0) return DSFFT_OK;
  if (count > SIZE_MAX / 64) return fail(DSFFT_ERR_INVALID, "count too large");
  const size_t cb = count * 2 * sizeof(double);
  // a, b: count x 16 B (emulate_call); the 40-byte entries go up separately
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(device);
  dsfft_entry* d_e = nullptr;
  if (cudaMalloc(&d_e, count * sizeof(dsfft_entry)) != cudaSuccess ||
      cudaMemcpy(d_e, entries, count * sizeof(dsfft_entry), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    cudaFree(d_e);
    return fail(DSFFT_ERR_CUDA, "emulation: upload failed");
  }
  const void* ins[2] = {a, b};
  const int rc = emulate_call(device, cb, ins, 2, out, 2 * cb, [&](void** d, void* o) {
    return dsfft::launch_butterflies(strategy, precision, static_cast<const double2*>(d[0]),
                                     static_cast<const double2*>(d[1]), d_e,
                                     static_cast<double*>(o), (long long)count, nullptr);
  });
  cudaFree(d_e);
  return rc;
}

int dsfft_dft_oracle(const double* in, double* out, size_t n, size_t batch, int device) {
  g_launches = 0;
  if (!in || !out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (n < 1 || n > (size_t(1) << 24)) return fail(DSFFT_ERR_INVALID, "dft_oracle: n out of range");
  if (batch == 0) return DSFFT_OK;
  if (batch > (SIZE_MAX / 32) / n)
    return fail(DSFFT_ERR_INVALID, "batch too large: byte count overflows size_t");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DSFFT_ERR_NO_DEVICE, "no CUDA device: dsfft has no CPU fallback");
  }
  if (device < 0 || device >= ndev) return fail(DSFFT_ERR_INVALID, "device ordinal out of range");
  DeviceGuard guard(device);
  const size_t bytes = batch * n * sizeof(double2);
  void *dx = nullptr, *dy = nullptr;
  if (cudaMalloc(&dx, bytes) != cudaSuccess || cudaMalloc(&dy, bytes) != cudaSuccess) {
    cudaFree(dx);
    cudaGetLastError();
    return fail(DSFFT_ERR_CUDA, "dft_oracle: device allocation failed");
  }
  int rc = DSFFT_OK;
  if (cudaMemcpy(dx, in, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(DSFFT_ERR_CUDA, "dft_oracle: upload failed");
  if (!rc) rc = dsfft_dft_device(dx, dy, n, batch, device, nullptr);
  if (!rc && cudaMemcpy(out, dy, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(DSFFT_ERR_CUDA, "dft_oracle: download failed");
  cudaFree(dx);
  cudaFree(dy);
  return rc;
}

int dsfft_measure_error(size_t n, int strategy, int precision, int metric, size_t trials,
                        uint64_t seed, int device, dsfft_error_report* out) {
  if (trials < 1) return fail(DSFFT_ERR_INVALID, "trials must be >= 1");
  dsfft_plan p = nullptr;
  int rc = dsfft_plan_create(n, strategy, precision, 1e-7, device, &p);
  if (rc) return rc;
  DeviceGuard guard(device);
  // the reference protocol: one SplitMix64 stream, 2n draws per trial, re then
  // im, uniform [-1, 1) (analysis.hpp:73-91, analysis.cpp:120-125), then
  // ingest-rounded (analysis.cpp:126-130)
  uint64_t state = seed;
  auto next = [&state]() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  std::vector<double> draws(2 * n * trials);
  for (double& d : draws) d = 2.0 * (static_cast<double>(next() >> 11) * 0x1p-53) - 1.0;
  const size_t tb = n * sample_bytes(precision);
  std::vector<uint8_t> host(tb * trials);
  rc = dsfft_round_to(draws.data(), host.data(), draws.size(), precision);
  void* d_x = nullptr;
  if (!rc && cudaMalloc(&d_x, host.size()) != cudaSuccess) rc = fail(DSFFT_ERR_CUDA, "alloc");
  if (!rc && cudaMemcpy(d_x, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(DSFFT_ERR_CUDA, "upload");
  // the reference's dft_oracle (bit-identical reports) wherever the O(n^2)
  // DFT stays cheap on the device; the fp64 FFT beyond
  const int ref = n <= (size_t(1) << 16) ? DSFFT_REF_DFT : DSFFT_REF_FFT64;
  if (!rc) rc = dsfft_error_device_ex(p, metric, ref, d_x, trials, nullptr, out, nullptr);
  if (!rc && out) out->seed = seed;
  if (d_x) cudaFree(d_x);
  dsfft_plan_destroy(p);
  return rc;
}

int dsfft_round_to(const double* in, void* out, size_t count, int precision) {
  if (!in || !out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (precision == DSFFT_FP16) {
    auto* o = static_cast<uint16_t*>(out);
    for (size_t i = 0; i < count; ++i) o[i] = dsfft::half_bits(in[i]);
  } else if (precision == DSFFT_FP32) {
    auto* o = static_cast<float*>(out);
    for (size_t i = 0; i < count; ++i) o[i] = float(dsfft::round_to(in[i], dsfft::kFp32));
  } else if (precision == DSFFT_FP64) {
    std::memcpy(out, in, count * sizeof(double));
  } else {
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  }
  return DSFFT_OK;
}

int dsfft_widen(const void* in, double* out, size_t count, int precision) {
  if (!in || !out) return fail(DSFFT_ERR_INVALID, "null buffer");
  if (precision == DSFFT_FP16) {
    auto* s = static_cast<const uint16_t*>(in);
    for (size_t i = 0; i < count; ++i) out[i] = dsfft::half_value(s[i]);
  } else if (precision == DSFFT_FP32) {
    auto* s = static_cast<const float*>(in);
    for (size_t i = 0; i < count; ++i) out[i] = double(s[i]);
  } else if (precision == DSFFT_FP64) {
    std::memcpy(out, in, count * sizeof(double));
  } else {
    return fail(DSFFT_ERR_INVALID, "unknown precision: " + std::to_string(precision));
  }
  return DSFFT_OK;
}

int dsfft_execute_f64(dsfft_plan p, int dir, const double* in, double* out, size_t batch) {
  g_launches = 0;
  int rc = check_exec_args(p, dir, in, out, batch);
  if (rc) return rc;
  const size_t count = 2 * p->n * batch;
  std::vector<uint8_t> a(count * (sample_bytes(p->precision) / 2) + 16);
  std::vector<uint8_t> b(a.size());
  // 16-byte alignment is not needed on the host side (copies are staged)
  rc = dsfft_round_to(in, a.data(), count, p->precision);
  if (rc) return rc;
  rc = dsfft_execute_host(p, dir, a.data(), b.data(), batch, nullptr);
  if (rc) return rc;
  return dsfft_widen(b.data(), out, count, p->precision);
}

}  // extern "C"
