// fp64.cu -- the Precision::fp64 device path.
//
// The reference's fp64 arithmetic is plain IEEE binary64 with a fused
// std::fma (precision.cpp:107-108), i.e. DFMA / DMUL / DADD on the GPU.  The
// dataflow is run_passes itself (fft.cpp:32-52): one launch per pass, each
// thread one butterfly X[j], X[j+N/2] -> Y[(j>>p)*2^(p+1) + (j mod 2^p)] (+2^p),
// ping-ponging through two scratch buffers so the last pass writes the output
// (in-place safe).  fp64 is the drop-in's accuracy path (the reference's own
// oracle-equivalence / op-count tests run at fp64), not a throughput path.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fp64.cuh"
#include "stream_alloc.cuh"

namespace dsfft {

namespace {
thread_local std::string g_f64_err;
}

const char* fp64_error() { return g_f64_err.c_str(); }

// Effective operands of one entry (host_table.cpp effective_operands):
// FMA strategies (t, w' = COS ? w : -w, w, cos); standard (omega_r, omega_i).
struct Rec64 {
  double a, b, c;
  int cos;
  int pad;
};

struct F64Plan {
  int m = 0, strategy = 0;
  Rec64* d_tab = nullptr;
  ~F64Plan() {
    if (d_tab) cudaFree(d_tab);
  }
};

template <bool STANDARD, bool CONJ_IN, bool SCALE_OUT>
__global__ void __launch_bounds__(256) fft64_pass(const double2* __restrict__ X,
                                                  double2* __restrict__ Y,
                                                  const Rec64* __restrict__ tab, long long total,
                                                  int m, int p, double scale) {
  const long long half = 1LL << (m - 1);
  const long long block = 1LL << p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i >> (m - 1), j = i & (half - 1);
    const double2* x = X + (b << m);
    double2 a = x[j], bb = x[j + half];
    if constexpr (CONJ_IN) {  // conj on load (fft.cpp:90-91)
      a.y = -a.y;
      bb.y = -bb.y;
    }
    const long long jq = j & (block - 1);
    const Rec64 e = tab[jq << (m - p - 1)];
    double2 A, B;
    if constexpr (STANDARD) {  // butterfly.cpp:37-53, every op rounded separately
      const double rr = __dmul_rn(e.a, bb.x), ii = __dmul_rn(e.b, bb.y);
      const double ir = __dmul_rn(e.b, bb.x), ri = __dmul_rn(e.a, bb.y);
      const double tr = __dsub_rn(rr, ii), ti = __dadd_rn(ir, ri);
      A = make_double2(__dadd_rn(a.x, tr), __dadd_rn(a.y, ti));
      B = make_double2(__dsub_rn(a.x, tr), __dsub_rn(a.y, ti));
    } else {  // unified cosine_core / sine_core (butterfly.cpp:10-33)
      const double xx = e.cos ? bb.x : bb.y, yy = e.cos ? bb.y : bb.x;
      const double u1 = __fma_rn(-e.a, yy, xx), u2 = __fma_rn(e.a, xx, yy);
      A = make_double2(__fma_rn(u1, e.b, a.x), __fma_rn(u2, e.c, a.y));
      B = make_double2(__fma_rn(-u1, e.b, a.x), __fma_rn(-u2, e.c, a.y));
    }
    if constexpr (SCALE_OUT) {  // conj + 1/n, one rounded mul each (fft.cpp:94-98)
      A = make_double2(__dmul_rn(A.x, scale), __dmul_rn(-A.y, scale));
      B = make_double2(__dmul_rn(B.x, scale), __dmul_rn(-B.y, scale));
    }
    double2* y = Y + (b << m);
    const long long base = ((j >> p) << (p + 1)) + jq;
    y[base] = A;
    y[base + block] = B;
  }
}

F64Plan* fp64_create(const std::vector<TableEntry>& table, int m, int strategy) {
  auto* fp = new F64Plan();
  fp->m = m;
  fp->strategy = strategy;
  std::vector<Rec64> recs(table.size());
  for (size_t k = 0; k < table.size(); ++k) {
    const TableEntry& e = table[k];
    if (strategy == kStandard) {
      recs[k] = Rec64{e.omega_r, e.omega_i, 0.0, 1, 0};
    } else {
      double t, w;
      bool cos;
      effective_operands(e, strategy, &t, &w, &cos);
      recs[k] = Rec64{t, cos ? w : -w, w, cos ? 1 : 0, 0};
    }
  }
  if (cudaMalloc(&fp->d_tab, recs.size() * sizeof(Rec64)) != cudaSuccess ||
      cudaMemcpy(fp->d_tab, recs.data(), recs.size() * sizeof(Rec64), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    g_f64_err = "fp64: table upload failed";
    delete fp;
    return nullptr;
  }
  return fp;
}

void fp64_destroy(F64Plan* fp) { delete fp; }

int fp64_execute(F64Plan& fp, bool inverse, const void* in, void* out, size_t batch,
                 double scale, int sm_count, cudaStream_t st, uint64_t* launches) {
  const int m = fp.m;
  const size_t tb = (size_t(1) << m) * sizeof(double2);
  // per-call, stream-ordered ping-pong buffers (plans may run on several
  // streams), at most 256 MiB each: the batch runs in chunks
  const size_t chunk = std::max<size_t>(1, std::min(batch, (size_t(256) << 20) / tb));
  double2* scratch[2] = {nullptr, nullptr};
  if (m > 1)
    for (auto*& sp : scratch)
      if (scratch_alloc(reinterpret_cast<void**>(&sp), chunk * tb, st) != cudaSuccess) {
        scratch_free(scratch[0], st);
        g_f64_err = "fp64: scratch allocation failed";
        return 1;
      }
  struct Release {
    double2** s;
    cudaStream_t st;
    ~Release() {
      scratch_free(s[0], st);
      scratch_free(s[1], st);
    }
  } release{scratch, st};
  const bool std_ = fp.strategy == kStandard;
  for (size_t b0 = 0; b0 < batch; b0 += chunk) {
    const size_t nb = std::min(chunk, batch - b0);
    const long long total = (long long)nb << (m - 1);
    const int grid = int(std::min<long long>((total + 255) / 256, (long long)sm_count * 8));
    const double2* src = static_cast<const double2*>(in) + (b0 << m);
    double2* dst = static_cast<double2*>(out) + (b0 << m);
    for (int p = 0; p < m; ++p) {
      const double2* X = p == 0 ? src : scratch[(p - 1) & 1];
      double2* Y = p == m - 1 ? dst : scratch[p & 1];
      const bool ci = inverse && p == 0, so = inverse && p == m - 1;
      auto go = [&](auto kern) { kern<<<grid, 256, 0, st>>>(X, Y, fp.d_tab, total, m, p, scale); };
      if (std_) {
        if (ci && so) go(fft64_pass<true, true, true>);
        else if (ci) go(fft64_pass<true, true, false>);
        else if (so) go(fft64_pass<true, false, true>);
        else go(fft64_pass<true, false, false>);
      } else {
        if (ci && so) go(fft64_pass<false, true, true>);
        else if (ci) go(fft64_pass<false, true, false>);
        else if (so) go(fft64_pass<false, false, true>);
        else go(fft64_pass<false, false, false>);
      }
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        g_f64_err = std::string("fft64_pass launch: ") + cudaGetErrorString(e);
        return 1;
      }
      if (launches) ++*launches;
    }
  }
  return 0;
}

}  // namespace dsfft
