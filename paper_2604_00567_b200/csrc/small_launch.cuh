// small_launch.cuh -- per-size instantiation and launch of fft_small_kernel.
//
// Each csrc/inst_m<M>.cu instantiates the 8 kernels (fp16/fp32 x
// FMA/standard x forward/inverse) of one transform size M = log2 N, so the
// heavily unrolled kernels compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "fft_kernels.cuh"

namespace dsfft {

// Runtime description of a compiled configuration (mirrors Sched<>).
struct SmallGeom {
  int m, log_e, warps, nstage;
  int s[4], P[4], tw_off[5];
  int tw_records, vals, k, buf_bytes, item_bytes, max_threads;
};

struct LaunchArgs {
  bool f16, standard, inverse;
  KernelParams kp;
  cudaStream_t stream;
  int grid, groups;
};

using SmallLaunchFn = cudaError_t (*)(const LaunchArgs&);

struct SmallEntry {
  SmallGeom geom;
  SmallLaunchFn launch;
  size_t (*smem_bytes)(int groups, int stages);
};

template <class Cfg>
SmallGeom make_geom() {
  SmallGeom g{};
  g.m = Cfg::LOG_N;
  g.log_e = Cfg::LOG_E;
  g.warps = Cfg::W;
  g.nstage = Cfg::NSTAGE;
  for (int i = 0; i < 4; ++i) {
    g.s[i] = Cfg::s(i);
    g.P[i] = Cfg::P(i);
  }
  for (int i = 0; i <= 4; ++i) g.tw_off[i] = i <= Cfg::NSTAGE ? Cfg::tw_off(i) : 0;
  g.tw_records = Cfg::TW_RECORDS;
  g.vals = Cfg::VALS;
  g.k = Cfg::K;
  g.buf_bytes = SmallLayout<Cfg>::kBufBytes;
  g.item_bytes = SmallLayout<Cfg>::kItemBytes;
  g.max_threads = Cfg::MAX_THREADS;
  return g;
}

template <class Cfg, bool F16, bool STD, bool INV>
cudaError_t launch_variant(const LaunchArgs& a) {
  auto kern = fft_small_kernel<Cfg, F16, STD, INV>;
  const size_t smem = SmallLayout<Cfg>::smem_bytes(a.groups, a.kp.stages);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(smem));
  if (e != cudaSuccess) return e;
  kern<<<a.grid, a.groups * Cfg::T, smem, a.stream>>>(a.kp);
  return cudaGetLastError();
}

template <class Cfg>
cudaError_t launch_small(const LaunchArgs& a) {
  if (a.f16) {
    if (a.standard)
      return a.inverse ? launch_variant<Cfg, true, true, true>(a)
                       : launch_variant<Cfg, true, true, false>(a);
    return a.inverse ? launch_variant<Cfg, true, false, true>(a)
                     : launch_variant<Cfg, true, false, false>(a);
  }
  if (a.standard)
    return a.inverse ? launch_variant<Cfg, false, true, true>(a)
                     : launch_variant<Cfg, false, true, false>(a);
  return a.inverse ? launch_variant<Cfg, false, false, true>(a)
                   : launch_variant<Cfg, false, false, false>(a);
}

template <class Cfg>
size_t small_smem_bytes(int groups, int stages) {
  return SmallLayout<Cfg>::smem_bytes(groups, stages);
}

template <class Cfg>
SmallEntry make_small_entry() {
  return SmallEntry{make_geom<Cfg>(), &launch_small<Cfg>, &small_smem_bytes<Cfg>};
}

// Defined in inst_m<M>.cu
SmallEntry small_entry_m1();
SmallEntry small_entry_m2();
SmallEntry small_entry_m3();
SmallEntry small_entry_m4();
SmallEntry small_entry_m5();
SmallEntry small_entry_m6();
SmallEntry small_entry_m7();
SmallEntry small_entry_m8();
SmallEntry small_entry_m9();
SmallEntry small_entry_m10();
SmallEntry small_entry_m11();
SmallEntry small_entry_m12();

}  // namespace dsfft
