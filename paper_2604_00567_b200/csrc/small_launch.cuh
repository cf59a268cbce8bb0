// small_launch.cuh -- per-size instantiation and launch of fft_small_kernel.
//
// Each csrc/inst_small.cu object (compiled with -DDSFFT_M=<log2 N>)
// instantiates the kernels of one transform size for three value layouts
// (fp32, fp16 transform-pairs, fp16 complex) x {FMA, standard} x {forward,
// inverse}, so the heavily unrolled kernels compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "fft_kernels.cuh"

namespace dsfft {

enum SmallVariantId : int { kVarF32 = 0, kVarF16P = 1, kVarF16C = 2 };

// Runtime description of a compiled configuration (mirrors Sched<>).
struct SmallGeom {
  int m, log_e, warps, nstage;
  int s[4], P[4], tw_off[5];
  int tw_records, vals, k, max_threads;
  int tpi;         // real transforms per item
  int item_bytes;  // bytes of one item in global memory
};

struct LaunchArgs {
  bool standard, inverse;
  KernelParams kp;
  cudaStream_t stream;
  int grid, groups;
};

using SmallLaunchFn = cudaError_t (*)(const LaunchArgs&);

struct SmallVariant {
  SmallGeom geom;
  SmallLaunchFn launch;
  size_t (*smem_bytes)(int groups, int stages);
};

struct SmallEntry {
  SmallVariant v[3];     // indexed by SmallVariantId
  int f16_default;       // kVarF16P or kVarF16C
  int stages[3];         // default item buffers per group, per variant (measured)
};

template <class Cfg, class A>
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
  g.max_threads = max_threads<Cfg, A>();
  g.tpi = SmallLayout<Cfg, A>::kTpi;
  g.item_bytes = SmallLayout<Cfg, A>::kItemBytes;
  return g;
}

template <class Cfg, class A, bool STD, bool INV>
cudaError_t launch_variant(const LaunchArgs& a) {
  auto kern = fft_small_kernel<Cfg, A, STD, INV>;
  const size_t smem = SmallLayout<Cfg, A>::smem_bytes(a.groups, a.kp.stages);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(smem));
  if (e != cudaSuccess) return e;
  kern<<<a.grid, a.groups * Cfg::T, smem, a.stream>>>(a.kp);
  return cudaGetLastError();
}

template <class Cfg, class A>
cudaError_t launch_small(const LaunchArgs& a) {
  if (a.standard)
    return a.inverse ? launch_variant<Cfg, A, true, true>(a) : launch_variant<Cfg, A, true, false>(a);
  return a.inverse ? launch_variant<Cfg, A, false, true>(a) : launch_variant<Cfg, A, false, false>(a);
}

template <class Cfg, class A>
size_t small_smem_bytes(int groups, int stages) {
  return SmallLayout<Cfg, A>::smem_bytes(groups, stages);
}

template <class Cfg, class A>
SmallVariant make_variant() {
  return SmallVariant{make_geom<Cfg, A>(), &launch_small<Cfg, A>, &small_smem_bytes<Cfg, A>};
}

// Defined in inst_small.cu (one object per M)
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
SmallEntry small_entry_m13();

}  // namespace dsfft
