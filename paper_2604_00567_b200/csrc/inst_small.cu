// inst_small.cu -- compiled once per transform size with -DDSFFT_M=<log2 N>;
// defines small_entry_m<M>() with that size's schedules (tools/
// schedule_check.cpp proves each dataflow-exact and counts its bank
// conflicts).  CfgW: two-word values (fp32 complex, fp16 transform pairs);
// CfgC: one-word values (fp16 complex in one f16x2 register).
#include "small_launch.cuh"

#ifndef DSFFT_M
#error "compile with -DDSFFT_M=<log2 N>"
#endif

namespace dsfft {

//            LOG_N LOG_E W  stages (passes per register stage)
#if DSFFT_M == 1
using CfgW = Sched<1, 5, 1, 1>;
using CfgC = CfgW;
#elif DSFFT_M <= 5
// A single register stage would have lane t read (and store) values t*32..:
// stride-N lanes, 32-way shared-memory conflicts and uncoalesced stores
// (schedule_check: 1024/32 load wavefronts at N=32).  Splitting off one-pass
// stages at both ends keeps the TMA tile reads and the global stores
// lane-contiguous (64/32) at the cost of two padded exchanges.
using CfgW = std::conditional_t<DSFFT_M == 2, Sched<2, 5, 1, 1, 1>,
             std::conditional_t<DSFFT_M == 3, Sched<3, 5, 1, 1, 1, 1>,
             std::conditional_t<DSFFT_M == 4, Sched<4, 5, 1, 1, 2, 1>, Sched<5, 5, 1, 1, 3, 1>>>>;
using CfgC = CfgW;
#elif DSFFT_M == 6
using CfgW = Sched<6, 5, 1, 3, 3>;
using CfgC = Sched<6, 5, 1, 1, 4, 1>;  // conflict-free for 4-byte values
#elif DSFFT_M == 7
using CfgW = Sched<7, 5, 1, 4, 3>;
using CfgC = Sched<7, 5, 1, 1, 5, 1>;
#elif DSFFT_M == 8
using CfgW = Sched<8, 5, 1, 4, 4>;
using CfgC = Sched<8, 5, 1, 1, 5, 2>;  // conflict-free for 4-byte values
#elif DSFFT_M == 9
using CfgW = Sched<9, 5, 1, 5, 4>;
using CfgC = CfgW;
#elif DSFFT_M == 10
using CfgW = Sched<10, 5, 1, 5, 5>;
using CfgC = CfgW;
#elif DSFFT_M == 11
// 32 values per thread over 2 warps: (E=64, 1 warp) needed ~210 registers and
// 33 KB per group, leaving ~4 resident warps per SM
using CfgW = Sched<11, 5, 2, 5, 5, 1>;
// one-word values: 64 per thread is ~64 data registers, so two stages fit
using CfgC = Sched<11, 6, 1, 5, 6>;
#elif DSFFT_M == 12
using CfgW = Sched<12, 5, 4, 5, 5, 2>;
using CfgC = Sched<12, 6, 2, 6, 6>;
#elif DSFFT_M == 13
// 8 warps per item, conflict-free for every value width (schedule_check);
// fp16 pairs: 64 KB of 8-byte records + two 66 KB items per SM
using CfgW = Sched<13, 5, 8, 5, 5, 3>;
using CfgC = CfgW;
#else
#error "single-kernel path covers N <= 8192"
#endif

#ifdef DSFFT_OV_E  // schedule experiments (tools/sched_variants.py)
using CfgWX = Sched<DSFFT_M, DSFFT_OV_E, DSFFT_OV_W, DSFFT_OV_S0, DSFFT_OV_S1, DSFFT_OV_S2,
                    DSFFT_OV_S3>;
#else
using CfgWX = CfgW;
#endif

// fp32 at N = 256 / 512: 16 values per thread (E=16, ~80 registers) and more
// resident warps beat E=32 (B200 sweep at >= 4 GiB per step: +2% / +4%)
#if DSFFT_M == 8
using CfgF = Sched<8, 4, 1, 4, 4>;
#elif DSFFT_M == 9
using CfgF = Sched<9, 4, 1, 4, 4, 1>;
#else
using CfgF = CfgWX;
#endif
#define DSFFT_CAT2(a, b) a##b
#define DSFFT_CAT(a, b) DSFFT_CAT2(a, b)
SmallEntry DSFFT_CAT(small_entry_m, DSFFT_M)() {
  SmallEntry e{};
  e.v[kVarF32] = make_variant<CfgF, ArithF32>();
  e.v[kVarF16P] = make_variant<CfgWX, ArithF16P>();
  e.v[kVarF16C] = make_variant<CfgC, ArithF16C>();
  // Defaults from B200 sweeps (profiles/README.md, "launch shapes"):
  // with 8-byte records, fp16 transform pairs win from N = 128 (95-97% of HBM
  // with a 1-deep ring vs 92% one-complex) up; one complex per register (3-deep
  // ring at N = 64) below.  N >= 2048 is
  // shared-memory bound (per-stage twiddle tables ~N*8 B plus 32 KB items),
  // where a 1-deep ring with more groups wins.
  e.f16_default = DSFFT_M >= 7 ? kVarF16P : kVarF16C;
  e.stages[kVarF32] = DSFFT_M >= 11 ? 1 : DSFFT_M == 8 ? 4 : DSFFT_M == 9 ? 2 : 3;
  // N=128 and N=1024: 1-deep rings, 16 one-warp groups (more warps beat deeper
  // rings, also under the board power cap: 84% vs 82.5% of HBM sustained at 1024)
  e.stages[kVarF16P] = (DSFFT_M >= 10 || DSFFT_M == 7) ? 1 : 2;
  e.stages[kVarF16C] = DSFFT_M >= 11 ? 1 : DSFFT_M == 6 ? 3 : 2;
  return e;
}

}  // namespace dsfft
