// inst_small.cu -- compiled once per transform size with -DDSFFT_M=<log2 N>;
// defines small_entry_m<M>() with that size's schedule (see schedule_check.cpp
// for the dataflow proof and bank-conflict counts of each choice).
#include "small_launch.cuh"

#ifndef DSFFT_M
#error "compile with -DDSFFT_M=<log2 N>"
#endif

namespace dsfft {

//            LOG_N LOG_E W  stages (passes per register stage)
#if DSFFT_M <= 5
using CfgM = Sched<DSFFT_M, 5, 1, DSFFT_M>;
#elif DSFFT_M == 6
using CfgM = Sched<6, 5, 1, 3, 3>;
#elif DSFFT_M == 7
using CfgM = Sched<7, 5, 1, 4, 3>;
#elif DSFFT_M == 8
using CfgM = Sched<8, 5, 1, 4, 4>;
#elif DSFFT_M == 9
using CfgM = Sched<9, 5, 1, 5, 4>;
#elif DSFFT_M == 10
using CfgM = Sched<10, 5, 1, 5, 5>;
#elif DSFFT_M == 11
using CfgM = Sched<11, 6, 1, 5, 6>;
#elif DSFFT_M == 12
using CfgM = Sched<12, 6, 2, 6, 6>;
#else
#error "single-kernel path covers N <= 4096"
#endif

#define DSFFT_CAT2(a, b) a##b
#define DSFFT_CAT(a, b) DSFFT_CAT2(a, b)
SmallEntry DSFFT_CAT(small_entry_m, DSFFT_M)() { return make_small_entry<CfgM>(); }

}  // namespace dsfft
