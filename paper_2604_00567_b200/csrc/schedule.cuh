// schedule.cuh -- index math of the regrouped Stockham schedule.
//
// Shared by the sm_100a kernels (fft_kernels.cuh) and the host-side schedule
// checker (tools/schedule_check.cpp), which proves on the CPU that a kernel
// configuration performs exactly the reference's butterfly dataflow graph and
// counts its shared-memory bank conflicts.
//
// Reference dataflow (run_passes, fft.cpp:32-52): pass p in [0, m) pairs
// X[j] with X[j + N/2] (j < N/2) under table entry (j mod 2^p) * N/2^(p+1)
// and writes Y[(j>>p)*2^(p+1) + (j mod 2^p)] = A, Y[... + 2^p] = B.
// After passes 0..P-1, buffer position q*2^P + r holds frequency r of the
// length-2^P DFT of x[q + s*N/2^P] (q < N/2^P).
//
// Regrouping (bit-exact): a *stage* runs passes
// [P, P+s) on independent *groups*.  Group g = q_low*2^P + r
// (q_low < N/2^(P+s), r < 2^P) gathers the 2^s values at positions
// g + c*N/2^s (c < 2^s), runs s local passes whose butterfly (pl, rl) uses
// global table entry (r + 2^P*rl) * N/2^(P+pl+1), and scatters its outputs to
// q_low*2^(P+s) + r + 2^P*c'.  Every butterfly keeps its operands, operand
// order and twiddle, so results are bit-identical to the reference.
//
// Items: a thread group of T threads processes an *item* of K "virtual
// transforms" of N values (a value is one FP32 complex, or for FP16 the same
// sample of two transforms packed as (re0,re1),(im0,im1)).  Thread t owns
// groups G = t + T*j (j < E/2^s) of every stage; G = k*(N/2^s) + g.
#pragma once

#if defined(__CUDACC__)
#define DSFFT_HD __host__ __device__ __forceinline__
#else
#define DSFFT_HD inline
#endif

namespace dsfft {

// Padded exchange layout: one 8-byte pad value after every 32 values keeps
// the column walks of the next stage on distinct banks.
constexpr int kPadShift = 5;
DSFFT_HD constexpr int pad_pos(int pos) { return pos + (pos >> kPadShift); }
DSFFT_HD constexpr int padded_size(int vals) { return vals + (vals >> kPadShift); }

// Stage geometry helpers (m = log2 N, P = first pass, s = passes in stage).
DSFFT_HD constexpr int grp_k(int m, int s, int G) { return G >> (m - s); }
DSFFT_HD constexpr int grp_g(int m, int s, int G) { return G & ((1 << (m - s)) - 1); }

// Logical position the c-th input of group G is read from.
DSFFT_HD constexpr int read_pos(int m, int /*P*/, int s, int G, int c) {
  return (grp_k(m, s, G) << m) + grp_g(m, s, G) + (c << (m - s));
}

// Logical position the c-th output of group G is written to.
DSFFT_HD constexpr int write_pos(int m, int P, int s, int G, int c) {
  const int g = grp_g(m, s, G);
  const int q = g >> P, r = g & ((1 << P) - 1);
  return (grp_k(m, s, G) << m) + (q << (P + s)) + r + (c << P);
}

// Frequency index r of group G (selects its twiddles).
DSFFT_HD constexpr int grp_r(int m, int P, int s, int G) {
  return grp_g(m, s, G) & ((1 << P) - 1);
}

// Global table entry used by local butterfly (pl, rl) of a group with freq r.
DSFFT_HD constexpr int tw_entry(int m, int P, int r, int pl, int rl) {
  return (r + (rl << P)) << (m - P - pl - 1);
}

// Slot of that twiddle in the per-stage device table: consecutive r are
// adjacent so lanes with consecutive groups read consecutive records (8 or 16 B).
DSFFT_HD constexpr int tw_slot(int P, int r, int pl, int rl) {
  return (((1 << pl) - 1 + rl) << P) + r;
}
DSFFT_HD constexpr int tw_stage_size(int P, int s) { return ((1 << s) - 1) << P; }

// A compile-time configuration of the single-kernel (N <= 4096) path.
//   LOG_N  transform size      LOG_E  values per thread
//   W      warps per group     S0..S3 passes per stage (sum == LOG_N)
template <int LOG_N_, int LOG_E_, int W_, int S0, int S1 = 0, int S2 = 0, int S3 = 0>
struct Sched {
  static constexpr int LOG_N = LOG_N_;
  static constexpr int N = 1 << LOG_N;
  static constexpr int LOG_E = LOG_E_;
  static constexpr int E = 1 << LOG_E;
  static constexpr int W = W_;
  static constexpr int T = 32 * W;
  static constexpr int VALS = T * E;
  static constexpr int K = VALS / N;  // virtual transforms per item
  static constexpr int NSTAGE = 1 + (S1 > 0) + (S2 > 0) + (S3 > 0);
  DSFFT_HD static constexpr int s(int i) {
    return i == 0 ? S0 : i == 1 ? S1 : i == 2 ? S2 : S3;
  }
  DSFFT_HD static constexpr int P(int i) {
    return i == 0 ? 0 : i == 1 ? S0 : i == 2 ? S0 + S1 : S0 + S1 + S2;
  }
  // Twiddle table offsets (in records) of each stage.
  DSFFT_HD static constexpr int tw_off(int i) {
    int off = 0;
    for (int k = 0; k < i; ++k) off += tw_stage_size(P(k), s(k));
    return off;
  }
  static constexpr int TW_RECORDS = tw_off(NSTAGE);
  static constexpr int BUF_VALS = padded_size(VALS);  // 8-byte values
  static_assert(S0 + S1 + S2 + S3 == LOG_N, "stages must cover every pass");
  static_assert(VALS % N == 0, "an item holds whole transforms");
  static_assert(S0 <= LOG_E && S1 <= LOG_E && S2 <= LOG_E && S3 <= LOG_E,
                "a stage's group must fit in a thread's registers");
};

}  // namespace dsfft
