// host_table.hpp -- host-side twiddle-table builder and device-record packer.
//
// The table stays on the host and is built with the reference's algorithm so
// that it is bit-identical to fmafft::make_plan's (checked against the
// reference library in tests/test_tables.py):
//   twiddle_angle           twiddle.cpp:55-57
//   build_*_table           twiddle.cpp:59-141 (dual = Algorithm 1, tie -> COS)
//   round once into p       fft.cpp:65-70 / round_to precision.cpp:61-75
// Compiled with -ffp-contract=off (the reference's rule, CMakeLists.txt:11-13)
// and glibc libm cos/sin, the reference's own trig.
#pragma once
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace dsfft {

enum Strategy : int { kStandard = 0, kLinzerFeig = 1, kCosine = 2, kDual = 3 };
enum Precision : int { kFp16 = 0, kFp32 = 1, kFp64 = 2 };
enum Path : int { kCos = 0, kSin = 1 };

struct TableEntry {
  double multiplier = 0.0;
  double ratio = 0.0;
  int path = kCos;
  bool clamped = false;
  double omega_r = 0.0;
  double omega_i = 0.0;
};

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// theta_k = -(2 pi) * (k / n)
double twiddle_angle(std::size_t k, std::size_t n);

// dft_oracle's twiddles (fft.cpp:103-121), indexed by r = (j k) mod n:
// interleaved (cos theta_r, sin theta_r), 2n doubles, any n >= 1.
std::vector<double> dft_table(std::size_t n);

// FP64 table of n/2 entries (throws InvalidArgument like the reference).
std::vector<TableEntry> build_table(std::size_t n, int strategy, double clamp_eps);

// make_plan's table: validated (n <= 2^24), FP64, then rounded once into p.
std::vector<TableEntry> plan_table(std::size_t n, int strategy, int precision,
                                   double clamp_eps);

// IEEE binary16 round-to-nearest-even of a double (== round_to(x, fp16)).
uint16_t half_bits(double x);
double half_value(uint16_t h);
double round_to(double x, int precision);

// Device twiddle record (see fft_kernels.cuh), 16 bytes:
//   FMA strategies: (t, w' = COS ? w : -w, w, PRMT selector)
//   standard:       (omega_r, omega_i, 0, 0)
// fp32 words hold binary32 bits.  fp16 transform pairs use 8 bytes,
//   x = (t | w' << 16), y = (selector | w << 16)   (standard: x = (omega_r | omega_i << 16))
// and the kernel broadcasts each half into both f16x2 lanes (folded into the
// HFMA2 operand selects .H0_H0 / .H1_H1, no extra instructions).  fp16 one
// complex per register: see pack_record.
struct Record {
  uint32_t x, y, z, w;
};
Record pack_record(const TableEntry& rounded, int strategy, int precision,
                   bool f16_complex = false);
// Bytes per device record for a precision / fp16 layout (8 or 16).
int record_bytes(int precision, bool f16_complex);
// Records -> device byte image (record_bytes each, padded to 16 bytes).
std::vector<uint8_t> serialize_records(const std::vector<Record>& recs, int rec_bytes);

// Effective (t, w, cos?) a butterfly uses for an entry: mirrors the operand
// choice of butterfly_linzer_feig / butterfly_cosine / butterfly_dual
// (butterfly.cpp:55-80), including LF's clamped k=0 -> cosine_core(omega_i, omega_r).
void effective_operands(const TableEntry& e, int strategy, double* t, double* w, bool* cos);

}  // namespace dsfft
