// host_table.cpp -- see host_table.hpp.  Build with -ffp-contract=off.
#include "host_table.hpp"

#include <cmath>
#include <cstring>

namespace dsfft {

namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi
constexpr std::size_t kMaxFftSize = std::size_t{1} << 24;  // fft.cpp:14

void check_size(std::size_t n) {
  if (n < 2 || (n & (n - 1)) != 0)
    throw InvalidArgument("FFT size must be a power of two >= 2, got " + std::to_string(n));
}

uint64_t bits_of(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}

uint32_t f32_bits(double x) {
  const float f = static_cast<float>(x);
  uint32_t b;
  std::memcpy(&b, &f, 4);
  return b;
}


}  // namespace

std::vector<double> dft_table(std::size_t n) {
  // dft_oracle (fft.cpp:103-121): theta = -two_pi_over_n * ((j k) mod n) with
  // two_pi_over_n = (2 pi) / n, then libm cos / sin -- tabulated per residue
  std::vector<double> t(2 * n);
  const double two_pi_over_n = (2.0 * kPi) / static_cast<double>(n);
  for (std::size_t r = 0; r < n; ++r) {
    const double theta = -two_pi_over_n * static_cast<double>(r);
    t[2 * r] = std::cos(theta);
    t[2 * r + 1] = std::sin(theta);
  }
  return t;
}

double twiddle_angle(std::size_t k, std::size_t n) {
  return -(2.0 * kPi) * (static_cast<double>(k) / static_cast<double>(n));
}

std::vector<TableEntry> build_table(std::size_t n, int strategy, double clamp_eps) {
  if (strategy < kStandard || strategy > kDual) throw InvalidArgument("unknown strategy");
  if (strategy == kLinzerFeig && !(clamp_eps > 0.0))
    throw InvalidArgument("clamp_eps must be positive");
  check_size(n);
  std::vector<TableEntry> t(n / 2);
  for (std::size_t k = 0; k < n / 2; ++k) {
    const double theta = twiddle_angle(k, n);
    TableEntry& e = t[k];
    e.omega_r = std::cos(theta);
    e.omega_i = std::sin(theta);
    switch (strategy) {
      case kStandard:
        e.multiplier = e.omega_r;
        e.ratio = 0.0;
        e.path = kCos;
        break;
      case kLinzerFeig:
        e.path = kSin;
        if (e.omega_i == 0.0) {  // k = 0: sin(-0) == -0, clamp to -eps
          e.multiplier = -clamp_eps;
          e.ratio = e.omega_r / -clamp_eps;
          e.clamped = true;
        } else {
          e.multiplier = e.omega_i;
          e.ratio = e.omega_r / e.omega_i;
        }
        break;
      case kCosine:
        e.path = kCos;
        e.multiplier = e.omega_r;
        e.ratio = e.omega_i / e.omega_r;
        break;
      case kDual:  // Algorithm 1: larger magnitude is the multiplier; tie -> COS
        if (std::fabs(e.omega_r) >= std::fabs(e.omega_i)) {
          e.path = kCos;
          e.multiplier = e.omega_r;
          e.ratio = e.omega_i / e.omega_r;
        } else {
          e.path = kSin;
          e.multiplier = e.omega_i;
          e.ratio = e.omega_r / e.omega_i;
        }
        break;
    }
  }
  return t;
}

std::vector<TableEntry> plan_table(std::size_t n, int strategy, int precision,
                                   double clamp_eps) {
  if (n > kMaxFftSize) throw InvalidArgument("FFT size exceeds 2^24");
  if (precision < kFp16 || precision > kFp64) throw InvalidArgument("unknown precision");
  std::vector<TableEntry> t = build_table(n, strategy, clamp_eps);
  for (TableEntry& e : t) {
    e.multiplier = round_to(e.multiplier, precision);
    e.ratio = round_to(e.ratio, precision);
    e.omega_r = round_to(e.omega_r, precision);
    e.omega_i = round_to(e.omega_i, precision);
  }
  return t;
}

uint16_t half_bits(double x) {
  const uint64_t b = bits_of(x);
  const uint16_t sign = uint16_t((b >> 48) & 0x8000u);
  const uint64_t a = b & 0x7FFFFFFFFFFFFFFFull;
  if (a > 0x7FF0000000000000ull) return uint16_t(sign | 0x7E00u);  // NaN
  if (a >= 0x40EFFE0000000000ull) return uint16_t(sign | 0x7C00u);  // |x| >= 65520 -> inf
  const int e = int(a >> 52) - 1023;
  if (e < -25) return sign;  // below half the smallest subnormal (incl. double subnormals)
  const uint64_t sig = (a & 0xFFFFFFFFFFFFFull) | (1ull << 52);
  const int shift = e >= -14 ? 42 : 42 + (-14 - e);  // 42..53
  uint64_t keep = sig >> shift;
  const uint64_t rest = sig & ((1ull << shift) - 1);
  const uint64_t halfway = 1ull << (shift - 1);
  if (rest > halfway || (rest == halfway && (keep & 1))) ++keep;
  if (e < -14) return uint16_t(sign | keep);  // subnormal (0x400 carries into exp 1)
  int he = e + 15;
  if (keep == 0x800) {
    keep >>= 1;
    ++he;
  }
  return uint16_t(sign | (he << 10) | (keep & 0x3FFu));
}

double half_value(uint16_t h) {
  const double sign = (h & 0x8000u) ? -1.0 : 1.0;
  const int e = (h >> 10) & 0x1F;
  const int f = h & 0x3FF;
  if (e == 31) return f ? std::nan("") : sign * INFINITY;
  if (e == 0) return sign * std::ldexp(double(f), -24);
  return sign * std::ldexp(double(1024 + f), e - 25);
}

double round_to(double x, int precision) {
  if (precision == kFp64 || x == 0.0 || std::isnan(x)) return x;
  if (precision == kFp16) return half_value(half_bits(x));
  if (std::fabs(x) >= 0x1.ffffffp+127) return std::copysign(INFINITY, x);
  return static_cast<double>(static_cast<float>(x));
}

void effective_operands(const TableEntry& e, int strategy, double* t, double* w, bool* cos) {
  switch (strategy) {
    case kLinzerFeig:
      if (e.clamped) {  // butterfly.cpp:59-63: cosine_core(a, b, omega_i, omega_r)
        *t = e.omega_i;
        *w = e.omega_r;
        *cos = true;
      } else {
        *t = e.ratio;
        *w = e.multiplier;
        *cos = false;
      }
      return;
    case kCosine:
      *t = e.ratio;
      *w = e.multiplier;
      *cos = true;
      return;
    default:  // dual (and the unused standard case)
      *t = e.ratio;
      *w = e.multiplier;
      *cos = e.path == kCos;
      return;
  }
}

Record pack_record(const TableEntry& e, int strategy, int precision, bool f16_complex) {
  double t, w;
  bool cos = true;
  if (strategy != kStandard) effective_operands(e, strategy, &t, &w, &cos);
  if (precision == kFp16 && f16_complex) {
    // one complex per f16x2 register: low half = re lane, high half = im lane
    auto pair = [](double lo, double hi) -> uint32_t {
      return uint32_t(half_bits(lo)) | (uint32_t(half_bits(hi)) << 16);
    };
    if (strategy == kStandard)
      return Record{pair(e.omega_r, e.omega_i), pair(e.omega_i, e.omega_r), 0u, 0u};
    // (-t, t), (w', w), PRMT selectors producing (x, y) and (y, x) from b
    return Record{pair(-t, t), pair(cos ? w : -w, w), cos ? 0x3210u : 0x1032u,
                  cos ? 0x1032u : 0x3210u};
  }
  if (precision == kFp16) {  // transform pairs: compact, halves broadcast on device
    auto pair = [](uint32_t lo, double hi) -> uint32_t {
      return lo | (uint32_t(half_bits(hi)) << 16);
    };
    if (strategy == kStandard) return Record{pair(half_bits(e.omega_r), e.omega_i), 0u, 0u, 0u};
    return Record{pair(half_bits(t), cos ? w : -w), pair(cos ? 0x3210u : 0x7654u, w), 0u, 0u};
  }
  if (strategy == kStandard) return Record{f32_bits(e.omega_r), f32_bits(e.omega_i), 0u, 0u};
  return Record{f32_bits(t), f32_bits(cos ? w : -w), f32_bits(w), cos ? 0x3210u : 0x7654u};
}

int record_bytes(int precision, bool f16_complex) {
  return precision == kFp16 && !f16_complex ? 8 : 16;
}

std::vector<uint8_t> serialize_records(const std::vector<Record>& recs, int rec_bytes) {
  std::vector<uint8_t> out((recs.size() * rec_bytes + 15) & ~size_t(15), 0);
  for (size_t i = 0; i < recs.size(); ++i)
    std::memcpy(out.data() + i * rec_bytes, &recs[i], rec_bytes);
  return out;
}

}  // namespace dsfft
