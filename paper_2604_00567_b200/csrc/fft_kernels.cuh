// fft_kernels.cuh -- the batched single-kernel radix-2 Stockham FFT for sm_100a.
//
// One persistent CTA per SM runs NG independent thread groups; each group owns
// an S-deep ring of item buffers in shared memory.  Per item (K transforms):
//   TMA bulk load (cp.async.bulk, mbarrier complete_tx)  -> smem
//   stage 0: gather 2^s0 values per group into registers, s0 passes in regs
//   exchange through padded smem (conflict-free, tools/schedule_check.cpp)
//   stage 1..: same, the last log2(E) passes entirely in registers
//   the buffer is released to the next TMA load right after the item's last
//   smem read; the last stage stores its natural-order results straight
//   from registers (each warp store covers whole 128-byte lines)
// Loads for the next S items are in flight while an item is computed.
//
// Arithmetic (the parity contract):
//  * FMA strategies (LF, cosine, dual) use the branch-free unified form of
//    cosine_core/sine_core (butterfly.cpp:10-33): the host packs per twiddle
//    (t, w' = COS ? w : -w, w, selector) and the COS/SIN operand swap is one
//    PRMT whose selector comes from the record, so COS and SIN butterflies
//    mix inside a warp without divergence:
//        (x, y) = COS ? (b.re, b.im) : (b.im, b.re)
//        u1 = fma(-t, y, x)   u2 = fma(t, x, y)
//        A = (fma(u1, w', a.re), fma(u2, w, a.im))
//        B = (fma(-u1, w', a.re), fma(-u2, w, a.im))
//    Bit-identical to the reference (sign flips are exact; IEEE fma depends
//    only on the exact product and the addend).
//  * standard (butterfly.cpp:37-53): 4 mul + 6 add/sub, each rounded
//    separately (mul.rn/add.rn/sub.rn, __fmul_rn/__fadd_rn/__fsub_rn).
//  * FP32 (ArithF32): a value is one complex, (re, im) in two registers; FFMA
//    == std::fmaf.
//  * FP16, two layouts; every HFMA2 lane is one correctly rounded binary16
//    FMA == ArithmeticContext::fma at fp16 (precision.cpp:98-111):
//      ArithF16P  a value is the same sample of two transforms,
//                 (re0,re1),(im0,im1): 6 HFMA2 + 2 PRMT per 2 butterflies;
//      ArithF16C  a value is one complex (re,im) in one f16x2 register:
//                 u = fma((-t,t), (y,x), (x,y)); A = fma(u, (w',w), a);
//                 B = fma(u, -(w',w), a): 3 HFMA2 + 2 PRMT per butterfly,
//                 half the registers and buffer bytes per transform.
#pragma once
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "schedule.cuh"

namespace dsfft {

struct KernelParams {
  const uint8_t* in;
  uint8_t* out;
  const uint4* tw;        // per-stage packed twiddle records (global)
  long long n_items;      // items = ceil(batch / transforms_per_item)
  long long batch;        // real transforms
  uint32_t scale;         // inverse: 1/n as f32 bits or f16x2 (s, s)
  int stages;             // S: item buffers per group
};

// ---- arithmetic back ends ---------------------------------------------------
struct F16Ops {
  __device__ __forceinline__ static uint32_t fma(uint32_t a, uint32_t b, uint32_t c) {
    return ptx::hfma2(a, b, c);
  }
  __device__ __forceinline__ static uint32_t neg(uint32_t a) { return ptx::hneg2(a); }
  __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) { return ptx::hadd2(a, b); }
  __device__ __forceinline__ static uint32_t sub(uint32_t a, uint32_t b) { return ptx::hsub2(a, b); }
  __device__ __forceinline__ static uint32_t mul(uint32_t a, uint32_t b) { return ptx::hmul2(a, b); }
};

// FP16, transform pairs: two words per value, two real transforms per
// virtual transform.
// Records are 8 bytes, (t | w' << 16, sel | w << 16), expanded by load_rec.
struct ArithF16P : F16Ops {
  static constexpr int kWords = 2, kPair = 2, kSampleBytes = 4, kRecBytes = 8;
};
// FP16, one complex per register.
struct ArithF16C : F16Ops {
  static constexpr int kWords = 1, kPair = 1, kSampleBytes = 4, kRecBytes = 16;
};

struct ArithF32 {
  static constexpr int kWords = 2, kPair = 1, kSampleBytes = 8, kRecBytes = 16;
  __device__ __forceinline__ static float f(uint32_t a) { return __uint_as_float(a); }
  __device__ __forceinline__ static uint32_t u(float a) { return __float_as_uint(a); }
  __device__ __forceinline__ static uint32_t fma(uint32_t a, uint32_t b, uint32_t c) {
    return u(__fmaf_rn(f(a), f(b), f(c)));
  }
  __device__ __forceinline__ static uint32_t neg(uint32_t a) { return a ^ 0x80000000u; }
  __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) { return u(__fadd_rn(f(a), f(b))); }
  __device__ __forceinline__ static uint32_t sub(uint32_t a, uint32_t b) { return u(__fsub_rn(f(a), f(b))); }
  __device__ __forceinline__ static uint32_t mul(uint32_t a, uint32_t b) { return u(__fmul_rn(f(a), f(b))); }
};

// A twiddle record from shared memory (byte address a) in the 4-word form the
// butterflies use; compact fp16 pair records expand to ((t,t), (w',w'), (w,w),
// sel) -- the broadcasts fold into the HFMA2 operands.
template <class A>
__device__ __forceinline__ uint4 expand_rec(uint32_t x, uint32_t y) {
  return make_uint4(ptx::bcast_lo(x), ptx::bcast_hi(x), ptx::bcast_hi(y), y);
}
template <class A>
__device__ __forceinline__ uint4 load_rec(uint32_t a) {
  if constexpr (A::kRecBytes == 8) {
    uint32_t x, y;
    ptx::lds64(a, x, y);
    return expand_rec<A>(x, y);
  } else {
    return ptx::lds128(a);
  }
}
// Same from global memory (read-only path).
template <class A>
__device__ __forceinline__ uint4 ldg_rec(const uint8_t* p) {
  if constexpr (A::kRecBytes == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    return expand_rec<A>(v.x, v.y);
  } else {
    return __ldg(reinterpret_cast<const uint4*>(p));
  }
}

// Bytes of one stored value (one complex or one transform-pair sample).
template <class A>
__host__ __device__ constexpr int value_bytes() { return A::kWords * 4; }

// CTA size cap (sets the register budget): 2E data registers for two-word
// values (E=32 -> 128 regs, 512 threads; E=16 -> ~80 regs, 768 threads), E for
// one-word values.
template <class Cfg, class A>
__host__ __device__ constexpr int max_threads() {
  return A::kWords == 2 ? (Cfg::LOG_E >= 6 ? 256 : Cfg::LOG_E <= 4 ? 768 : 512)
                        : (Cfg::LOG_E >= 6 ? 512 : 768);
}

// One radix-2 butterfly, A = a + W b, B = a - W b.
//   two-word values: (re, im) registers; one-word: f16x2 (re, im) in `re`.
template <class A, bool STANDARD>
__device__ __forceinline__ void butterfly(uint32_t are, uint32_t aim, uint32_t bre,
                                          uint32_t bim, const uint4& tw, uint32_t& Are,
                                          uint32_t& Aim, uint32_t& Bre, uint32_t& Bim) {
  if constexpr (A::kWords == 1) {
    if constexpr (STANDARD) {
      // record: ((wr, wi), (wi, wr), -, -)
      const uint32_t rr_ii = A::mul(bre, tw.x);  // (wr*br, wi*bi)
      const uint32_t ir_ri = A::mul(bre, tw.y);  // (wi*br, wr*bi)
      const uint32_t p = __byte_perm(rr_ii, ir_ri, 0x5410);  // (rr, ir)
      const uint32_t q = __byte_perm(rr_ii, ir_ri, 0x7632);  // (ii, ri)
      // (rr - ii, ir + ri): fma by -1 / +1 is one exact-product rounding
      const uint32_t t = A::fma(q, 0x3C00BC00u, p);
      Are = A::add(are, t);
      Bre = A::sub(are, t);
    } else {
      // record: ((-t, t), (w', w), sel_xy, sel_yx)
      const uint32_t xy = ptx::prmt(bre, bre, tw.z);
      const uint32_t yx = ptx::prmt(bre, bre, tw.w);
      const uint32_t u = A::fma(tw.x, yx, xy);
      Are = A::fma(u, tw.y, are);
      Bre = A::fma(u, A::neg(tw.y), are);
    }
  } else if constexpr (STANDARD) {
    // record: (omega_r, omega_i, -, -)
    const uint32_t rr = A::mul(tw.x, bre);
    const uint32_t ii = A::mul(tw.y, bim);
    const uint32_t ir = A::mul(tw.y, bre);
    const uint32_t ri = A::mul(tw.x, bim);
    const uint32_t tr = A::sub(rr, ii);
    const uint32_t ti = A::add(ir, ri);
    Are = A::add(are, tr);
    Aim = A::add(aim, ti);
    Bre = A::sub(are, tr);
    Bim = A::sub(aim, ti);
  } else {
    // record: (t, w', w, sel)
    const uint32_t x = ptx::prmt(bre, bim, tw.w);
    const uint32_t y = ptx::prmt(bim, bre, tw.w);
    const uint32_t u1 = A::fma(A::neg(tw.x), y, x);
    const uint32_t u2 = A::fma(tw.x, x, y);
    Are = A::fma(u1, tw.y, are);
    Aim = A::fma(u2, tw.z, aim);
    Bre = A::fma(A::neg(u1), tw.y, are);
    Bim = A::fma(A::neg(u2), tw.z, aim);
  }
}

// All local passes of stage ST on the thread's E values.
template <class Cfg, int ST, class A, bool STANDARD>
__device__ __forceinline__ void run_stage(uint32_t (&re)[Cfg::E], uint32_t (&im)[Cfg::E],
                                          uint32_t tw_base, int t) {
  constexpr int m = Cfg::LOG_N, s = Cfg::s(ST), P = Cfg::P(ST);
  constexpr int E = Cfg::E, NGRP = E >> s, H = 1 << (s - 1);
  constexpr bool kSharedR = (Cfg::T % (1 << P)) == 0;  // r independent of j
  constexpr int RB = A::kRecBytes;
  const uint32_t tws = tw_base + Cfg::tw_off(ST) * RB;
#pragma unroll
  for (int pl = 0; pl < s; ++pl) {
    uint32_t nre[E], nim[E];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl) {
      uint4 tw{};
      if constexpr (kSharedR) tw = load_rec<A>(tws + tw_slot(P, grp_r(m, P, s, t), pl, rl) * RB);
#pragma unroll
      for (int j = 0; j < NGRP; ++j) {
        if constexpr (!kSharedR)
          tw = load_rec<A>(tws + tw_slot(P, grp_r(m, P, s, t + Cfg::T * j), pl, rl) * RB);
#pragma unroll
        for (int q = 0; q < (H >> pl); ++q) {
          const int jl = (q << pl) | rl;
          const int ia = (j << s) + jl, ib = ia + H;
          const int oa = (j << s) + (q << (pl + 1)) + rl, ob = oa + (1 << pl);
          butterfly<A, STANDARD>(re[ia], im[ia], re[ib], im[ib], tw, nre[oa], nim[oa], nre[ob],
                                 nim[ob]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E; ++i) {
      re[i] = nre[i];
      if constexpr (A::kWords == 2) im[i] = nim[i];
    }
  }
}

// Gather stage ST's inputs from the padded exchange layout.
template <class Cfg, int ST, class A>
__device__ __forceinline__ void read_exchange(uint32_t (&re)[Cfg::E], uint32_t (&im)[Cfg::E],
                                              uint32_t buf, int t) {
  constexpr int m = Cfg::LOG_N, s = Cfg::s(ST), P = Cfg::P(ST);
#pragma unroll
  for (int j = 0; j < (Cfg::E >> s); ++j)
#pragma unroll
    for (int c = 0; c < (1 << s); ++c) {
      const uint32_t a = buf + pad_pos(read_pos(m, P, s, t + Cfg::T * j, c)) * value_bytes<A>();
      if constexpr (A::kWords == 2)
        ptx::lds64(a, re[(j << s) + c], im[(j << s) + c]);
      else
        re[(j << s) + c] = ptx::lds32(a);
    }
}

// Scatter stage ST's outputs into the padded exchange layout.
template <class Cfg, int ST, class A>
__device__ __forceinline__ void write_exchange(const uint32_t (&re)[Cfg::E],
                                               const uint32_t (&im)[Cfg::E], uint32_t buf,
                                               int t) {
  constexpr int m = Cfg::LOG_N, s = Cfg::s(ST), P = Cfg::P(ST);
#pragma unroll
  for (int j = 0; j < (Cfg::E >> s); ++j)
#pragma unroll
    for (int c = 0; c < (1 << s); ++c) {
      const uint32_t a = buf + pad_pos(write_pos(m, P, s, t + Cfg::T * j, c)) * value_bytes<A>();
      if constexpr (A::kWords == 2)
        ptx::sts64(a, re[(j << s) + c], im[(j << s) + c]);
      else
        ptx::sts32(a, re[(j << s) + c]);
    }
}

template <class Cfg>
__device__ __forceinline__ void group_sync(int gid) {
  if constexpr (Cfg::W == 1) {
    __syncwarp();
  } else {
    ptx::named_bar_sync(1 + gid, Cfg::T);
  }
}

template <class Cfg, int ST, class A, bool STANDARD, class Release>
__device__ __forceinline__ void later_stages(uint32_t (&re)[Cfg::E], uint32_t (&im)[Cfg::E],
                                             uint32_t buf, uint32_t tw_base, int t, int gid,
                                             Release& release) {
  if constexpr (ST < Cfg::NSTAGE) {
    group_sync<Cfg>(gid);  // every read of the previous layout is done
    write_exchange<Cfg, ST - 1, A>(re, im, buf, t);
    group_sync<Cfg>(gid);
    read_exchange<Cfg, ST, A>(re, im, buf, t);
    if constexpr (ST == Cfg::NSTAGE - 1) release();  // last smem read of this item
    run_stage<Cfg, ST, A, STANDARD>(re, im, tw_base, t);
    later_stages<Cfg, ST + 1, A, STANDARD>(re, im, buf, tw_base, t, gid, release);
  }
}

// Transform one item resident in smem (natural order in) and write it to
// global memory in natural order straight from registers.  `release()` runs
// as soon as the item's last shared-memory read is done, so the buffer is
// refilled by TMA while the last stage computes.  `valid` = real transforms
// of this item that exist (the batch tail).
template <class Cfg, class A, bool STANDARD, bool INVERSE, class Release>
__device__ __forceinline__ void transform_item(uint32_t buf, uint32_t tw_base, int t, int gid,
                                               uint32_t scale, uint8_t* gout, int valid,
                                               Release& release) {
  constexpr int m = Cfg::LOG_N, N = Cfg::N, E = Cfg::E;
  constexpr int s0 = Cfg::s(0), L = Cfg::NSTAGE - 1, sL = Cfg::s(L), PL = Cfg::P(L);
  uint32_t re[E], im[E];
  // ---- stage 0 gather from the natural (identity) layout -------------------
#pragma unroll
  for (int j = 0; j < (E >> s0); ++j)
#pragma unroll
    for (int c = 0; c < (1 << s0); ++c) {
      const int pos = read_pos(m, 0, s0, t + Cfg::T * j, c);
      const int v = (j << s0) + c;
      if constexpr (A::kPair == 2) {
        const int k = pos >> m, p = pos & (N - 1);
        const uint32_t lo = ptx::lds32(buf + ((2 * k) * N + p) * 4);
        const uint32_t hi = ptx::lds32(buf + ((2 * k + 1) * N + p) * 4);
        re[v] = __byte_perm(lo, hi, 0x5410);
        im[v] = __byte_perm(lo, hi, 0x7632);
        if constexpr (INVERSE) im[v] = A::neg(im[v]);  // conj on load (fft.cpp:90-91)
      } else if constexpr (A::kWords == 2) {
        ptx::lds64(buf + pos * 8, re[v], im[v]);
        if constexpr (INVERSE) im[v] = A::neg(im[v]);
      } else {
        re[v] = ptx::lds32(buf + pos * 4);
        if constexpr (INVERSE) re[v] ^= 0x80000000u;  // negate the im half only
      }
    }
  if constexpr (Cfg::NSTAGE == 1) release();
  run_stage<Cfg, 0, A, STANDARD>(re, im, tw_base, t);
  later_stages<Cfg, 1, A, STANDARD>(re, im, buf, tw_base, t, gid, release);
  // ---- last stage: natural-order stores from registers (coalesced) ---------
#pragma unroll
  for (int j = 0; j < (E >> sL); ++j)
#pragma unroll
    for (int c = 0; c < (1 << sL); ++c) {
      const int pos = write_pos(m, PL, sL, t + Cfg::T * j, c);
      const int v = (j << sL) + c;
      const int k = pos >> m, p = pos & (N - 1);
      if constexpr (A::kWords == 1) {
        uint32_t x = re[v];
        if constexpr (INVERSE)  // (re*s, (-im)*s), one rounded mul each (fft.cpp:94-98)
          x = A::mul(x ^ 0x80000000u, scale);
        if (k < valid) __stcs(reinterpret_cast<unsigned int*>(gout + size_t(pos) * 4), x);
      } else {
        uint32_t xr = re[v], xi = im[v];
        if constexpr (INVERSE) {  // conj + scale, one rounded mul each (fft.cpp:94-98)
          xr = A::mul(xr, scale);
          xi = A::mul(A::neg(xi), scale);
        }
        if constexpr (A::kPair == 2) {
          if (2 * k < valid)
            __stcs(reinterpret_cast<unsigned int*>(gout + (size_t(2 * k) * N + p) * 4),
                   __byte_perm(xr, xi, 0x5410));
          if (2 * k + 1 < valid)
            __stcs(reinterpret_cast<unsigned int*>(gout + (size_t(2 * k + 1) * N + p) * 4),
                   __byte_perm(xr, xi, 0x7632));
        } else {
          if (k < valid)
            __stcs(reinterpret_cast<uint2*>(gout + size_t(pos) * 8), make_uint2(xr, xi));
        }
      }
    }
}

template <class Cfg, class A>
struct SmallLayout {
  static constexpr int kBufBytes = Cfg::BUF_VALS * value_bytes<A>();
  static constexpr int kItemBytes = Cfg::VALS * value_bytes<A>();
  static constexpr int kTwBytes = (Cfg::TW_RECORDS * A::kRecBytes + 127) & ~127;
  static constexpr int kTpi = Cfg::K * A::kPair;            // real transforms per item
  static constexpr int kTb = Cfg::N * A::kSampleBytes;      // bytes per transform
  static size_t smem_bytes(int groups, int stages) {
    return size_t(kTwBytes) + size_t(groups) * stages * kBufBytes + size_t(groups) * stages * 8;
  }
};

// Persistent batched FFT over items.  blockDim = NG * T threads.
template <class Cfg, class A, bool STANDARD, bool INVERSE>
__global__ void __launch_bounds__(max_threads<Cfg, A>(), 1) fft_small_kernel(const KernelParams p) {
  using Lay = SmallLayout<Cfg, A>;
  extern __shared__ __align__(128) uint8_t smem[];
  const int ng = blockDim.x / Cfg::T;
  const int gid = threadIdx.x / Cfg::T;
  const int t = threadIdx.x % Cfg::T;
  const int S = p.stages;
  const uint32_t tw_base = ptx::smem_u32(smem);
  uint8_t* bufs = smem + Lay::kTwBytes + size_t(gid) * S * Lay::kBufBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::kTwBytes +
                                               size_t(ng) * S * Lay::kBufBytes) +
                   gid * S;
  // twiddle records -> smem (once per persistent CTA)
  for (int i = threadIdx.x; i < (Cfg::TW_RECORDS * A::kRecBytes + 15) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = p.tw[i];
  if (t == 0)
    for (int b = 0; b < S; ++b) ptx::mbar_init(&bars[b], 1);
  ptx::fence_mbar_init();
  __syncthreads();

  constexpr long long kTpi = Lay::kTpi;
  constexpr long long kTb = Lay::kTb;
  const long long first = (long long)blockIdx.x * ng + gid;
  const long long stride = (long long)gridDim.x * ng;
  const bool leader = (t == 0);
  uint64_t pol = 0;
  if (leader) pol = ptx::policy_evict_first();
  auto issue_load = [&](long long item, int b) {
    const long long left = p.batch - item * kTpi;
    const uint32_t bytes = uint32_t((left < kTpi ? left : kTpi) * kTb);
    ptx::mbar_arrive_expect_tx(&bars[b], bytes);
    ptx::bulk_g2s(bufs + size_t(b) * Lay::kBufBytes, p.in + item * Lay::kItemBytes, bytes,
                  &bars[b], pol);
  };
  if (leader)
    for (int b = 0; b < S; ++b) {
      const long long item = first + b * stride;
      if (item < p.n_items) issue_load(item, b);
    }
  int it = 0;
  for (long long item = first; item < p.n_items; item += stride, ++it) {
    const int b = it % S;
    ptx::mbar_wait(&bars[b], (it / S) & 1);
    uint8_t* bp = bufs + size_t(b) * Lay::kBufBytes;
    const long long left = p.batch - item * kTpi;
    const int valid = int(left < kTpi ? left : kTpi);
    auto release = [&]() {
      // all generic-proxy accesses of buffer b precede the next TMA write
      ptx::fence_proxy_async_smem();
      group_sync<Cfg>(gid);
      const long long nxt = item + (long long)S * stride;
      if (leader && nxt < p.n_items) issue_load(nxt, b);
    };
    transform_item<Cfg, A, STANDARD, INVERSE>(ptx::smem_u32(bp), tw_base, t, gid, p.scale,
                                              p.out + item * Lay::kItemBytes, valid, release);
  }
}

}  // namespace dsfft
