// multipass_impl.cuh -- internals shared by the large-N translation units:
// multipass.cu (pass groups as two or three launches over HBM intermediates)
// and multipass_fused.cu (both groups in one launch, L2-resident
// intermediate).  Twiddle-record layouts (host and device agree), the tile
// body both kernels run, the plan, and the host helpers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "fft_kernels.cuh"
#include "multipass.cuh"

namespace dsfft {

// ---- twiddle table layouts (host and device agree) ---------------------------
// first group (P = 0, twiddles independent of the column):
//   [0, 31)                      stage 1, slot1 = 2^pl - 1 + rl
//   31 + slot2*32 + r_l          stage 2, slot2 = 2^pl - 1 + rl, r_l < 32
// later groups, per block of 32 columns (rb = r / 32), base rb * mp_block:
//   slot1*32 + lane                          stage 1
//   31*32 + (slot2*32 + r_l)*32 + lane       stage 2
__host__ __device__ constexpr int mp_first_records(int S1) { return 31 + (((1 << S1) - 1) << 5); }
__host__ __device__ constexpr int mp_block_records(int S1) {
  return 31 * 32 + (((1 << S1) - 1) << 10);
}

// CW: columns per tile (32, or 16 -- narrower tiles, twice the tile groups
// per SM, same full-sector rows for 8-byte values).
template <int S1, class A, int CW = 32>
struct MpLayout {
  static constexpr int s = 5 + S1, L = 1 << s, T = CW << S1;
  static constexpr int VB = A::kWords * 4;
  // exchange layout [col][local pos]: column stride L + 1 values; 8-column
  // tiles (four row phases per warp) pad one value per 32 and use a column
  // stride = 2 mod 16 values: a 64-bit access is served per half-warp (8
  // columns x 2 row phases), whose 16 values then hit 16 distinct bank pairs
  static constexpr bool kPadX = CW == 8;
  static constexpr int kColStride = kPadX ? ((L + L / 32 + 13) / 16) * 16 + 2 : L + 1;
  __host__ __device__ static constexpr int xpos(int c, int pos) {
    return c * kColStride + (kPadX ? pos + (pos >> 5) : pos);
  }
  static constexpr int kBufBytes = CW * kColStride * VB;  // padded exchange >= TMA tile
  static constexpr int kTileBytes = CW * L * VB;
  // twiddle area rounded to 128 B: TMA tensor destinations are 128-B aligned.
  // Later groups keep their column block's whole twiddle slab in smem (stage 1
  // and 2) when it is at most 64 KB (8-byte fp16 pair records up to S1 = 3,
  // 16-byte records up to S1 = 2); otherwise only the stage-1 part, and stage
  // 2 reads its records through L1 (ldg).  A 130 KB fp32 slab would leave room
  // for one 256-thread tile group per SM.
  static constexpr bool kFullSlab = S1 <= 3 && mp_block_records(S1) * A::kRecBytes <= 65536;
  static constexpr int kSlabRecords = kFullSlab ? mp_block_records(S1) : 31 * 32;
  __host__ __device__ static constexpr int tw_bytes(bool first) {
    return ((first ? mp_first_records(S1) : kSlabRecords) * A::kRecBytes + 127) & ~127;
  }
  static size_t smem_bytes(bool first, int stages, int groups) {
    const int tw = tw_bytes(first);
    return size_t(tw) + size_t(groups) * stages * (kBufBytes + 8);
  }
};

// One tile: column block (q, rb) of one transform (pair) from smem slot
// c.buf.  release() hands the slot back to TMA after its last smem read;
// pre_store() runs right before the scatter (the fused kernel waits there
// until the scratch slot it writes is free).
//
// Threads: `sub` = warp * (32 / CW) + lane / CW takes rows sub + 2^S1 c of
// column `col` = lane % CW in stage 1.  Stage 2 groups (column, r_l): first
// group -- lanes walk r_l (column-contiguous output), columns warp + NW j;
// later groups -- lanes walk columns, r_l = sub + 2^S1 j.  col_off places a
// 16-column tile inside its 32-column block (twiddle slab, output columns).
template <int S1, class A, bool STANDARD, bool FIRST, bool CONJ_IN, bool SCALE_OUT, bool LAST,
          bool BOUT, int CW = 32, class Out, class Release, class PreStore>
__device__ __forceinline__ void mp_tile(uint32_t buf, uint32_t tw_base, const uint8_t* tw_g,
                                        uint32_t scale, int P, long long N, long long q, int rb,
                                        int col_off, bool second, int g, int warp, int lane,
                                        Out&& out, Release&& release, PreStore&& pre_store) {
  using Lay = MpLayout<S1, A, CW>;
  constexpr int L = Lay::L, T = Lay::T, NG2 = 32 >> S1, VB = Lay::VB;
  constexpr int NW = T / 32;           // warps per group
  constexpr int NSUB = 32 / CW;        // row phases per warp
  const int sub = warp * NSUB + (NSUB == 1 ? 0 : lane / CW);
  const int col = lane % CW, col32 = col_off + col;
  constexpr int RB = A::kRecBytes;
  constexpr int PAIR = A::kPair;
  constexpr int EB = A::kSampleBytes;  // bytes of one complex in memory
  constexpr int HALF = CW * L * EB;    // one transform's tile
  constexpr bool PIN = PAIR == 2 && !FIRST, POUT = PAIR == 2 && !LAST;
  constexpr int OEB = POUT ? 8 : EB;   // bytes per stored output element
  auto group_sync = [&]() {
    if (T == 32) __syncwarp(); else ptx::named_bar_sync(1 + g, T);
  };
  uint32_t re[32], im[32];
  // ---- stage 1: rows sub + c*2^S1 of column `col` (tile is [row][CW]) ----
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) {
    [[maybe_unused]] const uint32_t a = buf + ((sub + (cc << S1)) * CW + col) * VB;
    if constexpr (PAIR == 2 && !PIN) {  // (re0,re1), (im0,im1) from the two halves
      const uint32_t e = buf + ((sub + (cc << S1)) * CW + col) * EB;
      const uint32_t lo = ptx::lds32(e), hi = ptx::lds32(e + HALF);
      re[cc] = __byte_perm(lo, hi, 0x5410);
      im[cc] = __byte_perm(lo, hi, 0x7632);
      if constexpr (CONJ_IN) im[cc] = A::neg(im[cc]);  // conj on load (fft.cpp:90-91)
    } else if constexpr (A::kWords == 1) {
      re[cc] = ptx::lds32(a);
      if constexpr (CONJ_IN) re[cc] ^= 0x80000000u;  // conj on load (fft.cpp:90-91)
    } else {
      ptx::lds64(a, re[cc], im[cc]);
      if constexpr (CONJ_IN) im[cc] = A::neg(im[cc]);
    }
  }
#pragma unroll
  for (int pl = 0; pl < 5; ++pl) {
    uint32_t nre[32], nim[32];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl) {
      const int slot1 = (1 << pl) - 1 + rl;
      const uint4 tw = FIRST ? load_rec<A>(tw_base + slot1 * RB)
                             : load_rec<A>(tw_base + (slot1 * 32 + col32) * RB);
#pragma unroll
      for (int qq = 0; qq < (16 >> pl); ++qq) {
        const int jl = (qq << pl) | rl;
        const int oa = (qq << (pl + 1)) + rl;
        butterfly<A, STANDARD>(re[jl], im[jl], re[jl + 16], im[jl + 16], tw, nre[oa],
                               nim[oa], nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
      }
    }
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      re[x] = nre[x];
      if constexpr (A::kWords == 2) im[x] = nim[x];
    }
  }
  // ---- exchange through the padded slot: [col][local pos] ---------------
  group_sync();  // every stage-1 read of the TMA tile is done
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) {
    const uint32_t a = buf + Lay::xpos(col, sub * 32 + cc) * VB;
    if constexpr (A::kWords == 1) ptx::sts32(a, re[cc]); else ptx::sts64(a, re[cc], im[cc]);
  }
  group_sync();
  // stage 2 groups (column, r_l): first group lanes walk r_l (contiguous
  // column output), later groups lanes walk columns (contiguous rows)
#pragma unroll
  for (int j = 0; j < NG2; ++j) {
    const int col2 = FIRST ? warp + NW * j : col;
    const int rl_ = FIRST ? lane : sub + (j << S1);
#pragma unroll
    for (int cc = 0; cc < (1 << S1); ++cc) {
      const uint32_t a = buf + Lay::xpos(col2, rl_ + 32 * cc) * VB;
      const int v = (j << S1) + cc;
      if constexpr (A::kWords == 1) re[v] = ptx::lds32(a); else ptx::lds64(a, re[v], im[v]);
    }
  }
  // release the slot to this group's tile S ahead
  ptx::fence_proxy_async_smem();
  group_sync();
  release();
  // ---- stage 2 ----------------------------------------------------------
  [[maybe_unused]] const uint8_t* tw2 =
      FIRST ? nullptr
            : tw_g + ((long long)rb * mp_block_records(S1) + 31 * 32 + sub * 32 + col32) * RB;
#pragma unroll
  for (int pl = 0; pl < S1; ++pl) {
    uint32_t nre[32], nim[32];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl)
#pragma unroll
      for (int j = 0; j < NG2; ++j) {
        const int slot2 = (1 << pl) - 1 + rl;
        uint4 tw;
        if constexpr (FIRST)
          tw = load_rec<A>(tw_base + (31 + (slot2 << 5) + lane) * RB);
        else if constexpr (Lay::kFullSlab)  // record (slot2*32 + r_l)*32 + column
          tw = load_rec<A>(tw_base + (31 * 32 + (sub << 5) + col32 +
                                      (((slot2 << 5) + (j << S1)) << 5)) * RB);
        else  // r_l = sub + 2^S1 j
          tw = ldg_rec<A>(tw2 + ((slot2 << 5) + (j << S1)) * 32 * RB);
#pragma unroll
        for (int qq = 0; qq < ((1 << (S1 - 1)) >> pl); ++qq) {
          const int jl = (qq << pl) | rl;
          const int ia = (j << S1) + jl, ib = ia + (1 << (S1 - 1));
          const int oa = (j << S1) + (qq << (pl + 1)) + rl;
          butterfly<A, STANDARD>(re[ia], im[ia], re[ib], im[ib], tw, nre[oa], nim[oa],
                                 nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
        }
      }
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      re[x] = nre[x];
      if constexpr (A::kWords == 2) im[x] = nim[x];
    }
  }
  // ---- scatter ------------------------------------------------------------
  // Stockham order: q*2^(P+s) + r + 2^P*(r_l + 32 c').  BOUT (the group
  // feeding the last one) writes the blocked intermediate instead:
  //   Z[(r' >> 5) * 2^s3 + c][r' & 31],  r' = r + 2^P c', c = q,
  // so each last-group tile (32 columns r' x 2^s3 rows c) is one contiguous
  // block.  Element offsets in units of one stored complex (EB bytes).
  pre_store();
  uint8_t* gout = out();  // this transform (pair) in the group's output
  [[maybe_unused]] const long long S3 = N >> (P + Lay::s);  // rows of the last group (BOUT)
  uint8_t* base;
  long long jstride, cstride;  // bytes between groups j and rows c'
  if constexpr (FIRST && BOUT) {  // r' = lane + 32 c, c-index = column q CW + warp + NW j
    base = gout + ((q * CW + warp) * 32 + lane) * OEB;
    jstride = 32LL * NW * OEB;
    cstride = S3 * 32 * OEB;
  } else if constexpr (FIRST) {  // column-contiguous: ((q CW + col) L + r_l + 32 c')
    base = gout + ((q * CW + warp) * L + lane) * OEB;
    jstride = (long long)L * NW * OEB;
    cstride = 32 * OEB;
  } else if constexpr (BOUT) {  // r' = rb*32 + col32 + 2^P (sub + 2^S1 j + 32 c)
    base = gout + (((rb + ((long long)sub << (P - 5))) * S3 + q) * 32 + col32) * OEB;
    jstride = ((S3 * 32 * OEB) << (P - 5)) << S1;
    cstride = ((S3 * 32 * OEB) << (P - 5)) * 32;
  } else {
    base = gout + ((q << (P + Lay::s)) + rb * 32 + col32 + ((long long)sub << P)) * OEB;
    jstride = ((long long)OEB << P) << S1;
    cstride = ((long long)OEB << P) * 32;
  }
#pragma unroll
  for (int j = 0; j < NG2; ++j)
#pragma unroll
    for (int cc = 0; cc < (1 << S1); ++cc) {
      const int v = (j << S1) + cc;
      uint32_t xr = re[v];
      [[maybe_unused]] uint32_t xi = im[v];
      if constexpr (SCALE_OUT) {  // conj + 1/n, one rounded mul each (fft.cpp:94-98)
        if constexpr (A::kWords == 1) {
          xr = A::mul(xr ^ 0x80000000u, scale);
        } else {
          xr = A::mul(xr, scale);
          xi = A::mul(A::neg(xi), scale);
        }
      }
      uint8_t* dst = base + j * jstride + cc * cstride;
      if constexpr (POUT) {  // pair-packed intermediate
        __stcg(reinterpret_cast<uint2*>(dst), make_uint2(xr, xi));
      } else if constexpr (PAIR == 2) {  // unpack to transforms b and b+1
        unsigned int* d0 = reinterpret_cast<unsigned int*>(dst);
        unsigned int* d1 = reinterpret_cast<unsigned int*>(dst + N * EB);
        const uint32_t t0 = __byte_perm(xr, xi, 0x5410), t1 = __byte_perm(xr, xi, 0x7632);
        if constexpr (LAST) {
          __stcs(d0, t0);
          if (second) __stcs(d1, t1);
        } else {
          __stcg(d0, t0);
          if (second) __stcg(d1, t1);
        }
      } else if constexpr (A::kWords == 1) {
        if constexpr (LAST) __stcs(reinterpret_cast<unsigned int*>(dst), xr);
        else __stcg(reinterpret_cast<unsigned int*>(dst), xr);
      } else {
        if constexpr (LAST) __stcs(reinterpret_cast<uint2*>(dst), make_uint2(xr, xi));
        else __stcg(reinterpret_cast<uint2*>(dst), make_uint2(xr, xi));
      }
    }
}

// ---- plan and host helpers -----------------------------------------------------

struct MpGroup {
  int P, s;
  uint4* d_tw = nullptr;
};

struct MultipassPlan {
  int m = 0, strategy = 0, precision = 0, sm_count = 0;
  bool f16_pairs = true;  // fp16 value layout: transform pairs (else one complex/register)
  bool fused = false;     // both pass groups in one launch (mp_fused_kernel)
  size_t smem_optin = 0;
  std::vector<MpGroup> groups;
  size_t chunk_transforms = 0;
  ~MultipassPlan() {
    for (auto& g : groups)
      if (g.d_tw) cudaFree(g.d_tw);
  }
};

void set_mp_error(const std::string& msg);
// integer environment knob (tuning; documented in tools/gpu_tune.sh)
int env_or(const char* name, int dflt);
// TMA map over `batch` transforms at `base` for pass group [P, P+s) (see multipass.cu)
int make_in_map(CUtensorMap* map, const void* base, int m, int P, int s, int vb,
                long long batch, int box_cols = 32);
// one-launch execution of an eligible plan (multipass_fused.cu); returns
// kFusedUnfit, with nothing launched, when the device cannot hold one team
// co-resident (few SMs, small shared memory): the caller runs the same pass
// groups as two launches
constexpr int kFusedUnfit = 2;
int fused_execute(MultipassPlan& mp, bool inverse, const void* in, void* out, size_t batch,
                  uint32_t scale, cudaStream_t stream, uint64_t* launches);

}  // namespace dsfft
