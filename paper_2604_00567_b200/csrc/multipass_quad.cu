// multipass_quad.cu -- the one-launch N = 2^16 (s = 8 + 8) path with
// warp-independent tiles.
//
// mp_fused_kernel runs each 32-column x 256-row tile on an 8-warp group: the
// stage-1 / stage-2 exchange is a transpose across the 8 warps, so every tile
// costs three named barriers and the group moves in lock step (SM-latency
// bound: 44% FMA pipe, profiles/r02_fused_multipass.md).  Here a tile is split
// by COLUMNS instead: warp w owns a quad of 4 columns (all 256 rows), i.e. the
// whole length-256 column FFTs of its quad, and needs no other warp.
//   * lanes: c4 = lane & 3 (column in the quad), sub = lane >> 2; stage 1 takes
//     rows sub + 8 i (i < 32) of column c4 -- the same 32-point sub-FFT the
//     8-warp tile gives warp `sub` -- and runs passes 0..4 in registers;
//   * exchange in the warp's private 8 KB slot: output c of lane (c4, sub) is
//     stored at row 8 c + (sub ^ (c & 7)) (32-byte rows: 4 columns x 8 B), so
//     both the stores and the stage-2 loads -- group (column c4, r_l = sub + 8 t)
//     reads rows 8 r_l + (cc ^ sub) -- hit every bank exactly twice (the
//     2-wavefront minimum for 256 B); only __syncwarp in between;
//   * stage 2 runs passes 5..7 on 4 groups of 8 values per lane.
// Every warp has its own slot, filled by cp.async (16 B per lane-op; 32-byte
// row segments of the blocked intermediate, 16-byte halves of the user
// rows -- neighbour quads share the 32-byte sectors through L2), issued as
// soon as the warp's stage-2 loads are done.  So each of the 16 warps of an SM
// is an independent pipeline, like the single-kernel path's one-warp groups.
//
// The team / scratch-ring / counter protocol is mp_fused_kernel's (see
// multipass_fused.cu), at quad granularity: a unit is complete when all 8 K
// first-group quads are published, and its slot is free when all 8 K
// second-group quads have landed.  Second-group twiddles use a quad-ordered
// slab (quad_slab_index) so the 32 lanes of a stage-2 record load read 32
// consecutive records.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "host_table.hpp"
#include "multipass_impl.cuh"

namespace dsfft {

namespace {

constexpr int kQS1 = 3;                      // s = 8: 5 + 3 passes
constexpr int kQL = 256;                     // rows of a tile
constexpr int kQSlot = kQL * 4 * 8;          // 8 KB: 256 rows x 4 columns x 8-byte values
constexpr int kQWarps = 16;                  // warps per CTA (two unit streams of 8 quads)

// second-group stage-2 record (slot2, r_l, col) of a column block:
//   31*32 + ((slot2*4 + r_l/8)*8 + col/4)*32 + (col%4)*8 + r_l%8
__host__ __device__ constexpr int quad_slab_index(int slot2, int r_l, int col) {
  return 31 * 32 + (((slot2 * 4 + (r_l >> 3)) * 8 + (col >> 2)) << 5) + ((col & 3) << 3) +
         (r_l & 7);
}

template <class A>
struct QuadLayout {
  static constexpr int RB = A::kRecBytes;
  // 8-byte records (fp16 pairs): the whole 65 KB slab in smem; 16-byte (fp32):
  // stage 1 in smem, stage 2 through L1
  static constexpr bool kFullSlab = RB == 8;
  static constexpr int kTwA = (mp_first_records(kQS1) * RB + 127) & ~127;
  static constexpr int kTwB = ((kFullSlab ? mp_block_records(kQS1) : 31 * 32) * RB + 127) & ~127;
  static constexpr size_t kSmem = size_t(kTwA) + kTwB + size_t(kQWarps) * kQSlot;
};

// One quad tile, already in this warp's slot.  FIRST: the first pass group
// (user rows in, blocked pair-packed intermediate out); else the second group
// (blocked intermediate in, natural order out).  All addresses are a per-lane
// base plus compile-time offsets.
template <class A, bool STANDARD, bool INVERSE, bool FIRST, class Release, class PreStore>
__device__ __forceinline__ void quad_tile(uint32_t slot_s, uint32_t twA, uint32_t twB,
                                          const uint8_t* slab_g, uint8_t* obase,
                                          long long second_off, bool second, uint32_t scale,
                                          int quad, int lane, Release&& release,
                                          PreStore&& pre_store) {
  using Lay = QuadLayout<A>;
  constexpr int RB = A::kRecBytes, PAIR = A::kPair;
  const int c4 = lane & 3, sub = lane >> 2, col = quad * 4 + c4;
  uint32_t re[32], im[32];
  // ---- stage 1: rows sub + 8 i of column c4 ---------------------------------
  {
    const uint32_t a16 = slot_s + sub * 16 + c4 * 4;  // user halves: 16-byte rows
    const uint32_t a32 = slot_s + sub * 32 + c4 * 8;  // 8-byte values: 32-byte rows
#pragma unroll
    for (int ii = 0; ii < 32; ++ii) {
      if constexpr (FIRST && PAIR == 2) {
        const uint32_t lo = ptx::lds32(a16 + ii * 128);
        const uint32_t hi = ptx::lds32(a16 + 4096 + ii * 128);
        re[ii] = __byte_perm(lo, hi, 0x5410);
        im[ii] = __byte_perm(lo, hi, 0x7632);
      } else {
        ptx::lds64(a32 + ii * 256, re[ii], im[ii]);
      }
      if constexpr (FIRST && INVERSE) im[ii] = A::neg(im[ii]);  // conj on load (fft.cpp:90-91)
    }
  }
#pragma unroll
  for (int pl = 0; pl < 5; ++pl) {
    uint32_t nre[32], nim[32];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl) {
      const int slot1 = (1 << pl) - 1 + rl;
      const uint4 tw = FIRST ? load_rec<A>(twA + slot1 * RB)
                             : load_rec<A>(twB + (slot1 * 32 + col) * RB);
#pragma unroll
      for (int qq = 0; qq < (16 >> pl); ++qq) {
        const int jl = (qq << pl) | rl;
        const int oa = (qq << (pl + 1)) + rl;
        butterfly<A, STANDARD>(re[jl], im[jl], re[jl + 16], im[jl + 16], tw, nre[oa], nim[oa],
                               nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
      }
    }
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      re[x] = nre[x];
      im[x] = nim[x];
    }
  }
  // ---- exchange in the private slot: output c of lane (c4, sub) -> row
  // 8 c + (sub ^ (c & 7)); stage 2 reads group (c4, r_l = sub + 8 t), value cc
  // from row 8 r_l + (cc ^ sub)
  __syncwarp();  // every lane's stage-1 loads are done
  {
    const uint32_t base = slot_s + c4 * 8;
#pragma unroll
    for (int c7 = 0; c7 < 8; ++c7) {
      const uint32_t a = base + (sub ^ c7) * 32;
#pragma unroll
      for (int hi = 0; hi < 4; ++hi) {
        const int cc = hi * 8 + c7;
        ptx::sts64(a + cc * 256, re[cc], im[cc]);
      }
    }
  }
  __syncwarp();
  {
    const uint32_t base = slot_s + sub * 256 + c4 * 8;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const uint32_t a = base + (cc ^ sub) * 32;
#pragma unroll
      for (int t = 0; t < 4; ++t) ptx::lds64(a + t * 2048, re[(t << 3) + cc], im[(t << 3) + cc]);
    }
  }
  __syncwarp();
  release();  // the slot is free: the next tile's copies go out now
  // ---- stage 2: groups (column c4, r_l = sub + 8 t), 8 values each -----------
#pragma unroll
  for (int pl = 0; pl < kQS1; ++pl) {
    uint32_t nre[32], nim[32];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int slot2 = (1 << pl) - 1 + rl;
        const int r_l = sub + 8 * t;
        uint4 tw;
        if constexpr (FIRST)
          tw = load_rec<A>(twA + (31 + (slot2 << 5) + r_l) * RB);
        else if constexpr (Lay::kFullSlab)
          tw = load_rec<A>(twB + quad_slab_index(slot2, r_l, col) * RB);
        else
          tw = ldg_rec<A>(slab_g + quad_slab_index(slot2, r_l, col) * RB);
#pragma unroll
        for (int qq = 0; qq < ((1 << (kQS1 - 1)) >> pl); ++qq) {
          const int jl = (qq << pl) | rl;
          const int ia = (t << kQS1) + jl, ib = ia + (1 << (kQS1 - 1));
          const int oa = (t << kQS1) + (qq << (pl + 1)) + rl;
          butterfly<A, STANDARD>(re[ia], im[ia], re[ib], im[ib], tw, nre[oa], nim[oa],
                                 nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
        }
      }
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      re[x] = nre[x];
      im[x] = nim[x];
    }
  }
  // ---- stores ----------------------------------------------------------------
  pre_store();
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      uint32_t xr = re[(t << 3) + cc], xi = im[(t << 3) + cc];
      if constexpr (FIRST) {
        // value cc of group (q_col, r_l) -> second-group block cc, row q_col,
        // column r_l: obase = unit + ((32 j + col) * 32 + sub) * 8
        __stcg(reinterpret_cast<uint2*>(obase + cc * (kQL * 32 * 8) + t * 64),
               make_uint2(xr, xi));
      } else {
        // natural position 32 j + col + 2^8 (r_l + 32 cc):
        // obase = out + (b N + 32 j + col + 2^8 sub) * EB
        constexpr int EB = A::kSampleBytes;
        uint8_t* dst = obase + ((t * 8 + cc * 32) << 8) * EB;
        if constexpr (INVERSE) {  // conj + 1/n, one rounded mul each (fft.cpp:94-98)
          xr = A::mul(xr, scale);
          xi = A::mul(A::neg(xi), scale);
        }
        if constexpr (PAIR == 2) {
          __stcs(reinterpret_cast<unsigned int*>(dst), __byte_perm(xr, xi, 0x5410));
          if (second)
            __stcs(reinterpret_cast<unsigned int*>(dst + second_off),
                   __byte_perm(xr, xi, 0x7632));
        } else {
          __stcs(reinterpret_cast<uint2*>(dst), make_uint2(xr, xi));
        }
      }
    }
}

template <class A, bool STANDARD, bool INVERSE>
__global__ void __launch_bounds__(kQWarps * 32, 1) mp_quad_kernel(const FusedParams p) {
  using Lay = QuadLayout<A>;
  constexpr int RB = A::kRecBytes, PAIR = A::kPair, EB = A::kSampleBytes;
  constexpr long long kUnitScale = PAIR * EB;  // bytes per sample of a unit (8)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t ctr[2][2][16];  // [stream][A stored / B landed][slot]: quads of this member
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = w & 7, par = w >> 3;  // column quad of the block, unit stream
  const int c4 = lane & 3, sub = lane >> 2;
  const int K = p.K, R = p.R, D = p.D;
  const int tau = blockIdx.x / K, j = blockIdx.x - (blockIdx.x / K) * K;
  const long long N = 1LL << p.m;
  const long long NS = N >> 8;  // first-group row stride in samples (N / 2^s)
  const uint32_t twA = ptx::smem_u32(smem), twB = twA + Lay::kTwA;
  const uint32_t slot_s = twB + Lay::kTwB + uint32_t(w) * kQSlot;
  const int col = quad * 4 + c4;
  {  // both groups' twiddles, once per launch (member j = column block j)
    uint4* sa = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < (mp_first_records(kQS1) * RB + 15) / 16; i += blockDim.x)
      sa[i] = p.twA[i];
    const uint4* src = p.twB + (long long)j * mp_block_records(kQS1) * RB / 16;
    uint4* sb = reinterpret_cast<uint4*>(smem + Lay::kTwA);
    const int n16 = (Lay::kFullSlab ? mp_block_records(kQS1) : 31 * 32) * RB / 16;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) sb[i] = src[i];
    for (int i = threadIdx.x; i < 2 * 2 * 16; i += blockDim.x) (&ctr[0][0][0])[i] = 0;
  }
  __syncthreads();
  const uint8_t* slab_g = reinterpret_cast<const uint8_t*>(p.twB) +
                          (long long)j * mp_block_records(kQS1) * RB;

  // this warp's units: team-local v = par + 2 k, global u = tau + teams v
  const long long team_units = p.units > tau ? (p.units - tau + p.teams - 1) / p.teams : 0;
  const int nk = team_units > par ? int((team_units - par + 1) / 2) : 0;
  const int ntiles = 2 * nk;
  const int a0 = nk < D ? nk : D;
  const int c2 = nk > D ? nk - D : 0;
  auto tile_of = [&](int i, bool& is_b) -> int {
    if (i < a0) { is_b = false; return i; }
    const int i2 = i - a0;
    if (i2 < 2 * c2) { is_b = i2 & 1; return is_b ? i2 / 2 : D + i2 / 2; }
    is_b = true;
    return c2 + (i2 - 2 * c2);
  };
  auto unit_v = [&](int k) { return (long long)par + 2LL * k; };
  // flags count MEMBERS: the 8th quad warp of a member to finish a unit's
  // tile publishes for the member (smem counters ctr)
  auto spin = [&](const uint32_t* f, uint32_t want) {
    if (lane == 0) ptx::wait_at_least(f, want);
    __syncwarp();
  };

  // cp.async of tile i into this warp's slot (16 per lane)
  auto issue = [&](int i) {
    bool is_b;
    const long long v = unit_v(tile_of(i, is_b));
    if (!is_b) {  // first group: rows c of columns q = 32 j + 4 quad .. +3, from HBM
      const long long b = (tau + (long long)p.teams * v) * PAIR;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int idx = lane + 32 * k;
        if constexpr (PAIR == 2) {  // two 16-byte halves per row (transforms b, b+1)
          const int h = idx >> 8, r = idx & 255;
          const bool ok = b + h < p.nb;  // a missing pair partner is zero-filled
          const uint8_t* src =
              p.in + ((b + (ok ? h : 0)) * N + (long long)r * NS + j * 32 + quad * 4) * EB;
          ptx::cp_async16(slot_s + h * 4096 + r * 16, src, ok ? 16u : 0u);
        } else {  // one 32-byte row segment per row
          const int r = idx >> 1, hh = idx & 1;
          const uint8_t* src =
              p.in + (b * N + (long long)r * NS + j * 32 + quad * 4) * EB + hh * 16;
          ptx::cp_async16(slot_s + r * 32 + hh * 16, src, 16u);
        }
      }
    } else {  // second group: block j of the team's scratch slot, from L2
      const int slot = int(v % R);
      spin(p.done + tau * R + slot, uint32_t(K) * uint32_t(v / R + 1));
      const uint8_t* blk = p.mid + (long long)(tau * R + slot) * N * kUnitScale +
                           (long long)j * (kQL * 32 * 8) + quad * 32;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int idx = lane + 32 * k;
        const int r = idx >> 1, hh = idx & 1;
        ptx::cp_async16(slot_s + r * 32 + hh * 16, blk + r * 256 + hh * 16, 16u);
      }
    }
    ptx::cp_async_commit();
  };

  if (ntiles > 0) issue(0);
  for (int i = 0; i < ntiles; ++i) {
    bool is_b;
    const int k = tile_of(i, is_b);
    const long long v = unit_v(k);
    const int slot = int(v % R);
    const long long b = (tau + (long long)p.teams * v) * PAIR;
    bool next_b = false;
    const bool has_next = i + 1 < ntiles;
    const bool next_is_own = has_next && !is_b && tile_of(i + 1, next_b) == k && next_b;
    ptx::cp_async_wait_all();
    __syncwarp();
    auto release = [&] {
      if (has_next && !next_is_own) issue(i + 1);
    };
    if (!is_b) {
      uint8_t* obase = p.mid + (long long)(tau * R + slot) * N * kUnitScale +
                       ((long long)(j * 32 + col) * 32 + sub) * 8;
      quad_tile<A, STANDARD, INVERSE, true>(
          slot_s, twA, twB, slab_g, obase, 0, false, p.scale, quad, lane, release,
          [&] {  // the slot's previous unit has been read by every member
            spin(p.freed + tau * R + slot, uint32_t(K) * uint32_t(v / R));
          });
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        const uint32_t old = atomicAdd(&ctr[par][0][slot], 1u);
        if ((old & 7) == 7) ptx::red_release_add(p.done + tau * R + slot, 1);  // member done
      }
      if (next_is_own) issue(i + 1);
    } else {
      // landed: the 8th quad warp of the member drops the member's scratch
      // block from L2 (dead data, never written back) and frees the slot
      uint32_t last = 0;
      if (lane == 0) last = (atomicAdd(&ctr[par][1][slot], 1u) & 7) == 7;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        const uint8_t* blk =
            p.mid + (long long)(tau * R + slot) * N * kUnitScale + (long long)j * (kQL * 32 * 8);
        for (int off = lane * 128; off < kQL * 32 * 8; off += 32 * 128)
          ptx::discard_l2_line(blk + off);
        __syncwarp();
        if (lane == 0) ptx::red_release_add(p.freed + tau * R + slot, 1);
      }
      uint8_t* obase = p.out + (b * N + j * 32 + col + ((long long)sub << 8)) * EB;
      quad_tile<A, STANDARD, INVERSE, false>(slot_s, twA, twB, slab_g, obase, N * EB,
                                             b + 1 < p.nb, p.scale, quad, lane, release, [] {});
    }
  }
}

template <class A, bool STD>
cudaError_t quad_go(const FusedParams& p, bool inverse, int grid, cudaStream_t st) {
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(QuadLayout<A>::kSmem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kQWarps * 32);
    cfg.dynamicSmemBytes = QuadLayout<A>::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every team member co-resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  };
  return inverse ? go(mp_quad_kernel<A, STD, true>) : go(mp_quad_kernel<A, STD, false>);
}

}  // namespace

size_t quad_smem_bytes(int precision) {
  return precision == kFp16 ? QuadLayout<ArithF16P>::kSmem : QuadLayout<ArithF32>::kSmem;
}

cudaError_t quad_launch(const FusedParams& p, int precision, bool standard, bool inverse,
                        int grid, cudaStream_t st) {
  if (precision == kFp16)
    return standard ? quad_go<ArithF16P, true>(p, inverse, grid, st)
                    : quad_go<ArithF16P, false>(p, inverse, grid, st);
  return standard ? quad_go<ArithF32, true>(p, inverse, grid, st)
                  : quad_go<ArithF32, false>(p, inverse, grid, st);
}

std::vector<Record> quad_slab_records(const std::vector<TableEntry>& table, int m, int strategy,
                                      int precision) {
  // second group of the 8 + 8 split: P = 8, S1 = 3, K = 2^8 / 32 = 8 blocks
  const int P = 8;
  const long long blocks = (1LL << P) >> 5;
  const int per = mp_block_records(kQS1);
  std::vector<Record> recs(size_t(blocks) * per);
  auto rec = [&](long long k) { return pack_record(table[k], strategy, precision, false); };
  for (long long rb = 0; rb < blocks; ++rb) {
    Record* blk = recs.data() + rb * per;
    for (int c = 0; c < 32; ++c) {
      const long long r = rb * 32 + c;
      for (int pl = 0; pl < 5; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          blk[((1 << pl) - 1 + rl) * 32 + c] = rec((r + ((long long)rl << P)) << (m - P - pl - 1));
      for (int pl = 0; pl < kQS1; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          for (int r_l = 0; r_l < 32; ++r_l) {
            const long long lf = r_l + 32LL * rl;  // local frequency
            blk[quad_slab_index((1 << pl) - 1 + rl, r_l, c)] =
                rec((r + (lf << P)) << (m - P - 5 - pl - 1));
          }
    }
  }
  return recs;
}

}  // namespace dsfft
