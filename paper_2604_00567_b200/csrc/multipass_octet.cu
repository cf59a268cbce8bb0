// multipass_octet.cu -- the one-launch N = 2^16 (s = 8 + 8) path on 2-warp
// tile groups.
//
// mp_fused_kernel gives each 32-column x 256-row tile to an 8-warp group; the
// stage-1 / stage-2 exchange couples all 8 warps (three named barriers per
// tile), and the kernel is SM-latency bound (profiles/r02_fused_multipass.md).
// Splitting the tile into 4-column quads per warp removed the coupling but
// made every memory segment 16-32 bytes wide (1.4-2x slower).  The middle
// ground here: a tile group of 2 warps owns an OCTET of 8 columns (all 256
// rows) -- the whole column FFTs of its octet -- so
//   * the coupling is 64 threads (like the single-kernel path at N = 2048,
//     82% of HBM, against 8-warp groups' 58% at N = 8192);
//   * every memory segment is a whole 32-byte sector: 8 x 4 B user-row
//     halves, 8 x 8 B intermediate rows, 8 x 4 B output runs, stores of
//     4 x 8 B intermediate columns;
//   * one TMA box {8 columns, 256 rows} per transform half fills the group's
//     private 16 KB slot (dense rows: 32 B user halves, 64 B intermediate).
// Lanes: t = thread in the group (0..63), c8 = t & 7 (column), sub = t >> 3.
// Stage 1 takes rows sub + 8 i (i < 32) of column c8 -- warp `sub`'s 32-point
// sub-FFT of the 8-warp tile -- and runs passes 0..4 in registers.  The
// exchange stores output c of (c8, sub) at row 8 c + (sub ^ (c & 7)) of the
// slot (64-byte rows), and stage 2 -- group (c8, r_l = sub + 8 t), 8 values
// -- reads row 8 r_l + (cc ^ sub): each warp's 4 rows split 2 even / 2 odd,
// so both hit every bank exactly twice (the 2-wavefront minimum for 256 B).
// Second-group twiddles use an octet-ordered slab (octet_slab_index): the 32
// lanes of a warp read 32 consecutive records.
//
// Teams, scratch ring, lag and counters are mp_fused_kernel's protocol
// (multipass_fused.cu).  The four octet groups of a member tally their tiles
// of a unit in shared memory; the fourth publishes for the member, so the
// done / freed counters still count members.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "host_table.hpp"
#include "multipass_impl.cuh"

namespace dsfft {

namespace {

constexpr int kOS1 = 3;              // s = 8: 5 + 3 passes
constexpr int kOL = 256;             // rows of a tile
constexpr int kOSlot = kOL * 8 * 8;  // 16 KB: 256 rows x 8 columns x 8-byte values
constexpr int kOGroups = 8;          // 2-warp groups per CTA: 4 octets x 2 unit streams
constexpr int kOT = 64;              // threads per group

// second-group stage-2 record (slot2, r_l, col) of a column block:
//   31*32 + ((slot2*4 + r_l/8)*4 + col/8)*64 + (r_l%8)*8 + col%8
__host__ __device__ constexpr int octet_slab_index(int slot2, int r_l, int col) {
  return 31 * 32 + ((((slot2 * 4 + (r_l >> 3)) << 2) + (col >> 3)) << 6) + ((r_l & 7) << 3) +
         (col & 7);
}

template <class A>
struct OctetLayout {
  static constexpr int RB = A::kRecBytes;
  // 8-byte records (fp16 pairs): the whole 65 KB slab in smem; 16-byte (fp32):
  // stage 1 in smem, stage 2 through L1
  static constexpr bool kFullSlab = RB == 8;
  static constexpr int kTwA = (mp_first_records(kOS1) * RB + 127) & ~127;
  static constexpr int kTwB = ((kFullSlab ? mp_block_records(kOS1) : 31 * 32) * RB + 127) & ~127;
  static constexpr size_t kSmem =
      size_t(kTwA) + kTwB + size_t(kOGroups) * kOSlot + size_t(kOGroups) * 8;
};

// One octet tile in the group's slot.  FIRST: first pass group (user rows
// in, blocked pair-packed intermediate out); else the second group (blocked
// intermediate in, natural order out).  obase: this lane's output base.
template <class A, bool STANDARD, bool INVERSE, bool FIRST, class Sync, class Release,
          class PreStore>
__device__ __forceinline__ void octet_tile(uint32_t slot_s, uint32_t twA, uint32_t twB,
                                           const uint8_t* slab_g, uint8_t* obase,
                                           long long second_off, bool second, uint32_t scale,
                                           int oct, int t, Sync&& sync, Release&& release,
                                           PreStore&& pre_store) {
  using Lay = OctetLayout<A>;
  constexpr int RB = A::kRecBytes, PAIR = A::kPair;
  const int c8 = t & 7, sub = t >> 3, col = oct * 8 + c8;
  uint32_t re[32], im[32];
  // ---- stage 1: rows sub + 8 i of column c8 -----------------------------------
  {
    const uint32_t a32 = slot_s + sub * 32 + c8 * 4;  // user halves: 32-byte rows
    const uint32_t a64 = slot_s + sub * 64 + c8 * 8;  // 8-byte values: 64-byte rows
#pragma unroll
    for (int ii = 0; ii < 32; ++ii) {
      if constexpr (FIRST && PAIR == 2) {
        const uint32_t lo = ptx::lds32(a32 + ii * 256);
        const uint32_t hi = ptx::lds32(a32 + kOSlot / 2 + ii * 256);
        re[ii] = __byte_perm(lo, hi, 0x5410);
        im[ii] = __byte_perm(lo, hi, 0x7632);
      } else {
        ptx::lds64(a64 + ii * 512, re[ii], im[ii]);
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
  // ---- exchange in the group's slot -------------------------------------------
  sync();  // both warps' stage-1 loads are done
  {
    const uint32_t base = slot_s + c8 * 8;
#pragma unroll
    for (int c7 = 0; c7 < 8; ++c7) {
      const uint32_t a = base + (sub ^ c7) * 64;
#pragma unroll
      for (int hi = 0; hi < 4; ++hi) {
        const int cc = hi * 8 + c7;
        ptx::sts64(a + cc * 512, re[cc], im[cc]);
      }
    }
  }
  sync();
  {
    const uint32_t base = slot_s + sub * 512 + c8 * 8;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const uint32_t a = base + (cc ^ sub) * 64;
#pragma unroll
      for (int tt = 0; tt < 4; ++tt)
        ptx::lds64(a + tt * 4096, re[(tt << 3) + cc], im[(tt << 3) + cc]);
    }
  }
  ptx::fence_proxy_async_smem();  // generic reads of the slot precede the next TMA write
  sync();
  release();  // the slot is free: the next tile's TMA goes out now
  // ---- stage 2: groups (column c8, r_l = sub + 8 tt), 8 values each -----------
#pragma unroll
  for (int pl = 0; pl < kOS1; ++pl) {
    uint32_t nre[32], nim[32];
#pragma unroll
    for (int rl = 0; rl < (1 << pl); ++rl)
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) {
        const int slot2 = (1 << pl) - 1 + rl;
        const int r_l = sub + 8 * tt;
        uint4 tw;
        if constexpr (FIRST)
          tw = load_rec<A>(twA + (31 + (slot2 << 5) + r_l) * RB);
        else if constexpr (Lay::kFullSlab)
          tw = load_rec<A>(twB + octet_slab_index(slot2, r_l, col) * RB);
        else
          tw = ldg_rec<A>(slab_g + octet_slab_index(slot2, r_l, col) * RB);
#pragma unroll
        for (int qq = 0; qq < ((1 << (kOS1 - 1)) >> pl); ++qq) {
          const int jl = (qq << pl) | rl;
          const int ia = (tt << kOS1) + jl, ib = ia + (1 << (kOS1 - 1));
          const int oa = (tt << kOS1) + (qq << (pl + 1)) + rl;
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
  for (int tt = 0; tt < 4; ++tt)
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      uint32_t xr = re[(tt << 3) + cc], xi = im[(tt << 3) + cc];
      if constexpr (FIRST) {
        // value cc of group (q_col, r_l) -> second-group block cc, row q_col,
        // column r_l: obase = unit + ((32 j + col) * 32 + sub) * 8
        __stcg(reinterpret_cast<uint2*>(obase + cc * (kOL * 32 * 8) + tt * 64),
               make_uint2(xr, xi));
      } else {
        // natural position 32 j + col + 2^8 (r_l + 32 cc):
        // obase = out + (b N + 32 j + col + 2^8 sub) * EB
        constexpr int EB = A::kSampleBytes;
        uint8_t* dst = obase + ((tt * 8 + cc * 32) << 8) * EB;
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
__global__ void __launch_bounds__(kOGroups * kOT, 1)
    mp_octet_kernel(const __grid_constant__ CUtensorMap in_map,
                    const __grid_constant__ CUtensorMap mid_map, const FusedParams p) {
  using Lay = OctetLayout<A>;
  constexpr int RB = A::kRecBytes, PAIR = A::kPair, EB = A::kSampleBytes;
  constexpr long long kUnitScale = PAIR * EB;  // bytes per sample of a unit (8)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t ctr[2][2][16];  // [stream][A stored / B landed][slot]: octet tiles
  const int g = threadIdx.x / kOT, t = threadIdx.x % kOT;
  const int oct = g & 3, par = g >> 2;  // column octet of the block, unit stream
  const int c8 = t & 7, sub = t >> 3;
  const bool leader = t == 0;
  const int K = p.K, R = p.R, D = p.D;
  const int tau = blockIdx.x / K, j = blockIdx.x - (blockIdx.x / K) * K;
  const long long N = 1LL << p.m;
  const uint32_t twA = ptx::smem_u32(smem), twB = twA + Lay::kTwA;
  uint8_t* slot = smem + Lay::kTwA + Lay::kTwB + size_t(g) * kOSlot;
  const uint32_t slot_s = ptx::smem_u32(slot);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::kTwA + Lay::kTwB +
                                              size_t(kOGroups) * kOSlot) + g;
  const int col = oct * 8 + c8;
  {  // both groups' twiddles, once per launch (member j = column block j)
    uint4* sa = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < (mp_first_records(kOS1) * RB + 15) / 16; i += blockDim.x)
      sa[i] = p.twA[i];
    const uint4* src = p.twB + (long long)j * mp_block_records(kOS1) * RB / 16;
    uint4* sb = reinterpret_cast<uint4*>(smem + Lay::kTwA);
    const int n16 = (Lay::kFullSlab ? mp_block_records(kOS1) : 31 * 32) * RB / 16;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) sb[i] = src[i];
    for (int i = threadIdx.x; i < 2 * 2 * 16; i += blockDim.x) (&ctr[0][0][0])[i] = 0;
  }
  if (leader) ptx::mbar_init(bar, 1);
  ptx::fence_mbar_init();
  __syncthreads();
  const uint8_t* slab_g = reinterpret_cast<const uint8_t*>(p.twB) +
                          (long long)j * mp_block_records(kOS1) * RB;
  auto sync = [&] { ptx::named_bar_sync(1 + g, kOT); };

  // this group's units: team-local v = par + 2 k, global u = tau + teams v
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
  uint64_t pol = 0;
  if (leader) pol = ptx::policy_evict_first();

  auto issue = [&](int i) {  // leader only
    bool is_b;
    const long long v = unit_v(tile_of(i, is_b));
    if (!is_b) {  // first group: columns 32 j + 8 oct .. +7 of the unit's transform(s)
      ptx::mbar_arrive_expect_tx(bar, kOSlot);
      const int b = int((tau + (long long)p.teams * v) * PAIR);
#pragma unroll
      for (int h = 0; h < PAIR; ++h)
        ptx::tma_load_3d(slot + h * (kOSlot / 2), &in_map, j * 32 + oct * 8, 0, b + h, bar, pol);
    } else {  // second group: octet of block j of the team's scratch slot, from L2
      const int s = int(v % R);
      ptx::wait_at_least(p.done + tau * R + s, uint32_t(K) * uint32_t(v / R + 1));
      ptx::fence_proxy_async_global();  // generic-proxy stores -> TMA reads
      ptx::mbar_arrive_expect_tx(bar, kOSlot);
      ptx::tma_load_4d(slot, &mid_map, oct * 8, 0, j, tau * R + s, bar, pol);
    }
  };

  if (leader && ntiles > 0) issue(0);
  for (int i = 0; i < ntiles; ++i) {
    bool is_b;
    const int k = tile_of(i, is_b);
    const long long v = unit_v(k);
    const int s = int(v % R);
    const long long b = (tau + (long long)p.teams * v) * PAIR;
    bool next_b = false;
    const bool has_next = i + 1 < ntiles;
    const bool next_is_own = has_next && !is_b && tile_of(i + 1, next_b) == k && next_b;
    ptx::mbar_wait(bar, uint32_t(i & 1));
    auto release = [&] {
      if (leader && has_next && !next_is_own) issue(i + 1);
    };
    if (!is_b) {
      uint8_t* obase =
          p.mid + (long long)(tau * R + s) * N * kUnitScale + ((long long)(j * 32 + col) * 32 + sub) * 8;
      octet_tile<A, STANDARD, INVERSE, true>(
          slot_s, twA, twB, slab_g, obase, 0, false, p.scale, oct, t, sync, release, [&] {
            // the slot's previous unit has been read by every member
            if (leader) ptx::wait_at_least(p.freed + tau * R + s, uint32_t(K) * uint32_t(v / R));
            sync();
          });
      ptx::fence_proxy_async_global();
      sync();
      if (leader) {
        __threadfence();
        const uint32_t old = atomicAdd(&ctr[par][0][s], 1u);
        if ((old & 3) == 3) ptx::red_release_add(p.done + tau * R + s, 1);  // member done
        if (next_is_own) issue(i + 1);
      }
    } else {
      if (t < 32) {
        // landed: the member's fourth octet drops the member's scratch block
        // from L2 (dead data, never written back) and frees the slot
        uint32_t last = 0;
        if (leader) last = (atomicAdd(&ctr[par][1][s], 1u) & 3) == 3;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          const uint8_t* blk =
              p.mid + (long long)(tau * R + s) * N * kUnitScale + (long long)j * (kOL * 32 * 8);
          for (int off = t * 128; off < kOL * 32 * 8; off += 32 * 128)
            ptx::discard_l2_line(blk + off);
          __syncwarp();
          if (leader) ptx::red_release_add(p.freed + tau * R + s, 1);
        }
      }
      uint8_t* obase = p.out + (b * N + j * 32 + col + ((long long)sub << 8)) * EB;
      octet_tile<A, STANDARD, INVERSE, false>(slot_s, twA, twB, slab_g, obase, N * EB,
                                              b + 1 < p.nb, p.scale, oct, t, sync, release,
                                              [] {});
    }
  }
}

template <class A, bool STD>
cudaError_t octet_go(const CUtensorMap& in_map, const CUtensorMap& mid_map, const FusedParams& p,
                     bool inverse, int grid, cudaStream_t st) {
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(OctetLayout<A>::kSmem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kOGroups * kOT);
    cfg.dynamicSmemBytes = OctetLayout<A>::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every team member co-resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, in_map, mid_map, p);
  };
  return inverse ? go(mp_octet_kernel<A, STD, true>) : go(mp_octet_kernel<A, STD, false>);
}

}  // namespace

size_t octet_smem_bytes(int precision) {
  return precision == kFp16 ? OctetLayout<ArithF16P>::kSmem : OctetLayout<ArithF32>::kSmem;
}

cudaError_t octet_launch(const CUtensorMap& in_map, const CUtensorMap& mid_map,
                         const FusedParams& p, int precision, bool standard, bool inverse,
                         int grid, cudaStream_t st) {
  if (precision == kFp16)
    return standard ? octet_go<ArithF16P, true>(in_map, mid_map, p, inverse, grid, st)
                    : octet_go<ArithF16P, false>(in_map, mid_map, p, inverse, grid, st);
  return standard ? octet_go<ArithF32, true>(in_map, mid_map, p, inverse, grid, st)
                  : octet_go<ArithF32, false>(in_map, mid_map, p, inverse, grid, st);
}

std::vector<Record> octet_slab_records(const std::vector<TableEntry>& table, int m, int strategy,
                                       int precision) {
  // second group of the 8 + 8 split: P = 8, S1 = 3, K = 2^8 / 32 = 8 blocks
  const int P = 8;
  const long long blocks = (1LL << P) >> 5;
  const int per = mp_block_records(kOS1);
  std::vector<Record> recs(size_t(blocks) * per);
  auto rec = [&](long long k) { return pack_record(table[k], strategy, precision, false); };
  for (long long rb = 0; rb < blocks; ++rb) {
    Record* blk = recs.data() + rb * per;
    for (int c = 0; c < 32; ++c) {
      const long long r = rb * 32 + c;
      for (int pl = 0; pl < 5; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          blk[((1 << pl) - 1 + rl) * 32 + c] = rec((r + ((long long)rl << P)) << (m - P - pl - 1));
      for (int pl = 0; pl < kOS1; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          for (int r_l = 0; r_l < 32; ++r_l) {
            const long long lf = r_l + 32LL * rl;  // local frequency
            blk[octet_slab_index((1 << pl) - 1 + rl, r_l, c)] =
                rec((r + (lf << P)) << (m - P - 5 - pl - 1));
          }
    }
  }
  return recs;
}

}  // namespace dsfft
