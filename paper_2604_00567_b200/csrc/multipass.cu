// multipass.cu -- batched forward/inverse for N = 2^13 .. 2^24.
//
// The m = log2 N passes are split into 2-3 consecutive pass groups
// [P, P+s), s in 6..9, each one launch of mp_kernel (SURVEY.md A.1 item 3
// regrouping, bit-exact).  A pass group works on independent groups
// g = q*2^P + r: group g gathers x[g + c*N/2^s] (c < 2^s), runs s radix-2
// passes whose butterflies use the reference's table entries
// (r + 2^P*rl') * N/2^(P+pl'+1), and scatters to q*2^(P+s) + r + 2^P*c'.
//
// CTA tile = 32 consecutive groups ("columns") x 2^s rows:
//   * first group (P = 0): columns are 32 consecutive q; a column's outputs
//     are 2^s contiguous samples;
//   * later groups (P >= 5): columns are 32 consecutive r at fixed q, so
//     every row of the tile is 32 contiguous samples in and out.
// Inside the CTA: stage 1 = 5 passes in registers (lane = column, warp =
// row group), exchange through padded smem, stage 2 = s-5 passes in
// registers; lanes always walk contiguous samples, so each warp load/store
// moves whole 128-byte lines.  Twiddle records are laid out per kernel in
// exactly the order lanes consume them (coalesced 16-byte loads from L2).
//
// The batch runs in chunks whose intermediate fits in L2 (126 MB), so the
// pass groups after the first read their input from L2, not HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fft_kernels.cuh"
#include "multipass.cuh"

namespace dsfft {

namespace {
thread_local std::string g_mp_err;
}

const char* multipass_error() { return g_mp_err.c_str(); }

struct MpParams {
  const uint8_t* in;
  uint8_t* out;
  const uint4* tw;  // this pass group's records
  int m, P;         // log2 N, first pass of the group
  long long tiles_per_transform;
  long long tiles;  // chunk transforms x tiles_per_transform
  uint32_t scale;
  int last;         // output is the user's buffer (stream it out of L2)
};

// Twiddle record offsets inside one pass group's table.
//   stage 1 (local passes 0..4): slot (2^pl - 1 + rl) in 0..30
//   stage 2 (local passes 5..s-1): slot 31 + (2^pl - 1 + rl) * 32 + r_l
// and, for later groups, times 2^P + r (the column's global frequency).
__host__ __device__ constexpr int mp_slot1(int pl, int rl) { return (1 << pl) - 1 + rl; }
__host__ __device__ constexpr int mp_slot2(int pl, int rl, int r_l) {
  return 31 + (((1 << pl) - 1 + rl) << 5) + r_l;
}
__host__ __device__ constexpr int mp_slots(int s) { return 31 + (((1 << (s - 5)) - 1) << 5); }

template <class A>
__device__ __forceinline__ void mp_load(const uint8_t* base, long long idx, uint32_t& re,
                                        uint32_t& im, bool streaming) {
  if constexpr (A::kWords == 1) {
    const unsigned int* p = reinterpret_cast<const unsigned int*>(base) + idx;
    re = streaming ? __ldcs(p) : __ldcg(p);
  } else {
    const uint2* p = reinterpret_cast<const uint2*>(base) + idx;
    const uint2 v = streaming ? __ldcs(p) : __ldcg(p);
    re = v.x;
    im = v.y;
  }
}

template <class A>
__device__ __forceinline__ void mp_store(uint8_t* base, long long idx, uint32_t re, uint32_t im,
                                         bool streaming) {
  if constexpr (A::kWords == 1) {
    unsigned int* p = reinterpret_cast<unsigned int*>(base) + idx;
    if (streaming) __stcs(p, re); else __stcg(p, re);
  } else {
    uint2* p = reinterpret_cast<uint2*>(base) + idx;
    if (streaming) __stcs(p, make_uint2(re, im)); else __stcg(p, make_uint2(re, im));
  }
}

// One pass group over all tiles of a chunk.  T = 32 * 2^S1 threads; each
// thread owns 32 values in stage 1 and 2^(5-S1) groups of 2^S1 in stage 2.
template <int S1, class A, bool STANDARD, bool FIRST, bool CONJ_IN, bool SCALE_OUT>
__global__ void __launch_bounds__(32 << S1, (512 >> S1) / 32) mp_kernel(const MpParams p) {
  constexpr int s = 5 + S1, L = 1 << s, T = 32 << S1, NG2 = 32 >> S1;
  constexpr int VB = A::kWords * 4;                 // bytes per value
  constexpr int STRIDE = L + 1;                     // padded smem column (values)
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sbase = ptx::smem_u32(smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long N = 1LL << p.m;
  const long long rows_stride = N >> s;             // input row stride (samples)
  const int P = p.P;

  for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
    const long long b = tile / p.tiles_per_transform;  // transform within chunk
    const long long tt = tile - b * p.tiles_per_transform;
    const uint8_t* gin = p.in + b * N * (A::kPair == 1 ? A::kSampleBytes : 4);
    uint8_t* gout = p.out + b * N * (A::kPair == 1 ? A::kSampleBytes : 4);
    // column (group) of this lane in stage 1 and its global frequency r
    long long g;   // group index g = q*2^P + r
    int r;         // 0 for the first group
    if constexpr (FIRST) {
      g = tt * 32 + lane;
      r = 0;
    } else {
      const long long rblocks = (1LL << P) >> 5;
      const long long q = tt / rblocks;
      r = int((tt - q * rblocks) * 32 + lane);
      g = (q << P) + r;
    }
    const long long g0 = g - lane;
    uint32_t re[32], im[32];
    // ---- stage 1: rows warp + c*2^S1 of this lane's column ------------------
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int row = warp + (c << S1);
      mp_load<A>(gin, g + row * rows_stride, re[c], im[c], FIRST);
      if constexpr (CONJ_IN) {  // conj on load (fft.cpp:90-91)
        if constexpr (A::kWords == 1) re[c] ^= 0x80000000u; else im[c] = A::neg(im[c]);
      }
    }
#pragma unroll
    for (int pl = 0; pl < 5; ++pl) {
      uint32_t nre[32], nim[32];
#pragma unroll
      for (int rl = 0; rl < (1 << pl); ++rl) {
        const long long idx = FIRST ? mp_slot1(pl, rl)
                                    : ((long long)mp_slot1(pl, rl) << P) + r;
        const uint4 tw = __ldg(p.tw + idx);
#pragma unroll
        for (int q = 0; q < (16 >> pl); ++q) {
          const int jl = (q << pl) | rl;
          const int oa = (q << (pl + 1)) + rl;
          butterfly<A, STANDARD>(re[jl], im[jl], re[jl + 16], im[jl + 16], tw, nre[oa], nim[oa],
                                 nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        re[i] = nre[i];
        if constexpr (A::kWords == 2) im[i] = nim[i];
      }
    }
    // ---- exchange: local position warp*32 + c' of column lane ----------------
    __syncthreads();  // previous tile's stage-2 reads are done
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t a = sbase + (lane * STRIDE + warp * 32 + c) * VB;
      if constexpr (A::kWords == 1) ptx::sts32(a, re[c]); else ptx::sts64(a, re[c], im[c]);
    }
    __syncthreads();
    // ---- stage 2: groups (column, r_l), values at local rows r_l + 32*c ------
    int col[NG2], rloc[NG2];
#pragma unroll
    for (int j = 0; j < NG2; ++j) {
      const int glin = threadIdx.x + T * j;
      if constexpr (FIRST) {  // lanes walk r_l: contiguous column output
        rloc[j] = glin & 31;
        col[j] = glin >> 5;
      } else {                // lanes walk columns: contiguous row output
        col[j] = glin & 31;
        rloc[j] = glin >> 5;
      }
#pragma unroll
      for (int c = 0; c < (1 << S1); ++c) {
        const uint32_t a = sbase + (col[j] * STRIDE + rloc[j] + 32 * c) * VB;
        const int v = (j << S1) + c;
        if constexpr (A::kWords == 1) re[v] = ptx::lds32(a); else ptx::lds64(a, re[v], im[v]);
      }
    }
#pragma unroll
    for (int pl = 0; pl < S1; ++pl) {
      uint32_t nre[32], nim[32];
#pragma unroll
      for (int rl = 0; rl < (1 << pl); ++rl)
#pragma unroll
        for (int j = 0; j < NG2; ++j) {
          const int rcol = FIRST ? 0 : r - lane + col[j];  // global r of this group's column
          const long long idx = FIRST ? mp_slot2(pl, rl, rloc[j])
                                      : ((long long)mp_slot2(pl, rl, rloc[j]) << P) + rcol;
          const uint4 tw = __ldg(p.tw + idx);
#pragma unroll
          for (int q = 0; q < ((1 << (S1 - 1)) >> pl); ++q) {
            const int jl = (q << pl) | rl;
            const int ia = (j << S1) + jl, ib = ia + (1 << (S1 - 1));
            const int oa = (j << S1) + (q << (pl + 1)) + rl;
            butterfly<A, STANDARD>(re[ia], im[ia], re[ib], im[ib], tw, nre[oa], nim[oa],
                                   nre[oa + (1 << pl)], nim[oa + (1 << pl)]);
          }
        }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        re[i] = nre[i];
        if constexpr (A::kWords == 2) im[i] = nim[i];
      }
    }
    // ---- scatter: q*2^(P+s) + r + 2^P*(r_l + 32 c') ------------------------
#pragma unroll
    for (int j = 0; j < NG2; ++j)
#pragma unroll
      for (int c = 0; c < (1 << S1); ++c) {
        const int v = (j << S1) + c;
        uint32_t xr = re[v], xi = im[v];
        if constexpr (SCALE_OUT) {  // conj + 1/n, one rounded mul each (fft.cpp:94-98)
          if constexpr (A::kWords == 1) {
            xr = A::mul(xr ^ 0x80000000u, p.scale);
          } else {
            xr = A::mul(xr, p.scale);
            xi = A::mul(A::neg(xi), p.scale);
          }
        }
        const int lrow = rloc[j] + 32 * c;  // local output row c'
        long long pos;
        if constexpr (FIRST) {
          pos = (g0 + col[j]) * L + lrow;  // column-contiguous (P = 0)
        } else {
          const long long gc = g0 + col[j];
          const long long q = gc >> P, rr = gc & ((1LL << P) - 1);
          pos = (q << (P + s)) + rr + ((long long)lrow << P);
        }
        mp_store<A>(gout, pos, xr, xi, p.last != 0);
      }
  }
}

// ---- host side ---------------------------------------------------------------

struct MpGroup {
  int P, s;
  uint4* d_tw = nullptr;
};

struct MultipassPlan {
  int m = 0, strategy = 0, precision = 0, sm_count = 0;
  std::vector<MpGroup> groups;
  uint8_t* scratch[2] = {nullptr, nullptr};
  size_t chunk_transforms = 0;
  ~MultipassPlan() {
    for (auto& g : groups)
      if (g.d_tw) cudaFree(g.d_tw);
    for (auto* s : scratch)
      if (s) cudaFree(s);
  }
};

namespace {

std::vector<int> split_passes(int m) {
  // 2 groups up to m = 18, 3 beyond; every group 6..9 passes, first >= 5
  if (m <= 18) {
    const int a = (m + 1) / 2;
    return {a, m - a};
  }
  const int a = (m + 2) / 3, b = (m - a + 1) / 2;
  return {a, b, m - a - b};
}

template <int S1, class A, bool STD>
cudaError_t mp_launch_t(const MpParams& p, bool first, bool conj_in, bool scale_out, int grid,
                        cudaStream_t st) {
  constexpr int s = 5 + S1;
  const size_t smem = size_t(32) * ((1 << s) + 1) * A::kWords * 4;
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, 32 << S1, smem, st>>>(p);
    return cudaGetLastError();
  };
  if (first)
    return conj_in ? go(mp_kernel<S1, A, STD, true, true, false>)
                   : go(mp_kernel<S1, A, STD, true, false, false>);
  return scale_out ? go(mp_kernel<S1, A, STD, false, false, true>)
                   : go(mp_kernel<S1, A, STD, false, false, false>);
}

template <class A, bool STD>
cudaError_t mp_launch_a(int S1, const MpParams& p, bool first, bool conj_in, bool scale_out,
                        int grid, cudaStream_t st) {
  switch (S1) {
    case 1: return mp_launch_t<1, A, STD>(p, first, conj_in, scale_out, grid, st);
    case 2: return mp_launch_t<2, A, STD>(p, first, conj_in, scale_out, grid, st);
    case 3: return mp_launch_t<3, A, STD>(p, first, conj_in, scale_out, grid, st);
    case 4: return mp_launch_t<4, A, STD>(p, first, conj_in, scale_out, grid, st);
  }
  return cudaErrorInvalidValue;
}

size_t sample_bytes(int precision) { return precision == kFp16 ? 4 : 8; }

}  // namespace

MultipassPlan* multipass_create(const std::vector<TableEntry>& table, int m, int strategy,
                                int precision, int sm_count, size_t /*smem_optin*/) {
  auto* mp = new MultipassPlan();
  mp->m = m;
  mp->strategy = strategy;
  mp->precision = precision;
  mp->sm_count = sm_count;
  const bool f16c = precision == kFp16;  // one complex per f16x2 register
  int P = 0;
  for (int s : split_passes(m)) {
    MpGroup g;
    g.P = P;
    g.s = s;
    const int S1 = s - 5;
    const long long reps = P == 0 ? 1 : (1LL << P);
    std::vector<Record> rec(size_t(mp_slots(s)) * reps);
    for (long long r = 0; r < reps; ++r) {
      // stage 1: local passes pl < 5, local freq rl' = rl
      for (int pl = 0; pl < 5; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl) {
          const long long k = (r + ((long long)rl << P)) << (m - P - pl - 1);
          rec[size_t(mp_slot1(pl, rl)) * reps + r] =
              pack_record(table[k], strategy, precision, f16c);
        }
      // stage 2: local passes 5 + pl, local freq rl' = r_l + 32 rl
      for (int pl = 0; pl < S1; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          for (int r_l = 0; r_l < 32; ++r_l) {
            const long long lf = r_l + 32LL * rl;
            const long long k = (r + (lf << P)) << (m - P - 5 - pl - 1);
            rec[size_t(mp_slot2(pl, rl, r_l)) * reps + r] =
                pack_record(table[k], strategy, precision, f16c);
          }
    }
    if (cudaMalloc(&g.d_tw, rec.size() * sizeof(Record)) != cudaSuccess ||
        cudaMemcpy(g.d_tw, rec.data(), rec.size() * sizeof(Record), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      g_mp_err = "multipass: twiddle upload failed";
      mp->groups.push_back(g);
      delete mp;
      return nullptr;
    }
    mp->groups.push_back(g);
    P += s;
  }
  // chunk so the intermediate (one scratch buffer) stays L2-resident
  const size_t tb = (size_t(1) << m) * sample_bytes(precision);
  const size_t want = size_t(48) << 20;
  mp->chunk_transforms = std::max<size_t>(1, want / tb);
  const size_t bytes = mp->chunk_transforms * tb;
  for (auto*& s : mp->scratch)
    if (cudaMalloc(&s, bytes) != cudaSuccess) {
      g_mp_err = "multipass: scratch allocation failed";
      delete mp;
      return nullptr;
    }
  return mp;
}

void multipass_destroy(MultipassPlan* mp) { delete mp; }

int multipass_execute(MultipassPlan& mp, bool inverse, const void* in, void* out, size_t batch,
                      uint32_t scale, cudaStream_t stream, uint64_t* launches) {
  const size_t tb = (size_t(1) << mp.m) * sample_bytes(mp.precision);
  const bool f16 = mp.precision == kFp16;
  const bool std_ = mp.strategy == kStandard;
  const int ng = int(mp.groups.size());
  for (size_t b0 = 0; b0 < batch; b0 += mp.chunk_transforms) {
    const size_t nb = std::min(mp.chunk_transforms, batch - b0);
    for (int i = 0; i < ng; ++i) {
      const MpGroup& g = mp.groups[i];
      MpParams p{};
      p.in = i == 0 ? static_cast<const uint8_t*>(in) + b0 * tb : mp.scratch[(i - 1) & 1];
      p.out = i == ng - 1 ? static_cast<uint8_t*>(out) + b0 * tb : mp.scratch[i & 1];
      p.tw = g.d_tw;
      p.m = mp.m;
      p.P = g.P;
      p.tiles_per_transform = ((1LL << mp.m) >> g.s) / 32;
      p.tiles = p.tiles_per_transform * (long long)nb;
      p.scale = scale;
      p.last = i == ng - 1;
      const int threads = 32 << (g.s - 5);
      const int per_sm = std::max(1, 2048 / threads);
      const int grid = int(std::min<long long>(p.tiles, (long long)mp.sm_count * per_sm));
      const bool first = i == 0, last = i == ng - 1;
      cudaError_t e =
          f16 ? (std_ ? mp_launch_a<ArithF16C, true>(g.s - 5, p, first, first && inverse,
                                                     last && inverse, grid, stream)
                      : mp_launch_a<ArithF16C, false>(g.s - 5, p, first, first && inverse,
                                                      last && inverse, grid, stream))
              : (std_ ? mp_launch_a<ArithF32, true>(g.s - 5, p, first, first && inverse,
                                                    last && inverse, grid, stream)
                      : mp_launch_a<ArithF32, false>(g.s - 5, p, first, first && inverse,
                                                     last && inverse, grid, stream));
      if (e != cudaSuccess) {
        g_mp_err = std::string("mp_kernel launch: ") + cudaGetErrorString(e);
        return 1;
      }
      if (launches) ++*launches;
    }
  }
  return 0;
}

}  // namespace dsfft
