// multipass.cu -- batched forward/inverse for N = 2^14 .. 2^24 (and 2^13 on request).
//
// The m = log2 N passes are split into 2-3 consecutive pass groups
// [P, P+s), s in 6..10, each one launch of mp_kernel (SURVEY.md A.1 item 3
// regrouping, bit-exact).  A pass group works on independent groups
// g = q*2^P + r: group g gathers x[g + c*N/2^s] (c < 2^s), runs s radix-2
// passes whose butterflies use the reference's table entries
// (r + 2^P*rl') * N/2^(P+pl'+1), and scatters to q*2^(P+s) + r + 2^P*c'.
//
// CTA tile = CW consecutive groups ("columns") x 2^s rows (CW = 32; 16 or 8
// for s = 10, whose 32-column tiles would not fit shared memory):
//   * first group (P = 0): columns are 32 consecutive q; each column's
//     outputs are 2^s contiguous samples;
//   * later groups (P >= 6): columns are 32 consecutive r at fixed q; every
//     row of the tile is 32 contiguous samples in and out.
// A persistent CTA owns a contiguous range of tiles (transform index fastest,
// so consecutive tiles share their twiddles) and keeps S tiles in flight:
// TMA tensor loads (3-D / 4-D maps with the batch as a coordinate, SASS
// UTMALDG) land each tile row-major in a shared-memory ring slot.  Stage 1 =
// 5 passes in registers (lane = column), exchange through the padded slot,
// stage 2 = s-5 passes; the slot is handed back to TMA right after the last
// smem read and results are stored straight from registers (full lines).
//
// Between groups the intermediate is blocked for the last group (each of its
// tiles one contiguous block) and, for fp16, pair-packed (8-byte values of
// transforms b, b+1).  The batch runs in chunks of up to 1 GiB
// (DSFFT_MP_CHUNK_MB); L2-sized chunks were measured slower.  N = 2^14 /
// 2^16 (fp16) and 2^14 (fp32) take the one-launch path of multipass_fused.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "multipass_impl.cuh"
#include "stream_alloc.cuh"

namespace dsfft {

namespace {
thread_local std::string g_mp_err;
}

const char* multipass_error() { return g_mp_err.c_str(); }
void set_mp_error(const std::string& msg) { g_mp_err = msg; }

struct MpParams {
  uint8_t* out;      // output of this pass group (chunk base)
  const uint4* tw;   // this pass group's twiddle records (see mp_*_records)
  int m, P;          // log2 N, first pass of the group
  int stages;        // ring depth
  long long nb;      // transforms in this chunk
  long long b_off;   // first transform of the chunk (tensor-map coordinate)
  long long tiles;   // nb * tiles_per_transform
  uint32_t scale;
  int keep_l2;       // load tiles evict_normal (box rows narrower than a line)
  int prefetch;      // L2-prefetch the tile this many ring turns ahead (0: off)
};

// One pass group over all tiles of a chunk.  A CTA runs G = blockDim/T tile
// groups of T = 32 * 2^S1 threads; each thread owns 32 values in stage 1 and
// 2^(5-S1) groups of 2^S1 in stage 2.  The CTA's contiguous tile range is
// walked unit by unit (a unit = one column block tt, a range of transforms);
// later pass groups stage the unit's twiddle slab once, shared by all groups,
// and group g takes transforms b0+g, b0+g+G, ... of the unit with its own TMA
// ring.  Register budget: one-word values ~80, two-word ~128.
template <int S1, class A, bool STANDARD, bool FIRST, bool CONJ_IN, bool SCALE_OUT, bool LAST,
          bool BOUT, int CW>
__global__ void __launch_bounds__(512) __maxnreg__(A::kWords == 1 ? 80 : 128)
    mp_kernel(const __grid_constant__ CUtensorMap in_map, const MpParams p) {
  using Lay = MpLayout<S1, A, CW>;
  constexpr int L = Lay::L, T = Lay::T;
  constexpr int ROWS_BOX = L < 256 ? L : 256;
  extern __shared__ __align__(128) uint8_t smem[];
  const int G = blockDim.x / T;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int lane = t & 31, warp = t >> 5;
  const int S = p.stages;
  const int P = p.P;
  const long long N = 1LL << p.m;
  constexpr int tw_bytes = Lay::tw_bytes(FIRST);
  constexpr int RB = A::kRecBytes;  // bytes per twiddle record
  uint4* tws = reinterpret_cast<uint4*>(smem);
  const uint32_t tw_base = ptx::smem_u32(smem);
  uint8_t* bufs = smem + tw_bytes + size_t(g) * S * Lay::kBufBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tw_bytes + size_t(G) * S * Lay::kBufBytes) +
                   g * S;
  const long long rblocks = FIRST ? 1 : ((1LL << P) >> 5);
  const bool leader = t == 0;

  if constexpr (FIRST) {  // column-independent twiddles: stage once per CTA
    for (int i = threadIdx.x; i < (mp_first_records(S1) * RB + 15) / 16; i += blockDim.x)
      tws[i] = p.tw[i];
  }
  if (leader)
    for (int i = 0; i < S; ++i) ptx::mbar_init(&bars[i], 1);
  ptx::fence_mbar_init();
  __syncthreads();

  uint64_t pol = 0;
  if (leader) pol = p.keep_l2 ? ptx::policy_evict_normal() : ptx::policy_evict_first();
  const int nb = int(p.nb);
  // TMA load of transform b of column block (q, rb) into ring slot `slot`
  // (fp16 pairs: transforms b and b+1 land in the two halves of the slot; a
  // b+1 past the batch is zero-filled by TMA and never stored)
  constexpr int PAIR = A::kPair;
  constexpr int EB = A::kSampleBytes;           // bytes of one complex in memory
  constexpr int HALF = CW * L * EB;             // one transform's tile
  // fp16 pairs keep intermediates pair-packed: 8-byte values (re0,re1),(im0,im1)
  // of transforms (b, b+1) at pair index b/2 -- no unpack/repack between groups
  constexpr bool PIN = PAIR == 2 && !FIRST;
  // hf: which CW-wide part of a later group's 32-column block (CW = 16: 0, 1)
  auto issue_load = [&](long long q, int rb, int hf, int b, int slot) {
    uint8_t* dst = bufs + size_t(slot) * Lay::kBufBytes;
    ptx::mbar_arrive_expect_tx(&bars[slot], Lay::kTileBytes);
#pragma unroll
    for (int h = 0; h < (PIN ? 1 : PAIR); ++h)
#pragma unroll
      for (int r0 = 0; r0 < L; r0 += ROWS_BOX) {
        uint8_t* d = dst + h * HALF + size_t(r0) * CW * (PIN ? 8 : EB);
        const int bb = PIN ? b / 2 : int(b + h + p.b_off);
        if constexpr (FIRST)
          ptx::tma_load_3d(d, &in_map, int(q * CW), r0, bb, &bars[slot], pol);
        else if constexpr (LAST)  // blocked intermediate {r_l, c, rb, b}
          ptx::tma_load_4d(d, &in_map, hf * CW, r0, rb, bb, &bars[slot], pol);
        else
          ptx::tma_load_4d(d, &in_map, rb * 32 + hf * CW, int(q), r0, bb, &bars[slot], pol);
      }
  };
  auto prefetch_load = [&](long long q, int rb, int hf, int b) {
#pragma unroll
    for (int h = 0; h < (PIN ? 1 : PAIR); ++h)
#pragma unroll
      for (int r0 = 0; r0 < L; r0 += ROWS_BOX) {
        const int bb = PIN ? b / 2 : int(b + h + p.b_off);
        if constexpr (FIRST)
          ptx::tma_prefetch_3d(&in_map, int(q * CW), r0, bb);
        else if constexpr (LAST)
          ptx::tma_prefetch_4d(&in_map, hf * CW, r0, rb, bb);
        else
          ptx::tma_prefetch_4d(&in_map, rb * 32 + hf * CW, int(q), r0, bb);
      }
  };
  auto tile = [&](long long q, int rb, int hf, int b, bool second, uint32_t buf,
                  auto&& release) {
    mp_tile<S1, A, STANDARD, FIRST, CONJ_IN, SCALE_OUT, LAST, BOUT, CW>(
        buf, tw_base, reinterpret_cast<const uint8_t*>(p.tw), p.scale, P, N, q, rb, hf * CW,
        second, g, warp, lane, [&] { return p.out + b * N * EB; },  // pair b/2 * N * 8 if packed
        release, [] {});
  };

  if constexpr (FIRST) {
    // Tiles in transform-major order (column block fastest): a CTA walks all
    // column blocks of one transform (pair) before the next, so the rows it
    // reads share DRAM pages; the twiddles are column-independent.
    const long long nblk = (N >> Lay::s) / CW;
    const long long total = nblk * ((p.nb + PAIR - 1) / PAIR);
    const long long per = (total + gridDim.x - 1) / gridDim.x;
    const long long t_begin = blockIdx.x * per;
    const long long t_end = t_begin + per < total ? t_begin + per : total;
    const long long first_idx = t_begin + g;
    const int k = first_idx < t_end ? int((t_end - first_idx + G - 1) / G) : 0;
    auto load_tile = [&](int i) {
      const long long idx = first_idx + (long long)G * i;
      const long long pr = idx / nblk;
      issue_load(idx - pr * nblk, 0, 0, int(pr * PAIR), i % S);
      const int ip = i + p.prefetch * S;
      if (p.prefetch && ip < k) {
        const long long idp = first_idx + (long long)G * ip;
        const long long prp = idp / nblk;
        prefetch_load(idp - prp * nblk, 0, 0, int(prp * PAIR));
      }
    };
    if (leader)
      for (int i = 0; i < S && i < k; ++i) load_tile(i);
    for (int i = 0; i < k; ++i) {
      const long long idx = first_idx + (long long)G * i;
      const long long pr = idx / nblk;
      const int b = int(pr * PAIR);
      const int slot = i % S;
      ptx::mbar_wait(&bars[slot], uint32_t((i / S) & 1));
      tile(idx - pr * nblk, 0, 0, b, PAIR == 2 && b + 1 < nb,
           ptx::smem_u32(bufs + size_t(slot) * Lay::kBufBytes), [&] {
             if (leader && i + S < k) load_tile(i + S);
           });
    }
  } else {
    // units of PAIR transforms, column block outer: tile u -> (tt, pair v,
    // part hf of the block when CW = 16)
    constexpr int HPB = 32 / CW;
    const long long nbu = (p.nb + PAIR - 1) / PAIR;
    const long long per_blk = nbu * HPB;
    const long long total = ((N >> Lay::s) >> 5) * per_blk;
    const long long per = (total + gridDim.x - 1) / gridDim.x;
    const long long t_begin = blockIdx.x * per;
    const long long t_end = t_begin + per < total ? t_begin + per : total;
    long long it = 0;  // this group's running tile count (ring slot / phase)
    for (long long u0 = t_begin; u0 < t_end;) {
      const long long tt = u0 / per_blk;  // column block of this unit
      const long long w0 = u0 - tt * per_blk;
      const long long u1 = (tt + 1) * per_blk < t_end ? (tt + 1) * per_blk : t_end;
      const int units = int(u1 - u0);
      u0 = u1;
      const long long q = tt / rblocks;
      const int rb = int(tt - q * rblocks);
      {  // the unit's twiddle slab, shared by every group
        __syncthreads();
        // block records start 16-byte aligned: mp_block_records(S1) * RB % 16 == 0
        const uint4* src = p.tw + (long long)rb * mp_block_records(S1) * RB / 16;
        for (int i = threadIdx.x; i < Lay::kSlabRecords * RB / 16; i += blockDim.x)
          tws[i] = src[i];
        __syncthreads();
      }
      const int k = units > g ? (units - g + G - 1) / G : 0;  // this group's tiles
      auto item_b = [&](int i) { return int(PAIR * ((w0 + g + (long long)G * i) / HPB)); };
      auto item_hf = [&](int i) { return int((w0 + g + (long long)G * i) % HPB); };
      auto load_item = [&](int i) {
        issue_load(q, rb, item_hf(i), item_b(i), int((it + i) % S));
        const int ip = i + p.prefetch * S;
        if (p.prefetch && ip < k) prefetch_load(q, rb, item_hf(ip), item_b(ip));
      };
      if (leader)
        for (int i = 0; i < S && i < k; ++i) load_item(i);
      for (int i = 0; i < k; ++i) {
        const int b = item_b(i);
        const int slot = int((it + i) % S);
        ptx::mbar_wait(&bars[slot], uint32_t(((it + i) / S) & 1));
        tile(q, rb, item_hf(i), b, PAIR == 2 && b + 1 < nb,
             ptx::smem_u32(bufs + size_t(slot) * Lay::kBufBytes), [&] {
               if (leader && i + S < k) load_item(i + S);
             });
      }
      it += k;
    }
  }
}

// ---- host side ---------------------------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

namespace {

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeFn(nullptr);
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

std::vector<int> split_passes(int m, int max_s, bool fp32) {
  // DSFFT_MP_SPLIT="a,b[,c]" overrides (tuning; ignored unless every group is
  // 6..max_s passes and they sum to m)
  if (const char* env = std::getenv("DSFFT_MP_SPLIT")) {
    std::vector<int> v;
    int sum = 0;
    bool ok = true;
    for (const char* c = env; *c;) {
      const int s = std::atoi(c);
      ok = ok && s >= 6 && s <= max_s;
      v.push_back(s);
      sum += s;
      while (*c && *c != ',') ++c;
      if (*c == ',') ++c;
    }
    if (ok && sum == m && v.size() >= 2) return v;
  }
  // 2 groups up to m = 2*max_s, 3 beyond; every group 6..max_s passes.
  // max_s = 10 for 8-byte values (fp32, fp16 pairs): s = 10 runs 16-column x
  // 1024-row tiles (128 KiB, one 512-thread group per CTA), so N = 2^19 and
  // 2^20 take two HBM round trips; s = 9 tiles (32 x 512, 128 KiB) likewise
  // fall back to one 1-deep group per CTA (m = 17, 18), which measured within
  // +-3% of the 3-group splits that smaller tiles would force.  One-word fp16
  // values keep max_s = 9.
  if (m <= 2 * max_s) {
    if (max_s < 10) {  // one-word fp16 values
      const int a = (m + 1) / 2;
      return {a, m - a};
    }
    // 8-byte values: the larger group last (the first group reads the user's
    // rows, the last the blocked intermediate), except where the B200 sweep
    // (profiles/r02_fused_multipass.md, "pass-group splits") measured the
    // other way: m = 19 as 10 + 9 (fp16 +2% since its s = 10 first group
    // loads evict_normal; fp32 with that group on 8-column tiles) and fp32
    // m = 18 as 10 + 8 (+7% over 8 + 10, +18% over 9 + 9)
    const int a = m == 19 || (fp32 && m == 18) ? 10 : m / 2;
    return {a, m - a};
  }
  const int a = (m + 2) / 3, b = (m - a + 1) / 2;
  return {a, b, m - a - b};
}

size_t sample_bytes(int precision) { return precision == kFp16 ? 4 : 8; }

}  // namespace

int env_or(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Input map of a pass group over `batch` transforms starting at `base`.
int make_in_map(CUtensorMap* map, const void* base, int m, int P, int s, int vb,
                long long batch, int box_cols) {
  EncodeFn enc = encode_fn();
  if (!enc) return -1;
  const CUtensorMapDataType dt =
      vb == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  const cuuint64_t N = cuuint64_t(1) << m;
  const cuuint32_t rows_box = cuuint32_t(std::min(1 << s, 256));
  // 128-B promotion: a box row narrower than a line (16 fp16 columns = 64 B)
  // still fetches the whole line; the neighbouring tile, loaded evict_normal
  // (MpParams::keep_l2), then finds its half in L2
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r;
  if (P == 0) {  // {q (N/2^s), c (2^s), b}
    cuuint64_t dims[3] = {N >> s, cuuint64_t(1) << s, cuuint64_t(batch)};
    cuuint64_t strides[2] = {(N >> s) * vb, N * vb};
    cuuint32_t box[3] = {cuuint32_t(box_cols), rows_box, 1};
    r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (P + s == m) {  // last group: blocked intermediate {r_l, c, rb, b}
    cuuint64_t dims[4] = {32, cuuint64_t(1) << s, N >> (s + 5), cuuint64_t(batch)};
    cuuint64_t strides[3] = {32 * cuuint64_t(vb), (cuuint64_t(32) << s) * vb, N * vb};
    cuuint32_t box[4] = {cuuint32_t(box_cols), rows_box, 1, 1};
    r = enc(map, dt, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {  // {r (2^P), q (N/2^(P+s)), c (2^s), b}
    cuuint64_t dims[4] = {cuuint64_t(1) << P, N >> (P + s), cuuint64_t(1) << s,
                          cuuint64_t(batch)};
    cuuint64_t strides[3] = {(cuuint64_t(1) << P) * vb, (N >> s) * vb, N * vb};
    cuuint32_t box[4] = {cuuint32_t(box_cols), 1, rows_box, 1};
    r = enc(map, dt, 4, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return int(r);
}


namespace {

template <int S1, class A, bool STD, int CW>
cudaError_t mp_launch_t(const CUtensorMap& map, const MpParams& p, bool first, bool conj_in,
                        bool scale_out, bool last, bool bout, int sm_count, size_t smem_optin,
                        cudaStream_t st) {
  using Lay = MpLayout<S1, A, CW>;
  MpParams q = p;
  // ring depth S and tile groups per CTA G (later groups share one
  // column-block slab between their G groups; <= 512 threads).  Default: as
  // many independent groups as 512 threads hold (two 32-column groups, four
  // 16-column ones), giving up ring depth before groups when shared memory is
  // short -- two 1-deep groups beat one 2-deep group by 0-3% (B200 sweep).
  const char* es = std::getenv("DSFFT_MP_STAGES");
  const char* eg = std::getenv("DSFFT_MP_GROUPS");
  // 8-column tiles: one 2-deep group measured ahead of two 1-deep ones
  int stages = es && *es ? std::max(1, std::atoi(es)) : 2;
  int groups = eg && *eg ? std::max(1, std::atoi(eg)) : CW == 8 ? 1 : 512 / Lay::T;
  groups = std::min(groups, std::max(1, 512 / Lay::T));
  while (stages > 1 && Lay::smem_bytes(first, stages, groups) > smem_optin) --stages;
  while (groups > 1 && Lay::smem_bytes(first, stages, groups) > smem_optin) --groups;
  q.stages = stages;
  const size_t smem = Lay::smem_bytes(first, stages, groups);
  const int threads = groups * Lay::T;
  const int regs = A::kWords == 1 ? 80 : 128;
  const int per_sm = std::max(1, int(std::min<size_t>(
                                     {smem_optin / smem, size_t(2048 / threads),
                                      size_t(65536 / (threads * regs))})));
  const int grid = int(std::min<long long>((p.tiles + groups - 1) / groups,
                                           (long long)sm_count * per_sm));
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(map, q);
    return cudaGetLastError();
  };
  // the group before the last writes the blocked intermediate (bout)
  if (first && bout)  // never last: every split has >= 2 groups
    return conj_in ? go(mp_kernel<S1, A, STD, true, true, false, false, true, CW>)
                   : go(mp_kernel<S1, A, STD, true, false, false, false, true, CW>);
  if (first)
    return conj_in ? go(mp_kernel<S1, A, STD, true, true, false, false, false, CW>)
                   : go(mp_kernel<S1, A, STD, true, false, false, false, false, CW>);
  if (last)
    return scale_out ? go(mp_kernel<S1, A, STD, false, false, true, true, false, CW>)
                     : go(mp_kernel<S1, A, STD, false, false, false, true, false, CW>);
  return go(mp_kernel<S1, A, STD, false, false, false, false, true, CW>);  // middle of 3
}

// cw: columns per tile; 16-column tiles exist for two-word values (fp32, fp16
// pairs: 128-byte rows) at s >= 7
template <class A, bool STD>
cudaError_t mp_launch_a(int S1, int cw, const CUtensorMap& map, const MpParams& p, bool first,
                        bool conj_in, bool scale_out, bool last, bool bout, int sm_count,
                        size_t optin, cudaStream_t st) {
#define DSFFT_MP_GO(S, C) \
  mp_launch_t<S, A, STD, C>(map, p, first, conj_in, scale_out, last, bout, sm_count, optin, st)
  if constexpr (A::kWords == 2) {
    if (cw == 8 && S1 == 5) return DSFFT_MP_GO(5, 8);  // s = 10: 8 x 1024 tiles (64 KB)
    if (cw == 16) {
      switch (S1) {
        case 2: return DSFFT_MP_GO(2, 16);
        case 3: return DSFFT_MP_GO(3, 16);
        case 4: return DSFFT_MP_GO(4, 16);
        case 5: return DSFFT_MP_GO(5, 16);  // s = 10: 16 x 1024 tiles (128 KB)
      }
    }
  }
  switch (S1) {
    case 1: return DSFFT_MP_GO(1, 32);
    case 2: return DSFFT_MP_GO(2, 32);
    case 3: return DSFFT_MP_GO(3, 32);
    case 4: return DSFFT_MP_GO(4, 32);
  }
#undef DSFFT_MP_GO
  return cudaErrorInvalidValue;
}

}  // namespace

MultipassPlan* multipass_create(const std::vector<TableEntry>& table, int m, int strategy,
                                int precision, int sm_count, size_t smem_optin) {
  if (!encode_fn()) {
    g_mp_err = "multipass: cuTensorMapEncodeTiled unavailable";
    return nullptr;
  }
  auto* mp = new MultipassPlan();
  mp->m = m;
  mp->strategy = strategy;
  mp->precision = precision;
  mp->sm_count = sm_count;
  mp->smem_optin = smem_optin;
  // fp16: transform pairs share every twiddle record and per-tile overhead
  // between two transforms (DSFFT_MP_F16_LAYOUT=2 selects one complex/register)
  const char* lay = std::getenv("DSFFT_MP_F16_LAYOUT");
  mp->f16_pairs = !(lay && std::atoi(lay) == 2);
  const bool f16c = precision == kFp16 && !mp->f16_pairs;
  // one launch, L2-resident intermediate (multipass_fused.cu): m = 2s with s
  // in 7..9 (N = 2^14, 2^16, 2^18), two-word values (fp32, fp16 transform
  // pairs).  It moves 1.01x the algorithmic DRAM bytes (vs 2x) but, with two
  // 256-thread tile groups per SM (128 registers, ~200 KB smem), is bound by
  // SM latency; it is the default only where the B200 A/B measured it faster
  // (profiles/r02_fused_multipass.md): fp16 N = 2^14 (+0.6%), 2^16 (+3.9%)
  // and fp32 N = 2^14 (+11%), for the 6-FMA variants: the 10-op standard
  // butterfly makes the SM-bound fused kernel slower (fp16 2^14: 35% vs 42% of
  // the roofline).  DSFFT_MP_FUSED=1 / 0 forces it on / off.
  const bool fused_ok = !f16c && m % 2 == 0 && m >= 14 && m <= 18;
  const bool fused_auto = strategy != kStandard &&
                          (precision == kFp16 ? (m == 14 || m == 16) : m == 14);
  const int fused_env = env_or("DSFFT_MP_FUSED", -1);
  mp->fused = fused_ok && (fused_env < 0 ? fused_auto : fused_env != 0);
  auto rec = [&](long long k) { return pack_record(table[k], strategy, precision, f16c); };
  int P = 0;
  // two-word values (fp32, fp16 pairs) take s = 10 groups as 16-column tiles,
  // so N = 2^19, 2^20 need two HBM round trips instead of three
  const int max_s = f16c ? 9 : 10;
  const std::vector<int> split =
      mp->fused ? std::vector<int>{m / 2, m / 2} : split_passes(m, max_s, precision == kFp32);
  for (int s : split) {
    MpGroup g;
    g.P = P;
    g.s = s;
    const int S1 = s - 5;
    std::vector<Record> recs;
    if (P == 0) {
      recs.resize(mp_first_records(S1));
      for (int pl = 0; pl < 5; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          recs[(1 << pl) - 1 + rl] = rec((long long)rl << (m - pl - 1));
      for (int pl = 0; pl < S1; ++pl)
        for (int rl = 0; rl < (1 << pl); ++rl)
          for (int r_l = 0; r_l < 32; ++r_l)
            recs[31 + (((1 << pl) - 1 + rl) << 5) + r_l] =
                rec((r_l + 32LL * rl) << (m - 5 - pl - 1));
    } else {
      const long long blocks = (1LL << P) >> 5;
      const int per = mp_block_records(S1);
      recs.resize(size_t(blocks) * per);
      for (long long rb = 0; rb < blocks; ++rb)
        for (int lane = 0; lane < 32; ++lane) {
          const long long r = rb * 32 + lane;
          Record* blk = recs.data() + rb * per;
          for (int pl = 0; pl < 5; ++pl)
            for (int rl = 0; rl < (1 << pl); ++rl)
              blk[((1 << pl) - 1 + rl) * 32 + lane] =
                  rec((r + ((long long)rl << P)) << (m - P - pl - 1));
          for (int pl = 0; pl < S1; ++pl)
            for (int rl = 0; rl < (1 << pl); ++rl)
              for (int r_l = 0; r_l < 32; ++r_l) {
                const long long lf = r_l + 32LL * rl;  // local frequency
                blk[31 * 32 + ((((1 << pl) - 1 + rl) << 5) + r_l) * 32 + lane] =
                    rec((r + (lf << P)) << (m - P - 5 - pl - 1));
              }
        }
    }
    const std::vector<uint8_t> img = serialize_records(recs, record_bytes(precision, f16c));
    if (cudaMalloc(&g.d_tw, img.size()) != cudaSuccess ||
        cudaMemcpy(g.d_tw, img.data(), img.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
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
  const char* env = std::getenv("DSFFT_MP_CHUNK_MB");
  // measured on B200 (profiles/README.md): L2-sized 48 MiB chunks lose more to
  // per-launch ramp/tail than they gain from L2 residency; 1 GiB chunks win
  const size_t want = size_t(env && *env ? std::atoi(env) : 1024) << 20;
  mp->chunk_transforms = std::max<size_t>(1, want / tb);
  return mp;
}

void multipass_destroy(MultipassPlan* mp) { delete mp; }

int multipass_execute(MultipassPlan& mp, bool inverse, const void* in, void* out, size_t batch,
                      uint32_t scale, cudaStream_t stream, uint64_t* launches) {
  const int vb = int(sample_bytes(mp.precision));
  const size_t tb = (size_t(1) << mp.m) * vb;
  // columns per tile: 16 for s = 10 (a 32 x 1024 tile of 8-byte values would
  // not fit shared memory), or from s = 7 in every group (DSFFT_MP_CW=16) or
  // the groups of bit mask DSFFT_MP_CWMASK (tuning; no default gains > 1.5%,
  // profiles/r02_fused_multipass.md)
  const int cw_mask = env_or("DSFFT_MP_CW", 32) == 16 ? 7 : env_or("DSFFT_MP_CWMASK", 0);
  // s = 10 groups in the bit mask DSFFT_MP_CW10MASK take 8-column x 1024-row
  // tiles (64 KB, one 2-deep 256-thread group): default for the fp32 first
  // group, +11% at 2^19 and 2^20; fp16 (32-byte input rows, 32-byte unpacked
  // output runs) and later groups measured slower (profiles/r02_fused_multipass.md)
  const int cw10_mask = env_or("DSFFT_MP_CW10MASK", mp.precision == kFp32 ? 1 : 0);
  auto tile_cols = [&](int i) {
    const int s = mp.groups[i].s;
    if (s == 10) return (cw10_mask >> i) & 1 ? 8 : 16;
    return (((cw_mask >> i) & 1) && !(mp.precision == kFp16 && !mp.f16_pairs) &&
                       s >= 7)
               ? 16
               : 32;
  };
  const bool f16 = mp.precision == kFp16;
  const bool std_ = mp.strategy == kStandard;
  const int ng = int(mp.groups.size());
  if (mp.fused) {
    const int rc = fused_execute(mp, inverse, in, out, batch, scale, stream, launches);
    if (rc != kFusedUnfit) return rc;
  }
  // per-call, stream-ordered intermediates (plans may run on several streams)
  const size_t chunk = std::min(mp.chunk_transforms, batch);
  uint8_t* scratch[2] = {nullptr, nullptr};
  for (int i = 0; i < std::min(ng - 1, 2); ++i)
    // pair-packed fp16 intermediates hold whole pairs: round up to even
    if (scratch_alloc(reinterpret_cast<void**>(&scratch[i]), ((chunk + 1) & ~size_t(1)) * tb,
                      stream) !=
        cudaSuccess) {
      for (auto* sp : scratch) scratch_free(sp, stream);
      g_mp_err = "multipass: scratch allocation failed";
      return 1;
    }
  struct Release {
    uint8_t** s;
    cudaStream_t st;
    ~Release() {
      scratch_free(s[0], st);
      scratch_free(s[1], st);
    }
  } release{scratch, stream};
  // maps: the user input over the whole batch (chunk = coordinate offset) and
  // the scratch buffers
  std::vector<CUtensorMap> maps(ng);
  for (int i = 0; i < ng; ++i) {
    const void* base = i == 0 ? in : scratch[(i - 1) & 1];
    const long long nb = i == 0 ? (long long)batch : (long long)chunk;
    // groups after the first read pair-packed fp16 intermediates: 8-byte
    // elements, one map "batch" entry per transform pair
    const bool packed = i > 0 && f16 && mp.f16_pairs;
    const int rc = make_in_map(&maps[i], base, mp.m, mp.groups[i].P, mp.groups[i].s,
                               packed ? 8 : vb, packed ? (nb + 1) / 2 : nb,
                               tile_cols(i));
    if (rc != 0) {
      g_mp_err = "multipass: cuTensorMapEncodeTiled failed (CUresult " + std::to_string(rc) +
                 ", group " + std::to_string(i) + ", base " +
                 std::to_string(reinterpret_cast<uintptr_t>(base)) + ", batch " +
                 std::to_string(nb) + ")";
      return 1;
    }
  }
  for (size_t b0 = 0; b0 < batch; b0 += mp.chunk_transforms) {
    const size_t nb = std::min(mp.chunk_transforms, batch - b0);
    for (int i = 0; i < ng; ++i) {
      const MpGroup& g = mp.groups[i];
      MpParams p{};
      p.out = i == ng - 1 ? static_cast<uint8_t*>(out) + b0 * tb : scratch[i & 1];
      p.tw = g.d_tw;
      p.m = mp.m;
      p.P = g.P;
      p.nb = (long long)nb;
      p.b_off = i == 0 ? (long long)b0 : 0;
      p.tiles = (((1LL << mp.m) >> g.s) / tile_cols(i)) * (long long)nb;
      p.scale = scale;
      // first-group rows narrower than a 128-B line (fp16 s = 10: 16 x 4 B):
      // with evict_first the line's other half was evicted before the next
      // column block's tile read it -- 2x DRAM reads (ncu, 2^20 fp16); kept
      // evict_normal it hits L2: 1.12 -> 1.00 ms per 1 GiB step
      p.keep_l2 = env_or("DSFFT_MP_KEEP", i == 0 && tile_cols(i) * vb < 128);
      // later groups of s = 9 (and s = 10 for fp16 pairs) run 128 KB tiles
      // 1-deep: an L2 prefetch of the next tile, issued with this one's load,
      // hides part of its latency (+3-4% at 2^17 - 2^20).  First groups (user
      // input; 8-column / evict_normal loads) and fp32 s = 10 last groups
      // measured slower with it (profiles/r02_fused_multipass.md)
      const bool pf = i > 0 && (g.s == 9 || (g.s == 10 && f16 && mp.f16_pairs));
      p.prefetch = env_or("DSFFT_MP_PREFETCH",
                          (env_or("DSFFT_MP_PFMASK", pf ? 1 << i : 0) >> i) & 1);
      const bool first = i == 0, last = i == ng - 1;
      const int S1 = g.s - 5, cw = tile_cols(i);
      const bool ci = first && inverse, so = last && inverse, bo = i == ng - 2;
      const int sm = mp.sm_count;
      const size_t oi = mp.smem_optin;
      cudaError_t e;
      if (f16 && mp.f16_pairs)
        e = std_ ? mp_launch_a<ArithF16P, true>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream)
                 : mp_launch_a<ArithF16P, false>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream);
      else if (f16)
        e = std_ ? mp_launch_a<ArithF16C, true>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream)
                 : mp_launch_a<ArithF16C, false>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream);
      else
        e = std_ ? mp_launch_a<ArithF32, true>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream)
                 : mp_launch_a<ArithF32, false>(S1, cw, maps[i], p, first, ci, so, last, bo, sm, oi, stream);
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
