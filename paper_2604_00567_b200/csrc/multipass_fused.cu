// multipass_fused.cu -- N = 2^14, 2^16, 2^18 (m = 2 s): both pass groups of
// the regrouped Stockham FFT in ONE persistent launch, the intermediate kept
// in L2 (see the kernel comment).  HBM sees the input once and the output
// once, against twice each for the two-launch path in multipass.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "multipass_impl.cuh"
#include "stream_alloc.cuh"

namespace dsfft {

// ---- fused two-group kernel: one HBM round trip ------------------------------
// For m = 2s (N = 2^14, 2^16, 2^18) both pass groups run in ONE persistent
// launch and the intermediate never reaches HBM as a whole-batch array.
//
// Teams.  The first group of a transform has K = N/2^s/32 column blocks and
// the second K as well.  A team is K CTAs; member j owns column block j of
// BOTH groups, so it keeps the second group's twiddle slab for block j in
// shared memory for the whole launch (no per-unit restaging).  Units (fp16
// transform pairs / fp32 transforms) are dealt round robin to the teams;
// tile group g of every member takes the team's units g, g+G, g+2G, ...
//
// Per unit v: each member runs its first-group tile (TMA from the user
// input in HBM) and stores it, blocked and pair-packed, into scratch slot
// v mod R of its team, then publishes done[slot] += 1 (release).  D units
// later it runs its second-group tile of unit v: the TMA load is issued
// once done[slot] shows all K first-group tiles (acquire), reads the slot
// from L2 and frees it (freed[slot] += 1) as soon as it has landed.  A slot
// is rewritten only after all K members freed it.  The scratch is
// teams x R units (R = G (D + 2)): ~50 MB at 2^16, well inside the 126 MB L2,
// and it is rewritten every few units, so it stays resident: HBM sees the
// input once and the output once.
//
// Progress: every wait is on an item earlier in the same per-group sequence
// of another team member, and the launch is cooperative (all CTAs
// co-resident), so the earliest unfinished item can always run.
struct FusedParams {
  uint8_t* out;        // user output (batch base)
  uint8_t* mid;        // scratch: teams * R unit slots (blocked, pair-packed)
  const uint4* twA;    // first-group records (mp_first_records)
  const uint4* twB;    // second-group records, K column blocks of mp_block_records
  uint32_t* done;      // [teams * R] first-group tiles stored into the slot (monotonic)
  uint32_t* freed;     // [teams * R] second-group tiles that read the slot (monotonic)
  int m, s;            // log2 N = 2 s
  int K, teams, R, D;  // team size, teams, scratch slots per team, lag in units per group
  long long nb;        // transforms
  long long units;     // ceil(nb / PAIR)
  uint32_t scale;
};

template <int S1, class A, bool STANDARD, bool INVERSE>
__global__ void __launch_bounds__(512, 1)
    mp_fused_kernel(const __grid_constant__ CUtensorMap in_map,
                    const __grid_constant__ CUtensorMap mid_map, const FusedParams p) {
  using Lay = MpLayout<S1, A>;
  constexpr int L = Lay::L, T = Lay::T;
  constexpr int ROWS_BOX = L < 256 ? L : 256;
  constexpr int PAIR = A::kPair, EB = A::kSampleBytes, HALF = 32 * L * EB;
  constexpr int RB = A::kRecBytes;
  constexpr int twA_bytes = Lay::tw_bytes(true), twB_bytes = Lay::tw_bytes(false);
  constexpr long long kUnitScale = PAIR * EB;  // bytes per sample of one unit
  extern __shared__ __align__(128) uint8_t smem[];
  const int G = blockDim.x / T;
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int lane = t & 31, warp = t >> 5;
  const bool leader = t == 0;
  const int K = p.K, R = p.R, D = p.D;
  const int tau = blockIdx.x / K, j = blockIdx.x - (blockIdx.x / K) * K;
  const long long N = 1LL << p.m;
  const uint32_t twA_base = ptx::smem_u32(smem);
  const uint32_t twB_base = twA_base + twA_bytes;
  uint8_t* buf = smem + twA_bytes + twB_bytes + size_t(g) * Lay::kBufBytes;
  uint64_t* bar =
      reinterpret_cast<uint64_t*>(smem + twA_bytes + twB_bytes + size_t(G) * Lay::kBufBytes) + g;
  {  // both groups' twiddles, once per launch (member j = column block j)
    uint4* sa = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < (mp_first_records(S1) * RB + 15) / 16; i += blockDim.x)
      sa[i] = p.twA[i];
    const uint4* src = p.twB + (long long)j * mp_block_records(S1) * RB / 16;
    uint4* sb = reinterpret_cast<uint4*>(smem + twA_bytes);
    for (int i = threadIdx.x; i < Lay::kSlabRecords * RB / 16; i += blockDim.x) sb[i] = src[i];
  }
  if (leader) ptx::mbar_init(bar, 1);
  ptx::fence_mbar_init();
  __syncthreads();

  // this group's units: team-local v = g + G k, global u = tau + teams v
  const long long team_units = p.units > tau ? (p.units - tau + p.teams - 1) / p.teams : 0;
  const int nk = team_units > g ? int((team_units - g + G - 1) / G) : 0;
  const int ntiles = 2 * nk;
  const int a0 = nk < D ? nk : D;         // leading first-group tiles
  const int c2 = nk > D ? nk - D : 0;     // interleaved (A(k), B(k-D)) pairs
  // tile i of the sequence A(0..a0), [A(k), B(k-D)] for k in [D, nk), B(tail)
  auto tile_of = [&](int i, bool& is_b) -> int {
    if (i < a0) { is_b = false; return i; }
    const int i2 = i - a0;
    if (i2 < 2 * c2) { is_b = i2 & 1; return is_b ? i2 / 2 : D + i2 / 2; }
    is_b = true;
    return c2 + (i2 - 2 * c2);
  };
  auto unit_v = [&](int k) { return (long long)g + (long long)G * k; };
  uint64_t pol = 0;
  if (leader) pol = ptx::policy_evict_first();
  auto issue = [&](int i) {
    bool is_b;
    const long long v = unit_v(tile_of(i, is_b));
    ptx::mbar_arrive_expect_tx(bar, Lay::kTileBytes);
    if (!is_b) {  // first group: column block j of the unit's transform(s), from HBM
      const int b = int((tau + (long long)p.teams * v) * PAIR);
#pragma unroll
      for (int h = 0; h < PAIR; ++h)
#pragma unroll
        for (int r0 = 0; r0 < L; r0 += ROWS_BOX)
          ptx::tma_load_3d(buf + h * HALF + size_t(r0) * 32 * EB, &in_map, j * 32, r0, b + h, bar,
                           pol);
    } else {  // second group: block j of the team's scratch slot, from L2
      const int slot = int(v % R);
      ptx::wait_at_least(p.done + tau * R + slot, uint32_t(K) * uint32_t(v / R + 1));
      ptx::fence_proxy_async_global();  // generic-proxy stores -> TMA reads
#pragma unroll
      for (int r0 = 0; r0 < L; r0 += ROWS_BOX)
        ptx::tma_load_4d(buf + size_t(r0) * 32 * Lay::VB, &mid_map, 0, r0, j, tau * R + slot, bar,
                         pol);
    }
  };
  if (leader && ntiles > 0) issue(0);
  auto group_sync = [&]() {
    if (T == 32) __syncwarp(); else ptx::named_bar_sync(1 + g, T);
  };
  const uint32_t buf_s = ptx::smem_u32(buf);
  for (int i = 0; i < ntiles; ++i) {
    bool is_b;
    const int k = tile_of(i, is_b);
    const long long v = unit_v(k);
    const int slot = int(v % R);
    const long long b = (tau + (long long)p.teams * v) * PAIR;
    ptx::mbar_wait(bar, uint32_t(i & 1));
    // the next tile's load goes out as soon as this slot is free -- unless it
    // is the second-group tile of this very unit (only when a group has a
    // single unit), whose load must wait for this tile's own publish below
    bool next_b = false;
    const bool has_next = i + 1 < ntiles;
    const bool next_is_own = has_next && !is_b && tile_of(i + 1, next_b) == k && next_b;
    auto release = [&] {
      if (leader && has_next && !next_is_own) issue(i + 1);
    };
    if (!is_b) {
      uint32_t* done = p.done + tau * R + slot;
      const uint32_t* freed = p.freed + tau * R + slot;
      mp_tile<S1, A, STANDARD, true, INVERSE, false, false, true>(
          buf_s, twA_base, nullptr, p.scale, 0, N, j, 0, 0, true, g, warp, lane,
          [&] { return p.mid + (long long)(tau * R + slot) * N * kUnitScale; }, release,
          [&] {  // the slot's previous unit has been read by every member
            ptx::wait_at_least(freed, uint32_t(K) * uint32_t(v / R));
          });
      ptx::fence_proxy_async_global();
      group_sync();
      if (leader) {
        __threadfence();
        ptx::red_release_add(done, 1);
        if (next_is_own) issue(i + 1);
      }
    } else {
      // the tile has landed: its scratch lines are dead -- drop them from L2
      // without write-back, then (after the group barrier inside mp_tile)
      // free the slot for the unit R ahead
      const uint8_t* blk = p.mid + (long long)(tau * R + slot) * N * kUnitScale +
                           (long long)j * Lay::kTileBytes;
      for (int off = t * 128; off < Lay::kTileBytes; off += T * 128)
        ptx::discard_l2_line(blk + off);
      uint32_t* freed = p.freed + tau * R + slot;
      auto release_b = [&] {
        if (leader) {
          ptx::red_release_add(freed, 1);
          if (has_next) issue(i + 1);
        }
      };
      mp_tile<S1, A, STANDARD, false, false, INVERSE, true, false>(
          buf_s, twB_base, reinterpret_cast<const uint8_t*>(p.twB), p.scale, p.s, N, 0, j, 0,
          b + 1 < p.nb, g, warp, lane, [&] { return p.out + b * N * EB; }, release_b, [] {});
    }
  }
}

namespace {

// ---- fused launch -------------------------------------------------------------
struct FusedShape {
  int K = 0, teams = 0, R = 0, D = 0, G = 0;
  size_t smem = 0;
};

template <int S1, class A>
FusedShape fused_shape(int m, int sm_count, size_t smem_optin, long long units) {
  using Lay = MpLayout<S1, A>;
  FusedShape f;
  f.K = int((1LL << m) >> (5 + S1 + 5));  // column blocks per group (= 2^s / 32)
  const int gmax = std::max(1, 512 / Lay::T);
  f.G = std::min(gmax, std::max(1, env_or("DSFFT_FUSED_GROUPS", gmax)));
  auto smem_for = [&](int G) {
    return size_t(Lay::tw_bytes(true)) + size_t(Lay::tw_bytes(false)) +
           size_t(G) * (Lay::kBufBytes + 8);
  };
  while (f.G > 1 && smem_for(f.G) > smem_optin) --f.G;
  f.smem = smem_for(f.G);
  if (f.smem > smem_optin || f.K < 1 || f.K > sm_count) return FusedShape{};
  f.D = std::max(1, env_or("DSFFT_FUSED_LAG", 1));
  f.R = std::max(f.G * (f.D + 1), env_or("DSFFT_FUSED_SLOTS", f.G * (f.D + 2)));
  f.R = (f.R + f.G - 1) / f.G * f.G;  // groups own disjoint slots
  f.teams = int(std::min<long long>(sm_count / f.K, std::max(1LL, units)));
  f.teams = std::max(1, std::min(f.teams, env_or("DSFFT_FUSED_TEAMS", f.teams)));
  return f;
}

template <int S1, class A, bool STD>
cudaError_t fused_launch_t(const CUtensorMap& in_map, const CUtensorMap& mid_map,
                           const FusedParams& p, const FusedShape& f, bool inverse,
                           cudaStream_t st) {
  using Lay = MpLayout<S1, A>;
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(f.smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(f.teams * f.K));
    cfg.blockDim = dim3(unsigned(f.G * Lay::T));
    cfg.dynamicSmemBytes = f.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every team member co-resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, in_map, mid_map, p);
  };
  return inverse ? go(mp_fused_kernel<S1, A, STD, true>) : go(mp_fused_kernel<S1, A, STD, false>);
}

template <class A>
FusedShape fused_shape_a(int S1, int m, int sm, size_t optin, long long units) {
  switch (S1) {
    case 2: return fused_shape<2, A>(m, sm, optin, units);
    case 3: return fused_shape<3, A>(m, sm, optin, units);
    case 4: return fused_shape<4, A>(m, sm, optin, units);
  }
  return FusedShape{};
}

template <class A, bool STD>
cudaError_t fused_launch_a(int S1, const CUtensorMap& in_map, const CUtensorMap& mid_map,
                           const FusedParams& p, const FusedShape& f, bool inverse,
                           cudaStream_t st) {
  switch (S1) {
    case 2: return fused_launch_t<2, A, STD>(in_map, mid_map, p, f, inverse, st);
    case 3: return fused_launch_t<3, A, STD>(in_map, mid_map, p, f, inverse, st);
    case 4: return fused_launch_t<4, A, STD>(in_map, mid_map, p, f, inverse, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int fused_execute(MultipassPlan& mp, bool inverse, const void* in, void* out, size_t batch,
                  uint32_t scale, cudaStream_t stream, uint64_t* launches) {
  const bool f16 = mp.precision == kFp16;
  const bool std_ = mp.strategy == kStandard;
  const int s = mp.m / 2, S1 = s - 5;
  const long long units = f16 ? (long long)(batch + 1) / 2 : (long long)batch;
  // DSFFT_FUSED_SMS caps the SMs a team may span (tests the unfit fallback)
  const int sms = std::max(1, std::min(mp.sm_count, env_or("DSFFT_FUSED_SMS", mp.sm_count)));
  const FusedShape f = f16 ? fused_shape_a<ArithF16P>(S1, mp.m, sms, mp.smem_optin, units)
                           : fused_shape_a<ArithF32>(S1, mp.m, sms, mp.smem_optin, units);
  if (f.K == 0) return kFusedUnfit;
  const size_t unit_bytes = (size_t(1) << mp.m) * 8;  // pair-packed fp16 / one fp32 transform
  const size_t slots = size_t(f.teams) * f.R;
  const size_t flag_bytes = 2 * slots * sizeof(uint32_t);
  uint8_t* scratch = nullptr;
  if (scratch_alloc(reinterpret_cast<void**>(&scratch), slots * unit_bytes + flag_bytes,
                    stream) != cudaSuccess) {
    set_mp_error("multipass: scratch allocation failed");
    return 1;
  }
  struct Release {
    uint8_t* s;
    cudaStream_t st;
    ~Release() { scratch_free(s, st); }
  } release{scratch, stream};
  uint32_t* flags = reinterpret_cast<uint32_t*>(scratch + slots * unit_bytes);
  if (cudaMemsetAsync(flags, 0, flag_bytes, stream) != cudaSuccess) {
    set_mp_error("multipass: flag reset failed");
    return 1;
  }
  CUtensorMap in_map, mid_map;
  int rc = make_in_map(&in_map, in, mp.m, 0, s, f16 ? 4 : 8, (long long)batch);
  if (!rc) rc = make_in_map(&mid_map, scratch, mp.m, s, s, 8, (long long)slots);
  if (rc) {
    set_mp_error("multipass: cuTensorMapEncodeTiled failed (fused, CUresult " +
                 std::to_string(rc) + ")");
    return 1;
  }
  FusedParams p{};
  p.out = static_cast<uint8_t*>(out);
  p.mid = scratch;
  p.twA = mp.groups[0].d_tw;
  p.twB = mp.groups[1].d_tw;
  p.done = flags;
  p.freed = flags + slots;
  p.m = mp.m;
  p.s = s;
  p.K = f.K;
  p.teams = f.teams;
  p.R = f.R;
  p.D = f.D;
  p.nb = (long long)batch;
  p.units = units;
  p.scale = scale;
  cudaError_t e;
  if (f16)
    e = std_ ? fused_launch_a<ArithF16P, true>(S1, in_map, mid_map, p, f, inverse, stream)
             : fused_launch_a<ArithF16P, false>(S1, in_map, mid_map, p, f, inverse, stream);
  else
    e = std_ ? fused_launch_a<ArithF32, true>(S1, in_map, mid_map, p, f, inverse, stream)
             : fused_launch_a<ArithF32, false>(S1, in_map, mid_map, p, f, inverse, stream);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();  // not sticky: clear it for the two-launch path
    return kFusedUnfit;
  }
  if (e != cudaSuccess) {
    set_mp_error(std::string("mp_fused_kernel launch: ") + cudaGetErrorString(e));
    return 1;
  }
  if (launches) ++*launches;  // the fused kernel (plus a 2*slots*4-byte flag memset)
  return 0;
}

}  // namespace dsfft
