// Micro-benchmark: DRAM efficiency of the multipass access pattern.
// A "tile" = SEG bytes from each of ROWS rows at stride ROWSTRIDE bytes of one
// transform (TBYTES), copied to a contiguous destination.  Compared against
// a plain contiguous copy of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sc stride_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int SEG>
__global__ void tile_copy(const uint4* __restrict__ in, uint4* __restrict__ out, long long tiles,
                          int rows, long long rowstride, long long tbytes, int qblocks, int order) {
  // one warp per tile-row pass; each lane moves 16 B, SEG/16 lanes per row
  constexpr int LPR = SEG / 16;            // lanes per row
  constexpr int RPW = 32 / LPR;            // rows per warp instruction
  const long long warps = (long long)gridDim.x * blockDim.x / 32;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  for (long long t = wid; t < tiles; t += warps) {
    long long b, q;
    if (order == 0) { q = t % qblocks; b = t / qblocks; } else { b = t % (tiles / qblocks); q = t / (tiles / qblocks); }
    const char* src = reinterpret_cast<const char*>(in) + b * tbytes + q * SEG;
    char* dst = reinterpret_cast<char*>(out) + t * (long long)rows * SEG;
    for (int r0 = 0; r0 < rows; r0 += RPW * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * RPW + lane / LPR;
        v[u] = __ldcs(reinterpret_cast<const uint4*>(src + r * rowstride + (lane % LPR) * 16));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * RPW + lane / LPR;
        __stcs(reinterpret_cast<uint4*>(dst + (long long)r * SEG + (lane % LPR) * 16), v[u]);
      }
    }
  }
}

__global__ void plain_copy(const uint4* __restrict__ in, uint4* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

template <typename T>
__global__ void copy_w(const T* __restrict__ in, T* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}
// 16-byte loads, W-byte stores (the loaded vector written as 16/W stores)
template <int W>
__global__ void copy_st(const uint4* __restrict__ in, char* __restrict__ out, long long n) {
  const long long nthr = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr) {
    const uint4 v = __ldcs(in + i);
    // lane-interleaved so each store instruction covers contiguous lines:
    // element j of thread t goes to (block base) + j * (32 * W) + lane * W
    const long long warp_base = (i - (threadIdx.x & 31)) * 16;
    const int lane = threadIdx.x & 31;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (W == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) __stcs(reinterpret_cast<unsigned*>(out + warp_base + j * 128 + lane * 4), w[j]);
    } else if constexpr (W == 8) {
#pragma unroll
      for (int j = 0; j < 2; ++j) __stcs(reinterpret_cast<uint2*>(out + warp_base + j * 256 + lane * 8), make_uint2(w[2*j], w[2*j+1]));
    } else {
      __stcs(reinterpret_cast<uint4*>(out + warp_base + lane * 16), v);
    }
  }
}

int main() {
  const long long bytes = 1LL << 30;
  uint4 *a, *b;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto&& f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return 2.0 * bytes / (ms / 10 * 1e-3) / 1e9;
  };
  printf("plain copy: %.0f GB/s\n", timeit([&] { plain_copy<<<sms * 8, 256>>>(a, b, bytes / 16); }));
  printf("copy 4-byte ld/st: %.0f GB/s\n", timeit([&] { copy_w<unsigned><<<sms * 8, 256>>>((const unsigned*)a, (unsigned*)b, bytes / 4); }));
  printf("copy 8-byte ld/st: %.0f GB/s\n", timeit([&] { copy_w<uint2><<<sms * 8, 256>>>((const uint2*)a, (uint2*)b, bytes / 8); }));
  for (int occ : {2, 4, 8}) {
    printf("16-B loads, 4-B stores, %d CTAs/SM: %.0f GB/s\n", occ, timeit([&] { copy_st<4><<<sms * occ, 256>>>(a, (char*)b, bytes / 16); }));
    printf("16-B loads, 8-B stores, %d CTAs/SM: %.0f GB/s\n", occ, timeit([&] { copy_st<8><<<sms * occ, 256>>>(a, (char*)b, bytes / 16); }));
    printf("16-B loads, 16-B stores, %d CTAs/SM: %.0f GB/s\n", occ, timeit([&] { copy_st<16><<<sms * occ, 256>>>(a, (char*)b, bytes / 16); }));
  }
  // N = 2^16 fp16 complex (4 B): transform 256 KB, 256 rows x 1 KB
  struct Case { long long tb; int rows; long long rs; };
  for (Case c : {Case{1 << 18, 256, 1024}, Case{1 << 15, 128, 256}, Case{1 << 22, 256, 16384}}) {
    for (int order = 0; order < 2; ++order) {
      const int qb128 = int(c.rs / 128), qb256 = int(c.rs / 256);
      const long long nt = bytes / c.tb;
      double g128 = timeit([&] { tile_copy<128><<<sms * 8, 256>>>(a, b, nt * qb128, c.rows, c.rs, c.tb, qb128, order); });
      double g256 = timeit([&] { tile_copy<256><<<sms * 8, 256>>>(a, b, nt * qb256, c.rows, c.rs, c.tb, qb256, order); });
      printf("transform %lld B, %d rows x %lld B, order %s: 128-B segments %.0f GB/s, 256-B %.0f GB/s\n",
             c.tb, c.rows, c.rs, order ? "block-major" : "transform-major", g128, g256);
    }
  }
  return 0;
}
