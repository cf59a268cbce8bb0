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
