// Micro-benchmark: the multipass kernel's data movement without arithmetic.
// Persistent CTAs; one thread issues TMA tensor loads of column tiles
// (32 columns x ROWS rows of 4-byte values from a [batch][ROWS][COLS] tensor,
// the first pass group's view of N = ROWS*COLS) into an S-deep ring; W warps
// copy each tile from shared memory to a contiguous output with STG and
// release the slot through an "empty" mbarrier.  Reports GB/s (read + write).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_ring tma_ring.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}

template <int ROWS>
__global__ void __launch_bounds__(1024) ring(const __grid_constant__ CUtensorMap in, uint32_t* out,
                                             int tiles, int cols, int S) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int TB = 32 * ROWS * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * TB);
  uint64_t* empty = full + S;
  const int nw = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], nw);
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int qb = cols / 32;
  const int per = (tiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
  const int k = max(0, t1 - t0);
  auto load = [&](int i) {
    const int t = t0 + i, b = t / qb, q = t % qb;
    mbar_expect(&full[i % S], TB);
    for (int r0 = 0; r0 < ROWS; r0 += 256)
      tma3(smem + (i % S) * TB + r0 * 128, &in, q * 32, r0, b, &full[i % S]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < S && i < k; ++i) load(i);
  for (int i = 0; i < k; ++i) {
    const int slot = i % S;
    mbar_wait(&full[slot], (i / S) & 1);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(smem + slot * TB);
    uint32_t* dst = out + size_t(t0 + i) * 32 * ROWS;
    for (int r = warp; r < ROWS; r += nw) __stcs(dst + r * 32 + lane, src[r * 32 + lane]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (threadIdx.x == 0 && i + S < k) {
      mbar_wait(&empty[slot], (i / S) & 1);
      load(i + S);
    }
  }
}

int main() {
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  Enc enc = reinterpret_cast<Enc>(fn);
  const size_t bytes = size_t(1) << 30;
  uint32_t *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ROWS = 256;
  for (int cols : {256, 1024, 64}) {  // N = 2^16, 2^18, 2^14 (fp16 complex = 4 B)
    const long long per_t = (long long)ROWS * cols;
    const long long batch = bytes / 4 / per_t;
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(ROWS), cuuint64_t(batch)};
    cuuint64_t str[2] = {cuuint64_t(cols) * 4, cuuint64_t(per_t) * 4};
    cuuint32_t box[3] = {32, 256, 1}, es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tiles = int(batch * (cols / 32));
    for (int S : {2, 3, 4, 6})
      for (int ctas : {1, 2, 3})
        for (int threads : {256, 512}) {
          const size_t sm = size_t(S) * 32 * ROWS * 4 + 16 * S;
          if (sm * ctas > 227 * 1024 || threads * ctas > 2048) continue;
          cudaFuncSetAttribute(ring<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
          auto run = [&] { ring<256><<<sms * ctas, threads, sm>>>(m, b, tiles, cols, S); };
          run();
          cudaDeviceSynchronize();
          cudaEventRecord(e0);
          for (int it = 0; it < 10; ++it) run();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const cudaError_t err = cudaGetLastError();
          printf("N=%6d S=%d ctas/SM=%d threads=%d: %6.0f GB/s %s\n", ROWS * cols, S, ctas, threads,
                 2.0 * bytes / (ms / 10 * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
        }
  }
  return 0;
}
