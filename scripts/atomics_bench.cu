// atomics_bench.cu -- ceiling of the traversal's unit operation on this GPU:
// random 4-byte global atomics (returning ATOMG and fire-and-forget REDG) and
// random 4-byte loads, over footprints from L2-resident to DRAM-resident.
// Used to derive the "alu"/L2-atomic roofline in DESIGN.md §6.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics_bench atomics_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: atomicOr returning (result consumed), 1: RED (atomicOr, result
// unused), 2: ld.relaxed.gpu load, 3: atomicOr returning, 32 lanes of a warp
// on 32 consecutive words of one random line (coalesced, like 32 sources
// sharing a state line)
template <int MODE>
__global__ void kern(uint32_t *buf, uint32_t mask, int iters, uint32_t *sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0, h = tid * 2654435761u + 12345u;
  for (int i = 0; i < iters; i += 4) {
    uint32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      h = hash32(h + k);
      uint32_t idx = h & mask;
      if (MODE == 3) idx = (__shfl_sync(0xffffffffu, h, 0) & mask & ~31u) | (threadIdx.x & 31);
      if (MODE == 0 || MODE == 3) r[k] = atomicOr(buf + idx, 1u << (h >> 27));
      else if (MODE == 1) { atomicOr(buf + idx, 1u << (h >> 27)); r[k] = 0; }
      else {
        uint32_t v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(buf + idx));
        r[k] = v;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += r[k];
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  size_t maxw = (size_t)1 << 30;  // 4 GiB
  uint32_t *buf, *sink;
  cudaMalloc(&buf, maxw * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 0, maxw * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[4] = {"atomicOr-ret", "red.or", "ld.relaxed", "atomicOr-ret-coalesced"};
  for (int mode = 0; mode < 4; ++mode) {
    for (size_t words = (size_t)1 << 18; words <= maxw; words <<= 2) {
      for (int bpsm : {8, 16}) {
        const int threads = 256, grid = sms * bpsm, iters = 256;
        auto run = [&]() {
          if (mode == 0) kern<0><<<grid, threads>>>(buf, (uint32_t)(words - 1), iters, sink);
          if (mode == 1) kern<1><<<grid, threads>>>(buf, (uint32_t)(words - 1), iters, sink);
          if (mode == 2) kern<2><<<grid, threads>>>(buf, (uint32_t)(words - 1), iters, sink);
          if (mode == 3) kern<3><<<grid, threads>>>(buf, (uint32_t)(words - 1), iters, sink);
        };
        run();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 5.0 * grid * threads * (double)iters;
        printf("%-24s footprint %8.1f MiB  blocks/SM %2d : %7.1f Gop/s  (%.2f ns/op/SM)\n", names[mode],
               words * 4.0 / (1 << 20), bpsm, ops / ms / 1e6, ms * 1e6 / (ops / sms));
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
