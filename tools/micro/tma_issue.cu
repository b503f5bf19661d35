// Microbenchmark: TMA issue cost and per-SM TMA load throughput on B200.
// One CTA per SM; W warps issue 2-D bf16 box loads (64 cols x R rows, 128-B
// swizzle, the K4 token/weight box shape) into 12 smem slots, each slot with
// its own mbarrier; a round = 12 loads issued + all 12 waited.  Data is a 32 MB
// buffer each CTA walks with a stride (L2-resident after the first round, or
// DRAM-streamed with --stream: a 2 GB buffer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2512_13525_b200/csrc \
//        tma_issue.cu -o tma_issue -lcuda && ./tma_issue
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sm100.cuh"

using namespace janus::sm100;

constexpr int kSlots = 12;

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, uint64_t *bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(128, 1)
    tma_kernel(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows, int warps,
               int rounds, long long *out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kSlots * 16384);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = box_rows * 128;
  long long issue_cycles = 0, t_start = 0;
  int row = (blockIdx.x * 977 * box_rows) % (rows_total - box_rows);
  for (int r = 0; r < rounds; ++r) {
    if (r == 1) t_start = clock64();
    if (warp < warps) {
      const long long c0 = clock64();
      for (int s = warp; s < kSlots; s += warps) {
        if (lane == 0) {
          mbar_expect_tx(&bars[s], bytes);
          tma_load_2d(smem + s * 16384, &tm, &bars[s], 0, row + s * box_rows);
        }
        __syncwarp();
      }
      if (r > 0) issue_cycles += clock64() - c0;
    }
    for (int s = 0; s < kSlots; ++s) mbar_wait(&bars[s], r & 1);
    __syncthreads();
    row += kSlots * box_rows * 37;
    if (row + kSlots * box_rows >= rows_total) row = (row * 7) % (rows_total / 2);
  }
  const long long total = clock64() - t_start;
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = total;
    out[2 * blockIdx.x + 1] = issue_cycles;
  }
}

int main(int argc, char **argv) {
  const bool stream = argc > 1 && !strcmp(argv[1], "--stream");
  const size_t bytes = stream ? (2ull << 30) : (32ull << 20);
  const int rows_total = (int)(bytes / 128);
  void *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  long long *out;
  cudaMalloc(&out, 2 * sms * sizeof(long long));
  const int smem = kSlots * 16384 + 1024 + 256;
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 200;
  for (int box_rows : {128, 64, 16}) {
    CUtensorMap tm;
    if (!make_map(&tm, buf, rows_total, 64, box_rows)) {
      printf("map failed\n");
      return 1;
    }
    for (int warps : {1, 2, 4}) {
      for (int grid : {1, sms}) {
        tma_kernel<<<grid, 128, smem>>>(tm, rows_total, box_rows, warps, rounds, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        long long h[2 * 256];
        cudaMemcpy(h, out, 2 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double tot = 0, iss = 0;
        for (int i = 0; i < grid; ++i) {
          tot += h[2 * i];
          iss += h[2 * i + 1];
        }
        tot /= grid;
        iss /= grid;
        const double loads = (double)(rounds - 1) * kSlots;
        const double per_sm_gbs = loads * box_rows * 128 / (tot / (clk_khz * 1e3)) / 1e9;
        printf("{\"mode\": \"%s\", \"box_rows\": %d, \"warps\": %d, \"ctas\": %d, "
               "\"cycles_per_load\": %.1f, \"issue_cycles_per_load_per_warp\": %.1f, "
               "\"gbs_per_sm\": %.1f, \"gbs_total\": %.1f}\n",
               stream ? "dram" : "l2", box_rows, warps, grid, tot / loads,
               iss / (loads / warps), per_sm_gbs, per_sm_gbs * grid);
      }
    }
  }
  return 0;
}
