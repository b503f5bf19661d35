// Microbenchmark: per-step cycles of the one-lane greedy variants (not product code).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void loop_vmin(const uint4 *absent_g, int n, int reps, long long *cyc, int *out) {
  __shared__ uint4 am[256];
  __shared__ int chg[256];
  for (int i = threadIdx.x; i < n; i += blockDim.x) am[i] = absent_g[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t k[4] = {0x00010000u, 0x00030002u, 0x00050004u, 0x00070006u};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint4 a = am[0];
    for (int i = 0; i < n; ++i) {
      const uint4 a2 = am[(i + 1) & 255];
      const uint32_t t = __vminu2(__vminu2(k[0] | a.x, k[1] | a.y), __vminu2(k[2] | a.z, k[3] | a.w));
      const uint32_t best = min(t & 0xffffu, t >> 16);
      const uint32_t g = best & 7u;
      const uint32_t inc = 8u << ((g & 1u) << 4);
#pragma unroll
      for (int j = 0; j < 4; ++j) k[j] += (g >> 1) == (uint32_t)j ? inc : 0u;
      chg[i] = (int)g;
      a = a2;
    }
  }
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / ((long long)reps * n);
  out[0] = k[0] + k[1] + k[2] + k[3] + chg[n - 1];
}

// keys compared against the duplicated min; no scalar extraction of g on the chain
__global__ void loop_vmin2(const uint4 *absent_g, int n, int reps, long long *cyc, int *out) {
  __shared__ uint4 am[256];
  __shared__ int chg[256];
  for (int i = threadIdx.x; i < n; i += blockDim.x) am[i] = absent_g[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t k[4] = {0x00010000u, 0x00030002u, 0x00050004u, 0x00070006u};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint4 a = am[0];
    for (int i = 0; i < n; ++i) {
      const uint4 a2 = am[(i + 1) & 255];
      const uint32_t m0 = k[0] | a.x, m1 = k[1] | a.y, m2 = k[2] | a.z, m3 = k[3] | a.w;
      const uint32_t t = __vminu2(__vminu2(m0, m1), __vminu2(m2, m3));
      const uint32_t d = __vminu2(t, __byte_perm(t, 0, 0x1032));  // min in both halves
      k[0] += __vcmpeq2(m0, d) & 0x00080008u;
      k[1] += __vcmpeq2(m1, d) & 0x00080008u;
      k[2] += __vcmpeq2(m2, d) & 0x00080008u;
      k[3] += __vcmpeq2(m3, d) & 0x00080008u;
      chg[i] = (int)(d & 7u);
      a = a2;
    }
  }
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / ((long long)reps * n);
  out[0] = k[0] + k[1] + k[2] + k[3] + chg[n - 1];
}

// warp: lane g holds key_g; REDUX min
__global__ void loop_redux(const uint32_t *hostbits_g, int n, int reps, long long *cyc, int *out) {
  __shared__ uint32_t hb[256];
  __shared__ int chg[256];
  for (int i = threadIdx.x; i < n; i += blockDim.x) hb[i] = hostbits_g[i];
  __syncthreads();
  const int lane = threadIdx.x;
  uint32_t key = lane < 6 ? ((uint32_t)lane) : 0xffffffffu;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = 0; i < n; ++i) {
      const uint32_t drop = ((hb[i] >> lane) & 1u) ? 0u : 0xffffffffu;
      const uint32_t win = __reduce_min_sync(0xffffffffu, key | drop);
      key += (key == win) ? 32u : 0u;
      if (lane == 0) chg[i] = (int)(win & 31u);
    }
  }
  long long t1 = clock64();
  if (lane == 0) {
    cyc[0] = (t1 - t0) / ((long long)reps * n);
    out[0] = key + chg[n - 1];
  }
}

int main() {
  const int n = 68, reps = 100;
  std::vector<uint4> ab(256);
  std::vector<uint32_t> hbits(256);
  for (int i = 0; i < 256; ++i) {
    int a = i % 6, b = (i * 7 + 1) % 6;
    if (b == a) b = (a + 1) % 6;
    uint32_t f[4] = {0, 0, 0, 0};
    for (int g = 0; g < 8; ++g)
      if (g != a && g != b) f[g >> 1] |= 0xffffu << ((g & 1) * 16);
    ab[i] = make_uint4(f[0], f[1], f[2], f[3]);
    hbits[i] = (1u << a) | (1u << b);
  }
  uint4 *dab;
  uint32_t *dhb;
  long long *dc;
  int *dout;
  cudaMalloc(&dab, 256 * 16);
  cudaMalloc(&dhb, 256 * 4);
  cudaMalloc(&dc, 8);
  cudaMalloc(&dout, 4);
  cudaMemcpy(dab, ab.data(), 256 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dhb, hbits.data(), 256 * 4, cudaMemcpyHostToDevice);
  long long c;
  for (int w = 0; w < 2; ++w) {
    loop_vmin<<<1, 32>>>(dab, n, reps, dc, dout);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    if (w) printf("vmin one-lane: %lld cycles/step\n", c);
    loop_vmin2<<<1, 32>>>(dab, n, reps, dc, dout);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    if (w) printf("vmin2 (vcmpeq) one-lane: %lld cycles/step\n", c);
    loop_redux<<<1, 32>>>(dhb, n, reps, dc, dout);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    if (w) printf("warp redux: %lld cycles/step\n", c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
