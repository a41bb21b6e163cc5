// Shared-memory LDS.128 gather conflict behaviour on sm_100a: which lane groups must hit
// distinct 16-byte bank groups for a conflict-free 4-wavefront warp access.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
// mode 0: random slot; 1: slot = 8*rand + (lane & 7)  (each quarter-warp distinct groups)
// 2: slot = 8*rand + (lane >> 2)  (groups distinct across the 8 lanes {q, q+4, ...})
// 3: slot = 8*rand + ((lane + lane/8) & 7) (quarter-warps distinct, rotated)
// 4: slot = 8*rand + 0 (all lanes same bank group, different rows)
// 5: broadcast within quarter: slot = 8*rand(quarter) + 0
__global__ void k(float* out, int iters, int mode) {
  extern __shared__ float4 t[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = hsh((uint32_t)(i * 8 + u) * 977u + threadIdx.x * 131u) & 511u;
      const uint32_t rq = hsh((uint32_t)(i * 8 + u) * 977u + (threadIdx.x >> 3) * 131u) & 511u;
      int idx;
      if (mode == 0) idx = hsh(r + 7) & 4095;
      else if (mode == 1) idx = 8 * r + (lane & 7);
      else if (mode == 2) idx = 8 * r + (lane >> 2);
      else if (mode == 3) idx = 8 * r + ((lane + (lane >> 3)) & 7);
      else if (mode == 4) idx = 8 * r;
      else idx = 8 * rq;
      const float4 v = t[idx];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, blocks = sms * 4, thr = 256;
  for (int mode = 0; mode < 6; ++mode) {
    k<<<blocks, thr, 65536>>>(out, iters, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<blocks, thr, 65536>>>(out, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_lds = (double)blocks * (thr / 32) * iters * 8;
    const double cyc = ms * 1e-3 * 1.965e9 * sms;  // SM-cycles at max clock
    printf("{\"mode\": %d, \"ms\": %.3f, \"sm_cycles_per_warp_lds128\": %.3f}\n", mode, ms, cyc / warp_lds);
  }
  return 0;
}
