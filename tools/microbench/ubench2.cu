// FFMA2 (packed fp32x2, sm_100a) issue rate and near-sorted shared-memory gathers.
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 pk(float lo, float hi) { return ((u64)__float_as_uint(hi) << 32) | __float_as_uint(lo); }
__global__ void k_ffma2(float* out, int it, const float* ab) {
  u64 A = pk(ab[0], ab[0]), B = pk(ab[1], ab[1]); u64 x[8];
  for (int i = 0; i < 8; ++i) x[i] = pk(threadIdx.x + i, threadIdx.x * 2.f + i);
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = ffma2(x[j], A, B);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)x[i]) + __uint_as_float((unsigned)(x[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mode 0: idx = step (broadcast); 1: step + lane (consecutive); 2: step + (hash(lane,step) & 15) (near-sorted, spread 16);
// 3: step + (lane>>1); 4: fully random in 1024
__global__ void k_lds(float* out, int iters, int mode) {
  __shared__ float4 t[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  int lane = threadIdx.x & 31;
  uint32_t st = threadIdx.x * 2654435761u + 12345u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      st = st * 1664525u + 1013904223u;
      int base = (i * 8 + k) & 1023;
      int idx;
      if (mode == 0) idx = base; else if (mode == 1) idx = base + lane; else if (mode == 2) idx = base + (st >> 28);
      else if (mode == 3) idx = base + (lane >> 1); else idx = st >> 22;
      float4 v = t[idx];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 64 * 1024);
  float* ab; cudaMalloc(&ab, 8); float hab[2] = {0.999f, 0.001f}; cudaMemcpy(ab, hab, 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, thr = 256;
  auto timeit = [&](auto launch, double ops, const char* name) {
    launch(); cudaDeviceSynchronize(); float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"rate\": %.4e, \"per_sm_per_clk_at_max\": %.3f}\n", name, best, ops / (best * 1e-3), ops / (best * 1e-3) / sms / 1965e6);
  };
  timeit([&] { k_ffma2<<<blocks, thr>>>(out, 4096, ab); }, 4.0 * blocks * thr * 4096 * 128, "ffma2_flops");
  const char* nm[5] = {"lds_bcast", "lds_consec", "lds_near16", "lds_pairs", "lds_random"};
  for (int m = 0; m < 5; ++m) timeit([&] { k_lds<<<blocks, thr>>>(out, 2048, m); }, 1.0 * blocks * thr * 2048 * 8, nm[m]);
  return 0;
}
