// Micro-benchmarks of the sm_100a pipes the SPH interaction loops lean on:
// FFMA issue rate (the FP32 roofline denominator), MUFU rsqrt, I2F, shared-memory
// 128-bit gathers (broadcast vs random), shared-memory float atomics, and L1 gathers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ffma_reg(float* out, int iters, const float* ab) {
  // three-register form: multiplier/addend not compile-time immediates
  float a = ab[0], b = ab[1];
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_rsqrt(float* out, int iters) {
  float x0 = threadIdx.x + 1, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { x0 = rsqrtf(x0); x1 = rsqrtf(x1); x2 = rsqrtf(x2); x3 = rsqrtf(x3); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

__global__ void k_i2f(float* out, int iters) {
  int a0 = threadIdx.x, a1 = a0 + 7, a2 = a0 + 13, a3 = a0 + 17;
  float s = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      s += (float)a0 + (float)a1 + (float)a2 + (float)a3;
      a0 += 3; a1 += 5; a2 += 7; a3 += 11;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// shared-memory float4 gathers: mode 0 broadcast (all lanes same index), 1 random in 1024 entries
__global__ void k_lds(float* out, int iters, int mode) {
  __shared__ float4 t[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) t[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  uint32_t st = threadIdx.x * 2654435761u + 12345u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      st = st * 1664525u + 1013904223u;
      uint32_t idx = mode == 0 ? (uint32_t)(i * 8 + k) & 1023u : (st >> 22);
      float4 v = t[idx];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void k_atoms(float* out, int iters, int mode) {
  __shared__ float t[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = 0.f;
  __syncthreads();
  uint32_t st = threadIdx.x * 2654435761u + 12345u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      st = st * 1664525u + 1013904223u;
      uint32_t idx = mode == 0 ? threadIdx.x : (st >> 20);
      atomicAdd(&t[idx], 1.0f);
    }
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = t[threadIdx.x];
}

// global float4 gathers from a small (L1-resident) table, random lanes
__global__ void k_ldg(const float4* __restrict__ tab, float* out, int iters) {
  uint32_t st = threadIdx.x * 2654435761u + 12345u + blockIdx.x;
  float4 acc = make_float4(0, 0, 0, 0);
  const float4* base = tab + (blockIdx.x % 64) * 1024;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      st = st * 1664525u + 1013904223u;
      float4 v = __ldg(base + (st >> 22));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, clk);
  float* out; CK(cudaMalloc(&out, sizeof(float) * sms * 64 * 1024));
  float4* tab; CK(cudaMalloc(&tab, sizeof(float4) * 64 * 1024)); CK(cudaMemset(tab, 0, sizeof(float4) * 64 * 1024));
  float* ab; CK(cudaMalloc(&ab, 8)); float hab[2] = {0.999f, 0.001f}; CK(cudaMemcpy(ab, hab, 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, thr = 256;
  auto timeit = [&](auto launch, double ops, const char* name, const char* unit) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double rate = ops / (best * 1e-3);
    printf("{\"bench\": \"%s\", \"ms\": %.4f, \"rate\": %.4e, \"unit\": \"%s\", \"per_sm_per_clk_at_max\": %.3f}\n",
           name, best, rate, unit, rate / sms / (1965e6));
    fflush(stdout);
  };
  int it = 4096;
  timeit([&] { k_ffma<<<blocks, thr>>>(out, it, 0.999f, 0.001f); }, 2.0 * blocks * thr * it * 128, "ffma_imm", "flop/s");
  timeit([&] { k_ffma_reg<<<blocks, thr>>>(out, it, ab); }, 2.0 * blocks * thr * it * 128, "ffma_reg", "flop/s");
  timeit([&] { k_rsqrt<<<blocks, thr>>>(out, 1024); }, 1.0 * blocks * thr * 1024 * 64, "mufu_rsqrt", "op/s");
  timeit([&] { k_i2f<<<blocks, thr>>>(out, 1024); }, 1.0 * blocks * thr * 1024 * 64, "i2f", "op/s");
  timeit([&] { k_lds<<<blocks, thr>>>(out, 2048, 0); }, 1.0 * blocks * thr * 2048 * 8, "lds128_bcast", "lane-loads/s");
  timeit([&] { k_lds<<<blocks, thr>>>(out, 2048, 1); }, 1.0 * blocks * thr * 2048 * 8, "lds128_random", "lane-loads/s");
  timeit([&] { k_atoms<<<blocks, thr>>>(out, 512, 0); }, 1.0 * blocks * thr * 512 * 8, "atoms_f32_distinct", "lane-ops/s");
  timeit([&] { k_atoms<<<blocks, thr>>>(out, 512, 1); }, 1.0 * blocks * thr * 512 * 8, "atoms_f32_random", "lane-ops/s");
  timeit([&] { k_ldg<<<blocks, thr>>>(tab, out, 2048); }, 1.0 * blocks * thr * 2048 * 8, "ldg128_l1_random", "lane-loads/s");
  return 0;
}
