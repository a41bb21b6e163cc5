#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void k(float* out, int it, const float* ab) {
  float a = ab[0], b = ab[1];
  unsigned long long A = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  unsigned long long B = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) x[i] = ((unsigned long long)__float_as_uint(threadIdx.x + i) << 32) | __float_as_uint(threadIdx.x * 2.f + i);
  for (int i = 0; i < it; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = ffma2(x[j], A, B);
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)x[i]) + __uint_as_float((unsigned)(x[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() { return 0; }
