// Throughput of the scatter-add options for the j side of a pair-once force loop on sm_100a:
// shared-memory atomics (ATOMS.ADD int, CAS.128 float4 loop, float atomicAdd = CAS loop),
// plain shared RMW (LDS.128 + FADD + STS.128), and global reductions (REDG.F32, REDG.F32x4)
// into an L2-resident buffer.  Reports SM cycles per warp instruction (per 32 lane-ops).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__device__ __forceinline__ void cas128_add(float4* p, float4 d) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  float4 old = *p;
  for (;;) {
    const float4 nw = make_float4(old.x + d.x, old.y + d.y, old.z + d.z, old.w + d.w);
    unsigned long long olo, ohi;
    asm volatile("{ .reg .b128 c, s, d; mov.b128 c, {%2, %3}; mov.b128 s, {%4, %5}; atom.shared.cas.b128 d, [%6], c, s; mov.b128 {%0, %1}, d; }"
        : "=l"(olo), "=l"(ohi)
        : "l"(((unsigned long long)__float_as_uint(old.y) << 32) | __float_as_uint(old.x)),
          "l"(((unsigned long long)__float_as_uint(old.w) << 32) | __float_as_uint(old.z)),
          "l"(((unsigned long long)__float_as_uint(nw.y) << 32) | __float_as_uint(nw.x)),
          "l"(((unsigned long long)__float_as_uint(nw.w) << 32) | __float_as_uint(nw.z)), "r"(a)
        : "memory");
    const unsigned long long elo = ((unsigned long long)__float_as_uint(old.y) << 32) | __float_as_uint(old.x);
    const unsigned long long ehi = ((unsigned long long)__float_as_uint(old.w) << 32) | __float_as_uint(old.z);
    if (olo == elo && ohi == ehi) break;
    old = make_float4(__uint_as_float((unsigned)olo), __uint_as_float((unsigned)(olo >> 32)),
                      __uint_as_float((unsigned)ohi), __uint_as_float((unsigned)(ohi >> 32)));
  }
}

// mode 0 ATOMS.ADD int, 1 CAS.128 float4, 2 atomicAdd float smem, 3 plain LDS.128+STS.128 RMW,
// 4 REDG.F32, 5 REDG.F32x4, 6 LDS.128 only
__global__ void k(float4* g, int gmask, int iters, int mode) {
  extern __shared__ float4 t[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = make_float4(0, 0, 0, 0);
  __syncthreads();
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll 4
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = hsh((uint32_t)(i * 8 + u) * 977u + (blockIdx.x * blockDim.x + threadIdx.x) * 131u);
      const int idx = r & 4095;
      const float d = (float)(r & 7);
      if (mode == 0) atomicAdd(reinterpret_cast<int*>(t) + 4 * idx, (int)(r & 7));
      else if (mode == 1) cas128_add(&t[idx], make_float4(d, d, d, d));
      else if (mode == 2) atomicAdd(reinterpret_cast<float*>(t) + 4 * idx, d);
      else if (mode == 3) { float4 v = t[(idx & ~31) | (threadIdx.x & 31)]; v.x += d; v.y += d; v.z += d; v.w += d; t[(idx & ~31) | (threadIdx.x & 31)] = v; }
      else if (mode == 4) { float* p = reinterpret_cast<float*>(g + (r & gmask)); asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(d)); }
      else if (mode == 5) { float* p = reinterpret_cast<float*>(g + (r & gmask)); asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(d), "f"(d), "f"(d), "f"(d)); }
      else { const float4 v = t[idx]; acc += v.x + v.w; }
    }
  }
  if (acc == 12345.f) g[0].x = acc;
  __syncthreads();
  if (mode < 4 && threadIdx.x == 0) g[blockIdx.x].y = t[threadIdx.x].x;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4* g; const int gn = 1 << 18;  // 4 MB: L2-resident
  cudaMalloc(&g, sizeof(float4) * gn);
  cudaMemset(g, 0, sizeof(float4) * gn);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"atoms_add_s32", "atoms_cas128_f32x4", "atomicAdd_f32_smem", "lds128_sts128_rmw", "redg_f32", "redg_f32x4", "lds128"};
  for (int thr : {256, 512}) for (int mode = 0; mode < 7; ++mode) {
    const int iters = mode == 1 || mode == 2 ? 100 : 400, blocks = sms * (1024 / thr) * 2;
    k<<<blocks, thr, 65536>>>(g, gn - 1, iters, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0); k<<<blocks, thr, 65536>>>(g, gn - 1, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_ops = (double)blocks * (thr / 32) * iters * 8;
    const double cyc = ms * 1e-3 * 1.965e9 * sms;
    printf("{\"op\": \"%s\", \"threads\": %d, \"ms\": %.3f, \"sm_cycles_per_warp_op\": %.3f, \"lane_ops_per_sm_cycle\": %.3f, \"err\": \"%s\"}\n", names[mode], thr, ms, cyc / warp_ops, warp_ops * 32 / cyc, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
