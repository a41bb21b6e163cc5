// sph_kernels.cu -- sm_100a kernels of the SPH interaction loops of arXiv 2505.14538
// (density + h iteration, gradient + ghost, force + CFL dt).
//
// Decomposition.  The cell grid (side >= (1+skin) max support radius H = gamma_k h) is
// cut into CTA blocks of KZ cells of one grid column.  A block's TILE is the particles of
// the 3x3 neighbour columns over its z range +-1 cell: 9 contiguous ranges of the
// cell-sorted arrays, staged into shared memory with positions converted from fixed point
// to f32 offsets from the block centre.
//
// Neighbour lists.  k_lists tests, once per cell rebuild (and again only if an h outgrows
// its list radius), every candidate of the union of the 27-cell stencils of a warp's 32
// particles (warp-uniform, broadcast shared-memory reads) and stores, per particle, the
// tile slots j with r_ij < (1 + skin) max(H_i, H_j) as uint16, padded to a multiple of 8
// with a sentinel slot.  The density passes, the gradient loop and the force loop then run
// the pair arithmetic over these lists only: every lane works on a real (or skin)
// neighbour, no candidate is re-tested (the paper's pair tasks test all particle pairs of
// two cells).  Skin entries and the sentinel contribute exactly zero (compact
// support); membership (neighbour counts, v_sig) is decided in f32 with a rigorous band
// and re-decided in fp64 inside it, so counts equal the definition exactly.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "sph_internal.cuh"

namespace sph {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNW = 4;              // warps per CTA
constexpr float kFar = 1.0e12f;     // sentinel position (tile coordinates)

struct Tile {
  int ix, iy, z0, z1, nzt, nct, ntile, ib, ie, g0;
  uint32_t ref[3];
};

// Block geometry + tile cell table.  s_gst[c] = first global particle of tile cell c,
// s_off[c] = its offset in the tile; c = col * nzt + zz, col = (dx+1)*3 + (dy+1),
// zz = z - z0 + 1.  Ends with __syncthreads().
__device__ void tile_setup(const DevGrid& g, int b, const int* __restrict__ cell_start, int* s_off, int* s_gst,
                           Tile& T) {
  int zb = b % g.nzb;
  int col = b / g.nzb;
  T.iy = col % g.ny;
  T.ix = col / g.ny;
  T.z0 = zb * g.KZ;
  T.z1 = min(g.nz, T.z0 + g.KZ);
  T.nzt = T.z1 - T.z0 + 2;
  T.nct = 9 * T.nzt;
  T.ref[0] = (uint32_t)((((unsigned long long)(2 * T.ix + 1)) << 31) / (unsigned long long)g.nx);
  T.ref[1] = (uint32_t)((((unsigned long long)(2 * T.iy + 1)) << 31) / (unsigned long long)g.ny);
  T.ref[2] = (uint32_t)((((unsigned long long)(T.z0 + T.z1)) << 31) / (unsigned long long)g.nz);
  for (int t = threadIdx.x; t < T.nct; t += blockDim.x) {
    int c = t / T.nzt, zz = t - c * T.nzt;
    int cx = T.ix + c / 3 - 1, cy = T.iy + c % 3 - 1, cz = T.z0 - 1 + zz;
    cx += (cx < 0) ? g.nx : 0;
    cx -= (cx >= g.nx) ? g.nx : 0;
    cy += (cy < 0) ? g.ny : 0;
    cy -= (cy >= g.ny) ? g.ny : 0;
    cz += (cz < 0) ? g.nz : 0;
    cz -= (cz >= g.nz) ? g.nz : 0;
    int cell = (cx * g.ny + cy) * g.nz + cz;
    int gs = __ldg(cell_start + cell);
    s_gst[t] = gs;
    s_off[t + 1] = __ldg(cell_start + cell + 1) - gs;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int lane = threadIdx.x, carry = 0;
    for (int base = 0; base < T.nct; base += 32) {
      int t = base + lane;
      int v = t < T.nct ? s_off[t + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
      }
      if (t < T.nct) s_off[t + 1] = carry + v;
      carry += __shfl_sync(kFull, v, 31);
    }
    if (lane == 0) s_off[0] = 0;
  }
  __syncthreads();
  T.ntile = s_off[T.nct];
  T.ib = s_off[4 * T.nzt + 1];
  T.ie = s_off[4 * T.nzt + T.nzt - 1];
  T.g0 = s_gst[4 * T.nzt + 1];  // the block's own cells are consecutive in the cell order
}

// tile slot -> global particle index (binary search over the cell table)
__device__ __forceinline__ int slot_global(const int* s_off, const int* s_gst, int nct, int t) {
  int lo = 0, hi = nct;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (s_off[mid] <= t) lo = mid; else hi = mid;
  }
  return s_gst[lo] + (t - s_off[lo]);
}

__device__ __forceinline__ float3 rel_pos(const DevGrid& g, const Tile& T, uint4 x) {
  return make_float3((float)(int)(x.x - T.ref[0]) * g.scale[0], (float)(int)(x.y - T.ref[1]) * g.scale[1],
                     (float)(int)(x.z - T.ref[2]) * g.scale[2]);
}

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// M4 cubic spline: w(q), dw/dq; exactly zero for q >= 2 (compact support).
__device__ __forceinline__ void m4(float q, float& w, float& dw) {
  float q2 = q * q;
  float w_in = fmaf(q2, fmaf(0.75f, q, -1.5f), 1.f);
  float dw_in = q * fmaf(2.25f, q, -3.f);
  float t = fmaxf(2.f - q, 0.f);
  float t2 = t * t;
  bool inner = q < 1.f;
  w = inner ? w_in : 0.25f * t2 * t;
  dw = inner ? dw_in : -0.75f * t2;
}
__device__ __forceinline__ float m4_dw(float q) {
  float dw_in = q * fmaf(2.25f, q, -3.f);
  float t = fmaxf(2.f - q, 0.f);
  return q < 1.f ? dw_in : -0.75f * t * t;
}

// fp64 fixed-point neighbour test, operation for operation the oracle's (oracle.c sep2):
// r^2 = (dx*dx + dy*dy) + dz*dz < H2 with dx = (double)(int32)(X_i - X_j) * (L * 2^-32).
__device__ __noinline__ bool exact_neighbour(const uint4* __restrict__ xh, int gi, int gj, double H2, double sx,
                                             double sy, double sz) {
  uint4 a = xh[gi], b = xh[gj];
  double dx = __dmul_rn((double)(int)(a.x - b.x), sx);
  double dy = __dmul_rn((double)(int)(a.y - b.y), sy);
  double dz = __dmul_rn((double)(int)(a.z - b.z), sz);
  double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return r2 < H2 && r2 > 0.0;
}

__device__ __forceinline__ double h2_exact(float h, float gamma_k) {
  double H = __dmul_rn((double)gamma_k, (double)h);
  return __dmul_rn(H, H);
}

// Iterate a particle's padded neighbour list in groups of 8 (one 16-byte load each).
template <class PairF>
__device__ __forceinline__ void for_list(const uint16_t* __restrict__ list, int cnt, PairF&& pair) {
  const int mx = warp_max(cnt);
  for (int k0 = 0; k0 < mx; k0 += 8) {
    if (k0 < cnt) {
      const uint4 e = __ldg(reinterpret_cast<const uint4*>(list + k0));
      pair((int)(e.x & 0xffffu));
      pair((int)(e.x >> 16));
      pair((int)(e.y & 0xffffu));
      pair((int)(e.y >> 16));
      pair((int)(e.z & 0xffffu));
      pair((int)(e.z >> 16));
      pair((int)(e.w & 0xffffu));
      pair((int)(e.w >> 16));
    }
  }
}

// ========================================================== neighbour lists ==========
// For every particle i of the block: all tile slots j != i with
// r_ij^2 < ((1 + skin) gamma_k max(h_i, h_j))^2, in tile order, padded to 8 with the
// sentinel slot tcap.  Superset of every loop's neighbour set while each h stays within
// (1 + skin) of its value here (checked by the density epilogue).
__global__ void __launch_bounds__(kNW * 32) k_lists(DevGrid g, DevPhys ph, DevState s,
                                                    const int* __restrict__ cell_start,
                                                    DevCounters* __restrict__ ctr) {
  __shared__ int s_off[kMaxTileCells + 1];
  __shared__ int s_gst[kMaxTileCells];
  extern __shared__ float4 smem4[];
  float4* T0 = smem4;  // x, y, z, ((1+skin) H)^2
  uint16_t* L = reinterpret_cast<uint16_t*>(smem4 + g.tcap + 1);
  Tile T;
  tile_setup(g, blockIdx.x, cell_start, s_off, s_gst, T);
  if (T.ntile > g.tcap) {
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);
    return;
  }
  const float Hfac = (1.f + g.skin) * ph.gamma_k;
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    uint4 x = __ldg(&s.xh[slot_global(s_off, s_gst, T.nct, t)]);
    float3 p = rel_pos(g, T, x);
    float Hs = Hfac * __uint_as_float(x.w);
    T0[t] = make_float4(p.x, p.y, p.z, Hs * Hs);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ni = T.ie - T.ib;
  uint16_t* lst = L + warp * g.lcap * 32 + lane;
  int over = 0;
  for (int c = warp; c * 32 < ni; c += kNW) {
    const int k = c * 32 + lane;
    const bool valid = k < ni;
    const int ti = T.ib + (valid ? k : c * 32);
    const int* o = s_off + 4 * T.nzt;
    int zz = 1;
    while (zz < T.nzt - 2 && o[zz + 1] <= ti) ++zz;
    const int zf = warp_min(valid ? zz : 1 << 30), zl = warp_max(valid ? zz : -1);
    float4 pi4 = T0[ti];
    if (!valid) pi4.x = kFar;  // no hits
    int cnt = 0;
    for (int col = 0; col < 9; ++col) {
      const int a = s_off[col * T.nzt + zf - 1], e = s_off[col * T.nzt + zl + 2];
#pragma unroll 4
      for (int t = a; t < e; ++t) {
        const float4 p = T0[t];
        const float dx = pi4.x - p.x, dy = pi4.y - p.y, dz = pi4.z - p.z;
        const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (r2 < fmaxf(pi4.w, p.w) && r2 > 0.f) {
          if (cnt < g.lcap) lst[cnt * 32] = (uint16_t)t;
          ++cnt;
        }
      }
    }
    const int cntp = (cnt + 7) & ~7;
    if (cntp > g.lcap) over = max(over, cntp);
    if (valid && cntp <= g.lcap) {
      for (int kk = cnt; kk < cntp; ++kk) lst[kk * 32] = (uint16_t)g.tcap;
      const int gi = T.g0 + k;
      uint4* dst = reinterpret_cast<uint4*>(s.nbr + (size_t)gi * g.lcap);
      for (int k8 = 0; k8 < cntp; k8 += 8) {
        uint4 v;
        v.x = (uint32_t)lst[(k8 + 0) * 32] | ((uint32_t)lst[(k8 + 1) * 32] << 16);
        v.y = (uint32_t)lst[(k8 + 2) * 32] | ((uint32_t)lst[(k8 + 3) * 32] << 16);
        v.z = (uint32_t)lst[(k8 + 4) * 32] | ((uint32_t)lst[(k8 + 5) * 32] << 16);
        v.w = (uint32_t)lst[(k8 + 6) * 32] | ((uint32_t)lst[(k8 + 7) * 32] << 16);
        dst[k8 >> 3] = v;
      }
      s.ncount[gi] = cntp;
      s.hbuild[gi] = sqrtf(pi4.w) / Hfac;
    }
    __syncwarp();
  }
  over = warp_max(over);
  if (lane == 0 && over) atomicMax(&ctr->list_overflow, over);
}

// ============================================================== density loop ==========
// Eqs. 2-6 with the Newton-Raphson h update of the ghost (R7) and the
// density finalize (Eq. 8, EoS, Balsara; R8, R14) fused into the epilogue.
// Accumulators per particle i (q = r/h_i, w = M4, self term added in the epilogue):
//   S0 = sum w, S1 = sum q w', R0 = sum m_j w, R1 = sum m_j q w',
//   Dv = sum m_j w'/r (v_ij . r_ij),  Cv = sum m_j w'/r (v_ij x r_ij),  N_i.
// Then nhat = S0/(pi h^3), dn/dh = -(3 S0 + S1)/(pi h^4), rho = R0/(pi h^3),
// drho/dh = -(3 R0 + R1)/(pi h^4), div = -Dv/(rho pi h^4), curl = Cv/(rho pi h^4),
// g = nhat h^3 - eta^3 = S0/pi - eta^3, h g' = -S1/pi.
__global__ void __launch_bounds__(kNW * 32) k_density(DevGrid g, DevPhys ph, DevState s,
                                                      const int* __restrict__ cell_start, int pass,
                                                      const uint8_t* __restrict__ blk_in, uint8_t* __restrict__ blk_out,
                                                      DevCounters* __restrict__ ctr) {
  if (pass > 0 && !blk_in[blockIdx.x]) return;
  __shared__ int s_off[kMaxTileCells + 1];
  __shared__ int s_gst[kMaxTileCells];
  __shared__ int s_ni;
  __shared__ unsigned long long s_pairs, s_final;
  __shared__ int s_unconv, s_active;
  extern __shared__ float4 smem4[];
  float4* T0 = smem4;                  // x, y, z, m
  float4* T1 = T0 + (g.tcap + 1);      // vx, vy, vz, h
  int* ilist = reinterpret_cast<int*>(T1 + (g.tcap + 1));
  Tile T;
  if (threadIdx.x == 0) { s_ni = 0; s_pairs = 0; s_final = 0; s_unconv = 0; s_active = 0; }
  tile_setup(g, blockIdx.x, cell_start, s_off, s_gst, T);
  if (T.ntile > g.tcap) {
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);
    return;
  }
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    int gi = slot_global(s_off, s_gst, T.nct, t);
    uint4 x = __ldg(&s.xh[gi]);
    float4 v = __ldg(&s.vm[gi]);
    float3 p = rel_pos(g, T, x);
    T0[t] = make_float4(p.x, p.y, p.z, v.w);
    T1[t] = make_float4(v.x, v.y, v.z, __uint_as_float(x.w));
  }
  if (threadIdx.x == 0) {
    T0[g.tcap] = make_float4(kFar, kFar, kFar, 0.f);
    T1[g.tcap] = make_float4(0.f, 0.f, 0.f, 1.f);
  }
  const int ni_all = T.ie - T.ib;
  if (pass == 0) {
    if (threadIdx.x == 0) s_ni = ni_all;
  } else {
    for (int k = threadIdx.x; k < ni_all; k += blockDim.x)
      if (s.active[T.g0 + k]) ilist[atomicAdd(&s_ni, 1)] = k;
  }
  __syncthreads();
  const int ni = s_ni;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float inv_pi = 1.f / kPi;
  unsigned long long npairs = 0, nfinal = 0;

  for (int c = warp; c * 32 < ni; c += kNW) {
    const int kk = c * 32 + lane;
    const bool valid = kk < ni;
    const int li = pass == 0 ? (valid ? kk : c * 32) : ilist[valid ? kk : c * 32];
    const int ti = T.ib + li, gi = T.g0 + li;
    const float4 pi4 = T0[ti];
    const float4 vi4 = T1[ti];
    const float h = vi4.w, hinv = 1.f / h;
    const float qband = g.eabs * hinv + 8e-6f;  // |q - 2| below this: decide in fp64
    const double H2e = h2_exact(h, ph.gamma_k);
    const int cnt = valid ? s.ncount[gi] : 0;
    float S0 = 0.f, S1 = 0.f, R0 = 0.f, R1 = 0.f, Dv = 0.f, Cx = 0.f, Cy = 0.f, Cz = 0.f;
    int nn = 0;
    for_list(s.nbr + (size_t)gi * g.lcap, cnt, [&](int j) {
      const float4 p = T0[j];
      const float4 q4 = T1[j];
      const float dx = pi4.x - p.x, dy = pi4.y - p.y, dz = pi4.z - p.z;
      const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      const float rinv = rsqrtf(r2);
      const float q = r2 * rinv * hinv;
      bool in = q < 2.f;
      if (fabsf(q - 2.f) < qband)
        in = exact_neighbour(s.xh, gi, slot_global(s_off, s_gst, T.nct, j), H2e, g.dscale[0], g.dscale[1],
                             g.dscale[2]);
      nn += in;
      float w, dw;
      m4(q, w, dw);
      const float qdw = q * dw;
      S0 += w;
      S1 += qdw;
      R0 = fmaf(p.w, w, R0);
      R1 = fmaf(p.w, qdw, R1);
      const float F = p.w * dw * rinv;
      const float ux = vi4.x - q4.x, uy = vi4.y - q4.y, uz = vi4.z - q4.z;
      Dv = fmaf(F, fmaf(uz, dz, fmaf(uy, dy, ux * dx)), Dv);
      Cx = fmaf(F, fmaf(uy, dz, -uz * dy), Cx);
      Cy = fmaf(F, fmaf(uz, dx, -ux * dz), Cy);
      Cz = fmaf(F, fmaf(ux, dy, -uy * dx), Cz);
    });
    npairs += (unsigned long long)nn;
    if (valid) {
      // ---- epilogue: self term, closure, Newton / finalize
      const float mi = pi4.w;
      const float S0t = S0 + 1.f, R0t = R0 + mi;  // self: w(0) = 1, q w'(0) = 0
      const float ih3 = inv_pi * hinv * hinv * hinv;
      const float nhat = S0t * ih3;
      const float dndh = -(3.f * S0t + S1) * ih3 * hinv;
      const float rho = R0t * ih3;
      const float drho = -(3.f * R0t + R1) * ih3 * hinv;
      const float gres = S0t * inv_pi - ph.eta3;
      const bool conv = (ph.h_max_iter == 0) || fabsf(gres) <= ph.h_tol * ph.eta3;
      int it = pass == 0 ? 0 : s.iters[gi];
      const bool give_up = !conv && it >= ph.h_max_iter;
      if (conv || give_up) {
        const float ih4 = ih3 * hinv / rho;
        s.dens[gi] = make_float4(rho, drho, nhat, dndh);
        const float div = -Dv * ih4;
        const float cx = Cx * ih4, cy = Cy * ih4, cz = Cz * ih4;
        s.dvc[gi] = make_float4(cx, cy, cz, div);
        s.count[gi] = nn;
        // finalize: Eq. 8 (n_a = 3), ideal gas, Balsara (R8, R14)
        const float Omega = 1.f + h / (3.f * rho) * drho;
        const float f = ph.fh_mode ? Omega : 1.f / Omega;
        const float u = s.u[gi];
        const float P = (ph.gamma_eos - 1.f) * rho * u;
        const float cs = sqrtf(ph.gamma_eos * P / rho);
        const float adiv = fabsf(div), acurl = sqrtf(cx * cx + cy * cy + cz * cz);
        const float den = adiv + acurl + 1e-4f * cs * hinv;
        const float Bal = den > 0.f ? adiv / den : 0.f;
        s.fin[gi] = make_float4(f, P, cs, Bal);
        s.gq[gi] = make_float4(cs, u, mi / rho, rho);
        s.active[gi] = 0;
        s.iters[gi] = conv ? it : -1;
        nfinal += (unsigned long long)nn;
        if (give_up) atomicAdd(&s_unconv, 1);
      } else {
        // Newton with bracket + bisection (R7); g is non-decreasing in h
        float lo = pass == 0 ? 0.f : s.hlo[gi];
        float hi = pass == 0 ? CUDART_INF_F : s.hhi[gi];
        if (gres > 0.f) hi = h; else lo = h;
        float hn = (S1 < 0.f) ? h * (1.f + (S0t - ph.pi_eta3) / S1) : (gres < 0.f ? 2.f * h : 0.5f * h);
        hn = fminf(fmaxf(hn, 0.5f * h), 2.f * h);
        if (hn <= lo || hn >= hi) hn = isinf(hi) ? 2.f * h : 0.5f * (lo + hi);
        s.hlo[gi] = lo;
        s.hhi[gi] = hi;
        s.iters[gi] = it + 1;
        s.active[gi] = 1;
        reinterpret_cast<unsigned int*>(&s.xh[gi])[3] = __float_as_uint(hn);
        s_active = 1;
        const float Hn = ph.gamma_k * hn * (1.f + g.skin);
        if (Hn > g.side_min) atomicExch(&ctr->h_exceeds, 1);
        if (hn > (1.f + g.skin) * s.hbuild[gi]) atomicExch(&ctr->list_stale, 1);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    npairs += __shfl_xor_sync(kFull, npairs, o);
    nfinal += __shfl_xor_sync(kFull, nfinal, o);
  }
  if (lane == 0) {
    if (npairs) atomicAdd(&s_pairs, npairs);
    if (nfinal) atomicAdd(&s_final, nfinal);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_pairs) atomicAdd(&ctr->pairs_all, s_pairs);  // all pairs of this pass (h iteration work)
    if (s_final) atomicAdd(&ctr->pairs, s_final);
    if (s_unconv) atomicAdd(&ctr->unconverged, s_unconv);
    if (s_active) { blk_out[blockIdx.x] = 1; atomicAdd(&ctr->active_next, 1); }
  }
}

// ============================================================= gradient loop ==========
// v_sig,i = max(2 c_i, max_j (c_i + c_j - beta mu_ij)) (Eqs. 10-11, R15) and the
// Brookshaw Laplacian lap u_i = 2 sum_j (m_j/rho_j)(u_i - u_j) dW/dr / r (R16), gathered
// over r_ij < H_i; the gradient ghost (alpha_v Eqs. 12-15, alpha_c Eqs. 21-24; R17-R21)
// runs in the epilogue and writes the force-loop records.
__global__ void __launch_bounds__(kNW * 32) k_gradient(DevGrid g, DevPhys ph, DevState s,
                                                       const int* __restrict__ cell_start, float dt, int first_step,
                                                       DevCounters* __restrict__ ctr) {
  __shared__ int s_off[kMaxTileCells + 1];
  __shared__ int s_gst[kMaxTileCells];
  __shared__ unsigned long long s_pairs;
  extern __shared__ float4 smem4[];
  float4* T0 = smem4;                               // x, y, z, u
  float4* T1 = T0 + (g.tcap + 1);                   // vx, vy, vz, c
  float* T2 = reinterpret_cast<float*>(T1 + (g.tcap + 1));  // m/rho
  Tile T;
  if (threadIdx.x == 0) s_pairs = 0;
  tile_setup(g, blockIdx.x, cell_start, s_off, s_gst, T);
  if (T.ntile > g.tcap) {
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);
    return;
  }
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    int gi = slot_global(s_off, s_gst, T.nct, t);
    uint4 x = __ldg(&s.xh[gi]);
    float4 v = __ldg(&s.vm[gi]);
    float4 q = __ldg(&s.gq[gi]);
    float3 p = rel_pos(g, T, x);
    T0[t] = make_float4(p.x, p.y, p.z, q.y);
    T1[t] = make_float4(v.x, v.y, v.z, q.x);
    T2[t] = q.z;
  }
  if (threadIdx.x == 0) {
    T0[g.tcap] = make_float4(kFar, kFar, kFar, 0.f);
    T1[g.tcap] = make_float4(0.f, 0.f, 0.f, 0.f);
    T2[g.tcap] = 0.f;
  }
  __syncthreads();
  const int ni = T.ie - T.ib;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long npairs = 0;

  for (int c = warp; c * 32 < ni; c += kNW) {
    const int kk = c * 32 + lane;
    const bool valid = kk < ni;
    const int li = valid ? kk : c * 32;
    const int ti = T.ib + li, gi = T.g0 + li;
    const float4 pi4 = T0[ti];
    const float4 vi4 = T1[ti];
    const float h = __uint_as_float(s.xh[gi].w), hinv = 1.f / h;
    const float qband = g.eabs * hinv + 8e-6f;
    const double H2e = h2_exact(h, ph.gamma_k);
    const float ci = vi4.w, ui = pi4.w;
    const int cnt = valid ? s.ncount[gi] : 0;
    float vmax = 2.f * ci, lap = 0.f;
    int nn = 0;
    for_list(s.nbr + (size_t)gi * g.lcap, cnt, [&](int j) {
      const float4 p = T0[j];
      const float4 q4 = T1[j];
      const float Vj = T2[j];
      const float dx = pi4.x - p.x, dy = pi4.y - p.y, dz = pi4.z - p.z;
      const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      const float rinv = rsqrtf(r2);
      const float q = r2 * rinv * hinv;
      bool in = q < 2.f;
      if (fabsf(q - 2.f) < qband)
        in = exact_neighbour(s.xh, gi, slot_global(s_off, s_gst, T.nct, j), H2e, g.dscale[0], g.dscale[1],
                             g.dscale[2]);
      nn += in;
      const float dw = m4_dw(q);
      const float vr = fmaf(vi4.z - q4.z, dz, fmaf(vi4.y - q4.y, dy, (vi4.x - q4.x) * dx));
      const float mu = fminf(vr, 0.f) * rinv;
      const float vs = fmaf(-ph.beta, mu, ci + q4.w);
      vmax = fmaxf(vmax, in ? vs : 0.f);
      lap = fmaf(Vj * (ui - p.w), dw * rinv, lap);
    });
    if (valid) {
      npairs += (unsigned long long)nn;
      const float lap_u = 2.f * lap * hinv * hinv * hinv * hinv / kPi;
      const float vsig = vmax;
      // gradient ghost (R17-R21)
      const float H = ph.gamma_k * h;
      const float4 dvc = s.dvc[gi];
      const float4 fin = s.fin[gi];
      const float div = dvc.w;
      float av = s.av[gi], ac = s.ac[gi];
      const float Ddot = first_step ? 0.f : (div - s.dprev[gi]) / dt;
      const float S = H * H * fmaxf(-Ddot, 0.f);
      const float den = vsig * vsig + S;
      const float aloc = den > 0.f ? ph.alpha_v_max * S / den : 0.f;
      if (av < aloc) av = aloc;
      else av = aloc + (av - aloc) * expf(-ph.ell * ci * dt / H);
      const float src = ui > 0.f ? ph.beta_c * H * lap_u / sqrtf(ui) : 0.f;
      const float dac = src - (ac - ph.alpha_c_min) * vsig / H;
      ac = ac + dt * dac;
      const float ceil_ = fmaxf(ph.alpha_c_min, ph.alpha_c_max * (1.f - av / ph.alpha_v_max));
      ac = fmaxf(fminf(ac, ceil_), ph.alpha_c_min);
      s.grad[gi] = make_float2(vsig, lap_u);
      s.av[gi] = av;
      s.ac[gi] = ac;
      s.dprev[gi] = div;
      const float rho = s.dens[gi].x;
      const float f = fin.x, P = fin.y;
      s.fr1[gi] = make_float4(P / (rho * rho), f * hinv * hinv * hinv * hinv / kPi, ci, rho);
      s.fr2[gi] = make_float4(P, P * ac, ui, av);
      s.fr3[gi] = make_float2(fin.w, hinv);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) npairs += __shfl_xor_sync(kFull, npairs, o);
  if (lane == 0 && npairs) atomicAdd(&s_pairs, npairs);
  __syncthreads();
  if (threadIdx.x == 0 && s_pairs) atomicAdd(&ctr->pairs, s_pairs);
}

// ================================================================ force loop ==========
// Gather form of the pairwise sums of Eqs. 7, 17-19 over r_ij < max(H_i, H_j) (R3):
//   G = f dW/dr / r, A = P/rho^2, Pi_ij = -abar mu v_sig / rhobar (R9), Gbar = (G_i+G_j)/2,
//   S_ij = A_i G_i + A_j G_j + Pi_ij Gbar,  a_i = -sum_j m_j S_ij r_ij,
//   du_i = sum_j m_j [A_i G_i v.r + Pi Gbar v.r / 2 + D_ij]  (Eq. 18 + R10 + Eq. 19/R11),
//   D_ij = alpha_c,ij v_c,ij (u_i - u_j)(G_i + G_j) r / (rho_i + rho_j)  (Eqs. 20, 22; R12, R13).
// S_ij is evaluated from operands that are symmetric in (i, j), so the pair terms of i and
// j are exact negatives (momentum and energy conserving up to the summation rounding).
// The CFL dt = C_cfl min 2 gamma_k h / v_sig is reduced in the epilogue.
__global__ void __launch_bounds__(kNW * 32) k_force(DevGrid g, DevPhys ph, DevState s,
                                                    const int* __restrict__ cell_start,
                                                    DevCounters* __restrict__ ctr) {
  __shared__ int s_off[kMaxTileCells + 1];
  __shared__ int s_gst[kMaxTileCells];
  __shared__ unsigned long long s_pairs;
  __shared__ unsigned int s_dt;
  __shared__ int s_bad;
  extern __shared__ float4 smem4[];
  float4* T0 = smem4;                      // x, y, z, B
  float4* T1 = T0 + (g.tcap + 1);          // vx, vy, vz, m
  float4* T2 = T1 + (g.tcap + 1);          // A, Kf, c, rho
  float4* T3 = T2 + (g.tcap + 1);          // P, P alpha_c, u, alpha_v
  float* T4 = reinterpret_cast<float*>(T3 + (g.tcap + 1));  // 1/h
  Tile T;
  if (threadIdx.x == 0) { s_pairs = 0; s_dt = 0x7f800000u; s_bad = 0; }
  tile_setup(g, blockIdx.x, cell_start, s_off, s_gst, T);
  if (T.ntile > g.tcap) {
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);
    return;
  }
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    int gi = slot_global(s_off, s_gst, T.nct, t);
    uint4 x = __ldg(&s.xh[gi]);
    float3 p = rel_pos(g, T, x);
    float2 b3 = __ldg(&s.fr3[gi]);
    T0[t] = make_float4(p.x, p.y, p.z, b3.x);
    T1[t] = __ldg(&s.vm[gi]);
    T2[t] = __ldg(&s.fr1[gi]);
    T3[t] = __ldg(&s.fr2[gi]);
    T4[t] = b3.y;
  }
  if (threadIdx.x == 0) {
    T0[g.tcap] = make_float4(kFar, kFar, kFar, 0.f);
    T1[g.tcap] = make_float4(0.f, 0.f, 0.f, 0.f);
    T2[g.tcap] = make_float4(0.f, 0.f, 0.f, 1.f);
    T3[g.tcap] = make_float4(0.f, 0.f, 0.f, 0.f);
    T4[g.tcap] = 1.f;
  }
  __syncthreads();
  const int ni = T.ie - T.ib;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long npairs = 0;
  float dtmin = CUDART_INF_F;

  for (int c = warp; c * 32 < ni; c += kNW) {
    const int kk = c * 32 + lane;
    const bool valid = kk < ni;
    const int li = valid ? kk : c * 32;
    const int ti = T.ib + li, gi = T.g0 + li;
    const float4 pi4 = T0[ti];
    const float4 vi4 = T1[ti];
    const float4 ai = T2[ti];
    const float4 bi = T3[ti];
    const float hinv_i = T4[ti];
    const float hi_ = __uint_as_float(s.xh[gi].w);
    const double H2ei = h2_exact(hi_, ph.gamma_k);
    const float eq = g.eabs;
    const int cnt = valid ? s.ncount[gi] : 0;
    float ax = 0.f, ay = 0.f, az = 0.f, du = 0.f, vmax = 2.f * ai.z;
    int nn = 0;
    for_list(s.nbr + (size_t)gi * g.lcap, cnt, [&](int j) {
      const float4 p = T0[j];
      const float dx = pi4.x - p.x, dy = pi4.y - p.y, dz = pi4.z - p.z;
      const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      const float4 vj = T1[j];
      const float4 aj = T2[j];
      const float4 bj = T3[j];
      const float hinv_j = T4[j];
      const float rinv = rsqrtf(r2);
      const float r = r2 * rinv;
      const float qi = r * hinv_i, qj = r * hinv_j;
      const float qm = fminf(qi, qj);
      bool in = qm < 2.f;
      if (fabsf(qm - 2.f) < eq * fmaxf(hinv_i, hinv_j) + 8e-6f) {
        const int gj = slot_global(s_off, s_gst, T.nct, j);
        const double H2ej = h2_exact(__uint_as_float(s.xh[gj].w), ph.gamma_k);
        in = exact_neighbour(s.xh, gi, gj, fmax(H2ei, H2ej), g.dscale[0], g.dscale[1], g.dscale[2]);
      }
      nn += in;
      const float Gi = ai.y * m4_dw(qi) * rinv;
      const float Gj = aj.y * m4_dw(qj) * rinv;
      const float vr = fmaf(vi4.z - vj.z, dz, fmaf(vi4.y - vj.y, dy, (vi4.x - vj.x) * dx));
      const float mu = fminf(vr, 0.f) * rinv;
      const float vs = fmaf(-ph.beta, mu, ai.z + aj.z);
      vmax = fmaxf(vmax, in ? vs : 0.f);
      const float abar = 0.25f * (bi.w + bj.w) * (pi4.w + p.w);
      const float irs = __frcp_rn(ai.w + aj.w);
      const float PiV = -2.f * abar * mu * vs * irs;
      const float Gbar = 0.5f * (Gi + Gj);
      const float Sij = fmaf(PiV, Gbar, fmaf(ai.x, Gi, aj.x * Gj));
      const float mS = vj.w * Sij;
      ax = fmaf(-mS, dx, ax);
      ay = fmaf(-mS, dy, ay);
      az = fmaf(-mS, dz, az);
      const float Psum = bi.x + bj.x;
      const float acij = Psum > 0.f ? (bi.y + bj.y) * __frcp_rn(Psum) : 0.f;
      const float vc = fabsf(vr) * rinv + sqrtf(2.f * fabsf(bi.x - bj.x) * irs);
      const float D = acij * vc * (bi.z - bj.z) * (Gi + Gj) * r * irs;
      du = fmaf(vj.w, fmaf(ai.x * Gi, vr, fmaf(0.5f * PiV * Gbar, vr, D)), du);
    });
    if (valid) {
      s.acc[gi] = make_float4(ax, ay, az, du);
      s.vsig[gi] = vmax;
      s.countf[gi] = nn;
      npairs += (unsigned long long)nn;
      const float dti = ph.c_cfl * 2.f * ph.gamma_k * hi_ / vmax;
      if (!(isfinite(vmax) && isfinite(ax) && isfinite(ay) && isfinite(az) && isfinite(du)) || !(dti > 0.f))
        s_bad = 1;
      dtmin = fminf(dtmin, dti);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    npairs += __shfl_xor_sync(kFull, npairs, o);
    dtmin = fminf(dtmin, __shfl_xor_sync(kFull, dtmin, o));
  }
  if (lane == 0) {
    if (npairs) atomicAdd(&s_pairs, npairs);
    if (dtmin < CUDART_INF_F && dtmin > 0.f) atomicMin(&s_dt, __float_as_uint(dtmin));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_pairs) atomicAdd(&ctr->pairs, s_pairs);
    if (s_dt != 0x7f800000u) atomicMin(&ctr->dt_bits, s_dt);
    if (s_bad) atomicExch(&ctr->nonfinite, 1);
  }
}

// per-block tile size (max over blocks) -> sizes shared memory of the loops
__global__ void k_tile_sizes(DevGrid g, const int* __restrict__ cell_start, int* max_tile) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nblocks) return;
  int zb = b % g.nzb, col = b / g.nzb, iy = col % g.ny, ix = col / g.ny;
  int z0 = zb * g.KZ, z1 = min(g.nz, z0 + g.KZ);
  int tot = 0;
  for (int c = 0; c < 9; ++c) {
    int cx = (ix + c / 3 - 1 + g.nx) % g.nx, cy = (iy + c % 3 - 1 + g.ny) % g.ny;
    for (int z = z0 - 1; z <= z1; ++z) {
      int cz = (z + g.nz) % g.nz;
      int cell = (cx * g.ny + cy) * g.nz + cz;
      tot += cell_start[cell + 1] - cell_start[cell];
    }
  }
  atomicMax(max_tile, tot);
}

}  // namespace

int kernel_threads() { return kNW * 32; }

size_t lists_smem(const DevGrid& g) { return (size_t)(g.tcap + 1) * 16 + (size_t)kNW * g.lcap * 32 * 2; }
size_t density_smem(const DevGrid& g) { return (size_t)(g.tcap + 1) * (2 * 16 + 4); }
size_t gradient_smem(const DevGrid& g) { return (size_t)(g.tcap + 1) * (2 * 16 + 4); }
size_t force_smem(const DevGrid& g) { return (size_t)(g.tcap + 1) * (4 * 16 + 4); }

cudaError_t launch_tile_sizes(const DevGrid& g, const int* cell_start, int* max_tile, cudaStream_t st) {
  k_tile_sizes<<<(g.nblocks + 255) / 256, 256, 0, st>>>(g, cell_start, max_tile);
  return cudaGetLastError();
}

static cudaError_t set_smem(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_lists(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st) {
  size_t sm = lists_smem(g);
  cudaError_t e = set_smem((const void*)k_lists, sm);
  if (e != cudaSuccess) return e;
  k_lists<<<g.nblocks, kNW * 32, sm, st>>>(g, ph, s, cell_start, ctr);
  return cudaGetLastError();
}

cudaError_t launch_density(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, int pass,
                           const uint8_t* blk_in, uint8_t* blk_out, DevCounters* ctr, cudaStream_t st) {
  size_t sm = density_smem(g);
  cudaError_t e = set_smem((const void*)k_density, sm);
  if (e != cudaSuccess) return e;
  k_density<<<g.nblocks, kNW * 32, sm, st>>>(g, ph, s, cell_start, pass, blk_in, blk_out, ctr);
  return cudaGetLastError();
}

cudaError_t launch_gradient(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, float dt,
                            int first_step, DevCounters* ctr, cudaStream_t st) {
  size_t sm = gradient_smem(g);
  cudaError_t e = set_smem((const void*)k_gradient, sm);
  if (e != cudaSuccess) return e;
  k_gradient<<<g.nblocks, kNW * 32, sm, st>>>(g, ph, s, cell_start, dt, first_step, ctr);
  return cudaGetLastError();
}

cudaError_t launch_force(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st) {
  size_t sm = force_smem(g);
  cudaError_t e = set_smem((const void*)k_force, sm);
  if (e != cudaSuccess) return e;
  k_force<<<g.nblocks, kNW * 32, sm, st>>>(g, ph, s, cell_start, ctr);
  return cudaGetLastError();
}

}  // namespace sph
