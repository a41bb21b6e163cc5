// sph_wide.cu -- "wide" particles of the adaptive cell grid.
//
// A strong smoothing-length contrast (C3 Sedov: H from 0.63 to 5.6 H_0) makes a grid with
// side >= (1 + skin) gamma_k h_max hold thousands of particles per cell in the dense regions,
// far beyond what a shared-memory tile can stage.  The single-rank path then sizes the cells
// from a quantile of h instead (sph_api.cu rebuild()), and the few particles whose list
// radius (1 + skin) gamma_k h exceeds the side become WIDE:
//   - k_wide_lists: one warp per wide particle i scans the cells within +-k_a of its cell
//     (k_a = ceil(list radius / side_a) per axis) and lists, by global index, every j with
//     r_ij < (1 + skin) gamma_k max(h_i, h_j) -- the same criterion as the tile lists;
//   - k_wide_density / k_wide_gradient / k_wide_force: one warp per wide particle runs
//     the shared pair arithmetic (sph_pair.cuh) over its list, gathering the neighbour
//     records from global memory (L2), with the same epilogues as the tile loops;
//   - symmetry of the force set r < max(H_i, H_j) (R3): a partner j that did not list i
//     (a tile particle more than one cell away, or a wide particle whose own search range
//     stops short of i) gets its side of the pair from i, added with atomics (a, du/dt,
//     N_force) and atomicMax (v_sig); the CFL dt follows from the final v_sig (k_force_fin).
// The tile kernels skip wide particles as i (empty list, no epilogue) and see them as j like
// any other particle of their tile.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "sph_internal.cuh"
#include "sph_pair.cuh"

namespace sph {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int cell_axis(uint32_t x, int n) { return (int)(((unsigned long long)x * (unsigned)n) >> 32); }

// local x-plane of particle i: the plane its rank's binning put it in.  One rank: the periodic
// grid.  Slab path: owned particles on this slab's planes [G, G + nxo) (k_keys); the ghosts
// on their OWNER's planes (its last G planes -> [0, G), its first G -> [G + nxo, nx)), so the
// plane agrees with the ghost cell the particle was received into
// (PX: the grid is periodic along x, one rank; the kernels are instantiated for both cases so
// the single-rank build keeps its registers)
template <bool PX>
__device__ __forceinline__ int plane_of(const DevGrid& g, int i, uint32_t x) {
  if (PX) return cell_axis(x, g.nx);
  uint32_t lo = g.x_lo;
  unsigned long long w = g.wfix;
  int base = g.ix_first;
  if (i < g.gL) { lo = g.x_loL; w = g.wfixL; base = g.ix_first - g.nxo; }
  else if (i >= g.gL + g.n_own) { lo = g.x_loR; w = g.wfixR; base = g.ix_first + g.nxo; }
  const unsigned long long d = (unsigned long long)(uint32_t)(x - lo);
  const int p = (int)min((d * (unsigned long long)g.nxo) / w, (unsigned long long)(g.nxo - 1));
  return min(max(base + p, 0), g.nx - 1);
}

// search half-width in cells along each axis for a list radius R (capped to the whole axis)
__device__ __forceinline__ int reach(float R, float side, int n) {
  const int k = (int)ceilf(R / side);
  return min(k, (n - 1) / 2 + 1);
}

// cells i and j are within +-k of each other along an axis of n cells (periodic, or not: the
// slab path's local x planes)
__device__ __forceinline__ bool within(int a, int b, int k, int n, bool per = true) {
  int d = a - b;
  d = d < 0 ? -d : d;
  if (!per) return d <= k;
  if (2 * k + 1 >= n) return true;
  d = min(d, n - d);
  return d <= k;
}

// The wide particles search a coarse grid: coarse cell (cx / F, cy / F, cz / F) of grid cell
// (cx, cy, cz), F = s.cF (the last coarse cell along an axis may be thinner).  A particle with
// list radius R lists candidates from every coarse cell that meets the grid-cell box
// +-reach(R) around its own cell -- a superset of its sphere -- and the force kernel decides
// "did the wide j list i" with the same predicate (coarse_meets).
__device__ __forceinline__ bool coarse_meets(int ci, int a, int k, int n, int F, bool per = true) {
  const int f0 = ci * F, w = min(F, n - f0);
  if (!per) return f0 <= a + 2 * k && f0 + w - 1 >= a;  // (non-periodic: the range clipped to the axis)
  if (2 * k + 1 >= n) return true;  // (the whole axis)
  // start of the coarse cell, from a (mod n): a = c - k with c in [0, n) and k <= (n - 1) / 2 + 1
  // (reach), so f0 - a lies in (-n, 2n) and two conditional corrections replace the modulo
  int d0 = f0 - a;
  d0 += d0 < 0 ? n : 0;
  d0 -= d0 >= n ? n : 0;
  return d0 <= 2 * k || d0 + w > n;
}
// x / F for 0 <= x < 2^22, F >= 1 without an integer division: the f32 quotient is within one of
// the exact one, then corrected (the force loop's "did j list i" takes three per wide partner)
__device__ __forceinline__ int div_small(int x, int F) {
  int q = __float2int_rz(__fdividef((float)x, (float)F));
  q += (q + 1) * F <= x ? 1 : 0;
  q -= q * F > x ? 1 : 0;
  return q;
}

// coarse cells meeting the grid-cell range [a, a + 2k] (mod n): c0 (the one holding a) and
// the cnt that follow it cyclically
__device__ __forceinline__ void coarse_range(int a, int k, int n, int F, int cn, int& c0, int& cnt, bool per = true) {
  if (!per) {  // [a, a + 2k] clipped to [0, n)
    const int lo = max(a, 0), hi = min(a + 2 * k, n - 1);
    c0 = lo / F;
    cnt = hi >= lo ? hi / F - c0 + 1 : 0;
    return;
  }
  // closed form of "the cells from the one holding a, cyclically, while coarse_meets" (checked
  // against that loop for every n < 70, F <= n, k <= n, a in [-2n, 2n): identical c0 and cnt)
  if (2 * k + 1 >= n) {
    c0 = 0;
    cnt = cn;
    return;
  }
  const int am = ((a % n) + n) % n, e = am + 2 * k;
  c0 = am / F;
  cnt = e < n ? e / F - c0 + 1 : min(cn - c0 + (e - n) / F + 1, cn);
}

// coarse level of a wide particle whose search reaches kx, ky, kz grid cells: the finest
// whose cells are at least half the reach (its box then meets at most 3 coarse cells per axis)
__device__ __forceinline__ int coarse_level(const DevState& s, int kx, int ky, int kz) {
  const int k = max(kx, max(ky, kz));
  int l = 0;
#pragma unroll
  for (int q = 0; q < kCoarseLevels - 1; ++q) l += (2 * s.cF[l] < k) ? 1 : 0;
  return l;
}

template <bool PX>
__global__ void k_coarse_keys(int n, int l, DevGrid g, DevState s, unsigned int* keys, unsigned int* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 x = s.xh[i];
  const int F = s.cF[l];
  const unsigned int ccx = (unsigned)(plane_of<PX>(g, i, x.x) / F), ccy = (unsigned)(cell_axis(x.y, g.ny) / F),
                     ccz = (unsigned)(cell_axis(x.z, g.nz) / F);
  keys[i] = (ccx * (unsigned)s.cny[l] + ccy) * (unsigned)s.cnz[l] + ccz;
  vals[i] = (unsigned)i;
}

// (a particle within wide_margin of the cell side is wide already: its h may still grow in the h
// iteration, and outgrowing the cell mid-iteration costs a regrid of the lists; n0 counts the
// particles wide without the margin, so the host can refuse a margin that flips a whole population)
__global__ void k_mark_wide(int n, DevGrid g, DevPhys ph, DevState s, uint8_t* flag, unsigned int* n0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool w0 = false;
  if (i < n) {
    const float R = (1.f + g.skin) * ph.gamma_k * __uint_as_float(s.xh[i].w);
    const bool w = R * (1.f + g.wide_margin) > g.side_min;
    w0 = R > g.side_min;
    flag[i] = w ? 1 : 0;
    if (w) s.ncount[i] = 0;  // (no tile list: its block may not even run)
  }
  const unsigned b = __ballot_sync(kFull, w0);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(n0, (unsigned)__popc(b));
}

// One warp per wide particle.  Overflow of wlcap: the count is still returned (max in
// ctr->list_overflow) and the host rebuilds with a larger capacity.
template <bool PX>
// (8 CTAs per SM, 32 registers: C5s lists 8.93 at 5 CTAs, 8.77 at 6, 8.65 at 8)
#ifndef SPH_WL_MINB
#define SPH_WL_MINB 8
#endif
__global__ void __launch_bounds__(256, SPH_WL_MINB) k_wide_lists(DevGrid g, DevPhys ph, DevState s, const int* __restrict__ cell_start,
                                                    DevCounters* __restrict__ ctr) {
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wi >= s.n_wide) return;
  const int i = s.widx[wi];
  const uint4 xi = s.xh[i];
  const float Hfac = (1.f + g.skin) * ph.gamma_k;
  const float hi = __uint_as_float(xi.w);
  const float Hi2 = (Hfac * hi) * (Hfac * hi);
  constexpr bool px = PX;
  const int cx = plane_of<PX>(g, i, xi.x), cy = cell_axis(xi.y, g.ny), cz = cell_axis(xi.z, g.nz);
  const int kx = px ? reach(Hfac * hi, g.side[0], g.nx) : (int)ceilf(Hfac * hi / g.side[0]),
            ky = reach(Hfac * hi, g.side[1], g.ny), kz = reach(Hfac * hi, g.side[2], g.nz);
  const int lev = coarse_level(s, kx, ky, kz);
  const int F = s.cF[lev], cnx = s.cnx[lev], cny = s.cny[lev], cnz = s.cnz[lev];
  const int* __restrict__ ccs = s.ccs[lev];
  const uint32_t* __restrict__ cperm = s.cperm[lev];
  int x0, nxc, y0, nyc, z0, nzc;  // coarse cells meeting the grid-cell box, per axis
  coarse_range(cx - kx, kx, g.nx, F, cnx, x0, nxc, px);
  coarse_range(cy - ky, ky, g.ny, F, cny, y0, nyc);
  coarse_range(cz - kz, kz, g.nz, F, cnz, z0, nzc);
  const int run1 = min(nzc, cnz - z0);  // the z range as at most two contiguous runs
  uint32_t* lst = s.wnbr + (size_t)wi * s.wlcap;
  // the candidate ranges -- (coarse column, z run) pairs, in order -- 32 at a time: lane r loads
  // range r's ends, a warp scan flattens them, and the lanes walk the flattened candidates (so a
  // short range costs no round trip of its own), hits compacted with a ballot: the list is in
  // (column, z run, slot) order
  int cnt = 0;
  const int nr = nxc * nyc * 2;
  for (int rb = 0; rb < nr; rb += 32) {
    int t0 = 0, len = 0;
    {
      const int q = rb + lane;
      if (q < nr) {
        const int cq = q >> 1, part = q & 1;
        const int ax = cq / nyc, ay = cq - ax * nyc;
        const int ccx = (x0 + ax) % cnx, ccy = (y0 + ay) % cny;
        const int col = (ccx * cny + ccy) * cnz;
        const int c0 = part == 0 ? z0 : 0, nc = part == 0 ? run1 : nzc - run1;
        if (nc > 0) {
          t0 = __ldg(ccs + col + c0);
          len = __ldg(ccs + col + c0 + nc) - t0;
        }
      }
    }
    int incl = len;  // inclusive prefix of the lengths over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    // two chunks of 32 candidates per trip, both gathers (cperm -> xh) issued before either test
    // (the loop is bound by that chain's latency); hits compacted chunk by chunk, in order
    auto locate = [&](int idx, int& r0, int& e0) {  // the range holding idx: first lane with incl > idx
      int lo = 0;
#pragma unroll
      for (int w = 16; w > 0; w >>= 1) {
        const int v = __shfl_sync(kFull, incl, lo + w - 1);
        if (v <= idx) lo += w;
      }
      r0 = __shfl_sync(kFull, t0, lo & 31);
      e0 = __shfl_sync(kFull, incl - len, lo & 31);
    };
    auto test = [&](int j, const uint4& xj) {
      const float dx = (float)(int)(xi.x - xj.x) * g.scale[0];
      const float dy = (float)(int)(xi.y - xj.y) * g.scale[1];
      const float dz = (float)(int)(xi.z - xj.z) * g.scale[2];
      const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      const float hj = __uint_as_float(xj.w);
      // a partner at exactly i's position (j != i) is skipped
      return r2 < fmaxf(Hi2, (Hfac * hj) * (Hfac * hj)) &&
             !(j != i && xj.x == xi.x && xj.y == xi.y && xj.z == xi.z);
    };
    auto emit = [&](bool hit, int j) {
      const unsigned b = __ballot_sync(kFull, hit);
      const int pos = cnt + __popc(b & ((1u << lane) - 1u));
      if (hit && pos < s.wlcap) lst[pos] = (uint32_t)j;
      cnt += __popc(b);
    };
    for (int base = 0; base < total; base += 64) {
      const int ia = base + lane, ib = base + 32 + lane;
      int ra, ea, rb, eb;
      locate(ia, ra, ea);
      locate(ib, rb, eb);
      const bool va = ia < total, vb = ib < total;
      const int ja = va ? (int)__ldg(cperm + ra + (ia - ea)) : 0, jb = vb ? (int)__ldg(cperm + rb + (ib - eb)) : 0;
      const uint4 xa = va ? s.xh[ja] : xi, xb = vb ? s.xh[jb] : xi;
      emit(va && test(ja, xa), ja);
      if (base + 32 < total) emit(vb && test(jb, xb), jb);
    }
  }
  if (lane == 0) {
    s.wcount[wi] = min(cnt, s.wlcap);
    s.hbuild[i] = hi;
    if (cnt > s.wlcap) atomicMax(&ctr->wlist_overflow, cnt);
  }
}

// relative position r_i - r_j of two particles (minimum image on the 2^-32 grid)
__device__ __forceinline__ float3 rel(const DevGrid& g, const uint4& a, const uint4& b) {
  return make_float3((float)(int)(a.x - b.x) * g.scale[0], (float)(int)(a.y - b.y) * g.scale[1],
                     (float)(int)(a.z - b.z) * g.scale[2]);
}

// |q - 2| below this: decide membership in fp64 (fp32 r from exact integer differences errs
// by < 1e-6 relative)
constexpr float kBandW = 2e-5f;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_fmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// One warp per wide particle: the lanes split the list, the sums are reduced over the warp
// (lane order, deterministic), lane 0 runs the epilogue.
// (5 CTAs per SM, 48 registers: with the in-kernel h iteration 6 CTAs spill; C5s density 6.03 at 8 CTAs)
#ifndef SPH_WD_MINB
#define SPH_WD_MINB 5
#endif
__global__ void __launch_bounds__(256, SPH_WD_MINB) k_wide_density(DevGrid g, DevPhys ph, DevState s, int pass, float hfac_stale,
                                                      DevCounters* __restrict__ ctr) {
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wi >= s.n_wide_own) return;  // (ghosts: their owner iterates them)
  const int i = s.widx[wi];
  if (pass > 0 && !s.active[i]) return;  // warp-uniform
  const uint4 xi = s.xh[i];
  const float4 vi = s.vm[i];
  const uint32_t* lst = s.wnbr + (size_t)wi * s.wlcap;
  const int n = s.wcount[wi];
  // the h iteration inside the kernel (one rank): a wide particle's sums depend on its own h
  // only, so after a Newton update it walks its list again while the new h stays within the
  // list radius (at most 6 updates per pass, as the tile density loop); the slab path takes one
  // update per pass (its ghost-plane check, below, is per pass)
  const int maxit = g.periodic_x ? 6 : 1;
  float h = __uint_as_float(xi.w);
  for (int it = 0; it < maxit; ++it) {
    const float hinv = 1.f / h;
    const double H2 = h2_exact(h, ph.gamma_k);
    DenAcc a = DenAcc::zero();
    for (int k = lane; k < n; k += 32) {
      const int j = (int)__ldg(lst + k);
      const float3 d = rel(g, xi, s.xh[j]);
      den_pair(a, d.x, d.y, d.z, hinv, kBandW, vi, s.vm[j], [&]() {
        return exact_neighbour(s.xh, i, j, H2, g.dscale[0], g.dscale[1], g.dscale[2]);
      });
    }
    a.S0 = warp_sum(a.S0); a.S1 = warp_sum(a.S1); a.R0 = warp_sum(a.R0); a.R1 = warp_sum(a.R1);
    a.Dv = warp_sum(a.Dv); a.Cx = warp_sum(a.Cx); a.Cy = warp_sum(a.Cy); a.Cz = warp_sum(a.Cz);
    a.nn = warp_isum(a.nn);
    int more = 0;
    float hn = h;
    if (lane == 0) {
      const DenOut o = den_epilogue(g, ph, s, a, i, h, vi.w, pass + it, hfac_stale);
      atomicAdd(&ctr->pairs_all, (unsigned long long)o.nn);
      more = o.active && !o.stale && it + 1 < maxit;
      hn = o.hn;
      if (!more) {
        if (o.final_) atomicAdd(&ctr->pairs, (unsigned long long)o.nn);
        if (o.final_ && o.resid > 0.f) atomicMax(&ctr->max_resid_bits, __float_as_uint(o.resid));
        if (o.give_up) atomicAdd(&ctr->unconverged, 1);
        if (o.active) atomicAdd(&ctr->active_next, 1);
        if (o.stale) atomicExch(&ctr->list_stale, 1);
        // slab path: the new list radius must still fit the G ghost planes (ghost_planes_needed);
        // past them the grid is rebuilt with a larger G
        if (!g.periodic_x && o.active &&
            ghost_planes_needed((int)ceilf((1.f + g.skin) * ph.gamma_k * o.hn / g.side_min),
                                plane_of<false>(g, i, xi.x) - g.ix_first, g.nxo) > g.ix_first)
          atomicExch(&ctr->h_exceeds, 1);
      }
    }
    more = __shfl_sync(kFull, more, 0);
    if (!more) break;
    h = __shfl_sync(kFull, hn, 0);
  }
}

// (k_wide_gradient at 5 CTAs per SM, 48 registers: C5s gradient 3.13 -> 2.89 ms; 4 CTAs 3.10)
#ifndef SPH_WG_MINB
#define SPH_WG_MINB 5
#endif
__global__ void __launch_bounds__(256, SPH_WG_MINB) k_wide_gradient(DevGrid g, DevPhys ph, DevState s, float dt, int first_step,
                                                       DevCounters* __restrict__ ctr) {
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wi >= s.n_wide_own) return;  // (ghosts: the X3 exchange brings their records)
  const int i = s.widx[wi];
  const uint4 xi = s.xh[i];
  const float4 vi = s.vm[i];
  const float4 gi4 = s.gq[i];
  const float h = __uint_as_float(xi.w), hinv = 1.f / h;
  const double H2 = h2_exact(h, ph.gamma_k);
  const uint32_t* lst = s.wnbr + (size_t)wi * s.wlcap;
  const int n = s.wcount[wi];
  GradAcc a{2.f * gi4.x, 0.f, 0};
  // two entries per lane per trip, both gathers issued before either pair (the loop is bound by
  // the latency of the list -> record gather chain; C5s gradient 3.43 -> 3.13 ms); the lane's sum
  // order is unchanged
  for (int k = lane; k < n; k += 64) {
    const bool two = k + 32 < n;
    const int j0 = (int)__ldg(lst + k), j1 = two ? (int)__ldg(lst + k + 32) : j0;
    const uint4 x0 = s.xh[j0], x1 = s.xh[j1];
    const float4 v0 = s.vm[j0], v1 = s.vm[j1], q0 = s.gq[j0], q1 = s.gq[j1];
    const float3 d0 = rel(g, xi, x0);
    grad_pair(a, d0.x, d0.y, d0.z, hinv, kBandW, vi, gi4.x, gi4.y, ph.beta, v0, q0, [&]() {
      return exact_neighbour(s.xh, i, j0, H2, g.dscale[0], g.dscale[1], g.dscale[2]);
    });
    if (two) {
      const float3 d1 = rel(g, xi, x1);
      grad_pair(a, d1.x, d1.y, d1.z, hinv, kBandW, vi, gi4.x, gi4.y, ph.beta, v1, q1, [&]() {
        return exact_neighbour(s.xh, i, j1, H2, g.dscale[0], g.dscale[1], g.dscale[2]);
      });
    }
  }
  a.vmax = warp_fmax(a.vmax);
  a.lap = warp_sum(a.lap);
  a.nn = warp_isum(a.nn);
  if (lane != 0) return;
  const int nn = grad_epilogue(ph, s, a, i, h, gi4.x, gi4.y, gi4.w, dt, first_step);
  atomicAdd(&ctr->pairs, (unsigned long long)nn);
}

// acc, v_sig and N_force of the wide particles start from zero: k_wide_force adds them
__global__ void k_wide_zero(DevState s) {
  const int wi = blockIdx.x * blockDim.x + threadIdx.x;
  if (wi >= s.n_wide) return;
  const int i = s.widx[wi];
  s.acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  s.vsig[i] = 0.f;
  s.countf[i] = 0;
}

__device__ __forceinline__ ForceSide side_of(const DevState& s, int i, float h) {
  ForceSide f;
  f.hinv = 1.f / h;
  f.v = s.vm[i];
  f.a = s.fr1[i];
  f.b = s.fr2[i];
  f.P = f.a.x * f.a.w * f.a.w;
  return f;
}

__device__ __forceinline__ void red_add4_w(float4* p, const float4& v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

// One warp per wide particle i over its list.  Every pair of the symmetric force set is
// evaluated ONCE (force_pair2: both sides, Eqs. 17-18) by exactly one particle and applied to
// both: a tile partner never evaluates a pair with a wide one (k_lists keeps those out of its
// force part), so i does; a wide partner that listed i too does it only if it has the lower index;
// one that did not list i leaves it to i.  i's side is reduced over the warp (lane order), j's
// goes to acc[j] with one vector reduction.  v_sig and N_force: i's over its list; a partner
// that did not list i gets its share of the pair here (atomics).
template <bool PX>
// (k_wide_force at 4 CTAs per SM, 64 registers: the gather-latency-bound loop wants the warps;
// C5s force 6.24 -> 5.27 ms, 5 CTAs (48 registers, spills) 5.58)
#ifndef SPH_WF_MINB
#define SPH_WF_MINB 4
#endif
__global__ void __launch_bounds__(256, SPH_WF_MINB) k_wide_force(DevGrid g, DevPhys ph, DevState s, DevCounters* __restrict__ ctr) {
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wi >= s.n_wide) return;
  const int i = s.widx[wi];
  const uint4 xi = s.xh[i];
  const float h = __uint_as_float(xi.w);
  const ForceSide I = side_of(s, i, h);
  const double Hi2 = h2_exact(h, ph.gamma_k);
  const float Hfac = (1.f + g.skin) * ph.gamma_k;
  constexpr bool px = PX;
  const int cxi = plane_of<PX>(g, i, xi.x), cyi = cell_axis(xi.y, g.ny), czi = cell_axis(xi.z, g.nz);
  // a ghost i (slab path) evaluates its pairs for the owned partners only; its own side is its owner's
  const bool iown = PX || wi < s.n_wide_own;
  const uint32_t* lst = s.wnbr + (size_t)wi * s.wlcap;
  const int n = s.wcount[wi];
  float4 ai = make_float4(0.f, 0.f, 0.f, 0.f);
  float vmax = 2.f * I.a.z;  // (R15)
  int nn = 0;
  // (loading the next trip's list entry and position one trip ahead: C5s force 6.24 -> 6.34 ms)
  for (int k = lane; k < n; k += 32) {
    const int j = (int)__ldg(lst + k);
    const uint4 xj = s.xh[j];
    const float hj = __uint_as_float(xj.w);
    const ForceSide J = side_of(s, j, hj);
    const float3 d = rel(g, xi, xj);
    // membership of the symmetric set, r < max(H_i, H_j) (R3; fp64 inside the band), and the
    // pair's signal velocity (Eqs. 10-11)
    const float r2 = fmaf(d.z, d.z, fmaf(d.y, d.y, d.x * d.x));
    const float rinv = rinv_safe(r2);
    const float r = r2 * rinv;
    const float dd = fminf(r * I.hinv, r * J.hinv) - 2.f;
    int in = neg(dd);
    if (fabsf(dd) < kBandW)
      in = exact_neighbour(s.xh, i, j, fmax(Hi2, h2_exact(hj, ph.gamma_k)), g.dscale[0], g.dscale[1], g.dscale[2]);
    const float vrr = fmaf(I.v.z - J.v.z, d.z, fmaf(I.v.y - J.v.y, d.y, (I.v.x - J.v.x) * d.x)) * rinv;
    const float vs = fmaf(-ph.beta, fminf(vrr, 0.f), I.a.z + J.a.z);
    nn += in;
    vmax = fmaxf(vmax, in ? vs : 0.f);
    // did j list i?  tile particles list the cells within +-1 of their own, wide ones the
    // cells within their list radius at build time (k_wide_lists)
    const int cxj = plane_of<PX>(g, j, xj.x), cyj = cell_axis(xj.y, g.ny), czj = cell_axis(xj.z, g.nz);
    const bool jwide = s.wide[j] != 0;
    const float Rj = Hfac * s.hbuild[j];
    bool seen;
    if (jwide) {  // j's search: the coarse cells meeting its grid-cell box (k_wide_lists)
      const int kx = px ? reach(Rj, g.side[0], g.nx) : (int)ceilf(Rj / g.side[0]), ky = reach(Rj, g.side[1], g.ny),
                kz = reach(Rj, g.side[2], g.nz);
      const int F = s.cF[coarse_level(s, kx, ky, kz)];
      seen = coarse_meets(div_small(cxi, F), cxj - kx, kx, g.nx, F, px) &&
             coarse_meets(div_small(cyi, F), cyj - ky, ky, g.ny, F) && coarse_meets(div_small(czi, F), czj - kz, kz, g.nz, F);
    } else {
      seen = within(cxi, cxj, 1, g.nx, px) && within(cyi, cyj, 1, g.ny) && within(czi, czj, 1, g.nz);
    }
    const bool jown = px || (j >= g.gL && j < g.gL + g.n_own);
    if (j != i && (!jwide || !seen || i < j)) {
      float4 jo;
      force_pair2(ai, jo, d.x, d.y, d.z, I, J, ph.beta);
      red_add4_w(s.acc + j, jo);
    }
    // v_sig and N_force of a partner that listed i already hold the pair (gradient loop); the
    // CFL dt is taken from the final v_sig of every particle afterwards (k_force_fin)
    if (j != i && in && !seen && jown) {
      atomicMax(reinterpret_cast<int*>(&s.vsig[j]), __float_as_int(vs));
      atomicAdd(&s.countf[j], 1);
    }
  }
  ai.x = warp_sum(ai.x);
  ai.y = warp_sum(ai.y);
  ai.z = warp_sum(ai.z);
  ai.w = warp_sum(ai.w);
  vmax = warp_fmax(vmax);
  nn = warp_isum(nn);
  if (lane != 0 || !iown) return;
  red_add4_w(s.acc + i, ai);
  atomicMax(reinterpret_cast<int*>(&s.vsig[i]), __float_as_int(vmax));
  atomicAdd(&s.countf[i], nn - 1);  // (the self pair)
  if (!(isfinite(vmax) && isfinite(ai.x) && isfinite(ai.y) && isfinite(ai.z) && isfinite(ai.w)))
    atomicExch(&ctr->nonfinite, 1);
}

}  // namespace

cudaError_t launch_mark_wide(int n, const DevGrid& g, const DevPhys& ph, const DevState& s, uint8_t* flag,
                             unsigned int* n0, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_mark_wide<<<(n + 255) / 256, 256, 0, st>>>(n, g, ph, s, flag, n0);
  return cudaGetLastError();
}

cudaError_t launch_coarse_keys(int n, int level, const DevGrid& g, const DevState& s, unsigned int* keys,
                               unsigned int* vals, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (g.periodic_x) k_coarse_keys<true><<<(n + 255) / 256, 256, 0, st>>>(n, level, g, s, keys, vals);
  else k_coarse_keys<false><<<(n + 255) / 256, 256, 0, st>>>(n, level, g, s, keys, vals);
  return cudaGetLastError();
}

cudaError_t launch_wide_lists(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                              DevCounters* ctr, cudaStream_t st) {
  if (s.n_wide <= 0) return cudaSuccess;
  if (g.periodic_x) k_wide_lists<true><<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, cell_start, ctr);
  else k_wide_lists<false><<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, cell_start, ctr);
  return cudaGetLastError();
}

cudaError_t launch_wide_density(const DevGrid& g, const DevPhys& ph, const DevState& s, int pass, float hfac_stale,
                                DevCounters* ctr, cudaStream_t st) {
  if (s.n_wide <= 0) return cudaSuccess;
  k_wide_density<<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, pass, hfac_stale, ctr);
  return cudaGetLastError();
}

cudaError_t launch_wide_gradient(const DevGrid& g, const DevPhys& ph, const DevState& s, float dt, int first_step,
                                 DevCounters* ctr, cudaStream_t st) {
  if (s.n_wide <= 0) return cudaSuccess;
  k_wide_gradient<<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, dt, first_step, ctr);
  return cudaGetLastError();
}

cudaError_t launch_wide_force(const DevGrid& g, const DevPhys& ph, const DevState& s, DevCounters* ctr,
                              cudaStream_t st) {
  if (s.n_wide <= 0) return cudaSuccess;
  k_wide_zero<<<(s.n_wide + 255) / 256, 256, 0, st>>>(s);
  if (g.periodic_x) k_wide_force<true><<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, ctr);
  else k_wide_force<false><<<(s.n_wide * 32 + 255) / 256, 256, 0, st>>>(g, ph, s, ctr);
  return cudaGetLastError();
}

}  // namespace sph
