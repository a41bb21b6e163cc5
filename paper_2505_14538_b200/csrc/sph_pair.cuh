// sph_pair.cuh -- the per-pair arithmetic and per-particle epilogues of the three SPH loops
// (arXiv 2505.14538), shared by the tile kernels (sph_kernels.cu: neighbours
// gathered from a shared-memory tile) and the wide-particle kernels (sph_wide.cu: neighbours
// gathered from global memory).  Each function states the equations it evaluates; the
// readings R* are DESIGN.md §3.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "sph_internal.cuh"

namespace sph {

// 1 if d < 0 (sign bit), i.e. q < 2 for d = q - 2
__device__ __forceinline__ int neg(float d) { return (int)(__float_as_uint(d) >> 31); }

// r^-1 with the self pair (r = 0, listed) mapped to a finite value: every pair term of the
// self pair then carries w'(0) = 0 or v_ij = 0 and vanishes exactly.
__device__ __forceinline__ float rinv_safe(float r2) { return rsqrtf(fmaxf(r2, 1e-30f)); }

// fp64 fixed-point neighbour test, operation for operation the oracle's (oracle.c sep2):
// r^2 = (dx*dx + dy*dy) + dz*dz < H2 with dx = (double)(int32)(X_i - X_j) * (L * 2^-32).
// Only reached for pairs within the f32 error band of the support radius (rare).
__device__ __forceinline__ bool exact_neighbour(const uint4* __restrict__ xh, int gi, int gj, double H2, double sx,
                                                double sy, double sz) {
  const uint4 a = xh[gi], b = xh[gj];
  const double dx = __dmul_rn((double)(int)(a.x - b.x), sx);
  const double dy = __dmul_rn((double)(int)(a.y - b.y), sy);
  const double dz = __dmul_rn((double)(int)(a.z - b.z), sz);
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return r2 < H2 && r2 > 0.0;
}

__device__ __forceinline__ double h2_exact(float h, float gamma_k) {
  const double H = __dmul_rn((double)gamma_k, (double)h);
  return __dmul_rn(H, H);
}

// -dW/dq / 0.75 of M4: q (4 - 3q) for q < 1, (2 - q)^2 for 1 <= q < 2, 0 beyond, as the
// truncated powers t^2 - 4 s^2 (t = (2 - q)+, s = (1 - q)+): no branch or predicate
__device__ __forceinline__ float m4_dwp(float q) {
  const float t = fmaxf(2.f - q, 0.f), s = fmaxf(1.f - q, 0.f);
  return fmaf(t, t, -4.f * (s * s));
}

// alpha_c weight floor of the force records (force_pair2, Eq. 20 / R13)
constexpr float kPeps = 1e-30f;

// ---------------------------------------------------------------- density (Eqs. 2-6) ----
// Accumulators per particle i (q = r/h_i, w = M4; the self pair is in the list: w(0) = 1):
//   S0 = sum w, S1 = sum q w', R0 = sum m_j w, R1 = sum m_j q w',
//   Dv = sum m_j w'/r (v_ij . r_ij),  Cv = sum m_j w'/r (v_ij x r_ij),  N_i.
// Then nhat = S0/(pi h^3), dn/dh = -(3 S0 + S1)/(pi h^4), rho = R0/(pi h^3),
// drho/dh = -(3 R0 + R1)/(pi h^4), div = -Dv/(rho pi h^4), curl = Cv/(rho pi h^4),
// g = nhat h^3 - eta^3 = S0/pi - eta^3, h g' = -S1/pi.
struct DenAcc {
  float S0, S1, R0, R1, Dv, Cx, Cy, Cz;
  int nn;
  __device__ static DenAcc zero() { return DenAcc{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0}; }
  __device__ void add(const DenAcc& o) {
    S0 += o.S0; S1 += o.S1; R0 += o.R0; R1 += o.R1; Dv += o.Dv; Cx += o.Cx; Cy += o.Cy; Cz += o.Cz; nn += o.nn;
  }
};

// One directed pair: r_ij = (dx, dy, dz) = r_i - r_j (R4), vi = v_i, vj = (v_j, m_j);
// |q - 2| < qband re-decides membership with exact() (fp64).
template <class Exact>
__device__ __forceinline__ void den_pair(DenAcc& a, float dx, float dy, float dz, float hinv, float qband,
                                         const float4& vi, const float4& vj, Exact&& exact) {
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float rinv = rinv_safe(r2);
  const float q = r2 * rinv * hinv;
  const float d = q - 2.f;
  a.nn += neg(d);
  if (fabsf(d) < qband) a.nn += (int)exact() - neg(d);
  // M4 as truncated powers: w = t^3/4 - s^3, w' = -3/4 t^2 + 3 s^2 (t = (2-q)+, s = (1-q)+)
  const float tq = fmaxf(-d, 0.f), sq = fmaxf(1.f - q, 0.f);
  const float t2 = tq * tq, s2 = sq * sq;
  const float w = fmaf(0.25f * tq, t2, -sq * s2);
  const float dw = fmaf(3.f, s2, -0.75f * t2);
  const float qdw = q * dw;
  a.S0 += w;
  a.S1 += qdw;
  a.R0 = fmaf(vj.w, w, a.R0);
  a.R1 = fmaf(vj.w, qdw, a.R1);
  const float F = vj.w * dw * rinv;
  const float ux = vi.x - vj.x, uy = vi.y - vj.y, uz = vi.z - vj.z;
  a.Dv = fmaf(F, fmaf(uz, dz, fmaf(uy, dy, ux * dx)), a.Dv);
  a.Cx = fmaf(F, fmaf(uy, dz, -uz * dy), a.Cx);
  a.Cy = fmaf(F, fmaf(uz, dx, -ux * dz), a.Cy);
  a.Cz = fmaf(F, fmaf(ux, dy, -uy * dx), a.Cz);
}

// Epilogue of particle gi (h, mass mi) for density pass `pass`: closure test, then
// either the density finalize (Eq. 8 with R8, ideal-gas EoS, Balsara switch R14) or one
// Newton update of h with bracket and bisection (R7).
struct DenOut {
  int nn;        // neighbours (self excluded)
  bool final_;   // converged (or given up): results stored
  bool give_up;
  bool active;   // another pass needed
  bool exceeds;  // the new support outgrows the cell side
  bool stale;    // the new h outgrows the list radius
  float hn;      // the new h (active)
  float resid;   // final: |nhat h^3 - eta^3| / eta^3 (the closure residual)
};
__device__ __forceinline__ DenOut den_epilogue(const DevGrid& g, const DevPhys& ph, const DevState& s, const DenAcc& a,
                                               int gi, float h, float mi, int pass, float hfac_stale) {
  DenOut o{a.nn - 1, false, false, false, false, false, h, 0.f};  // (the self pair)
  const float inv_pi = 1.f / kPi;
  const float hinv = 1.f / h;
  const float ih3 = inv_pi * hinv * hinv * hinv;
  const float nhat = a.S0 * ih3;
  const float dndh = -(3.f * a.S0 + a.S1) * ih3 * hinv;
  const float rho = a.R0 * ih3;
  const float drho = -(3.f * a.R0 + a.R1) * ih3 * hinv;
  const float gres = a.S0 * inv_pi - ph.eta3;
  const bool conv = (ph.h_max_iter == 0) || fabsf(gres) <= ph.h_tol * ph.eta3;
  const int it = pass == 0 ? 0 : s.iters[gi];
  const bool give_up = !conv && it >= ph.h_max_iter;
  if (conv || give_up) {
    const float ih4 = ih3 * hinv / rho;
    s.dens[gi] = make_float4(rho, drho, nhat, dndh);
    const float div = -a.Dv * ih4;
    const float cx = a.Cx * ih4, cy = a.Cy * ih4, cz = a.Cz * ih4;
    s.dvc[gi] = make_float4(cx, cy, cz, div);
    s.count[gi] = o.nn;
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
    const float4 vmi = s.vm[gi];
    s.vc[gi] = make_float4(vmi.x, vmi.y, vmi.z, cs);
    s.um[gi] = make_float2(u, mi / rho);
    // halo put (X2): a boundary-plane particle's gradient records and h go straight to the
    // neighbours (peer stores; the exchange then carries only an ordering token)
#pragma unroll
    for (int d = 0; d < 2; ++d)
      if (s.put_gq[d] && gi >= s.put_lo[d] && gi < s.put_hi[d]) {
        const int t = gi - s.put_lo[d];
        s.put_gq[d][t] = make_float4(cs, u, mi / rho, rho);
        s.put_vc[d][t] = make_float4(vmi.x, vmi.y, vmi.z, cs);
        s.put_um[d][t] = make_float2(u, mi / rho);
        s.put_h[d][t] = h;
      }
    s.active[gi] = 0;
    s.iters[gi] = conv ? it : -1;
    o.final_ = true;
    o.give_up = give_up;
    o.resid = fabsf(gres) / ph.eta3;
  } else {
    // Newton with bracket + bisection (R7); g is non-decreasing in h
    float lo = pass == 0 ? 0.f : s.hlo[gi];
    float hi = pass == 0 ? CUDART_INF_F : s.hhi[gi];
    if (gres > 0.f) hi = h; else lo = h;
    float hn = (a.S1 < 0.f) ? h * (1.f + (a.S0 - ph.pi_eta3) / a.S1) : (gres < 0.f ? 2.f * h : 0.5f * h);
    hn = fminf(fmaxf(hn, 0.5f * h), 2.f * h);
    if (hn <= lo || hn >= hi) hn = isinf(hi) ? 2.f * h : 0.5f * (lo + hi);
    s.hlo[gi] = lo;
    s.hhi[gi] = hi;
    s.iters[gi] = it + 1;
    s.active[gi] = 1;
    reinterpret_cast<unsigned int*>(&s.xh[gi])[3] = __float_as_uint(hn);
    o.active = true;
    o.hn = hn;
    // a particle already wide may grow past the cell: its list search widens instead
    const bool wide = s.wide && s.wide[gi];
    o.exceeds = !wide && ph.gamma_k * hn * (1.f + g.skin) > g.side_min;
    o.stale = hn > hfac_stale * s.hbuild[gi];
  }
  return o;
}

// ------------------------------------------------------------- gradient (Eqs. 10-16) ----
// v_sig,i = max(2 c_i, max_j (c_i + c_j - beta mu_ij)) (Eqs. 10-11, R15) and the Brookshaw
// Laplacian lap u_i = 2 sum_j (m_j/rho_j)(u_i - u_j) dW/dr / r (R16), over r_ij < H_i.
// vmaxs and the high half of nn: the force loop's signal velocity and neighbour count over the
// symmetric set r_ij < max(H_i, H_j) (R3, R15), taken by the tile gradient loop (same v and
// c_s as the force loop; the pair-once force loop then carries no per-pair maximum or count).
// nn = gather count | symmetric count << 16 (16 bytes per accumulator record).
struct GradAcc {
  float vmax, lap;  // vmax > 0: max over its f32 bits as int
  int nn;
  float vmaxs;
  __device__ static GradAcc zero() { return GradAcc{0.f, 0.f, 0, 0.f}; }
  __device__ void add(const GradAcc& o) {
    vmax = fmaxf(vmax, o.vmax); lap += o.lap; nn += o.nn; vmaxs = fmaxf(vmaxs, o.vmaxs);
  }
};

// vj = (v_j, m_j), gj = (c_j, u_j, m_j/rho_j, rho_j)
template <class Exact>
__device__ __forceinline__ void grad_pair(GradAcc& a, float dx, float dy, float dz, float hinv, float qband,
                                          const float4& vi, float ci, float ui, float beta, const float4& vj,
                                          const float4& gj, Exact&& exact) {
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float rinv = rinv_safe(r2);
  const float q = r2 * rinv * hinv;
  const float d = q - 2.f;
  int in = neg(d);
  if (fabsf(d) < qband) in = exact();
  a.nn += in;
  const float tq = fmaxf(-d, 0.f), sq = fmaxf(1.f - q, 0.f);
  const float dw = fmaf(3.f * sq, sq, -0.75f * tq * tq);  // M4 w'(q)
  const float vr = fmaf(vi.z - vj.z, dz, fmaf(vi.y - vj.y, dy, (vi.x - vj.x) * dx));
  const float mu = fminf(vr, 0.f) * rinv;
  const float vs = fmaf(-beta, mu, ci + gj.x);
  a.vmax = fmaxf(a.vmax, in ? vs : 0.f);
  a.lap = fmaf(gj.z * (ui - gj.y), dw * rinv, a.lap);
}

// The tile loop's pair: grad_pair plus membership of the symmetric force set,
// min(q_i, q_j) < 2 (qj = r / h_j; fp64 inside the band `sband`).
template <class Exact, class ExactS>
__device__ __forceinline__ void grad_pair_sym(GradAcc& a, float dx, float dy, float dz, float hinv, float hinvj,
                                              float qband, float sband, const float4& vi, float ci, float ui, float beta,
                                              const float4& vj, const float4& gj, Exact&& exact, ExactS&& exact_s) {
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float rinv = rinv_safe(r2);
  const float r = r2 * rinv;
  const float q = r * hinv;
  const float d = q - 2.f;
  int in = neg(d);
  if (fabsf(d) < qband) in = exact();
  const float ds = fminf(q, r * hinvj) - 2.f;
  int ins = neg(ds);
  if (fabsf(ds) < sband) ins = exact_s();
  a.nn += in + (ins << 16);
  const float tq = fmaxf(-d, 0.f), sq = fmaxf(1.f - q, 0.f);
  const float dw = fmaf(3.f * sq, sq, -0.75f * tq * tq);  // M4 w'(q)
  const float vr = fmaf(vi.z - vj.z, dz, fmaf(vi.y - vj.y, dy, (vi.x - vj.x) * dx));
  const float mu = fminf(vr, 0.f) * rinv;
  const float vs = fmaf(-beta, mu, ci + gj.x);
  a.vmax = fmaxf(a.vmax, in ? vs : 0.f);
  a.vmaxs = fmaxf(a.vmaxs, ins ? vs : 0.f);
  a.lap = fmaf(gj.z * (ui - gj.y), dw * rinv, a.lap);
}

// Gradient ghost of particle gi (R17-R21): alpha_v (Eqs. 12-15), alpha_c (Eqs. 21-24), and
// the force-loop records fr1 = (A = P/rho^2, K = -0.75 f/(pi h^4), c, rho) and fr2 = (B,
// (P + kPeps) alpha_c -- Eq. 20's weight, with its P_i + P_j = 0 case (R13), see force_pair2 --,
// u, alpha_v).  Returns N_i (self excluded).
__device__ __forceinline__ int grad_epilogue(const DevPhys& ph, const DevState& s, const GradAcc& a, int gi, float h,
                                             float ci, float ui, float rho, float dt, int first_step) {
  const float hinv = 1.f / h;
  const float lap_u = 2.f * a.lap * hinv * hinv * hinv * hinv / kPi;
  const float vsig = a.vmax;
  const float H = ph.gamma_k * h;
  const float4 dvc = s.dvc[gi];
  const float4 fin = s.fin[gi];
  const float div = dvc.w;
  float av = s.av[gi], ac = s.ac[gi];
  const float Ddot = first_step ? 0.f : (div - s.dprev[gi]) / dt;
  const float Sx = H * H * fmaxf(-Ddot, 0.f);
  const float den = vsig * vsig + Sx;
  const float aloc = den > 0.f ? ph.alpha_v_max * Sx / den : 0.f;
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
  const float f = fin.x, P = fin.y;
  const float4 r1 = make_float4(P / (rho * rho), -0.75f * f * hinv * hinv * hinv * hinv / kPi, ci, rho);
  const float4 r2 = make_float4(fin.w, (P + kPeps) * ac, ui, av);
  s.fr1[gi] = r1;
  s.fr2[gi] = r2;
  // halo put: a boundary-plane particle's records also go straight to the neighbours' ghost
  // slots (peer stores; the X3 exchange then carries only an ordering token)
#pragma unroll
  for (int d = 0; d < 2; ++d)
    if (s.put_fr1[d] && gi >= s.put_lo[d] && gi < s.put_hi[d]) {
      s.put_fr1[d][gi - s.put_lo[d]] = r1;
      s.put_fr2[d][gi - s.put_lo[d]] = r2;
    }
  return (a.nn & 0xffff) - 1;
}

// ------------------------------------------------------------ force (Eqs. 7, 17-24) ----
// Pairwise sums over r_ij < max(H_i, H_j) (R3), written with g = G r = f dW/dr (the r
// factors cancel):
//   A = P/rho^2, Pi_ij = -abar mu v_sig / rhobar (R9), gbar = (g_i + g_j)/2,
//   T = A_i g_i + A_j g_j + Pi_ij gbar  (= S_ij r),   a_i = -sum_j m_j T r_ij / r,
//   du_i = sum_j m_j [(A_i g_i + Pi gbar / 2)(v_ij . r_hat) + D_ij]  (Eq. 18 + R10 + Eq. 19/R11),
//   D_ij = alpha_c,ij v_c,ij (u_i - u_j)(g_i + g_j) / (rho_i + rho_j)  (Eqs. 20, 22; R12, R13).
// T is evaluated from operands symmetric in (i, j), so the pair terms of i and j are exact
// negatives (momentum and energy conserving up to the summation rounding).

// Operands of one side of a force pair: 1/h, v, m, the fr1 / fr2 records, P = A rho^2.
struct ForceSide {
  float hinv;
  float4 v;  // (v, m)
  float4 a;  // fr1: A, K, c, rho
  float4 b;  // fr2: B, (P + kPeps) alpha_c, u, alpha_v
  float P;
};

// Both sides of the unordered pair (i, j) (pair-once force loop), r_ij = (dx, dy, dz) = r_i - r_j:
// i's terms added to acc (a_i, du_i), j's returned in jo (a_j, du_j):
//   a_i -= m_j T r_ij / r,  a_j += m_i T r_ij / r  (Eq. 17: antisymmetric, momentum exact),
//   du_i += m_j [(A_i g_i + Pi gbar / 2)(v_ij . r_hat) + D_ij],
//   du_j += m_i [(A_j g_j + Pi gbar / 2)(v_ij . r_hat) - D_ij]  (v_ji . r_ji = v_ij . r_ij, D_ji = -D_ij).
// Membership needs no test: g_i = g_j = 0 beyond both supports, so every term vanishes.
// alpha_c,ij (Eq. 20) = (P_i ac_i + P_j ac_j) / (P_i + P_j), the mean when P_i + P_j = 0 (R13),
// is ((P_i + e) ac_i + (P_j + e) ac_j) / (P_i + P_j + 2e) with e = kPeps (grad_epilogue stores
// (P + e) ac): the mean when both P vanish, the weighted mean to a relative 1e-30 / P otherwise.
// Returns whether the pair has any term (g_i + g_j != 0).
__device__ __forceinline__ bool force_pair2(float4& acc, float4& jo, float dx, float dy, float dz, const ForceSide& I,
                                            const ForceSide& J, float beta) {
  // (r^2 + 1e-30: rinv_safe's floor folded into the first FMA; no pair has 0 < r^2 < 1e-20)
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, 1e-30f)));
  const float rinv = rsqrtf(r2);
  const float r = r2 * rinv;
  const float gI = I.a.y * m4_dwp(r * I.hinv);  // g_i = G_i r = f_i dW/dr(h_i)
  const float gJ = J.a.y * m4_dwp(r * J.hinv);
  const float vr = fmaf(I.v.z - J.v.z, dz, fmaf(I.v.y - J.v.y, dy, (I.v.x - J.v.x) * dx));
  const float vrr = vr * rinv;
  const float mu = fminf(vrr, 0.f);
  const float vs = fmaf(-beta, mu, I.a.z + J.a.z);
  const float irs = __fdividef(1.f, I.a.w + J.a.w);
  const float gs = gI + gJ;
  const float gsr = gs * irs;
  // X = 4 abar mu v_sig (g_i + g_j) / (rho_i + rho_j):  Pi_ij gbar = -X / 4
  const float X = ((I.b.w + J.b.w) * (I.b.x + J.b.x)) * (mu * vs) * gsr;
  const float AgI = I.a.x * gI, AgJ = J.a.x * gJ;
  const float Tr = fmaf(-0.25f, X, AgI + AgJ) * rinv;  // S_ij = T / r
  const float mTi = J.v.w * Tr, mTj = I.v.w * Tr;
  acc.x = fmaf(-mTi, dx, acc.x);
  acc.y = fmaf(-mTi, dy, acc.y);
  acc.z = fmaf(-mTi, dz, acc.z);
  jo.x = mTj * dx;
  jo.y = mTj * dy;
  jo.z = mTj * dz;
  const float acij = __fdividef(I.b.y + J.b.y, I.P + J.P + 2.f * kPeps);
  const float vc = fabsf(vrr) + sqrtf(2.f * fabsf(I.P - J.P) * irs);
  const float D = acij * vc * (I.b.z - J.b.z) * gsr;
  const float hX = -0.125f * X;
  acc.w = fmaf(J.v.w, fmaf(hX + AgI, vrr, D), acc.w);
  jo.w = I.v.w * fmaf(hX + AgJ, vrr, -D);
  return gs != 0.f;
}

}  // namespace sph
