// sph_api.cu -- the C-ABI of libsph (include/sph.h): context, cell binning (device radix
// sort by cell key, SWIFT's cell tree + sort tasks replaced), orchestration
// of the three interaction loops and the h iteration, kick/drift, read-back.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "../../include/sph.h"
#include "sph_internal.cuh"

using namespace sph;

namespace {

constexpr int kLcapInit = 96;         // neighbour-list capacity per particle (entries, multiple of 8)
constexpr size_t kSmemMax = 227 * 1024;
constexpr size_t kSmemTarget = 106 * 1024;  // two CTAs per SM for the largest (force) tile (+ static smem)

__global__ void k_hmax(int n, const uint4* __restrict__ xh, unsigned int* out) {
  unsigned int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, xh[i].w);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);  // positive f32 order as u32
}

__global__ void k_keys(int n, const uint4* __restrict__ xh, int nx, int ny, int nz, unsigned int* keys,
                       unsigned int* perm) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint4 x = xh[i];
  unsigned int cx = (unsigned int)(((unsigned long long)x.x * (unsigned)nx) >> 32);
  unsigned int cy = (unsigned int)(((unsigned long long)x.y * (unsigned)ny) >> 32);
  unsigned int cz = (unsigned int)(((unsigned long long)x.z * (unsigned)nz) >> 32);
  keys[i] = (cx * ny + cy) * nz + cz;
  perm[i] = i;
}

// cell_start[c] = first sorted index with key >= c, for c in [0, ncells]
__global__ void k_cell_start(int n, int ncells, const unsigned int* __restrict__ keys, int* cell_start) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  int lo = (p == 0) ? 0 : (int)keys[p - 1] + 1;
  int hi = (p == n) ? ncells : (int)keys[p];
  for (int c = lo; c <= hi; ++c) cell_start[c] = p;
}

struct Persist {
  uint4* xh;
  float4* vm;
  float* u;
  float* av;
  float* ac;
  float* dprev;
  int64_t* uid;
  int32_t* orig;
  float4* acc;
};

__global__ void k_permute(int n, const unsigned int* __restrict__ perm, Persist src, Persist dst) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int i = (int)perm[p];
  dst.xh[p] = src.xh[i];
  dst.vm[p] = src.vm[i];
  dst.u[p] = src.u[i];
  dst.av[p] = src.av[i];
  dst.ac[p] = src.ac[i];
  dst.dprev[p] = src.dprev[i];
  dst.uid[p] = src.uid[i];
  dst.orig[p] = src.orig[i];
  dst.acc[p] = src.acc[i];
}

// caller arrays (any order) -> persistent state (caller order; the next rebuild sorts it)
__global__ void k_ingest(int n, const uint32_t* __restrict__ X, const float* __restrict__ v,
                         const float* __restrict__ m, const float* __restrict__ u, const float* __restrict__ h,
                         const float* __restrict__ av, const float* __restrict__ ac, const float* __restrict__ dp,
                         const int64_t* __restrict__ id, Persist d) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  d.xh[i] = make_uint4(X[3 * i], X[3 * i + 1], X[3 * i + 2], __float_as_uint(h[i]));
  d.vm[i] = make_float4(v[3 * i], v[3 * i + 1], v[3 * i + 2], m[i]);
  d.u[i] = u[i];
  d.av[i] = av ? av[i] : 0.1f;
  d.ac[i] = ac ? ac[i] : 0.0f;
  d.dprev[i] = dp ? dp[i] : 0.0f;
  d.uid[i] = id ? id[i] : (int64_t)i;
  d.orig[i] = i;
  d.acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Kick v += a dt_k, u = max(0, u + du dt_k); drift x += v dt_d on the 2^-32 L
// grid, rounded to nearest, wrapping mod 2^32 (R25).
__global__ void k_kick_drift(int n, uint4* xh, float4* vm, float* u, const float4* __restrict__ acc, float dtk,
                             float dtd, double fx, double fy, double fz, const float4* __restrict__ dvc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (dvc && dtd != 0.f) {
    // h prediction in the drift: d ln h/dt = -(1/3) d ln rho/dt = (div v)/3 (continuity)
    float h = __uint_as_float(xh[i].w) * __expf(dtd * dvc[i].w * (1.f / 3.f));
    reinterpret_cast<unsigned int*>(&xh[i])[3] = __float_as_uint(h);
  }
  float4 a = acc[i];
  float4 v = vm[i];
  v.x = fmaf(a.x, dtk, v.x);
  v.y = fmaf(a.y, dtk, v.y);
  v.z = fmaf(a.z, dtk, v.z);
  vm[i] = v;
  u[i] = fmaxf(0.f, fmaf(a.w, dtk, u[i]));
  if (dtd != 0.f) {
    uint4 x = xh[i];
    x.x += (unsigned int)(long long)llrint((double)v.x * (double)dtd * fx);
    x.y += (unsigned int)(long long)llrint((double)v.y * (double)dtd * fy);
    x.z += (unsigned int)(long long)llrint((double)v.z * (double)dtd * fz);
    xh[i] = x;
  }
}

// out[orig[p] * comps + c] = src[p * stride + off + c]   (32-bit or 64-bit elements)
__global__ void k_scatter32(int n, const uint32_t* __restrict__ src, int stride, int off, int comps,
                            const int32_t* __restrict__ orig, uint32_t* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int o = orig[p];
  for (int c = 0; c < comps; ++c) out[(size_t)o * comps + c] = src[(size_t)p * stride + off + c];
}
__global__ void k_scatter64(int n, const uint64_t* __restrict__ src, const int32_t* __restrict__ orig, uint64_t* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  out[orig[p]] = src[p];
}

inline int nblk(long long n, int t) { return (int)((n + t - 1) / t); }

}  // namespace

struct sph_ctx {
  sph_config cfg{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int device = 0;
  int n = 0;
  bool poisoned = false;
  bool stale = true;          // grid must be rebuilt before the next loop
  bool lists_stale = true;    // neighbour lists must be rebuilt before the next loop
  size_t nbr_cap = 0;         // allocated list entries (n x lcap)
  int lcap = kLcapInit;
  bool dprev_valid = false;
  bool dvc_valid = false;     // dvc (div v) is from a density pass in the current particle order
  bool density_done = false, gradient_done = false;
  std::string err;
  DevGrid grid{};
  DevPhys phys{};
  DevState s{};
  Persist alt{};              // second buffers of the persistent arrays (permutation target)
  int* cell_start = nullptr;
  size_t cell_cap = 0;
  unsigned int *keys = nullptr, *keys_alt = nullptr, *perm = nullptr, *perm_alt = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  uint8_t* blk[2] = {nullptr, nullptr};
  size_t blk_cap = 0;
  DevCounters* ctr = nullptr;     // device
  DevCounters* ctr_h = nullptr;   // pinned host mirror
  unsigned int* scratch = nullptr;  // device scalars
  unsigned int* scratch_h = nullptr;
  void* out_tmp = nullptr;
  size_t out_tmp_bytes = 0;
  sph_counters counters{};
  long long launches = 0;
};

namespace {

sph_status fail(sph_ctx* c, sph_status st, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (st == SPH_ERR_CUDA || st == SPH_ERR_NCCL) c->poisoned = true;
  }
  return st;
}

#define CK(expr)                                                                                    \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      if (e_ == cudaErrorMemoryAllocation) return fail(c, SPH_ERR_OOM, std::string(#expr) + ": out of device memory"); \
      return fail(c, SPH_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));           \
    }                                                                                               \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

sph_status alloc_state(sph_ctx* c) {
  const size_t n = (size_t)c->n;
  DevState& s = c->s;
  CK(dalloc(&s.xh, n)); CK(dalloc(&s.vm, n)); CK(dalloc(&s.u, n)); CK(dalloc(&s.av, n)); CK(dalloc(&s.ac, n));
  CK(dalloc(&s.dprev, n)); CK(dalloc(&s.uid, n)); CK(dalloc(&s.orig, n)); CK(dalloc(&s.acc, n));
  Persist& a = c->alt;
  CK(dalloc(&a.xh, n)); CK(dalloc(&a.vm, n)); CK(dalloc(&a.u, n)); CK(dalloc(&a.av, n)); CK(dalloc(&a.ac, n));
  CK(dalloc(&a.dprev, n)); CK(dalloc(&a.uid, n)); CK(dalloc(&a.orig, n)); CK(dalloc(&a.acc, n));
  CK(dalloc(&s.dens, n)); CK(dalloc(&s.dvc, n)); CK(dalloc(&s.count, n)); CK(dalloc(&s.fin, n));
  CK(dalloc(&s.gq, n)); CK(dalloc(&s.hlo, n)); CK(dalloc(&s.hhi, n)); CK(dalloc(&s.iters, n));
  CK(dalloc(&s.active, n)); CK(dalloc(&s.grad, n)); CK(dalloc(&s.fr1, n)); CK(dalloc(&s.fr2, n));
  CK(dalloc(&s.fr3, n)); CK(dalloc(&s.vsig, n)); CK(dalloc(&s.countf, n));
  CK(dalloc(&s.ncount, n)); CK(dalloc(&s.hbuild, n));
  CK(dalloc(&s.nbr, n * (size_t)c->lcap));
  c->nbr_cap = n * (size_t)c->lcap;
  CK(dalloc(&c->keys, n)); CK(dalloc(&c->keys_alt, n)); CK(dalloc(&c->perm, n)); CK(dalloc(&c->perm_alt, n));
  CK(dalloc(&c->ctr, 1));
  CK(cudaMallocHost((void**)&c->ctr_h, sizeof(DevCounters)));
  CK(dalloc(&c->scratch, 16));
  CK(cudaMallocHost((void**)&c->scratch_h, 16 * sizeof(unsigned int)));
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, c->keys, c->keys_alt, c->perm, c->perm_alt, (int)n, 0, 32);
  c->sort_tmp_bytes = tmp;
  CK(cudaMalloc(&c->sort_tmp, std::max<size_t>(tmp, 1)));
  return SPH_OK;
}

Persist persist_of(const DevState& s) {
  return Persist{s.xh, s.vm, s.u, s.av, s.ac, s.dprev, s.uid, s.orig, s.acc};
}

void set_persist(DevState& s, const Persist& p) {
  s.xh = p.xh; s.vm = p.vm; s.u = p.u; s.av = p.av; s.ac = p.ac; s.dprev = p.dprev; s.uid = p.uid;
  s.orig = p.orig; s.acc = p.acc;
}

sph_status validate_cfg(sph_ctx* c, const sph_config* cfg) {
  if (!cfg) return fail(c, SPH_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->struct_size != sizeof(sph_config)) return fail(c, SPH_ERR_INVALID_ARG, "sph_config.struct_size mismatch");
  if (cfg->gamma_k != 2.0f) return fail(c, SPH_ERR_INVALID_ARG, "gamma_k must be 2 (M4 kernel support, R1)");
  for (int a = 0; a < 3; ++a)
    if (!(cfg->box[a] > 0.0)) return fail(c, SPH_ERR_INVALID_ARG, "box sides must be > 0");
  if (!(cfg->eta > 0.f) || !(cfg->h_tol > 0.f) || cfg->h_max_iter < 0 || !(cfg->gamma_eos > 1.f) ||
      !(cfg->alpha_v_max > 0.f) || !(cfg->c_cfl > 0.f) || cfg->cell_skin < 0.f)
    return fail(c, SPH_ERR_INVALID_ARG, "invalid physics parameter");
  if (cfg->nranks != 1 || cfg->rank != 0)
    return fail(c, SPH_ERR_INVALID_ARG, "multi-rank contexts are not supported by this build (nranks must be 1)");
  return SPH_OK;
}

void fill_phys(sph_ctx* c) {
  const sph_config& k = c->cfg;
  DevPhys& p = c->phys;
  p.gamma_k = k.gamma_k;
  p.eta3 = k.eta * k.eta * k.eta;
  p.h_tol = k.h_tol;
  p.pi_eta3 = kPi * p.eta3;
  p.h_max_iter = k.h_max_iter;
  p.fh_mode = k.fh_mode;
  p.gamma_eos = k.gamma_eos;
  p.beta = k.beta;
  p.alpha_v_max = k.alpha_v_max;
  p.ell = k.ell;
  p.alpha_c_min = k.alpha_c_min;
  p.alpha_c_max = k.alpha_c_max;
  p.beta_c = k.beta_c;
  p.c_cfl = k.c_cfl;
}

sph_status ingest(sph_ctx* c, const sph_particles_in* in) {
  if (!in || in->n != c->n) return fail(c, SPH_ERR_INVALID_ARG, "particle count mismatch");
  if (!in->X || !in->v || !in->m || !in->u || !in->h) return fail(c, SPH_ERR_INVALID_ARG, "required particle array is NULL");
  const size_t n = (size_t)c->n;
  // stage host arrays through the (reused) output buffer region on the device
  const uint32_t* X = in->X;
  const float *v = in->v, *m = in->m, *u = in->u, *h = in->h, *av = in->alpha_v, *ac = in->alpha_c,
              *dp = in->div_prev;
  const int64_t* id = in->id;
  void* tmp = nullptr;
  if (!in->on_device) {
    size_t bytes = n * (12 + 12 + 4 * 3) + (av ? 4 * n : 0) + (ac ? 4 * n : 0) + (dp ? 4 * n : 0) + (id ? 8 * n : 0);
    if (c->out_tmp_bytes < bytes) {
      if (c->out_tmp) cudaFree(c->out_tmp);
      c->out_tmp = nullptr;
      c->out_tmp_bytes = 0;
      CK(cudaMalloc(&c->out_tmp, bytes));
      c->out_tmp_bytes = bytes;
    }
    tmp = c->out_tmp;
    char* d = (char*)tmp;
    auto up = [&](const void* src, size_t b) -> void* {
      void* dst = d;
      cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, c->stream);
      d += (b + 15) & ~size_t(15);
      return dst;
    };
    X = (const uint32_t*)up(in->X, 12 * n);
    v = (const float*)up(in->v, 12 * n);
    m = (const float*)up(in->m, 4 * n);
    u = (const float*)up(in->u, 4 * n);
    h = (const float*)up(in->h, 4 * n);
    if (av) av = (const float*)up(in->alpha_v, 4 * n);
    if (ac) ac = (const float*)up(in->alpha_c, 4 * n);
    if (dp) dp = (const float*)up(in->div_prev, 4 * n);
    if (id) id = (const int64_t*)up(in->id, 8 * n);
    CK(cudaGetLastError());
  }
  k_ingest<<<nblk(n, 256), 256, 0, c->stream>>>((int)n, X, v, m, u, h, av, ac, dp, id, persist_of(c->s));
  c->launches++;
  CK(cudaGetLastError());
  c->dprev_valid = dp != nullptr;
  c->dvc_valid = false;
  c->stale = true;
  c->density_done = c->gradient_done = false;
  return SPH_OK;
}

sph_status sync_ctr(sph_ctx* c) {
  CK(cudaMemcpyAsync(c->ctr_h, c->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return SPH_OK;
}

sph_status reset_ctr(sph_ctx* c) {
  CK(cudaMemsetAsync(c->ctr, 0, sizeof(DevCounters), c->stream));
  return SPH_OK;
}

float ulp_of(float x) {
  int e;
  std::frexp(x, &e);  // x = f 2^e, f in [0.5, 1)
  return std::ldexp(1.0f, e - 24);
}

// Choose the grid for the current h, sort, permute, and size the CTA tiles.
sph_status rebuild(sph_ctx* c) {
  const int n = c->n;
  CK(cudaMemsetAsync(c->scratch, 0, 16 * sizeof(unsigned int), c->stream));
  k_hmax<<<std::min(nblk(n, 256), 1184), 256, 0, c->stream>>>(n, c->s.xh, c->scratch);
  c->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->scratch_h, c->scratch, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  float hmax;
  std::memcpy(&hmax, c->scratch_h, 4);
  if (!(hmax > 0.f) || !std::isfinite(hmax)) return fail(c, SPH_ERR_INVALID_ARG, "smoothing lengths must be finite and > 0");
  const double Hs = (double)c->cfg.gamma_k * hmax * (1.0 + c->cfg.cell_skin);
  DevGrid& g = c->grid;
  int nc[3];
  for (int a = 0; a < 3; ++a) {
    double k = std::floor(c->cfg.box[a] / Hs);
    if (k < 3) {
      char b[256];
      snprintf(b, sizeof b, "support radius %.6g leaves fewer than 3 cells along axis %d (box %.6g)", Hs, a, c->cfg.box[a]);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
    nc[a] = (int)std::min(k, 1024.0);
  }
  while ((long long)nc[0] * nc[1] * nc[2] > (1LL << 30)) { for (int a = 0; a < 3; ++a) nc[a] = std::max(3, nc[a] / 2); }
  g.nx = nc[0]; g.ny = nc[1]; g.nz = nc[2];
  g.ncells = g.nx * g.ny * g.nz;
  for (int a = 0; a < 3; ++a) {
    g.side[a] = (float)(c->cfg.box[a] / nc[a]);
    g.scale[a] = (float)(c->cfg.box[a] * std::ldexp(1.0, -32));
    g.dscale[a] = c->cfg.box[a] * std::ldexp(1.0, -32);
  }
  g.side_min = std::min(g.side[0], std::min(g.side[1], g.side[2]));
  // keys, sort, cell ranges, permutation
  if (c->cell_cap < (size_t)g.ncells + 1) {
    if (c->cell_start) cudaFree(c->cell_start);
    c->cell_start = nullptr;
    CK(dalloc(&c->cell_start, (size_t)g.ncells + 1));
    c->cell_cap = (size_t)g.ncells + 1;
  }
  k_keys<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->s.xh, g.nx, g.ny, g.nz, c->keys, c->perm);
  c->launches++;
  CK(cudaGetLastError());
  int bits = 1;
  while ((1LL << bits) < g.ncells) ++bits;
  size_t tmp = c->sort_tmp_bytes;
  CK(cub::DeviceRadixSort::SortPairs(c->sort_tmp, tmp, c->keys, c->keys_alt, c->perm, c->perm_alt, n, 0, bits,
                                     c->stream));
  c->launches += 1 + (bits + 7) / 8;
  k_cell_start<<<nblk(n + 1, 256), 256, 0, c->stream>>>(n, g.ncells, c->keys_alt, c->cell_start);
  c->launches++;
  k_permute<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->perm_alt, persist_of(c->s), c->alt);
  c->launches++;
  CK(cudaGetLastError());
  Persist old = persist_of(c->s);
  set_persist(c->s, c->alt);
  c->alt = old;
  // CTA blocks: BX x BY grid columns x KZ cells (BX, BY = 2 when the grid allows: the tile of
  // (BX+2)(BY+2) columns is then ~2x smaller per owned particle than with single columns)
  g.bx = g.nx >= 6 ? 2 : 1;
  g.by = g.ny >= 6 ? 2 : 1;
  g.nbx = (g.nx + g.bx - 1) / g.bx;
  g.nby = (g.ny + g.by - 1) / g.by;
  const double occ = (double)n / g.ncells;
  const int kz_max = std::min(kMaxTileCellsZ - 2, g.nz > 3 ? g.nz - 3 : 1);
  int KZ = (int)std::lround(kernel_threads() / std::max(occ * g.bx * g.by, 1e-3));
  if (c->cfg.tile_cells_z > 0) KZ = c->cfg.tile_cells_z;
  KZ = std::max(1, std::min(KZ, kz_max));
  for (;;) {
    g.KZ = KZ;
    g.nzb = (g.nz + KZ - 1) / KZ;
    g.nblocks = g.nbx * g.nby * g.nzb;
    CK(cudaMemsetAsync(c->scratch + 1, 0, 4, c->stream));
    CK(launch_tile_sizes(g, c->cell_start, (int*)(c->scratch + 1), c->stream));
    c->launches++;
    CK(cudaMemcpyAsync(c->scratch_h + 1, c->scratch + 1, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    g.tcap = std::max(32, (int)c->scratch_h[1]);
    g.lcap = c->lcap;
    g.skin = c->cfg.cell_skin;
    const bool fits = force_smem(g) <= kSmemMax && lists_smem(g) <= kSmemMax && g.tcap < 65535;
    if (fits && (force_smem(g) <= kSmemTarget || KZ == 1)) break;
    if (fits && c->cfg.tile_cells_z > 0) break;
    if (KZ == 1) {
      char b[256];
      snprintf(b, sizeof b, "largest cell tile (%d particles) exceeds shared memory; h contrast too high for one grid", g.tcap);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
    KZ = std::max(1, KZ - 1);
  }
  // rounding error of a tile coordinate: offsets reach (B/2 + 1) cells from the block centre
  const float max_off = std::max(std::max((0.5f * g.bx + 1.0f) * g.side[0], (0.5f * g.by + 1.0f) * g.side[1]),
                                 (0.5f * g.KZ + 1.0f) * g.side[2]);
  g.eabs = 4.0f * ulp_of(max_off) * 2.0f;  // 8 x (ulp/2): two coordinates per difference, with margin
  if ((size_t)g.nblocks > c->blk_cap) {
    for (int k = 0; k < 2; ++k) {
      if (c->blk[k]) cudaFree(c->blk[k]);
      c->blk[k] = nullptr;
      CK(dalloc(&c->blk[k], (size_t)g.nblocks));
    }
    c->blk_cap = (size_t)g.nblocks;
  }
  c->stale = false;
  c->lists_stale = true;
  c->dvc_valid = false;
  return SPH_OK;
}

// Build the neighbour lists for the current grid and h (growing the capacity if needed).
sph_status build_lists(sph_ctx* c) {
  for (int attempt = 0; attempt < 4; ++attempt) {
    c->grid.lcap = c->lcap;
    CK(cudaMemsetAsync(&c->ctr->list_overflow, 0, sizeof(int), c->stream));
    CK(cudaMemsetAsync(&c->ctr->nonfinite, 0, sizeof(int), c->stream));
    if (lists_smem(c->grid) > kSmemMax) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "neighbour lists exceed shared memory");
    CK(launch_lists(c->grid, c->phys, c->s, c->cell_start, c->ctr, c->stream));
    c->launches++;
    sph_status st = sync_ctr(c);
    if (st != SPH_OK) return st;
    int over = c->ctr_h->list_overflow;
    if (c->ctr_h->nonfinite == 2) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
    if (over == 0) {
      c->lists_stale = false;
      return SPH_OK;
    }
    int need = ((int)(over * 1.25) + 7) & ~7;
    if (need > 8192) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "neighbour list longer than 8192 entries");
    c->lcap = need;
    size_t want = (size_t)c->n * c->lcap;
    if (want > c->nbr_cap) {
      cudaFree(c->s.nbr);
      c->s.nbr = nullptr;
      CK(dalloc(&c->s.nbr, want));
      c->nbr_cap = want;
    }
  }
  return fail(c, SPH_ERR_CUDA, "internal: neighbour list capacity did not converge");
}

}  // namespace

extern "C" {

int sph_abi_version(void) { return SPH_ABI_VERSION; }

void sph_config_default(sph_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->struct_size = sizeof(sph_config);
  cfg->box[0] = cfg->box[1] = cfg->box[2] = 1.0;
  cfg->gamma_k = 2.0f;
  cfg->eta = 1.2348f;
  cfg->h_tol = 1e-4f;
  cfg->h_max_iter = 32;
  cfg->cell_skin = 0.05f;
  cfg->gamma_eos = 5.0f / 3.0f;
  cfg->beta = 3.0f;
  cfg->alpha_v_max = 2.0f;
  cfg->ell = 0.05f;
  cfg->alpha_c_min = 0.0f;
  cfg->alpha_c_max = 1.0f;
  cfg->beta_c = 1.0f;
  cfg->c_cfl = 0.1f;
  cfg->fh_mode = 0;
  cfg->device = 0;
  cfg->stream = nullptr;
  cfg->rank = 0;
  cfg->nranks = 1;
  cfg->tile_cells_z = 0;
  cfg->predict_h = 1;
}

sph_status sph_create(const sph_config* cfg, const sph_particles_in* in, sph_ctx** out) {
  if (!out) return SPH_ERR_INVALID_ARG;
  *out = nullptr;
  sph_ctx* c = new (std::nothrow) sph_ctx();
  if (!c) return SPH_ERR_OOM;
  sph_status st = validate_cfg(c, cfg);
  if (st != SPH_OK) { delete c; return st; }
  if (!in || in->n <= 0 || in->n > (int64_t)0x7fffffff) { delete c; return SPH_ERR_INVALID_ARG; }
  c->cfg = *cfg;
  c->n = (int)in->n;
  c->device = cfg->device;
  auto bail = [&](sph_status s) { sph_destroy(c); return s; };
  if (cudaSetDevice(c->device) != cudaSuccess) return bail(SPH_ERR_CUDA);
  if (cfg->stream) {
    c->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SPH_ERR_CUDA);
    c->own_stream = true;
  }
  fill_phys(c);
  if ((st = alloc_state(c)) != SPH_OK) return bail(st);
  if ((st = ingest(c, in)) != SPH_OK) return bail(st);
  if ((st = rebuild(c)) != SPH_OK) return bail(st);
  *out = c;
  return SPH_OK;
}

#define GUARD(c)                                                   \
  do {                                                             \
    if (!(c)) return SPH_ERR_INVALID_ARG;                          \
    if ((c)->poisoned) return SPH_ERR_STATE;                       \
    if (cudaSetDevice((c)->device) != cudaSuccess) return SPH_ERR_CUDA; \
  } while (0)

sph_status sph_set_particles(sph_ctx* c, const sph_particles_in* in) {
  GUARD(c);
  return ingest(c, in);
}

sph_status sph_rebuild_cells(sph_ctx* c) {
  GUARD(c);
  return rebuild(c);
}

sph_status sph_density(sph_ctx* c, sph_density_stats* stats) {
  GUARD(c);
  sph_status st;
  if (c->stale && (st = rebuild(c)) != SPH_OK) return st;
  if (c->lists_stale && (st = build_lists(c)) != SPH_OK) return st;
  int rebuilds = 0;
  long long pairs_all = 0;
  int pass = 0, passes_run = 0;
  unsigned long long final_pairs = 0;
  int unconverged = 0;
  if ((st = reset_ctr(c)) != SPH_OK) return st;
  for (;;) {
    uint8_t* bin = c->blk[pass & 1];
    uint8_t* bout = c->blk[(pass + 1) & 1];
    CK(cudaMemsetAsync(bout, 0, (size_t)c->grid.nblocks, c->stream));
    CK(cudaMemsetAsync(&c->ctr->active_next, 0, 3 * sizeof(int), c->stream));  // active_next, list_stale, overflow
    CK(cudaMemsetAsync(&c->ctr->h_exceeds, 0, sizeof(int), c->stream));
    CK(launch_density(c->grid, c->phys, c->s, c->cell_start, pass, bin, bout, 1.f + c->cfg.cell_skin, c->ctr,
                      c->stream));
    c->launches++;
    ++passes_run;
    if ((st = sync_ctr(c)) != SPH_OK) return st;
    if (c->ctr_h->nonfinite == 2) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
    if (c->ctr_h->active_next == 0) break;
    if (c->ctr_h->h_exceeds) {
      // an h grew past what the cell grid holds: rebin with the new h and restart the passes
      if (++rebuilds > 8) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "h kept outgrowing the cell grid");
      pairs_all += (long long)c->ctr_h->pairs_all;
      if ((st = rebuild(c)) != SPH_OK) return st;
      if ((st = build_lists(c)) != SPH_OK) return st;
      if ((st = reset_ctr(c)) != SPH_OK) return st;
      pass = 0;
      continue;
    }
    if (c->ctr_h->list_stale) {
      // an h outgrew its list radius: rebuild the lists for the current h, keep iterating
      if ((st = build_lists(c)) != SPH_OK) return st;
    }
    ++pass;
  }
  final_pairs = c->ctr_h->pairs;
  pairs_all += (long long)c->ctr_h->pairs_all;
  unconverged = c->ctr_h->unconverged;
  c->counters.pairs_density = (int64_t)final_pairs;
  c->counters.pairs_h_iter = pairs_all;
  c->density_done = true;
  c->gradient_done = false;
  c->dvc_valid = true;
  if (stats) {
    stats->iterations = passes_run;
    stats->unconverged = unconverged;
    stats->rebuilds = rebuilds;
    stats->reserved = 0;
    stats->pairs_density = (int64_t)final_pairs;
    stats->pairs_h_iter = pairs_all;
  }
  if (unconverged > 0) {
    char b[160];
    snprintf(b, sizeof b, "h iteration: %d particles not converged after %d Newton updates", unconverged,
             c->cfg.h_max_iter);
    c->err = b;
    return SPH_ERR_NOT_CONVERGED;
  }
  return SPH_OK;
}

sph_status sph_gradient(sph_ctx* c, float dt) {
  GUARD(c);
  if (!c->density_done) return fail(c, SPH_ERR_STATE, "sph_gradient needs a completed sph_density");
  if (!(dt > 0.f) || !std::isfinite(dt)) return fail(c, SPH_ERR_INVALID_ARG, "sph_gradient: dt must be > 0 (S:246)");
  sph_status st;
  if ((st = reset_ctr(c)) != SPH_OK) return st;
  CK(launch_gradient(c->grid, c->phys, c->s, c->cell_start, dt, c->dprev_valid ? 0 : 1, c->ctr, c->stream));
  c->launches++;
  CK(cudaMemcpyAsync(&c->counters.pairs_gradient, &c->ctr->pairs, 8, cudaMemcpyDeviceToHost, c->stream));
  c->dprev_valid = true;
  c->gradient_done = true;
  return SPH_OK;
}

sph_status sph_force(sph_ctx* c, float* dt_next) {
  GUARD(c);
  if (!c->gradient_done) return fail(c, SPH_ERR_STATE, "sph_force needs a completed sph_gradient");
  sph_status st;
  if ((st = reset_ctr(c)) != SPH_OK) return st;
  unsigned int inf_bits = 0x7f800000u;
  CK(cudaMemcpyAsync(&c->ctr->dt_bits, &inf_bits, 4, cudaMemcpyHostToDevice, c->stream));
  CK(launch_force(c->grid, c->phys, c->s, c->cell_start, c->ctr, c->stream));
  c->launches++;
  if ((st = sync_ctr(c)) != SPH_OK) return st;
  c->counters.pairs_force = (int64_t)c->ctr_h->pairs;
  float dt;
  std::memcpy(&dt, &c->ctr_h->dt_bits, 4);
  if (dt_next) *dt_next = dt;
  if (c->ctr_h->nonfinite == 2) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
  if (c->ctr_h->nonfinite || !std::isfinite(dt)) return fail(c, SPH_ERR_NUMERIC, "non-finite acceleration, v_sig or dt (S:262)");
  return SPH_OK;
}

sph_status sph_kick_drift(sph_ctx* c, float dt_kick, float dt_drift) {
  GUARD(c);
  if (!std::isfinite(dt_kick) || !std::isfinite(dt_drift)) return fail(c, SPH_ERR_INVALID_ARG, "non-finite dt");
  const double f[3] = {std::ldexp(1.0, 32) / c->cfg.box[0], std::ldexp(1.0, 32) / c->cfg.box[1],
                       std::ldexp(1.0, 32) / c->cfg.box[2]};
  const float4* dvc = (c->cfg.predict_h && c->dvc_valid) ? c->s.dvc : nullptr;
  k_kick_drift<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->s.xh, c->s.vm, c->s.u, c->s.acc, dt_kick, dt_drift, f[0],
                                                     f[1], f[2], dvc);
  c->launches++;
  CK(cudaGetLastError());
  if (dt_drift != 0.f) c->stale = true;
  c->density_done = c->gradient_done = false;
  return SPH_OK;
}

sph_status sph_get(sph_ctx* c, int field, void* dst, int on_device) {
  GUARD(c);
  if (!dst) return fail(c, SPH_ERR_INVALID_ARG, "dst is NULL");
  const DevState& s = c->s;
  const void* src = nullptr;
  int stride = 1, off = 0, comps = 1, wide = 0;
  switch (field) {
    case SPH_F_X: src = s.xh; stride = 4; comps = 3; break;
    case SPH_F_H: src = s.xh; stride = 4; off = 3; break;
    case SPH_F_V: src = s.vm; stride = 4; comps = 3; break;
    case SPH_F_M: src = s.vm; stride = 4; off = 3; break;
    case SPH_F_U: src = s.u; break;
    case SPH_F_RHO: src = s.dens; stride = 4; off = 0; break;
    case SPH_F_DRHO_DH: src = s.dens; stride = 4; off = 1; break;
    case SPH_F_NHAT: src = s.dens; stride = 4; off = 2; break;
    case SPH_F_DN_DH: src = s.dens; stride = 4; off = 3; break;
    case SPH_F_CURL: src = s.dvc; stride = 4; comps = 3; break;
    case SPH_F_DIV: src = s.dvc; stride = 4; off = 3; break;
    case SPH_F_COUNT: src = s.count; break;
    case SPH_F_F: src = s.fin; stride = 4; off = 0; break;
    case SPH_F_P: src = s.fin; stride = 4; off = 1; break;
    case SPH_F_C: src = s.fin; stride = 4; off = 2; break;
    case SPH_F_B: src = s.fin; stride = 4; off = 3; break;
    case SPH_F_VSIG_GRAD: src = s.grad; stride = 2; off = 0; break;
    case SPH_F_LAP_U: src = s.grad; stride = 2; off = 1; break;
    case SPH_F_ALPHA_V: src = s.av; break;
    case SPH_F_ALPHA_C: src = s.ac; break;
    case SPH_F_DIV_PREV: src = s.dprev; break;
    case SPH_F_A: src = s.acc; stride = 4; comps = 3; break;
    case SPH_F_DU: src = s.acc; stride = 4; off = 3; break;
    case SPH_F_VSIG: src = s.vsig; break;
    case SPH_F_COUNT_FORCE: src = s.countf; break;
    case SPH_F_ITERS: src = s.iters; break;
    case SPH_F_ID: src = s.uid; wide = 1; break;
    default: return fail(c, SPH_ERR_INVALID_ARG, "unknown field");
  }
  const size_t bytes = (size_t)c->n * comps * (wide ? 8 : 4);
  void* d = dst;
  if (!on_device) {
    if (c->out_tmp_bytes < bytes) {
      if (c->out_tmp) cudaFree(c->out_tmp);
      c->out_tmp = nullptr;
      c->out_tmp_bytes = 0;
      CK(cudaMalloc(&c->out_tmp, bytes));
      c->out_tmp_bytes = bytes;
    }
    d = c->out_tmp;
  }
  if (wide)
    k_scatter64<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, (const uint64_t*)src, s.orig, (uint64_t*)d);
  else
    k_scatter32<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, (const uint32_t*)src, stride, off, comps, s.orig,
                                                        (uint32_t*)d);
  c->launches++;
  CK(cudaGetLastError());
  if (!on_device) {
    CK(cudaMemcpyAsync(dst, d, bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return SPH_OK;
}

sph_status sph_get_counters(sph_ctx* c, sph_counters* out) {
  GUARD(c);
  if (!out) return SPH_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(c->stream));
  c->counters.coincident = -1;  // not tracked by the GPU loops
  c->counters.kernel_launches = c->launches;
  *out = c->counters;
  return SPH_OK;
}

sph_status sph_synchronize(sph_ctx* c) {
  GUARD(c);
  CK(cudaStreamSynchronize(c->stream));
  return SPH_OK;
}

const char* sph_last_error(const sph_ctx* c) { return c ? c->err.c_str() : "context is NULL"; }

sph_status sph_destroy(sph_ctx* c) {
  if (!c) return SPH_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  DevState& s = c->s;
  void* ptrs[] = {s.xh, s.vm, s.u, s.av, s.ac, s.dprev, s.uid, s.orig, s.acc, c->alt.xh, c->alt.vm, c->alt.u,
                  c->alt.av, c->alt.ac, c->alt.dprev, c->alt.uid, c->alt.orig, c->alt.acc, s.dens, s.dvc, s.count,
                  s.fin, s.gq, s.hlo, s.hhi, s.iters, s.active, s.grad, s.fr1, s.fr2, s.fr3, s.vsig, s.countf, s.nbr,
                  s.ncount, s.hbuild,
                  c->cell_start, c->keys, c->keys_alt, c->perm, c->perm_alt, c->sort_tmp, c->blk[0], c->blk[1],
                  c->ctr, c->scratch, c->out_tmp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->ctr_h) cudaFreeHost(c->ctr_h);
  if (c->scratch_h) cudaFreeHost(c->scratch_h);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return SPH_OK;
}

}  // extern "C"
