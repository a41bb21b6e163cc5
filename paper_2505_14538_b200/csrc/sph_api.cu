// sph_api.cu -- the C-ABI of libsph (include/sph.h): context, cell binning (device radix
// sort by cell key, SWIFT's cell tree + sort tasks replaced), orchestration
// of the three interaction loops and the h iteration, kick/drift, read-back, and
// the slab decomposition across ranks with its halo exchanges.
//
// Local particle layout (every array, cell order):  [left ghosts | owned | right ghosts].
// One rank: no ghosts, periodic grid.  Several ranks: rank r owns the grid planes
// [r nx/R, (r+1) nx/R) along x; the planes on either side are ghost planes received from the
// neighbours (cell side >= (1+skin) max H, so one plane is the whole halo).  The local grid
// has P + 2 planes along x (ghost, owned..., ghost) and is periodic in y and z.
#include <thrust/iterator/counting_iterator.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>
#include <nvtx3/nvtx3.hpp>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "../../include/sph.h"
#include "sph_comm.cuh"
#include "sph_internal.cuh"

using namespace sph;

namespace {

constexpr int kLcapInit = 96;         // neighbour-list capacity per particle (entries, multiple of 8)
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kMaxGhostPlanes = 16;     // slab path: ghost planes per side (wide particles)
constexpr size_t kSmemTarget = 107 * 1024;  // two CTAs per SM for the largest (force) tile (+ static smem)

__global__ void k_hmax(int n, const uint4* __restrict__ xh, unsigned int* out) {
  unsigned int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, xh[i].w);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);  // positive f32 order as u32
}

// histogram of the owned particles' x over nb equal bins of the box (balanced slab cuts)
__global__ void k_xhist(int n, const uint4* __restrict__ xh, int nb, unsigned int* hist) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&hist[(int)(((unsigned long long)xh[i].x * (unsigned)nb) >> 32)], 1u);
}

// ghost planes the owned particle needs (ghost_planes_needed) for a list radius Hfac h; a
// particle that left the slab counts at its nearest owned plane
__global__ void k_ghost_need(int n, const uint4* __restrict__ xh, DevGrid g, float Hfac, unsigned int* out) {
  unsigned int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint4 x = xh[i];
    long long d = (long long)(unsigned int)(x.x - g.x_lo);
    if ((unsigned long long)d >= g.wfix + ((1ull << 32) - g.wfix) / 2) d -= (1ll << 32);
    const long long q = d * (long long)g.nxo, w = (long long)g.wfix;
    long long pl = q >= 0 ? q / w : -((-q + w - 1) / w);
    pl = pl < 0 ? 0 : (pl >= g.nxo ? g.nxo - 1 : pl);
    const int k = (int)ceilf(Hfac * __uint_as_float(x.w) / g.side_min);
    m = max(m, (unsigned int)ghost_planes_needed(k, (int)pl, g.nxo));
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// cell key of each particle in the local grid (DevGrid slab fields); a particle outside the
// local planes gets the key ncells (sorted last) and is counted
__global__ void k_keys(int n, const uint4* __restrict__ xh, DevGrid g, unsigned int* keys, unsigned int* perm,
                       int* outside) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  uint4 x = xh[i];
  // offset from the slab start; the complement of the slab is split at its middle into
  // "left of the slab" (negative) and "right of the slab"
  long long d = (long long)(unsigned int)(x.x - g.x_lo);
  if ((unsigned long long)d >= g.wfix + ((1ull << 32) - g.wfix) / 2) d -= (1ll << 32);
  const long long q = d * (long long)g.nxo;
  const long long w = (long long)g.wfix;
  const long long pl = q >= 0 ? q / w : -((-q + w - 1) / w);  // floor
  const long long cx = pl + g.ix_first;
  unsigned int cy = (unsigned int)(((unsigned long long)x.y * (unsigned)ny) >> 32);
  const unsigned long long zq = (unsigned long long)x.z * (unsigned)nz;
  const unsigned int cz = (unsigned int)(zq >> 32);
  // low bits: the top zbits of the position inside the cell along z, so each cell's
  // particles come out sorted by z up to one bucket (the list kernel's z windows)
  const unsigned int zf = g.zbits ? (unsigned int)zq >> (32 - g.zbits) : 0u;
  if (cx < 0 || cx >= nx) {
    keys[i] = ((unsigned)nx * ny * nz) << g.zbits;
    atomicAdd(outside, 1);
  } else {
    keys[i] = ((((unsigned)cx * ny + cy) * nz + cz) << g.zbits) | zf;
  }
  perm[i] = i;
}

// cell_start[c] = first sorted index with cell(key) >= c, for c in [0, ncells]
__global__ void k_cell_start(int n, int ncells, int zbits, const unsigned int* __restrict__ keys, int* cell_start) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  int lo = (p == 0) ? 0 : min((int)(keys[p - 1] >> zbits) + 1, ncells + 1);
  int hi = (p == n) ? ncells : min((int)(keys[p] >> zbits), ncells);
  for (int c = lo; c <= hi; ++c) cell_start[c] = p;
}

// Coincident particles (a pair with r_ij = 0, j != i, contributes nothing and is counted).
// Exactly equal fixed-point positions give equal sort keys (cell + z sub-bucket), so a particle's
// coincident partners lie in its run of equal keys: flag every particle that has one and count the
// directed pairs.  p indexes the sorted owned particles (keys[p] belongs to xh[p]).
// (dup must be zero before the launch; each unordered pair is found once, by its first particle,
// which flags both and counts it twice)
__global__ void k_dup(int n, const unsigned int* __restrict__ keys, const uint4* __restrict__ xh, uint8_t* dup,
                      unsigned int* npairs) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const unsigned int k = keys[p];
  if (p + 1 >= n || keys[p + 1] != k) return;  // (most particles: the next key differs)
  const uint4 a = xh[p];
  unsigned int m = 0;
  for (int q = p + 1; q < n && keys[q] == k; ++q) {
    const uint4 b = xh[q];
    if (b.x == a.x && b.y == a.y && b.z == a.z) {
      dup[q] = 1;
      ++m;
    }
  }
  if (m) {
    dup[p] = 1;
    atomicAdd(npairs, 2u * m);
  }
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

Persist offset(const Persist& p, int o) {
  return Persist{p.xh + o, p.vm + o, p.u + o, p.av + o, p.ac + o, p.dprev + o, p.uid + o, p.orig + o, p.acc + o};
}

// dst[p] = src[perm[p0 + p]] for p < n
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

// one migrating particle, all persistent fields (80 bytes)
struct MigRec {
  uint4 xh;
  float4 vm;
  float4 acc;
  float u, av, ac, dprev;
  long long uid;
  int orig, pad;
};

__global__ void k_pack_mig(int n, const unsigned int* __restrict__ perm, Persist src, MigRec* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int i = (int)perm[p];
  MigRec r;
  r.xh = src.xh[i];
  r.vm = src.vm[i];
  r.acc = src.acc[i];
  r.u = src.u[i];
  r.av = src.av[i];
  r.ac = src.ac[i];
  r.dprev = src.dprev[i];
  r.uid = src.uid[i];
  r.orig = src.orig[i];
  r.pad = 0;
  out[p] = r;
}

__global__ void k_set_u32(unsigned int* p, unsigned int v) { *p = v; }

// Zero n bytes (memsets of the context stream as a kernel: a cudaMemsetAsync can queue on the
// copy engines behind a pipelined upload, see copy_chunked)
__global__ void k_zero(uint8_t* p, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t head = (16 - ((uintptr_t)p & 15)) & 15;
  if (head >= n) {
    for (; i < n; i += stride) p[i] = 0;
    return;
  }
  const size_t n16 = (n - head) / 16;
  uint4* p4 = reinterpret_cast<uint4*>(p + head);
  for (size_t k = i; k < n16; k += stride) p4[k] = make_uint4(0u, 0u, 0u, 0u);
  for (size_t k = i; k < head; k += stride) p[k] = 0;
  for (size_t k = head + 16 * n16 + i; k < n; k += stride) p[k] = 0;
}
__global__ void k_copy_u32(const unsigned int* __restrict__ s, unsigned int* d) { *d = *s; }

// The pipelined host I/O's large copies.  Page-locked, device-mapped host memory is copied by a
// kernel (loads or stores over PCIe from a few CTAs on the copy stream): the copy engines, which
// take the copies, memsets and read-backs of every stream in submission order, stay free for the
// context stream's small operations -- with a 738 MB upload queued on them, those waited up to
// ~13 ms each (C4 e2e 35.6 to 140 ms per step from run to run; by kernel 41 ms every run: the
// kernel's PCIe reads reach ~18 GB/s against the copy engines' ~55).  Other host memory goes
// through cudaMemcpyAsync in pieces of at most 4 MB.  The context stream's own memsets are
// kernels too (zero_async).
__global__ void __launch_bounds__(256) k_copy_words(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                    size_t nw) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n16 = ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) ? nw / 4 : 0;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (; i + 3 * stride < n16; i += 4 * stride) {  // four 16-byte loads in flight per thread
    const uint4 a = s4[i], b = s4[i + stride], c = s4[i + 2 * stride], e = s4[i + 3 * stride];
    d4[i] = a;
    d4[i + stride] = b;
    d4[i + 2 * stride] = c;
    d4[i + 3 * stride] = e;
  }
  for (; i < n16; i += stride) d4[i] = s4[i];
  for (size_t w = 4 * n16 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) dst[w] = src[w];
}

cudaError_t copy_chunked(void* dst, const void* src, size_t b, cudaMemcpyKind kind, cudaStream_t st) {
  const void* host = kind == cudaMemcpyHostToDevice ? src : dst;
  cudaPointerAttributes at{};
  // (uploads by copy engine with SPH_H2D_CE: C4 e2e 41.4 / 65.3 ms against 43.2 / 42.4 by kernel on one box)
  static const bool h2d_kernel = getenv("SPH_H2D_CE") == nullptr;
  if ((kind == cudaMemcpyDeviceToHost || h2d_kernel) && b % 4 == 0 && ((uintptr_t)src & 3) == 0 && ((uintptr_t)dst & 3) == 0 &&
      cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer) {
    const ptrdiff_t off = static_cast<const char*>(host) - static_cast<const char*>(at.hostPointer);
    void* mapped = static_cast<char*>(at.devicePointer) + off;
    const uint32_t* s = static_cast<const uint32_t*>(kind == cudaMemcpyHostToDevice ? mapped : src);
    uint32_t* d = static_cast<uint32_t*>(kind == cudaMemcpyHostToDevice ? dst : mapped);
    // (CTAs, C4 e2e ms: 8 69, 16 40-42, 32 39.0-39.2, 64 43, 148 81, 296 48 -- the PCIe reads saturate
    // near 19 GB/s and more CTAs only take SM slots from the loops; SPH_COPY_CTAS overrides)
    static const int ctas = getenv("SPH_COPY_CTAS") ? std::max(1, atoi(getenv("SPH_COPY_CTAS"))) : 32;
    k_copy_words<<<(unsigned)std::min<size_t>(ctas, (b / 4 + 1023) / 1024), 256, 0, st>>>(s, d, b / 4);
    return cudaGetLastError();
  }
  cudaGetLastError();  // (cudaPointerGetAttributes on pageable memory)
  constexpr size_t kPiece = 4u << 20;
  for (size_t o = 0; o < b; o += kPiece) {
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                                          std::min(kPiece, b - o), kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t zero_async(void* p, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const size_t blocks = std::min<size_t>((n / 16 + 255) / 256 + 1, 1184);
  k_zero<<<(unsigned)blocks, 256, 0, st>>>(static_cast<uint8_t*>(p), n);
  return cudaGetLastError();
}

// Halo put (X2): the ghosts' final h, stored into hin by the neighbours' density epilogues,
// into the ghost positions' h (after the token; ghost slots [0, gL) and [gL + n_own, + gR)).
__global__ void k_ghost_h(int gL, int n_own, int gR, const float* __restrict__ hin, uint4* xh) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= gL + gR) return;
  if (p >= gL) p += n_own;
  reinterpret_cast<unsigned int*>(&xh[p])[3] = __float_as_uint(hin[p]);
}

__global__ void k_unpack_mig(int n, const MigRec* __restrict__ in, Persist dst) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  MigRec r = in[p];
  dst.xh[p] = r.xh;
  dst.vm[p] = r.vm;
  dst.acc[p] = r.acc;
  dst.u[p] = r.u;
  dst.av[p] = r.av;
  dst.ac[p] = r.ac;
  dst.dprev[p] = r.dprev;
  dst.uid[p] = r.uid;
  dst.orig[p] = r.orig;
}

// per-cell particle counts of one x plane of the owned cell_start
__global__ void k_plane_counts(int plane_cells, const int* __restrict__ cs, int first_cell, int* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= plane_cells) return;
  out[k] = cs[first_cell + k + 1] - cs[first_cell + k];
}

// final cell_start of the [ghost | owned | ghost] layout: owned planes shifted by gL, ghost
// planes from the exclusive scans of the received per-cell counts
__global__ void k_final_cs(int ncells, int plane_cells, int G, int P, int gL, int n_own, const int* __restrict__ scanL,
                           const int* __restrict__ scanR, int n_loc, int* cs) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > ncells) return;
  if (c == ncells) { cs[c] = n_loc; return; }
  const int plane = c / plane_cells;
  if (plane < G) cs[c] = scanL[c];                                          // left ghost planes
  else if (plane >= G + P) cs[c] = gL + n_own + scanR[c - (G + P) * plane_cells];  // right ghost planes
  else cs[c] = cs[c] + gL;
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
// grid, rounded to nearest, wrapping mod 2^32 (R25); h prediction (R29).
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

// out[(orig ? orig[p] : p) * comps + c] = src[p * stride + off + c]   (32-bit or 64-bit)
__global__ void k_scatter32(int n, const uint32_t* __restrict__ src, int stride, int off, int comps,
                            const int32_t* __restrict__ orig, uint32_t* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int o = orig ? orig[p] : p;
  for (int c = 0; c < comps; ++c) out[(size_t)o * comps + c] = src[(size_t)p * stride + off + c];
}
__global__ void k_scatter64(int n, const uint64_t* __restrict__ src, const int32_t* __restrict__ orig, uint64_t* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  out[orig ? orig[p] : p] = src[p];
}

inline int nblk(long long n, int t) { return (int)((n + t - 1) / t); }

}  // namespace

struct sph_ctx {
  sph_config cfg{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int device = 0;
  // particle layout: [gL ghosts | n_own owned | gR ghosts], capacity cap
  int n_in = 0;               // particles given at creation / set_particles
  int cap = 0;
  int n_own = 0, gL = 0, gR = 0;
  int nranks = 1, rank = 0;
  bool slab = false;          // slab path (a transport was given; always when nranks > 1)
  Comm* comm = nullptr;
  bool ghost_v_stale = false;   // owners' v changed since the ghosts were received
  int planeL = 0, planeR = 0;   // owned particles in the first / last G owned planes (ghost sources)
  int gplanes = 1;              // G: ghost planes on each side of the slab
  bool poisoned = false;
  bool stale = true;          // grid must be rebuilt before the next loop
  bool lists_stale = true;    // neighbour lists must be rebuilt before the next loop
  size_t nbr_cap = 0;         // allocated list entries (cap x lcap)
  int lcap = kLcapInit;
  // wide particles (adaptive cell side, sph_wide.cu)
  float h_side = 0.f;          // h the cell side is sized from (0: the global h_max)
  double adapt_q = 0.0;        // its quantile (0: none)
  uint8_t* wide_flag = nullptr;
  int32_t* widx = nullptr;
  int32_t* wcount = nullptr;
  int* n_wide_dev = nullptr;
  uint32_t* wnbr = nullptr;
  size_t wnbr_cap = 0;         // allocated wide-list entries
  int wlcap = 256;
  void* sel_tmp = nullptr;
  size_t sel_tmp_bytes = 0;
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
  uint8_t* act_flag = nullptr;  // [nblocks] block has i particles
  int* blk_list = nullptr;      // [nact] active block ids
  int* run_list = nullptr;      // [nrun] active indices of the blocks with a non-wide i particle
  size_t run_cap = 0;
  // slab path: the halo exchanges after the density (X2) and gradient (X3) loops run on a
  // communication stream while the next loop's interior blocks (tiles without ghost particles)
  // run on the context stream; its boundary blocks wait for the exchange
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_main = nullptr, ev_x2 = nullptr, ev_x3 = nullptr;
  // halo put (sph_config.halo_put): the neighbours' fr1 / fr2 buffers mapped into this process
  // ([0] left, [1] right), so the gradient epilogue stores X3's ghost records there itself
  // pipelined host I/O (sph_stage_particles / sph_set_particles_staged / sph_get_async)
  static constexpr int kGetSlots = 8;
  cudaStream_t hstream = nullptr, dstream = nullptr;  // host -> device, device -> host copies
  cudaStream_t h2stream = nullptr;                    // (host -> device by copy engine, SPH_H2D_CE_FRAC)
  cudaEvent_t ev_h2 = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_stage_free = nullptr;
  void* stage_buf = nullptr;
  size_t stage_bytes = 0;
  sph_particles_in staged{};
  bool has_staged = false, stage_used = false;
  void* gbuf[kGetSlots] = {};
  size_t gbuf_bytes[kGetSlots] = {};
  bool gused[kGetSlots] = {};
  cudaEvent_t ev_gready[kGetSlots] = {}, ev_gfree[kGetSlots] = {};
  int gnext = 0;
  bool halo_put = false;
  // slab cuts on the 2^-32 grid: rank r owns [cut[r], cut[r+1]) (sph_config.balance moves them)
  std::vector<unsigned long long> cut;
  bool balance = false;
  unsigned int* xhist = nullptr;  // [kHistBins] device histogram of x (balance)
  float4* peer_fr1[2] = {nullptr, nullptr};
  float4* peer_fr2[2] = {nullptr, nullptr};
  float4* peer_gq[2] = {nullptr, nullptr};
  float4* peer_vc[2] = {nullptr, nullptr};
  float2* peer_um[2] = {nullptr, nullptr};
  float* peer_h[2] = {nullptr, nullptr};
  float* hin = nullptr;  // [cap] ghost h stored by the neighbours' density epilogues (X2 put)
  bool x2_pending = false, x3_pending = false;
  uint8_t* side_flag = nullptr;  // [2 nact]: interior, boundary flags
  int* side_list = nullptr;      // [2 nact]: interior active indices at 0, boundary ones at nact
  size_t side_cap = 0, side_flag_cap = 0;
  int n_int = 0, n_bnd = 0;
  int kz_hint = 0;              // KZ chosen at the last rebuild (first probe of the next)
  bool kz_hint_1cta = false;    // ... with one force CTA per SM
  long long n_coinc = 0;        // directed coincident pairs of the owned particles (k_dup)
  unsigned long long* pairs_grad_h = nullptr;  // pinned: the last gradient loop's directed pairs
  float wide_margin = 0.2f;     // adaptive grid: DevGrid::wide_margin (env SPH_WIDE_MARGIN overrides)
  int sparse_wide = 64;         // adaptive grid: blocks with fewer tile particles go wide (env SPH_SPARSE_WIDE; 0 = off)
  double coarse_q = 0.99;       // wide search grid: the h quantile its coarse cells are sized from (env SPH_COARSE_Q)
  // distinct wide search grids (env SPH_COARSE_LEVELS, 1..kCoarseLevels); C5s ms per step with 1 / 2 / 3:
  // 29.5 / 29.0 / 29.2 (the wide list build is bound by its gather latency, not by the candidates)
  int coarse_levels = 2;
  uint32_t* cperm[kCoarseLevels] = {};  // wide search grids: particles in coarse-cell order
  size_t cperm_cap[kCoarseLevels] = {};
  int* ccs[kCoarseLevels] = {};         // their coarse cell starts
  size_t ccs_cap[kCoarseLevels] = {};
  size_t act_cap = 0;
  size_t list_cap = 0;
  char* desc_buf = nullptr;   // tile descriptors, nblocks x tile_desc_bytes()
  size_t desc_cap = 0;
  int* pref_buf = nullptr;    // per-block list-group prefixes (k_lists)
  size_t pref_cap = 0;
  size_t blk_cap = 0;
  DevCounters* ctr = nullptr;     // device
  DevCounters* ctr_h = nullptr;   // pinned host mirror
  unsigned int* scratch = nullptr;  // device scalars
  unsigned int* scratch_h = nullptr;
  void* out_tmp = nullptr;
  size_t out_tmp_bytes = 0;
  // halo exchange buffers
  MigRec *mig_send = nullptr, *mig_recv = nullptr;
  size_t mig_cap = 0;
  int *pc_send = nullptr, *pc_recv = nullptr, *pc_scan = nullptr;  // per-cell plane counts
  size_t pc_cap = 0;
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
  long long* cnt_dev = nullptr;  // 4 message sizes
  long long* cnt_h = nullptr;
  sph_counters counters{};
  long long launches = 0;
  // per-phase device timing (sph_set_timing): event pairs resolved by sph_get_timings
  bool timing = false;
  struct TEv { int kind; cudaEvent_t a, b; };
  std::vector<TEv> tev;
  std::vector<cudaEvent_t> pool;
  double tms[SPH_T_COUNT] = {};
  long long tcnt[SPH_T_COUNT] = {};
};

namespace {

cudaEvent_t ev_get(sph_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Scope of one timed phase on the context stream (no-op unless timing is on).
// (every timed phase is also an NVTX range, named after the phase: visible in nsys / ncu
// --nvtx timelines, free when no tool is attached)
const char* const kPhaseName[SPH_T_COUNT] = {"sph:rebuild", "sph:lists", "sph:density", "sph:gradient",
                                             "sph:force", "sph:kick_drift", "sph:exchange", "sph:other"};
struct Timed {
  sph_ctx* c;
  int kind;
  cudaEvent_t a = nullptr;
  nvtx3::scoped_range range;
  Timed(sph_ctx* ctx, int k) : c(ctx), kind(k), range(kPhaseName[k]) {
    if (c->timing) {
      a = ev_get(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~Timed() {
    if (a) {
      cudaEvent_t b = ev_get(c);
      cudaEventRecord(b, c->stream);
      c->tev.push_back({kind, a, b});
    }
  }
};

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

#define CKC(expr)                                          \
  do {                                                     \
    std::string e_ = (expr);                               \
    if (!e_.empty()) return fail(c, SPH_ERR_NCCL, e_);     \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

sph_status alloc_state(sph_ctx* c) {
  const size_t n = (size_t)c->cap;
  DevState& s = c->s;
  CK(dalloc(&s.xh, n)); CK(dalloc(&s.vm, n)); CK(dalloc(&s.u, n)); CK(dalloc(&s.av, n)); CK(dalloc(&s.ac, n));
  CK(dalloc(&s.dprev, n)); CK(dalloc(&s.uid, n)); CK(dalloc(&s.orig, n)); CK(dalloc(&s.acc, n));
  Persist& a = c->alt;
  CK(dalloc(&a.xh, n)); CK(dalloc(&a.vm, n)); CK(dalloc(&a.u, n)); CK(dalloc(&a.av, n)); CK(dalloc(&a.ac, n));
  CK(dalloc(&a.dprev, n)); CK(dalloc(&a.uid, n)); CK(dalloc(&a.orig, n)); CK(dalloc(&a.acc, n));
  CK(dalloc(&s.dens, n)); CK(dalloc(&s.dvc, n)); CK(dalloc(&s.count, n)); CK(dalloc(&s.fin, n));
  CK(dalloc(&s.gq, n)); CK(dalloc(&s.hlo, n)); CK(dalloc(&s.hhi, n)); CK(dalloc(&s.iters, n));
  CK(dalloc(&s.vc, n)); CK(dalloc(&s.um, n));
  CK(dalloc(&s.active, n)); CK(dalloc(&s.grad, n)); CK(dalloc(&s.fr1, n)); CK(dalloc(&s.fr2, n));
  CK(dalloc(&s.vsig, n)); CK(dalloc(&s.countf, n)); CK(dalloc(&s.dup, n));
  CK(cudaMemset(s.dup, 0, n));
  CK(dalloc(&s.ncount, n)); CK(dalloc(&s.hbuild, n));
  CK(cudaMemset(s.ncount, 0, n * sizeof(int32_t)));  // k_lists reads it as a length hint
  CK(dalloc(&s.nbr, n * (size_t)c->lcap));
  CK(dalloc(&s.nbr_raw, n * (size_t)c->lcap));
  c->nbr_cap = n * (size_t)c->lcap;
  CK(dalloc(&c->keys, n)); CK(dalloc(&c->keys_alt, n)); CK(dalloc(&c->perm, n)); CK(dalloc(&c->perm_alt, n));
  CK(dalloc(&c->ctr, 1));
  CK(cudaMallocHost((void**)&c->ctr_h, sizeof(DevCounters)));
  CK(cudaMallocHost((void**)&c->pairs_grad_h, sizeof(unsigned long long)));
  *c->pairs_grad_h = 0;
  CK(dalloc(&c->scratch, 16));
  CK(cudaMallocHost((void**)&c->scratch_h, 16 * sizeof(unsigned int)));
  CK(dalloc(&c->cnt_dev, 8));
  CK(cudaMallocHost((void**)&c->cnt_h, 8 * sizeof(long long)));
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

void swap_persist(sph_ctx* c) {
  Persist old = persist_of(c->s);
  set_persist(c->s, c->alt);
  c->alt = old;
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
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks)
    return fail(c, SPH_ERR_INVALID_ARG, "rank/nranks out of range");
  if (cfg->nranks > 1 || cfg->nccl_uid || (cfg->transport == SPH_TRANSPORT_LOOPBACK && cfg->loopback)) {
    if (cfg->transport == SPH_TRANSPORT_NCCL && !cfg->nccl_uid)
      return fail(c, SPH_ERR_INVALID_ARG, "NCCL transport needs nccl_uid (sph_nccl_unique_id on rank 0, broadcast)");
    if (cfg->transport == SPH_TRANSPORT_LOOPBACK && !cfg->loopback)
      return fail(c, SPH_ERR_INVALID_ARG, "loopback transport needs a group (sph_loopback_create)");
    if (cfg->n_total <= 0) return fail(c, SPH_ERR_INVALID_ARG, "multi-rank contexts need n_total");
  }
  const bool slabs = (cfg->decomp[0] == 0 && cfg->decomp[1] == 0 && cfg->decomp[2] == 0) ||
                     (cfg->decomp[0] == cfg->nranks && cfg->decomp[1] == 1 && cfg->decomp[2] == 1);
  if (!slabs)
    return fail(c, SPH_ERR_INVALID_ARG, "decomp: only x-slabs {nranks, 1, 1} are implemented (DESIGN.md §9)");
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
  if (!in || !in->X || !in->v || !in->m || !in->u || !in->h)
    return fail(c, SPH_ERR_INVALID_ARG, "required particle array is NULL");
  if (in->n < 0 || (c->nranks == 1 && in->n != c->n_in) || in->n > c->cap)
    return fail(c, SPH_ERR_INVALID_ARG, "particle count mismatch / above capacity");
  const size_t n = (size_t)in->n;
  const uint32_t* X = in->X;
  const float *v = in->v, *m = in->m, *u = in->u, *h = in->h, *av = in->alpha_v, *ac = in->alpha_c,
              *dp = in->div_prev;
  const int64_t* id = in->id;
  if (!in->on_device && n > 0) {
    // stage host arrays through the (reused) output buffer region on the device
    size_t bytes = n * (12 + 12 + 4 * 3) + (av ? 4 * n : 0) + (ac ? 4 * n : 0) + (dp ? 4 * n : 0) + (id ? 8 * n : 0) +
                   9 * 16;
    if (c->out_tmp_bytes < bytes) {
      if (c->out_tmp) cudaFree(c->out_tmp);
      c->out_tmp = nullptr;
      c->out_tmp_bytes = 0;
      CK(cudaMalloc(&c->out_tmp, bytes));
      c->out_tmp_bytes = bytes;
    }
    char* d = (char*)c->out_tmp;
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
  if (n > 0) {
    k_ingest<<<nblk(n, 256), 256, 0, c->stream>>>((int)n, X, v, m, u, h, av, ac, dp, id, persist_of(c->s));
    c->launches++;
    CK(cudaGetLastError());
  }
  c->n_own = (int)n;
  c->gL = c->gR = 0;
  c->dprev_valid = dp != nullptr;
  c->dvc_valid = false;
  c->stale = true;
  c->density_done = c->gradient_done = false;
  return SPH_OK;
}

sph_status sync_ctr(sph_ctx* c) {
  CK(copy_chunked(c->ctr_h, c->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  return SPH_OK;
}

sph_status reset_ctr(sph_ctx* c) {
  CK(zero_async(c->ctr, sizeof(DevCounters), c->stream));
  c->launches++;
  return SPH_OK;
}

float ulp_of(float x) {
  int e;
  std::frexp(x, &e);  // x = f 2^e, f in [0.5, 1)
  return std::ldexp(1.0f, e - 24);
}

int left_of(const sph_ctx* c) { return (c->rank + c->nranks - 1) % c->nranks; }
int right_of(const sph_ctx* c) { return (c->rank + 1) % c->nranks; }

// Exchange two int64 sizes with the slab neighbours: sends (to_right, to_left), returns
// (from_left, from_right).
sph_status exchange_sizes(sph_ctx* c, long long to_right, long long to_left, long long& from_left,
                          long long& from_right) {
  c->cnt_h[0] = to_right;
  c->cnt_h[1] = to_left;
  CK(cudaMemcpyAsync(c->cnt_dev, c->cnt_h, 2 * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
  Xfer s[2] = {{right_of(c), c->cnt_dev, 8}, {left_of(c), c->cnt_dev + 1, 8}};
  Xfer r[2] = {{left_of(c), c->cnt_dev + 2, 8}, {right_of(c), c->cnt_dev + 3, 8}};
  CKC(c->comm->exchange(s, 2, r, 2, c->stream));
  CK(copy_chunked(c->cnt_h + 2, c->cnt_dev + 2, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  from_left = c->cnt_h[2];
  from_right = c->cnt_h[3];
  return SPH_OK;
}

template <class T>
sph_status grow(sph_ctx* c, T** p, size_t& cap, size_t need) {
  if (need <= cap) return SPH_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  cap = 0;
  CK(dalloc(p, need));
  cap = need;
  return SPH_OK;
}

// grow() with 25 % headroom, for buffers sized by counts that drift from rebuild to rebuild
// (active blocks): a realloc (and the device sync of cudaFree) only every so often
template <class T>
sph_status grow_h(sph_ctx* c, T** p, size_t& cap, size_t need) {
  return need <= cap ? SPH_OK : grow(c, p, cap, need + need / 4);
}

// Ghost halo exchange of one per-particle array (elem bytes each): the first owned plane goes
// to the left neighbour (its right ghosts), the last owned plane to the right neighbour (its
// left ghosts).  Ghost sets are fixed between rebuilds, so no sizes are exchanged.
sph_status halo(sph_ctx* c, void* base, size_t elem) {
  if (!c->slab) return SPH_OK;
  Timed tm(c, SPH_T_EXCHANGE);
  char* b = static_cast<char*>(base);
  Xfer s[2] = {{right_of(c), b + (size_t)(c->gL + c->n_own - c->planeR) * elem, (size_t)c->planeR * elem},
               {left_of(c), b + (size_t)c->gL * elem, (size_t)c->planeL * elem}};
  Xfer r[2] = {{left_of(c), b, (size_t)c->gL * elem},
               {right_of(c), b + (size_t)(c->gL + c->n_own) * elem, (size_t)c->gR * elem}};
  CKC(c->comm->exchange(s, 2, r, 2, c->stream));
  return SPH_OK;
}

// The same exchange enqueued on stream st (untimed: it overlaps the interior blocks' loop).
sph_status halo_on(sph_ctx* c, void* base, size_t elem, cudaStream_t st) {
  char* b = static_cast<char*>(base);
  Xfer s[2] = {{right_of(c), b + (size_t)(c->gL + c->n_own - c->planeR) * elem, (size_t)c->planeR * elem},
               {left_of(c), b + (size_t)c->gL * elem, (size_t)c->planeL * elem}};
  Xfer r[2] = {{left_of(c), b, (size_t)c->gL * elem},
               {right_of(c), b + (size_t)(c->gL + c->n_own) * elem, (size_t)c->gR * elem}};
  CKC(c->comm->exchange(s, 2, r, 2, st));
  return SPH_OK;
}

// Start an asynchronous halo exchange of `n` arrays on the communication stream after the work
// enqueued so far on the context stream; `ev` marks its completion.
sph_status halo_async(sph_ctx* c, void* const* bases, const size_t* elems, int n, cudaEvent_t ev) {
  CK(cudaEventRecord(c->ev_main, c->stream));
  CK(cudaStreamWaitEvent(c->cstream, c->ev_main, 0));
  for (int k = 0; k < n; ++k) {
    const sph_status st = halo_on(c, bases[k], elems[k], c->cstream);
    if (st != SPH_OK) return st;
  }
  CK(cudaEventRecord(ev, c->cstream));
  return SPH_OK;
}

// Halo put: a zero-payload exchange (8 bytes each way with both neighbours) on the
// communication stream after the work enqueued so far on the context stream.  Stream order
// makes it leave after the kernels whose epilogues stored into the neighbours' buffers, and
// arrive after theirs: the ordering NCCL send/recv of the data would have given.
sph_status halo_token(sph_ctx* c) {
  CK(cudaEventRecord(c->ev_main, c->stream));
  CK(cudaStreamWaitEvent(c->cstream, c->ev_main, 0));
  Xfer ts[2] = {{right_of(c), c->cnt_dev + 4, 8}, {left_of(c), c->cnt_dev + 5, 8}};
  Xfer tr[2] = {{left_of(c), c->cnt_dev + 6, 8}, {right_of(c), c->cnt_dev + 7, 8}};
  CKC(c->comm->exchange(ts, 2, tr, 2, c->cstream));
  return SPH_OK;
}

// The context stream waits for every pending asynchronous exchange.
sph_status join_comm(sph_ctx* c) {
  if (c->x2_pending) CK(cudaStreamWaitEvent(c->stream, c->ev_x2, 0));
  if (c->x3_pending) CK(cudaStreamWaitEvent(c->stream, c->ev_x3, 0));
  c->x2_pending = c->x3_pending = false;
  return SPH_OK;
}

// global reduction of host scalars (no-op on one rank)
sph_status allreduce(sph_ctx* c, double* v, int n, ReduceOp op) {
  if (!c->slab) return SPH_OK;
  CKC(c->comm->allreduce(v, n, op, c->stream));
  return SPH_OK;
}

// global reduction of uint32 values in device memory, enqueued on the context stream (no host
// synchronisation over NCCL; no-op on one rank).  The next read-back sees the global values.
sph_status allreduce_dev(sph_ctx* c, void* d, int n, ReduceOp op) {
  if (!c->slab) return SPH_OK;
  CKC(c->comm->allreduce_dev_u32(static_cast<uint32_t*>(d), n, op, c->stream));
  return SPH_OK;
}

// Collective error agreement: every rank takes the same branch (a rank that fails alone
// would leave its neighbours waiting in the next exchange).
sph_status agree(sph_ctx* c, bool bad, sph_status code, const char* msg) {
  if (c->slab) {
    double v = bad ? 1.0 : 0.0;
    sph_status st = allreduce(c, &v, 1, kMax);
    if (st != SPH_OK) return st;
    if (v > 0 && !bad) return fail(c, code, std::string("another rank failed: ") + msg);
  }
  return bad ? fail(c, code, msg) : SPH_OK;
}

// keys + radix sort of n particles starting at `base` (persistent arrays) into cell order;
// fills c->perm_alt (sorted -> input index) and the owned-relative cell_start
sph_status sort_cells(sph_ctx* c, int base, int n, int* outside) {
  DevGrid& g = c->grid;
  CK(zero_async(c->scratch + 2, 4, c->stream));
  c->launches++;
  if (n > 0) {
    k_keys<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->s.xh + base, g, c->keys, c->perm, (int*)(c->scratch + 2));
    c->launches++;
    CK(cudaGetLastError());
    int bits = 1;
    while ((1LL << bits) <= g.ncells) ++bits;
    bits += g.zbits;
    size_t tmp = c->sort_tmp_bytes;
    CK(cub::DeviceRadixSort::SortPairs(c->sort_tmp, tmp, c->keys, c->keys_alt, c->perm, c->perm_alt, n, 0, bits,
                                       c->stream));
    c->launches += 1 + (bits + 7) / 8;
  }
  k_cell_start<<<nblk(n + 1, 256), 256, 0, c->stream>>>(n, g.ncells, g.zbits, c->keys_alt, c->cell_start);
  c->launches++;
  CK(cudaGetLastError());
  CK(copy_chunked(c->scratch_h + 2, c->scratch + 2, 4, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  *outside = (int)c->scratch_h[2];
  return SPH_OK;
}

sph_status read_cs(sph_ctx* c, int cell, int* v) {
  k_copy_u32<<<1, 1, 0, c->stream>>>(reinterpret_cast<const unsigned int*>(c->cell_start + cell),
                                     reinterpret_cast<unsigned int*>(c->scratch + 4));
  c->launches++;
  CK(cudaGetLastError());
  CK(copy_chunked(c->scratch_h + 4, c->scratch + 4, 4, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  *v = (int)c->scratch_h[4];
  return SPH_OK;
}

// Choose the grid for the current h, migrate (several ranks), sort, exchange ghost planes, and
// size the CTA tiles.
sph_status rebuild_impl(sph_ctx* c);
sph_status mark_wide(sph_ctx* c);
sph_status h_quantile(sph_ctx* c, double q, float* out, bool global = true);

// Cell grid for the current h.  adaptive_h: when cells sized from h_max do not fit the tiles
// (strong h contrast), size them from decreasing quantiles of h instead (on the slab path the
// largest of the ranks' quantiles, so every rank takes the same grid); the particles whose
// support exceeds a cell then become wide (sph_wide.cu).
sph_status rebuild(sph_ctx* c) {
  Timed tm(c, SPH_T_REBUILD);
  const bool adaptive = c->cfg.adaptive_h;
  sph_status st;
  if (adaptive && c->adapt_q > 0.0) {  // the quantile that worked last time, first
    float hq;
    const auto t0 = std::chrono::steady_clock::now();
    if ((st = h_quantile(c, c->adapt_q, &hq)) != SPH_OK) return st;
    const auto t1 = std::chrono::steady_clock::now();
    c->h_side = hq;
    st = rebuild_impl(c);
    const auto t2 = std::chrono::steady_clock::now();
    if (st == SPH_OK) {
      st = mark_wide(c);
      if (getenv("SPH_DEBUG")) {
        cudaStreamSynchronize(c->stream);
        const auto t3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        fprintf(stderr, "[sph] rebuild ms: quantile %.3f grid %.3f wide %.3f (n_wide %d)\n", ms(t0, t1), ms(t1, t2),
                ms(t2, t3), c->s.n_wide);
      }
      return st;
    }
    if (st != SPH_ERR_H_EXCEEDS_CELL) return st;
  }
  c->h_side = 0.f;
  c->adapt_q = 0.0;
  st = rebuild_impl(c);
  if (st == SPH_ERR_H_EXCEEDS_CELL && adaptive) {
    const std::string first = c->err;
    float tried = std::numeric_limits<float>::infinity();
    for (double q : {0.99, 0.95, 0.9, 0.8, 0.65, 0.5, 0.35, 0.2}) {
      float hq;
      const sph_status sq = h_quantile(c, q, &hq);
      if (sq != SPH_OK) return sq;
      if (!(hq < tried)) continue;
      tried = hq;
      c->h_side = hq;
      st = rebuild_impl(c);
      if (getenv("SPH_DEBUG"))
        fprintf(stderr, "[sph] adaptive grid: h quantile %.2f = %.6g -> status %d (%s)\n", q, hq, (int)st,
                st == SPH_OK ? "ok" : c->err.c_str());
      if (st != SPH_ERR_H_EXCEEDS_CELL) {
        c->adapt_q = q;
        break;
      }
    }
    if (st == SPH_ERR_H_EXCEEDS_CELL) {
      c->h_side = 0.f;
      c->adapt_q = 0.0;
      return fail(c, st, first);
    }
  }
  if (st != SPH_OK) return st;
  return mark_wide(c);
}

// Balanced slab cuts (sph_config.balance): a global histogram of the owned particles' x
// (kHistBins bins, device-side SUM allreduce, one read-back), and every cut r moved toward the x
// where the cumulative count reaches r N / R (linear inside its bin) -- by at most a quarter of
// the thinner adjacent slab's cell plane, so that migrants stay within one ghost plane, and
// keeping every slab at least half the uniform width.  Every rank computes the same cuts from
// the same histogram.
constexpr int kHistBins = 4096;
sph_status rebalance_cuts(sph_ctx* c, int base, int n) {
  const int R = c->nranks;
  if (!c->xhist) CK(cudaMalloc(&c->xhist, kHistBins * sizeof(unsigned int)));
  CK(zero_async(c->xhist, kHistBins * sizeof(unsigned int), c->stream));
  c->launches++;
  if (n > 0) {
    k_xhist<<<std::min(nblk(n, 256), 1184), 256, 0, c->stream>>>(n, c->s.xh + base, kHistBins, c->xhist);
    c->launches++;
  }
  CK(cudaGetLastError());
  sph_status st = allreduce_dev(c, c->xhist, kHistBins, kSum);
  if (st != SPH_OK) return st;
  std::vector<unsigned int> h(kHistBins);
  CK(copy_chunked(h.data(), c->xhist, kHistBins * sizeof(unsigned int), cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  for (unsigned int v : h) tot += v;
  if (!(tot > 0.0)) return SPH_OK;
  const double two32 = std::ldexp(1.0, 32), bw = two32 / kHistBins;
  const long long wmin = (long long)((two32 / R) / 2);
  std::vector<unsigned long long> cut = c->cut;
  double cum = 0.0;
  int b = 0;
  for (int r = 1; r < R; ++r) {
    const double target = tot * r / R;
    while (b < kHistBins - 1 && cum + h[b] < target) cum += h[b++];
    const double frac = h[b] > 0 ? (target - cum) / h[b] : 0.5;
    const double want = (b + std::min(1.0, std::max(0.0, frac))) * bw;
    const double wl = (double)(c->cut[r] - c->cut[r - 1]), wr = (double)(c->cut[r + 1] - c->cut[r]);
    const double step = 0.25 * std::min(wl, wr) / std::max(c->grid.nxo, 1);
    const double d = std::min(step, std::max(-step, want - (double)c->cut[r]));
    long long nc = (long long)c->cut[r] + (long long)d;
    nc = std::max(nc, (long long)cut[r - 1] + wmin);  // (the left neighbour's cut already moved)
    nc = std::min(nc, (long long)c->cut[r + 1] - wmin);
    cut[r] = (unsigned long long)std::max(nc, (long long)cut[r - 1] + 1);
  }
  c->cut = cut;
  return SPH_OK;
}

sph_status rebuild_impl(sph_ctx* c) {
  // SPH_DEBUG: elapsed ms at the stages of the rebuild (synchronising)
  const bool dbg = getenv("SPH_DEBUG") != nullptr;
  const auto tr0 = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[sph]   rebuild %s at %.3f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count());
  };
  sph_status st;
  // the owned particles sit at [base, base + n); the old ghosts are dropped (re-received below)
  const int base = c->gL;
  int n = c->n_own;
  // global h_max -> cell side (identical on every rank)
  CK(zero_async(c->scratch, 4, c->stream));
  c->launches++;
  if (n > 0) {
    k_hmax<<<std::min(nblk(n, 256), 1184), 256, 0, c->stream>>>(n, c->s.xh + base, c->scratch);
    c->launches++;
  }
  CK(cudaGetLastError());
  // global h_max (positive f32 bits order as uint32): device-side reduction, one read-back
  if ((st = allreduce_dev(c, c->scratch, 1, kMax)) != SPH_OK) return st;
  CK(copy_chunked(c->scratch_h, c->scratch, 4, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  float hmax;
  std::memcpy(&hmax, c->scratch_h, 4);
  if (!(hmax > 0.f) || !std::isfinite(hmax)) return fail(c, SPH_ERR_INVALID_ARG, "smoothing lengths must be finite and > 0");
  const float hcell = c->h_side > 0.f ? std::min(c->h_side, hmax) : hmax;  // adaptive: an h quantile
  const double Hs = (double)c->cfg.gamma_k * hcell * (1.0 + c->cfg.cell_skin);
  DevGrid& g = c->grid;
  const int R = c->nranks;
  int G = c->gplanes;  // ghost planes per side (slab path; more with wide particles, below)
  const bool slab = c->slab;
  // slab of this rank on the 2^-32 grid (fixed by position, independent of h)
  const double two32 = std::ldexp(1.0, 32);
  if (slab && R > 1 && c->balance && c->grid.nxo > 0) {
    if ((st = rebalance_cuts(c, base, n)) != SPH_OK) return st;
  }
  auto slab_lo = [&](int r) { return c->cut[r]; };
  unsigned long long wmin = ~0ull;
  for (int r = 0; r < R; ++r) wmin = std::min(wmin, slab_lo(r + 1) - slab_lo(r));
  g.x_lo = (unsigned int)slab_lo(c->rank);
  g.wfix = slab_lo(c->rank + 1) - slab_lo(c->rank);
  int nc[3];
  for (int a = 0; a < 3; ++a) {
    // planes along x per slab (same on every rank), cells along y, z
    const double len = a == 0 ? c->cfg.box[0] * ((double)wmin / two32) : c->cfg.box[a];
    double k = std::floor(len / Hs);
    // (x planes of a slab: checked against the ghost planes below)
    const double kmin = (a == 0 && slab) ? 1 : 3;
    if (k < kmin) {
      char b[256];
      snprintf(b, sizeof b, "support radius %.6g leaves fewer than %g cells along axis %d (length %.6g over %d ranks)",
               Hs, kmin, a, c->cfg.box[a], a == 0 ? R : 1);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
    nc[a] = (int)std::min(k, 1024.0);
  }
  auto ncells_of = [&]() { return (long long)(nc[0] + (slab ? 2 * kMaxGhostPlanes : 0)) * nc[1] * nc[2]; };
  while (ncells_of() > (1LL << 30)) { for (int a = 0; a < 3; ++a) nc[a] = std::max(3, nc[a] / 2); }
  g.nxo = nc[0];
  g.ny = nc[1];
  g.nz = nc[2];
  for (int a = 0; a < 3; ++a) {
    g.side[a] = (float)(c->cfg.box[a] / nc[a]);
    g.scale[a] = (float)(c->cfg.box[a] * std::ldexp(1.0, -32));
    g.dscale[a] = c->cfg.box[a] * std::ldexp(1.0, -32);
  }
  float side_x_min = g.side[0];
  if (slab) {
    g.side[0] = (float)(c->cfg.box[0] * ((double)g.wfix / two32) / nc[0]);          // this slab's planes
    side_x_min = (float)(c->cfg.box[0] * ((double)wmin / two32) / nc[0]);           // thinnest planes of any slab
  }
  g.side_min = std::min(side_x_min, std::min(g.side[1], g.side[2]));
  if (slab && c->h_side > 0.f) {
    // wide particles on the slab path: G ghost planes per side such that every particle whose
    // list radius (+25 % for its growth in the h iteration; k_wide_density asks for a rebuild
    // past it) crosses a slab face lies within G planes of it, and its own search stays inside
    // the local planes (ghost_planes_needed; the largest over the ranks)
    CK(zero_async(c->scratch + 5, 4, c->stream));
    c->launches++;
    if (n > 0) {
      k_ghost_need<<<std::min(nblk(n, 256), 1184), 256, 0, c->stream>>>(
          n, c->s.xh + base, g, (1.f + c->cfg.cell_skin) * c->cfg.gamma_k * 1.25f, c->scratch + 5);
      c->launches++;
    }
    CK(cudaGetLastError());
    if ((st = allreduce_dev(c, c->scratch + 5, 1, kMax)) != SPH_OK) return st;
    CK(copy_chunked(c->scratch_h + 5, c->scratch + 5, 4, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
    G = std::max(G, (int)c->scratch_h[5]);
    if (G > kMaxGhostPlanes) {
      char b[256];
      snprintf(b, sizeof b, "wide particles reach %d cell planes past their slab (at most %d ghost planes)", G,
               kMaxGhostPlanes);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
  }
  if (slab) {
    // the G ghost planes on each side are distinct from each other and, for R = 1, from the
    // owned planes they image: nxo >= 2G + 1 (R = 1), 2G (R = 2), G (R >= 3)
    const int kmin = R == 1 ? 2 * G + 1 : R == 2 ? 2 * G : G;
    if (g.nxo < kmin) {
      char b[256];
      snprintf(b, sizeof b, "support radius %.6g leaves fewer than %d cells along axis 0 (length %.6g over %d ranks, "
               "%d ghost planes)", Hs, kmin, c->cfg.box[0], R, G);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
    g.nx = g.nxo + 2 * G;
    g.periodic_x = 0;
    g.ix_first = G;
  } else {
    g.nx = g.nxo;
    g.periodic_x = 1;
    g.ix_first = 0;
  }
  g.ncells = g.nx * g.ny * g.nz;
  {
    int cbits = 1;
    while ((1LL << cbits) <= g.ncells) ++cbits;
    g.zbits = std::max(0, std::min(12, 32 - cbits));
  }
  g.zbucket = (float)(c->cfg.box[2] / nc[2] * std::ldexp(1.0, -g.zbits));
  if ((st = grow(c, &c->cell_start, c->cell_cap, (size_t)g.ncells + 1)) != SPH_OK) return st;
  const int pcells = g.ny * g.nz;
  int outside = 0;
  if ((st = sort_cells(c, base, n, &outside)) != SPH_OK) return st;
  const Persist cur = offset(persist_of(c->s), base);
  if (slab) {
    // ---- migration (X6): particles now in a ghost plane belong to the neighbour
    if ((st = agree(c, outside > 0, SPH_ERR_INVALID_ARG, "a particle moved more than G cell planes out of its slab")) !=
        SPH_OK)
      return st;
    const int P = g.nxo;
    int c1, cP1;
    if ((st = read_cs(c, G * pcells, &c1)) != SPH_OK) return st;          // first owned plane
    if ((st = read_cs(c, (G + P) * pcells, &cP1)) != SPH_OK) return st;  // first right ghost plane
    const long long nL = c1, nR = n - cP1, nmid = cP1 - c1;
    long long mL = 0, mR = 0;
    if ((st = exchange_sizes(c, nR, nL, mL, mR)) != SPH_OK) return st;
    const long long nnew = nmid + mL + mR;
    if ((st = agree(c, nnew > c->cap, SPH_ERR_OOM, "slab holds more particles than the context capacity")) != SPH_OK)
      return st;
    const size_t mig_old = c->mig_cap;
    if ((st = grow(c, &c->mig_send, c->mig_cap, (size_t)std::max(nL + nR, mL + mR) * 2 + 16)) != SPH_OK) return st;
    if (!c->mig_recv || c->mig_cap != mig_old) {  // (same capacity as mig_send)
      if (c->mig_recv) cudaFree(c->mig_recv);
      c->mig_recv = nullptr;
      CK(dalloc(&c->mig_recv, c->mig_cap));
    }
    MigRec* sR = c->mig_send;
    MigRec* sL = c->mig_send + nR;
    if (nR > 0) k_pack_mig<<<nblk(nR, 256), 256, 0, c->stream>>>((int)nR, c->perm_alt + cP1, cur, sR);
    if (nL > 0) k_pack_mig<<<nblk(nL, 256), 256, 0, c->stream>>>((int)nL, c->perm_alt, cur, sL);
    c->launches += 2;
    CK(cudaGetLastError());
    Xfer s[2] = {{right_of(c), sR, (size_t)nR * sizeof(MigRec)}, {left_of(c), sL, (size_t)nL * sizeof(MigRec)}};
    Xfer r[2] = {{left_of(c), c->mig_recv, (size_t)mL * sizeof(MigRec)},
                 {right_of(c), c->mig_recv + mL, (size_t)mR * sizeof(MigRec)}};
    CKC(c->comm->exchange(s, 2, r, 2, c->stream));
    if (nmid > 0) {
      k_permute<<<nblk(nmid, 256), 256, 0, c->stream>>>((int)nmid, c->perm_alt + c1, cur, c->alt);
      c->launches++;
    }
    if (mL + mR > 0) {
      k_unpack_mig<<<nblk(mL + mR, 256), 256, 0, c->stream>>>((int)(mL + mR), c->mig_recv, offset(c->alt, (int)nmid));
      c->launches++;
    }
    CK(cudaGetLastError());
    swap_persist(c);
    n = (int)nnew;
    c->n_own = n;
    c->gL = c->gR = 0;
    if ((st = sort_cells(c, 0, n, &outside)) != SPH_OK) return st;
    if ((st = agree(c, outside > 0, SPH_ERR_INVALID_ARG, "migrated particle outside its slab")) != SPH_OK) return st;
    // ---- ghost planes (X1): sizes and per-cell counts first
    // (the owned planes are [G, G + P); the ghost sources are the first and the last G of them)
    const int gpc = G * pcells;
    int cP;
    if ((st = read_cs(c, P * pcells, &cP)) != SPH_OK) return st;  // start of the last G owned planes
    int c2;
    if ((st = read_cs(c, 2 * gpc, &c2)) != SPH_OK) return st;  // end of the first G owned planes
    c->planeL = c2;        // first G owned planes: [0, c2) of the sorted owned set
    c->planeR = n - cP;    // last G owned planes: [cP, n)
    long long gL = 0, gR = 0;
    if ((st = exchange_sizes(c, c->planeR, c->planeL, gL, gR)) != SPH_OK) return st;
    if ((st = agree(c, gL + n + gR > c->cap, SPH_ERR_OOM, "owned + ghost particles exceed the context capacity")) !=
        SPH_OK)
      return st;
    c->gL = (int)gL;
    c->gR = (int)gR;
    if (c->halo_put) {
      // halo put targets: the first G owned planes go to the left neighbour's right ghosts (at
      // its gL + n_own, which it sends us), the last G to the right neighbour's left ghosts (at 0)
      long long dstL = 0, unused = 0;
      if ((st = exchange_sizes(c, (long long)c->gL + n, 0, dstL, unused)) != SPH_OK) return st;
      DevState& ds = c->s;
      ds.put_fr1[0] = c->peer_fr1[0] + dstL;
      ds.put_fr2[0] = c->peer_fr2[0] + dstL;
      ds.put_lo[0] = c->gL;
      ds.put_hi[0] = c->gL + c->planeL;
      ds.put_gq[0] = c->peer_gq[0] + dstL;
      ds.put_vc[0] = c->peer_vc[0] + dstL;
      ds.put_um[0] = c->peer_um[0] + dstL;
      ds.put_h[0] = c->peer_h[0] + dstL;
      ds.put_fr1[1] = c->peer_fr1[1];
      ds.put_fr2[1] = c->peer_fr2[1];
      ds.put_gq[1] = c->peer_gq[1];
      ds.put_vc[1] = c->peer_vc[1];
      ds.put_um[1] = c->peer_um[1];
      ds.put_h[1] = c->peer_h[1];
      ds.put_lo[1] = c->gL + n - c->planeR;
      ds.put_hi[1] = c->gL + n;
    }
    g.gL = c->gL;
    g.n_own = n;
    g.x_loL = (unsigned int)slab_lo((c->rank + R - 1) % R);
    g.wfixL = slab_lo((c->rank + R - 1) % R + 1) - slab_lo((c->rank + R - 1) % R);
    g.x_loR = (unsigned int)slab_lo((c->rank + 1) % R);
    g.wfixR = slab_lo((c->rank + 1) % R + 1) - slab_lo((c->rank + 1) % R);
    const size_t pc_old = c->pc_cap;
    if ((st = grow(c, &c->pc_send, c->pc_cap, (size_t)4 * gpc + 64)) != SPH_OK) return st;
    if (!c->pc_recv || c->pc_cap != pc_old) {  // (same capacity as pc_send)
      if (c->pc_recv) cudaFree(c->pc_recv);
      if (c->pc_scan) cudaFree(c->pc_scan);
      c->pc_recv = c->pc_scan = nullptr;
      CK(dalloc(&c->pc_recv, c->pc_cap));
      CK(dalloc(&c->pc_scan, c->pc_cap));
    }
    k_plane_counts<<<nblk(gpc, 256), 256, 0, c->stream>>>(gpc, c->cell_start, P * pcells, c->pc_send);
    k_plane_counts<<<nblk(gpc, 256), 256, 0, c->stream>>>(gpc, c->cell_start, gpc, c->pc_send + gpc);
    c->launches += 2;
    CK(cudaGetLastError());
    {
      Xfer s2[2] = {{right_of(c), c->pc_send, (size_t)gpc * 4}, {left_of(c), c->pc_send + gpc, (size_t)gpc * 4}};
      Xfer r2[2] = {{left_of(c), c->pc_recv, (size_t)gpc * 4}, {right_of(c), c->pc_recv + gpc, (size_t)gpc * 4}};
      CKC(c->comm->exchange(s2, 2, r2, 2, c->stream));
    }
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, c->pc_recv, c->pc_scan, gpc, c->stream);
    if (need > c->scan_tmp_bytes) {
      if (c->scan_tmp) cudaFree(c->scan_tmp);
      c->scan_tmp = nullptr;
      CK(cudaMalloc(&c->scan_tmp, need));
      c->scan_tmp_bytes = need;
    }
    CK(cub::DeviceScan::ExclusiveSum(c->scan_tmp, need, c->pc_recv, c->pc_scan, gpc, c->stream));
    CK(cub::DeviceScan::ExclusiveSum(c->scan_tmp, need, c->pc_recv + gpc, c->pc_scan + gpc, gpc, c->stream));
    c->launches += 2;
    // owned particles into their final place, then the ghost payload straight into the ghost slots
    if (n > 0) {
      k_permute<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->perm_alt, persist_of(c->s), offset(c->alt, c->gL));
      c->launches++;
    }
    k_final_cs<<<nblk(g.ncells + 1, 256), 256, 0, c->stream>>>(g.ncells, pcells, G, P, c->gL, n, c->pc_scan,
                                                               c->pc_scan + gpc, c->gL + n + c->gR, c->cell_start);
    c->launches++;
    CK(cudaGetLastError());
    swap_persist(c);
    if ((st = halo(c, c->s.xh, sizeof(uint4))) != SPH_OK) return st;
    if ((st = halo(c, c->s.vm, sizeof(float4))) != SPH_OK) return st;
    c->ghost_v_stale = false;
  } else {
    if (outside) return fail(c, SPH_ERR_INVALID_ARG, "internal: particle outside the periodic grid");
    g.gL = 0;
    g.n_own = n;
    if (n > 0) {
      k_permute<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->perm_alt, cur, c->alt);
      c->launches++;
    }
    CK(cudaGetLastError());
    swap_persist(c);
  }
  stage("binned");
  // coincident particles: flags for k_lists and the directed pair count (read with the
  // tile sizes below)
  CK(zero_async(c->scratch + 14, 4, c->stream));
  c->launches++;
  if (n > 0) {
    CK(zero_async(c->s.dup + c->gL, (size_t)n, c->stream));
    c->launches++;
    k_dup<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->keys_alt, c->s.xh + c->gL, c->s.dup + c->gL, c->scratch + 14);
    c->launches++;
  }
  CK(cudaGetLastError());
  CK(copy_chunked(c->scratch_h + 14, c->scratch + 14, 4, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  // CTA blocks: BX x BY grid columns x KZ cells (BX, BY = 2 when the grid allows: the tile of
  // (BX+2)(BY+2) columns is then ~2x smaller per owned particle than with single columns)
  g.bx = (g.periodic_x ? g.nx >= 6 : g.nxo >= 2) ? 2 : 1;
  g.by = g.ny >= 6 ? 2 : 1;
  g.nbx = (g.nxo + g.bx - 1) / g.bx;
  g.nby = (g.ny + g.by - 1) / g.by;
  double ntot = n;
  if ((st = allreduce(c, &ntot, 1, kSum)) != SPH_OK) return st;  // same KZ on every rank
  const double occ = std::max(ntot, 1.0) / ((double)R * g.nxo * g.ny * g.nz);
  const int kz_max = std::min(kMaxTileCellsZ - 2, g.nz > 3 ? g.nz - 3 : 1);
  // largest KZ whose force tile (64 B per slot + 32 B per block particle) fits the target,
  // from the mean occupancy with a 10% margin; then checked against the real maximum below
  int KZ = 1;
  for (int k = 2; k <= kz_max; ++k) {
    const double slots = 1.1 * occ * (g.bx + 2) * (g.by + 2) * (k + 2);
    const double icnt = 1.1 * occ * g.bx * g.by * k;
    if (64.0 * slots + 32.0 * icnt > (double)kSmemTarget) break;
    KZ = k;
  }
  // the last rebuild's KZ is only a first probe: one above it (tiles may have shrunk since), then
  // the hint itself if that does not fit, then a bisection below
  const int hint = (c->kz_hint > 0 && c->kz_hint < KZ) ? c->kz_hint : 0;
  // (a KZ taken at one force CTA per SM: a taller block cannot fit two CTAs, and one CTA takes at
  // most KZ = 2 -- probe the hint itself first)
  if (hint) KZ = c->kz_hint_1cta ? hint : hint + 1;
  if (c->cfg.tile_cells_z > 0) KZ = c->cfg.tile_cells_z;
  KZ = std::max(1, std::min(KZ, kz_max));
  g.lists_warps = 8;  // (the largest k_lists CTA for the fit test)
  // the largest KZ <= the estimate whose tiles fit (tile sizes grow with KZ): the estimate
  // first, then a bisection over [1, KZ) when it does not fit (several probes on a grid
  // whose densest tiles are far above the mean, e.g. clustered boxes)
  int kz_lo = 0, kz_hi = KZ + 1;  // fits at kz_lo (0: none known), not at kz_hi
  bool probing = false;
  for (;;) {
    g.KZ = KZ;
    g.nzb = (g.nz + KZ - 1) / KZ;
    g.nblocks = g.nbx * g.nby * g.nzb;
    CK(zero_async(c->scratch + 6, 8, c->stream));
    c->launches++;
    // the blocks with i particles (flagged from the occupied cells, compacted in block order: one
    // loop CTA each), then the largest tile and i count over those blocks only (a clustered box
    // on a fine grid has mostly empty blocks); the last probe is at the chosen KZ
    if ((st = grow_h(c, &c->act_flag, c->act_cap, (size_t)g.nblocks)) != SPH_OK) return st;
    if ((st = grow_h(c, &c->blk_list, c->list_cap, (size_t)g.nblocks)) != SPH_OK) return st;
    CK(zero_async(c->act_flag, (size_t)g.nblocks, c->stream));
    c->launches++;
    CK(launch_block_flags(n, c->keys_alt, g, c->act_flag, c->stream));
    {
      thrust::counting_iterator<int> it(0);
      size_t need = 0;
      int* nact_dev = reinterpret_cast<int*>(c->scratch + 12);
      CK(cub::DeviceSelect::Flagged(nullptr, need, it, c->act_flag, c->blk_list, nact_dev, g.nblocks, c->stream));
      if (need > c->sel_tmp_bytes) {
        if (c->sel_tmp) cudaFree(c->sel_tmp);
        c->sel_tmp = nullptr;
        CK(cudaMalloc(&c->sel_tmp, need));
        c->sel_tmp_bytes = need;
      }
      CK(cub::DeviceSelect::Flagged(c->sel_tmp, need, it, c->act_flag, c->blk_list, nact_dev, g.nblocks, c->stream));
      CK(launch_tile_sizes_list(g, c->cell_start, c->blk_list, nact_dev, (int*)(c->scratch + 6),
                                (int*)(c->scratch + 7), c->stream));
    }
    c->launches += 3;
    if ((st = allreduce_dev(c, c->scratch + 6, 2, kMax)) != SPH_OK) return st;  // same capacities on every rank
    CK(copy_chunked(c->scratch_h + 6, c->scratch + 6, 8, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(copy_chunked(c->scratch_h + 12, c->scratch + 12, 4, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
    double tmax[2] = {(double)c->scratch_h[6], (double)c->scratch_h[7]};
    g.tcap = std::max(32, (int)tmax[0]);
    g.icap = std::max(32, (int)tmax[1]);
    g.lcap = c->lcap;
    g.skin = c->cfg.cell_skin;
    // force: 256 threads when two CTAs fit an SM, else one CTA of 512
    g.force_threads = 448;
    if (force_smem(g) > kSmemTarget) g.force_threads = 512;
    const bool fits = force_smem(g) <= kSmemMax && lists_smem(g) <= kSmemMax && density_smem(g) <= kSmemMax &&
                      gradient_smem(g) <= kSmemMax && g.tcap < 32760;  // (list entries: 15-bit slots)
    // (KZ <= 2 is taken at one force CTA per SM too: C3 Sedov 128^3 at KZ = 2 with one CTA 6.66 ms
    // per step against 7.90 at KZ = 1 with two -- the list build gains more from the taller blocks)
    const bool ok = fits && (force_smem(g) <= kSmemTarget || KZ <= 2);
    if (fits && c->cfg.tile_cells_z > 0) break;
    if (!probing && ok) break;  // the estimate fits
    if (ok) kz_lo = KZ; else kz_hi = KZ;
    if (!ok && KZ == 1) {
      char b[256];
      snprintf(b, sizeof b, "largest cell tile (%d particles) exceeds shared memory; h contrast too high for one grid", g.tcap);
      return fail(c, SPH_ERR_H_EXCEEDS_CELL, b);
    }
    probing = true;
    if (kz_hi - kz_lo <= 1) {
      if (KZ == kz_lo) break;  // (the state of the last probe is the answer)
      KZ = kz_lo;              // re-probe the answer so g holds its sizes
      continue;
    }
    KZ = kz_lo == 0 ? (hint && hint < kz_hi ? hint : std::max(1, kz_hi / 2)) : (kz_lo + kz_hi) / 2;
  }
  c->kz_hint = g.KZ;
  c->kz_hint_1cta = force_smem(g) > kSmemTarget;
  {
    const char* e = getenv("SPH_DENS_INNER");  // (tuning: Newton iterations per pass inside the CTA)
    g.dens_inner = e ? std::max(1, atoi(e)) : 6;
  }
  c->n_coinc = (long long)c->scratch_h[14];  // (the tile-size probes synchronised the stream)
  g.coinc = c->n_coinc > 0 ? 1 : 0;
  stage("KZ chosen");
  // the blocks with i particles of the last probe (its KZ), in block order
  g.nact = n > 0 ? (int)c->scratch_h[12] : 0;
  g.blk_list = c->blk_list;
  // k_lists: about one warp per 32 particles of a mean block (+10 %); the warps of a larger CTA
  // would only wait at its final barrier (the tile, not the warp count, limits CTAs per SM)
  g.lists_warps = std::max(2, std::min(8, (int)std::ceil(1.1 * n / std::max(g.nact, 1) / 32.0)));
  // rounding error of a tile coordinate: offsets reach (B/2 + 1) cells from the block centre
  const float max_off = std::max(std::max((0.5f * g.bx + 1.0f) * g.side[0], (0.5f * g.by + 1.0f) * g.side[1]),
                                 (0.5f * g.KZ + 1.0f) * g.side[2]);
  g.eabs = 4.0f * ulp_of(max_off) * 2.0f;  // 8 x (ulp/2): two coordinates per difference, with margin
  {
    // k_lists tests candidates in fp16 (unit roundoff 2^-11) on coordinates of magnitude <= C
    // cells: each coordinate difference errs by <= 2^-11 (2 C + |d|), |d| <= ~1.5 cells near
    // the list radius, the squares and sums by a few more ulps; the margin covers all of it
    const float C = max_off / g.side_min;
    g.lpad = std::ldexp(1.0f, -11) * (1.7321f * (2.0f * C + 3.0f) + 4.0f);
  }
  if (getenv("SPH_DEBUG")) {
    std::vector<int> cs(std::min(g.ncells, 1 << 24) + 1);  // (the monotonicity check on small grids only)
    copy_chunked(cs.data(), c->cell_start, cs.size() * 4, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    int bad = 0;
    for (size_t k = 0; k + 1 < cs.size(); ++k) bad += cs[k + 1] < cs[k];
    fprintf(stderr, "[sph rank %d] nx %d ny %d nz %d nxo %d ix_first %d bx %d by %d nbx %d nby %d KZ %d nzb %d nblocks %d "
            "nact %d tcap %d n_own %d gL %d gR %d planeL %d planeR %d cs0 %d csN %d nonmono %d x_lo %u wfix %llu\n",
            c->rank, g.nx, g.ny, g.nz, g.nxo, g.ix_first, g.bx, g.by, g.nbx, g.nby, g.KZ, g.nzb, g.nblocks, g.nact, g.tcap,
            c->n_own, c->gL, c->gR, c->planeL, c->planeR, cs[0], cs[cs.size() - 1], bad, g.x_lo, g.wfix);
  }
  stage("active blocks");
  // per-block tile descriptors for the loop kernels (k_tile_desc)
  const size_t na = (size_t)std::max(g.nact, 1);
  if ((st = grow_h(c, &c->desc_buf, c->desc_cap, na * tile_desc_bytes())) != SPH_OK) return st;
  g.desc = c->desc_buf;
  g.desc_cells = c->desc_buf + na * tile_desc_header_bytes();
  if ((st = grow_h(c, &c->pref_buf, c->pref_cap, 2 * na * (g.icap + 1))) != SPH_OK) return st;
  g.desc_pref = c->pref_buf;
  g.desc_prefF = c->pref_buf + na * (g.icap + 1);
  // (the i columns of every active block now; the full descriptors once the blocks the loops run
  // are known, at the end of mark_wide)
  CK(launch_tile_icols(g, c->cell_start, c->stream));
  c->launches++;
  const size_t blk_old = c->blk_cap;
  if ((st = grow_h(c, &c->blk[0], c->blk_cap, na)) != SPH_OK) return st;
  if (!c->blk[1] || c->blk_cap != blk_old) {  // (same capacity as blk[0])
    if (c->blk[1]) cudaFree(c->blk[1]);
    c->blk[1] = nullptr;
    CK(dalloc(&c->blk[1], c->blk_cap));
  }
  stage("descriptors");
  g.nrun = g.nact;  // (mark_wide narrows it to the blocks with tile particles)
  g.run_list = nullptr;
  if (slab) {
    // interior / boundary active blocks (the halo exchanges overlap the interior ones)
    if ((st = grow_h(c, &c->side_flag, c->side_flag_cap, 2 * na)) != SPH_OK) return st;
    if ((st = grow_h(c, &c->side_list, c->side_cap, 2 * na)) != SPH_OK) return st;
    CK(launch_block_side(g, c->side_flag, c->side_flag + na, c->stream));
    c->launches++;
    thrust::counting_iterator<int> it(0);
    size_t need = 0;
    int* n_dev = reinterpret_cast<int*>(c->scratch + 8);
    CK(cub::DeviceSelect::Flagged(nullptr, need, it, c->side_flag, c->side_list, n_dev, g.nact, c->stream));
    if (need > c->sel_tmp_bytes) {
      if (c->sel_tmp) cudaFree(c->sel_tmp);
      c->sel_tmp = nullptr;
      CK(cudaMalloc(&c->sel_tmp, need));
      c->sel_tmp_bytes = need;
    }
    CK(cub::DeviceSelect::Flagged(c->sel_tmp, need, it, c->side_flag, c->side_list, n_dev, g.nact, c->stream));
    CK(cub::DeviceSelect::Flagged(c->sel_tmp, need, it, c->side_flag + na, c->side_list + na, n_dev + 1, g.nact,
                                  c->stream));
    c->launches += 2;
    CK(copy_chunked(c->scratch_h + 8, c->scratch + 8, 8, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
    c->n_int = g.nact > 0 ? (int)c->scratch_h[8] : 0;
    c->n_bnd = g.nact > 0 ? (int)c->scratch_h[9] : 0;
  }
  c->stale = false;
  c->lists_stale = true;
  c->dvc_valid = false;
  // the particles were re-sorted: every per-particle result of the loops is in the old order
  c->density_done = c->gradient_done = false;
  return SPH_OK;
}

__global__ void k_h_keys(int n, const uint4* __restrict__ xh, unsigned int* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = xh[i].w;  // positive f32: ordered as unsigned
}

// q-quantile of the owned particles' h (device radix sort of the f32 bits).  global (slab
// path): the largest of the ranks' quantiles (a collective: every rank calls it)
sph_status h_quantile(sph_ctx* c, double q, float* out, bool global) {
  const int n = c->n_own;
  global = global && c->slab;
  if (n <= 0 && !global) return fail(c, SPH_ERR_INVALID_ARG, "no particles");
  CK(zero_async(c->scratch + 9, 4, c->stream));
  c->launches++;
  if (n > 0) {
    k_h_keys<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->s.xh + c->gL, c->keys);
    c->launches++;
    CK(cudaGetLastError());
    size_t tmp = c->sort_tmp_bytes;
    CK(cub::DeviceRadixSort::SortKeys(c->sort_tmp, tmp, c->keys, c->keys_alt, n, 0, 32, c->stream));
    const int k = std::min(n - 1, std::max(0, (int)(q * (n - 1))));
    k_copy_u32<<<1, 1, 0, c->stream>>>(c->keys_alt + k, reinterpret_cast<unsigned int*>(c->scratch + 9));
    c->launches++;
    CK(cudaGetLastError());
  }
  sph_status st;
  if (global && (st = allreduce_dev(c, c->scratch + 9, 1, kMax)) != SPH_OK) return st;
  CK(copy_chunked(c->scratch_h + 9, c->scratch + 9, 4, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  std::memcpy(out, c->scratch_h + 9, 4);
  if (!(*out > 0.f)) return fail(c, SPH_ERR_INVALID_ARG, "no particles");
  return SPH_OK;
}

// a wide ghost (index outside the owned range [lo, hi))
struct GhostFlag {
  const uint8_t* w;
  int lo, hi;
  __host__ __device__ bool operator()(int i) const { return w[i] != 0 && (i < lo || i >= hi); }
};

// Flag and list the wide particles of the current grid (none unless the side was sized from
// an h quantile).
sph_status mark_wide_impl(sph_ctx* c);

// The wide set and the loops' run list (mark_wide_impl), then the tile descriptors of the blocks
// the loops run (k_tile_desc; every active block without wide particles).
sph_status mark_wide(sph_ctx* c) {
  const sph_status st = mark_wide_impl(c);
  if (st != SPH_OK) return st;
  CK(launch_tile_desc(c->grid, c->cell_start, c->stream));
  c->launches++;
  return SPH_OK;
}

sph_status mark_wide_impl(sph_ctx* c) {
  DevState& s = c->s;
  s.n_wide = s.n_wide_own = 0;
  s.wide = nullptr;
  c->grid.nrun = c->grid.nact;
  c->grid.run_list = nullptr;
  if (c->h_side <= 0.f) return SPH_OK;
  const int n = c->n_own;
  // slab path: the ghosts are flagged too (a ghost whose support reaches an owned particle beyond
  // the neighbouring cells evaluates that pair here, k_wide_force)
  const int n_loc = c->gL + n + c->gR;
  if (!c->wide_flag) {
    CK(dalloc(&c->wide_flag, (size_t)c->cap));
    CK(dalloc(&c->widx, (size_t)c->cap));
    CK(dalloc(&c->wcount, (size_t)c->cap));
    CK(dalloc(&c->n_wide_dev, 2));
  }
  // widx: the owned wide particles (ascending), then the ghost ones
  int nw = 0, nw_own = 0;
  auto select = [&]() -> sph_status {
    thrust::counting_iterator<int> it(c->gL);
    thrust::counting_iterator<int> it0(0);
    const GhostFlag gf{c->wide_flag, c->gL, c->gL + n};
    size_t need = 0, need2 = 0;
    CK(cub::DeviceSelect::Flagged(nullptr, need, it, c->wide_flag + c->gL, c->widx, c->n_wide_dev, n, c->stream));
    if (n_loc > n)
      CK(cub::DeviceSelect::If(nullptr, need2, it0, c->widx, c->n_wide_dev + 1, n_loc, gf, c->stream));
    need = std::max(need, need2);
    if (need > c->sel_tmp_bytes) {
      if (c->sel_tmp) cudaFree(c->sel_tmp);
      c->sel_tmp = nullptr;
      CK(cudaMalloc(&c->sel_tmp, need));
      c->sel_tmp_bytes = need;
    }
    CK(cub::DeviceSelect::Flagged(c->sel_tmp, need, it, c->wide_flag + c->gL, c->widx, c->n_wide_dev, n, c->stream));
    c->launches++;
    // (with the population counter n0 in the same read-back)
    CK(copy_chunked(c->scratch_h + 10, c->n_wide_dev, 4, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(copy_chunked(c->scratch_h + 15, c->scratch + 15, 4, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
    std::memcpy(&nw_own, c->scratch_h + 10, 4);
    nw = nw_own;
    if (n_loc > n) {
      CK(cub::DeviceSelect::If(c->sel_tmp, need, it0, c->widx + nw_own, c->n_wide_dev + 1, n_loc, gf, c->stream));
      c->launches++;
      CK(copy_chunked(c->scratch_h + 10, c->n_wide_dev + 1, 4, cudaMemcpyDeviceToHost, c->stream));
      c->launches++;
      CK(cudaStreamSynchronize(c->stream));
      int ng;
      std::memcpy(&ng, c->scratch_h + 10, 4);
      nw += ng;
    }
    return SPH_OK;
  };
  // wide: support past the cell side, or within wide_margin of it (the margin is dropped when it
  // would add more than 10 % to the wide set, e.g. a uniform region whose h sits at the threshold)
  sph_status sq;
  for (float margin : {c->wide_margin, 0.f}) {
    c->grid.wide_margin = margin;
    CK(zero_async(c->scratch + 15, 4, c->stream));
    c->launches++;
    CK(launch_mark_wide(n_loc, c->grid, c->phys, s, c->wide_flag, c->scratch + 15, c->stream));
    c->launches++;
    if ((sq = select()) != SPH_OK) return sq;
    const int n0 = (int)c->scratch_h[15];
    if (margin == 0.f || nw <= n0 + n0 / 10 + 1024) break;
  }
  // sparse blocks' tile particles are handled as wide too (k_sparse_wide)
  if (c->sparse_wide > 0 && nw > 0) {
    CK(launch_sparse_wide(c->grid, c->wide_flag, s.ncount, c->sparse_wide, c->stream));
    c->launches++;
    if ((sq = select()) != SPH_OK) return sq;
  }
  s.n_wide = nw;
  s.n_wide_own = nw_own;
  s.wide = c->wide_flag;
  if (nw > 0) {
    // the wide particles' search grid (sph_wide.cu): coarse cells of F^3 grid cells, F such
    // that a particle at the 99th percentile of h reaches about two coarse cells (this rank's
    // quantile: not a collective, the ranks' wide sets differ); all local particles, ghosts too
    DevGrid& g = c->grid;
    float hq = 0.f;
    if (n > 0 && (sq = h_quantile(c, c->coarse_q, &hq, false)) != SPH_OK) return sq;
    if (!(hq > 0.f)) hq = c->h_side;
    const float R = (1.f + c->cfg.cell_skin) * c->cfg.gamma_k * hq;
    const float side = std::min(g.side[0], std::min(g.side[1], g.side[2]));
    const int Ftop = std::max(1, std::min(64, (int)std::ceil(R / (2.f * side))));
    // levels F/9, F/3, F (finest first; coarse_level takes the finest at least half a particle's
    // reach; with coarse_levels < kCoarseLevels the finest ones repeat the next), each capped to
    // 2^26 coarse cells
    for (int l = 0; l < kCoarseLevels; ++l) {
      int F = Ftop;
      for (int q = l; q < kCoarseLevels - 1; ++q) F = q + c->coarse_levels >= kCoarseLevels ? std::max(1, F / 3) : F;
      while ((long long)((g.nx + F - 1) / F) * ((g.ny + F - 1) / F) * ((g.nz + F - 1) / F) > (1LL << 26)) ++F;
      if (l > 0) F = std::max(F, s.cF[l - 1]);
      s.cF[l] = F;
      s.cnx[l] = (g.nx + F - 1) / F;
      s.cny[l] = (g.ny + F - 1) / F;
      s.cnz[l] = (g.nz + F - 1) / F;
    }
    for (int l = 0; l < kCoarseLevels; ++l) {
      if (l > 0 && s.cF[l] == s.cF[l - 1]) {  // (a repeated level shares the finer one's arrays)
        s.cperm[l] = s.cperm[l - 1];
        s.ccs[l] = s.ccs[l - 1];
        continue;
      }
      const long long ncc = (long long)s.cnx[l] * s.cny[l] * s.cnz[l];
      if ((sq = grow_h(c, &c->cperm[l], c->cperm_cap[l], (size_t)std::max(n_loc, 1))) != SPH_OK) return sq;
      if ((sq = grow_h(c, &c->ccs[l], c->ccs_cap[l], (size_t)ncc + 1)) != SPH_OK) return sq;
      CK(launch_coarse_keys(n_loc, l, g, s, c->keys, c->perm, c->stream));
      c->launches++;
      int bits = 1;
      while ((1LL << bits) <= ncc) ++bits;
      size_t tmp = c->sort_tmp_bytes;
      CK(cub::DeviceRadixSort::SortPairs(c->sort_tmp, tmp, c->keys, c->keys_alt, c->perm, c->cperm[l], n_loc, 0,
                                         bits, c->stream));
      c->launches++;
      k_cell_start<<<nblk(n_loc + 1, 256), 256, 0, c->stream>>>(n_loc, (int)ncc, 0, c->keys_alt, c->ccs[l]);
      c->launches++;
      CK(cudaGetLastError());
      s.cperm[l] = c->cperm[l];
      s.ccs[l] = c->ccs[l];
    }
  }
  if (nw > 0 && c->grid.nact > 0) {
    // the loop kernels run only the blocks with a non-wide i particle
    DevGrid& g = c->grid;
    const sph_status st = grow_h(c, &c->run_list, c->run_cap, (size_t)g.nact);
    if (st != SPH_OK) return st;
    CK(launch_block_run(g, s, c->act_flag, c->stream));
    c->launches++;
    size_t need2 = 0;
    thrust::counting_iterator<int> it(0);
    int* nrun_dev = reinterpret_cast<int*>(c->scratch + 13);
    CK(cub::DeviceSelect::Flagged(nullptr, need2, it, c->act_flag, c->run_list, nrun_dev, g.nact, c->stream));
    if (need2 > c->sel_tmp_bytes) {
      if (c->sel_tmp) cudaFree(c->sel_tmp);
      c->sel_tmp = nullptr;
      CK(cudaMalloc(&c->sel_tmp, need2));
      c->sel_tmp_bytes = need2;
    }
    CK(cub::DeviceSelect::Flagged(c->sel_tmp, need2, it, c->act_flag, c->run_list, nrun_dev, g.nact, c->stream));
    c->launches++;
    CK(copy_chunked(c->scratch_h + 13, c->scratch + 13, 4, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
    g.nrun = (int)c->scratch_h[13];
    g.run_list = c->run_list;
  }
  s.widx = c->widx;
  s.wcount = c->wcount;
  s.wlcap = c->wlcap;
  const size_t want = (size_t)std::max(nw, 1) * c->wlcap;
  if (want > c->wnbr_cap) {  // (with headroom: the wide set changes a little every rebuild)
    if (c->wnbr) cudaFree(c->wnbr);
    c->wnbr = nullptr;
    CK(dalloc(&c->wnbr, want + want / 2));
    c->wnbr_cap = want + want / 2;
  }
  s.wnbr = c->wnbr;
  return SPH_OK;
}

// Build the neighbour lists for the current grid and h (growing the capacity if needed).
sph_status build_lists(sph_ctx* c) {
  for (int attempt = 0; attempt < 4; ++attempt) {
    c->grid.lcap = c->lcap;
    CK(zero_async(&c->ctr->list_overflow, sizeof(int), c->stream));
    c->launches++;
    CK(zero_async(&c->ctr->wlist_overflow, sizeof(int), c->stream));
    c->launches++;
    CK(zero_async(&c->ctr->nonfinite, sizeof(int), c->stream));
    c->launches++;
    if (lists_smem(c->grid) > kSmemMax) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "neighbour lists exceed shared memory");
    {
      Timed tm(c, SPH_T_LISTS);
      CK(launch_lists(c->grid, c->phys, c->s, c->cell_start, c->ctr, c->stream));
      CK(launch_bank(c->gL, c->n_own, c->grid, c->s, c->stream));
      CK(launch_wide_lists(c->grid, c->phys, c->s, c->cell_start, c->ctr, c->stream));
    }
    c->launches += 2 + (c->s.n_wide > 0 ? 1 : 0);
    sph_status st = sync_ctr(c);
    if (st != SPH_OK) return st;
    const int wover = c->ctr_h->wlist_overflow;
    if (wover > 0) {  // wide lists: grow this rank's capacity (the retry below is collective)
      c->wlcap = ((int)(wover * 1.25) + 31) & ~31;
      c->s.wlcap = c->wlcap;
      const size_t want = (size_t)std::max(c->s.n_wide, 1) * c->wlcap;
      if (want > c->wnbr_cap) {
        if (c->wnbr) cudaFree(c->wnbr);
        c->wnbr = nullptr;
        CK(dalloc(&c->wnbr, want));
        c->wnbr_cap = want;
      }
      c->s.wnbr = c->wnbr;
    }
    double over = c->ctr_h->list_overflow, bad = c->ctr_h->nonfinite == 2 ? 1 : 0;
    double v[3] = {over, bad, (double)wover};
    if ((st = allreduce(c, v, 3, kMax)) != SPH_OK) return st;
    if (v[1] > 0) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
    if (v[0] == 0 && v[2] == 0) {
      c->lists_stale = false;
      return SPH_OK;
    }
    if (v[0] == 0) continue;  // (a wide list overflowed on some rank)
    int need = ((int)(v[0] * 1.25) + 7) & ~7;
    if (need > 8192) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "neighbour list longer than 8192 entries");
    c->lcap = need;
    size_t want = (size_t)c->cap * c->lcap;
    if (want > c->nbr_cap) {
      cudaFree(c->s.nbr);
      cudaFree(c->s.nbr_raw);
      c->s.nbr = c->s.nbr_raw = nullptr;
      CK(dalloc(&c->s.nbr, want));
      CK(dalloc(&c->s.nbr_raw, want));
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
  cfg->transport = SPH_TRANSPORT_NCCL;
  cfg->nccl_uid = nullptr;
  cfg->loopback = nullptr;
  cfg->adaptive_h = 1;
  cfg->decomp[0] = cfg->decomp[1] = cfg->decomp[2] = 0;
  cfg->halo_put = -1;
}

sph_status sph_nccl_unique_id(void* out128) {
  if (!out128) return SPH_ERR_INVALID_ARG;
  return nccl_unique_id(out128).empty() ? SPH_OK : SPH_ERR_NCCL;
}

sph_status sph_loopback_create(int nranks, void** out) {
  if (!out || nranks < 1) return SPH_ERR_INVALID_ARG;
  *out = loopback_group_create(nranks);
  return SPH_OK;
}

sph_status sph_loopback_destroy(void* group) {
  if (group) loopback_group_destroy(group);
  return SPH_OK;
}

sph_status sph_create(const sph_config* cfg, const sph_particles_in* in, sph_ctx** out) {
  if (!out) return SPH_ERR_INVALID_ARG;
  *out = nullptr;
  sph_ctx* c = new (std::nothrow) sph_ctx();
  if (!c) return SPH_ERR_OOM;
  sph_status st = validate_cfg(c, cfg);
  if (st != SPH_OK) { delete c; return st; }
  if (!in || in->n < 0 || in->n > (int64_t)0x3fffffff || (cfg->nranks == 1 && in->n <= 0)) {
    delete c;
    return SPH_ERR_INVALID_ARG;
  }
  c->cfg = *cfg;
  c->n_in = (int)in->n;
  c->nranks = cfg->nranks;
  c->rank = cfg->rank;
  c->device = cfg->device;
  c->slab = cfg->nranks > 1 || cfg->nccl_uid || (cfg->transport == SPH_TRANSPORT_LOOPBACK && cfg->loopback);
  if (!c->slab) {
    c->cap = c->n_in;
  } else {
    // SPH_GHOST_PLANES: more than one ghost plane per side (a test hook for the G-plane layout)
    if (const char* e = getenv("SPH_GHOST_PLANES")) c->gplanes = std::max(1, std::min(kMaxGhostPlanes, atoi(e)));
    const double per = (double)cfg->n_total / c->nranks;
    const double plane = std::pow((double)cfg->n_total, 2.0 / 3.0);
    // ghosts: ~3 particle layers per cell plane; adaptive_h may need up to kMaxGhostPlanes per side
    const double gmax = cfg->adaptive_h ? kMaxGhostPlanes : c->gplanes;
    c->cap = (int)std::min<double>(0x3fffffff, 1.5 * std::max<double>(per, c->n_in) +
                                                   (4.0 + 3.0 * 2.0 * gmax) * plane + 65536);
  }
  auto bail = [&](sph_status s) { sph_destroy(c); return s; };
  if (cudaSetDevice(c->device) != cudaSuccess) return bail(SPH_ERR_CUDA);
  if (cfg->stream) {
    c->stream = (cudaStream_t)cfg->stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SPH_ERR_CUDA);
    c->own_stream = true;
  }
  if (c->slab) {
    if (cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_main, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_x2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_x3, cudaEventDisableTiming) != cudaSuccess)
      return bail(SPH_ERR_CUDA);
    std::string e;
    c->comm = cfg->transport == SPH_TRANSPORT_LOOPBACK ? make_loopback_comm(cfg->loopback, c->rank, e)
                                                       : make_nccl_comm(cfg->nccl_uid, c->rank, c->nranks, e);
    if (!c->comm) {
      fail(c, SPH_ERR_NCCL, e);
      fprintf(stderr, "sph_create: %s\n", e.c_str());
      return bail(SPH_ERR_NCCL);
    }
  }
  fill_phys(c);
  if (const char* m = getenv("SPH_WIDE_MARGIN")) c->wide_margin = (float)std::max(0.0, atof(m));
  if (const char* m = getenv("SPH_SPARSE_WIDE")) c->sparse_wide = std::max(0, atoi(m));
  if (const char* m = getenv("SPH_COARSE_Q")) c->coarse_q = std::min(1.0, std::max(0.01, atof(m)));
  if (const char* m = getenv("SPH_COARSE_LEVELS")) c->coarse_levels = std::min(kCoarseLevels, std::max(1, atoi(m)));
  c->cut.resize(c->nranks + 1);
  for (int r = 0; r <= c->nranks; ++r)
    c->cut[r] = (unsigned long long)(((unsigned __int128)r << 32) / (unsigned)c->nranks);
  c->balance = cfg->balance != 0;
  if ((st = alloc_state(c)) != SPH_OK) return bail(st);
  if (c->slab) {
    c->halo_put = cfg->halo_put == 1 ||
                  (cfg->halo_put < 0 && (cfg->transport == SPH_TRANSPORT_LOOPBACK || c->nranks == 1));
    if (c->halo_put) {
      if (dalloc(&c->hin, (size_t)c->cap) != cudaSuccess) return bail(SPH_ERR_OOM);
      void* const mine[6] = {c->s.fr1, c->s.fr2, c->s.gq, c->s.vc, c->s.um, c->hin};
      void* p[6][2];
      std::string e;
      for (int k = 0; k < 6 && e.empty(); ++k)
        e = c->comm->map_peer(mine[k], left_of(c), right_of(c), &p[k][0], &p[k][1], c->stream);
      if (!e.empty()) {
        fail(c, SPH_ERR_NCCL, "halo put: " + e);
        fprintf(stderr, "sph_create: %s\n", c->err.c_str());
        return bail(SPH_ERR_NCCL);
      }
      for (int d = 0; d < 2; ++d) {
        c->peer_fr1[d] = static_cast<float4*>(p[0][d]);
        c->peer_fr2[d] = static_cast<float4*>(p[1][d]);
        c->peer_gq[d] = static_cast<float4*>(p[2][d]);
        c->peer_vc[d] = static_cast<float4*>(p[3][d]);
        c->peer_um[d] = static_cast<float2*>(p[4][d]);
        c->peer_h[d] = static_cast<float*>(p[5][d]);
      }
    }
  }
  if ((st = ingest(c, in)) != SPH_OK) return bail(st);
  if ((st = rebuild(c)) != SPH_OK) {
    fprintf(stderr, "sph_create: %s\n", c->err.c_str());
    return bail(st);
  }
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
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  return ingest(c, in);
}

sph_status sph_rebuild_cells(sph_ctx* c) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  return rebuild(c);
}

sph_status sph_density(sph_ctx* c, sph_density_stats* stats) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  sph_status st;
  if (c->stale && (st = rebuild(c)) != SPH_OK) return st;
  if (c->ghost_v_stale && (st = halo(c, c->s.vm, sizeof(float4))) != SPH_OK) return st;
  c->ghost_v_stale = false;
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
    CK(zero_async(bout, (size_t)std::max(c->grid.nact, 1), c->stream));
    c->launches++;
    CK(zero_async(&c->ctr->active_next, 3 * sizeof(int), c->stream));
  c->launches++;  // active_next, list_stale, overflow
    CK(zero_async(&c->ctr->h_exceeds, sizeof(int), c->stream));
    c->launches++;
    {
      Timed tm(c, SPH_T_DENSITY);
      CK(launch_density(c->grid, c->phys, c->s, c->cell_start, pass, bin, bout, 1.f + c->cfg.cell_skin, c->ctr,
                        c->stream));
      CK(launch_wide_density(c->grid, c->phys, c->s, pass, 1.f + c->cfg.cell_skin, c->ctr, c->stream));
    }
    c->launches += 1 + (c->s.n_wide > 0 ? 1 : 0);
    ++passes_run;
    // every rank takes the same branch: the pass's flags (unconverged .. max_resid_bits, nine
    // uint32 in DevCounters) are reduced over ranks on the device (MAX), then read back once; the
    // unconverged count is then the largest over ranks (no host allreduce after the pass loop, so
    // the X2 exchange below overlaps the gradient loop's interior blocks)
    if ((st = allreduce_dev(c, &c->ctr->unconverged, 9, kMax)) != SPH_OK) return st;
    if ((st = sync_ctr(c)) != SPH_OK) return st;
    double fl[4] = {(double)c->ctr_h->active_next, (double)c->ctr_h->h_exceeds, (double)c->ctr_h->list_stale,
                    c->ctr_h->nonfinite == 2 ? 1.0 : 0.0};
    if (fl[3] > 0) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
    if (fl[0] == 0) break;
    if (fl[1] > 0) {
      // an h grew past what the cell grid holds: rebin with the new h and restart the passes
      // (adaptive grid: the particle just becomes wide, no rebinning)
      if (++rebuilds > 8) return fail(c, SPH_ERR_H_EXCEEDS_CELL, "h kept outgrowing the cell grid");
      pairs_all += (long long)c->ctr_h->pairs_all;
      if (c->h_side > 0.f && !c->slab) {
        Timed tm(c, SPH_T_REBUILD);
        if ((st = mark_wide(c)) != SPH_OK) return st;
      } else if ((st = rebuild(c)) != SPH_OK) {
        return st;
      }
      if ((st = build_lists(c)) != SPH_OK) return st;
      if ((st = reset_ctr(c)) != SPH_OK) return st;
      pass = 0;
      continue;
    }
    if (fl[2] > 0) {
      // an h outgrew its list radius: refresh the ghosts' h, rebuild the lists, keep iterating
      if ((st = halo(c, c->s.xh, sizeof(uint4))) != SPH_OK) return st;
      if ((st = build_lists(c)) != SPH_OK) return st;
    }
    ++pass;
  }
  final_pairs = c->ctr_h->pairs;
  pairs_all += (long long)c->ctr_h->pairs_all;
  unconverged = c->ctr_h->unconverged;
  // ghosts need the final h and the gradient-loop record of their owners (X2)
  if (c->slab) {
    if (c->halo_put) {
      // the density epilogues stored gq / vc / um in the neighbours' ghost slots and h in their
      // hin: the token orders that before this rank takes its ghost h from hin (and before the
      // neighbours' gradient boundary blocks)
      if ((st = halo_token(c)) != SPH_OK) return st;
      if (c->gL + c->gR > 0) {
        k_ghost_h<<<nblk(c->gL + c->gR, 256), 256, 0, c->cstream>>>(c->gL, c->n_own, c->gR, c->hin, c->s.xh);
        CK(cudaGetLastError());
      }
      CK(cudaEventRecord(c->ev_x2, c->cstream));
    } else {
      void* const b[4] = {c->s.xh, c->s.gq, c->s.vc, c->s.um};
      const size_t e[4] = {sizeof(uint4), sizeof(float4), sizeof(float4), sizeof(float2)};
      if ((st = halo_async(c, b, e, 4, c->ev_x2)) != SPH_OK) return st;
    }
    c->x2_pending = true;
  }
  const double un = unconverged;  // (already the maximum over ranks)
  c->counters.pairs_density = (int64_t)final_pairs;
  c->counters.pairs_h_iter = pairs_all;
  c->density_done = true;
  c->gradient_done = false;
  c->dvc_valid = true;
  if (stats) {
    stats->iterations = passes_run;
    stats->unconverged = unconverged;
    stats->rebuilds = rebuilds;
    float mr;
    std::memcpy(&mr, &c->ctr_h->max_resid_bits, 4);
    stats->max_rel_resid = mr;
    stats->pairs_density = (int64_t)final_pairs;
    stats->pairs_h_iter = pairs_all;
  }
  if (un > 0) {
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
  if (!c->density_done || c->stale || c->lists_stale)
    return fail(c, SPH_ERR_STATE, "sph_gradient needs a completed sph_density on the current cells");
  if (!(dt > 0.f) || !std::isfinite(dt)) return fail(c, SPH_ERR_INVALID_ARG, "sph_gradient: dt must be > 0 (S:246)");
  sph_status st;
  if ((st = reset_ctr(c)) != SPH_OK) return st;
  const int first = c->dprev_valid ? 0 : 1;
  {
    Timed tm(c, SPH_T_GRADIENT);
    if (c->slab && c->x2_pending && !c->grid.run_list) {
      // interior blocks while the X2 halo (ghost h and gradient records) is in flight, then the
      // boundary blocks
      DevGrid gi = c->grid, gb = c->grid;
      gi.run_list = c->side_list;
      gi.nrun = c->n_int;
      gb.run_list = c->side_list + std::max(c->grid.nact, 1);
      gb.nrun = c->n_bnd;
      CK(launch_gradient(gi, c->phys, c->s, c->cell_start, dt, first, c->ctr, c->stream));
      if ((st = join_comm(c)) != SPH_OK) return st;
      CK(launch_gradient(gb, c->phys, c->s, c->cell_start, dt, first, c->ctr, c->stream));
      c->launches += 1;
    } else {
      if ((st = join_comm(c)) != SPH_OK) return st;
      CK(launch_gradient(c->grid, c->phys, c->s, c->cell_start, dt, first, c->ctr, c->stream));
    }
    CK(launch_wide_gradient(c->grid, c->phys, c->s, dt, first, c->ctr, c->stream));
  }
  c->launches += 1 + (c->s.n_wide > 0 ? 1 : 0);
  // (into pinned memory: a pageable destination would block the host until the loop ends;
  // sph_get_counters synchronises and reads it)
  CK(copy_chunked(c->pairs_grad_h, &c->ctr->pairs, 8, cudaMemcpyDeviceToHost, c->stream));
  c->launches++;
  // ghosts need their owners' force-loop records (X3): on the communication stream, overlapping
  // the force loop's interior blocks
  if (c->slab) {
    if (c->halo_put) {
      // the gradient epilogues stored the ghost records in the neighbours' buffers already: the
      // token orders the neighbours' boundary force blocks after them, and theirs before ours
      if ((st = halo_token(c)) != SPH_OK) return st;
      CK(cudaEventRecord(c->ev_x3, c->cstream));
    } else {
      void* const b[2] = {c->s.fr1, c->s.fr2};
      const size_t e[2] = {sizeof(float4), sizeof(float4)};
      if ((st = halo_async(c, b, e, 2, c->ev_x3)) != SPH_OK) return st;
    }
    c->x3_pending = true;
  }
  c->dprev_valid = true;
  c->gradient_done = true;
  return SPH_OK;
}

sph_status sph_force(sph_ctx* c, float* dt_next) {
  GUARD(c);
  if (!c->gradient_done || c->stale || c->lists_stale)
    return fail(c, SPH_ERR_STATE, "sph_force needs a completed sph_gradient on the current cells");
  sph_status st;
  if ((st = reset_ctr(c)) != SPH_OK) return st;
  // (dt_bits = +inf by a kernel, not a host copy: a copy would queue on the copy engines behind a
  // pipelined upload, sph_stage_particles, and a pageable one would block the host with it)
  k_set_u32<<<1, 1, 0, c->stream>>>(&c->ctr->dt_bits, 0x7f800000u);
  c->launches++;
  CK(cudaGetLastError());
  {
    Timed tm(c, SPH_T_FORCE);
    // the pair-once loop adds both sides of every pair into acc (ghost slots included)
    CK(zero_async(c->s.acc, sizeof(float4) * (size_t)(c->gL + c->n_own + c->gR), c->stream));
    c->launches++;
    if (c->slab && c->x3_pending && !c->grid.run_list) {
      // interior blocks while the X3 halo (ghost force records) is in flight, then the boundary
      DevGrid gi = c->grid, gb = c->grid;
      gi.run_list = c->side_list;
      gi.nrun = c->n_int;
      gb.run_list = c->side_list + std::max(c->grid.nact, 1);
      gb.nrun = c->n_bnd;
      CK(launch_force(gi, c->phys, c->s, c->cell_start, c->ctr, c->stream));
      if ((st = join_comm(c)) != SPH_OK) return st;
      CK(launch_force(gb, c->phys, c->s, c->cell_start, c->ctr, c->stream));
      c->launches += 1;
    } else {
      if ((st = join_comm(c)) != SPH_OK) return st;
      CK(launch_force(c->grid, c->phys, c->s, c->cell_start, c->ctr, c->stream));
    }
    CK(launch_wide_force(c->grid, c->phys, c->s, c->ctr, c->stream));
    CK(launch_force_fin(c->gL, c->n_own, c->phys, c->s, c->ctr, c->stream));
  }
  c->launches += 2 + (c->s.n_wide > 0 ? 2 : 0);
  // CFL dt: global minimum (X4; positive f32 bits order as uint32) and the error flag, reduced
  // on the device, one read-back
  if ((st = allreduce_dev(c, &c->ctr->dt_bits, 1, kMin)) != SPH_OK) return st;
  if ((st = allreduce_dev(c, &c->ctr->nonfinite, 1, kMax)) != SPH_OK) return st;
  if ((st = sync_ctr(c)) != SPH_OK) return st;
  c->counters.pairs_force = (int64_t)c->ctr_h->pairs;
  float dt;
  std::memcpy(&dt, &c->ctr_h->dt_bits, 4);
  const int mx = c->ctr_h->nonfinite;
  if (dt_next) *dt_next = dt;
  if (mx == 2) return fail(c, SPH_ERR_CUDA, "internal: tile larger than its capacity");
  if (mx > 0 || !std::isfinite(dt)) return fail(c, SPH_ERR_NUMERIC, "non-finite acceleration, v_sig or dt (S:262)");
  return SPH_OK;
}

sph_status sph_kick_drift(sph_ctx* c, float dt_kick, float dt_drift) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  if (!std::isfinite(dt_kick) || !std::isfinite(dt_drift)) return fail(c, SPH_ERR_INVALID_ARG, "non-finite dt");
  const double f[3] = {std::ldexp(1.0, 32) / c->cfg.box[0], std::ldexp(1.0, 32) / c->cfg.box[1],
                       std::ldexp(1.0, 32) / c->cfg.box[2]};
  const int o = c->gL, n = c->n_own;
  const float4* dvc = (c->cfg.predict_h && c->dvc_valid) ? c->s.dvc + o : nullptr;
  if (n > 0) {
    Timed tm(c, SPH_T_KICK_DRIFT);
    k_kick_drift<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->s.xh + o, c->s.vm + o, c->s.u + o, c->s.acc + o, dt_kick,
                                                      dt_drift, f[0], f[1], f[2], dvc);
    c->launches++;
  }
  CK(cudaGetLastError());
  if (dt_drift != 0.f) c->stale = true;
  else if (c->slab && dt_kick != 0.f) c->ghost_v_stale = true;
  c->density_done = c->gradient_done = false;
  return SPH_OK;
}

}  // extern "C"

namespace {
// Gather one field of the owned particles (caller order on one rank) into device memory d
// (sph_get / sph_get_async); *bytes = its size.  d = nullptr: size only.
sph_status gather_field(sph_ctx* c, int field, void* d, size_t* bytes) {
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
  // one rank: the caller's original order; several ranks: the owned particles in the local
  // (cell) order -- SPH_F_ID maps them to the caller's ids
  const int n = c->n_own;
  const int32_t* orig = c->nranks == 1 ? s.orig + c->gL : nullptr;
  *bytes = (size_t)n * comps * (wide ? 8 : 4);
  if (n == 0 || !d) return SPH_OK;
  if (wide)
    k_scatter64<<<nblk(n, 256), 256, 0, c->stream>>>(n, (const uint64_t*)src + c->gL, orig, (uint64_t*)d);
  else
    k_scatter32<<<nblk(n, 256), 256, 0, c->stream>>>(n, (const uint32_t*)src + (size_t)c->gL * stride, stride, off,
                                                     comps, orig, (uint32_t*)d);
  c->launches++;
  CK(cudaGetLastError());
  return SPH_OK;
}

// the copy streams and events of the pipelined host I/O (created on first use)
sph_status ensure_io(sph_ctx* c) {
  if (c->hstream) return SPH_OK;
  CK(cudaStreamCreateWithFlags(&c->hstream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->dstream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->h2stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_h2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_stage_free, cudaEventDisableTiming));
  for (int k = 0; k < sph_ctx::kGetSlots; ++k) {
    CK(cudaEventCreateWithFlags(&c->ev_gready[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_gfree[k], cudaEventDisableTiming));
  }
  return SPH_OK;
}
}  // namespace

extern "C" {

sph_status sph_get(sph_ctx* c, int field, void* dst, int on_device) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  if (!dst) return fail(c, SPH_ERR_INVALID_ARG, "dst is NULL");
  size_t bytes = 0;
  sph_status st = gather_field(c, field, nullptr, &bytes);
  if (st != SPH_OK || bytes == 0) return st;
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
  if ((st = gather_field(c, field, d, &bytes)) != SPH_OK) return st;
  if (!on_device) {
    CK(copy_chunked(dst, d, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->launches++;
    CK(cudaStreamSynchronize(c->stream));
  }
  return SPH_OK;
}

sph_status sph_get_async(sph_ctx* c, int field, void* dst) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;
  if (!dst) return fail(c, SPH_ERR_INVALID_ARG, "dst is NULL");
  sph_status st;
  if ((st = ensure_io(c)) != SPH_OK) return st;
  size_t bytes = 0;
  if ((st = gather_field(c, field, nullptr, &bytes)) != SPH_OK || bytes == 0) return st;
  const int k = c->gnext;
  c->gnext = (c->gnext + 1) % sph_ctx::kGetSlots;
  if (c->gbuf_bytes[k] < bytes) {
    if (c->gbuf[k]) cudaFree(c->gbuf[k]);  // (synchronises the device: the slot's copy is done)
    c->gbuf[k] = nullptr;
    c->gbuf_bytes[k] = 0;
    CK(cudaMalloc(&c->gbuf[k], bytes));
    c->gbuf_bytes[k] = bytes;
  } else if (c->gused[k]) {
    CK(cudaStreamWaitEvent(c->stream, c->ev_gfree[k], 0));  // the slot's previous copy is done
  }
  if ((st = gather_field(c, field, c->gbuf[k], &bytes)) != SPH_OK) return st;
  CK(cudaEventRecord(c->ev_gready[k], c->stream));
  CK(cudaStreamWaitEvent(c->dstream, c->ev_gready[k], 0));
  CK(copy_chunked(dst, c->gbuf[k], bytes, cudaMemcpyDeviceToHost, c->dstream));
  CK(cudaEventRecord(c->ev_gfree[k], c->dstream));
  c->gused[k] = true;
  return SPH_OK;
}

sph_status sph_stage_particles(sph_ctx* c, const sph_particles_in* in) {
  GUARD(c);
  if (!in || !in->X || !in->v || !in->m || !in->u || !in->h)
    return fail(c, SPH_ERR_INVALID_ARG, "required particle array is NULL");
  if (in->on_device) return fail(c, SPH_ERR_INVALID_ARG, "sph_stage_particles takes host arrays");
  if (in->n < 0 || (c->nranks == 1 && in->n != c->n_in) || in->n > c->cap)
    return fail(c, SPH_ERR_INVALID_ARG, "particle count mismatch / above capacity");
  sph_status st;
  if ((st = ensure_io(c)) != SPH_OK) return st;
  const size_t n = (size_t)in->n;
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  const size_t bytes = al(12 * n) * 2 + al(4 * n) * 3 + (in->alpha_v ? al(4 * n) : 0) + (in->alpha_c ? al(4 * n) : 0) +
                       (in->div_prev ? al(4 * n) : 0) + (in->id ? al(8 * n) : 0) + 16;
  if (c->stage_bytes < bytes) {
    if (c->stage_buf) cudaFree(c->stage_buf);  // (synchronises the device: no copy or ingest reads it)
    c->stage_buf = nullptr;
    c->stage_bytes = 0;
    CK(cudaMalloc(&c->stage_buf, bytes));
    c->stage_bytes = bytes;
  } else if (c->stage_used) {
    CK(cudaStreamWaitEvent(c->hstream, c->ev_stage_free, 0));  // the last staged upload was taken
    CK(cudaStreamWaitEvent(c->h2stream, c->ev_stage_free, 0));
  }
  // (SPH_H2D_CE_FRAC: the leading fraction of every array goes through the copy engines on a
  // second stream, the rest by kernel -- an experiment knob, default 0)
  static const double ce_frac = getenv("SPH_H2D_CE_FRAC") ? std::min(1.0, std::max(0.0, atof(getenv("SPH_H2D_CE_FRAC")))) : 0.0;
  char* d = static_cast<char*>(c->stage_buf);
  auto up = [&](const void* src, size_t b) -> void* {
    if (!src) return nullptr;
    void* dst = d;
    const size_t bce = ce_frac > 0.0 ? std::min(b, (size_t)(ce_frac * b) & ~size_t(15)) : 0;
    constexpr size_t kPiece = 4u << 20;
    for (size_t o = 0; o < bce; o += kPiece)
      cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kPiece, bce - o),
                      cudaMemcpyHostToDevice, c->h2stream);
    if (b > bce) {
      cudaError_t e_ = copy_chunked(static_cast<char*>(dst) + bce, static_cast<const char*>(src) + bce, b - bce,
                                    cudaMemcpyHostToDevice, c->hstream);
      (void)e_;
    }
    d += al(b);
    return dst;
  };
  sph_particles_in& sp = c->staged;
  sp = *in;
  sp.on_device = 1;
  sp.X = (const uint32_t*)up(in->X, 12 * n);
  sp.v = (const float*)up(in->v, 12 * n);
  sp.m = (const float*)up(in->m, 4 * n);
  sp.u = (const float*)up(in->u, 4 * n);
  sp.h = (const float*)up(in->h, 4 * n);
  sp.alpha_v = (const float*)up(in->alpha_v, 4 * n);
  sp.alpha_c = (const float*)up(in->alpha_c, 4 * n);
  sp.div_prev = (const float*)up(in->div_prev, 4 * n);
  sp.id = (const int64_t*)up(in->id, 8 * n);
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_h2, c->h2stream));
  CK(cudaStreamWaitEvent(c->hstream, c->ev_h2, 0));
  CK(cudaEventRecord(c->ev_staged, c->hstream));
  c->has_staged = true;
  return SPH_OK;
}

sph_status sph_set_particles_staged(sph_ctx* c) {
  GUARD(c);
  if (!c->has_staged) return fail(c, SPH_ERR_STATE, "sph_set_particles_staged: nothing staged");
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;  // (pending halo exchanges)
  CK(cudaStreamWaitEvent(c->stream, c->ev_staged, 0));
  const sph_status st = ingest(c, &c->staged);
  CK(cudaEventRecord(c->ev_stage_free, c->stream));
  c->has_staged = false;
  c->stage_used = true;
  return st;
}

int64_t sph_local_count(const sph_ctx* c) { return c ? (int64_t)c->n_own : -1; }

sph_status sph_get_counters(sph_ctx* c, sph_counters* out) {
  GUARD(c);
  if (!out) return SPH_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(c->stream));
  c->counters.pairs_gradient = (int64_t)*c->pairs_grad_h;
  c->counters.coincident = c->n_coinc;  // directed pairs, skipped by the loops (k_dup)
  c->counters.kernel_launches = c->launches;
  c->counters.wide_particles = c->s.n_wide;
  *out = c->counters;
  return SPH_OK;
}

sph_status sph_synchronize(sph_ctx* c) {
  GUARD(c);
  if (join_comm(c) != SPH_OK) return SPH_ERR_CUDA;
  CK(cudaStreamSynchronize(c->stream));
  if (c->hstream) CK(cudaStreamSynchronize(c->hstream));
  if (c->h2stream) CK(cudaStreamSynchronize(c->h2stream));
  if (c->dstream) CK(cudaStreamSynchronize(c->dstream));
  return SPH_OK;
}

sph_status sph_set_timing(sph_ctx* c, int on) {
  GUARD(c);
  c->timing = on != 0;
  return SPH_OK;
}

sph_status sph_get_timings(sph_ctx* c, sph_timings* out, int reset) {
  GUARD(c);
  CK(cudaStreamSynchronize(c->stream));
  for (const auto& t : c->tev) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    c->tms[t.kind] += ms;
    c->tcnt[t.kind] += 1;
    c->pool.push_back(t.a);
    c->pool.push_back(t.b);
  }
  c->tev.clear();
  if (out) {
    for (int k = 0; k < SPH_T_COUNT; ++k) {
      out->ms[k] = c->tms[k];
      out->count[k] = c->tcnt[k];
    }
  }
  if (reset) {
    for (int k = 0; k < SPH_T_COUNT; ++k) {
      c->tms[k] = 0.0;
      c->tcnt[k] = 0;
    }
  }
  return SPH_OK;
}

const char* sph_last_error(const sph_ctx* c) { return c ? c->err.c_str() : "context is NULL"; }

sph_status sph_destroy(sph_ctx* c) {
  if (!c) return SPH_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->cstream) cudaStreamSynchronize(c->cstream);
  for (cudaStream_t x : {c->hstream, c->dstream, c->h2stream})
    if (x) {
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
  for (cudaEvent_t e : {c->ev_staged, c->ev_stage_free, c->ev_h2})
    if (e) cudaEventDestroy(e);
  for (int k = 0; k < sph_ctx::kGetSlots; ++k) {
    if (c->ev_gready[k]) cudaEventDestroy(c->ev_gready[k]);
    if (c->ev_gfree[k]) cudaEventDestroy(c->ev_gfree[k]);
    if (c->gbuf[k]) cudaFree(c->gbuf[k]);
  }
  if (c->stage_buf) cudaFree(c->stage_buf);
  DevState& s = c->s;
  void* ptrs[] = {s.xh, s.vm, s.u, s.av, s.ac, s.dprev, s.uid, s.orig, s.acc, c->alt.xh, c->alt.vm, c->alt.u,
                  c->alt.av, c->alt.ac, c->alt.dprev, c->alt.uid, c->alt.orig, c->alt.acc, s.dens, s.dvc, s.count,
                  s.fin, s.gq, s.hlo, s.hhi, s.iters, s.active, s.grad, s.fr1, s.fr2, s.vsig, s.countf, s.nbr, s.nbr_raw,
                  s.ncount, s.hbuild, c->cell_start, c->keys, c->keys_alt, c->perm, c->perm_alt, c->sort_tmp,
                  c->blk[0], c->blk[1], c->ctr, c->scratch, c->out_tmp, c->mig_send, c->mig_recv, c->pc_send,
                  c->pc_recv, c->pc_scan, c->scan_tmp, c->cnt_dev, c->wide_flag, c->widx, c->wcount,
                  c->n_wide_dev, c->wnbr, c->sel_tmp, c->desc_buf, c->pref_buf,
                  c->act_flag, c->blk_list, c->run_list, c->cperm[0], c->cperm[1], c->cperm[2], c->ccs[0],
                  c->ccs[1], c->ccs[2], s.dup, c->side_flag, c->side_list,
                  s.vc, s.um, c->hin, c->xhist};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->ctr_h) cudaFreeHost(c->ctr_h);
  if (c->pairs_grad_h) cudaFreeHost(c->pairs_grad_h);
  if (c->scratch_h) cudaFreeHost(c->scratch_h);
  if (c->cnt_h) cudaFreeHost(c->cnt_h);
  for (const auto& t : c->tev) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  delete c->comm;
  for (cudaEvent_t e : {c->ev_main, c->ev_x2, c->ev_x3})
    if (e) cudaEventDestroy(e);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return SPH_OK;
}

}  // extern "C"
