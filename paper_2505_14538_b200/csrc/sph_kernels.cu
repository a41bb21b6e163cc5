// sph_kernels.cu -- sm_100a kernels of the SPH interaction loops of arXiv 2505.14538
// (density + h iteration, gradient + ghost, force + CFL dt).
//
// Decomposition.  The cell grid (side >= (1+skin) max support radius H = gamma_k h) is
// cut into CTA blocks of BX x BY grid columns x KZ cells.  A block's TILE is the
// particles of the (BX+2) x (BY+2) neighbour columns over its z range +-1 cell: at most
// 3 contiguous ranges of the cell-sorted arrays per column, staged into shared memory with
// cp.async (LDGSTS) and converted from fixed point to f32 offsets from the block centre.
//
// Bank-aware rows.  A loop gathers the records of 8 list entries per lane and step from the
// shared tile with one 16-byte load per record; the 8 lanes of a quarter-warp (one
// shared-memory phase) are conflict-free when their 8 slots lie in distinct 16-byte bank
// groups (slot mod 8).  The walk reads row entry (u + lane) mod 8 at sub-step u, so a row
// whose entry w lies in bank group w gives distinct groups to the 8 lanes at every sub-step,
// whatever rows and particles they are on.  k_bank therefore places the t-th entry of group
// b at row t, column b (t < R = ceil(n / 8)); the rare overflow of a group past R rows fills
// the free cells left (those gathers may conflict), every other free cell gets the sentinel
// slot of its group (tcap + group, a far-away zero record).  Lists longer than 8 kCellRows,
// or with a group of more than kCellRows entries, keep the natural order (correct, more
// conflicts).
//
// Neighbour lists.  k_lists tests, once per cell rebuild (and again only if an h outgrows
// its list radius), each particle's candidates in its 3 x 3 neighbour columns inside a z
// window of +-R (cells are z-sorted by the binning key, so a binary search finds the
// window) and stores, per particle, the tile slots j with r_ij < (1 + skin) max(H_i, H_j)
// (self included) as uint16, padded to a multiple of 8 with sentinel slots, in ROWS of 8 whose
// entry w lies in shared-memory bank group w (see "Bank-aware rows").  The density passes, the gradient loop and the force
// loop then run the pair arithmetic over these lists only: every lane works on a real (or
// skin) neighbour, no candidate is re-tested (the paper's pair tasks test all particle
// pairs of two cells).  Skin entries, the sentinel and the self pair contribute
// exactly zero (compact support, w'(0) = 0); membership (neighbour counts, v_sig) is decided
// in f32 with a rigorous band and re-decided in fp64 inside it, so counts equal the
// definition exactly.
#include <algorithm>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "sph_internal.cuh"
#include "sph_pair.cuh"

namespace sph {

extern __shared__ float4 smem4[];  // dynamic shared memory of every loop kernel

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNW = 8;              // warps per CTA
constexpr float kFar = 1.0e12f;     // sentinel position (tile coordinates)
constexpr int kMaxICols = 4;        // BX * BY <= 4
constexpr int kMaxSeg = 3 * 16;     // <= 3 contiguous segments per tile column
constexpr int kNSent = 8;           // sentinel slots tcap .. tcap+7, one per 16-byte bank group

struct Tile {
  int ix0, iy0, z0, z1, nzt, ntc, nct, ntile, ncol, ni;
  uint32_t ref[3];
};

// Shared block bookkeeping (static shared memory of every loop kernel).
struct BlockShared {
  int off[kMaxTileCells + 1];  // tile offset of each tile cell (exclusive prefix)
  int gst[kMaxTileCells];      // global index of the first particle of each tile cell
  int4 seg[kMaxSeg];           // contiguous segments (tile start, global start, length)
  int ib[kMaxICols];           // tile start of each i column of the block
  int g0[kMaxICols];           // global start of each i column
  int tc[kMaxICols];           // tile column of each i column
  int pre[kMaxICols + 1];      // prefix of i counts over the i columns
};

// A block's tile descriptor, computed once per rebuild (k_tile_desc: the tile geometry, the
// contiguous segments to stage, the i columns) and loaded by the loop kernels with one
// coalesced read instead of redoing tile_setup's cell scans and serial steps every launch.
struct TileDesc {
  Tile T;                      // 13 ints
  int ib[kMaxICols], g0[kMaxICols], tc[kMaxICols], pre[kMaxICols + 1];
  int pad[2];                  // (128-byte header)
  int4 seg[kMaxSeg];           // (tile start, global start, length) per segment
};
static_assert(sizeof(TileDesc) % 16 == 0, "TileDesc size");

// Launch order of the blocks: z fastest, then block columns in strips of kStrip columns
// along y, column-major inside a strip, so the blocks whose tiles share a column (its x and
// y neighbours) run within ~kStrip * nzb launches of each other and re-read the column's
// records from L2 rather than HBM (the tiles of one launch wave are ~20 MB).
constexpr int kStrip = 8;
__device__ __forceinline__ void block_coords(const DevGrid& g, int b, int& jx, int& jy, int& zb) {
  zb = b % g.nzb;
  const int c = b / g.nzb;
  const int s = c / (kStrip * g.nbx);
  const int hs = min(kStrip, g.nby - s * kStrip);
  const int local = c - s * kStrip * g.nbx;
  jx = local / hs;
  jy = s * kStrip + local % hs;
}

// Block geometry + tile cell table + i columns + segments.  Tile cell c = tc * nzt + zz,
// tile column tc = (dx+1) * (BY+2) + (dy+1) for dx in [-1, BX], dy in [-1, BY],
// zz = z - z0 + 1.  Ends with __syncthreads().
__device__ void tile_setup(const DevGrid& g, int b, const int* __restrict__ cell_start, BlockShared& S, Tile& T) {
  int jx, jy, zb;
  block_coords(g, b, jx, jy, zb);
  T.ix0 = g.ix_first + jx * g.bx;
  T.iy0 = jy * g.by;
  T.z0 = zb * g.KZ;
  T.z1 = min(g.nz, T.z0 + g.KZ);
  T.nzt = T.z1 - T.z0 + 2;
  T.ntc = (g.bx + 2) * (g.by + 2);
  T.nct = T.ntc * T.nzt;
  // block centre on the global 2^-32 grid (wraps mod 2^32 past the box edge)
  T.ref[0] = g.x_lo + (uint32_t)(((unsigned long long)(2 * (T.ix0 - g.ix_first) + g.bx) * g.wfix) /
                                 (2ull * (unsigned long long)g.nxo));
  T.ref[1] = (uint32_t)((((unsigned long long)(2 * T.iy0 + g.by)) << 31) / (unsigned long long)g.ny);
  T.ref[2] = (uint32_t)((((unsigned long long)(T.z0 + T.z1)) << 31) / (unsigned long long)g.nz);
  for (int t = threadIdx.x; t < T.nct; t += blockDim.x) {
    const int c = t / T.nzt, zz = t - c * T.nzt;
    int cx = T.ix0 + c / (g.by + 2) - 1, cy = T.iy0 + c % (g.by + 2) - 1, cz = T.z0 - 1 + zz;
    bool empty = false;
    if (g.periodic_x) {
      cx += (cx < 0) ? g.nx : 0;
      cx -= (cx >= g.nx) ? g.nx : 0;
    } else {
      empty = cx >= g.nx;  // past the right ghost plane (odd owned plane count)
      cx = min(cx, g.nx - 1);
    }
    cy += (cy < 0) ? g.ny : 0;
    cy -= (cy >= g.ny) ? g.ny : 0;
    cz += (cz < 0) ? g.nz : 0;
    cz -= (cz >= g.nz) ? g.nz : 0;
    const int cell = (cx * g.ny + cy) * g.nz + cz;
    const int gs = __ldg(cell_start + cell);
    S.gst[t] = empty ? 0 : gs;
    S.off[t + 1] = empty ? 0 : __ldg(cell_start + cell + 1) - gs;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int carry = 0;
    for (int base = 0; base < T.nct; base += 32) {
      const int t = base + lane;
      int v = t < T.nct ? S.off[t + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
      }
      if (t < T.nct) S.off[t + 1] = carry + v;
      carry += __shfl_sync(kFull, v, 31);
    }
    if (lane == 0) S.off[0] = 0;
  }
  __syncthreads();
  // i columns of the block (edge blocks may own fewer than BX x BY columns)
  if (threadIdx.x == 0) {
    int k = 0, acc = 0;
    for (int ex = 0; ex < g.bx; ++ex)
      for (int ey = 0; ey < g.by; ++ey) {
        if (T.ix0 + ex >= g.ix_first + g.nxo || T.iy0 + ey >= g.ny) continue;
        const int tc = (ex + 1) * (g.by + 2) + (ey + 1);
        S.tc[k] = tc;
        S.ib[k] = S.off[tc * T.nzt + 1];
        S.g0[k] = S.gst[tc * T.nzt + 1];  // an i column's cells are consecutive in the cell order
        S.pre[k] = acc;
        acc += S.off[tc * T.nzt + T.nzt - 1] - S.off[tc * T.nzt + 1];
        ++k;
      }
    S.pre[k] = acc;
    for (int r = k; r < kMaxICols; ++r) { S.tc[r] = 0; S.ib[r] = 0; S.g0[r] = 0; S.pre[r + 1] = acc; }
  }
  // contiguous segments: one thread per tile column
  if (threadIdx.x >= 32 && threadIdx.x < 32 + T.ntc) {
    const int col = threadIdx.x - 32;
    int n = 0;
    int4 cur = make_int4(0, 0, 0, 0);
    for (int zz = 0; zz < T.nzt; ++zz) {
      const int c = col * T.nzt + zz;
      const int len = S.off[c + 1] - S.off[c];
      // empty cells never split a segment (at most 3 per column: the two z wraps)
      if (zz > 0 && (len == 0 || cur.y + cur.z == S.gst[c])) {
        cur.z += len;
      } else if (zz > 0 && cur.z == 0) {
        cur = make_int4(S.off[c], S.gst[c], len, 0);
      } else {
        if (zz > 0) S.seg[col * 3 + n++] = cur;
        cur = make_int4(S.off[c], S.gst[c], len, 0);
      }
    }
    S.seg[col * 3 + n++] = cur;
    for (; n < 3; ++n) S.seg[col * 3 + n] = make_int4(0, 0, 0, 0);
  }
  __syncthreads();
  T.ntile = S.off[T.nct];
  int k = 0;
  while (k < kMaxICols && S.pre[k + 1] > S.pre[k]) ++k;
  T.ncol = k;
  T.ni = S.pre[kMaxICols];
}

// block-local i index -> (tile slot, global index)
template <class SS>
__device__ __forceinline__ void i_slot(const SS& S, int li, int& ti, int& gi) {
  int k = 0;
#pragma unroll
  for (int r = 1; r < kMaxICols; ++r) k += (li >= S.pre[r]) ? 1 : 0;
  ti = S.ib[k] + (li - S.pre[k]);
  gi = S.g0[k] + (li - S.pre[k]);
}

// tile slot -> global particle index from the staged segments (rare path)
__device__ __forceinline__ int slot_global(const TileDesc& D, int nseg, int t) {
  for (int k = 0; k < nseg; ++k) {
    const int4 sg = D.seg[k];
    if (t >= sg.x && t < sg.x + sg.z) return sg.y + (t - sg.x);
  }
  return 0;  // (unreachable for a slot of the tile)
}

__device__ __forceinline__ void cp_async16(const void* smem_dst, const void* gmem_src) {
  const unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async8(const void* smem_dst, const void* gmem_src) {
  const unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async4(const void* smem_dst, const void* gmem_src) {
  const unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// 16-byte shared-memory load at a 32-bit shared address: the loops gather their neighbour
// records this way from record-array bases held in registers (smem_base's opaque move keeps
// the compiler from rebuilding the shared window address before every gather)
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t smem_base(int rec) {
  uint32_t a;
  asm volatile("mov.u32 %0, %1;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(smem4) + (uint32_t)rec * 16u));
  return a;
}

// The tile staging's mbarrier (one per CTA, used once: phase 0).  Thread 0 initialises it
// before the kernel's first barrier (stage_mbar_init), stage_records waits on it.
__shared__ __align__(8) unsigned long long s_stage_mbar;
__device__ __forceinline__ uint32_t stage_mbar() { return (uint32_t)__cvta_generic_to_shared(&s_stage_mbar); }
__device__ __forceinline__ void stage_mbar_init() {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n"
               "fence.mbarrier_init.release.cluster;" ::"r"(stage_mbar())
               : "memory");
}

// Stage nrec16 16-byte per-particle records (at smem4[o16[r] + slot]) of every tile slot:
// each of the tile's contiguous segments (<= 3 per tile column, TileDesc::seg) is one 1-D
// bulk copy per record array (cp.async.bulk on the TMA engine, no per-lane loop), counted in
// bytes on the CTA's mbarrier (armed by thread 0 before the copies, __syncthreads of the
// prologue); lane 0 of every warp issues a share of them (the copies of one lane issue one
// after another).  Every thread then waits on the mbarrier (and on its own earlier cp.async
// copies), and the block synchronises.
template <int nrec16, class SS>
__device__ __forceinline__ void stage_records(const SS& S, int nseg, const float4* const* src16, const int* o16,
                                              int ntile) {
  const uint32_t mbar = stage_mbar();
  if (threadIdx.x == 0)
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(mbar),
                 "r"((uint32_t)(nrec16 * 16 * ntile))
                 : "memory");
  __syncthreads();
  {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem4);
    // copy c = (segment, record) of the CTA's nseg * nrec16: lane (c / nw) % 32 of warp c % nw
    for (int c = warp + nw * lane; c < nseg * nrec16; c += 32 * nw) {
      const int k = c % nseg, r = c / nseg;
      const int4 sg = S.seg[k];
      if (sg.z <= 0) continue;
      // (record r by selects: a dynamic index into src16 / o16 would put them in local memory)
      const float4* src = src16[0];
      int o = o16[0];
#pragma unroll
      for (int q = 1; q < nrec16; ++q)
        if (r == q) { src = src16[q]; o = o16[q]; }
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sbase + 16u * (uint32_t)(o + sg.x)),
          "l"(src + sg.y), "r"(16u * (uint32_t)sg.z), "r"(mbar)
          : "memory");
    }
  }
  cp_async_wait_all();
  asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W%=; }" ::"r"(mbar)
               : "memory");
  __syncthreads();
}

__device__ __forceinline__ float3 rel_pos(const DevGrid& g, const Tile& T, uint4 x) {
  return make_float3((float)(int)(x.x - T.ref[0]) * g.scale[0], (float)(int)(x.y - T.ref[1]) * g.scale[1],
                     (float)(int)(x.z - T.ref[2]) * g.scale[2]);
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Loop kernels: the block's descriptor from k_tile_desc (S.seg, S.ib, ... and T), one barrier.
// The active-block index of this CTA (the index of the per-block arrays).
__device__ __forceinline__ int blk_a(const DevGrid& g) { return g.run_list ? g.run_list[blockIdx.x] : (int)blockIdx.x; }

#define DESC_PROLOGUE()                                                          \
  __shared__ TileDesc S;                                                         \
  const int ba = blk_a(g); /* active-block index: descriptor, prefix, density flags */ \
  {                                                                              \
    const int* src_ = reinterpret_cast<const int*>(g.desc) + (size_t)ba * (sizeof(TileDesc) / 4); \
    int* dst_ = reinterpret_cast<int*>(&S);                                      \
    for (int q_ = threadIdx.x; q_ < (int)(sizeof(TileDesc) / 4); q_ += blockDim.x) dst_[q_] = __ldg(src_ + q_); \
    if (threadIdx.x == 0) stage_mbar_init();                                     \
  }                                                                              \
  __syncthreads();                                                               \
  const Tile T = S.T;                                                            \
  if (T.ntile > g.tcap) {                                                        \
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);                        \
    return;                                                                      \
  }                                                                              \
  const int nseg = 3 * T.ntc;                                                    \
  const int SP = g.tcap + kNSent; /* slots per record array (the last kNSent are sentinels) */

// ========================================================== neighbour lists ==========
// For every particle i of the block: all tile slots j (self included) with
// r_ij^2 < ((1 + skin) gamma_k max(h_i, h_j))^2, in tile order, padded to 8 with the
// sentinel slot tcap.  Superset of every loop's neighbour set while each h stays within
// (1 + skin) of its value here (checked by the density epilogue).
// One lane per particle i, each walking its OWN candidates: in each of the 3 x 3 tile
// columns around i's column, only the slots with |z_j - z_i| <= R (R = the largest list
// radius in the tile, plus the sort bucket and rounding slack), rounded out to 1/16-cell
// sub-buckets: each cell's particles are sorted by the top z bits of the sort key, so a
// per-block table of each sub-bucket's first slot (s_zw) gives both window ends with two
// loads.  This tests ~2R/(3 side) of the 27-cell candidates.
// The tile is staged pair-interleaved, P[8p .. 8p+7] = (x_2p, x_2p+1, y_2p, y_2p+1, z_2p,
// z_2p+1, H2_2p, H2_2p+1), so one lane tests two consecutive candidates with two LDS.128
// and packed f32x2 arithmetic (FADD2 / FMUL2 / FFMA2).  Hits go to a per-lane column of a
// per-warp buffer in shared memory and leave for global memory 8 at a time (16-byte stores);
// k_bank then lays each list out in bank-aware rows.  The CTA has about one warp per 32 of
// the mean block's particles (DevGrid::lists_warps).
__device__ void block_exclusive_scan(int* a, int n);
constexpr int kMaxICells = kMaxICols * (kMaxTileCellsZ - 2);
constexpr int kListRows = 32;  // ring rows per lane (<= 7 left + 2 single tests + 16 per group)
constexpr int kCellRows = 16;  // k_bank grid rows per list (longer lists keep the natural order)
constexpr int kZSub = 16;      // z sub-buckets per cell in k_lists' window table
// k_lists' dynamic shared memory after the pair array: the per-warp list rings and the group
// counts (holding one z sub-bucket byte per slot before the walk), then the z window table
// k_lists' dynamic shared memory: region A (the staged raw records; after the conversion to
// the fp16 candidate records, the per-warp list rings and the group counts), the candidate
// records P16, the slots' z sub-bucket bytes, the z window table, the wide flags
__host__ __device__ __forceinline__ size_t lists_a_bytes(const DevGrid& g, int nw) {
  const size_t raw = (size_t)((g.tcap + kNSent + 1) & ~1) * 16;
  const size_t ring = (size_t)nw * kListRows * 32 * 2 + (size_t)(g.icap + 1) * 8;
  return ((raw > ring ? raw : ring) + 15) & ~(size_t)15;
}
__host__ __device__ __forceinline__ size_t lists_slot_bytes(const DevGrid& g) {
  return ((size_t)g.tcap + kNSent + 15) & ~(size_t)15;
}
__host__ __device__ __forceinline__ size_t lists_zw_bytes(const DevGrid& g) {
  return ((((size_t)(g.bx + 2) * (g.by + 2) * (g.KZ + 2) * kZSub + 1) * 2 + 15) & ~(size_t)15);
}
// (the per-lane list buffers are touched only through these volatile asm statements, which
// keep their order; no memory clobber, so the compiler may move tile loads across them)
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_u16_if(uint32_t a, uint32_t v, bool p) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }\n" ::"r"(a),
               "h"((unsigned short)v), "r"((uint32_t)p));
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(a));
  return v;
}
// kTag: tag each entry as it leaves the ring (wide particles or ghost planes present); else the
// list is sorted by slot and its force part is simply its tail (position >= the count of
// entries up to the particle's own slot).
template <bool kWide, bool kTag>
__global__ void __launch_bounds__(kNW * 32, 4) k_lists(DevGrid g, DevPhys ph, DevState s,
                                                       const int* __restrict__ cell_start,
                                                       DevCounters* __restrict__ ctr) {
  __shared__ int s_cp[kMaxICells + 1];  // prefix of particle counts over the block's i cells
  __shared__ int s_ct[kMaxICells];      // tile start of each i cell
  __shared__ int s_cg[kMaxICells];      // global start of each i cell
  __shared__ unsigned int s_hmax;       // largest h of the tile (f32 bits)
  if (threadIdx.x == 0) s_hmax = 0u;
  const int nw = blockDim.x >> 5;  // warps (host-chosen from the mean block particle count)
  // the block's tile from its descriptor (k_tile_desc) instead of tile_setup
  __shared__ BlockShared S;
  const int ba = blk_a(g);
  __shared__ Tile Tsh;
  {
    const TileDesc* D = reinterpret_cast<const TileDesc*>(g.desc) + ba;
    if (threadIdx.x == 0) Tsh = D->T;
    if (threadIdx.x < kMaxICols) {
      S.ib[threadIdx.x] = D->ib[threadIdx.x];
      S.g0[threadIdx.x] = D->g0[threadIdx.x];
      S.tc[threadIdx.x] = D->tc[threadIdx.x];
    }
    if (threadIdx.x <= kMaxICols) S.pre[threadIdx.x] = D->pre[threadIdx.x];
    for (int q = threadIdx.x; q < kMaxSeg; q += blockDim.x) S.seg[q] = D->seg[q];
    const int nct = D->T.nct;
    const int2* C = reinterpret_cast<const int2*>(g.desc_cells) + (size_t)ba * (kMaxTileCells + 1);
    for (int c = threadIdx.x; c <= nct; c += blockDim.x) {
      const int2 v = __ldg(C + c);
      S.off[c] = v.x;
      if (c < nct) S.gst[c] = v.y;
    }
    if (threadIdx.x == 0) stage_mbar_init();
  }
  __syncthreads();
  const Tile T = Tsh;
  if (T.ntile > g.tcap) {
    if (threadIdx.x == 0) atomicExch(&ctr->nonfinite, 2);
    return;
  }
  const int nseg = 3 * T.ntc;
  const int SP = g.tcap + kNSent;
  const int NP = (SP + 1) >> 1;  // slot pairs
  float* P = reinterpret_cast<float*>(smem4);
  // z window table: s_zw[16 c + k] = first slot of tile cell c in z sub-bucket >= k (16 per
  // cell, the top 4 z bits inside the cell -- the sort key's, so exact), s_zw[16 nct] = end
  // (layout: lists_a_bytes)
  const size_t abytes = lists_a_bytes(g, nw);
  char* ring0 = reinterpret_cast<char*>(P);  // (after the conversion below)
  uint4* P16 = reinterpret_cast<uint4*>(reinterpret_cast<char*>(P) + abytes);
  unsigned char* zsb = reinterpret_cast<unsigned char*>(P16 + NP);
  unsigned short* s_zw = reinterpret_cast<unsigned short*>(zsb + lists_slot_bytes(g));
  // wide particles (adaptive grid): one flag byte per slot after the window table (a wide
  // partner's pair is never in the force part: k_wide_force applies it to both sides)
  unsigned char* wfl = reinterpret_cast<unsigned char*>(s_zw) + lists_zw_bytes(g);  // (lists_slot_bytes)
  // (bit 0: wide, bit 1: a coincident partner exists, k_dup)
  if (kWide || g.coinc) {
    const int lane_ = threadIdx.x & 31;
    for (int k = threadIdx.x >> 5; k < nseg; k += nw) {
      const int4 sg = S.seg[k];
      for (int t = lane_; t < sg.z; t += 32)
        wfl[sg.x + t] = (kWide ? s.wide[sg.y + t] : 0) | (g.coinc ? (s.dup[sg.y + t] << 1) : 0);
    }
  }
  {
    const float4* src[1] = {reinterpret_cast<const float4*>(s.xh)};
    const int o16[1] = {0};
    stage_records<1>(S, nseg, src, o16, T.ntile);
  }
  const float Hfac = (1.f + g.skin) * ph.gamma_k;
  unsigned int hm = 0u;
  // each slot's z sub-bucket (bytes; the region of the list ring, not yet in use)
  const int zb4 = min(g.zbits, 4);
  const uint32_t zmask = (1u << (4 - zb4)) - 1u;  // (coarse sort keys: fewer sub-buckets)
  // Candidate records in fp16, pair-interleaved: P16[p] = (x, y, z, H^2) of slots 2p, 2p+1 as
  // half2, coordinates in units of the smallest cell side from the block centre.  The test
  // r^2 < max(H_i^2, H_j^2) in half precision only has to keep every pair of the f32 list
  // criterion: each list radius carries g.lpad cells for the fp16 rounding of the coordinates
  // and of the squares (host: from the largest tile offset), and H^2 is rounded up.  The extra
  // entries are skin entries (exactly zero in every loop).
  const float cs = 1.f / g.side_min;
  for (int pp = threadIdx.x; pp < NP; pp += blockDim.x) {
    float4 q[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = 2 * pp + u;
      q[u] = make_float4(3.0e4f, 3.0e4f, 3.0e4f, 0.f);
      if (t < T.ntile) {
        const uint4 x = reinterpret_cast<const uint4*>(smem4)[t];
        const float3 r = rel_pos(g, T, x);
        const float Hs = Hfac * __uint_as_float(x.w) * cs + g.lpad;
        hm = max(hm, x.w);
        q[u] = make_float4(r.x * cs, r.y * cs, r.z * cs, Hs * Hs);
        zsb[t] = (unsigned char)((((uint32_t)((unsigned long long)x.z * (unsigned)g.nz)) >> 28) & ~zmask);
      }
    }
    const __half2 hx = __floats2half2_rn(q[0].x, q[1].x), hy = __floats2half2_rn(q[0].y, q[1].y),
                  hz = __floats2half2_rn(q[0].z, q[1].z);
    const __half2 hh = __halves2half2(__float2half_ru(q[0].w), __float2half_ru(q[1].w));
    P16[pp] = make_uint4(*reinterpret_cast<const uint32_t*>(&hx), *reinterpret_cast<const uint32_t*>(&hy),
                         *reinterpret_cast<const uint32_t*>(&hz), *reinterpret_cast<const uint32_t*>(&hh));
  }
  hm = warp_max((int)hm);
  if ((threadIdx.x & 31) == 0) atomicMax(&s_hmax, hm);
  __syncthreads();
  {  // the z window table, one warp per tile cell
    const int lane = threadIdx.x & 31;
    for (int c = threadIdx.x >> 5; c < T.nct; c += nw) {
      const int s0 = S.off[c], s1 = S.off[c + 1];
      unsigned short* row = s_zw + c * kZSub;
      if (s0 == s1 && lane < kZSub) row[lane] = (unsigned short)s0;
      for (int u = s0 + lane; u < s1; u += 32) {
        const int b = zsb[u];
        const int bp = u > s0 ? (int)zsb[u - 1] : -1;
        for (int k = bp + 1; k <= b; ++k) row[k] = (unsigned short)u;
        if (u == s1 - 1)
          for (int k = b + 1; k < kZSub; ++k) row[k] = (unsigned short)s1;
      }
    }
    if (threadIdx.x == 0) s_zw[T.nct * kZSub] = (unsigned short)S.off[T.nct];
  }
  int ncolI = 0;
#pragma unroll
  for (int r = 0; r < kMaxICols; ++r) ncolI += (r == 0 || S.tc[r] != 0) ? 1 : 0;
  const int nicell = (T.nzt - 2) * ncolI;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < nicell; ++e) {
      // column-major: a warp's 32 particles share a column (coherent candidate windows)
      const int k = e / (T.nzt - 2), zz = e - k * (T.nzt - 2) + 1;
      const int c = S.tc[k] * T.nzt + zz;
      s_cp[e] = acc;
      s_ct[e] = S.off[c];
      s_cg[e] = S.gst[c];
      acc += S.off[c + 1] - S.off[c];
    }
    s_cp[nicell] = acc;
  }
  __syncthreads();
  // window half-width: the largest list radius of any pair in the tile, plus the z-order
  // bucket and the coordinate rounding bound
  const float zpad = Hfac * __uint_as_float(s_hmax) + g.zbucket + g.eabs + 2.f * g.lpad * g.side_min;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t sP = (uint32_t)__cvta_generic_to_shared(P);
  const float sub_scale = (float)kZSub / g.side[2];
  auto zbound = [&](int cz) {  // tile-relative z of the lower boundary of grid cell cz (may wrap)
    const int c = cz < 0 ? cz + g.nz : cz;
    const uint32_t b = (uint32_t)((((unsigned long long)c) << 32) / (unsigned long long)g.nz);
    return (float)(int)(b - T.ref[2]) * g.scale[2];
  };
  // kListRows x 32-lane uint16 ring per warp after the pair array (row stride 64 bytes):
  // entries leave 8 at a time from 512-byte aligned ring positions, nothing is moved
  const uint32_t buf = sP + (uint32_t)(warp * kListRows * 32 + lane) * 2u;
  int* grp = reinterpret_cast<int*>(ring0 + (size_t)nw * kListRows * 32 * 2);
  int* grpF = grp + (g.icap + 1);  // force-part groups
  constexpr uint32_t kRing = kListRows * 64u;
  const int ni = s_cp[nicell];
  int over = 0;
  // slots of the slab's ghost planes (several ranks): the tile's x-columns outside the owned
  // planes, [0, gLo) and [gHi, ...)
  int gLo = 0, gHi = 0x7fffffff;
  if (!g.periodic_x) {
    const int colx = (g.by + 2) * T.nzt;  // tile cells per tile x-column
    if (T.ix0 == g.ix_first) gLo = S.off[colx];
    const int xr = g.ix_first + g.nxo - T.ix0 + 1;  // first tile x-column past the owned planes
    if (xr <= g.bx + 1) gHi = S.off[xr * colx];
  }
  for (int c = warp; c * 32 < ni; c += nw) {
    const int k = c * 32 + lane;
    bool valid = k < ni;
    const int kk = valid ? k : c * 32;
    int lo = 0, hi = nicell;  // s_cp[lo] <= kk < s_cp[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_cp[mid] <= kk) lo = mid; else hi = mid;
    }
    const int col = lo / (T.nzt - 2), zz = lo - col * (T.nzt - 2) + 1;
    const int ti = s_ct[lo] + (kk - s_cp[lo]);
    const int gi = s_cg[lo] + (kk - s_cp[lo]);
    const __half* pi = reinterpret_cast<const __half*>(P16 + (ti >> 1)) + (ti & 1);
    const __half2 nX = __half2half2(__hneg(pi[0])), nY = __half2half2(__hneg(pi[2])),
                  nZ = __half2half2(__hneg(pi[4])), Hi2 = __half2half2(pi[6]);
    const float zi = __half2float(pi[4]) * g.side_min;  // (length units, for the z windows)
    const int tc = S.tc[col];
    const float zc = zbound(T.z0 + zz - 2);  // bottom of tile cell zz - 1
    // (kTag: k_bank lays the tagged list out; else the list leaves in its final layout)
    uint4* dst = reinterpret_cast<uint4*>((kTag ? s.nbr_raw : s.nbr) + (size_t)gi * g.lcap);
    if (valid && kWide && s.wide[gi]) {  // a wide particle's list is built by k_wide_lists
      s.ncount[gi] = 0;
      valid = false;
    }
    int mygrp = 0, mygrpF = 0;  // list groups of this lane's particle, all / force part (0: none / wide)
    uint32_t w = 0u, rd = 0u;  // ring byte offsets: next write, next flush
    int flushed = 0;           // entries already in global memory
    uint32_t nF2 = 0u;         // force-part entries flushed (two 16-bit halves)
    // Force part (bit 15, set as the entries leave the ring): each unordered pair is evaluated
    // once, by the particle whose partner has the later tile slot.  Tile columns run in the
    // order of their (x, y) cell offsets and each column in z order, so "later slot" is "the
    // partner's cell lies in the upper half of the 3x3x3 stencil (minimum-image cell offset
    // lexicographically positive), or the same cell and a later global index": the same
    // decision seen from either particle's block, whatever the periodic wraps.  A ghost partner
    // (slot outside [gLo, gHi)) is always in it: the other rank evaluates its own side.
    const uint32_t uti = (uint32_t)ti;
    auto ftag = [&](uint32_t t) -> uint32_t {
      if (!kTag) return t;
      bool f = t < (uint32_t)g.tcap && (t > uti || t < (uint32_t)gLo || t >= (uint32_t)gHi);
      if (kWide) f = f && !(wfl[t] & 1);
      return f ? 0x8000u | t : t;
    };
    auto hit = [&](bool h, int t) {
      if (h) {
        sts_u16(buf + w, (uint32_t)t);
        w = (w + 64u) & (kRing - 1u);
      }
    };
    auto test_one = [&](int t) {  // a single candidate (window ends)
      const uint4 A = P16[t >> 1];
      __half2 dx = __hadd2(*reinterpret_cast<const __half2*>(&A.x), nX);
      __half2 dy = __hadd2(*reinterpret_cast<const __half2*>(&A.y), nY);
      __half2 dz = __hadd2(*reinterpret_cast<const __half2*>(&A.z), nZ);
      __half2 r2 = __hmul2(dx, dx);
      r2 = __hfma2(dy, dy, r2);
      r2 = __hfma2(dz, dz, r2);
      const unsigned mk = __hlt2_mask(r2, __hmax2(Hi2, *reinterpret_cast<const __half2*>(&A.w)));
      hit(((mk >> (16 * (t & 1))) & 1u) != 0u, t);
    };
    auto drain = [&]() {  // buffered entries -> global memory, 8 at a time
      while (((w - rd) & (kRing - 1u)) >= 8u * 64u) {
        if (flushed + 8 <= g.lcap) {
          const uint32_t r = buf + rd;
          uint4 v;
          v.x = ftag(lds_u16(r + 0 * 64)) | (ftag(lds_u16(r + 1 * 64)) << 16);
          v.y = ftag(lds_u16(r + 2 * 64)) | (ftag(lds_u16(r + 3 * 64)) << 16);
          v.z = ftag(lds_u16(r + 4 * 64)) | (ftag(lds_u16(r + 5 * 64)) << 16);
          v.w = ftag(lds_u16(r + 6 * 64)) | (ftag(lds_u16(r + 7 * 64)) << 16);
          dst[flushed >> 3] = v;
          if (kTag)
            nF2 += ((v.x >> 15) & 0x10001u) + ((v.y >> 15) & 0x10001u) + ((v.z >> 15) & 0x10001u) +
                   ((v.w >> 15) & 0x10001u);
        }
        rd = (rd + 8u * 64u) & (kRing - 1u);
        flushed += 8;
      }
    };
    // window ends in sub-buckets above the bottom of the column's first window cell (a
    // margin of 1/100 sub-bucket covers the rounding of the tile coordinates)
    const float ulo = (zi - zpad - zc) * sub_scale - 0.01f, uhi = (zi + zpad - zc) * sub_scale + 0.01f;
    const int klo = (int)(min(max(floorf(ulo), 0.f), (float)(3 * kZSub))) & ~(int)zmask;
    const int khi = (((int)(min(max(ceilf(uhi), 0.f), (float)(3 * kZSub))) - 1) | (int)zmask) + 1;
    int c1 = 0;  // (!kTag) entries with a slot <= ti: the part outside the force loop
    // one window [a, e) of a tile column, in slot order
    auto scan = [&](int a, int e) {
      if (a >= e) return;
      if (a & 1) test_one(a++);
      if ((e - a) & 1) test_one(--e);
      drain();
      for (int p0 = a >> 1; p0 < (e >> 1); p0 += 8) {
          const int pn = min(e >> 1, p0 + 8);
#pragma unroll 4
          for (int pp = p0; pp < pn; ++pp) {
            const uint4 A = P16[pp];  // (one 16-byte load, packed half2 arithmetic: two candidates)
            const __half2 dx = __hadd2(*reinterpret_cast<const __half2*>(&A.x), nX);
            const __half2 dy = __hadd2(*reinterpret_cast<const __half2*>(&A.y), nY);
            const __half2 dz = __hadd2(*reinterpret_cast<const __half2*>(&A.z), nZ);
            __half2 r2 = __hmul2(dx, dx);
            r2 = __hfma2(dy, dy, r2);
            r2 = __hfma2(dz, dz, r2);
            const unsigned mk = __hlt2_mask(r2, __hmax2(Hi2, *reinterpret_cast<const __half2*>(&A.w)));
            hit((mk & 1u) != 0u, 2 * pp);
            hit((mk >> 16) != 0u, 2 * pp + 1);
          }
          drain();
        }
    };
    if (valid) {
#pragma unroll 1
      for (int d = 0; d < 9; ++d) {
        const int tcol = tc + (d / 3 - 1) * (g.by + 2) + (d % 3 - 1);
        const int cb = tcol * T.nzt + zz;
        // every slot of the 3 window cells with |z - zi| <= zpad lies in [a, e): the table
        // rows are the cells' sub-bucket starts, consecutive down the tile column
        const int a = s_zw[(cb - 1) * kZSub + klo];
        const int e = s_zw[(cb - 1) * kZSub + khi];
        // the columns come in slot order, so the hits do: in the own column (d = 4) the
        // window is cut after the particle's own slot and the count there taken
        if (!kTag && d == 4) {
          scan(a, min(e, ti + 1));
          // the rest of the list is the force part: close the row with sentinels
          c1 = flushed + (int)(((w - rd) & (kRing - 1u)) >> 6);
          for (int k = c1; k & 7; ++k) hit(true, g.tcap + (k & 7));
          scan(max(a, ti + 1), e);
        } else {
          scan(a, e);
        }
      }
      // pad to a multiple of 8 with sentinel slots (one per bank group, not in the force part), flush
      int nb = (int)(((w - rd) & (kRing - 1u)) >> 6);
      const int cnt = flushed + nb;
      const int cntp = (cnt + 7) & ~7;
      for (; nb < ((nb + 7) & ~7); ++nb) hit(true, g.tcap + (nb & 7));
      drain();
      const int nF = kTag ? (int)((nF2 & 0xffffu) + (nF2 >> 16)) : cnt - ((c1 + 7) & ~7);
      const int nL = kTag ? cnt - nF : c1;
      const int gF = (nF + 7) >> 3, gL = (nL + 7) >> 3;  // k_bank pads each part to rows of 8
      const int need = max(cntp, 8 * (gF + gL));
      if (need > g.lcap) over = max(over, need);
      const bool fits = need <= g.lcap;
      // bit 31: the list is already in its final layout (no k_bank pass)
      s.ncount[gi] = fits ? (nF | (nL << 16) | (kTag ? 0 : (int)0x80000000u)) : 0;
      mygrp = fits ? gF + gL : 0;
      mygrpF = fits ? gF : 0;
      // a partner at exactly i's position (j != i) is dropped: its entry becomes the
      // sentinel of its column (after the list is written, so the hot drain stays lean; only on
      // grids where k_dup found such particles, only for the particles it flagged)
      if (g.coinc && fits && s.dup[gi]) {
        uint16_t* L = (kTag ? s.nbr_raw : s.nbr) + (size_t)gi * g.lcap;
        for (int q = 0; q < cntp; ++q) {
          const uint32_t t = L[q] & 0x7fffu;
          if (t >= (uint32_t)g.tcap || t == uti || !(wfl[t] & 2)) continue;
          int gj = 0;
          for (int sq = 0; sq < nseg; ++sq) {
            const int4 sg = S.seg[sq];
            if ((int)t >= sg.x && (int)t < sg.x + sg.z) gj = sg.y + ((int)t - sg.x);
          }
          const uint4 xa = s.xh[gi], xb = s.xh[gj];
          if (xa.x == xb.x && xa.y == xb.y && xa.z == xb.z) L[q] = (uint16_t)((L[q] & 0x8000u) | (g.tcap + (q & 7)));
        }
      }
      s.hbuild[gi] = __uint_as_float(__ldg(&s.xh[gi].w));
    }
    if (k < ni) {
      grp[k] = mygrp;
      grpF[k] = mygrpF;
    }
  }
  over = warp_max(over);
  if (lane == 0 && over) atomicMax(&ctr->list_overflow, over);
  // the block's list-group prefix, in the loops' block-local particle order (column-major,
  // as here), for the loop kernels' walks (walk_prefix_pre)
  __syncthreads();
  block_exclusive_scan(grp, ni);
  block_exclusive_scan(grpF, ni);
  int* out = g.desc_pref + (size_t)ba * (g.icap + 1);
  int* outF = g.desc_prefF + (size_t)ba * (g.icap + 1);
  for (int k = threadIdx.x; k <= ni; k += blockDim.x) {
    out[k] = grp[k];
    outF[k] = grpF[k];
  }
}

// k_bank: a TAGGED list of k_lists (ghost planes or wide particles present: the force part
// is not a tail of the slot order) -> the two-part layout of nbr (sph_internal.cuh): rows
// [0, RL) the non-force part, rows [RL, RL + RF) the force part, each part in bank-aware rows
// ("Bank-aware rows" above).  One lane per list, one pass over the raw list: the t-th real
// entry of group b of part p goes straight to cell (row0_p + t, b) of the lane's grid in
// shared memory while t < R_p = ceil(n_p / 8), past that into the part's overflow queue.  The
// rows are then written out cell by cell: a grid entry where the column has one, else the
// part's next queued entry, else the column's sentinel (tcap + its bank group).  Counts are
// 4-bit fields (8 groups per 32-bit word per part).  A list of more than kCellRows rows, a
// group of more than 15 entries or more than kBankQ overflowing entries in a part takes the
// natural-order path (still split in the two parts).  Untagged lists (ncount bit 31) left
// k_lists in their final layout and are skipped.
constexpr int kBankThreads = 256;
constexpr int kBankQ = 8;  // overflow queue entries per lane and part
__global__ void __launch_bounds__(kBankThreads) k_bank(int i0, int n, DevGrid g, DevState s) {
  // cell (r, w) of thread t at kb[(8 r + w) T + t]; queue entry q of part p at kb[(8 kCellRows + p kBankQ + q) T + t]
  extern __shared__ unsigned short kb[];
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i0 + n) return;
  const int packed = s.ncount[i];
  if (packed <= 0) return;  // (final already, or no list)
  const int nF = packed & 0xffff, nL = (packed >> 16) & 0x7fff;
  const int RF = (nF + 7) >> 3, RL = (nL + 7) >> 3, Rraw = (nF + nL + 7) >> 3;
  const uint4* raw = reinterpret_cast<const uint4*>(s.nbr_raw + (size_t)i * g.lcap);
  uint4* lst = reinterpret_cast<uint4*>(s.nbr + (size_t)i * g.lcap);
  const uint32_t tcap = (uint32_t)g.tcap;
  constexpr uint32_t kStride = 2u * kBankThreads;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(kb) + 2u * threadIdx.x;
  const uint32_t qbF = base + 8u * kCellRows * kStride, qbL = qbF + kBankQ * kStride;
  auto cell = [&](uint32_t r, uint32_t w) { return base + (8u * r + w) * kStride; };
  bool grid_ok = RF + RL <= kCellRows;
  uint32_t cF = 0u, cL = 0u;  // 4-bit entry counts of the 8 groups, per part
  int qF = 0, qL = 0;         // queued entries per part
  if (grid_ok) {
    const uint32_t rf = (uint32_t)RF, rl = (uint32_t)RL;
    for (int r = 0; r < Rraw; ++r) {
      const uint4 v = __ldg(raw + r);
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t e = (wv[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        const uint32_t sl = e & 0x7fffu, b = e & 7u;
        const bool lpart = e < 0x8000u, real = sl < tcap;
        const uint32_t c = lpart ? cL : cF;
        const uint32_t tb = (c >> (4u * b)) & 15u;
        const uint32_t R = lpart ? rl : rf;
        const bool ovf = real && tb >= R;
        sts_u16_if(cell((lpart ? 0u : rl) + tb, b), sl, real && tb < R);
        const int qn = lpart ? qL : qF;
        sts_u16_if((lpart ? qbL : qbF) + (uint32_t)min(qn, kBankQ - 1) * kStride, sl, ovf);
        if (lpart) qL += ovf ? 1 : 0; else qF += ovf ? 1 : 0;
        const uint32_t inc = (real ? 1u : 0u) << (4u * b);
        if (lpart) cL += inc; else cF += inc;
      }
    }
    // (a group past 15 entries carries into the next field: the sums no longer match)
    uint32_t sF = 0u, sL = 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q) { sF += (cF >> (4 * q)) & 15u; sL += (cL >> (4 * q)) & 15u; }
    grid_ok = qF <= kBankQ && qL <= kBankQ && sF == (uint32_t)nF && sL == (uint32_t)nL;
  }
  if (grid_ok) {
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {  // p = 0: the non-force part (rows from 0), 1: the force part
      const int R = p ? RF : RL, row0 = p ? RL : 0, qn = p ? qF : qL;
      const uint32_t c = p ? cF : cL, qb = p ? qbF : qbL;
      int cw[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) cw[w] = (int)((c >> (4 * w)) & 15u);
      int q = 0;
      for (int r = 0; r < R; ++r) {
        uint32_t o[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          uint32_t hv = tcap + (((uint32_t)w - tcap) & 7u);  // the column's sentinel
          if (r < cw[w]) hv = lds_u16(cell((uint32_t)(row0 + r), (uint32_t)w));
          else if (q < qn) hv = lds_u16(qb + (uint32_t)(q++) * kStride);
          o[w] = hv;
        }
        lst[row0 + r] = make_uint4(o[0] | (o[1] << 16), o[2] | (o[3] << 16), o[4] | (o[5] << 16), o[6] | (o[7] << 16));
      }
    }
    return;
  }
  // natural order, split in the two parts (each padded with sentinels to a row of 8)
#pragma unroll 1
  for (uint32_t p = 0; p < 2; ++p) {
    int orow = p ? RL : 0, m = 0;
    uint4 buf = make_uint4(0u, 0u, 0u, 0u);
    auto put = [&](uint32_t sl) {
      const int k = m & 7;
      const uint32_t lo = (k & 1) ? 0xffffu : 0u, hi = (k & 1) ? (sl << 16) : sl;
      const int wd = k >> 1;
      if (wd == 0) buf.x = (buf.x & lo) | hi;
      else if (wd == 1) buf.y = (buf.y & lo) | hi;
      else if (wd == 2) buf.z = (buf.z & lo) | hi;
      else buf.w = (buf.w & lo) | hi;
      if (k == 7) lst[orow++] = buf;
      ++m;
    };
    for (int r = 0; r < Rraw; ++r) {
      const uint4 v = __ldg(raw + r);
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t e = (wv[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        const uint32_t sl = e & 0x7fffu;
        if (sl < tcap && (e >= 0x8000u) == (p == 1u)) put(sl);
      }
    }
    while (m & 7) put(tcap + (uint32_t)(m & 7));
  }
}

// ================================================ balanced walk over the lists ==========
// The loops below run over the block's i particles' neighbour lists cut into groups of 8
// entries (one 16-byte load each).  Instead of one lane per particle (a block holds only a
// few chunks of 32 particles, so most warps would idle while the last chunk finishes), the
// block's G list groups are split evenly over its 256 threads: thread t walks groups
// [t G / 256, (t+1) G / 256) in particle order, in one flat loop (every thread runs the same
// number of iterations up to one; only the particle switch diverges).  A particle whose
// groups lie inside one thread's range is summed by that thread alone and stored; a particle
// split across threads leaves one partial record per thread it touches (the thread's head
// record if the thread's range starts inside it, else -- the one thread whose range ends
// inside it -- the particle's own record), summed by the epilogue in thread order
// (gather_acc): no atomics, and the sums are the same every run.
constexpr int kMaxNW = 16;  // loop kernels run 256 or 512 threads (blockDim.x)
__device__ __forceinline__ int group_start(int t, int G) { return (int)(((long long)t * G) / blockDim.x); }

// In-place exclusive scan of a[0..n) by the whole block; a[n] = total.  Ends with a barrier.
__device__ void block_exclusive_scan(int* a, int n) {
  __shared__ int s_w[kMaxNW + 1];
  const int nw = blockDim.x >> 5, nt = blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int base = 0; base < n; base += nt) {
    const int k = base + threadIdx.x;
    const int v0 = k < n ? a[k] : 0;
    int v = v0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < nw; ++w) {
        const int t = s_w[w];
        s_w[w] = acc;
        acc += t;
      }
      s_w[nw] = acc;
    }
    __syncthreads();
    if (k < n) a[k] = carry + s_w[warp] + v - v0;
    carry += s_w[nw];
    __syncthreads();
  }
  if (threadIdx.x == 0) a[n] = carry;
  __syncthreads();
}

// A pair2 of two calls of a one-entry pair (the loops without packed pair arithmetic).
template <class P>
__device__ __forceinline__ auto pair2_of(P p) {
  return [=](int j0, int j1) { p(j0); p(j1); };
}

// Walk this thread's groups.  list_of(k) is particle k's list; begin(k) sets up particle k
// (i state, accumulators); pair2(j0, j1) accumulates two entries; take() returns the
// accumulators.
// finish(k, part): particle k's rows in this thread's range are done; part = 0 when they are
// all of its rows, 1 when this thread's range starts inside it (its head), 2 otherwise (tail).
template <class ListOf, class Begin, class Pair2, class Finish>
__device__ __forceinline__ void walk_rows(int ni, const int* __restrict__ pref, ListOf&& list_of, Begin&& begin,
                                          Pair2&& pair2, Finish&& finish_k) {
  const int G = pref[ni];
  if (G == 0) return;
  const int g0 = group_start(threadIdx.x, G), g1 = group_start(threadIdx.x + 1, G);
  if (g0 >= g1) return;
  int lo = 0, hi = ni;  // pref[lo] <= g0 < pref[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= g0) lo = mid; else hi = mid;
  }

  int k = lo;
  int p0 = pref[k], p1 = pref[k + 1];
  const uint4* list = reinterpret_cast<const uint4*>(list_of(k)) + (g0 - p0);
  begin(k);
  // a particle whose rows lie in this thread's range is stored whole; a split one goes to
  // this thread's head record (the particle its range starts in) or tail record (the one it
  // ends in), summed by the epilogue (gather_acc) in thread order -- no atomics
  auto finish = [&]() { finish_k(k, (g0 <= p0 && p1 <= g1) ? 0 : (k == lo ? 1 : 2)); };
  // each row is loaded one iteration ahead (its global-load latency was ~8 % of the loop
  // kernels' warp stalls when the row was used right after its load)
  uint4 enext = __ldg(list);
  for (int gg = g0; gg < g1; ++gg, ++list) {
    if (gg == p1) {
      finish();
      // next particle with a non-empty list (wide particles have none)
      do {
        ++k;
        p0 = p1;
        p1 = pref[k + 1];
      } while (p1 == p0);
      list = reinterpret_cast<const uint4*>(list_of(k));
      begin(k);
      enext = __ldg(list);
    }
    uint4 e = enext;
    if (gg + 1 < g1 && gg + 1 != p1) enext = __ldg(list + 1);
    // rotate the row so that its first entry (slot s0) is read at sub-step (lane - s0) mod 8:
    // the 8 lanes of a shared-memory phase then gather from 8 distinct 16-byte bank groups at
    // every sub-step for rows of consecutive slots (natural order) and for k_bank's rows
    // (entry w in bank group w, s0 = 0 mod 8: the rotation is the lane index); C4, against a
    // fixed rotation by the lane index: density 5.81 -> 5.73, gradient 6.60 -> 6.46, force
    // 7.24 -> 6.97 ms
    const uint32_t rot = ((uint32_t)threadIdx.x - e.x) & 7u;
    const uint32_t sh = 16u * (rot & 1u);
    if (rot & 4) { const uint32_t a = e.x, b = e.y; e.x = e.z; e.y = e.w; e.z = a; e.w = b; }
    if (rot & 2) { const uint32_t a = e.x; e.x = e.y; e.y = e.z; e.z = e.w; e.w = a; }
    {
      const uint32_t a = e.x;
      e.x = __funnelshift_r(e.x, e.y, sh);
      e.y = __funnelshift_r(e.y, e.z, sh);
      e.z = __funnelshift_r(e.z, e.w, sh);
      e.w = __funnelshift_r(e.w, a, sh);
    }
    pair2((int)(e.x & 0xffffu), (int)(e.x >> 16));
    pair2((int)(e.y & 0xffffu), (int)(e.y >> 16));
    pair2((int)(e.z & 0xffffu), (int)(e.z >> 16));
    pair2((int)(e.w & 0xffffu), (int)(e.w >> 16));
  }
  finish();
}

template <class Acc, class ListOf, class Begin, class Pair2, class Take>
__device__ __forceinline__ void walk_lists(int ni, const int* __restrict__ pref, Acc* fin, Acc* head,
                                           ListOf&& list_of, Begin&& begin, Pair2&& pair2, Take&& take) {
  walk_rows(ni, pref, list_of, begin, pair2, [&](int k, int part) {
    if (part == 1) head[threadIdx.x] = take();
    else fin[k] = take();  // (whole, or the split particle's part in the thread ending inside it)
  });
}

// Walk-area layout after a kernel's tile records (byte offset `base`, 16-aligned).
template <class Acc>
struct WalkArea {
  int* pref;  // [icap + 1]
  int* kl;    // [icap]  walk index -> block-local i index
  Acc* fin;   // [icap]  whole particles (split ones: the part of the thread whose range ends inside)
  Acc* head;  // [threads] split particle a thread's range starts in
};
#ifndef SPH_DENS_T
#define SPH_DENS_T 256
#endif
#ifndef SPH_GRAD_T
#define SPH_GRAD_T 256
#endif
constexpr int kDensT = SPH_DENS_T;  // k_density threads per CTA (3 CTAs per SM)
constexpr int kGradT = SPH_GRAD_T;  // k_gradient threads per CTA (3 CTAs per SM)
#ifndef SPH_FORCE_T
#define SPH_FORCE_T 448
#endif
constexpr int kForceT = SPH_FORCE_T;  // k_force threads per CTA when two CTAs fit an SM
template <class Acc>
__host__ __device__ __forceinline__ size_t walk_bytes(int icap, int threads = kNW * 32) {
  return (((size_t)(icap + 1) * 4 + 15) & ~(size_t)15) + (((size_t)icap * 4 + 15) & ~(size_t)15) +
         (((size_t)icap * sizeof(Acc) + 15) & ~(size_t)15) + (size_t)threads * sizeof(Acc);
}
template <class Acc>
__device__ __forceinline__ WalkArea<Acc> walk_area(char* base, int icap) {
  WalkArea<Acc> w;
  w.pref = reinterpret_cast<int*>(base);
  base += ((size_t)(icap + 1) * 4 + 15) & ~(size_t)15;
  w.kl = reinterpret_cast<int*>(base);
  base += ((size_t)icap * 4 + 15) & ~(size_t)15;
  w.fin = reinterpret_cast<Acc*>(base);
  base += ((size_t)icap * sizeof(Acc) + 15) & ~(size_t)15;
  w.head = reinterpret_cast<Acc*>(base);
  return w;
}

// Accumulators of walk particle k: its whole record, or the sum, in thread order, of the
// records of the threads its rows were split over (walk_lists).
template <class Acc>
__device__ __forceinline__ Acc gather_acc(const WalkArea<Acc>& W, int ni, int k) {
  const long long G = W.pref[ni];
  const int a = W.pref[k], b = W.pref[k + 1];
  if (b <= a) return Acc::zero();
  const long long nt = blockDim.x;
  const int ta = (int)((nt * (a + 1) - 1) / G), tb = (int)((nt * b - 1) / G);
  if (ta == tb) return W.fin[k];
  Acc s = Acc::zero();
  for (int t2 = ta; t2 <= tb; ++t2) {
    const int s0 = (int)(((long long)t2 * G) / nt), s1 = (int)(((long long)(t2 + 1) * G) / nt);
    if (s0 >= s1) continue;  // (a thread without rows)
    s.add(s0 >= a ? W.head[t2] : W.fin[k]);
  }
  return s;
}

// Fill pref[] with the list groups of the walk's particles (kl[0..ni)), scan it, and clear
// the accumulators.
// The same for a walk over all the block's particles (kl[k] = k): the prefix k_lists stored.
template <class Acc>
// Issued with cp.async before the tile staging, whose wait + barrier completes it.
__device__ __forceinline__ void walk_prefix_pre(const DevGrid& g, WalkArea<Acc>& W, int ni, bool force_part = false) {
  const int* src = (force_part ? g.desc_prefF : g.desc_pref) + (size_t)blk_a(g) * (g.icap + 1);
  for (int k = threadIdx.x; k <= ni; k += blockDim.x) cp_async4(W.pref + k, src + k);
}

template <class Acc, class SS>
__device__ __forceinline__ void walk_prefix(const SS& S, const DevState& s, WalkArea<Acc>& W, int ni) {
  const int* kl = W.kl;
  int* pref = W.pref;
  for (int k = threadIdx.x; k < ni; k += blockDim.x) {
    int ti, gi;
    i_slot(S, kl[k], ti, gi);
    const int c = __ldg(s.ncount + gi);
    pref[k] = (((c & 0xffff) + 7) >> 3) + ((((c >> 16) & 0x7fff) + 7) >> 3);
  }
  __syncthreads();
  block_exclusive_scan(pref, ni);
}

// ============================================================== density loop ==========
// Eqs. 2-6 with the Newton-Raphson h update of the ghost (R7) and the
// density finalize (Eq. 8, EoS, Balsara; R8, R14) fused into the epilogue.
// Accumulators per particle i (q = r/h_i, w = M4; the self pair is in the list: w(0) = 1):
//   S0 = sum w, S1 = sum q w', R0 = sum m_j w, R1 = sum m_j q w',
//   Dv = sum m_j w'/r (v_ij . r_ij),  Cv = sum m_j w'/r (v_ij x r_ij),  N_i.
// Then nhat = S0/(pi h^3), dn/dh = -(3 S0 + S1)/(pi h^4), rho = R0/(pi h^3),
// drho/dh = -(3 R0 + R1)/(pi h^4), div = -Dv/(rho pi h^4), curl = Cv/(rho pi h^4),
// g = nhat h^3 - eta^3 = S0/pi - eta^3, h g' = -S1/pi.
__global__ void __launch_bounds__(kDensT, 3) k_density(DevGrid g, DevPhys ph, DevState s,
                                                      const int* __restrict__ cell_start, int pass,
                                                      const uint8_t* __restrict__ blk_in, uint8_t* __restrict__ blk_out,
                                                      float hfac_stale, DevCounters* __restrict__ ctr) {
  if (pass > 0 && !blk_in[blk_a(g)]) return;
  __shared__ int s_ni;
  __shared__ unsigned long long s_pairs, s_final;
  __shared__ int s_unconv, s_active;
  __shared__ unsigned int s_rmax;
  if (threadIdx.x == 0) { s_ni = 0; s_pairs = 0; s_final = 0; s_unconv = 0; s_active = 0; s_rmax = 0u; }
  DESC_PROLOGUE();
  const int O1 = SP;  // T0 = smem4[j]: x, y, z, h   T1 = smem4[O1 + j]: vx, vy, vz, m
  WalkArea<DenAcc> W = walk_area<DenAcc>(reinterpret_cast<char*>(smem4 + 2 * SP), g.icap);
  if (pass == 0) walk_prefix_pre(g, W, T.ni);
  {
    const float4* src[2] = {reinterpret_cast<const float4*>(s.xh), s.vm};
    const int o16[2] = {0, O1};
    stage_records<2>(S, nseg, src, o16, T.ntile);
  }
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    const uint4 x = reinterpret_cast<const uint4*>(smem4)[t];
    const float3 p = rel_pos(g, T, x);
    smem4[t] = make_float4(p.x, p.y, p.z, __uint_as_float(x.w));
  }
  if (threadIdx.x < kNSent) {
    smem4[g.tcap + threadIdx.x] = make_float4(kFar, kFar, kFar, 1.f);
    smem4[O1 + g.tcap + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // the walk's particles: all of the block (pass 0) or the still active ones, compacted in
  // block order (deterministic)
  if (pass == 0) {
    for (int k = threadIdx.x; k < T.ni; k += blockDim.x) W.kl[k] = k;
    if (threadIdx.x == 0) s_ni = T.ni;
  } else {
    for (int k = threadIdx.x; k < T.ni; k += blockDim.x) {
      int ti, gi;
      i_slot(S, k, ti, gi);
      W.pref[k] = s.active[gi] ? 1 : 0;
    }
    __syncthreads();
    block_exclusive_scan(W.pref, T.ni);
    for (int k = threadIdx.x; k < T.ni; k += blockDim.x)
      if (W.pref[k + 1] > W.pref[k]) W.kl[W.pref[k]] = k;
    if (threadIdx.x == 0) s_ni = W.pref[T.ni];
  }
  __syncthreads();
  int ni = s_ni;
  if (pass > 0) walk_prefix(S, s, W, ni);
  // Newton iterations inside the CTA (h iteration, R7): a particle's density sums depend
  // only on the positions and its own h (gather, W(r_ij, h_i)), so while its new h stays within
  // its list radius and the cell, the next iteration walks its list again over the tile still in
  // shared memory.  Only the particles that outgrow their list or cell (or reach DevGrid::dens_inner
  // iterations here) are left active for another pass of the host loop (sph_density).
  unsigned long long npairs = 0, nfinal = 0;
  float rmax = 0.f;  // largest closure residual of the particles finished here
  for (int it = 0;; ++it) {
    {
      float4 pi4, vi4;
      float hinv = 0.f, qband = 0.f;
      double H2 = 0.0;
      int gi = 0;
      DenAcc a;
      const uint32_t sb0 = smem_base(0), sb1 = smem_base(O1);
      int ti_c = 0;  // tile slot of the walk's current particle (list_of -> begin)
      walk_lists(
          ni, W.pref, W.fin, W.head,
          [&](int k) {  // (list_of runs right before begin: the slot lookup is shared)
            i_slot(S, W.kl[k], ti_c, gi);
            return s.nbr + (size_t)gi * g.lcap;
          },
          [&](int) {
            const int ti = ti_c;
            pi4 = smem4[ti];
            vi4 = smem4[O1 + ti];
            hinv = 1.f / pi4.w;
            qband = g.eabs * hinv + 8e-6f;  // |q - 2| below this: decide in fp64
            H2 = h2_exact(pi4.w, ph.gamma_k);
            a = DenAcc{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0};
          },
          pair2_of([&](int j) {
            const uint32_t o = (uint32_t)j << 4;
            const float4 p = lds4(sb0 + o);
            den_pair(a, pi4.x - p.x, pi4.y - p.y, pi4.z - p.z, hinv, qband, vi4, lds4(sb1 + o), [&]() {
              return exact_neighbour(s.xh, gi, slot_global(S, nseg, j), H2, g.dscale[0], g.dscale[1], g.dscale[2]);
            });
          }),
          [&]() { return a; });
    }
    __syncthreads();
    // (the continue flags stay in a register mask until every thread's epilogue has read the walk
    // area -- gather_acc reads W.pref -- then go to W.pref for the compaction)
    const bool more = it + 1 < g.dens_inner && ni <= 32 * (int)blockDim.x;
    uint32_t cmask = 0u;
    for (int k = threadIdx.x, q = 0; k < ni; k += blockDim.x, ++q) {
      const DenAcc a = gather_acc(W, ni, k);
      int ti, gi;
      const int kl = W.kl[k];
      i_slot(S, kl, ti, gi);
      bool cont = false;
      if (!(s.wide && s.wide[gi])) {  // wide particles: k_wide_density
        const DenOut o = den_epilogue(g, ph, s, a, gi, smem4[ti].w, smem4[O1 + ti].w, pass + it, hfac_stale);
        npairs += (unsigned long long)o.nn;
        if (o.final_) nfinal += (unsigned long long)o.nn;
        if (o.final_) rmax = fmaxf(rmax, o.resid);
        if (o.give_up) atomicAdd(&s_unconv, 1);
        if (o.exceeds) atomicExch(&ctr->h_exceeds, 1);
        if (o.stale) atomicExch(&ctr->list_stale, 1);
        cont = o.active && !o.exceeds && !o.stale && more;
        if (o.active && !cont) s_active = 1;
        if (cont) smem4[ti].w = o.hn;
      }
      if (cont) cmask |= 1u << q;
    }
    __syncthreads();
    for (int k = threadIdx.x, q = 0; k < ni; k += blockDim.x, ++q) W.pref[k] = (int)((cmask >> q) & 1u);
    __syncthreads();
    // the particles that keep iterating, compacted in block order (deterministic), through the
    // walk's record area (consumed by the epilogue above)
    block_exclusive_scan(W.pref, ni);
    const int nnext = W.pref[ni];
    if (nnext == 0) break;
    int* tmp = reinterpret_cast<int*>(W.fin);
    for (int k = threadIdx.x; k < ni; k += blockDim.x)
      if (W.pref[k + 1] > W.pref[k]) tmp[W.pref[k]] = W.kl[k];
    __syncthreads();
    for (int k = threadIdx.x; k < nnext; k += blockDim.x) W.kl[k] = tmp[k];
    __syncthreads();
    ni = nnext;
    walk_prefix(S, s, W, ni);
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    npairs += __shfl_xor_sync(kFull, npairs, o);
    nfinal += __shfl_xor_sync(kFull, nfinal, o);
  }
  rmax = __int_as_float(warp_max(__float_as_int(rmax)));  // (non-negative: int order)
  if (lane == 0) {
    if (npairs) atomicAdd(&s_pairs, npairs);
    if (nfinal) atomicAdd(&s_final, nfinal);
    if (rmax > 0.f) atomicMax(&s_rmax, __float_as_uint(rmax));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_rmax) atomicMax(&ctr->max_resid_bits, s_rmax);
    if (s_pairs) atomicAdd(&ctr->pairs_all, s_pairs);  // all pairs of this pass (h iteration work)
    if (s_final) atomicAdd(&ctr->pairs, s_final);
    if (s_unconv) atomicAdd(&ctr->unconverged, s_unconv);
    if (s_active) { blk_out[ba] = 1; atomicAdd(&ctr->active_next, 1); }
  }
}

// ============================================================= gradient loop ==========
// v_sig,i = max(2 c_i, max_j (c_i + c_j - beta mu_ij)) (Eqs. 10-11, R15) and the
// Brookshaw Laplacian lap u_i = 2 sum_j (m_j/rho_j)(u_i - u_j) dW/dr / r (R16), gathered
// over r_ij < H_i; the gradient ghost (alpha_v Eqs. 12-15, alpha_c Eqs. 21-24; R17-R21)
// runs in the epilogue and writes the force-loop records.
// the gradient tile's (u, m/rho) array, 16-byte aligned
__host__ __device__ __forceinline__ size_t gradient_t2_bytes(const DevGrid& g) {
  return (((size_t)(g.tcap + kNSent) * 8) + 15) & ~(size_t)15;
}
__global__ void __launch_bounds__(kGradT, 3) k_gradient(DevGrid g, DevPhys ph, DevState s,
                                                       const int* __restrict__ cell_start, float dt, int first_step,
                                                       DevCounters* __restrict__ ctr) {
  __shared__ unsigned long long s_pairs;
  __shared__ unsigned int s_hinv_max;  // largest 1/h of the tile (f32 bits)
  if (threadIdx.x == 0) { s_pairs = 0; s_hinv_max = 0u; }
  DESC_PROLOGUE();
  // T0 = smem4[j]: x, y, z, 1/h   T1 = smem4[O1 + j]: vx, vy, vz, c (the density loop's vc record)
  // T2 = float2 [j]: u, m/rho (um): a pair gathers 16 + 16 + 8 bytes
  const int O1 = SP;
  float2* T2 = reinterpret_cast<float2*>(smem4 + 2 * SP);
  WalkArea<GradAcc> W = walk_area<GradAcc>(reinterpret_cast<char*>(T2) + gradient_t2_bytes(g), g.icap);
  walk_prefix_pre(g, W, T.ni);
  {
    // (the 8-byte records with cp.async, completed by the staging's wait + barrier)
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int k = threadIdx.x >> 5; k < nseg; k += nw) {
      const int4 sg = S.seg[k];
      for (int t = lane; t < sg.z; t += 32) cp_async8(T2 + sg.x + t, s.um + sg.y + t);
    }
    const float4* src[2] = {reinterpret_cast<const float4*>(s.xh), s.vc};
    const int o16[2] = {0, O1};
    stage_records<2>(S, nseg, src, o16, T.ntile);
  }
  {
    unsigned int hm = 0u;
    for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
      const uint4 x = reinterpret_cast<const uint4*>(smem4)[t];
      const float3 p = rel_pos(g, T, x);
      const float hinv = 1.f / __uint_as_float(x.w);
      smem4[t] = make_float4(p.x, p.y, p.z, hinv);
      hm = max(hm, __float_as_uint(hinv));
    }
    hm = (unsigned int)warp_max((int)hm);
    if ((threadIdx.x & 31) == 0 && hm) atomicMax(&s_hinv_max, hm);
  }
  if (threadIdx.x < kNSent) {
    smem4[g.tcap + threadIdx.x] = make_float4(kFar, kFar, kFar, 1.f);
    smem4[O1 + g.tcap + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    T2[g.tcap + threadIdx.x] = make_float2(0.f, 0.f);
  }
  const int ni = T.ni;
  for (int k = threadIdx.x; k < ni; k += blockDim.x) W.kl[k] = k;
  __syncthreads();
  {
    float4 pi4, vi4;
    float hinv = 0.f, qband = 0.f, ci = 0.f, ui = 0.f;
    // |min(q_i, q_j) - 2| below this: decide the symmetric set in fp64 (eabs / min h of the tile)
    const float sband = g.eabs * __uint_as_float(s_hinv_max) + 8e-6f;
    double H2 = 0.0;
    int gi = 0;
    GradAcc a;
    const uint32_t sb0 = smem_base(0), sb1 = smem_base(O1), sb2 = smem_base(2 * SP);
    int ti_c = 0;  // tile slot of the walk's current particle (list_of -> begin)
    walk_lists(
        ni, W.pref, W.fin, W.head,
        [&](int k) {  // (list_of runs right before begin: the slot lookup is shared)
          i_slot(S, W.kl[k], ti_c, gi);
          return s.nbr + (size_t)gi * g.lcap;
        },
        [&](int) {
          const int ti = ti_c;
          pi4 = smem4[ti];
          vi4 = smem4[O1 + ti];
          hinv = pi4.w;
          qband = g.eabs * hinv + 8e-6f;
          H2 = h2_exact(__uint_as_float(__ldg(&s.xh[gi].w)), ph.gamma_k);  // (the exact h: fp64 edge test)
          ci = vi4.w;
          ui = T2[ti].x;
          a = GradAcc{2.f * ci, 0.f, 0, 2.f * ci};
        },
        pair2_of([&](int j) {
          const uint32_t o = (uint32_t)j << 4;
          const float4 p = lds4(sb0 + o);
          const float4 vj = lds4(sb1 + o);
          const float2 uj = lds2(sb2 + ((uint32_t)j << 3));
          grad_pair_sym(
              a, pi4.x - p.x, pi4.y - p.y, pi4.z - p.z, hinv, p.w, qband, sband, vi4, ci, ui, ph.beta, vj,
              make_float4(vj.w, uj.x, uj.y, 0.f),
              [&]() {
                return exact_neighbour(s.xh, gi, slot_global(S, nseg, j), H2, g.dscale[0], g.dscale[1], g.dscale[2]);
              },
              [&]() {
                const int gj = slot_global(S, nseg, j);
                return exact_neighbour(s.xh, gi, gj, fmax(H2, h2_exact(__uint_as_float(s.xh[gj].w), ph.gamma_k)),
                                       g.dscale[0], g.dscale[1], g.dscale[2]);
              });
        }),
        [&]() { return a; });
  }
  __syncthreads();
  unsigned long long npairs = 0;
  for (int k = threadIdx.x; k < ni; k += blockDim.x) {
    const GradAcc a = gather_acc(W, ni, k);
    int ti, gi;
    i_slot(S, k, ti, gi);
    if (s.wide && s.wide[gi]) continue;  // wide particles: k_wide_gradient, k_wide_force
    npairs += (unsigned long long)grad_epilogue(ph, s, a, gi, __uint_as_float(s.xh[gi].w), smem4[O1 + ti].w,
                                                T2[ti].x, s.gq[gi].w, dt, first_step);
    // the force loop's v_sig and N_force (symmetric set; a wide partner that did not list this
    // particle adds its pair in k_wide_force)
    s.vsig[gi] = a.vmaxs;
    s.countf[gi] = (a.nn >> 16) - 1;  // (the self pair)
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) npairs += __shfl_xor_sync(kFull, npairs, o);
  if (lane == 0 && npairs) atomicAdd(&s_pairs, npairs);
  __syncthreads();
  if (threadIdx.x == 0 && s_pairs) atomicAdd(&ctr->pairs, s_pairs);
}

// ================================================================ force loop ==========
// Pair-once form of the pairwise sums of Eqs. 7, 17-19 over r_ij < max(H_i, H_j) (R3): each
// unordered pair is evaluated ONCE, by the particle whose list holds it in its force part
// (k_lists: partner in the upper half of the cell stencil), and applied to both particles with
// opposite signs (force_pair2): the i side accumulates in registers and is added to acc[i]
// when the thread's rows of i end, the j side is added to acc[j] with one vector reduction
// (red.global.add.v4.f32) per pair that has a term.  acc is zeroed before the launch; the CFL
// dt and the finiteness check run over the finished sums in k_force_fin.  v_sig and N_force
// of the symmetric set were taken by the gradient loop.
__host__ __device__ __forceinline__ size_t force_records_bytes(int tcap) {
  const size_t sp = (size_t)tcap + kNSent;
  return sp * (4 * 16) + ((sp + 3) & ~(size_t)3) * 4;  // four records + the slot's global index
}

// (no "memory" clobber: the reductions target global memory the kernel never reads, so the
// shared-memory gathers of the next pair may be scheduled across them)
__device__ __forceinline__ void red_add4(float4* p, const float4& v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}
// the same under a predicate (no branch around it in the pair loop)
__device__ __forceinline__ void red_add4_if(float4* p, const float4& v, bool on) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %5, 0; @q red.global.add.v4.f32 [%0], {%1, %2, %3, %4}; }" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((uint32_t)on));
}
__device__ __forceinline__ int lds1(uint32_t a) {
  int v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// (NT threads, MINB CTAs per SM: 448 x 2 when two tiles fit an SM -- 28 warps to hide the
// gather latency, registers <= 73; C4 force: 256 x 2 7.29, 384 x 2 7.32, 448 x 2 7.07, 512 x 2 7.27 ms
// (spills) --, else 512 x 1)
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_force(DevGrid g, DevPhys ph, DevState s,
                                                    const int* __restrict__ cell_start,
                                                    DevCounters* __restrict__ ctr) {
  DESC_PROLOGUE();
  // T0 = [j]: x, y, z, 1/h   T1 = [O1+j]: vx, vy, vz, m   T2 = [O2+j]: A, Kf, c, rho
  // T3 = [O3+j]: B, (P + kPeps) alpha_c, u, alpha_v  (P = A rho^2)   GI[j]: global index of slot j
  const int O1 = SP, O2 = 2 * SP, O3 = 3 * SP;
  int* GI = reinterpret_cast<int*>(smem4 + 4 * SP);
  int* pref = GI + ((SP + 3) & ~3);  // [icap + 1] force-part group prefix (k_lists)
  int* prefA = pref + (g.icap + 1);  // [icap + 1] whole-list group prefix
  {
    const int* src = g.desc_prefF + (size_t)ba * (g.icap + 1);
    const int* srcA = g.desc_pref + (size_t)ba * (g.icap + 1);
    for (int k = threadIdx.x; k <= T.ni; k += blockDim.x) {
      cp_async4(pref + k, src + k);
      cp_async4(prefA + k, srcA + k);
    }
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int k = threadIdx.x >> 5; k < nseg; k += nw) {
      const int4 sg = S.seg[k];
      for (int t = lane; t < sg.z; t += 32) GI[sg.x + t] = sg.y + t;
    }
    if (threadIdx.x < kNSent) GI[g.tcap + threadIdx.x] = 0;  // (sentinels: never a term)
  }
  {
    const float4* src[4] = {reinterpret_cast<const float4*>(s.xh), s.vm, s.fr1, s.fr2};
    const int o16[4] = {0, O1, O2, O3};
    stage_records<4>(S, nseg, src, o16, T.ntile);
  }
  for (int t = threadIdx.x; t < T.ntile; t += blockDim.x) {
    const uint4 x = reinterpret_cast<const uint4*>(smem4)[t];
    const float3 p = rel_pos(g, T, x);
    smem4[t] = make_float4(p.x, p.y, p.z, 1.f / __uint_as_float(x.w));
  }
  if (threadIdx.x < kNSent) {
    smem4[g.tcap + threadIdx.x] = make_float4(kFar, kFar, kFar, 1.f);
    smem4[O1 + g.tcap + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    smem4[O2 + g.tcap + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 1.f);
    smem4[O3 + g.tcap + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const float4* __restrict__ T0 = smem4;
  const float4* __restrict__ T1 = smem4 + O1;
  const float4* __restrict__ T2 = smem4 + O2;
  const float4* __restrict__ T3 = smem4 + O3;
  float4 pi4;
  ForceSide I;
  int gi = 0;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t sb0 = smem_base(0), sb1 = smem_base(O1), sb2 = smem_base(O2), sb3 = smem_base(O3);
  const uint32_t sbg = smem_base(4 * SP);
  int ti_c = 0;  // tile slot of the walk's current particle (list_of -> begin)
  walk_rows(
      T.ni, pref,
      [&](int k) {  // (list_of runs right before begin: the slot lookup is shared)
        i_slot(S, k, ti_c, gi);
        // the force part follows the RL rows of the rest of the list
        const int RL = (prefA[k + 1] - prefA[k]) - (pref[k + 1] - pref[k]);
        return s.nbr + (size_t)gi * g.lcap + 8 * RL;
      },
      [&](int) {
        const int ti = ti_c;
        pi4 = T0[ti];
        I.hinv = pi4.w;
        I.v = T1[ti];
        I.a = T2[ti];
        I.b = T3[ti];
        I.P = I.a.x * I.a.w * I.a.w;
        a = make_float4(0.f, 0.f, 0.f, 0.f);
      },
      // (one entry at a time: a packed f32x2 version over two entries, force_pair2 with
      // FFMA2 / FMUL2, ran 17 % fewer loop instructions but needs 128 registers -- 256 x 2
      // threads per SM: 7.60 ms against 7.06 on C4; the loop is latency-bound, not issue-bound)
      pair2_of([&](int j) {
        const uint32_t o = (uint32_t)j << 4;
        const float4 p = lds4(sb0 + o);
        ForceSide J;
        J.hinv = p.w;
        J.v = lds4(sb1 + o);
        J.a = lds4(sb2 + o);
        J.b = lds4(sb3 + o);
        J.P = J.a.x * J.a.w * J.a.w;
        float4 jo;
        const bool term = force_pair2(a, jo, pi4.x - p.x, pi4.y - p.y, pi4.z - p.z, I, J, ph.beta);
        red_add4_if(s.acc + lds1(sbg + ((uint32_t)j << 2)), jo, term);
      }),
      [&](int, int) { red_add4(s.acc + gi, a); });
}

// After k_force (and the wide particles' k_wide_force): the CFL dt = C_cfl min 2 gamma_k h / v_sig
// (S:261), the finiteness check of a, du/dt and v_sig, and sum N_force.
__global__ void __launch_bounds__(256) k_force_fin(int i0, int n, DevPhys ph, DevState s,
                                                   DevCounters* __restrict__ ctr) {
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  float dtmin = CUDART_INF_F;
  unsigned long long npairs = 0;
  bool bad = false;
  if (i < i0 + n) {
    const float h = __uint_as_float(s.xh[i].w);
    const float vs = s.vsig[i];
    const float4 a = s.acc[i];
    const float dti = ph.c_cfl * 2.f * ph.gamma_k * h / vs;
    bad = !(isfinite(vs) && isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w)) || !(dti > 0.f);
    dtmin = dti > 0.f ? dti : CUDART_INF_F;
    npairs = (unsigned long long)max(s.countf[i], 0);
  }
  __shared__ unsigned long long s_pairs;
  __shared__ unsigned int s_dt;
  __shared__ int s_bad;
  if (threadIdx.x == 0) { s_pairs = 0; s_dt = 0x7f800000u; s_bad = 0; }
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    npairs += __shfl_xor_sync(kFull, npairs, o);
    dtmin = fminf(dtmin, __shfl_xor_sync(kFull, dtmin, o));
  }
  if (bad) s_bad = 1;
  if ((threadIdx.x & 31) == 0) {
    if (npairs) atomicAdd(&s_pairs, npairs);
    if (dtmin < CUDART_INF_F) atomicMin(&s_dt, __float_as_uint(dtmin));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_pairs) atomicAdd(&ctr->pairs, s_pairs);
    if (s_dt != 0x7f800000u) atomicMin(&ctr->dt_bits, s_dt);
    if (s_bad) atomicExch(&ctr->nonfinite, 1);
  }
}

// One CTA per block: tile_setup, then the descriptor out (k_tile_desc, once per rebuild).
__global__ void __launch_bounds__(64) k_tile_desc(DevGrid g, const int* __restrict__ cell_start) {
  __shared__ BlockShared S;
  Tile T;
  const int a = blk_a(g);  // (the blocks the loops run: run_list, else every active block)
  tile_setup(g, g.blk_list[a], cell_start, S, T);
  TileDesc* D = reinterpret_cast<TileDesc*>(const_cast<void*>(g.desc)) + a;
  if (threadIdx.x == 0) D->T = T;
  if (threadIdx.x < kMaxICols) {
    D->ib[threadIdx.x] = S.ib[threadIdx.x];
    D->g0[threadIdx.x] = S.g0[threadIdx.x];
    D->tc[threadIdx.x] = S.tc[threadIdx.x];
  }
  if (threadIdx.x <= kMaxICols) D->pre[threadIdx.x] = S.pre[threadIdx.x];
  if (threadIdx.x < kMaxSeg) D->seg[threadIdx.x] = S.seg[threadIdx.x];
  // per tile cell (tile offset, global start) for k_lists' window searches
  int2* C = reinterpret_cast<int2*>(const_cast<void*>(g.desc_cells)) + (size_t)a * (kMaxTileCells + 1);
  for (int c = threadIdx.x; c <= T.nct; c += blockDim.x) C[c] = make_int2(S.off[c], c < T.nct ? S.gst[c] : 0);
}

// The i columns of every active block (TileDesc::pre, g0, tc), one thread per block: all that
// k_sparse_wide and k_block_run read; the full descriptors (k_tile_desc) are then made for the
// blocks the loops run only (on a clustered box a few thousand of ~0.9 M active blocks).
__global__ void k_tile_icols(DevGrid g, const int* __restrict__ cell_start) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= g.nact) return;
  int jx, jy, zb;
  block_coords(g, g.blk_list[a], jx, jy, zb);
  const int ix0 = g.ix_first + jx * g.bx, iy0 = jy * g.by, z0 = zb * g.KZ, z1 = min(g.nz, z0 + g.KZ);
  TileDesc* D = reinterpret_cast<TileDesc*>(const_cast<void*>(g.desc)) + a;
  int k = 0, acc = 0;
  for (int ex = 0; ex < g.bx; ++ex)
    for (int ey = 0; ey < g.by; ++ey) {
      if (ix0 + ex >= g.ix_first + g.nxo || iy0 + ey >= g.ny) continue;
      const int col = ((ix0 + ex) * g.ny + (iy0 + ey)) * g.nz;  // an i column's cells are consecutive
      const int s0 = __ldg(cell_start + col + z0), s1 = __ldg(cell_start + col + z1);
      D->tc[k] = (ex + 1) * (g.by + 2) + (ey + 1);
      D->g0[k] = s0;
      D->pre[k] = acc;
      acc += s1 - s0;
      ++k;
    }
  D->pre[k] = acc;
  for (int r = k; r < kMaxICols; ++r) { D->tc[r] = 0; D->g0[r] = 0; D->pre[r + 1] = acc; }
}

// tile size and i count of block b
__device__ void block_counts(const DevGrid& g, const int* __restrict__ cell_start, int b, int& tot_out, int& ni_out) {
  int jx, jy, zb;
  block_coords(g, b, jx, jy, zb);
  const int ix0 = g.ix_first + jx * g.bx, iy0 = jy * g.by;
  const int z0 = zb * g.KZ, z1 = min(g.nz, z0 + g.KZ);
  int tot = 0, ni = 0;
  for (int dx = -1; dx <= g.bx; ++dx)
    for (int dy = -1; dy <= g.by; ++dy) {
      if (!g.periodic_x && ix0 + dx >= g.nx) continue;
      const int cx = (ix0 + dx + g.nx) % g.nx, cy = (iy0 + dy + g.ny) % g.ny;
      const int c0 = (cx * g.ny + cy) * g.nz;
      const bool own = dx >= 0 && dx < g.bx && dy >= 0 && dy < g.by && ix0 + dx < g.ix_first + g.nxo &&
                       iy0 + dy < g.ny;
      for (int z = z0 - 1; z <= z1; ++z) {
        const int cz = (z + g.nz) % g.nz;
        const int c = cell_start[c0 + cz + 1] - cell_start[c0 + cz];
        tot += c;
        if (own && z >= z0 && z < z1) ni += c;
      }
    }
  tot_out = tot;
  ni_out = ni;
}

// per-block tile size and i count (max over blocks) -> sizes shared memory of the loops
// (and, with `flag`, which blocks have i particles: the active-block flags of this grid)
__global__ void k_tile_sizes(DevGrid g, const int* __restrict__ cell_start, int* max_tile, int* max_i,
                             uint8_t* flag) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nblocks) return;
  int tot, ni;
  block_counts(g, cell_start, b, tot, ni);
  if (flag) flag[b] = ni > 0 ? 1 : 0;
  if (tot) atomicMax(max_tile, tot);
  if (ni) atomicMax(max_i, ni);
}

// Block id of grid column (jx, jy), z block zb: the inverse of block_coords.
__device__ __forceinline__ int block_of(const DevGrid& g, int jx, int jy, int zb) {
  const int sgm = jy / kStrip;
  const int hs = min(kStrip, g.nby - sgm * kStrip);
  const int c = sgm * kStrip * g.nbx + jx * hs + (jy - sgm * kStrip);
  return c * g.nzb + zb;
}

// Flag the blocks holding an owned particle (cell ids from the sorted keys, cell << zbits): the
// active blocks without a pass over every block of the grid (a clustered box's fine grid has
// ~70x more blocks than occupied ones).  flag must be zero before the launch.
__global__ void k_block_flags(int n, const unsigned int* __restrict__ keys, DevGrid g, uint8_t* flag) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const unsigned int cell = keys[p] >> g.zbits;
  if (p > 0 && (keys[p - 1] >> g.zbits) == cell) return;  // (one thread per occupied cell)
  if ((int)cell >= g.ncells) return;
  const int cz = (int)(cell % (unsigned)g.nz);
  const int cxy = (int)(cell / (unsigned)g.nz);
  const int cy = cxy % g.ny, cx = cxy / g.ny;
  if (cx < g.ix_first || cx >= g.ix_first + g.nxo) return;
  flag[block_of(g, (cx - g.ix_first) / g.bx, cy / g.by, cz / g.KZ)] = 1;
}

// tile size and i count (max over the listed blocks), grid-stride over the device-side count
__global__ void k_tile_sizes_list(DevGrid g, const int* __restrict__ cell_start, const int* __restrict__ list,
                                  const int* __restrict__ nlist, int* max_tile, int* max_i) {
  const int n = *nlist;
  int mt = 0, mi = 0;
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
    int tot, ni;
    block_counts(g, cell_start, list[a], tot, ni);
    mt = max(mt, tot);
    mi = max(mi, ni);
  }
  mt = warp_max(mt);
  mi = warp_max(mi);
  if ((threadIdx.x & 31) == 0) {
    if (mt) atomicMax(max_tile, mt);
    if (mi) atomicMax(max_i, mi);
  }
}

// Sparse blocks (adaptive grid): a block with fewer than kmin tile (non-wide) i particles pays a
// whole tile staging for them; its particles are handled as wide instead (global-index lists, one
// warp each), cheaper per particle on a clustered box's mostly empty fine grid.
__global__ void k_sparse_wide(DevGrid g, uint8_t* wide, int32_t* ncount, int kmin) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= g.nact) return;
  const TileDesc* D = reinterpret_cast<const TileDesc*>(g.desc) + a;
  int cnt = 0;
  for (int r = 0; r < kMaxICols; ++r) {
    const int c = D->pre[r + 1] - D->pre[r], g0 = D->g0[r];
    for (int k = 0; k < c; ++k)
      if (!wide[g0 + k] && ++cnt >= kmin) return;
  }
  if (cnt == 0) return;
  for (int r = 0; r < kMaxICols; ++r) {
    const int c = D->pre[r + 1] - D->pre[r], g0 = D->g0[r];
    for (int k = 0; k < c; ++k)
      if (!wide[g0 + k]) {
        wide[g0 + k] = 1;
        ncount[g0 + k] = 0;  // (no tile list)
      }
  }
}

// active blocks with a non-wide i particle (the loop kernels run only these)
__global__ void k_block_run(DevGrid g, DevState s, uint8_t* flag) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= g.nact) return;
  const TileDesc* D = reinterpret_cast<const TileDesc*>(g.desc) + a;
  int run = 0;
  for (int r = 0; r < kMaxICols && !run; ++r) {
    const int c = D->pre[r + 1] - D->pre[r], g0 = D->g0[r];
    for (int k = 0; k < c; ++k)
      if (!s.wide[g0 + k]) { run = 1; break; }
  }
  flag[a] = (uint8_t)run;
}


}  // namespace

// Slab decomposition: which active blocks have a tile inside the owned planes (interior: no
// ghost particle in the tile, so the loop can run before the halo arrives) and which touch a
// ghost plane (boundary).  Tile x-planes are [ix0 - 1, ix0 + bx]; the owned planes are
// [ix_first, ix_first + nxo).
__global__ void k_block_side(DevGrid g, uint8_t* interior, uint8_t* boundary) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= g.nact) return;
  int jx, jy, zb;
  block_coords(g, g.blk_list[a], jx, jy, zb);
  const int ix0 = g.ix_first + jx * g.bx;
  const bool in = g.periodic_x || (ix0 - 1 >= g.ix_first && ix0 + g.bx < g.ix_first + g.nxo);
  interior[a] = in ? 1 : 0;
  boundary[a] = in ? 0 : 1;
}

cudaError_t launch_block_flags(int n, const unsigned int* keys, const DevGrid& g, uint8_t* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_block_flags<<<(n + 255) / 256, 256, 0, st>>>(n, keys, g, flag);
  return cudaGetLastError();
}

cudaError_t launch_tile_sizes_list(const DevGrid& g, const int* cell_start, const int* list, const int* nlist,
                                   int* max_tile, int* max_i, cudaStream_t st) {
  k_tile_sizes_list<<<148 * 4, 256, 0, st>>>(g, cell_start, list, nlist, max_tile, max_i);
  return cudaGetLastError();
}

cudaError_t launch_block_side(const DevGrid& g, uint8_t* interior, uint8_t* boundary, cudaStream_t st) {
  if (g.nact == 0) return cudaSuccess;
  k_block_side<<<(g.nact + 255) / 256, 256, 0, st>>>(g, interior, boundary);
  return cudaGetLastError();
}

int kernel_threads() { return kNW * 32; }
size_t tile_desc_bytes() { return sizeof(TileDesc) + (size_t)(kMaxTileCells + 1) * sizeof(int2); }
size_t tile_desc_header_bytes() { return sizeof(TileDesc); }

cudaError_t launch_tile_desc(const DevGrid& g, const int* cell_start, cudaStream_t st) {
  const int nb = g.run_list ? g.nrun : g.nact;
  if (nb == 0) return cudaSuccess;
  k_tile_desc<<<nb, 64, 0, st>>>(g, cell_start);
  return cudaGetLastError();
}

cudaError_t launch_tile_icols(const DevGrid& g, const int* cell_start, cudaStream_t st) {
  if (g.nact == 0) return cudaSuccess;
  k_tile_icols<<<(g.nact + 255) / 256, 256, 0, st>>>(g, cell_start);
  return cudaGetLastError();
}

cudaError_t launch_sparse_wide(const DevGrid& g, uint8_t* wide, int32_t* ncount, int kmin, cudaStream_t st) {
  if (g.nact == 0 || kmin <= 0) return cudaSuccess;
  k_sparse_wide<<<(g.nact + 255) / 256, 256, 0, st>>>(g, wide, ncount, kmin);
  return cudaGetLastError();
}

cudaError_t launch_block_run(const DevGrid& g, const DevState& s, uint8_t* flag, cudaStream_t st) {
  if (g.nact == 0) return cudaSuccess;
  k_block_run<<<(g.nact + 255) / 256, 256, 0, st>>>(g, s, flag);
  return cudaGetLastError();
}

size_t lists_smem(const DevGrid& g) {
  const int nw = g.lists_warps > 0 ? g.lists_warps : kNW;
  return lists_a_bytes(g, nw) + (size_t)((g.tcap + kNSent + 1) >> 1) * 16 + lists_slot_bytes(g) +
         lists_zw_bytes(g) + lists_slot_bytes(g);
}
size_t density_smem(const DevGrid& g) {
  return (size_t)(g.tcap + kNSent) * (2 * 16) + walk_bytes<DenAcc>(g.icap, kDensT);
}
size_t gradient_smem(const DevGrid& g) {
  return (size_t)(g.tcap + kNSent) * (2 * 16) + gradient_t2_bytes(g) + walk_bytes<GradAcc>(g.icap, kGradT);
}
size_t force_smem(const DevGrid& g) { return force_records_bytes(g.tcap) + (size_t)(g.icap + 1) * 8; }

cudaError_t launch_tile_sizes(const DevGrid& g, const int* cell_start, int* max_tile, int* max_i, uint8_t* flag,
                              cudaStream_t st) {
  k_tile_sizes<<<(g.nblocks + 255) / 256, 256, 0, st>>>(g, cell_start, max_tile, max_i, flag);
  return cudaGetLastError();
}

static cudaError_t set_smem(const void* fn, size_t bytes) {
  // (SPH_CARVEOUT: the shared-memory carveout in percent of the unified L1 / shared storage, -1 =
  // the driver's choice; an experiment knob)
  static const int carve = getenv("SPH_CARVEOUT") ? atoi(getenv("SPH_CARVEOUT")) : -1;
  if (carve >= 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_lists(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st) {
  const size_t sm = lists_smem(g);
  const bool wide = s.wide != nullptr && s.n_wide > 0, tag = wide || !g.periodic_x;
  const void* fn = wide ? (const void*)k_lists<true, true>
                        : (tag ? (const void*)k_lists<false, true> : (const void*)k_lists<false, false>);
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  if (g.nrun == 0) return cudaSuccess;
  const int thr = (g.lists_warps > 0 ? g.lists_warps : kNW) * 32;
  if (wide) k_lists<true, true><<<g.nrun, thr, sm, st>>>(g, ph, s, cell_start, ctr);
  else if (tag) k_lists<false, true><<<g.nrun, thr, sm, st>>>(g, ph, s, cell_start, ctr);
  else k_lists<false, false><<<g.nrun, thr, sm, st>>>(g, ph, s, cell_start, ctr);
  return cudaGetLastError();
}

cudaError_t launch_bank(int i0, int n, const DevGrid& g, const DevState& s, cudaStream_t st) {
  // (k_lists tags lists, and leaves them to k_bank, only with ghost planes or wide particles)
  if (n <= 0 || (g.periodic_x && !(s.wide != nullptr && s.n_wide > 0))) return cudaSuccess;
  const size_t sm = (size_t)(8 * kCellRows + 2 * kBankQ) * kBankThreads * 2;
  cudaError_t e = set_smem((const void*)k_bank, sm);
  if (e != cudaSuccess) return e;
  k_bank<<<(n + kBankThreads - 1) / kBankThreads, kBankThreads, sm, st>>>(i0, n, g, s);
  return cudaGetLastError();
}


cudaError_t launch_density(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, int pass,
                           const uint8_t* blk_in, uint8_t* blk_out, float hfac_stale, DevCounters* ctr,
                           cudaStream_t st) {
  const size_t sm = density_smem(g);
  cudaError_t e = set_smem((const void*)k_density, sm);
  if (e != cudaSuccess) return e;
  if (g.nrun == 0) return cudaSuccess;
  k_density<<<g.nrun, kDensT, sm, st>>>(g, ph, s, cell_start, pass, blk_in, blk_out, hfac_stale, ctr);
  return cudaGetLastError();
}

cudaError_t launch_gradient(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, float dt,
                            int first_step, DevCounters* ctr, cudaStream_t st) {
  const size_t sm = gradient_smem(g);
  cudaError_t e = set_smem((const void*)k_gradient, sm);
  if (e != cudaSuccess) return e;
  if (g.nrun == 0) return cudaSuccess;
  k_gradient<<<g.nrun, kGradT, sm, st>>>(g, ph, s, cell_start, dt, first_step, ctr);
  return cudaGetLastError();
}

cudaError_t launch_force(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st) {
  const size_t sm = force_smem(g);
  const void* fn = g.force_threads == 512 ? (const void*)k_force<512, 1> : (const void*)k_force<kForceT, 2>;
  cudaError_t e = set_smem(fn, sm);
  if (e != cudaSuccess) return e;
  if (g.nrun == 0) return cudaSuccess;
  if (g.force_threads == 512) k_force<512, 1><<<g.nrun, 512, sm, st>>>(g, ph, s, cell_start, ctr);
  else k_force<kForceT, 2><<<g.nrun, kForceT, sm, st>>>(g, ph, s, cell_start, ctr);
  return cudaGetLastError();
}

cudaError_t launch_force_fin(int i0, int n, const DevPhys& ph, const DevState& s, DevCounters* ctr, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_force_fin<<<(n + 255) / 256, 256, 0, st>>>(i0, n, ph, s, ctr);
  return cudaGetLastError();
}

}  // namespace sph
