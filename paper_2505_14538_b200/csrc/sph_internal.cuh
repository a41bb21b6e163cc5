// sph_internal.cuh -- device-side data layout and kernel launch interface of libsph.
//
// Layout in HBM: every per-particle array is stored in CELL ORDER (the
// order produced by the last sph_rebuild_cells), structure-of-arrays with the fields
// the interaction loops read together packed into 16-byte records:
//   xh   uint4  (X, Y, Z fixed point, h as f32 bits)        density/gradient/force tiles
//   vm   float4 (vx, vy, vz, m)                              density/gradient/force tiles
//   gq   float4 (c_s, u, m/rho, rho)                         gradient tile (+ xh, vm)
//   fr1  float4 (A = P/rho^2, Kf = f/(pi h^4), c_s, rho)     force tile
//   fr2  float4 (B, (P + kPeps) alpha_c, u, alpha_v)         force tile (P = A rho^2)
// plus plain f32 arrays for state and outputs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sph {

constexpr int kMaxTileCellsZ = 16;          // z cells per block + 2 halo cells
constexpr int kMaxTileCells = 16 * kMaxTileCellsZ;  // (BX+2)(BY+2) <= 16 tile columns
constexpr float kPi = 3.14159265358979323846f;

// Cell grid and CTA block decomposition.  A CTA owns the cells of BX x BY grid columns
// over z0..z1-1; its tile is the (BX+2) x (BY+2) neighbour columns over z0-1..z1 (wrapped).
struct DevGrid {
  int nx, ny, nz;     // cells per axis (each >= 3)
  int bx, by;         // grid columns per block along x, y (1 or 2)
  int nbx, nby;       // blocks along x, y
  int nzb, KZ;        // z blocks per column, cells per block
  int nblocks;        // nbx * nby * nzb
  int nact;           // blocks with i particles: the loop kernels' CTAs (a = blockIdx.x)
  const int* blk_list;  // [nact] active index a -> block id (per-block arrays are indexed by a)
  int nrun;           // blocks the loop kernels run: those with a non-wide i particle
  const int* run_list;  // [nrun] -> active index a (null: all nact, a = blockIdx.x)
  int ncells;
  int tcap;           // tile capacity (particles) the launch is sized for; slot tcap = sentinel
  int icap;           // most i particles (owned by the block) of any block
  int lcap;           // neighbour-list capacity per particle (multiple of 16)
  float skin;         // list radius = (1 + skin) max(H_i, H_j)
  int force_threads;  // block size of the force kernel: 448 (two CTAs per SM), or 512 when one CTA fills an SM
  int lists_warps;    // warps per k_lists CTA: ~ the mean block particle count / 32 (a warp per 32)
  const void* desc;   // [nblocks] tile descriptors (sph_kernels.cu TileDesc, k_tile_desc)
  const void* desc_cells;  // [nblocks][kMaxTileCells + 1] per tile cell (tile offset, global start)
  int* desc_pref;     // [nblocks][icap + 1] list-group prefix of the block's particles (k_lists)
  int* desc_prefF;    // [nblocks][icap + 1] the same over the force part of each list (k_lists)
  int dens_inner;     // Newton iterations per density pass inside the CTA (k_density; >= 1)
  float wide_margin;  // adaptive grid: wide when (1 + skin)(1 + wide_margin) gamma_k h > the cell side
  int coinc;          // some particles share their exact position with another (k_dup): the lists drop
                      // those pairs
  float scale[3];     // L_a / 2^32 as f32 (fixed point -> length)
  double dscale[3];   // L_a * 2^-32 exact (fp64 exact neighbour test)
  float side[3];      // cell side per axis
  float side_min;
  float eabs;         // 8 x max rounding error of a tile coordinate (length units)
  float lpad;         // k_lists' fp16 candidate test: list radius margin (units of side_min)
  int zbits;          // particles of a cell sorted by the top zbits of their z inside the cell
  float zbucket;      // side_z 2^-zbits: z order inside a cell holds up to this
  // Slab decomposition along x.  The rank owns x in [x_lo, x_lo + wfix) on the 2^-32 grid,
  // cut into nxo planes; local plane of x = ix_first + floor((x - x_lo) nxo / wfix).
  // One rank: x_lo = 0, wfix = 2^32, ix_first = 0, nxo = nx, periodic.  Several ranks:
  // local planes = [G ghost, nxo owned, G ghost] (nx = nxo + 2G, ix_first = G), not periodic
  // along x.  The left / right neighbours' slabs (x_loL, wfixL / x_loR, wfixR) place the
  // ghosts, local indices [0, gL) and [gL + n_own, ...), on their owners' planes.
  unsigned long long wfix, wfixL, wfixR;
  unsigned int x_lo, x_loL, x_loR;
  int periodic_x;
  int ix_first, nxo;
  int gL, n_own;
};

// Slab path, wide particles: ghost planes per side needed by an owned particle whose search
// reaches k planes (list radius / side, rounded up) from owned plane pl of nxo.  Its search
// [pl - k, pl + k] must stay inside the local planes (G >= k - distance to the nearer face),
// and when it crosses a face the neighbour must hold it as a ghost (G > its distance to that
// face, in whole planes), so that every pair with an owned particle has its evaluator on the
// owner's rank.
__host__ __device__ inline int ghost_planes_needed(int k, int pl, int nxo) {
  const int dl = pl, dr = nxo - 1 - pl;
  int need = k - (dl < dr ? dl : dr);
  if (k > dl && dl + 1 > need) need = dl + 1;
  if (k > dr && dr + 1 > need) need = dr + 1;
  return need > 1 ? need : 1;
}

struct DevPhys {
  float gamma_k, eta3, h_tol, pi_eta3;
  int h_max_iter, fh_mode;
  float gamma_eos, beta, alpha_v_max, ell, alpha_c_min, alpha_c_max, beta_c, c_cfl;
};

constexpr int kCoarseLevels = 3;  // wide search grids (cell factors F, F/3, F/9 of the p99 one)

struct DevState {
  uint4* xh;
  float4* vm;
  float* u;
  float* av;
  float* ac;
  float* dprev;
  int64_t* uid;       // caller id
  int32_t* orig;      // caller index 0..n-1 (for sph_get)
  // density
  float4* dens;       // rho, drho_dh, nhat, dn_dh
  float4* dvc;        // curl x, y, z, div
  int32_t* count;
  float4* fin;        // f, P, c, B
  float4* gq;         // c, u, m/rho, rho
  float4* vc;         // v, c      (the gradient tile's j records: 16 + 16 + 8 bytes per pair)
  float2* um;         // u, m/rho
  float* hlo;
  float* hhi;
  int32_t* iters;
  uint8_t* active;
  // gradient
  float2* grad;       // v_sig, lap_u
  float4* fr1;
  float4* fr2;
  // halo put (X3 over peer memory): the gradient epilogue also stores the fr1 /
  // fr2 records of the owned particles gi in [put_lo[d], put_hi[d]) at put_fr1[d][gi - put_lo[d]]
  // / put_fr2[d][...]: the ghost slots of the left (d = 0) / right (d = 1) neighbour; null = off
  float4* put_fr1[2];
  float4* put_fr2[2];
  int put_lo[2], put_hi[2];
  // and X2 from the density epilogue (finished particles): gq, vc, um into the neighbours'
  // ghost slots, h into their `hin` (their density loop still reads its ghost h; a copy kernel
  // moves it into xh after the token)
  float4* put_gq[2];
  float4* put_vc[2];
  float2* put_um[2];
  float* put_h[2];
  // force
  float4* acc;        // a, du
  float* vsig;
  int32_t* countf;
  // neighbour lists: tile-relative uint16 slots in two parts, each padded with sentinel slots
  // (tcap .. tcap+7) to a multiple of 8 and laid out in ROWS of 8 whose entry w lies in
  // shared-memory bank group w (slot mod 8; k_bank, sph_kernels.cu); [n][lcap]:
  //   rows [0, nL8)          the rest (self included): density and gradient walk both parts
  //   rows [nL8, nL8 + nF8)  the FORCE part: the pairs this particle evaluates once for both sides
  //                          (partner in the "upper" half of the cell stencil, or a ghost)
  // Lists without ghost planes or wide particles leave k_lists in this layout in slot order
  // (no bank-aware rows: ncount bit 31); the others go through k_bank.
  uint16_t* nbr;
  uint16_t* nbr_raw;  // k_lists' tagged output before k_bank: natural order, bit 15 = force part
  int32_t* ncount;    // nF | nL << 16 | final << 31: real entries of the two parts (k_lists)
  float* hbuild;      // h when the list was built
  // wide particles (adaptive cell side, sph_wide.cu): support past the cell side; nullptr /
  // 0 when there are none
  uint8_t* wide;      // [n] flag
  uint8_t* dup;       // [n] 1: another particle has exactly this position (k_dup, sph_api.cu)
  int32_t* widx;      // [n_wide] their indices, ascending
  uint32_t* wnbr;     // [n_wide][wlcap] neighbour lists, global indices
  int32_t* wcount;    // [n_wide] list lengths
  int n_wide, wlcap;
  int n_wide_own;     // widx[0, n_wide_own): the owned ones (then the slab path's ghosts)
  // the wide particles' search grids: kCoarseLevels coarse grids, level l of cells of cF[l]^3
  // grid cells (cnx x cny x cnz, the last along an axis possibly thinner), particles sorted by
  // coarse cell (cperm), ranges ccs; a wide particle searches the finest level whose cells are
  // at least half its reach (coarse_level, sph_wide.cu), so its box meets <= 3 cells per axis
  const uint32_t* cperm[kCoarseLevels];  // [n local] particle indices in coarse-cell order
  const int* ccs[kCoarseLevels];         // [cnx cny cnz + 1] coarse cell starts in cperm
  int cF[kCoarseLevels], cnx[kCoarseLevels], cny[kCoarseLevels], cnz[kCoarseLevels];
};

struct DevCounters {
  unsigned long long pairs;     // directed neighbour pairs of the loop (density: at the final h)
  unsigned long long pairs_all; // density: directed pairs evaluated over all h passes
  int unconverged;
  int h_exceeds;
  unsigned int dt_bits;         // min dt as f32 bits (positive)
  int nonfinite;
  int active_next;
  int list_stale;               // an h outgrew its list radius
  int list_overflow;            // max list length seen above lcap (0 = none)
  int wlist_overflow;           // max wide-list length seen above wlcap (0 = none)
  unsigned int max_resid_bits;  // density: max |nhat h^3 - eta^3| / eta^3 of the finished particles (f32 bits)
};

// Launchers (sph_kernels.cu).  All enqueue on `st`.
cudaError_t launch_lists(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st);
cudaError_t launch_density(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, int pass,
                           const uint8_t* blk_in, uint8_t* blk_out, float hfac_stale, DevCounters* ctr,
                           cudaStream_t st);
cudaError_t launch_gradient(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start, float dt,
                            int first_step, DevCounters* ctr, cudaStream_t st);
cudaError_t launch_force(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                         DevCounters* ctr, cudaStream_t st);
cudaError_t launch_force_fin(int i0, int n, const DevPhys& ph, const DevState& s, DevCounters* ctr, cudaStream_t st);
cudaError_t launch_tile_sizes(const DevGrid& g, const int* cell_start, int* max_tile, int* max_i, uint8_t* flag,
                              cudaStream_t st);
size_t lists_smem(const DevGrid& g);
size_t density_smem(const DevGrid& g);
size_t gradient_smem(const DevGrid& g);
size_t force_smem(const DevGrid& g);
cudaError_t launch_bank(int i0, int n, const DevGrid& g, const DevState& s, cudaStream_t st);
// wide particles (sph_wide.cu)
cudaError_t launch_mark_wide(int n, const DevGrid& g, const DevPhys& ph, const DevState& s, uint8_t* flag,
                             unsigned int* n0, cudaStream_t st);
cudaError_t launch_coarse_keys(int n, int level, const DevGrid& g, const DevState& s, unsigned int* keys,
                               unsigned int* vals, cudaStream_t st);
cudaError_t launch_wide_lists(const DevGrid& g, const DevPhys& ph, const DevState& s, const int* cell_start,
                              DevCounters* ctr, cudaStream_t st);
cudaError_t launch_wide_density(const DevGrid& g, const DevPhys& ph, const DevState& s, int pass, float hfac_stale,
                                DevCounters* ctr, cudaStream_t st);
cudaError_t launch_wide_gradient(const DevGrid& g, const DevPhys& ph, const DevState& s, float dt, int first_step,
                                 DevCounters* ctr, cudaStream_t st);
cudaError_t launch_wide_force(const DevGrid& g, const DevPhys& ph, const DevState& s, DevCounters* ctr,
                              cudaStream_t st);
int kernel_threads();
size_t tile_desc_bytes();  // descriptor + per-cell table, per block
size_t tile_desc_header_bytes();  // the descriptor alone
cudaError_t launch_tile_icols(const DevGrid& g, const int* cell_start, cudaStream_t st);
cudaError_t launch_tile_desc(const DevGrid& g, const int* cell_start, cudaStream_t st);
cudaError_t launch_block_run(const DevGrid& g, const DevState& s, uint8_t* flag, cudaStream_t st);
cudaError_t launch_sparse_wide(const DevGrid& g, uint8_t* wide, int32_t* ncount, int kmin, cudaStream_t st);
cudaError_t launch_block_side(const DevGrid& g, uint8_t* interior, uint8_t* boundary, cudaStream_t st);
cudaError_t launch_block_flags(int n, const unsigned int* keys, const DevGrid& g, uint8_t* flag, cudaStream_t st);
cudaError_t launch_tile_sizes_list(const DevGrid& g, const int* cell_start, const int* list, const int* nlist,
                                   int* max_tile, int* max_i, cudaStream_t st);

}  // namespace sph
