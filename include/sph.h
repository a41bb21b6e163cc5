/*
 * sph.h -- C-ABI of libsph, the B200-native (sm_100a) hot path of SWIFT's SPHENIX SPH
 * solver as described in arXiv 2505.14538 ("Task-parallelism in SWIFT for heterogeneous
 * compute architectures").  Citations: "P:n" = line n of the paper text,
 * "S:n" = line n of SPEC.md, "Rk" = reading k of DESIGN.md §3.
 *
 * The path: density loop with the Newton-Raphson smoothing-length
 * iteration (Eqs. 2-6), density finalize (Eq. 8 + EoS + Balsara switch), gradient
 * loop (Eqs. 10-11 + Laplacian of u) with the gradient ghost (Eqs. 12-15, 21-24), force
 * loop (Eqs. 7, 9, 16-20, 22) with the CFL timestep, and kick/drift.
 *
 * Conventions
 *  - Positions are uint32 fixed point on a 2^-32 L grid per axis: x_a = X_a * L_a / 2^32,
 *    periodic (R25).  Interleaved [n][3] arrays for X and v.
 *  - Ownership: the context owns all device state; inputs are copied by sph_create /
 *    sph_set_particles; sph_get writes into caller buffers (host or device), in the
 *    caller's ORIGINAL particle order (by id).
 *  - Synchrony: work is enqueued on cfg.stream (NULL -> a library-owned stream).
 *    sph_density and sph_force return after the small synchronising read-backs they need
 *    (convergence count, dt); the other calls are asynchronous and report CUDA errors at
 *    the next synchronisation point.
 *  - Errors: no C++ exception crosses the ABI.  After any CUDA error the context is
 *    poisoned: every later call except sph_destroy / sph_last_error returns SPH_ERR_STATE.
 *    SPH_ERR_NOT_CONVERGED leaves the context valid (last h iterate kept).
 *  - Threading: a context is not thread-safe.  Contexts of a loopback group (below) are
 *    driven from one host thread each.
 *  - There is no CPU fallback: a call that cannot run on the GPU fails.
 *
 * Several ranks: nranks > 1 splits the box into
 * x-slabs, rank r owning x in [floor(r 2^32 / R), floor((r+1) 2^32 / R)) on the fixed-point
 * grid.  Each rank keeps one cell plane of ghosts on either side (cell side >= support
 * radius, so one plane is the whole halo of P:82's neighbour search) and exchanges, per
 * step: migrating particles + ghost positions/velocities at each rebuild (X1), ghost h and
 * gradient-loop records after the density loop (X2), force-loop records after the gradient
 * loop (X3), and the global flags / h_max / dt as allreduces (X4).  Every call below is then
 * COLLECTIVE: all ranks make the same calls in the same order.  The transport is NCCL (one
 * process per GPU; grouped ncclSend/ncclRecv between slab neighbours) or a loopback group
 * (several contexts in one process, one host thread each, any devices; device copies) used
 * to test the multi-rank path on one GPU.  sph_get returns the rank's OWNED particles in
 * its local order (n = sph_local_count; SPH_F_ID identifies them).
 */
#ifndef SPH_H_
#define SPH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_ABI_VERSION 5

typedef enum {
  SPH_OK = 0,
  SPH_ERR_INVALID_ARG = 1,    /* bad argument or configuration                              */
  SPH_ERR_CUDA = 2,           /* CUDA runtime error (context poisoned)                      */
  SPH_ERR_NCCL = 3,           /* multi-rank exchange error (context poisoned)               */
  SPH_ERR_OOM = 4,            /* device allocation failed                                   */
  SPH_ERR_NOT_CONVERGED = 5,  /* h iteration hit h_max_iter (R7); state kept          */
  SPH_ERR_H_EXCEEDS_CELL = 6, /* a smoothing length outgrew what the cell grid can hold      */
  SPH_ERR_NUMERIC = 7,        /* non-finite v_sig / dt                              */
  SPH_ERR_STATE = 8           /* call order violated or context poisoned                    */
} sph_status;

typedef struct sph_ctx sph_ctx; /* opaque */

typedef enum { SPH_TRANSPORT_NCCL = 0, SPH_TRANSPORT_LOOPBACK = 1 } sph_transport;

/* Configuration.  Defaults (sph_config_default) follow DESIGN.md §3 readings R1, R7, R8,
 * R22, R23 and SPEC S:72-74. */
typedef struct {
  uint32_t struct_size;   /* = sizeof(sph_config); ABI check                                */
  int64_t n_total;        /* total particle count over all ranks (nranks > 1: sizes buffers)*/
  double box[3];          /* periodic box side lengths L_a                                 */
  float gamma_k;          /* kernel support ratio H = gamma_k h; must be 2 (M4, R1)         */
  float eta;              /* target nhat h^3 = eta^3 (R1), default 1.2348            */
  float h_tol;            /* closure tolerance |g|/eta^3 (1e-4)                       */
  int32_t h_max_iter;     /* Newton cap (R7), default 32; 0 = density at the given h       */
  float cell_skin;        /* cell side >= gamma_k h_max (1 + cell_skin), default 0.05      */
  float gamma_eos;        /* 5/3                                                    */
  float beta;             /* Eq. 10, default 3                                              */
  float alpha_v_max;      /* Eq. 13, default 2                                              */
  float ell;              /* Eq. 12 decay length, default 0.05                      */
  float alpha_c_min, alpha_c_max, beta_c; /* Eqs. 21-24, defaults 0, 1, 1                  */
  float c_cfl;            /* S:261, default 0.1                                             */
  int32_t fh_mode;        /* R8: 0 -> f = 1/Omega (default), 1 -> f = Omega (Eq. 8 literal)*/
  int32_t device;         /* CUDA device ordinal                                            */
  void* stream;           /* cudaStream_t to enqueue on, or NULL                            */
  int32_t rank, nranks;   /* slab decomposition over nranks ranks (default 0, 1)            */
  int32_t tile_cells_z;   /* cells per CTA block along z (0 = auto)                         */
  int32_t predict_h;      /* drift also advances h with d ln h/dt = (div v)/3 (continuity),   */
                          /* a better Newton start; the converged h does not depend on it     */
  int32_t transport;      /* sph_transport, used when nranks > 1                            */
  const void* nccl_uid;   /* NCCL: 128-byte id from sph_nccl_unique_id on rank 0, same on all*/
  void* loopback;         /* LOOPBACK: group from sph_loopback_create (shared by the ranks)  */
  int32_t adaptive_h;     /* strong h contrast: when the cells sized from      */
                          /* h_max overflow the tiles, size them from an h quantile and treat  */
                          /* the particles whose support exceeds a cell as "wide" (global-index*/
                          /* lists); default 1, 0 = fail instead.  Slab path:   */
                          /* the largest of the ranks' quantiles, and up to 16 ghost cell planes*/
                          /* per side (more: SPH_ERR_H_EXCEEDS_CELL)                           */
  int32_t decomp[3];      /* ranks per axis of the domain decomposition;*/
                          /* {0,0,0} (default) = x-slabs {nranks, 1, 1}, the one implemented:   */
                          /* any other product of nranks is SPH_ERR_INVALID_ARG                */
  int32_t halo_put;       /* X2 / X3 halos: 1 = the density and gradient  */
                          /* loops' epilogues store each boundary-plane particle's records      */
                          /* straight into the neighbours' ghost slots over peer memory (NVLink */
                          /* P2P stores through CUDA IPC mappings; loopback: the other contexts'*/
                          /* buffers) and each exchange sends only a zero-payload token that    */
                          /* orders the neighbours' next loop after them; 0 = NCCL send/recv of */
                          /* the planes after the loop; -1 (default) = 1 for loopback and one   */
                          /* rank, 0 for NCCL over several ranks (not yet run on multi-GPU      */
                          /* hardware).  DESIGN.md §9.                                          */
  int32_t balance;        /* slab cuts (several ranks): 0 (default) = fixed, rank r owns          */
                          /* [floor(r 2^32 / R), floor((r+1) 2^32 / R)); 1 = every rebuild moves */
                          /* each cut toward equal owned-particle counts (a global histogram of  */
                          /* x, at most a quarter of a cell plane per rebuild so migrants stay   */
                          /* within one plane; slabs kept >= half the uniform width) -- the 1-D  */
                          /* orthogonal recursive bisection of the slab path       */
} sph_config;

/* Particle input.  n particles; arrays are host pointers (on_device = 0) or device
 * pointers (on_device = 1).  alpha_v / alpha_c / id may be NULL (defaults 0.1 / 0 /
 * 0..n-1, R23).  div_prev may be NULL (the next sph_gradient is then a first step,
 * R19). */
typedef struct {
  int64_t n;
  int32_t on_device;
  const uint32_t* X;      /* [n][3] fixed-point positions                                  */
  const float* v;         /* [n][3] velocities                                             */
  const float* m;         /* [n] masses                                                    */
  const float* u;         /* [n] internal energies                                         */
  const float* h;         /* [n] smoothing lengths (initial guess for the h iteration)     */
  const float* alpha_v;   /* [n] viscosity switch, nullable                                */
  const float* alpha_c;   /* [n] conduction switch, nullable                               */
  const float* div_prev;  /* [n] div v of the previous step, nullable                      */
  const int64_t* id;      /* [n] caller ids, nullable                                      */
} sph_particles_in;

typedef struct {
  int32_t iterations;      /* density passes run (1 = converged on the first pass)         */
  int32_t unconverged;     /* particles not converged after the last pass (several ranks:   */
                           /* the largest count of any rank)                                */
  int32_t rebuilds;        /* cell-grid rebuilds forced by growing h                       */
  float max_rel_resid;     /* max over the particles of |nhat h^3 - eta^3| / eta^3 at their  */
                           /* final h (the closure residual; <= h_tol when converged)  */
  int64_t pairs_density;   /* sum_i N_i at the final h (directed pairs, j != i)            */
  int64_t pairs_h_iter;    /* directed pairs evaluated over all density passes             */
} sph_density_stats;

typedef struct {
  int64_t pairs_density;   /* last sph_density: sum_i N_i                                  */
  int64_t pairs_gradient;  /* last sph_gradient: directed pairs                            */
  int64_t pairs_force;     /* last sph_force: directed pairs (= 2 x unordered)             */
  int64_t pairs_h_iter;    /* last sph_density: directed pairs over all passes             */
  int64_t coincident;      /* pairs with r_ij = 0, j != i, skipped                 */
  int64_t kernel_launches; /* kernels launched by this context since creation              */
  int64_t wide_particles;  /* particles handled as wide by the adaptive grid (last rebuild) */
} sph_counters;

/* Device-time phases (sph_get_timings). */
typedef enum {
  SPH_T_REBUILD = 0,    /* binning: sort, permute, migration + ghost exchange (a1, X1, X6)     */
  SPH_T_LISTS = 1,      /* neighbour-list build (one per rebuild or list refresh)              */
  SPH_T_DENSITY = 2,    /* one density pass each (a2-a4)                                        */
  SPH_T_GRADIENT = 3,   /* a5-a6                                                                */
  SPH_T_FORCE = 4,      /* a7-a8                                                                */
  SPH_T_KICK_DRIFT = 5, /* a9                                                                   */
  SPH_T_EXCHANGE = 6,   /* halo exchanges outside the rebuild (X2, X3)                          */
  SPH_T_COUNT = 8
} sph_phase;

typedef struct {
  double ms[SPH_T_COUNT];     /* summed device time per phase (CUDA events on the context stream) */
  int64_t count[SPH_T_COUNT]; /* timed launches / scopes per phase                               */
} sph_timings;

/* Fields for sph_get (element type; components). */
typedef enum {
  SPH_F_X = 0,        /* uint32 x3  fixed-point position                                   */
  SPH_F_V = 1,        /* f32 x3                                                             */
  SPH_F_M = 2,        /* f32                                                                */
  SPH_F_U = 3,        /* f32                                                                */
  SPH_F_H = 4,        /* f32  smoothing length                                              */
  SPH_F_RHO = 5,      /* f32  Eq. 2                                                         */
  SPH_F_DRHO_DH = 6,  /* f32                                                                */
  SPH_F_NHAT = 7,     /* f32  Eq. 5                                                         */
  SPH_F_DN_DH = 8,    /* f32  Eq. 6                                                         */
  SPH_F_DIV = 9,      /* f32  Eq. 3 (R5)                                                    */
  SPH_F_CURL = 10,    /* f32 x3  Eq. 4 (R5)                                                 */
  SPH_F_COUNT = 11,   /* int32  N_i, density neighbours j != i                              */
  SPH_F_F = 12,       /* f32  h-factor f (Eq. 8, R8)                                        */
  SPH_F_P = 13,       /* f32  pressure                                                      */
  SPH_F_C = 14,       /* f32  sound speed                                                   */
  SPH_F_B = 15,       /* f32  Balsara switch (R14)                                          */
  SPH_F_VSIG_GRAD = 16, /* f32  v_sig from the gradient loop (R15)                         */
  SPH_F_LAP_U = 17,   /* f32  Laplacian of u (R16)                                          */
  SPH_F_ALPHA_V = 18, /* f32                                                                */
  SPH_F_ALPHA_C = 19, /* f32                                                                */
  SPH_F_DIV_PREV = 20,/* f32                                                                */
  SPH_F_A = 21,       /* f32 x3  dv/dt (Eqs. 7 + 17)                                        */
  SPH_F_DU = 22,      /* f32  du/dt (Eqs. 18 + 19 + R10)                                    */
  SPH_F_VSIG = 23,    /* f32  v_sig from the force loop                                     */
  SPH_F_COUNT_FORCE = 24, /* int32  force neighbours (r < max(H_i, H_j), j != i)            */
  SPH_F_ID = 25,      /* int64                                                              */
  SPH_F_ITERS = 26    /* int32  Newton updates in the last sph_density (-1 = unconverged)   */
} sph_field;

/* Fill a configuration with the defaults listed above (box = unit cube). */
void sph_config_default(sph_config* cfg);

/* Create a context on cfg->device and copy the particles in (S:104 build_tree: the cell
 * grid is built here).  On success *out is a valid context.  nranks > 1: collective; each
 * rank passes the particles of its slab (a particle up to one cell plane outside migrates,
 * farther is SPH_ERR_INVALID_ARG) and cfg->n_total > 0. */
sph_status sph_create(const sph_config* cfg, const sph_particles_in* in, sph_ctx** out);

/* Replace every particle field (one rank: same n as at creation; several ranks: the
 * rank's slab, at most the capacity derived from n_total).  Resets div_prev validity
 * unless in->div_prev is given.  Asynchronous on the context stream. */
sph_status sph_set_particles(sph_ctx* ctx, const sph_particles_in* in);

/* Wrap positions, bin particles into the cell grid (side >= gamma_k h_max (1+skin)) with a
 * device radix sort by cell key, and permute every particle array into cell order
 * (replaces SWIFT's cell tree + sort tasks). */
sph_status sph_rebuild_cells(sph_ctx* ctx);

/* Density loop + h iteration (Eqs. 2-6) fused with the density finalize
 * (Eq. 8, EoS, Balsara).  Newton with bracket/bisection safeguard (R7) on the particles
 * not yet within h_tol; the grid is rebuilt if an h outgrows it.  stats may be NULL. */
sph_status sph_density(sph_ctx* ctx, sph_density_stats* stats);

/* Gradient loop (v_sig, Laplacian of u; Eqs. 10-11, R15, R16) fused with the gradient
 * ghost (alpha_v Eqs. 12-15, alpha_c Eqs. 21-24; R17-R21).  dt > 0 is the step used by
 * the switch integration; if div_prev is not valid (first step) Ddot = 0 (R19). */
sph_status sph_gradient(sph_ctx* ctx, float dt);

/* Force loop (Eqs. 7, 9, 16-20, 22; R3, R9-R13) fused with the CFL reduction
 * dt = C_cfl min_i 2 gamma_k h_i / v_sig,i.  dt_next may be NULL. */
sph_status sph_force(sph_ctx* ctx, float* dt_next);

/* Kick v += a dt_kick, u = max(0, u + du dt_kick); drift x += v dt_drift on the
 * fixed-point grid with periodic wrap.  Marks the cell grid
 * stale: the next sph_density rebuilds it. */
sph_status sph_kick_drift(sph_ctx* ctx, float dt_kick, float dt_drift);

/* Copy one field out, in the caller's original order (by id), to host (on_device = 0)
 * or device memory.  dst must hold n x components elements of the field's type (several
 * ranks: the owned particles in local order, n = sph_local_count). */
sph_status sph_get(sph_ctx* ctx, int field, void* dst, int on_device);

/* Pipelined host I/O (a host loop that uploads step k+1 while step k computes and reads step
 * k's results back while step k+1 computes; bench.py's e2e).  Copies run on the context's
 * two copy streams (host-to-device, device-to-host), never on the context stream.
 * sph_stage_particles: enqueue the host -> device copy of every array of `in` (on_device must
 *   be 0; page-locked memory for real overlap) into the context's staging buffers and return;
 *   the copy waits until the previous staged upload has been taken by
 *   sph_set_particles_staged.  The host arrays must stay unchanged until the copy is done
 *   (sph_synchronize, or the next sph_set_particles_staged has returned).
 * sph_set_particles_staged: sph_set_particles from the last staged upload (the context
 *   stream waits for its copy; SPH_ERR_STATE if nothing is staged).
 * sph_get_async: sph_get into host memory `dst`, the device -> host copy enqueued after the
 *   work enqueued so far; `dst` is written by the next sph_synchronize (at most 8 reads in
 *   flight; a ninth waits for the oldest). */
sph_status sph_stage_particles(sph_ctx* ctx, const sph_particles_in* in);
sph_status sph_set_particles_staged(sph_ctx* ctx);
sph_status sph_get_async(sph_ctx* ctx, int field, void* dst);

/* Particles owned by this rank (= n for one rank); -1 for NULL. */
int64_t sph_local_count(const sph_ctx* ctx);

/* NCCL transport: write a fresh 128-byte ncclUniqueId to out128 (call on rank 0, then
 * broadcast it to the other ranks out of band, e.g. torch.distributed). */
sph_status sph_nccl_unique_id(void* out128);

/* Loopback transport: a group of nranks in-process ranks; destroy after every context of
 * the group is destroyed. */
sph_status sph_loopback_create(int32_t nranks, void** group);
sph_status sph_loopback_destroy(void* group);

/* Counters of the last calls (pairs per loop, launches). */
sph_status sph_get_counters(sph_ctx* ctx, sph_counters* out);

/* Per-phase device timing with CUDA events recorded around every launch on the context
 * stream (off by default; a few microseconds per launch when on). */
sph_status sph_set_timing(sph_ctx* ctx, int on);

/* Synchronise the stream and return the summed phase times since the last reset; reset != 0
 * zeroes them afterwards. */
sph_status sph_get_timings(sph_ctx* ctx, sph_timings* out, int reset);

/* Block until all work enqueued by the context has finished. */
sph_status sph_synchronize(sph_ctx* ctx);

/* Human-readable message for the last error of this context ("" if none). */
const char* sph_last_error(const sph_ctx* ctx);

/* Destroy the context and free its device memory.  Always safe (NULL, poisoned ctx). */
sph_status sph_destroy(sph_ctx* ctx);

/* Library ABI version (SPH_ABI_VERSION). */
int sph_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPH_H_ */
