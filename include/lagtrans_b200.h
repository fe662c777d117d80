/*
 * lagtrans_b200.h — C ABI of liblagtrans_b200.so, the B200 drop-in for the
 * particle time step of the reference `lagtrans` package
 * (/root/reference/pkg/src/lagtrans).
 *
 * The reference has no native layer: its hot path is reached through three
 * Python surfaces, and every entry point below replaces one
 * of them.  Citations are reference file:line.
 *
 *   module API    physics.module_*(ctl, ens, met0, met1, dt, [rnd], [cache], work)
 *                 physics.py:82-301            -> lt_run (one module bit each)
 *   RNG API       rng.generate_random_nums      rng.py:156-181 -> lt_rng_fill
 *   runtime API   DevicePool.region_create / region_update_device /
 *                 region_update_host / region_delete / device_wait
 *                 device_runtime.py:165-230,118-127
 *                 -> lt_ctx_create / lt_particles_alloc / lt_field_h2d /
 *                    lt_met_load / lt_field_d2h / lt_ctx_destroy / lt_sync
 *
 * Conventions
 *   - Every function returns an int status: LT_OK (0) or a negative code;
 *     lt_last_error() gives the message of the calling thread's last failure.
 *     The Python layer maps codes onto the reference exception types
 *     (ValueError, IndexError, device_runtime.LifecycleError, RuntimeError).
 *   - No function throws; no torch types appear in any signature.
 *   - Host arrays are borrowed for the duration of the call only and must be
 *     C-contiguous.  Copies into device memory are ordered on the context's
 *     compute stream; D2H copies return after the data has landed.
 *   - One context per GPU; a context is driven by one host thread at a time
 *     (the DevicePool worker model, device_runtime.py:100-102).
 */
#ifndef LAGTRANS_B200_H
#define LAGTRANS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LT_ABI_VERSION 1

/* status codes */
#define LT_OK 0
#define LT_ERR_ARG (-1)    /* invalid argument          -> ValueError      */
#define LT_ERR_RANGE (-2)  /* work range out of bounds  -> IndexError      */
#define LT_ERR_STATE (-3)  /* lifecycle violation       -> LifecycleError  */
#define LT_ERR_CUDA (-4)   /* CUDA failure              -> RuntimeError    */
#define LT_ERR_NOMEM (-5)  /* device allocation failed  -> MemoryError     */

/* module bits for lt_run (pipeline order driver_cli.py:31-33; decay is new) */
#define LT_MOD_TIMESTEPS    (1u << 0)  /* physics.py:82-88   */
#define LT_MOD_ADVECTION    (1u << 1)  /* physics.py:91-116  */
#define LT_MOD_TURB         (1u << 2)  /* physics.py:119-147 */
#define LT_MOD_MESO         (1u << 3)  /* physics.py:150-188 */
#define LT_MOD_CONVECTION   (1u << 4)  /* physics.py:191-203 */
#define LT_MOD_SEDI         (1u << 5)  /* physics.py:206-222 */
#define LT_MOD_DECAY        (1u << 6)  /* new: exponential decay of q[decay_slot] */
#define LT_MOD_ISOSURF      (1u << 7)  /* physics.py:238-264 */
#define LT_MOD_POSITION     (1u << 8)  /* physics.py:267-287 */
#define LT_MOD_METEO        (1u << 9)  /* physics.py:290-301 */
#define LT_MOD_ISOSURF_INIT (1u << 10) /* physics.py:225-235 */

/* lt_run flags */
#define LT_RUN_RNG_INKERNEL (1u << 0) /* draw randoms in-kernel (else read the batch) */
#define LT_RUN_DT_ARRAY     (1u << 1) /* read dt from the dt array (else inline)       */
#define LT_RUN_WRITE_DT     (1u << 2) /* store dt computed by TIMESTEPS               */
#define LT_RUN_MODULE_CLOCKS (1u << 3) /* fused launch charges SM cycles per module (generic
                                          kernel; read with lt_module_cycles) — the PHYSICS
                                          timer rows of driver_cli.py:151-183 / timers.py */
#define LT_RUN_SORT_KEYS    (1u << 4) /* the launch also writes the box-sort keys of the
                                          particles' end positions; an lt_sort_by_box of the
                                          same range as the very next call on the context
                                          uses them instead of computing its own (no effect
                                          before the context's first sort) */

/* rng modes (model_state.py:15 plus the fast Philox mode) */
#define LT_RNG_FAITHFUL 0
#define LT_RNG_COUNTER 1
#define LT_RNG_PHILOX 2

/* isosurface modes (model_state.py:14) */
#define LT_ISO_OFF 0
#define LT_ISO_PRESSURE 1
#define LT_ISO_THETA 2

/* per-particle fields (ParticleEnsemble model_state.py:92-110,
   CacheState :184-195, dt, RandomBatch rng.py:32-44) */
#define LT_F_TIME 0
#define LT_F_P 1
#define LT_F_ZETA 2
#define LT_F_LON 3
#define LT_F_LAT 4
#define LT_F_Q 5        /* row = quantity slot 0..nq-1            */
#define LT_F_UVWP 6     /* row = component 0..2                   */
#define LT_F_ISO_VAR 7
#define LT_F_DT 8
#define LT_F_RND_CONV 9 /* n doubles                              */
#define LT_F_RND_TURB 10 /* 3n doubles, [3i:3i+3] for particle i  */
#define LT_F_RND_MESO 11 /* 3n doubles                            */
#define LT_F_ID 12      /* uint32 global particle index (sorted layouts) */

/* met storage precision for lt_met_grid */
#define LT_MET_F32 4
#define LT_MET_F64 8
/* lt_met_load flags */
#define LT_MET_CLOSE_LON (1u << 0) /* source lacks the +360 column: append column 0
                                      (ingest.py:195-207 met_periodic) */
#define LT_MET_DEVICE_SRC (1u << 1) /* source pointers are device memory (e.g. an
                                       NCCL-broadcast buffer): pack without staging */

/* kernel-relevant Control fields (model_state.py:18-45) + decay */
typedef struct lt_control {
  double t_stop, dt_model, met_dt;
  double turb_dx, turb_dz, turb_meso;
  double conv_prob, conv_p_top, p_surf, p_top;
  double sedi_radius, sedi_density;
  double decay_tau;          /* s, <= 0 disables */
  int32_t isosurf_mode;      /* LT_ISO_*  */
  int32_t rng_mode;          /* LT_RNG_*  */
  uint64_t rng_seed_global;  /* counter / philox key */
  int32_t decay_slot;        /* q row decayed by LT_MOD_DECAY */
  int32_t precision;         /* 0 exact (bit-faithful fp64), 1 fast (mixed) */
} lt_control;

typedef struct lt_ctx lt_ctx;

/* library / device discovery (device_runtime.py:39-55) */
int lt_abi_version(void);
int lt_device_count(int32_t *n);
const char *lt_last_error(void);

/* context = one GPU's data region (device_runtime.py:165-186) */
int lt_ctx_create(int32_t device, lt_ctx **out);
int lt_ctx_destroy(lt_ctx *ctx);                  /* region_delete */
int lt_sync(lt_ctx *ctx);                         /* device_wait   */
int lt_stream(lt_ctx *ctx, void **cuda_stream);   /* interop       */

/* particle store: SoA in HBM, `capacity` particles, nq quantity rows */
int lt_particles_alloc(lt_ctx *ctx, int64_t capacity, int32_t nq, int32_t with_batch);
int lt_field_h2d(lt_ctx *ctx, int32_t field, int32_t row, int64_t offset,
                 int64_t count, const void *host);
int lt_field_d2h(lt_ctx *ctx, int32_t field, int32_t row, int64_t offset,
                 int64_t count, void *host);
int lt_field_fill(lt_ctx *ctx, int32_t field, int32_t row, int64_t offset,
                  int64_t count, double value);
int lt_field_devptr(lt_ctx *ctx, int32_t field, int32_t row, void **dev);
int lt_ids_reset(lt_ctx *ctx, int64_t offset, int64_t count, int64_t first_id);

/* met store: up to 3 snapshot slots on one grid (MeteoField model_state.py:126-153) */
int lt_met_grid(lt_ctx *ctx, int32_t nx, int32_t ny, int32_t nz, const double *lons,
                const double *lats, const double *levs, int32_t precision);
int lt_met_load(lt_ctx *ctx, int32_t slot, double t_met, int32_t src_bytes,
                const void *u, const void *v, const void *w, const void *T,
                uint32_t flags);
int lt_met_load_nodes(lt_ctx *ctx, int32_t slot, double t_met, const float *uvwT,
                      uint32_t flags);
int lt_met_use(lt_ctx *ctx, int32_t slot0, int32_t slot1);
/* replicate a packed snapshot to another context (peer copy over NVLink;
   a device-to-device copy when both share a GPU) — the single-process
   met broadcast replacing the per-device deep copies of
   device_runtime.py:178-186; both contexts must hold the same grid */
int lt_met_copy_slot(lt_ctx *dst, int32_t dst_slot, lt_ctx *src, int32_t src_slot);
/* the met broadcast of the one-process-drives-all-GPUs design
   (arXiv 2211.12616; replaces the deep copy of met0/met1 into every device
   image on each rotation, driver_cli.py:146-149 -> device_runtime.py:178-186):
   slot slots[root] of ctxs[root] is replicated into slot slots[i] of every
   other context by ONE ncclBroadcast group over the distinct GPUs (NCCL is
   loaded at run time, communicators from ncclCommInitAll, cached per device
   list), each rank on its context's copy stream; contexts sharing a GPU get
   a device-to-device copy.  Asynchronous: lt_met_use orders the compute
   stream after the transfer, as after lt_met_load. */
int lt_met_broadcast(lt_ctx *const *ctxs, int32_t n, int32_t root, const int32_t *slots);
/* NCCL version code of the loaded libnccl (LT_ERR_STATE if none loads) and
   the number of NCCL ranks the process has created */
int lt_nccl_version(int32_t *version);
int lt_nccl_ranks(int32_t *nranks);
/* NCCL end to end on the GPUs present: a communicator over devices
   0..ndev-1 and one broadcast group of `bytes` from device 0 into a
   separate buffer on every device, checked byte for byte */
int lt_nccl_selftest(int32_t ndev, int64_t bytes);
int lt_met_slot_time(lt_ctx *ctx, int32_t slot, double *t_met);

/* climatology tables for module_meteo (ClimData model_state.py:156-181) */
int lt_clim_load(lt_ctx *ctx, int32_t nlat, int32_t np_, const double *lat_grid,
                 const double *p_grid, const double *hno3, const double *p_trop);

/* compute: apply the modules in `modules` to particles [start, end) */
int lt_run(lt_ctx *ctx, const lt_control *ctl, uint32_t modules, int64_t start,
           int64_t end, int64_t step, uint64_t faithful_state,
           int64_t faithful_base, uint32_t flags);
/* nsteps consecutive steps; results identical to nsteps lt_run calls.  The
   production chain (timesteps|advection|turb|meso|position) with in-kernel
   counter or philox draws, and the advection chain (timesteps|advection|
   position), run as one launch, each particle's state held in
   registers across the steps (a pending box-sort permutation is applied by
   a first single step); anything else as nsteps launches.  The selected met
   pair must cover all the steps. */
int lt_run_steps(lt_ctx *ctx, const lt_control *ctl, uint32_t modules, int64_t start,
                 int64_t end, int64_t step, int32_t nsteps, uint32_t flags);
/* host-buffer step (the module API's numpy path, physics.py:82-301 called
   on host arrays): particles [0, n) live in host memory (pinned for full
   PCIe overlap).  They stream through the context's particle store in
   chunks of `chunk` particles: H2D on the copy stream, the fused modules on
   the compute stream, D2H on a third stream, so both PCIe directions and
   the kernel overlap.  Particle i has global id first_id + i (RNG key).
   The store (and its ids) is scratch for the duration of the call; the
   call returns after every result has landed in host memory. */
typedef struct lt_host_soa {
  double *time, *p, *lon, *lat; /* required (read + write) */
  double *uvwp;                 /* 3 rows of `stride` doubles; LT_MOD_MESO */
  double *iso_var;              /* LT_MOD_ISOSURF / LT_MOD_ISOSURF_INIT */
  double *q;                    /* nq rows of `stride` doubles; METEO / DECAY */
  int64_t stride;               /* row stride of uvwp and q (>= n) */
  int32_t nq;
} lt_host_soa;
int lt_run_host(lt_ctx *ctx, const lt_control *ctl, uint32_t modules, int64_t n,
                int64_t step, int64_t first_id, uint64_t faithful_state,
                const lt_host_soa *io, int64_t chunk);
/* nsteps consecutive host-buffer steps (step, step+1, ...; the faithful
   state advances 7n draws per step): every step still moves every particle
   host -> device -> host, but chunk c of step s+1 starts as soon as chunk c
   of step s has landed, so the pipeline fills and drains once per call */
int lt_run_host_steps(lt_ctx *ctx, const lt_control *ctl, uint32_t modules, int64_t n,
                      int64_t step, int32_t nsteps, int64_t first_id, uint64_t faithful_state,
                      const lt_host_soa *io, int64_t chunk);

/* fill the device RandomBatch for [start, end) (rng.py:156-181); counter and
   philox draws are keyed by the slot's global particle id (LT_F_ID) once the
   store has ids (a shard or a sorted layout), else by the slot index */
int lt_rng_fill(lt_ctx *ctx, int32_t mode, uint64_t seed_or_state, int64_t step,
                int64_t start, int64_t end);
/* the in-kernel Philox4x32-10 block function (the north star's counter-based
   generator; words of particle gid at step s are blocks (gid lo, gid hi, s,
   0|1) under key (seed lo, seed hi)) on n explicit host (ctr[4], key[2])
   pairs, run on the device: out = n x 4 words.  A known-answer hook:
   Random123's kat_vectors must come back bit for bit. */
int lt_philox4x32_10(lt_ctx *ctx, int32_t n, const uint32_t *ctr, const uint32_t *key,
                     uint32_t *out);
/* interpolate_met (physics.py:69-79) at n host points: out = u,v,w,T rows (4n) */
int lt_interpolate(lt_ctx *ctx, int64_t n, const double *t, const double *lon,
                   const double *lat, const double *p, double *out);
/* the cell lookup of the exact (precision 0) or fast (1, f32 store) kernels
   at n host points: out = i, j, k rows (3n int32), which must equal the
   reference's _locate (physics.py:31-47: searchsorted(side='left') - 1,
   clipped; reversed levels) — the box-index audit; needs lt_met_grid only */
int lt_locate_cells(lt_ctx *ctx, int32_t precision, int64_t n, const double *lon,
                    const double *lat, const double *p, int32_t *out);
/* theta-isosurface non-convergence counter (CacheState.iso_nonconverged) */
int lt_iso_counter(lt_ctx *ctx, int64_t *value, int32_t reset);

/* Row groups that may stay in particle ("home") order while the store is
   box-sorted: the element of global particle id g sits at index
   g - home_base (home_base = first_id of the last lt_ids_reset, which must
   start at offset 0), so the sort need not move them; kernels reach them
   through the id row.  lt_set_home_rows converts the current layout.
   With every cold group (Q, ZETA, DT, ISO) in home order, lt_sort_by_box
   of the whole store defers the row permutation and the next lt_run of the
   production chain (timesteps + advection + turb + meso + position, drawing
   in-kernel) applies it while it streams the rows; any other call touching
   particle rows applies it first. */
#define LT_HOME_Q    (1u << 0)
#define LT_HOME_ZETA (1u << 1)
#define LT_HOME_DT   (1u << 2)
#define LT_HOME_ISO  (1u << 3)
int lt_set_home_rows(lt_ctx *ctx, uint32_t mask);

/* box sort: stable radix sort of [start, end) by met0 cell, ids travel along */
int lt_sort_by_box(lt_ctx *ctx, int64_t start, int64_t end);

/* sorts run on this context, and how many of them used the keys of the
   launch just before (LT_RUN_SORT_KEYS) instead of computing their own */
int lt_sort_info(lt_ctx *ctx, int64_t *sorts, int64_t *sorts_with_step_keys);
/* copies that undo the sort permutation (ids must be a permutation of
   [first_id, first_id + count)) */
int lt_field_d2h_ordered(lt_ctx *ctx, int32_t field, int32_t row, int64_t offset,
                         int64_t count, int64_t first_id, void *host);
int lt_field_h2d_ordered(lt_ctx *ctx, int32_t field, int32_t row, int64_t offset,
                         int64_t count, int64_t first_id, const void *host);

/* output-side statistics over particles [start, end) of the store
   (output.py:28-64), reduced in HBM:
   lt_grid_counts  write_grid (output.py:28-44): counts[ix * ny + iy] (int64,
                   nx*ny, overwritten), ix = clip(floor((lon+180)/(360/nx)),0,nx-1)
   lt_group_stats  write_ens (output.py:47-64): groups = int64(q[slot]) (must
                   be >= 0), ascending; count and mean/std (ddof 0) of lon,
                   lat, p.  mean/std are [3][max_groups] (lon, lat, p rows).
                   *ngroups receives the group count; LT_ERR_RANGE when it
                   exceeds max_groups (nothing else written), LT_ERR_ARG for a
                   negative group id (ValueError in the reference). */
int lt_grid_counts(lt_ctx *ctx, int32_t nx, int32_t ny, int64_t start, int64_t end,
                   int64_t *counts);
int lt_group_stats(lt_ctx *ctx, int32_t slot, int64_t start, int64_t end, int64_t max_groups,
                   int64_t *ngroups, int64_t *gid, int64_t *count, double *mean, double *std);

/* write_atm (output.py:17-25): one CSV row per particle "time,p,zeta,lon,
   lat,q0.." with every double formatted exactly as Python's repr() — the
   reference's bytes — by `threads` host threads (0: all cores).  q is nq
   rows of q_stride doubles.  lt_format_double formats one value. */
int lt_write_atm(const char *path, int64_t n, int32_t nq, const double *time, const double *p,
                 const double *zeta, const double *lon, const double *lat, const double *q,
                 int64_t q_stride, int32_t threads);
int lt_format_double(double x, char *out, int32_t cap, int32_t *len);

/* SM cycles the LT_RUN_MODULE_CLOCKS launches spent per module, summed
   over particles, in the order timesteps, random draws, advection, turb,
   meso, convection, sedi, decay, isosurf, position, meteo, isosurf_init;
   shares of a launch's event time give the reference's per-module
   PHYSICS timer rows for a fused step (timers.py:40-54) */
#define LT_N_MODULE_CLOCKS 12
int lt_module_cycles(lt_ctx *ctx, uint64_t *cycles, int32_t reset);

/* event timing of the last lt_run / lt_sort_by_box on this context */
int lt_timing(lt_ctx *ctx, int32_t enable);
int lt_last_elapsed_ms(lt_ctx *ctx, float *ms);

/* pinned host memory for streaming met snapshots */
int lt_host_alloc(int64_t bytes, void **out);
int lt_host_free(void *p);

#ifdef __cplusplus
}
#endif
#endif /* LAGTRANS_B200_H */
