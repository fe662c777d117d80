// lt_step.cuh — the fused per-particle time step kernel.
//
// One thread advances one particle through the enabled modules in the
// reference pipeline order (driver_cli.py:31-33, :151-183):
//   timesteps -> [random draws] -> advection -> turb -> meso -> convection
//   -> sedi -> decay -> isosurf -> position -> meteo
// Particle state lives in registers between modules, so a fused step reads
// and writes each SoA field once.  Per-module calls from the drop-in module
// API launch the same kernel with a single module bit.
#pragma once

#include "lt_device.cuh"

namespace lt {

// Per-launch constants of a full step (dt == ctl.dt_model, the common case):
// the same fp64 expressions the kernel evaluates per particle, computed once
// on the host (sqrt and division are correctly rounded on both sides, so a
// particle taking them gets bit-identical values)
struct StepConst {
  double dt;        // ctl.dt_model
  double turb_sx;   // sqrt(2 turb_dx dt)
  double turb_sz;   // sqrt(2 turb_dz dt)
  double meso_r;    // clip(1 - 2 dt / met_dt, 0, 1)
  double meso_amp;  // sqrt(1 - r^2)
  double decay;     // exp(-dt / decay_tau) (host libm; 1 when decay is off)
  double conv_scale;  // (p_surf - conv_p_top) / conv_prob (fast path only)
  uint32_t philox_rk[20];  // Philox round keys of ctl.rng_seed_global (lt_device.cuh)
};

template <class Rec>
struct StepArgs {
  // particle store (SoA, row stride `cap` for q and uvwp)
  double* time;
  double* p;
  double* lon;
  double* lat;
  double* dt;
  double* uvwp[3];  // AR(1) mesoscale perturbations (CacheState.uvwp rows)
  double* iso_var;
  double* q;
  const uint32_t* ids;  // global particle index per slot, or null (= slot)
  uint32_t home_mask;   // HOME_* row groups kept in particle order (index id - home_base)
  int64_t home_base;
  // pending box-sort permutation (PERM kernels): slot s of the new order
  // holds old slot perm_start + perm[s - perm_start]; the hot rows and ids
  // are gathered through it and written to the o_* rows
  const uint32_t* perm;
  int64_t perm_start;
  double *o_time, *o_p, *o_lon, *o_lat;
  double* o_uvwp[3];
  uint32_t* o_ids;
  const double* rnd_conv;
  const double* rnd_turb;
  const double* rnd_meso;
  int64_t cap, start, end;
  int32_t nq;
  uint32_t modules, flags;
  int64_t step;
  int32_t nsteps;  // steps per launch (MULTI kernels: in-kernel counter/Philox draws)
  uint64_t faithful_state;
  int64_t faithful_base;
  unsigned long long* iso_nonconv;
  unsigned long long* mod_cycles;  // CK_N counters (F_MODULE_CLOCKS launches)
  // F_SORT_KEYS: the compressed box-sort key of each particle's end position
  // (the keys lt_sort_by_box's own box_key + compress kernels would make:
  // rank[Morton column] * sk_nocc + (level box - sk_kmin)) into sk_keys[s -
  // start], s - start into sk_vals; a level box outside the window sets *sk_bad
  uint32_t* sk_keys;
  uint32_t* sk_vals;
  const uint32_t* sk_rank;
  uint32_t sk_kmin, sk_nocc;
  unsigned int* sk_bad;
  Control ctl;
  StepConst kc;
  MetView<Rec> met;
  Clim clim;
};

__device__ __forceinline__ void prefetch_l2(const void* ptr) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}
__device__ __forceinline__ void prefetch_l1(const void* ptr) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr));
}

// particle-state rows are touched once per step: stream them past L1
// (evict-first) so L1 keeps the met records the gathers reuse
#ifndef LT_NO_STREAM_STATE
__device__ __forceinline__ double ld_state(const double* p) { return __ldcs(p); }
__device__ __forceinline__ void st_state(double* p, double v) { __stcs(p, v); }
#else
__device__ __forceinline__ double ld_state(const double* p) { return *p; }
__device__ __forceinline__ void st_state(double* p, double v) { *p = v; }
#endif

#ifndef LT_STEP_BLOCK
#define LT_STEP_BLOCK 256
#endif
#ifndef LT_STEP_MIN_BLOCKS
#define LT_STEP_MIN_BLOCKS (1024 / LT_STEP_BLOCK)
#endif
// resident blocks per SM the exact (FAST = 0) kernels are compiled for: 4
// (64 registers), except the adv+turb+meso chain with in-kernel Philox draws,
// whose fp64 Box-Muller pairs spill less at 3 blocks (80 registers): -3.2 %
// at cfg3, where the counter-word and full-chain kernels measured +0.7 % and
// +5 % slower at 3
#ifndef LT_EXACT_MIN_BLOCKS
#define LT_EXACT_MIN_BLOCKS 4
#endif
#ifndef LT_EXACT_PHILOX_MIN_BLOCKS
#define LT_EXACT_PHILOX_MIN_BLOCKS 3
#endif
constexpr int step_min_blocks(uint32_t fixed, int fast, int rm) {
  return fast ? LT_STEP_MIN_BLOCKS
              : (fixed == (M_TIMESTEPS | M_ADVECTION | M_TURB | M_MESO | M_POSITION) && rm == RNG_PHILOX
                     ? LT_EXACT_PHILOX_MIN_BLOCKS : LT_EXACT_MIN_BLOCKS);
}

// Arithmetic policy: FAST = 0 reproduces numpy's operation sequence in
// fp64; FAST = 1 is the mixed-precision path of lt_device.cuh (fp32 store
// only), FAST = 2 the same on a geographic grid (locate_h / locate_v).
template <class Rec, int FAST>
struct Ops {
  static constexpr bool kFast = false;
  __device__ static void sample(const MetView<Rec>& m, double t, double lon, double lat,
                                double p, int fmask, double out[4], uint32_t* col = nullptr) {
    lt::sample(m, t, lon, lat, p, fmask, out, col);
  }
  __device__ static double over_cos(double x, double lat) { return x / cos_lat(lat); }
  // one midpoint stage (physics.py:91-116): (xs, ys, zs) <- (lon, lat, p) +
  // h * wind sampled at (ts, xs, ys, zs)
  __device__ static void adv_stage(const MetView<Rec>& m, double ts, double& xs, double& ys,
                                   double& zs, double lon, double lat, double p, double h) {
    double w[4];
    sample(m, ts, xs, ys, zs, 7, w);
    const double nlon = lon + over_cos(w[0] * h * kDegPerM, ys);
    const double nlat = lat + w[1] * h * kDegPerM;
    const double np_ = p + w[2] * h;
    xs = nlon; ys = nlat; zs = np_;
  }
  // physics.py:199-203: the convective target level of a uniform u < conv_prob
  __device__ static double conv_target(const Control& ctl, const StepConst&, double u) {
    return ctl.conv_p_top + (u / ctl.conv_prob) * (ctl.p_surf - ctl.conv_p_top);
  }
  // physics.py:206-222 (module_sedi): Stokes settling hop of p
  __device__ static double sedi_hop(const Control& ctl, double p, double temp, double dt) {
    const double rho = 100.0 * p / (kRAir * temp);
    constexpr double k9eta = 9.0 * kEtaAir;
    const double vs = div_cr(2.0 * (ctl.sedi_radius * ctl.sedi_radius) * (ctl.sedi_density - rho) *
                             kG0, k9eta, 1.0 / k9eta);
    return p + div_cr(rho * kG0 * vs * dt, 100.0, 0.01);
  }
  // physics.py:238-264 (module_isosurf, theta): up to 10 fixed-point steps
  // p <- 1000 (T(p) / theta0)^(1/kappa) while |dp| >= 0.1; false if still pending
  __device__ static bool isosurf_theta(const MetView<Rec>& m, double time, double lon, double lat,
                                       double& p, double theta0) {
    bool pending = true;
    for (int it = 0; it < 10 && pending; ++it) {
      double v[4];
      sample(m, time, lon, lat, p, 8, v);
      const double pn = 1000.0 * power(v[3] / theta0, kInvKappa);
      const double dp = pn - p;
      p = pn;
      pending = fabs(dp) >= 0.1;
    }
    return !pending;
  }
  // physics.py turb vertical hop: p - rho g dz / 100 with rho = 100 p / (R T)
  __device__ static double vertical_hop(double p, double temp, double dz) {
    const double rho = 100.0 * p / (kRAir * temp);
    return p + div_cr(-(rho * kG0 * dz), 100.0, 0.01);
  }
  __device__ static uint32_t cell(const MetView<Rec>& m, double lon, double lat, double p) {
    return cell_of(m, lon, lat, p).r00;
  }
  // the cell of a point whose lon/lat column is already known
  __device__ static uint32_t cell_in_column(const MetView<Rec>& m, uint32_t col, double p) {
    double frev;
    return col * (m.nz - 1) + (m.nz - 2 - locate(m.lev, p, frev));
  }
  // corner spreads of u, v, w in met0 around record r00 (meso diffusion)
  // (run_typed builds the table of met0 before any launch with meso)
  __device__ static void spreads(const MetView<Rec>& m, uint32_t r00, double sig[3]) {
    load_spreads(m.sig0, r00, sig);
  }
  // x^e (isosurface potential temperature, physics.py:233-234, 256-257)
  __device__ static double power(double x, double e) { return pow(x, e); }
  __device__ static void normals(uint64_t seed, int64_t step, uint64_t gid, int stream, double z[3]) {
    counter_normals(seed, step, gid, stream, z);
  }
};

template <int G>
struct OpsFast {
  static constexpr bool kFast = true;
  __device__ static void sample(const MetView<RecF>& m, double t, double lon, double lat,
                                double p, int fmask, double out[4], uint32_t* col = nullptr) {
    sample_fast<G>(m, t, lon, lat, p, fmask, out, col);
  }
  __device__ static double over_cos(double x, double lat) { return x * inv_cos_lat_fast(lat); }
  // the same stage with fp32 increments (the winds are fp32 already; the
  // positions they are added to stay fp64)
  __device__ static void adv_stage(const MetView<RecF>& m, double ts, double& xs, double& ys,
                                   double& zs, double lon, double lat, double p, double h) {
    float w[4];
    sample_fast_f<G>(m, ts, xs, ys, zs, 7, w);
    const float hf = static_cast<float>(h);
    const float hk = hf * static_cast<float>(kDegPerM);
    const float ic = inv_cos_lat_f(ys);
    xs = lon + static_cast<double>(w[0] * hk * ic);
    ys = lat + static_cast<double>(w[1] * hk);
    zs = p + static_cast<double>(w[2] * hf);
  }
  __device__ static double conv_target(const Control& ctl, const StepConst& kc, double u) {
    return ctl.conv_p_top + u * kc.conv_scale;
  }
  // the same settling with an fp32 reciprocal of T and no fp64 divisions
  __device__ static double sedi_hop(const Control& ctl, double p, double temp, double dt) {
    const double rho = p * (100.0 / kRAir) *
                       static_cast<double>(rcp_approx(static_cast<float>(temp)));
    const double vs = (2.0 * kG0 / (9.0 * kEtaAir)) * (ctl.sedi_radius * ctl.sedi_radius) *
                      (ctl.sedi_density - rho);
    return p + rho * vs * (dt * (kG0 / 100.0));
  }
  // the theta iteration on the column found once (lon/lat do not move
  // inside it): per step a level lookup, a T-only gather and fp32 pow
  __device__ static bool isosurf_theta(const MetView<RecF>& m, double time, double lon,
                                       double lat, double& p, double theta0) {
    float fx, fy;
    const int i = locate_h<G>(m.lon, lon, fx);
    const int j = locate_h<G>(m.lat, lat, fy);
    const uint32_t col = static_cast<uint32_t>(i) * m.ny + j;
    const float gx = 1.0f - fx, gy = 1.0f - fy;
    const float xy[4] = {gx * gy, fx * gy, gx * fy, fx * fy};
    const float wt = static_cast<float>((time - m.t0) * m.inv_dt);
    const f32x2 w2 = bc2(fminf(fmaxf(wt, 0.0f), 1.0f));
    const float inv_theta0 = rcp_approx(static_cast<float>(theta0));
    const uint32_t dcol = m.nz - 1, drow = static_cast<uint32_t>(m.ny) * dcol;
    bool pending = true;
    // the column's T at the two levels of the current level cell, already
    // weighted over the 4 columns and blended in time: the iteration moves
    // only p, so while p stays in that cell (most iterations) T(p) is one
    // FMA on (T(k), T(k+1)) and the records are not gathered again
    int kcell = -1;
    f32x2 tz = pk2(0.0f, 0.0f);
    double cx = 0.0;    // lower node and fp32 1/width of the current level cell:
    float cinv = 0.0f;  // while p stays inside it, no lookup either
#pragma unroll 1
    for (int it = 0; it < 10 && pending; ++it) {
      float frev = static_cast<float>(p - cx) * cinv;
      int krev = kcell;
      if (!(kcell >= 0 && frev > kNodeEps && frev < 1.0f - kNodeEps)) {
        krev = locate_v<G>(m.lev, p, frev, m.levc);
        const double2 c = G == 2 ? m.levc[krev] : __ldg(m.lev.cell + krev);
        cx = c.x;
        cinv = __int_as_float(static_cast<int>(__double2loint(c.y)));
      }
      if (krev != kcell) {
        const uint32_t r00 = col * dcol + (m.nz - 2 - krev);
        f32x2 a = pk2(0.0f, 0.0f), b = pk2(0.0f, 0.0f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t r = r00 + (c & 1 ? drow : 0) + (c & 2 ? dcol : 0);
          f32x2 t0, t1;
          asm("ld.global.nc.b64 %0, [%1];" : "=l"(t0) : "l"(m.s0[r].x + 6));
          asm("ld.global.nc.b64 %0, [%1];" : "=l"(t1) : "l"(m.s1[r].x + 6));
          a = fma2(t0, bc2(xy[c]), a);
          b = fma2(t1, bc2(xy[c]), b);
        }
        tz = fma2(w2, sub2(b, a), a);   // w2 = 0 with equal snapshot times (inv_dt = 0)
        kcell = krev;
      }
      // (level k, level k+1) weights (frev, 1 - frev)
      const float temp = fmaf(lo2(tz), frev, hi2(tz) * (1.0f - frev));
      const double pn = static_cast<double>(
          1000.0f * ex2_approx(static_cast<float>(kInvKappa) * lg2_approx(temp * inv_theta0)));
      const double dp = pn - p;
      p = pn;
      pending = fabs(dp) >= 0.1;
    }
    return !pending;
  }
  // the same hop as p (1 - g dz / (R T)) with an fp32 reciprocal of T
  __device__ static double vertical_hop(double p, double temp, double dz) {
    const double k = static_cast<double>(
        rcp_approx(static_cast<float>(temp) * static_cast<float>(kRAir / kG0)));
    return p - p * (dz * k);
  }
  __device__ static uint32_t cell(const MetView<RecF>& m, double lon, double lat, double p) {
    return cell_fast<G>(m, lon, lat, p).r00;
  }
  __device__ static uint32_t cell_in_column(const MetView<RecF>& m, uint32_t col, double p) {
    float frev;
    return col * (m.nz - 1) + (m.nz - 2 - locate_v<G>(m.lev, p, frev, m.levc));
  }
  __device__ static void spreads(const MetView<RecF>& m, uint32_t r00, double sig[3]) {
    load_spreads(m.sig0, r00, sig);
  }
  __device__ static double power(double x, double e) {
    return static_cast<double>(ex2_approx(static_cast<float>(e) * lg2_approx(static_cast<float>(x))));
  }
  __device__ static void normals(uint64_t seed, int64_t step, uint64_t gid, int stream, double z[3]) {
    counter_normals_fast(seed, step, gid, stream, z);
  }
};
template <> struct Ops<RecF, 1> : OpsFast<1> {};
template <> struct Ops<RecF, 2> : OpsFast<2> {};

// Draws of one stream for particle slot s / global id gid: stream 0 = the
// convection uniform (x[0]), 1 = turbulent normals, 2 = mesoscale normals.
// RM >= 0 fixes the in-kernel generator at compile time (RNG_COUNTER,
// RNG_PHILOX or RNG_FAITHFUL, no batch); RM = -1 decides at run time.
template <class O, int RM, class Rec>
__device__ __forceinline__ void draws(const StepArgs<Rec>& a, int64_t s, uint64_t gid, int stream,
                                      double x[3], int64_t step) {
  const Control& ctl = a.ctl;
  if (RM == RNG_COUNTER) {
    if (stream == 0) x[0] = to_unit(counter_word(ctl.rng_seed_global, step, gid, 0, 0));
    else O::normals(ctl.rng_seed_global, step, gid, stream, x);
    return;
  }
  if (RM == RNG_PHILOX) {
    philox_stream(a.kc.philox_rk, step, gid, stream, x);
    return;
  }
  if (RM == RNG_FAITHFUL) {
    faithful_stream(a.faithful_state, gid - static_cast<uint64_t>(a.faithful_base), stream, x);
    return;
  }
  if (!(a.flags & F_RNG_INKERNEL)) {  // the caller's RandomBatch
    if (stream == 0) {
      x[0] = a.rnd_conv[s];
    } else {
      const double* b = stream == 1 ? a.rnd_turb : a.rnd_meso;
      x[0] = b[3 * s]; x[1] = b[3 * s + 1]; x[2] = b[3 * s + 2];
    }
    return;
  }
  if (ctl.rng_mode == RNG_COUNTER) {
    if (stream == 0) x[0] = to_unit(counter_word(ctl.rng_seed_global, step, gid, 0, 0));
    else O::normals(ctl.rng_seed_global, step, gid, stream, x);
  } else if (ctl.rng_mode == RNG_FAITHFUL) {
    faithful_stream(a.faithful_state, gid - static_cast<uint64_t>(a.faithful_base), stream, x);
  } else {
    philox_stream(a.kc.philox_rk, step, gid, stream, x);
  }
}

// index of a particle in a row group that may be kept in particle order:
// slot s (source slot `src` of a pending permutation) or its id - home_base
template <class Rec>
__device__ __forceinline__ int64_t row_index(const StepArgs<Rec>& a, int64_t s, int64_t src,
                                             uint32_t group) {
  return (a.home_mask & group) && a.ids ? static_cast<int64_t>(a.ids[src]) - a.home_base : s;
}

// PM: 0 one step, 1 one step applying a pending permutation (PERM), 2
// a.nsteps steps per particle (MULTI)
template <class Rec, uint32_t FIXED, int FAST, int RM, int PM>
__global__ void __launch_bounds__(LT_STEP_BLOCK, step_min_blocks(FIXED, FAST, RM))
    step_kernel(const __grid_constant__ StepArgs<Rec> a) {
  using O = Ops<Rec, FAST>;
  constexpr bool PERM = PM == 1, MULTI = PM == 2;
  const uint32_t mods = FIXED ? FIXED : a.modules;
  const Control& ctl = a.ctl;
  // each block walks its own contiguous run of (box-sorted) particles tile
  // by tile, so consecutive tiles reuse the met records left in L1
  const int64_t ntile = (a.end - a.start + blockDim.x - 1) / blockDim.x;
  const int64_t per = (ntile + gridDim.x - 1) / gridDim.x;
  const int64_t s_lo = a.start + static_cast<int64_t>(blockIdx.x) * per * blockDim.x;
  const int64_t s_hi = min(a.end, s_lo + per * blockDim.x);
  // 32-bit slots in the loop (capacity < 2^31, lt_particles_alloc): every
  // row address is one IMAD.WIDE.U32 on the kernel-parameter base instead
  // of a 64-bit add pair
  const uint32_t lo32 = static_cast<uint32_t>(min(s_lo, s_hi)), hi32 = static_cast<uint32_t>(s_hi);
  const uint32_t stride = blockDim.x;
  const uint32_t pstart = static_cast<uint32_t>(a.perm_start);
  unsigned long long nonconv = 0;

  // per-launch switches, decided once outside the particle loop
  // F_MODULE_CLOCKS (generic kernels only; the specialised ones compile it
  // out): SM cycles between module boundaries are charged to the module
  // that ends there (draws to CK_RNG), summed over threads — the per-module
  // split of a fused launch behind the reference's PHYSICS timer rows
  const bool clocks = FIXED == 0 && (a.flags & F_MODULE_CLOCKS);
  unsigned long long cyc[CK_N];
  long long t_last = 0;
  if (FIXED == 0) {
#pragma unroll
    for (int k = 0; k < CK_N; ++k) cyc[k] = 0;
  }
#define LT_CLOCK(slot)                                  \
  do {                                                  \
    if (FIXED == 0 && clocks) {                         \
      const long long t_ = clock64();                   \
      cyc[slot] += static_cast<unsigned long long>(t_ - t_last); \
      t_last = t_;                                      \
    }                                                   \
  } while (0)

  const bool want_turb = (mods & M_TURB) && (ctl.turb_dx != 0.0 || ctl.turb_dz != 0.0);
  const bool want_meso = (mods & M_MESO) && ctl.turb_meso != 0.0;
  const bool want_conv = (mods & M_CONVECTION) && ctl.conv_prob != 0.0;
  const bool turb_h = ctl.turb_dx > 0.0, turb_v = ctl.turb_dz > 0.0;

  for (uint32_t s = lo32 + threadIdx.x; s < hi32; s += stride) {
    // PERM: this slot's particle comes from old slot `src` (box sort applied
    // on the fly: gathered reads, coalesced writes to the o_* rows)
    const uint32_t src = PERM ? pstart + a.perm[s - pstart] : s;
    // stage the next particle's state rows into L2 while this one runs
    // (costs no registers; the loads below then hit L2 instead of HBM)
#ifndef LT_NO_PREFETCH
    if (!PERM && s + stride < hi32) {
      const uint32_t nx = s + stride;
      prefetch_l2(a.time + nx); prefetch_l2(a.lon + nx); prefetch_l2(a.lat + nx);
      prefetch_l2(a.p + nx);
      if (mods & M_MESO) {
        prefetch_l2(a.uvwp[0] + nx); prefetch_l2(a.uvwp[1] + nx); prefetch_l2(a.uvwp[2] + nx);
      }
      if (a.ids && (mods & (M_TURB | M_MESO | M_CONVECTION))) prefetch_l2(a.ids + nx);
    }
    if (PERM && s + stride < hi32) {  // the next tile's gathered source rows
      const uint32_t nx = pstart + a.perm[s + stride - pstart];
      prefetch_l2(a.time + nx); prefetch_l2(a.lon + nx); prefetch_l2(a.lat + nx);
      prefetch_l2(a.p + nx);
      prefetch_l2(a.uvwp[0] + nx); prefetch_l2(a.uvwp[1] + nx); prefetch_l2(a.uvwp[2] + nx);
      prefetch_l2(a.ids + nx);
    }
#endif
#ifndef LT_NO_L1PF_UVWP
    // exact kernels: this particle's AR(1) state into L1 now, so the meso
    // step's loads of it (issued late, after the gathers) hit L1 (-0.5 %;
    // the fast kernels measured +2.6 % with it — their L1 holds the records)
    if (FAST == 0 && (mods & M_MESO)) {
      prefetch_l1(a.uvwp[0] + src); prefetch_l1(a.uvwp[1] + src); prefetch_l1(a.uvwp[2] + src);
    }
#endif
    if (FIXED == 0 && clocks) t_last = clock64();
    double time = ld_state(a.time + src), lon = ld_state(a.lon + src), lat = ld_state(a.lat + src),
           p = ld_state(a.p + src);

    // random draws (rng.py:156-181) are made where they are consumed, which
    // keeps them out of the registers live across the advection gathers —
    // except on the fast counter path, below
    const uint64_t gid = (RM >= 0 || (a.flags & F_RNG_INKERNEL)) && (want_turb || want_meso || want_conv)
                             ? (a.ids ? static_cast<uint64_t>(a.ids[src]) : static_cast<uint64_t>(s))
                             : 0ull;

    // the particle's index in the home-ordered row groups (one ids load,
    // not one per row access: the row stores would keep the compiler from
    // reusing it)
    // (fast kernels with the isosurface / decay / meteo rows; the exact
    // kernels re-read the id at each use — a value live across the whole
    // iteration costs them more in spills)
    const bool need_home = FAST != 0 && (mods & (M_ISOSURF | M_ISOSURF_INIT | M_DECAY | M_METEO));
    const int64_t home = need_home && a.home_mask && a.ids
                             ? static_cast<int64_t>(a.ids[src]) - a.home_base
                             : static_cast<int64_t>(s);
#define LT_ROW(group) (need_home ? ((a.home_mask & (group)) && a.ids ? home : static_cast<int64_t>(s)) \
                                 : row_index(a, s, src, (group)))
#ifndef LT_NO_L1PF_UVWP
    // fast kernels: the decay module's q element (read late, after the
    // gathers, from the home-ordered q rows) into L1
    if (FAST != 0 && (mods & M_DECAY) && ctl.decay_tau > 0.0 && ctl.decay_slot >= 0 &&
        ctl.decay_slot < a.nq)
      prefetch_l1(a.q + static_cast<int64_t>(ctl.decay_slot) * a.cap + LT_ROW(HOME_Q));
#endif

    // nsteps consecutive steps of this particle with its state in registers
    // (particles are independent within a step; the caller keeps the met
    // pair valid for all of them)
    const int nk = MULTI ? a.nsteps : 1;
    bool meso_wrote = false;  // the (single) PERM step wrote the o_uvwp rows
#pragma unroll 1
    for (int ks = 0; ks < nk; ++ks) {
      const int64_t stp = a.step + ks;
      // physics.py:82-88 (module_timesteps)
      double dt;
      if ((mods & M_TIMESTEPS) || !(a.flags & F_DT_ARRAY)) {
        dt = np_min(ctl.t_stop - time, ctl.dt_model);
        dt = np_min(np_max(dt, 0.0), ctl.dt_model);
        if ((mods & M_TIMESTEPS) && (a.flags & F_WRITE_DT)) a.dt[row_index(a, s, src, HOME_DT)] = dt;
      } else {
        dt = a.dt[row_index(a, s, src, HOME_DT)];
      }
      const bool act = dt > 0.0;
      if (PERM) meso_wrote = want_meso && act;
      LT_CLOCK(CK_TIMESTEPS);

#ifndef LT_LATE_DRAWS
      // fast path with a compile-time generator: the six normals are pure ALU
      // work on the id, done (fp32, SFU) before the first gather so they fill
      // issue slots the gathers leave idle
      // (the exact path measured slower this way: its fp64 normals cost twice
      // the registers)
      constexpr bool kEarly = FAST != 0 && RM >= 0;
      float early[6];
      if (kEarly && act) {
        if (RM == RNG_FAITHFUL) {
          faithful_normals_fast(a.faithful_state, gid - static_cast<uint64_t>(a.faithful_base), early);
        } else if (RM == RNG_PHILOX) {
#ifdef LT_PROBE_NO_RNG  // timing probe only: what the draws cost
          for (int q = 0; q < 6; ++q) early[q] = 0.25f * static_cast<float>((gid >> q) & 3) - 0.3f;
#else
          philox_normals_fast(a.kc.philox_rk, stp, gid, early);
#endif
        } else {
          double z[3];
          if (want_turb) {
            O::normals(ctl.rng_seed_global, stp, gid, 1, z);
            early[0] = z[0]; early[1] = z[1]; early[2] = z[2];
          }
          if (want_meso) {
            O::normals(ctl.rng_seed_global, stp, gid, 2, z);
            early[3] = z[0]; early[4] = z[1]; early[5] = z[2];
          }
        }
      }
#endif

      // physics.py:225-235 (module_isosurf_init)
      if ((mods & M_ISOSURF_INIT) && ctl.isosurf_mode != ISO_OFF) {
        if (ctl.isosurf_mode == ISO_PRESSURE) {
          a.iso_var[LT_ROW(HOME_ISO)] = p;
        } else {
          double v[4];
          O::sample(a.met, time, lon, lat, p, 8, v);
          a.iso_var[LT_ROW(HOME_ISO)] = v[3] * O::power(1000.0 / p, kKappa);
        }
        LT_CLOCK(CK_ISOSURF_INIT);
      }

      // physics.py:91-116 (module_advection): explicit midpoint.  The two
      // stages share one (rolled) sample call site to keep the kernel small.
      if ((mods & M_ADVECTION) && act) {
        const double half = 0.5 * dt;
        double ts = time, xs = lon, ys = lat, zs = p, h = half;
#pragma unroll 1
        for (int stage = 0; stage < 2; ++stage) {
          // stage 0: midpoint from (lon, lat, p) with half a step;
          // stage 1: full step from (lon, lat, p) with the midpoint winds
          O::adv_stage(a.met, ts, xs, ys, zs, lon, lat, p, h);
          ts = time + half;
          h = dt;
        }
        lon = xs; lat = ys; p = zs;
        time = time + dt;
        LT_CLOCK(CK_ADVECTION);
      }

      constexpr uint32_t kNoColumn = 0xFFFFFFFFu;
      uint32_t tcol = kNoColumn;  // lon/lat column of the turb T sample (reused by meso)
      // exact kernels with a compile-time generator: the turb and meso
      // normals are drawn at ONE call site before the turbulence step (one
      // inlined copy of the fp64 log / cos / sincospi code instead of two —
      // the exact kernels stall on instruction fetch); Philox's two streams
      // also share block 1 and a Box-Muller pair there
      constexpr bool kBoth = !kEarly && RM >= 0 && ((FIXED & (M_TURB | M_MESO)) == (M_TURB | M_MESO));
      double zturb[3] = {0.0, 0.0, 0.0}, zmeso[3] = {0.0, 0.0, 0.0};
      if (kBoth && (want_turb || want_meso) && act) {
        if (RM == RNG_PHILOX) {
          philox_turb_meso(a.kc.philox_rk, stp, gid, zturb, zmeso);
        } else {
#pragma unroll 1
          for (int st = 1; st <= 2; ++st) {
            double z[3];
            draws<O, RM>(a, s, gid, st, z, stp);
            if (st == 1) { zturb[0] = z[0]; zturb[1] = z[1]; zturb[2] = z[2]; }
            else { zmeso[0] = z[0]; zmeso[1] = z[1]; zmeso[2] = z[2]; }
          }
        }
        LT_CLOCK(CK_RNG);
      }

      // physics.py:119-147 (module_diffusion_turb); the vertical part sees the
      // post-hop lon/lat and pre-hop p (numpy view aliasing)
      if (want_turb && act) {
        double xt[3];
#ifndef LT_LATE_DRAWS
        if (kEarly) { xt[0] = early[0]; xt[1] = early[1]; xt[2] = early[2]; }
        else
#endif
        if (kBoth) { xt[0] = zturb[0]; xt[1] = zturb[1]; xt[2] = zturb[2]; }
        else { draws<O, RM>(a, s, gid, 1, xt, stp); LT_CLOCK(CK_RNG); }
        if (turb_h) {
          double sig = a.kc.turb_sx;
          if (__builtin_expect(dt != a.kc.dt, 0)) sig = sqrt(2.0 * ctl.turb_dx * dt);
          const double nlon = lon + O::over_cos(sig * xt[0] * kDegPerM, lat);
          lat = lat + sig * xt[1] * kDegPerM;
          lon = nlon;
        }
        if (turb_v) {
          double v[4];
          O::sample(a.met, time, lon, lat, p, 8, v, &tcol);
          double sz = a.kc.turb_sz;
          if (__builtin_expect(dt != a.kc.dt, 0)) sz = sqrt(2.0 * ctl.turb_dz * dt);
          const double dz = sz * xt[2];
          p = O::vertical_hop(p, v[3], dz);
        }
        LT_CLOCK(CK_TURB);
      }

      // physics.py:150-188 (module_diffusion_meso): AR(1) with met0 cell spread
      if (want_meso && act) {
        double xm[3];
#ifndef LT_LATE_DRAWS
        if (kEarly) { xm[0] = early[3]; xm[1] = early[4]; xm[2] = early[5]; }
        else
#endif
        if (kBoth) { xm[0] = zmeso[0]; xm[1] = zmeso[1]; xm[2] = zmeso[2]; }
        else { draws<O, RM>(a, s, gid, 2, xm, stp); LT_CLOCK(CK_RNG); }
        // the vertical hop moved only p: the T sample's lon/lat column holds
        const uint32_t r00 = tcol != kNoColumn ? O::cell_in_column(a.met, tcol, p)
                                               : O::cell(a.met, lon, lat, p);
        // the AR(1) state loads go out before the spread-table load so the two
        // latencies overlap
        double prev[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) prev[f] = ld_state(a.uvwp[f] + src);
        double sig[3];
        O::spreads(a.met, r00, sig);
        double r = a.kc.meso_r, amp = a.kc.meso_amp;
        if (__builtin_expect(dt != a.kc.dt, 0)) {
          r = 1.0 - 2.0 * dt / ctl.met_dt;
          r = np_min(np_max(r, 0.0), 1.0);
          amp = sqrt(1.0 - r * r);
        }
        double pert[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double sigma = ctl.turb_meso * sig[f];
          pert[f] = r * prev[f] + amp * sigma * xm[f];
          st_state((PERM ? a.o_uvwp[f] : a.uvwp[f]) + s, pert[f]);
        }
        const double nlon = lon + O::over_cos(pert[0] * dt * kDegPerM, lat);
        lat = lat + pert[1] * dt * kDegPerM;
        lon = nlon;
        p = p + pert[2] * dt;
        LT_CLOCK(CK_MESO);
      }

      // physics.py:191-203 (module_convection)
      if (want_conv && act) {
        double xc[3];
        draws<O, RM>(a, s, gid, 0, xc, stp);
        LT_CLOCK(CK_RNG);
        if (p > ctl.conv_p_top && xc[0] < ctl.conv_prob)
          p = O::conv_target(ctl, a.kc, xc[0]);
        LT_CLOCK(CK_CONVECTION);
      }

      // physics.py:206-222 (module_sedi): Stokes settling
      if ((mods & M_SEDI) && ctl.sedi_radius != 0.0 && act) {
        double v[4];
        O::sample(a.met, time, lon, lat, p, 8, v);
        p = O::sedi_hop(ctl, p, v[3], dt);
        LT_CLOCK(CK_SEDI);
      }

      // decay (new module): q[slot] *= exp(-dt / tau) while active
      if ((mods & M_DECAY) && ctl.decay_tau > 0.0 && act && ctl.decay_slot >= 0 &&
          ctl.decay_slot < a.nq) {
        double* qs = a.q + static_cast<int64_t>(ctl.decay_slot) * a.cap + LT_ROW(HOME_Q);
        *qs = *qs * (dt == a.kc.dt ? a.kc.decay : exp(-dt / ctl.decay_tau));
        LT_CLOCK(CK_DECAY);
      }

      // physics.py:238-264 (module_isosurf): applies to every particle
      if ((mods & M_ISOSURF) && ctl.isosurf_mode != ISO_OFF) {
        if (ctl.isosurf_mode == ISO_PRESSURE) {
          p = a.iso_var[LT_ROW(HOME_ISO)];
        } else {
          const double theta0 = a.iso_var[LT_ROW(HOME_ISO)];
          nonconv += O::isosurf_theta(a.met, time, lon, lat, p, theta0) ? 0ull : 1ull;
        }
        LT_CLOCK(CK_ISOSURF);
      }

      // physics.py:267-287 (module_position): pole reflection, lon wrap, clamp
      if (mods & M_POSITION) {
        while (fabs(lat) > 90.0) {
          lat = (lat > 0.0 ? 1.0 : -1.0) * (180.0 - fabs(lat));
          lon = lon + 180.0;
        }
        if (lon < -180.0 || lon >= 180.0) {
          double m = fmod(lon + 180.0, 360.0);  // np.mod: result takes the divisor's sign
          if (m != 0.0) {
            if (m < 0.0) m += 360.0;
          } else {
            m = 0.0;
          }
          lon = m - 180.0;
        }
        p = np_min(np_max(p, ctl.p_top), ctl.p_surf);
        LT_CLOCK(CK_POSITION);
      }

      // physics.py:290-301 (module_meteo): sample T,u,v and climatology
      if (mods & M_METEO) {
        double v[4];
        O::sample(a.met, time, lon, lat, p, 11, v);
        const int64_t qi = LT_ROW(HOME_Q);
        a.q[qi] = v[3];
        a.q[a.cap + qi] = v[0];
        a.q[2 * a.cap + qi] = v[1];
        a.q[3 * a.cap + qi] = clim_hno3(a.clim, lat, p);
        a.q[4 * a.cap + qi] = p < clim_ptrop(a.clim, lat) ? 1.0 : 0.0;
        LT_CLOCK(CK_METEO);
      }

    }  // steps

    // the box-sort key of the end position (a sort follows this launch)
    if (!PERM && (a.flags & F_SORT_KEYS)) {
      int ci, cj, ck;
      if constexpr (FAST != 0) {
        float fx, fy, fz;
        ci = locate_h<FAST>(a.met.lon, lon, fx);
        cj = locate_h<FAST>(a.met.lat, lat, fy);
        ck = a.met.nz - 2 - locate_v<FAST>(a.met.lev, p, fz, a.met.levc);
      } else {
        const Cell c = cell_of(a.met, lon, lat, p);
        ci = c.i; cj = c.j; ck = c.k;
      }
      const uint32_t code = (part1by1(static_cast<uint32_t>(ci) >> LT_BOX_SHIFT) << 1) |
                            part1by1(static_cast<uint32_t>(cj) >> LT_BOX_SHIFT);
      const uint32_t kb = static_cast<uint32_t>(ck) / LT_BOX_ZDIV - a.sk_kmin;
      const uint32_t t = s - static_cast<uint32_t>(a.start);
      a.sk_keys[t] = __ldg(a.sk_rank + code) * a.sk_nocc + kb;
      a.sk_vals[t] = t;
      if (kb >= a.sk_nocc) atomicOr(a.sk_bad, 1u);
    }

    if (mods & (M_ADVECTION | M_TURB | M_MESO | M_CONVECTION | M_SEDI | M_ISOSURF | M_POSITION)) {
      st_state((PERM ? a.o_p : a.p) + s, p);
      st_state((PERM ? a.o_lon : a.lon) + s, lon);
      st_state((PERM ? a.o_lat : a.lat) + s, lat);
      if (mods & M_ADVECTION) st_state((PERM ? a.o_time : a.time) + s, time);
    }
    if (PERM) {  // every hot row moves with its particle, touched this step or not
      if (!(mods & (M_ADVECTION | M_TURB | M_MESO | M_CONVECTION | M_SEDI | M_ISOSURF |
                    M_POSITION))) {
        st_state(a.o_p + s, p);
        st_state(a.o_lon + s, lon);
        st_state(a.o_lat + s, lat);
      }
      if (!(mods & M_ADVECTION)) st_state(a.o_time + s, time);
      if (!meso_wrote) {
#pragma unroll
        for (int f = 0; f < 3; ++f) st_state(a.o_uvwp[f] + s, ld_state(a.uvwp[f] + src));
      }
      a.o_ids[s] = a.ids[src];
    }
  }

#undef LT_CLOCK
#undef LT_ROW
  if (FIXED == 0 && clocks) {  // warp sums, one atomic per warp and module
#pragma unroll
    for (int k = 0; k < CK_N; ++k) {
      unsigned long long v = cyc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(a.mod_cycles + k, v);
    }
  }
  if (mods & M_ISOSURF) {
    // warp-aggregated counter (CacheState.iso_nonconverged)
    unsigned long long tot = nonconv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(a.iso_nonconv, tot);
  }
}

}  // namespace lt
