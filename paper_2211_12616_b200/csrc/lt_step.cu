// lt_step.cu — launch of the fused step kernel (+ CUB sort wrapper).
#include <cub/cub.cuh>

#include "lt_kernels.cuh"

namespace lt {

// module sets compiled as their own specialisation (dead modules removed)
constexpr uint32_t kChainAdv = M_TIMESTEPS | M_ADVECTION | M_POSITION;
constexpr uint32_t kChainAdvDiff = M_TIMESTEPS | M_ADVECTION | M_TURB | M_MESO | M_POSITION;
// cfg4's plume chain and the full chain (engine.FULL), fp32 met store only
constexpr uint32_t kChainPlume = kChainAdvDiff | M_SEDI | M_DECAY;
constexpr uint32_t kChainFull = kChainAdvDiff | M_CONVECTION | M_SEDI | M_DECAY | M_ISOSURF | M_METEO;

template <class Rec, uint32_t FIXED, int FAST, int RM, int PM = 0>
static cudaError_t launch_fixed(const StepArgs<Rec>& a, cudaStream_t st) {
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (!blocks_per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, step_kernel<Rec, FIXED, FAST, RM, PM>, LT_STEP_BLOCK, 0);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t n = a.end - a.start;
  if (n <= 0) return cudaSuccess;
  int64_t grid = (n + LT_STEP_BLOCK - 1) / LT_STEP_BLOCK;
#ifndef LT_GRID_WAVES
#define LT_GRID_WAVES 48
#endif
  const int64_t cap = static_cast<int64_t>(sms) * blocks_per_sm * LT_GRID_WAVES;
  if (grid > cap) grid = cap;
  step_kernel<Rec, FIXED, FAST, RM, PM><<<static_cast<unsigned>(grid), LT_STEP_BLOCK, 0, st>>>(a);
  return cudaGetLastError();
}

template <class Rec, int FAST>
static cudaError_t launch_prec(const StepArgs<Rec>& a, cudaStream_t st) {
  // per-module cycle attribution runs in the generic kernel (the
  // specialised ones carry no instrumentation)
  if (a.flags & F_MODULE_CLOCKS) return launch_fixed<Rec, 0, FAST, -1>(a, st);
  // the production chain gets its in-kernel generator fixed at compile time;
  // with a pending box-sort permutation it applies it on the fly
  if (a.perm) {
    if (a.ctl.rng_mode == RNG_COUNTER) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_COUNTER, 1>(a, st);
    if (a.ctl.rng_mode == RNG_PHILOX) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_PHILOX, 1>(a, st);
    return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_FAITHFUL, 1>(a, st);
  }
  // several steps per launch (lt_run_steps checked the chain and generator)
  if (a.nsteps > 1) {
    if (a.modules == kChainAdv) return launch_fixed<Rec, kChainAdv, FAST, -1, 2>(a, st);
    if (a.ctl.rng_mode == RNG_PHILOX) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_PHILOX, 2>(a, st);
    return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_COUNTER, 2>(a, st);
  }
  if (a.modules == kChainAdvDiff && (a.flags & F_RNG_INKERNEL)) {
    if (a.ctl.rng_mode == RNG_COUNTER) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_COUNTER>(a, st);
    if (a.ctl.rng_mode == RNG_PHILOX) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_PHILOX>(a, st);
    if (a.ctl.rng_mode == RNG_FAITHFUL) return launch_fixed<Rec, kChainAdvDiff, FAST, RNG_FAITHFUL>(a, st);
  }
  if constexpr (sizeof(Rec) == sizeof(RecF)) {
    if ((a.flags & F_RNG_INKERNEL) && (a.modules == kChainPlume || a.modules == kChainFull)) {
      const bool full = a.modules == kChainFull;
      if (a.ctl.rng_mode == RNG_PHILOX)
        return full ? launch_fixed<Rec, kChainFull, FAST, RNG_PHILOX>(a, st)
                    : launch_fixed<Rec, kChainPlume, FAST, RNG_PHILOX>(a, st);
      if (a.ctl.rng_mode == RNG_COUNTER)
        return full ? launch_fixed<Rec, kChainFull, FAST, RNG_COUNTER>(a, st)
                    : launch_fixed<Rec, kChainPlume, FAST, RNG_COUNTER>(a, st);
    }
  }
  if (a.modules == kChainAdvDiff) return launch_fixed<Rec, kChainAdvDiff, FAST, -1>(a, st);
  if (a.modules == kChainAdv) return launch_fixed<Rec, kChainAdv, FAST, -1>(a, st);
  return launch_fixed<Rec, 0, FAST, -1>(a, st);
}

// launches that can apply a pending box-sort permutation on the fly: the
// production chain (it reads and writes every hot row) with a compile-time
// in-kernel generator
bool perm_capable(uint32_t modules, uint32_t flags, int rng_mode) {
  return modules == kChainAdvDiff && (flags & F_RNG_INKERNEL) && !(flags & F_MODULE_CLOCKS) &&
         (rng_mode == RNG_COUNTER || rng_mode == RNG_PHILOX || rng_mode == RNG_FAITHFUL);
}

template <class Rec>
cudaError_t launch_step(const StepArgs<Rec>& a, cudaStream_t st) {
  // the fast (mixed-precision) kernels exist for the fp32 met store only;
  // a geographic grid (uniform lon/lat, levels with the log2 guess) gets
  // its axis lookups fixed at compile time
  if constexpr (sizeof(Rec) == sizeof(RecF)) {
    if (a.ctl.precision == 1) {
      const bool geo = a.met.lon.uniform && a.met.lat.uniform && !a.met.lev.uniform &&
                       a.met.lev.logscale && a.met.lev.n - 1 <= kLevCap;
      return geo ? launch_prec<Rec, 2>(a, st) : launch_prec<Rec, 1>(a, st);
    }
  }
  return launch_prec<Rec, 0>(a, st);
}
template cudaError_t launch_step<RecF>(const StepArgs<RecF>&, cudaStream_t);
template cudaError_t launch_step<RecD>(const StepArgs<RecD>&, cudaStream_t);

cudaError_t sort_pairs(void* temp, size_t& temp_bytes, const uint32_t* keys_in,
                       uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                       int64_t n, int end_bit, cudaStream_t st) {
  return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out,
                                         static_cast<int>(n), 0, end_bit, st);
}

}  // namespace lt
