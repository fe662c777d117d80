// lt_kernels.cuh — launcher declarations shared by the kernels and the C ABI.
#pragma once

#include "lt_step.cuh"

namespace lt {

// node `which` (0: level k, 1: level k+1) of a record (layout in lt_device.cuh)
__device__ __forceinline__ void store_node(RecF& r, int which, double u, double v, double w,
                                           double T) {
  r.x[2 * which] = static_cast<float>(u);
  r.x[2 * which + 1] = static_cast<float>(v);
  r.x[4 + which] = static_cast<float>(w);
  r.x[6 + which] = static_cast<float>(T);
}
__device__ __forceinline__ void store_node(RecD& r, int which, double u, double v, double w,
                                           double T) {
  r.x[2 * which] = u; r.x[2 * which + 1] = v;
  r.x[4 + which] = w; r.x[6 + which] = T;
}

template <class Src, class Rec>
cudaError_t launch_pack_fields(Rec* out, const Src* u, const Src* v, const Src* w, const Src* T,
                               int nx, int ny, int nz, int nx_src, cudaStream_t st);
template <class Rec>
cudaError_t launch_pack_nodes(Rec* out, const float4* nodes, int nx, int ny, int nz, int nx_src,
                              cudaStream_t st);
// per-cell mesoscale spreads of the met0 records (MetView::sig0)
template <class Rec>
cudaError_t launch_spread_table(const MetView<Rec>& m, int nx, double* out, cudaStream_t st);
cudaError_t launch_rng_fill(int mode, uint64_t seed, int64_t step, int64_t start, int64_t end,
                            const uint32_t* ids, double* conv, double* turb, double* meso,
                            cudaStream_t st);
template <class Rec>
cudaError_t launch_box_keys(const MetView<Rec>& m, const double* lon, const double* lat,
                            const double* p, int64_t start, int64_t n, uint32_t* keys,
                            uint32_t* vals, int morton, unsigned int* kzone, cudaStream_t st);
cudaError_t launch_compress_keys(uint32_t* keys, int64_t n, const uint32_t* rank, uint32_t nlev,
                                 uint32_t kmin, uint32_t nocc, cudaStream_t st);
constexpr int kRowSet = 4;
struct RowSet {
  const double* src[kRowSet];
  double* dst[kRowSet];
  int n;
};
cudaError_t launch_permute_rows(const RowSet& r, const uint32_t* perm, int64_t start, int64_t n,
                               cudaStream_t st);
template <class T>
cudaError_t launch_permute(T* dst, const T* src, const uint32_t* perm, int64_t start, int64_t n,
                           cudaStream_t st);
cudaError_t launch_unsort(double* out, const double* in, const uint32_t* ids, int64_t offset,
                          int64_t count, int64_t first_id, int* bad, int stride, cudaStream_t st);
cudaError_t launch_resort(double* out, const double* in, const uint32_t* ids, int64_t offset,
                          int64_t count, int64_t first_id, int* bad, int stride, cudaStream_t st);
template <class Rec>
cudaError_t launch_sample(const MetView<Rec>& m, const double* t, const double* lon,
                          const double* lat, const double* p, double* out, int64_t n,
                          cudaStream_t st);
template <class Rec>
cudaError_t launch_locate(const MetView<Rec>& m, int fast, const double* lon, const double* lat,
                          const double* p, int32_t* out, int64_t n, cudaStream_t st);
cudaError_t launch_philox_kat(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int n,
                              cudaStream_t st);
cudaError_t launch_iota(uint32_t* ids, int64_t offset, int64_t count, int64_t first,
                        cudaStream_t st);
cudaError_t launch_fill(double* x, int64_t n, double v, cudaStream_t st);

cudaError_t launch_grid_counts(const double* lon, const double* lat, int64_t start, int64_t n,
                               int nx, int ny, unsigned long long* counts, int sms,
                               cudaStream_t st);
cudaError_t group_stats(const double* lon, const double* lat, const double* p, const double* qrow,
                        const uint32_t* ids, int64_t qbase, int64_t start, int64_t n, int64_t max_groups, void* ws,
                        size_t ws_bytes, size_t* ws_need, int* bad_dev, int64_t* ngroups_out,
                        uint32_t* gid_out, int64_t* count_out, double* mean_out, double* std_out,
                        cudaStream_t st);

template <class Rec>
cudaError_t launch_step(const StepArgs<Rec>& a, cudaStream_t st);
bool perm_capable(uint32_t modules, uint32_t flags, int rng_mode);

cudaError_t sort_pairs(void* temp, size_t& temp_bytes, const uint32_t* keys_in,
                       uint32_t* keys_out, const uint32_t* vals_in, uint32_t* vals_out,
                       int64_t n, int end_bit, cudaStream_t st);

}  // namespace lt
