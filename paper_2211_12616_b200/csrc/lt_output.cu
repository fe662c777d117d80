// lt_output.cu — output-side statistics on the device:
//   * grid counts   output.py:28-44 (write_grid): particles per lon/lat bin;
//   * group stats   output.py:47-64 (write_ens): count, mean, std of lon,
//                   lat, p per group id taken from one quantity slot.
// Both reduce the shard in HBM and return a few KB, instead of copying the
// whole ensemble back for a host loop (write_atm is a per-particle Python
// loop, unusable at 1e8 particles).
#include <cub/cub.cuh>

#include "lt_kernels.cuh"

namespace lt {

// output.py:35-36: ix = clip(floor((lon + 180) / wx), 0, nx - 1) (same for lat)
__device__ __forceinline__ int grid_bin(double x, double off, double w, int n) {
  const double f = floor((x + off) / w);
  if (!(f >= 0.0)) return 0;  // also NaN -> 0 (numpy: int64 min, clipped to 0)
  return f > static_cast<double>(n - 1) ? n - 1 : static_cast<int>(f);
}

// block-privatised histogram in shared memory, flushed with one atomic per bin
__global__ void grid_count_shared_kernel(const double* lon, const double* lat, int64_t start,
                                         int64_t n, int nx, int ny, double wx, double wy,
                                         unsigned long long* counts) {
  extern __shared__ unsigned int bins[];
  const int nb = nx * ny;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) bins[b] = 0u;
  __syncthreads();
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ix = grid_bin(lon[start + t], 180.0, wx, nx);
    const int iy = grid_bin(lat[start + t], 90.0, wy, ny);
    atomicAdd(&bins[ix * ny + iy], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (bins[b]) atomicAdd(&counts[b], static_cast<unsigned long long>(bins[b]));
}

__global__ void grid_count_global_kernel(const double* lon, const double* lat, int64_t start,
                                         int64_t n, int nx, int ny, double wx, double wy,
                                         unsigned long long* counts) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ix = grid_bin(lon[start + t], 180.0, wx, nx);
    const int iy = grid_bin(lat[start + t], 90.0, wy, ny);
    atomicAdd(&counts[static_cast<int64_t>(ix) * ny + iy], 1ull);
  }
}

cudaError_t launch_grid_counts(const double* lon, const double* lat, int64_t start, int64_t n,
                               int nx, int ny, unsigned long long* counts, int sms,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const double wx = 360.0 / nx, wy = 180.0 / ny;  // output.py:34
  const size_t shmem = sizeof(unsigned int) * static_cast<size_t>(nx) * ny;
  int64_t g = (n + 255) / 256;
  if (shmem <= 48 * 1024) {
    if (g > 4 * sms) g = 4 * sms;
    grid_count_shared_kernel<<<static_cast<unsigned>(g), 256, shmem, st>>>(lon, lat, start, n, nx, ny,
                                                                          wx, wy, counts);
  } else {
    if (g > 64 * sms) g = 64 * sms;
    grid_count_global_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(lon, lat, start, n, nx, ny,
                                                                      wx, wy, counts);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- group stats
//
// output.py:52-63: gid = int64(q[slot]) (truncation), must be >= 0; per
// group (ascending) count and mean/std (ddof 0) of lon, lat, p.  Device
// plan: stable radix sort of (gid, slot) pairs, run-length encode, gather
// the three fields in sorted order, segmented sums for the means, then a
// second segmented pass over (x - mean)^2 (numpy's two-pass std).  CUB's
// reductions use a fixed tree, so results are reproducible run to run.

// key = (group id << 32) | particle id: groups ascending, and inside a group
// particles in id order whatever the store's (box-sorted) slot order
__global__ void group_keys_kernel(const double* qrow, const uint32_t* ids, int64_t qbase,
                                  int64_t start, int64_t n, uint64_t* keys, uint32_t* vals,
                                  int* bad) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // qbase >= 0: the q rows are in particle (home) order
    const int64_t qi = qbase >= 0 ? static_cast<int64_t>(ids[start + t]) - qbase : start + t;
    const double g = trunc(qrow[qi]);
    uint64_t gid = 0;
    if (!(g >= 0.0)) *bad = 1;
    else if (g > 4294967295.0) *bad = 2;
    else gid = static_cast<uint64_t>(g);
    const uint64_t id = ids ? ids[start + t] : static_cast<uint64_t>(start + t);
    keys[t] = (gid << 32) | id;
    vals[t] = static_cast<uint32_t>(t);
  }
}

__global__ void high_words_kernel(const uint64_t* keys, int64_t n, uint32_t* out) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[t] = static_cast<uint32_t>(keys[t] >> 32);
}

__global__ void gather3_kernel(const double* a, const double* b, const double* c, int64_t start,
                               const uint32_t* perm, int64_t n, double* out) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = start + perm[t];
    out[t] = a[s];
    out[n + t] = b[s];
    out[2 * n + t] = c[s];
  }
}

// element t of field f minus its group mean, squared; run id from the
// sorted-order offsets by binary search
__global__ void sqdev_kernel(const double* x, const int64_t* offsets, const double* means,
                             int ngroups, int64_t n, double* out) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = ngroups;  // last run with offsets[run] <= t
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (offsets[mid] <= t) lo = mid; else hi = mid;
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double d = x[f * n + t] - means[f * ngroups + lo];
      out[f * n + t] = d * d;
    }
  }
}

__global__ void finish_means_kernel(const double* sums, const int64_t* counts, int ngroups,
                                    double* means) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < 3 * ngroups; g += gridDim.x * blockDim.x)
    means[g] = sums[g] / static_cast<double>(counts[g % ngroups]);
}

static int grid_n(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

// Everything temporary is carved from one device workspace (call once with
// ws = null for the size).  *ngroups_out > max_groups means the result
// arrays were too small and nothing was written.
cudaError_t group_stats(const double* lon, const double* lat, const double* p, const double* qrow,
                        const uint32_t* ids, int64_t qbase, int64_t start, int64_t n, int64_t max_groups, void* ws, size_t ws_bytes,
                        size_t* ws_need, int* bad_dev, int64_t* ngroups_out, uint32_t* gid_out,
                        int64_t* count_out, double* mean_out, double* std_out, cudaStream_t st) {
  // layout: keys_in, keys_out (u64 n) | vals_in, vals_out, gids (u32 n) | fields 3n f64 |
  //         sq 3n f64 | uniq u32 G | counts i64 G | offsets i64 G+1 | sums 3G | means 3G | nruns
  //         | cub temp
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int64_t G = max_groups;
  size_t off = 0;
  const size_t o_keys = off; off = align(off + 2 * sizeof(uint64_t) * n);
  const size_t o_vals = off; off = align(off + 3 * sizeof(uint32_t) * n);
  const size_t o_fields = off; off = align(off + 3 * sizeof(double) * n);
  const size_t o_sq = off; off = align(off + 3 * sizeof(double) * n);
  // run-length outputs can hold up to n runs before the count is known
  const size_t o_uniq = off; off = align(off + sizeof(uint32_t) * n);
  const size_t o_cnt = off; off = align(off + sizeof(int64_t) * (n + 1));
  const size_t o_offs = off; off = align(off + sizeof(int64_t) * (n + 1));
  const size_t o_sums = off; off = align(off + 3 * sizeof(double) * G);
  const size_t o_means = off; off = align(off + 3 * sizeof(double) * G);
  const size_t o_nruns = off; off = align(off + sizeof(int64_t));
  // CUB temp requirement: max over the calls below
  size_t t_sort = 0, t_rle = 0, t_scan = 0, t_seg = 0;
  uint32_t* dk = nullptr;
  uint64_t* dk64 = nullptr;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, dk64, dk64, dk, dk, static_cast<int>(n), 0, 64, st);
  cub::DeviceRunLengthEncode::Encode(nullptr, t_rle, dk, dk, static_cast<int64_t*>(nullptr),
                                     static_cast<int64_t*>(nullptr), static_cast<int>(n), st);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, static_cast<int64_t*>(nullptr),
                                static_cast<int64_t*>(nullptr), static_cast<int>(n + 1), st);
  cub::DeviceSegmentedReduce::Sum(nullptr, t_seg, static_cast<double*>(nullptr),
                                  static_cast<double*>(nullptr), static_cast<int>(std::max<int64_t>(G, 1)),
                                  static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr), st);
  const size_t t_need = std::max(std::max(t_sort, t_rle), std::max(t_scan, t_seg));
  const size_t o_tmp = off; off = align(off + t_need);
  *ws_need = off;
  if (!ws || ws_bytes < off) return cudaSuccess;  // size query

  char* base = static_cast<char*>(ws);
  uint64_t* keys_in = reinterpret_cast<uint64_t*>(base + o_keys);
  uint64_t* keys_out = keys_in + n;
  uint32_t* vals_in = reinterpret_cast<uint32_t*>(base + o_vals);
  uint32_t* vals_out = vals_in + n;
  uint32_t* gids = vals_out + n;
  double* fields = reinterpret_cast<double*>(base + o_fields);
  double* sq = reinterpret_cast<double*>(base + o_sq);
  uint32_t* uniq = reinterpret_cast<uint32_t*>(base + o_uniq);
  int64_t* cnt = reinterpret_cast<int64_t*>(base + o_cnt);
  int64_t* offs = reinterpret_cast<int64_t*>(base + o_offs);
  double* sums = reinterpret_cast<double*>(base + o_sums);
  double* means = reinterpret_cast<double*>(base + o_means);
  int64_t* nruns = reinterpret_cast<int64_t*>(base + o_nruns);
  void* tmp = base + o_tmp;
  size_t tb = t_need;
  cudaError_t e;

  group_keys_kernel<<<grid_n(n), 256, 0, st>>>(qrow, ids, qbase, start, n, keys_in, vals_in, bad_dev);
  if ((e = cub::DeviceRadixSort::SortPairs(tmp, tb, keys_in, keys_out, vals_in, vals_out,
                                           static_cast<int>(n), 0, 64, st))) return e;
  high_words_kernel<<<grid_n(n), 256, 0, st>>>(keys_out, n, gids);
  tb = t_need;
  if ((e = cub::DeviceRunLengthEncode::Encode(tmp, tb, gids, uniq, cnt, nruns,
                                              static_cast<int>(n), st))) return e;
  int64_t ng = 0;
  if ((e = cudaMemcpyAsync(&ng, nruns, sizeof ng, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  *ngroups_out = ng;
  if (ng > G) return cudaSuccess;  // caller re-sizes
  // offsets[g] = sum of counts before g; offsets[ng] = n
  if ((e = cudaMemsetAsync(cnt + ng, 0, sizeof(int64_t), st))) return e;
  tb = t_need;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, offs, static_cast<int>(ng + 1), st))) return e;
  gather3_kernel<<<grid_n(n), 256, 0, st>>>(lon, lat, p, start, vals_out, n, fields);
  for (int f = 0; f < 3; ++f) {
    tb = t_need;
    if ((e = cub::DeviceSegmentedReduce::Sum(tmp, tb, fields + f * n, sums + f * ng,
                                             static_cast<int>(ng), offs, offs + 1, st)))
      return e;
  }
  finish_means_kernel<<<grid_n(3 * ng), 256, 0, st>>>(sums, cnt, static_cast<int>(ng), means);
  sqdev_kernel<<<grid_n(n), 256, 0, st>>>(fields, offs, means, static_cast<int>(ng), n, sq);
  for (int f = 0; f < 3; ++f) {
    tb = t_need;
    if ((e = cub::DeviceSegmentedReduce::Sum(tmp, tb, sq + f * n, sums + f * ng,
                                             static_cast<int>(ng), offs, offs + 1, st)))
      return e;
  }
  finish_means_kernel<<<grid_n(3 * ng), 256, 0, st>>>(sums, cnt, static_cast<int>(ng), sums);
  if ((e = cudaGetLastError())) return e;
  // results to the host: gid, count, mean[3][ng], var[3][ng] (std on the host)
  if ((e = cudaMemcpyAsync(gid_out, uniq, sizeof(uint32_t) * ng, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaMemcpyAsync(count_out, cnt, sizeof(int64_t) * ng, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaMemcpyAsync(mean_out, means, 3 * sizeof(double) * ng, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaMemcpyAsync(std_out, sums, 3 * sizeof(double) * ng, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  for (int64_t k = 0; k < 3 * ng; ++k) std_out[k] = sqrt(std_out[k]);
  return cudaSuccess;
}

}  // namespace lt
