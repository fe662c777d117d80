// lt_kernels.cu — kernels other than the step: met packing, random-batch
// fill, box keys for the sort, SoA permutation and ordered copies.
#include "lt_kernels.cuh"

namespace lt {

// Pack (nx_src, ny, nz) field arrays into node-pair records (u,v,w,T at k
// and k+1 per (i,j,k), k < nz-1).  With close_lon the destination has one
// more longitude column, a copy of column 0 (ingest.py:195-207).
template <class Src, class Rec>
__global__ void pack_fields_kernel(Rec* out, const Src* u, const Src* v, const Src* w,
                                   const Src* T, int nx, int ny, int nz, int nx_src) {
  const int64_t nrec = static_cast<int64_t>(nx) * ny * (nz - 1);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nrec;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(r % (nz - 1));
    const int64_t col = r / (nz - 1);
    const int j = static_cast<int>(col % ny);
    int i = static_cast<int>(col / ny);
    if (i >= nx_src) i -= nx_src;
    const int64_t b = (static_cast<int64_t>(i) * ny + j) * nz + k;
    Rec rec;
    store_node(rec, 0, u[b], v[b], w[b], T[b]);
    store_node(rec, 1, u[b + 1], v[b + 1], w[b + 1], T[b + 1]);
    out[r] = rec;
  }
}

template <class Rec>
__global__ void pack_nodes_kernel(Rec* out, const float4* nodes, int nx, int ny, int nz,
                                  int nx_src) {
  const int64_t nrec = static_cast<int64_t>(nx) * ny * (nz - 1);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < nrec;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(r % (nz - 1));
    const int64_t col = r / (nz - 1);
    const int j = static_cast<int>(col % ny);
    int i = static_cast<int>(col / ny);
    if (i >= nx_src) i -= nx_src;
    const int64_t b = (static_cast<int64_t>(i) * ny + j) * nz + k;
    const float4 n0 = nodes[b], n1 = nodes[b + 1];
    Rec rec;
    store_node(rec, 0, n0.x, n0.y, n0.z, n0.w);
    store_node(rec, 1, n1.x, n1.y, n1.z, n1.w);
    out[r] = rec;
  }
}

// rng.py:156-181: fill the RandomBatch of [start, end).  Counter and Philox
// draws are keyed by the particle's global index: ids[s] when the store
// holds a shard (or a sorted layout), else the slot s itself.  Faithful
// draws walk the device stream from the range start (rng.py:105-126).
__global__ void rng_fill_kernel(int mode, uint64_t seed_or_state, int64_t step, int64_t start,
                                int64_t end, const uint32_t* ids, double* conv, double* turb,
                                double* meso) {
  for (int64_t s = start + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < end;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double c, t[3], m[3];
    const uint64_t gid = ids ? static_cast<uint64_t>(ids[s]) : static_cast<uint64_t>(s);
    if (mode == RNG_COUNTER) {
      c = to_unit(counter_word(seed_or_state, step, gid, 0, 0));
      counter_normals(seed_or_state, step, gid, 1, t);
      counter_normals(seed_or_state, step, gid, 2, m);
    } else if (mode == RNG_FAITHFUL) {
      faithful_draws(seed_or_state, static_cast<uint64_t>(s - start), c, t, m);
    } else {
      philox_draws(seed_or_state, step, gid, c, t, m);
    }
    conv[s] = c;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      turb[3 * s + k] = t[k];
      meso[3 * s + k] = m[k];
    }
  }
}

// The mesoscale spreads of every met0 cell (sigma_u, sigma_v, sigma_w of
// its eight corners, physics.py:168-176) with the exact kernels' own code
// (gather + corner_std, numpy's pairwise order in fp64): the step kernels
// then read one 32-byte entry per particle instead of gathering the four
// corner records and reducing them.  Identical values, computed once per
// met0 snapshot instead of once per particle and step.  Cells on the last
// lon/lat row are never a corner-000 cell (locate clips to n - 2): zeros.
template <class Rec>
__global__ void spread_table_kernel(const __grid_constant__ MetView<Rec> m, int nx, double4* out) {
  const uint32_t dcol = static_cast<uint32_t>(m.nz - 1);
  const uint32_t nrec = static_cast<uint32_t>(nx) * m.ny * dcol;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
    const uint32_t col = r / dcol;
    const uint32_t i = col / m.ny, j = col - i * m.ny;
    double4 o = make_double4(0.0, 0.0, 0.0, 0.0);
    if (i + 1 < static_cast<uint32_t>(nx) && j + 1 < static_cast<uint32_t>(m.ny)) {
      Corners<Rec> q;
      gather(m.s0, m, r, q, 7);
      o.x = corner_std(q, 0);
      o.y = corner_std(q, 1);
      o.z = corner_std(q, 2);
    }
    out[r] = o;
  }
}

// Box keys from the fast kernels' cell lookup: it returns searchsorted's
// cells bit for bit (near-node guesses are settled exactly, lt_device.cuh),
// so the keys — and the stable sort's permutation — are the oracle's
// box_keys, at a fraction of the fp64 bracketing's cost.  G = 2 on a
// geographic grid (computed lon/lat cells, log-guessed levels), 1 elsewhere.
// kzone[0] / kzone[1] collect the smallest and largest level box (the
// occupied level range, for compress_keys_kernel)
template <class Rec, int G>
__global__ void box_key_kernel(const __grid_constant__ MetView<Rec> m, const double* lon, const double* lat,
                               const double* p, int64_t start, int64_t n, uint32_t* keys,
                               uint32_t* vals, int morton, unsigned int* kzone) {
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = start + t;
    float fx, fy, fz;
    const int i = locate_h<G>(m.lon, __ldcs(lon + s), fx);
    const int j = locate_h<G>(m.lat, __ldcs(lat + s), fy);
    const int k = m.nz - 2 - locate_v<G>(m.lev, __ldcs(p + s), fz, m.levc);
    const uint32_t r00 = (static_cast<uint32_t>(i) * m.ny + j) * (m.nz - 1) + k;
    keys[t] = morton ? box_key_morton(i, j, k, m.nz) : r00;
    vals[t] = static_cast<uint32_t>(t);
    const uint32_t kb = static_cast<uint32_t>(k) / LT_BOX_ZDIV;
    kmin = min(kmin, kb);
    kmax = max(kmax, kb);
  }
  if (kzone) {
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(kzone, kmin);
      atomicMax(kzone + 1, kmax);
    }
  }
}

// The same order with fewer key bits: Morton column codes are sparse (0.25
// deg: 2.5e6 codes for 1.04e6 columns) and most level boxes hold no
// particle, so key = column * nlev + kb becomes rank[column] * nocc +
// (kb - kmin) — strictly monotone on the keys present, hence the same
// stable permutation, in 24 bits instead of 28 at cfg3 (three onesweep
// passes instead of four)
__global__ void compress_keys_kernel(uint32_t* keys, int64_t n, const uint32_t* __restrict__ rank,
                                     uint32_t nlev, uint32_t kmin, uint32_t nocc) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t key = keys[t];
    const uint32_t col = key / nlev;
    keys[t] = __ldg(rank + col) * nocc + (key - col * nlev - kmin);
  }
}

template <class T>
__global__ void permute_kernel(T* dst, const T* src, const uint32_t* perm, int64_t start,
                               int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[start + t] = src[start + perm[t]];
}

// gather up to kRowSet rows through one permutation (perm read once per particle)
__global__ void permute_rows_kernel(RowSet r, const uint32_t* perm, int64_t start, int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t from = start + perm[t];
    double v[kRowSet];
#pragma unroll
    for (int k = 0; k < kRowSet; ++k)
      if (k < r.n) v[k] = __ldg(r.src[k] + from);
#pragma unroll
    for (int k = 0; k < kRowSet; ++k)
      if (k < r.n) r.dst[k][start + t] = v[k];
  }
}

// scatter a sorted slice into original order: out[id - first] = in[s]
template <class T>
__global__ void unsort_kernel(T* out, const T* in, const uint32_t* ids, int64_t offset,
                              int64_t count, int64_t first_id, int* bad, int stride_in) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t dst = static_cast<int64_t>(ids[offset + t]) - first_id;
    if (dst < 0 || dst >= count) { *bad = 1; continue; }
    for (int c = 0; c < stride_in; ++c) out[dst * stride_in + c] = in[(offset + t) * stride_in + c];
  }
}

// gather original order into the sorted slice: out[s] = in[id - first]
template <class T>
__global__ void resort_kernel(T* out, const T* in, const uint32_t* ids, int64_t offset,
                              int64_t count, int64_t first_id, int* bad, int stride_in) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t src = static_cast<int64_t>(ids[offset + t]) - first_id;
    if (src < 0 || src >= count) { *bad = 1; continue; }
    for (int c = 0; c < stride_in; ++c) out[(offset + t) * stride_in + c] = in[src * stride_in + c];
  }
}

// physics.py:69-79 as a standalone call (interpolate_met at arbitrary points)
template <class Rec>
__global__ void sample_kernel(MetView<Rec> m, const double* t, const double* lon, const double* lat,
                              const double* p, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v[4];
    sample(m, t[i], lon[i], lat[i], p[i], 15, v);
#pragma unroll
    for (int f = 0; f < 4; ++f) out[f * n + i] = v[f];
  }
}

// physics.py:31-47 cell lookup alone, for the cell audit (lt_locate_cells):
// FAST = 0 the exact bracketing every exact kernel uses (cell_of), 1 / 2
// the fast kernels' lookups (cell_fast<G>) on any / a geographic grid
template <class Rec, int FAST>
__global__ void locate_kernel(MetView<Rec> m, const double* lon, const double* lat,
                              const double* p, int32_t* out, int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int i, j, k;
    if constexpr (FAST == 0) {
      const Cell c = cell_of(m, lon[t], lat[t], p[t]);
      i = c.i; j = c.j; k = c.k;
    } else {
      const CellF c = cell_fast<FAST>(m, lon[t], lat[t], p[t]);
      i = static_cast<int>(c.col / m.ny);
      j = static_cast<int>(c.col % m.ny);
      k = static_cast<int>(c.r00 - c.col * static_cast<uint32_t>(m.nz - 1));
    }
    out[t] = i;
    out[n + t] = j;
    out[2 * n + t] = k;
  }
}

__global__ void iota_kernel(uint32_t* ids, int64_t offset, int64_t count, int64_t first) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ids[offset + t] = static_cast<uint32_t>(first + t);
}

__global__ void fill_kernel(double* x, int64_t n, double v) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[t] = v;
}

// ---------------------------------------------------------------- launchers

static int grid_for(int64_t n, int block = 256) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return static_cast<int>(g);
}

template <class Rec>
cudaError_t launch_spread_table(const MetView<Rec>& m, int nx, double* out, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(nx) * m.ny * (m.nz - 1);
  spread_table_kernel<Rec><<<grid_for(n), 256, 0, st>>>(m, nx, reinterpret_cast<double4*>(out));
  return cudaGetLastError();
}
template cudaError_t launch_spread_table<RecF>(const MetView<RecF>&, int, double*, cudaStream_t);
template cudaError_t launch_spread_table<RecD>(const MetView<RecD>&, int, double*, cudaStream_t);


template <class Src, class Rec>
cudaError_t launch_pack_fields(Rec* out, const Src* u, const Src* v, const Src* w, const Src* T,
                               int nx, int ny, int nz, int nx_src, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(nx) * ny * (nz - 1);
  pack_fields_kernel<Src, Rec><<<grid_for(n), 256, 0, st>>>(out, u, v, w, T, nx, ny, nz, nx_src);
  return cudaGetLastError();
}
template cudaError_t launch_pack_fields<float, RecF>(RecF*, const float*, const float*, const float*, const float*, int, int, int, int, cudaStream_t);
template cudaError_t launch_pack_fields<double, RecF>(RecF*, const double*, const double*, const double*, const double*, int, int, int, int, cudaStream_t);
template cudaError_t launch_pack_fields<float, RecD>(RecD*, const float*, const float*, const float*, const float*, int, int, int, int, cudaStream_t);
template cudaError_t launch_pack_fields<double, RecD>(RecD*, const double*, const double*, const double*, const double*, int, int, int, int, cudaStream_t);

template <class Rec>
cudaError_t launch_pack_nodes(Rec* out, const float4* nodes, int nx, int ny, int nz, int nx_src,
                              cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(nx) * ny * (nz - 1);
  pack_nodes_kernel<Rec><<<grid_for(n), 256, 0, st>>>(out, nodes, nx, ny, nz, nx_src);
  return cudaGetLastError();
}
template cudaError_t launch_pack_nodes<RecF>(RecF*, const float4*, int, int, int, int, cudaStream_t);
template cudaError_t launch_pack_nodes<RecD>(RecD*, const float4*, int, int, int, int, cudaStream_t);

cudaError_t launch_rng_fill(int mode, uint64_t seed, int64_t step, int64_t start, int64_t end,
                            const uint32_t* ids, double* conv, double* turb, double* meso,
                            cudaStream_t st) {
  if (end <= start) return cudaSuccess;
  rng_fill_kernel<<<grid_for(end - start), 256, 0, st>>>(mode, seed, step, start, end, ids, conv,
                                                         turb, meso);
  return cudaGetLastError();
}

// the in-kernel generator's block function on explicit (counter, key)
// pairs: the known-answer hook for Philox4x32-10 (Random123's kat_vectors)
__global__ void philox_kat_kernel(const uint4* ctr, const uint2* key, uint4* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // both forms of the block function: a disagreement poisons the answer
  uint32_t rk[20];
  philox_round_keys(key[i].x, key[i].y, rk);
  const uint4 a = philox(ctr[i], key[i]), b = philox_rk(ctr[i], rk);
  const bool same = a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
  out[i] = same ? a : make_uint4(~a.x, ~a.y, ~a.z, ~a.w);
}

cudaError_t launch_philox_kat(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int n,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  philox_kat_kernel<<<(n + 127) / 128, 128, 0, st>>>(reinterpret_cast<const uint4*>(ctr),
                                                     reinterpret_cast<const uint2*>(key),
                                                     reinterpret_cast<uint4*>(out), n);
  return cudaGetLastError();
}

template <class Rec>
cudaError_t launch_box_keys(const MetView<Rec>& m, const double* lon, const double* lat,
                            const double* p, int64_t start, int64_t n, uint32_t* keys,
                            uint32_t* vals, int morton, unsigned int* kzone, cudaStream_t st) {
  const bool geo = m.lon.uniform && m.lat.uniform && !m.lev.uniform && m.lev.logscale &&
                   m.lev.n - 1 <= kLevCap;
  if (geo) box_key_kernel<Rec, 2><<<grid_for(n), 256, 0, st>>>(m, lon, lat, p, start, n, keys, vals, morton, kzone);
  else box_key_kernel<Rec, 1><<<grid_for(n), 256, 0, st>>>(m, lon, lat, p, start, n, keys, vals, morton, kzone);
  return cudaGetLastError();
}

cudaError_t launch_compress_keys(uint32_t* keys, int64_t n, const uint32_t* rank, uint32_t nlev,
                                 uint32_t kmin, uint32_t nocc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  compress_keys_kernel<<<grid_for(n), 256, 0, st>>>(keys, n, rank, nlev, kmin, nocc);
  return cudaGetLastError();
}
template cudaError_t launch_box_keys<RecF>(const MetView<RecF>&, const double*, const double*, const double*, int64_t, int64_t, uint32_t*, uint32_t*, int, unsigned int*, cudaStream_t);
template cudaError_t launch_box_keys<RecD>(const MetView<RecD>&, const double*, const double*, const double*, int64_t, int64_t, uint32_t*, uint32_t*, int, unsigned int*, cudaStream_t);

template <class T>
cudaError_t launch_permute(T* dst, const T* src, const uint32_t* perm, int64_t start, int64_t n,
                           cudaStream_t st) {
  permute_kernel<T><<<grid_for(n), 256, 0, st>>>(dst, src, perm, start, n);
  return cudaGetLastError();
}
template cudaError_t launch_permute<double>(double*, const double*, const uint32_t*, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_permute<uint32_t>(uint32_t*, const uint32_t*, const uint32_t*, int64_t, int64_t, cudaStream_t);

cudaError_t launch_permute_rows(const RowSet& r, const uint32_t* perm, int64_t start, int64_t n,
                               cudaStream_t st) {
  if (n <= 0 || r.n <= 0) return cudaSuccess;
  permute_rows_kernel<<<grid_for(n), 256, 0, st>>>(r, perm, start, n);
  return cudaGetLastError();
}

cudaError_t launch_unsort(double* out, const double* in, const uint32_t* ids, int64_t offset,
                          int64_t count, int64_t first_id, int* bad, int stride, cudaStream_t st) {
  unsort_kernel<double><<<grid_for(count), 256, 0, st>>>(out, in, ids, offset, count, first_id, bad, stride);
  return cudaGetLastError();
}
cudaError_t launch_resort(double* out, const double* in, const uint32_t* ids, int64_t offset,
                          int64_t count, int64_t first_id, int* bad, int stride, cudaStream_t st) {
  resort_kernel<double><<<grid_for(count), 256, 0, st>>>(out, in, ids, offset, count, first_id, bad, stride);
  return cudaGetLastError();
}
template <class Rec>
cudaError_t launch_sample(const MetView<Rec>& m, const double* t, const double* lon,
                          const double* lat, const double* p, double* out, int64_t n,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  sample_kernel<Rec><<<grid_for(n), 256, 0, st>>>(m, t, lon, lat, p, out, n);
  return cudaGetLastError();
}
template cudaError_t launch_sample<RecF>(const MetView<RecF>&, const double*, const double*, const double*, const double*, double*, int64_t, cudaStream_t);
template cudaError_t launch_sample<RecD>(const MetView<RecD>&, const double*, const double*, const double*, const double*, double*, int64_t, cudaStream_t);

template <class Rec>
cudaError_t launch_locate(const MetView<Rec>& m, int fast, const double* lon, const double* lat,
                          const double* p, int32_t* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (fast == 0) {
    locate_kernel<Rec, 0><<<grid_for(n), 256, 0, st>>>(m, lon, lat, p, out, n);
  } else if constexpr (sizeof(Rec) == sizeof(RecF)) {
    // the same dispatch as launch_step: geographic grids get the G = 2 lookups
    const bool geo = m.lon.uniform && m.lat.uniform && !m.lev.uniform && m.lev.logscale &&
                   m.lev.n - 1 <= kLevCap;
    if (geo) locate_kernel<Rec, 2><<<grid_for(n), 256, 0, st>>>(m, lon, lat, p, out, n);
    else locate_kernel<Rec, 1><<<grid_for(n), 256, 0, st>>>(m, lon, lat, p, out, n);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template cudaError_t launch_locate<RecF>(const MetView<RecF>&, int, const double*, const double*, const double*, int32_t*, int64_t, cudaStream_t);
template cudaError_t launch_locate<RecD>(const MetView<RecD>&, int, const double*, const double*, const double*, int32_t*, int64_t, cudaStream_t);

cudaError_t launch_iota(uint32_t* ids, int64_t offset, int64_t count, int64_t first, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  iota_kernel<<<grid_for(count), 256, 0, st>>>(ids, offset, count, first);
  return cudaGetLastError();
}
cudaError_t launch_fill(double* x, int64_t n, double v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fill_kernel<<<grid_for(n), 256, 0, st>>>(x, n, v);
  return cudaGetLastError();
}

}  // namespace lt
