// lt_capi.cu — the extern "C" boundary (include/lagtrans_b200.h).
//
// A context is one GPU's data region: the SoA particle store, up to three
// met snapshot slots on one grid, the climatology tables, two streams
// (compute, copy) and the scratch used by the sort and ordered copies.
// The reference equivalent is one DevicePool worker's ModelImage
// (device_runtime.py:58-69,165-230).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/lagtrans_b200.h"
#include "lt_comm.cuh"
#include "lt_kernels.cuh"

using namespace lt;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(e_ == cudaErrorMemoryAllocation ? LT_ERR_NOMEM : LT_ERR_CUDA,      \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

struct AxisHost {
  double* dev = nullptr;
  double* rinv = nullptr;  // per cell RN(1 / (x[i+1] - x[i])) (exact path: Markstein quotient)
  double2* cell = nullptr;  // per cell {x[i], fp32 1/(x[i+1]-x[i]) in the low word}
  double lo = 0.0, hi = 0.0;
  int n = 0;
  int logscale = 0;
  float g0 = 0.f, ginv = 0.f;
  int uniform = 0;
  double dinv = 0.0, dorg = 0.0;
  std::vector<double2> host_cell;  // host copy of `cell` (the level table in kernel parameters)
};

struct Slot {
  void* rec = nullptr;  // RecF[] or RecD[]
  double t_met = 0.0;
  bool valid = false;
  cudaEvent_t ready = nullptr;  // recorded on the copy stream after packing
};

}  // namespace

struct lt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t copy = nullptr;    // met streaming, host-path H2D
  cudaStream_t d2h = nullptr;     // host-path D2H
  std::vector<cudaEvent_t> ring_ev;  // host-path chunk events (3 per ring slot)
  std::vector<cudaEvent_t> host_ev;  // host-path: chunk k's results are back in host memory
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  cudaEvent_t compute_mark = nullptr;  // last compute-stream work touching met slots
  bool marked = false;
  bool timing = false;
  bool timed_once = false;

  // particles
  int64_t cap = 0;
  int32_t nq = 0;
  double *time = nullptr, *p = nullptr, *zeta = nullptr, *lon = nullptr, *lat = nullptr;
  double *q = nullptr, *iso_var = nullptr, *dt = nullptr;
  double* uvwp[3] = {nullptr, nullptr, nullptr};  // separate rows: the sort swaps row pointers
  double *rnd_conv = nullptr, *rnd_turb = nullptr, *rnd_meso = nullptr;
  uint32_t* ids = nullptr;
  uint32_t home_mask = 0;        // LT_HOME_* row groups kept in particle order
  int64_t home_base = 0;         // first id of the last lt_ids_reset (offset 0)
  int64_t home_n = 0;            // particles [0, home_n) carry home-order ids
  double* scratch = nullptr;     // cap doubles (ordered copies)
  double* pool[8] = {};          // cap doubles each: gather targets (swapped with rows)
  uint32_t* ids_alt = nullptr;   // cap: the id row a fused sort-and-step writes
  bool pending = false;          // a box-sort permutation is waiting to be applied
  int64_t pend_start = 0, pend_n = 0;
  uint32_t* sort_buf = nullptr;  // 4 * cap (keys in/out, vals in/out)
  uint32_t* col_rank = nullptr;  // dense rank of each Morton column code (key compression)
  int64_t col_rank_n = 0;        // its length (0: not built for the current grid)
  uint32_t col_count = 0;        // number of columns (nx * ny)
  // the occupied level-box range of the last sort that computed its keys
  // (the window of keys written by LT_RUN_SORT_KEYS launches)
  bool zone_known = false;
  uint32_t zone_min = 0, zone_max = 0;
  // API calls on the context (check_ctx); keys written by the launch of call
  // sk_call serve an lt_sort_by_box of [sk_start, sk_end) that is call sk_call + 1
  uint64_t calls = 0, sk_call = ~0ull;
  int64_t sk_start = 0, sk_end = 0;
  uint32_t sk_nocc = 1;
  int64_t n_sorts = 0, n_sorts_fused = 0;  // lt_sort_info
  void* cub_temp = nullptr;
  size_t cub_bytes = 0;
  unsigned long long* counters = nullptr;  // [0] iso_nonconverged, [8, 8 + CK_N) module cycles
  int* bad = nullptr;

  // met
  int nx = 0, ny = 0, nz = 0, prec = 0;
  AxisHost ax_lon, ax_lat, ax_lev;
  Slot slots[3];
  int use0 = -1, use1 = -1;
  // per-cell mesoscale spreads (MetView::sig0): two tables tagged with the
  // met slot they describe — met0's, and met1's, prebuilt on the copy stream
  // while the steps run, so a rotation finds its new met0's table ready
  double* sig_buf[2] = {nullptr, nullptr};
  int sig_of[2] = {-1, -1};
  cudaEvent_t sig_ready[2] = {nullptr, nullptr};
  cudaEvent_t sig_mark = nullptr;  // compute work that may still read a table
  bool meso_seen = false;          // prebuild met1's table only once meso has run
  void* staging = nullptr;
  size_t staging_bytes = 0;
  cudaEvent_t staging_free = nullptr;

  // climatology
  AxisHost cl_lat, cl_p;
  double *hno3 = nullptr, *p_trop = nullptr;
};

namespace {

void free_dev(void* p) {
  if (p) cudaFree(p);
}

int alloc_dev(void** p, size_t bytes, const char* what) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? LT_ERR_NOMEM : LT_ERR_CUDA,
                "cudaMalloc(%s, %zu bytes): %s", what, bytes, cudaGetErrorString(e));
  }
  return LT_OK;
}

// choose the cell-guess mapping of an axis: linear in x, or in log2(x)
// (geometric pressure levels).  Only speed depends on it, never results.
int upload_axis(AxisHost& ax, const double* x, int n, cudaStream_t st) {
  if (n < 2) return fail(LT_ERR_ARG, "axis needs at least 2 nodes, got %d", n);
  for (int i = 1; i < n; ++i)
    if (!(x[i] > x[i - 1])) return fail(LT_ERR_ARG, "axis not strictly increasing at %d", i);
  auto spread = [&](auto f) {
    const double a = f(x[0]), b = f(x[n - 1]);
    double worst = 0;
    for (int i = 0; i < n; ++i) {
      const double ideal = a + (b - a) * i / (n - 1);
      worst = fmax(worst, fabs(f(x[i]) - ideal) / ((b - a) / (n - 1)));
    }
    return worst;
  };
  const double lin = spread([](double v) { return v; });
  double lg = 1e300;
  if (x[0] > 0) lg = spread([](double v) { return log2(v); });
  ax.logscale = lg < lin ? 1 : 0;
  const double a = ax.logscale ? log2(x[0]) : x[0];
  const double b = ax.logscale ? log2(x[n - 1]) : x[n - 1];
  ax.g0 = static_cast<float>(a);
  ax.ginv = static_cast<float>((n - 1) / (b - a));
  ax.lo = x[0];
  ax.hi = x[n - 1];
  ax.uniform = lin <= 1e-9 ? 1 : 0;
  ax.dinv = (n - 1) / (x[n - 1] - x[0]);
  ax.dorg = -x[0] * ax.dinv;
  if (ax.dev && ax.n != n) {
    cudaFree(ax.dev);
    cudaFree(ax.cell);
    cudaFree(ax.rinv);
    ax.dev = nullptr;
    ax.cell = nullptr;
    ax.rinv = nullptr;
  }
  ax.n = n;
  if (!ax.dev) {
    int rc = alloc_dev(reinterpret_cast<void**>(&ax.dev), sizeof(double) * n, "axis");
    if (rc) return rc;
    rc = alloc_dev(reinterpret_cast<void**>(&ax.cell), sizeof(double2) * n, "axis cells");
    if (rc) return rc;
    rc = alloc_dev(reinterpret_cast<void**>(&ax.rinv), sizeof(double) * n, "axis reciprocals");
    if (rc) return rc;
  }
  // correctly rounded reciprocal cell widths: with them the exact kernels'
  // fraction (x - x[i]) / (x[i+1] - x[i]) is one multiply and two FMAs and
  // still the correctly rounded quotient numpy computes (lt_device.cuh div_cr)
  std::vector<double> rinv(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) rinv[i] = 1.0 / (x[i + 1] - x[i]);
  CK(cudaMemcpyAsync(ax.rinv, rinv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  std::vector<double2> cell(n);
  for (int i = 0; i < n; ++i) {
    const float r = i + 1 < n ? static_cast<float>(1.0 / (x[i + 1] - x[i])) : 0.0f;
    uint32_t bits;
    std::memcpy(&bits, &r, 4);
    const uint64_t word = bits;
    cell[i].x = x[i];
    std::memcpy(&cell[i].y, &word, 8);
  }
  CK(cudaMemcpyAsync(ax.dev, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ax.cell, cell.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, st));
  ax.host_cell = cell;
  CK(cudaStreamSynchronize(st));
  return LT_OK;
}

Axis view(const AxisHost& a) {
  Axis v;
  v.x = a.dev;
  v.cell = a.cell;
  v.rinv = a.rinv;
  v.lo = a.lo;
  v.hi = a.hi;
  v.n = a.n;
  v.nm2 = a.n - 2;
  v.logscale = a.logscale;
  v.g0 = a.g0;
  v.ginv = a.ginv;
  v.uniform = a.uniform;
  v.dinv = a.dinv;
  v.dorg = a.dorg;
  return v;
}

size_t rec_bytes(const lt_ctx* c) { return c->prec == LT_MET_F64 ? sizeof(RecD) : sizeof(RecF); }
int64_t n_rec(const lt_ctx* c) { return static_cast<int64_t>(c->nx) * c->ny * (c->nz - 1); }

template <class Rec>
MetView<Rec> met_view(const lt_ctx* c) {
  MetView<Rec> m;
  m.lon = view(c->ax_lon);
  m.lat = view(c->ax_lat);
  m.lev = view(c->ax_lev);
  m.ny = c->ny;
  m.nz = c->nz;
  m.s0 = static_cast<const Rec*>(c->slots[c->use0].rec);
  m.s1 = static_cast<const Rec*>(c->slots[c->use1].rec);
  m.t0 = c->slots[c->use0].t_met;
  m.t1 = c->slots[c->use1].t_met;
  m.inv_dt = m.t1 != m.t0 ? 1.0 / (m.t1 - m.t0) : 0.0;
  m.sig0 = nullptr;
  const int ncell = c->ax_lev.n - 1;
  if (ncell <= kLevCap) std::memcpy(m.levc, c->ax_lev.host_cell.data(), sizeof(double2) * ncell);
  return m;
}

double* field_ptr(lt_ctx* c, int field, int row, int64_t* len, int* rc) {
  *rc = LT_OK;
  *len = c->cap;
  switch (field) {
    case LT_F_TIME: return c->time;
    case LT_F_P: return c->p;
    case LT_F_ZETA: return c->zeta;
    case LT_F_LON: return c->lon;
    case LT_F_LAT: return c->lat;
    case LT_F_Q:
      if (row < 0 || row >= c->nq) { *rc = fail(LT_ERR_ARG, "q row %d outside [0, %d)", row, c->nq); return nullptr; }
      return c->q + static_cast<int64_t>(row) * c->cap;
    case LT_F_UVWP:
      if (row < 0 || row >= 3) { *rc = fail(LT_ERR_ARG, "uvwp row %d outside [0, 3)", row); return nullptr; }
      return c->uvwp[row];
    case LT_F_ISO_VAR: return c->iso_var;
    case LT_F_DT: return c->dt;
    case LT_F_RND_CONV:
    case LT_F_RND_TURB:
    case LT_F_RND_MESO:
      if (!c->rnd_conv) { *rc = fail(LT_ERR_STATE, "context allocated without a random batch"); return nullptr; }
      if (field == LT_F_RND_CONV) return c->rnd_conv;
      *len = 3 * c->cap;
      return field == LT_F_RND_TURB ? c->rnd_turb : c->rnd_meso;
    default:
      *rc = fail(LT_ERR_ARG, "unknown field id %d", field);
      return nullptr;
  }
}

int check_ctx(lt_ctx* c) {
  if (!c) return fail(LT_ERR_STATE, "null context (deleted region?)");
  ++c->calls;
  CK(cudaSetDevice(c->device));
  return LT_OK;
}

// entry points that leave the particles and their slot order alone: they do
// not count as calls between a LT_RUN_SORT_KEYS launch and its sort
int check_ctx_keep(lt_ctx* c) {
  const int rc = check_ctx(c);
  if (rc == LT_OK) --c->calls;
  return rc;
}

int check_particles(lt_ctx* c) {
  if (!c->time) return fail(LT_ERR_STATE, "particle store not allocated");
  return LT_OK;
}

int ensure_scratch(lt_ctx* c) {
  if (!c->scratch)
    return alloc_dev(reinterpret_cast<void**>(&c->scratch), sizeof(double) * c->cap, "scratch");
  return LT_OK;
}

int ensure_pool(lt_ctx* c, int rows = 4) {
  for (int k = 0; k < rows; ++k)
    if (!c->pool[k])
      if (int rc = alloc_dev(reinterpret_cast<void**>(&c->pool[k]), sizeof(double) * c->cap, "sort pool"))
        return rc;
  return LT_OK;
}

int ensure_ids(lt_ctx* c) {
  if (!c->ids) {
    int rc = alloc_dev(reinterpret_cast<void**>(&c->ids), sizeof(uint32_t) * c->cap, "ids");
    if (rc) return rc;
    CK(launch_iota(c->ids, 0, c->cap, 0, c->stream));
  }
  return LT_OK;
}

}  // namespace

static int settle(lt_ctx* c);  // apply a pending box-sort permutation (below)

extern "C" {

int lt_abi_version(void) { return LT_ABI_VERSION; }

const char* lt_last_error(void) { return g_err.c_str(); }

int lt_device_count(int32_t* n) {
  int k = 0;
  cudaError_t e = cudaGetDeviceCount(&k);
  if (e != cudaSuccess) {
    *n = 0;
    return fail(LT_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *n = k;
  return LT_OK;
}

static int ctx_init(lt_ctx* c);

int lt_ctx_create(int32_t device, lt_ctx** out) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
    return fail(LT_ERR_ARG, "device_id %d out of range [0, %d)", device, n);
  CK(cudaSetDevice(device));
  lt_ctx* c = new lt_ctx();
  c->device = device;
  if (int rc = ctx_init(c)) {  // release what was created before the failure
    std::string msg = lt_last_error();
    lt_ctx_destroy(c);
    return fail(rc, "%s", msg.c_str());
  }
  *out = c;
  return LT_OK;
}

static int ctx_init(lt_ctx* c) {
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  CK(cudaEventCreate(&c->ev_start));
  CK(cudaEventCreate(&c->ev_stop));
  CK(cudaEventCreateWithFlags(&c->staging_free, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->compute_mark, cudaEventDisableTiming));
  for (auto& s : c->slots) CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
  for (auto& e : c->sig_ready) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->sig_mark, cudaEventDisableTiming));
  int rc = alloc_dev(reinterpret_cast<void**>(&c->counters), 32 * sizeof(unsigned long long), "counters");
  if (rc) return rc;
  rc = alloc_dev(reinterpret_cast<void**>(&c->bad), sizeof(int), "flag");
  if (rc) return rc;
  CK(cudaMemsetAsync(c->counters, 0, 32 * sizeof(unsigned long long), c->stream));
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

static void free_particles(lt_ctx* c) {
  for (double** p : {&c->time, &c->p, &c->zeta, &c->lon, &c->lat, &c->q, &c->uvwp[0], &c->uvwp[1], &c->uvwp[2], &c->iso_var,
                     &c->dt, &c->rnd_conv, &c->rnd_turb, &c->rnd_meso, &c->scratch}) {
    free_dev(*p);
    *p = nullptr;
  }
  free_dev(c->ids); c->ids = nullptr;
  c->home_mask = 0; c->home_base = 0; c->home_n = 0;
  for (double*& r : c->pool) { free_dev(r); r = nullptr; }
  free_dev(c->ids_alt); c->ids_alt = nullptr;
  c->pending = false;
  free_dev(c->sort_buf); c->sort_buf = nullptr;
  free_dev(c->col_rank); c->col_rank = nullptr; c->col_rank_n = 0;
  free_dev(c->cub_temp); c->cub_temp = nullptr; c->cub_bytes = 0;
  c->cap = 0;
}

int lt_ctx_destroy(lt_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  cudaError_t e1 = cudaStreamSynchronize(c->stream);
  cudaError_t e2 = cudaStreamSynchronize(c->copy);
  if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(c->d2h);
  free_particles(c);
  for (auto& s : c->slots) {
    free_dev(s.rec);
    cudaEventDestroy(s.ready);
  }
  free_dev(c->staging);
  for (AxisHost* a : {&c->ax_lon, &c->ax_lat, &c->ax_lev, &c->cl_lat, &c->cl_p}) {
    free_dev(a->dev);
    free_dev(a->cell);
    free_dev(a->rinv);
  }
  free_dev(c->hno3);
  free_dev(c->p_trop);
  free_dev(c->counters);
  free_dev(c->bad);
  cudaEventDestroy(c->ev_start);
  cudaEventDestroy(c->ev_stop);
  cudaEventDestroy(c->staging_free);
  cudaEventDestroy(c->compute_mark);
  for (int b = 0; b < 2; ++b) {
    free_dev(c->sig_buf[b]);
    cudaEventDestroy(c->sig_ready[b]);
  }
  cudaEventDestroy(c->sig_mark);
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->copy);
  cudaStreamDestroy(c->d2h);
  for (cudaEvent_t e : c->ring_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : c->host_ev) cudaEventDestroy(e);
  delete c;
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    return fail(LT_ERR_CUDA, "pending work failed before destroy: %s",
                cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  return LT_OK;
}

int lt_sync(lt_ctx* c) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->copy));
  CK(cudaStreamSynchronize(c->d2h));
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

int lt_stream(lt_ctx* c, void** s) {
  int rc = check_ctx(c);
  if (rc) return rc;
  *s = c->stream;
  return LT_OK;
}

int lt_particles_alloc(lt_ctx* c, int64_t capacity, int32_t nq, int32_t with_batch) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (capacity < 0) return fail(LT_ERR_ARG, "capacity %lld < 0", (long long)capacity);
  // particle ids and the kernels' slot arithmetic are 32-bit (2^31 particles
  // would need > 180 GB of state alone)
  if (capacity > INT32_MAX) return fail(LT_ERR_ARG, "capacity %lld > 2^31 - 1", (long long)capacity);
  if (nq < 5) return fail(LT_ERR_ARG, "nq >= 5 violated (meteo sampling needs slots 0..4)");
  CK(cudaStreamSynchronize(c->stream));
  free_particles(c);
  c->cap = capacity;
  c->nq = nq;
  const size_t b = sizeof(double) * static_cast<size_t>(capacity);
  struct { double** p; size_t mult; const char* name; } plan[] = {
      {&c->time, 1, "time"}, {&c->p, 1, "p"}, {&c->zeta, 1, "zeta"}, {&c->lon, 1, "lon"},
      {&c->lat, 1, "lat"}, {&c->q, static_cast<size_t>(nq), "q"}, {&c->uvwp[0], 1, "uvwp"},
      {&c->uvwp[1], 1, "uvwp"}, {&c->uvwp[2], 1, "uvwp"},
      {&c->iso_var, 1, "iso_var"}, {&c->dt, 1, "dt"}};
  for (auto& e : plan) {
    rc = alloc_dev(reinterpret_cast<void**>(e.p), b * e.mult, e.name);
    if (rc) { free_particles(c); return rc; }
    CK(cudaMemsetAsync(*e.p, 0, b * e.mult, c->stream));
  }
  if (with_batch) {
    struct { double** p; size_t mult; } bplan[] = {{&c->rnd_conv, 1}, {&c->rnd_turb, 3}, {&c->rnd_meso, 3}};
    for (auto& e : bplan) {
      rc = alloc_dev(reinterpret_cast<void**>(e.p), b * e.mult, "random batch");
      if (rc) { free_particles(c); return rc; }
      CK(cudaMemsetAsync(*e.p, 0, b * e.mult, c->stream));
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

int lt_field_devptr(lt_ctx* c, int32_t field, int32_t row, void** dev) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (field == LT_F_ID) {
    if ((rc = ensure_ids(c))) return rc;
    *dev = c->ids;
    return LT_OK;
  }
  int64_t len;
  double* p = field_ptr(c, field, row, &len, &rc);
  if (rc) return rc;
  *dev = p;
  return LT_OK;
}

static int slice_check(lt_ctx* c, int64_t off, int64_t cnt, int64_t len) {
  if (off < 0 || cnt < 0 || off + cnt > len)
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside field of %lld elements", (long long)off,
                (long long)(off + cnt), (long long)len);
  return LT_OK;
}

int lt_field_h2d(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt, const void* host) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (field == LT_F_ID) {
    if ((rc = ensure_ids(c)) || (rc = slice_check(c, off, cnt, c->cap))) return rc;
    if (cnt) CK(cudaMemcpyAsync(c->ids + off, host, 4 * cnt, cudaMemcpyHostToDevice, c->stream));
    return LT_OK;
  }
  int64_t len;
  double* p = field_ptr(c, field, row, &len, &rc);
  if (rc || (rc = slice_check(c, off, cnt, len))) return rc;
  if (cnt) CK(cudaMemcpyAsync(p + off, host, sizeof(double) * cnt, cudaMemcpyHostToDevice, c->stream));
  return LT_OK;
}

int lt_field_d2h(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt, void* host) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (field == LT_F_ID) {
    if ((rc = ensure_ids(c)) || (rc = slice_check(c, off, cnt, c->cap))) return rc;
    if (cnt) CK(cudaMemcpyAsync(host, c->ids + off, 4 * cnt, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return LT_OK;
  }
  int64_t len;
  double* p = field_ptr(c, field, row, &len, &rc);
  if (rc || (rc = slice_check(c, off, cnt, len))) return rc;
  if (cnt) CK(cudaMemcpyAsync(host, p + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

int lt_field_fill(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt, double value) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  int64_t len;
  double* p = field_ptr(c, field, row, &len, &rc);
  if (rc || (rc = slice_check(c, off, cnt, len))) return rc;
  CK(launch_fill(p + off, cnt, value, c->stream));
  return LT_OK;
}

int lt_ids_reset(lt_ctx* c, int64_t off, int64_t cnt, int64_t first_id) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if ((rc = ensure_ids(c)) || (rc = slice_check(c, off, cnt, c->cap))) return rc;
  if (first_id < 0 || first_id + cnt > (int64_t(1) << 32))
    return fail(LT_ERR_ARG, "particle ids must fit in 32 bits");
  CK(launch_iota(c->ids, off, cnt, first_id, c->stream));
  if (off == 0) {   // slot s now holds particle first_id + s: home order == slot order
    c->home_base = first_id;
    c->home_n = cnt;
  }
  return LT_OK;
}

// Convert row groups between slot order and particle ("home") order.  With
// ids a permutation of [home_base, home_base + home_n) over slots
// [0, home_n): slot -> home scatters out[id - base] = in[s]; home -> slot
// gathers out[s] = in[id - base].
static int convert_row(lt_ctx* c, double** row, bool separate, bool to_home) {
  const int64_t n = c->home_n;
  if (n == 0 || !c->ids) return LT_OK;
  if (int rc = ensure_pool(c)) return rc;
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  double* tmp = c->pool[0];
  if (to_home) CK(launch_unsort(tmp, *row, c->ids, 0, n, c->home_base, c->bad, 1, c->stream));
  else CK(launch_resort(tmp, *row, c->ids, 0, n, c->home_base, c->bad, 1, c->stream));
  if (separate && n == c->cap) std::swap(*row, c->pool[0]);
  else CK(cudaMemcpyAsync(*row, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return LT_OK;
}

int lt_set_home_rows(lt_ctx* c, uint32_t mask) {
  int rc = check_ctx_keep(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (mask & ~(LT_HOME_Q | LT_HOME_ZETA | LT_HOME_DT | LT_HOME_ISO))
    return fail(LT_ERR_ARG, "unknown home row bits");
  const uint32_t change = mask ^ c->home_mask;
  if (!change) return LT_OK;
  if (change & LT_HOME_ZETA)
    if ((rc = convert_row(c, &c->zeta, true, mask & LT_HOME_ZETA))) return rc;
  if (change & LT_HOME_DT)
    if ((rc = convert_row(c, &c->dt, true, mask & LT_HOME_DT))) return rc;
  if (change & LT_HOME_ISO)
    if ((rc = convert_row(c, &c->iso_var, true, mask & LT_HOME_ISO))) return rc;
  if (change & LT_HOME_Q)
    for (int k = 0; k < c->nq; ++k) {
      double* r = c->q + static_cast<int64_t>(k) * c->cap;
      if ((rc = convert_row(c, &r, false, mask & LT_HOME_Q))) return rc;
    }
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (bad) return fail(LT_ERR_STATE, "particle ids of [0, %lld) are not a permutation of the home range",
                       (long long)c->home_n);
  c->home_mask = mask;
  return LT_OK;
}

// ------------------------------------------------------------------ met

int lt_met_grid(lt_ctx* c, int32_t nx, int32_t ny, int32_t nz, const double* lons,
                const double* lats, const double* levs, int32_t precision) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (nx < 2 || ny < 2 || nz < 2) return fail(LT_ERR_ARG, "meteo grid needs nx, ny, nz >= 2");
  if (precision != LT_MET_F32 && precision != LT_MET_F64)
    return fail(LT_ERR_ARG, "met precision must be 4 or 8 bytes");
  if (static_cast<int64_t>(nx) * ny * (nz - 1) >= (int64_t(1) << 32))
    return fail(LT_ERR_ARG, "met grid too large: cell records must fit 32-bit indices");
  std::vector<double> asc(levs, levs + nz);
  for (int k = 1; k < nz; ++k)
    if (!(levs[k] < levs[k - 1])) return fail(LT_ERR_ARG, "pressure levels must be strictly decreasing");
  for (int k = 0; k < nz; ++k) asc[k] = levs[nz - 1 - k];
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->copy));
  if ((rc = upload_axis(c->ax_lon, lons, nx, c->stream))) return rc;
  if ((rc = upload_axis(c->ax_lat, lats, ny, c->stream))) return rc;
  if ((rc = upload_axis(c->ax_lev, asc.data(), nz, c->stream))) return rc;
  const bool same_size = c->nx == nx && c->ny == ny && c->nz == nz && c->prec == precision;
  c->nx = nx; c->ny = ny; c->nz = nz; c->prec = precision;
  c->col_rank_n = 0;  // the key-compression table belongs to the old grid
  c->zone_known = false;
  for (int b = 0; b < 2; ++b) {  // so do the spread tables
    free_dev(c->sig_buf[b]);
    c->sig_buf[b] = nullptr;
    c->sig_of[b] = -1;
  }
  for (auto& s : c->slots) {
    s.valid = false;
    if (!same_size) { free_dev(s.rec); s.rec = nullptr; }
  }
  c->use0 = c->use1 = -1;
  return LT_OK;
}

static int met_prepare(lt_ctx* c, int slot) {
  if (!c->nx) return fail(LT_ERR_STATE, "met grid not set");
  if (slot < 0 || slot > 2) return fail(LT_ERR_ARG, "met slot %d outside [0, 3)", slot);
  Slot& s = c->slots[slot];
  for (int& t : c->sig_of)
    if (t == slot) t = -1;  // its spread table goes stale
  // never overwrite a slot the compute stream may still be reading: the copy
  // stream waits (on the device) for the compute work issued so far
  if (c->marked) CK(cudaStreamWaitEvent(c->copy, c->compute_mark, 0));
  if (!s.rec) {
    int rc = alloc_dev(&s.rec, rec_bytes(c) * n_rec(c), "met slot");
    if (rc) return rc;
  }
  s.valid = false;
  return LT_OK;
}

static int ensure_staging(lt_ctx* c, size_t bytes) {
  if (c->staging_bytes < bytes) {
    CK(cudaStreamSynchronize(c->copy));
    free_dev(c->staging);
    c->staging = nullptr;
    c->staging_bytes = 0;
    int rc = alloc_dev(&c->staging, bytes, "met staging");
    if (rc) return rc;
    c->staging_bytes = bytes;
  }
  return LT_OK;
}

int lt_met_load(lt_ctx* c, int32_t slot, double t_met, int32_t src_bytes, const void* u,
                const void* v, const void* w, const void* T, uint32_t flags) {
  int rc = check_ctx(c);
  if (rc || (rc = met_prepare(c, slot))) return rc;
  if (src_bytes != 4 && src_bytes != 8) return fail(LT_ERR_ARG, "met source must be f32 or f64");
  const int nx_src = (flags & LT_MET_CLOSE_LON) ? c->nx - 1 : c->nx;
  const size_t fbytes = static_cast<size_t>(nx_src) * c->ny * c->nz * src_bytes;
  const void* src[4] = {u, v, w, T};
  if (!(flags & LT_MET_DEVICE_SRC)) {
    // host fields: stage all four on the device (copy stream), then pack
    if ((rc = ensure_staging(c, 4 * fbytes))) return rc;
    char* st = static_cast<char*>(c->staging);
    for (int f = 0; f < 4; ++f) {
      CK(cudaMemcpyAsync(st + f * fbytes, src[f], fbytes, cudaMemcpyHostToDevice, c->copy));
      src[f] = st + f * fbytes;
    }
  }
  Slot& s = c->slots[slot];
  cudaError_t e;
  if (src_bytes == 4) {
    const float* const* b = reinterpret_cast<const float* const*>(src);
    e = c->prec == LT_MET_F64
            ? launch_pack_fields<float, RecD>(static_cast<RecD*>(s.rec), b[0], b[1], b[2], b[3], c->nx, c->ny, c->nz, nx_src, c->copy)
            : launch_pack_fields<float, RecF>(static_cast<RecF*>(s.rec), b[0], b[1], b[2], b[3], c->nx, c->ny, c->nz, nx_src, c->copy);
  } else {
    const double* const* b = reinterpret_cast<const double* const*>(src);
    e = c->prec == LT_MET_F64
            ? launch_pack_fields<double, RecD>(static_cast<RecD*>(s.rec), b[0], b[1], b[2], b[3], c->nx, c->ny, c->nz, nx_src, c->copy)
            : launch_pack_fields<double, RecF>(static_cast<RecF*>(s.rec), b[0], b[1], b[2], b[3], c->nx, c->ny, c->nz, nx_src, c->copy);
  }
  CK(e);
  CK(cudaEventRecord(s.ready, c->copy));
  s.t_met = t_met;
  s.valid = true;
  return LT_OK;
}

int lt_met_load_nodes(lt_ctx* c, int32_t slot, double t_met, const float* uvwT, uint32_t flags) {
  int rc = check_ctx(c);
  if (rc || (rc = met_prepare(c, slot))) return rc;
  const int nx_src = (flags & LT_MET_CLOSE_LON) ? c->nx - 1 : c->nx;
  const size_t bytes = static_cast<size_t>(nx_src) * c->ny * c->nz * 4 * sizeof(float);
  const float4* nodes = reinterpret_cast<const float4*>(uvwT);
  if (!(flags & LT_MET_DEVICE_SRC)) {
    if ((rc = ensure_staging(c, bytes))) return rc;
    CK(cudaMemcpyAsync(c->staging, uvwT, bytes, cudaMemcpyHostToDevice, c->copy));
    nodes = static_cast<const float4*>(c->staging);
  }
  Slot& s = c->slots[slot];
  CK(c->prec == LT_MET_F64
         ? launch_pack_nodes<RecD>(static_cast<RecD*>(s.rec), nodes, c->nx, c->ny, c->nz, nx_src, c->copy)
         : launch_pack_nodes<RecF>(static_cast<RecF*>(s.rec), nodes, c->nx, c->ny, c->nz, nx_src, c->copy));
  CK(cudaEventRecord(s.ready, c->copy));
  s.t_met = t_met;
  s.valid = true;
  return LT_OK;
}

int lt_met_use(lt_ctx* c, int32_t s0, int32_t s1) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (s0 < 0 || s0 > 2 || s1 < 0 || s1 > 2) return fail(LT_ERR_ARG, "met slots must be in [0, 3)");
  if (!c->slots[s0].valid || !c->slots[s1].valid) return fail(LT_ERR_STATE, "met slot not loaded");
  // the compute stream waits for the packing of both snapshots (copy stream)
  CK(cudaStreamWaitEvent(c->stream, c->slots[s0].ready, 0));
  CK(cudaStreamWaitEvent(c->stream, c->slots[s1].ready, 0));
  c->use0 = s0;
  c->use1 = s1;
  return LT_OK;
}

// Direct peer access dst -> src (NVLink), so peer copies do not stage
// through host memory; a no-op when the pair cannot (the copy then still
// works, through the driver's staging).  Leaves dst's device current.
static int enable_peer(int dst, int src) {
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, dst, src));
  if (can) {
    CK(cudaSetDevice(dst));
    cudaError_t e = cudaDeviceEnablePeerAccess(src, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();  // clear the sticky-free error
    else CK(e);
  }
  return LT_OK;
}

// Replicate a packed snapshot GPU to GPU (NVLink peer copy, or a D2D copy
// when both contexts share a GPU): the single-process counterpart of the
// met broadcast.  The copy runs on the destination's copy stream after the
// source slot's packing; the destination slot's ready event follows it.
int lt_met_copy_slot(lt_ctx* dst, int32_t dslot, lt_ctx* src, int32_t sslot) {
  int rc = check_ctx(src);
  if (rc || (rc = check_ctx(dst))) return rc;
  if (sslot < 0 || sslot > 2) return fail(LT_ERR_ARG, "met slot %d outside [0, 3)", sslot);
  if (!src->slots[sslot].valid) return fail(LT_ERR_STATE, "source met slot %d not loaded", sslot);
  if (dst->nx != src->nx || dst->ny != src->ny || dst->nz != src->nz || dst->prec != src->prec)
    return fail(LT_ERR_ARG, "met grids of the two contexts differ (call lt_met_grid first)");
  if ((rc = met_prepare(dst, dslot))) return rc;  // also orders after dst's compute
  const size_t bytes = rec_bytes(src) * n_rec(src);
  CK(cudaStreamWaitEvent(dst->copy, src->slots[sslot].ready, 0));
  if (dst->device == src->device) {
    CK(cudaMemcpyAsync(dst->slots[dslot].rec, src->slots[sslot].rec, bytes, cudaMemcpyDeviceToDevice, dst->copy));
  } else {
    if ((rc = enable_peer(dst->device, src->device))) return rc;
    CK(cudaMemcpyPeerAsync(dst->slots[dslot].rec, dst->device, src->slots[sslot].rec, src->device, bytes, dst->copy));
  }
  CK(cudaEventRecord(dst->slots[dslot].ready, dst->copy));
  // the source slot must not be refilled (on src's copy stream) before this
  // copy has read it
  CK(cudaStreamWaitEvent(src->copy, dst->slots[dslot].ready, 0));
  dst->slots[dslot].t_met = src->slots[sslot].t_met;
  dst->slots[dslot].valid = true;
  return LT_OK;
}

// The met broadcast of the one-process design: slot slots[root] of
// ctxs[root] reaches slot slots[i] of every other context.  Distinct GPUs
// receive it by ONE ncclBroadcast group (NVLink / NVSwitch, each rank on its
// context's copy stream); further contexts on an already-served GPU (test
// setups mapping several devices onto one B200) get a device-to-device copy
// from the context that received it there.  Every destination slot is
// ordered after that context's compute work (met_prepare) and its ready event
// follows the transfer, exactly as for an upload.
int lt_met_broadcast(lt_ctx* const* ctxs, int32_t n, int32_t root, const int32_t* slots) {
  if (!ctxs || !slots || n < 1) return fail(LT_ERR_ARG, "lt_met_broadcast needs n >= 1 contexts and slots");
  if (root < 0 || root >= n) return fail(LT_ERR_ARG, "broadcast root %d outside [0, %d)", root, n);
  lt_ctx* src = ctxs[root];
  int rc = check_ctx(src);
  if (rc) return rc;
  const int sslot = slots[root];
  if (sslot < 0 || sslot > 2) return fail(LT_ERR_ARG, "met slot %d outside [0, 3)", sslot);
  if (!src->slots[sslot].valid) return fail(LT_ERR_STATE, "root met slot %d not loaded", sslot);
  for (int i = 0; i < n; ++i) {
    lt_ctx* d = ctxs[i];
    if (!d) return fail(LT_ERR_STATE, "null context %d (deleted region?)", i);
    if (d->nx != src->nx || d->ny != src->ny || d->nz != src->nz || d->prec != src->prec)
      return fail(LT_ERR_ARG, "met grid of context %d differs from the root's (call lt_met_grid first)", i);
    for (int j = 0; j < i; ++j)
      if (ctxs[j] == d) return fail(LT_ERR_ARG, "context %d appears twice in the broadcast", i);
  }
  const size_t bytes = rec_bytes(src) * n_rec(src);
  // one representative per GPU (the root's GPU: the root itself)
  std::vector<int> rep_of(n, -1), devs, reps;
  devs.push_back(src->device);
  reps.push_back(root);
  rep_of[root] = root;
  for (int i = 0; i < n; ++i) {
    if (i == root) continue;
    auto it = std::find(devs.begin(), devs.end(), ctxs[i]->device);
    if (it == devs.end()) {
      devs.push_back(ctxs[i]->device);
      reps.push_back(i);
      rep_of[i] = i;
    } else {
      rep_of[i] = reps[it - devs.begin()];
    }
  }
  for (int i = 0; i < n; ++i) {
    if (i == root) continue;
    if ((rc = check_ctx(ctxs[i])) || (rc = met_prepare(ctxs[i], slots[i]))) return rc;
  }
  // the root's copy stream sends once the root slot is packed (it is its own stream)
  CK(cudaSetDevice(src->device));
  CK(cudaStreamWaitEvent(src->copy, src->slots[sslot].ready, 0));
  if (devs.size() > 1) {
    std::vector<void*> bufs;
    std::vector<cudaStream_t> streams;
    for (int r : reps) {
      bufs.push_back(ctxs[r]->slots[slots[r]].rec);
      streams.push_back(ctxs[r]->copy);
    }
    std::string err;
    if (lt_comm::broadcast(devs, bufs, bytes, 0, streams, &err))
      return fail(LT_ERR_CUDA, "met broadcast over %zu GPUs: %s", devs.size(), err.c_str());
    for (int r : reps) {
      if (r == root) continue;
      CK(cudaSetDevice(ctxs[r]->device));
      CK(cudaEventRecord(ctxs[r]->slots[slots[r]].ready, ctxs[r]->copy));
    }
    CK(cudaSetDevice(src->device));
  }
  // contexts sharing a GPU with a representative: device-local copies
  for (int i = 0; i < n; ++i) {
    if (rep_of[i] == i) continue;
    lt_ctx* d = ctxs[i];
    lt_ctx* from = ctxs[rep_of[i]];
    const int fslot = slots[rep_of[i]];
    CK(cudaSetDevice(d->device));
    CK(cudaStreamWaitEvent(d->copy, from->slots[fslot].ready, 0));
    CK(cudaMemcpyAsync(d->slots[slots[i]].rec, from->slots[fslot].rec, bytes, cudaMemcpyDeviceToDevice, d->copy));
    CK(cudaEventRecord(d->slots[slots[i]].ready, d->copy));
    CK(cudaStreamWaitEvent(from->copy, d->slots[slots[i]].ready, 0));  // source not refilled early
  }
  for (int i = 0; i < n; ++i) {
    if (i == root) continue;
    ctxs[i]->slots[slots[i]].t_met = src->slots[sslot].t_met;
    ctxs[i]->slots[slots[i]].valid = true;
  }
  return LT_OK;
}

int lt_nccl_version(int32_t* version) {
  std::string err;
  int v = 0;
  if (lt_comm::version(&v, &err)) return fail(LT_ERR_STATE, "%s", err.c_str());
  *version = v;
  return LT_OK;
}

// NCCL on this box, end to end with the GPUs there are: a communicator over
// `ndev` devices (ncclCommInitAll), one broadcast group of `bytes` from
// device 0 into a separate buffer on every device (device 0 too: send and
// receive buffers differ), checked byte for byte.  Returns LT_ERR_STATE when
// NCCL cannot be loaded, LT_ERR_CUDA on a mismatch.
int lt_nccl_selftest(int32_t ndev, int64_t bytes) {
  int have = 0;
  CK(cudaGetDeviceCount(&have));
  if (ndev < 1 || ndev > have) return fail(LT_ERR_ARG, "ndev %d outside [1, %d]", ndev, have);
  if (bytes < 1) return fail(LT_ERR_ARG, "bytes must be positive");
  std::vector<int> devs(ndev);
  std::vector<void*> send(ndev, nullptr), recv(ndev, nullptr);
  std::vector<cudaStream_t> streams(ndev, nullptr);
  std::vector<unsigned char> pattern(static_cast<size_t>(bytes)), back(static_cast<size_t>(bytes));
  for (size_t b = 0; b < pattern.size(); ++b) pattern[b] = static_cast<unsigned char>((b * 131u + 7u) & 0xFF);
  int rc = LT_OK;
  std::string err;
  for (int d = 0; d < ndev && !rc; ++d) {
    devs[d] = d;
    if (cudaSetDevice(d) != cudaSuccess || cudaStreamCreateWithFlags(&streams[d], cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&send[d], bytes) != cudaSuccess || cudaMalloc(&recv[d], bytes) != cudaSuccess ||
        cudaMemset(recv[d], 0, bytes) != cudaSuccess)
      rc = fail(LT_ERR_CUDA, "selftest allocation on device %d failed", d);
  }
  if (!rc && cudaMemcpy(send[0], pattern.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(LT_ERR_CUDA, "selftest upload failed");
  if (!rc) {
    // rank 0 sends from its own buffer; every rank receives into recv[d]
    std::vector<void*> bufs(recv);
    std::vector<void*> sendbufs(send);
    if (lt_comm::broadcast_from(devs, sendbufs[0], bufs, static_cast<size_t>(bytes), streams, &err))
      rc = fail(LT_ERR_STATE, "%s", err.c_str());
  }
  for (int d = 0; d < ndev && !rc; ++d) {
    cudaSetDevice(d);
    if (cudaStreamSynchronize(streams[d]) != cudaSuccess ||
        cudaMemcpy(back.data(), recv[d], bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = fail(LT_ERR_CUDA, "selftest readback on device %d failed", d);
    else if (std::memcmp(back.data(), pattern.data(), static_cast<size_t>(bytes)) != 0)
      rc = fail(LT_ERR_CUDA, "NCCL broadcast delivered wrong bytes to device %d", d);
  }
  for (int d = 0; d < ndev; ++d) {
    cudaSetDevice(d);
    if (send[d]) cudaFree(send[d]);
    if (recv[d]) cudaFree(recv[d]);
    if (streams[d]) cudaStreamDestroy(streams[d]);
  }
  return rc;
}

int lt_nccl_ranks(int32_t* nranks) {
  std::string err;
  *nranks = lt_comm::communicators(&err);
  return LT_OK;
}

int lt_met_slot_time(lt_ctx* c, int32_t slot, double* t) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  if (slot < 0 || slot > 2) return fail(LT_ERR_ARG, "met slot outside [0, 3)");
  if (!c->slots[slot].valid) return fail(LT_ERR_STATE, "met slot %d not loaded", slot);
  *t = c->slots[slot].t_met;
  return LT_OK;
}

int lt_clim_load(lt_ctx* c, int32_t nlat, int32_t np_, const double* lat_grid,
                 const double* p_grid, const double* hno3, const double* p_trop) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = upload_axis(c->cl_lat, lat_grid, nlat, c->stream))) return rc;
  if ((rc = upload_axis(c->cl_p, p_grid, np_, c->stream))) return rc;
  free_dev(c->hno3);
  free_dev(c->p_trop);
  c->hno3 = c->p_trop = nullptr;
  if ((rc = alloc_dev(reinterpret_cast<void**>(&c->hno3), sizeof(double) * nlat * np_, "hno3")))
    return rc;
  if ((rc = alloc_dev(reinterpret_cast<void**>(&c->p_trop), sizeof(double) * nlat, "p_trop")))
    return rc;
  CK(cudaMemcpyAsync(c->hno3, hno3, sizeof(double) * nlat * np_, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->p_trop, p_trop, sizeof(double) * nlat, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

// ------------------------------------------------------------------ compute

extern "C++" {
// The spread table of met slot `slot`: an existing one, or built into the
// buffer that describes neither met0 nor met1 — on the compute stream (after
// any prebuild still writing that buffer), or on the copy stream (after the
// slot's packing and after every compute launch issued so far, which may
// still read the buffer's previous table)
template <class Rec>
static int spread_table_for(lt_ctx* c, int slot, bool on_copy, int* idx) {
  for (int b = 0; b < 2; ++b)
    if (c->sig_of[b] == slot) { *idx = b; return LT_OK; }
  int b = 0;
  while (b < 2 && (c->sig_of[b] == c->use0 || c->sig_of[b] == c->use1) && c->sig_of[b] >= 0) ++b;
  if (b == 2) return fail(LT_ERR_STATE, "no free spread table (slots %d/%d)", c->use0, c->use1);
  if (!c->sig_buf[b]) {
    if (int rc = alloc_dev(reinterpret_cast<void**>(&c->sig_buf[b]), 4 * sizeof(double) * n_rec(c), "spread table"))
      return rc;
  }
  MetView<Rec> m = met_view<Rec>(c);
  m.s0 = static_cast<const Rec*>(c->slots[slot].rec);
  cudaStream_t st = c->stream;
  if (on_copy) {
    st = c->copy;
    CK(cudaEventRecord(c->sig_mark, c->stream));
    CK(cudaStreamWaitEvent(c->copy, c->sig_mark, 0));
    CK(cudaStreamWaitEvent(c->copy, c->slots[slot].ready, 0));
  } else {
    CK(cudaStreamWaitEvent(c->stream, c->sig_ready[b], 0));
  }
  CK(launch_spread_table<Rec>(m, c->nx, c->sig_buf[b], st));
  CK(cudaEventRecord(c->sig_ready[b], st));
  c->sig_of[b] = slot;
  *idx = b;
  return LT_OK;
}

template <class Rec>
static int run_typed(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t start,
                     int64_t end, int64_t step, uint64_t fstate, int64_t fbase, uint32_t flags,
                     bool fuse_perm = false, int32_t nsteps = 1) {
  StepArgs<Rec> a;
  a.perm = nullptr;
  a.perm_start = 0;
  a.o_time = a.o_p = a.o_lon = a.o_lat = nullptr;
  a.o_uvwp[0] = a.o_uvwp[1] = a.o_uvwp[2] = nullptr;
  a.o_ids = nullptr;
  if (fuse_perm) {  // apply the pending sort on the fly: hot rows into the pool
    if (int rc = ensure_pool(c, 7)) return rc;
    if (!c->ids_alt)
      if (int rc = alloc_dev(reinterpret_cast<void**>(&c->ids_alt), sizeof(uint32_t) * c->cap, "ids"))
        return rc;
    a.perm = c->sort_buf + 3 * c->cap;
    a.perm_start = c->pend_start;
    a.o_time = c->pool[0]; a.o_p = c->pool[1]; a.o_lon = c->pool[2]; a.o_lat = c->pool[3];
    for (int k = 0; k < 3; ++k) a.o_uvwp[k] = c->pool[4 + k];
    a.o_ids = c->ids_alt;
  }
  a.time = c->time; a.p = c->p; a.lon = c->lon; a.lat = c->lat; a.dt = c->dt;
  for (int k = 0; k < 3; ++k) a.uvwp[k] = c->uvwp[k];
  a.iso_var = c->iso_var; a.q = c->q;
  a.ids = c->ids;
  a.home_mask = c->home_mask;
  a.home_base = c->home_base;
  a.rnd_conv = c->rnd_conv; a.rnd_turb = c->rnd_turb; a.rnd_meso = c->rnd_meso;
  a.cap = c->cap; a.start = start; a.end = end; a.nq = c->nq;
  a.modules = modules; a.flags = flags; a.step = step; a.nsteps = nsteps;
  a.faithful_state = fstate; a.faithful_base = fbase;
  a.iso_nonconv = c->counters;
  a.mod_cycles = c->counters + 8;
  a.flags &= ~F_SORT_KEYS;
  a.sk_keys = a.sk_vals = nullptr;
  a.sk_rank = nullptr;
  a.sk_kmin = 0;
  a.sk_nocc = 1;
  a.sk_bad = nullptr;
  bool sort_keys = false;
  // (the key lookup needs the met axes: launches that bind a met pair only)
  const bool met_bound = (modules & (M_ADVECTION | M_TURB | M_MESO | M_SEDI | M_ISOSURF | M_METEO |
                                     M_ISOSURF_INIT)) && c->use0 >= 0;
  if ((flags & LT_RUN_SORT_KEYS) && !fuse_perm && met_bound && c->zone_known && c->col_rank &&
      c->sort_buf && c->col_count > 0) {
    // the level window: as wide as the radix passes of the occupied range
    // allow, centred on it (a particle outside it flags the keys invalid and
    // the sort computes its own)
    const uint32_t nlev = box_levels(c->nz);
    const uint32_t occ = c->zone_max - c->zone_min + 1;
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= static_cast<uint64_t>(c->col_count) * occ - 1) ++bits;
    bits = (bits + 7) / 8 * 8;
    const uint64_t room = bits >= 32 ? nlev : (1ull << bits) / c->col_count;
    const uint32_t nocc = static_cast<uint32_t>(std::max<uint64_t>(occ, std::min<uint64_t>(nlev, room)));
    uint32_t kmin = c->zone_min - std::min(c->zone_min, (nocc - occ) / 2);
    if (kmin + nocc > nlev) kmin = nlev - nocc;
    a.sk_keys = c->sort_buf;
    a.sk_vals = c->sort_buf + 2 * c->cap;
    a.sk_rank = c->col_rank;
    a.sk_kmin = kmin;
    a.sk_nocc = nocc;
    a.sk_bad = reinterpret_cast<unsigned int*>(c->counters + 5);
    CK(cudaMemsetAsync(a.sk_bad, 0, sizeof(unsigned int), c->stream));
    a.flags |= F_SORT_KEYS;
    sort_keys = true;
  }
  static_assert(sizeof(lt_control) == sizeof(Control), "control layout");
  std::memcpy(&a.ctl, ctl, sizeof(Control));
  {
    // the kernel's own expressions at dt = dt_model (lt_step.cuh StepConst);
    // volatile keeps the host compiler from contracting 1 - r*r into an FMA
    StepConst& k = a.kc;
    const double dt = ctl->dt_model;
    k.dt = dt;
    k.turb_sx = std::sqrt(2.0 * ctl->turb_dx * dt);
    k.turb_sz = std::sqrt(2.0 * ctl->turb_dz * dt);
    double r = 1.0 - 2.0 * dt / ctl->met_dt;
    r = std::fmin(std::fmax(r, 0.0), 1.0);
    volatile double rr = r * r;
    k.meso_r = r;
    k.meso_amp = std::sqrt(1.0 - rr);
    k.decay = ctl->decay_tau > 0.0 ? std::exp(-dt / ctl->decay_tau) : 1.0;
    k.conv_scale = ctl->conv_prob != 0.0 ? (ctl->p_surf - ctl->conv_p_top) / ctl->conv_prob : 0.0;
    philox_round_keys(static_cast<uint32_t>(ctl->rng_seed_global),
                      static_cast<uint32_t>(ctl->rng_seed_global >> 32), k.philox_rk);
  }
  const bool need_met = modules & (M_ADVECTION | M_TURB | M_MESO | M_SEDI | M_ISOSURF | M_METEO |
                                   M_ISOSURF_INIT);
  if (need_met) {
    if (c->use0 < 0) return fail(LT_ERR_STATE, "no met snapshots selected (lt_met_use)");
    a.met = met_view<Rec>(c);
    if ((modules & M_MESO) && ctl->turb_meso != 0.0) {
      // the mesoscale spreads of met0 (built here on the compute stream if
      // no prebuilt table describes it), then met1's prebuilt on the copy
      // stream for the next rotation
      int b = -1;
      if (int rc = spread_table_for<Rec>(c, c->use0, false, &b)) return rc;
      CK(cudaStreamWaitEvent(c->stream, c->sig_ready[b], 0));
      a.met.sig0 = c->sig_buf[b];
      c->meso_seen = true;
      if (c->use1 != c->use0) {
        int b1 = -1;
        if (int rc = spread_table_for<Rec>(c, c->use1, true, &b1)) return rc;
      }
    }
  } else {
    std::memset(&a.met, 0, sizeof(a.met));
  }
  if (modules & M_METEO) {
    if (!c->hno3) return fail(LT_ERR_STATE, "climatology not loaded (lt_clim_load)");
    a.clim.lat = view(c->cl_lat);
    a.clim.p = view(c->cl_p);
    a.clim.hno3 = c->hno3;
    a.clim.p_trop = c->p_trop;
  } else {
    std::memset(&a.clim, 0, sizeof(a.clim));
  }
  CK(launch_step<Rec>(a, c->stream));
  if (sort_keys) {
    c->sk_call = c->calls;
    c->sk_start = start;
    c->sk_end = end;
    c->sk_nocc = a.sk_nocc;
  } else {
    c->sk_call = ~0ull;
  }
  if (fuse_perm) {  // the pool rows now hold the sorted state
    std::swap(c->time, c->pool[0]); std::swap(c->p, c->pool[1]);
    std::swap(c->lon, c->pool[2]); std::swap(c->lat, c->pool[3]);
    for (int k = 0; k < 3; ++k) std::swap(c->uvwp[k], c->pool[4 + k]);
    std::swap(c->ids, c->ids_alt);
    c->pending = false;
  }
  return LT_OK;
}
}  // extern C++

static int run_impl(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t start,
                    int64_t end, int64_t step, int32_t nsteps, uint64_t fstate, int64_t fbase,
                    uint32_t flags);

int lt_run(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t start, int64_t end,
           int64_t step, uint64_t fstate, int64_t fbase, uint32_t flags) {
  return run_impl(c, ctl, modules, start, end, step, 1, fstate, fbase, flags);
}

// nsteps consecutive steps of [start, end) in one launch (each particle's
// state stays in registers across them): in-kernel counter or Philox draws
// only, and the met pair must cover all the steps (no rotation inside)
int lt_run_steps(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t start,
                 int64_t end, int64_t step, int32_t nsteps, uint32_t flags) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (nsteps < 1) return fail(LT_ERR_ARG, "nsteps %d < 1", nsteps);
  if ((modules & (M_TURB | M_MESO | M_CONVECTION)) && ctl->rng_mode == RNG_FAITHFUL)
    return fail(LT_ERR_ARG, "faithful draws need the per-step stream state: use lt_run per step");
  // one launch for the production chain with an in-kernel counter or Philox
  // generator; anything else runs as nsteps single-step launches
  const bool multi =
      modules == (M_TIMESTEPS | M_ADVECTION | M_POSITION) ||
      (modules == (M_TIMESTEPS | M_ADVECTION | M_TURB | M_MESO | M_POSITION) &&
       (flags & LT_RUN_RNG_INKERNEL) && (ctl->rng_mode == RNG_COUNTER || ctl->rng_mode == RNG_PHILOX));
  // the event timing (lt_timing) spans every launch of the call
  const bool timing = c->timing;
  if (timing) CK(cudaEventRecord(c->ev_start, c->stream));
  c->timing = false;
  if (!multi) {
    for (int32_t k = 0; k < nsteps && !rc; ++k)
      rc = run_impl(c, ctl, modules, start, end, step + k, 1, 0, 0, flags);
  } else {
    // a pending sort rides along with the first step alone
    if (c->pending && nsteps > 1) {
      rc = run_impl(c, ctl, modules, start, end, step, 1, 0, 0, flags);
      ++step;
      --nsteps;
    }
    if (!rc) rc = run_impl(c, ctl, modules, start, end, step, nsteps, 0, 0, flags);
  }
  c->timing = timing;
  if (rc) return rc;
  if (timing) {
    CK(cudaEventRecord(c->ev_stop, c->stream));
    c->timed_once = true;
  }
  return LT_OK;
}

static int run_impl(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t start,
                    int64_t end, int64_t step, int32_t nsteps, uint64_t fstate, int64_t fbase,
                    uint32_t flags) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if (!(0 <= start && start <= end && end <= c->cap))
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside ensemble of %lld particles",
                (long long)start, (long long)end, (long long)c->cap);
  if (!(flags & LT_RUN_RNG_INKERNEL) && (modules & (M_TURB | M_MESO | M_CONVECTION)) && !c->rnd_conv)
    return fail(LT_ERR_STATE, "random batch not allocated and in-kernel draws not requested");
  if ((flags & LT_RUN_RNG_INKERNEL) && ctl->rng_mode == RNG_FAITHFUL &&
      (modules & (M_TURB | M_MESO | M_CONVECTION)) && c->ids == nullptr && fbase > start)
    return fail(LT_ERR_ARG, "faithful base beyond range start");
  // a pending box sort rides along with a whole-store production step;
  // anything else applies it first
  bool fuse = false;
  if (c->pending) {
    fuse = perm_capable(modules, flags, ctl->rng_mode) && start == 0 && end == c->cap &&
           c->pend_start == 0 && c->pend_n == c->cap;
    if (!fuse && (rc = settle(c))) return rc;
  }
  if (fuse && nsteps > 1) return fail(LT_ERR_STATE, "a pending sort fuses with one step only");
  if (c->timing) CK(cudaEventRecord(c->ev_start, c->stream));
  if (end > start) {
    rc = c->prec == LT_MET_F64
             ? run_typed<RecD>(c, ctl, modules, start, end, step, fstate, fbase, flags, fuse, nsteps)
             : run_typed<RecF>(c, ctl, modules, start, end, step, fstate, fbase, flags, fuse, nsteps);
    if (rc) return rc;
  }
  CK(cudaEventRecord(c->compute_mark, c->stream));
  c->marked = true;
  if (c->timing) {
    CK(cudaEventRecord(c->ev_stop, c->stream));
    c->timed_once = true;
  }
  return LT_OK;
}

// Chunked host-buffer step: H2D (copy stream) -> fused step (compute
// stream) -> D2H (d2h stream), one ring slot per chunk in the particle
// store.  Events order each slot's three stages and keep a slot from being
// refilled before its results have been copied out.
int lt_run_host(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t n, int64_t step,
                int64_t first_id, uint64_t fstate, const lt_host_soa* io, int64_t chunk) {
  return lt_run_host_steps(c, ctl, modules, n, step, 1, first_id, fstate, io, chunk);
}

// nsteps steps, each a full round trip of every particle through the GPU.
// Particles are independent, so chunk c of step s+1 only has to wait for
// chunk c of step s to land back in host memory: the pipeline never drains
// between steps (one fill and one drain per call instead of per step).
int lt_run_host_steps(lt_ctx* c, const lt_control* ctl, uint32_t modules, int64_t n, int64_t step,
                      int32_t nsteps, int64_t first_id, uint64_t fstate, const lt_host_soa* io,
                      int64_t chunk) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (!io || !io->time || !io->p || !io->lon || !io->lat)
    return fail(LT_ERR_ARG, "host SoA needs time, p, lon and lat");
  if (n < 0) return fail(LT_ERR_ARG, "negative particle count");
  if (nsteps < 0) return fail(LT_ERR_ARG, "negative step count");
  if (first_id < 0 || first_id + n > (int64_t(1) << 32))
    return fail(LT_ERR_ARG, "particle ids must fit in 32 bits");
  const bool meso = modules & M_MESO;
  const bool iso_in = modules & M_ISOSURF, iso_out = modules & M_ISOSURF_INIT;
  const bool meteo = modules & M_METEO;
  const bool decay = (modules & M_DECAY) && ctl->decay_slot >= 0;
  if (meso && !io->uvwp) return fail(LT_ERR_ARG, "meso needs the uvwp rows");
  if ((iso_in || iso_out) && !io->iso_var) return fail(LT_ERR_ARG, "isosurf needs iso_var");
  if ((meteo || decay) && !io->q) return fail(LT_ERR_ARG, "meteo/decay need the q rows");
  if ((meso || meteo || decay) && io->stride < n) return fail(LT_ERR_ARG, "row stride < n");
  if (meteo && (io->nq < 5 || c->nq < 5)) return fail(LT_ERR_ARG, "meteo needs 5 q rows");
  if (decay && (ctl->decay_slot >= io->nq || ctl->decay_slot >= c->nq))
    return fail(LT_ERR_ARG, "decay_slot outside the q rows");
  if (n == 0 || nsteps == 0) return LT_OK;
  // the store is scratch for this call: every row in slot order
  c->home_mask = 0;
  c->home_n = 0;
  // 1M-particle chunks (~8 MB per row): short pipeline fill and drain, few
  // enough copy calls (best of 1M/2M/4M/n/16 on B200, PCIe Gen5)
  if (chunk <= 0) chunk = std::min<int64_t>(c->cap, int64_t(1) << 20);
  chunk = std::min(chunk, c->cap);
  if (chunk <= 0) return fail(LT_ERR_STATE, "particle store has no capacity");
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int nbuf = static_cast<int>(std::min<int64_t>({nchunks, c->cap / chunk, 32}));
  if ((rc = ensure_ids(c))) return rc;
  while (c->ring_ev.size() < static_cast<size_t>(3 * nbuf)) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ring_ev.push_back(e);
  }
  // rows: (device row, host row, copy in, copy out)
  struct Row { double* dev; double* host; bool in, out; };
  std::vector<Row> rows;
  const bool moves = modules & (M_ADVECTION | M_TURB | M_MESO | M_CONVECTION | M_SEDI | M_ISOSURF |
                                M_POSITION);
  rows.push_back({c->time, io->time, true, (modules & M_ADVECTION) != 0});
  rows.push_back({c->p, io->p, true, moves});
  rows.push_back({c->lon, io->lon, true, moves});
  rows.push_back({c->lat, io->lat, true, moves});
  if (meso)
    for (int k = 0; k < 3; ++k) rows.push_back({c->uvwp[k], io->uvwp + k * io->stride, true, true});
  if (iso_in || iso_out) rows.push_back({c->iso_var, io->iso_var, iso_in, iso_out});
  if (meteo)
    for (int k = 0; k < 5; ++k) rows.push_back({c->q + k * c->cap, io->q + k * io->stride, false, true});
  if (decay && !(meteo && ctl->decay_slot < 5))
    rows.push_back({c->q + ctl->decay_slot * c->cap, io->q + ctl->decay_slot * io->stride, true, true});
  else if (decay)
    rows[rows.size() - 5 + ctl->decay_slot].in = true;
  if (c->timing) CK(cudaEventRecord(c->ev_start, c->stream));
  // the copy stream must not overwrite slots the compute stream still reads
  CK(cudaEventRecord(c->compute_mark, c->stream));
  CK(cudaStreamWaitEvent(c->copy, c->compute_mark, 0));
  while (c->host_ev.size() < static_cast<size_t>(nchunks)) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->host_ev.push_back(e);
  }
  for (int32_t st = 0; st < nsteps; ++st) {
    // faithful device stream after st fills of n particles (rng.py:125)
    const uint64_t fs = fstate + static_cast<uint64_t>(st) * 7ull * static_cast<uint64_t>(n) * kGamma;
    for (int64_t k = 0; k < nchunks; ++k) {
      const int64_t g = st * nchunks + k;  // global chunk sequence number
      const int b = static_cast<int>(g % nbuf);
      const int64_t off = b * chunk, lo = k * chunk, cnt = std::min(chunk, n - lo);
      cudaEvent_t h2d_done = c->ring_ev[3 * b], run_done = c->ring_ev[3 * b + 1],
                  d2h_done = c->ring_ev[3 * b + 2];
      if (g >= nbuf) CK(cudaStreamWaitEvent(c->copy, d2h_done, 0));        // slot free
      if (st > 0) CK(cudaStreamWaitEvent(c->copy, c->host_ev[k], 0));      // host rows landed
      for (const Row& r : rows)
        if (r.in) CK(cudaMemcpyAsync(r.dev + off, r.host + lo, sizeof(double) * cnt, cudaMemcpyHostToDevice, c->copy));
      CK(cudaEventRecord(h2d_done, c->copy));
      CK(cudaStreamWaitEvent(c->stream, h2d_done, 0));
      CK(launch_iota(c->ids, off, cnt, first_id + lo, c->stream));
      rc = c->prec == LT_MET_F64
               ? run_typed<RecD>(c, ctl, modules, off, off + cnt, step + st, fs, first_id, LT_RUN_RNG_INKERNEL)
               : run_typed<RecF>(c, ctl, modules, off, off + cnt, step + st, fs, first_id, LT_RUN_RNG_INKERNEL);
      if (rc) return rc;
      CK(cudaEventRecord(run_done, c->stream));
      CK(cudaStreamWaitEvent(c->d2h, run_done, 0));
      for (const Row& r : rows)
        if (r.out) CK(cudaMemcpyAsync(r.host + lo, r.dev + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->d2h));
      CK(cudaEventRecord(d2h_done, c->d2h));
      CK(cudaEventRecord(c->host_ev[k], c->d2h));
    }
  }
  const int64_t last = static_cast<int64_t>(nsteps) * nchunks - 1;
  CK(cudaEventRecord(c->compute_mark, c->stream));
  c->marked = true;
  if (c->timing) {
    CK(cudaStreamWaitEvent(c->stream, c->ring_ev[3 * (last % nbuf) + 2], 0));
    CK(cudaEventRecord(c->ev_stop, c->stream));
    c->timed_once = true;
  }
  CK(cudaStreamSynchronize(c->d2h));
  CK(cudaStreamSynchronize(c->stream));
  return LT_OK;
}

int lt_rng_fill(lt_ctx* c, int32_t mode, uint64_t seed, int64_t step, int64_t start, int64_t end) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (!c->rnd_conv) return fail(LT_ERR_STATE, "context allocated without a random batch");
  if (!(0 <= start && start <= end && end <= c->cap))
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside ensemble of %lld particles",
                (long long)start, (long long)end, (long long)c->cap);
  if (mode < 0 || mode > 2) return fail(LT_ERR_ARG, "unknown rng mode %d", mode);
  if (c->timing) CK(cudaEventRecord(c->ev_start, c->stream));
  CK(launch_rng_fill(mode, seed, step, start, end, c->ids, c->rnd_conv, c->rnd_turb, c->rnd_meso, c->stream));
  if (c->timing) { CK(cudaEventRecord(c->ev_stop, c->stream)); c->timed_once = true; }
  return LT_OK;
}

int lt_module_cycles(lt_ctx* c, uint64_t* cycles, int32_t reset) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  static_assert(CK_N <= LT_N_MODULE_CLOCKS, "clock slots");
  unsigned long long v[LT_N_MODULE_CLOCKS] = {};
  CK(cudaMemcpyAsync(v, c->counters + 8, sizeof(unsigned long long) * CK_N, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (reset) CK(cudaMemsetAsync(c->counters + 8, 0, sizeof(unsigned long long) * CK_N, c->stream));
  for (int k = 0; k < LT_N_MODULE_CLOCKS; ++k) cycles[k] = v[k];
  return LT_OK;
}

int lt_philox4x32_10(lt_ctx* c, int32_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (n < 0) return fail(LT_ERR_ARG, "negative block count");
  if (n == 0) return LT_OK;
  void* d = nullptr;
  // counters (16 B each), keys (8 B), outputs (16 B): each array 16-byte aligned
  const size_t b_ctr = 16 * static_cast<size_t>(n), b_key = (8 * static_cast<size_t>(n) + 15) & ~size_t(15);
  if ((rc = alloc_dev(&d, 2 * b_ctr + b_key, "philox kat"))) return rc;
  char* base = static_cast<char*>(d);
  cudaError_t e = cudaMemcpyAsync(base, ctr, b_ctr, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(base + b_ctr, key, b_key, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = launch_philox_kat(reinterpret_cast<uint32_t*>(base), reinterpret_cast<uint32_t*>(base + b_ctr),
                          reinterpret_cast<uint32_t*>(base + b_ctr + b_key), n, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, base + b_ctr + b_key, b_ctr, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  free_dev(d);
  CK(e);
  return LT_OK;
}

int lt_iso_counter(lt_ctx* c, int64_t* value, int32_t reset) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&v, c->counters, sizeof v, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (reset) {
    CK(cudaMemsetAsync(c->counters, 0, sizeof v, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  *value = static_cast<int64_t>(v);
  return LT_OK;
}

int lt_interpolate(lt_ctx* c, int64_t n, const double* t, const double* lon, const double* lat,
                   const double* p, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->use0 < 0) return fail(LT_ERR_STATE, "no met snapshots selected (lt_met_use)");
  if (n < 0) return fail(LT_ERR_ARG, "negative point count");
  if (n == 0) return LT_OK;
  double* buf = nullptr;
  if ((rc = alloc_dev(reinterpret_cast<void**>(&buf), sizeof(double) * 8 * n, "interp points")))
    return rc;
  const double* src[4] = {t, lon, lat, p};
  cudaError_t e = cudaSuccess;
  for (int f = 0; f < 4 && e == cudaSuccess; ++f)
    e = cudaMemcpyAsync(buf + f * n, src[f], sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = c->prec == LT_MET_F64
            ? launch_sample<RecD>(met_view<RecD>(c), buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, n, c->stream)
            : launch_sample<RecF>(met_view<RecF>(c), buf, buf + n, buf + 2 * n, buf + 3 * n, buf + 4 * n, n, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, buf + 4 * n, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(buf);
  CK(e);
  return LT_OK;
}

// the cell lookup of the exact (precision 0) or fast (1) kernels at n host
// points: out = i, j, k rows (3n int32) — the cell audit against the
// reference's _locate (physics.py:31-47); needs the grid only
int lt_locate_cells(lt_ctx* c, int32_t precision, int64_t n, const double* lon, const double* lat,
                    const double* p, int32_t* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->nx) return fail(LT_ERR_STATE, "met grid not set");
  if (precision != 0 && precision != 1) return fail(LT_ERR_ARG, "precision must be 0 or 1");
  if (precision == 1 && c->prec != LT_MET_F32)
    return fail(LT_ERR_ARG, "the fast kernels run on the f32 met store only");
  if (n < 0) return fail(LT_ERR_ARG, "negative point count");
  if (n == 0) return LT_OK;
  char* buf = nullptr;
  if ((rc = alloc_dev(reinterpret_cast<void**>(&buf), (sizeof(double) * 3 + sizeof(int32_t) * 3) * n,
                      "locate points")))
    return rc;
  double* d = reinterpret_cast<double*>(buf);
  int32_t* o = reinterpret_cast<int32_t*>(buf + sizeof(double) * 3 * n);
  const double* src[3] = {lon, lat, p};
  cudaError_t e = cudaSuccess;
  for (int f = 0; f < 3 && e == cudaSuccess; ++f)
    e = cudaMemcpyAsync(d + f * n, src[f], sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) {
    if (c->prec == LT_MET_F64) {
      MetView<RecD> m{};
      m.lon = view(c->ax_lon); m.lat = view(c->ax_lat); m.lev = view(c->ax_lev);
      m.ny = c->ny; m.nz = c->nz;
      e = launch_locate<RecD>(m, precision, d, d + n, d + 2 * n, o, n, c->stream);
    } else {
      MetView<RecF> m{};
      m.lon = view(c->ax_lon); m.lat = view(c->ax_lat); m.lev = view(c->ax_lev);
      m.ny = c->ny; m.nz = c->nz;
      e = launch_locate<RecF>(m, precision, d, d + n, d + 2 * n, o, n, c->stream);
    }
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, o, sizeof(int32_t) * 3 * n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(buf);
  CK(e);
  return LT_OK;
}

// ------------------------------------------------------------------ sort

extern "C++" {
template <class Rec>
static int sort_typed(lt_ctx* c, int64_t start, int64_t end) {
  const int64_t n = end - start;
  uint32_t* keys_in = c->sort_buf;
  uint32_t* keys_out = keys_in + c->cap;
  uint32_t* vals_in = keys_out + c->cap;
  uint32_t* vals_out = vals_in + c->cap;
  const MetView<Rec> m = met_view<Rec>(c);
  // Morton column order when its keys fit 32 bits (they do up to ~0.1 deg
  // grids; measured -1.6 % step time against row-major cells at cfg3), else
  // the record index
  const uint64_t max_morton =
      static_cast<uint64_t>((part1by1(static_cast<uint32_t>(c->nx - 1) >> LT_BOX_SHIFT) << 1) |
                            part1by1(static_cast<uint32_t>(c->ny - 1) >> LT_BOX_SHIFT)) *
          box_levels(c->nz) + (box_levels(c->nz) - 1);
  const int morton = c->nx <= 65536 && c->ny <= 65536 && max_morton < (uint64_t(1) << 32);
  auto nbits = [](uint64_t v) { int b = 1; while (b < 32 && (1ull << b) <= v) ++b; return b; };
  // keys written by the step launch just before (LT_RUN_SORT_KEYS), unless a
  // particle left their level window
  bool fresh = morton && n > 0 && c->calls == c->sk_call + 1 && start == c->sk_start &&
               end == c->sk_end && c->col_rank;
  if (fresh) {
    unsigned int bad = 1;
    CK(cudaMemcpyAsync(&bad, c->counters + 5, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    fresh = bad == 0;
  }
  c->sk_call = ~0ull;
  uint64_t max_key = morton ? max_morton : static_cast<uint64_t>(n_rec(c));
  ++c->n_sorts;
  if (fresh) {
    ++c->n_sorts_fused;
    max_key = static_cast<uint64_t>(c->col_count) * c->sk_nocc - 1;
  } else {
  unsigned int* kzone = reinterpret_cast<unsigned int*>(c->counters + 2);
  if (morton) {
    const unsigned int init[2] = {0xFFFFFFFFu, 0u};
    CK(cudaMemcpyAsync(kzone, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
  }
  CK(launch_box_keys<Rec>(m, c->lon, c->lat, c->p, start, n, keys_in, vals_in, morton,
                          morton ? kzone : nullptr, c->stream));
  if (morton && n > 0) {
    // the same order in fewer key bits when that saves an 8-bit radix pass:
    // dense column ranks times the occupied level boxes (compress_keys_kernel)
    const uint32_t nlev = box_levels(c->nz);
    const uint64_t ncode = max_morton / nlev + 1;
    if (c->col_rank_n != static_cast<int64_t>(ncode)) {
      std::vector<uint32_t> rank(ncode, 0u);
      std::vector<unsigned char> used(ncode, 0);
      for (int i = 0; i < c->nx; ++i)
        for (int j = 0; j < c->ny; ++j)
          used[(part1by1(static_cast<uint32_t>(i) >> LT_BOX_SHIFT) << 1) |
               part1by1(static_cast<uint32_t>(j) >> LT_BOX_SHIFT)] = 1;
      uint32_t r = 0;
      for (uint64_t code = 0; code < ncode; ++code) {
        rank[code] = r;
        r += used[code];
      }
      free_dev(c->col_rank);
      c->col_rank = nullptr;
      if (int rc = alloc_dev(reinterpret_cast<void**>(&c->col_rank), sizeof(uint32_t) * ncode, "column ranks"))
        return rc;
      CK(cudaMemcpy(c->col_rank, rank.data(), sizeof(uint32_t) * ncode, cudaMemcpyHostToDevice));
      c->col_rank_n = static_cast<int64_t>(ncode);
      c->col_count = r;
    }
    unsigned int zone[2];
    CK(cudaMemcpyAsync(zone, kzone, sizeof zone, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const uint32_t nocc = zone[1] - zone[0] + 1;
    c->zone_known = true;
    c->zone_min = zone[0];
    c->zone_max = zone[1];
    const uint64_t max_c = static_cast<uint64_t>(c->col_count) * nocc - 1;
    if ((nbits(max_c) + 7) / 8 < (nbits(max_key) + 7) / 8) {
      CK(launch_compress_keys(keys_in, n, c->col_rank, nlev, zone[0], nocc, c->stream));
      max_key = max_c;
    }
  }
  }
  const int bits = nbits(max_key);
  size_t need = 0;
  CK(sort_pairs(nullptr, need, keys_in, keys_out, vals_in, vals_out, n, bits, c->stream));
  if (need > c->cub_bytes) {
    CK(cudaStreamSynchronize(c->stream));
    free_dev(c->cub_temp);
    c->cub_temp = nullptr;
    int rc = alloc_dev(&c->cub_temp, need, "sort temp");
    if (rc) return rc;
    c->cub_bytes = need;
  }
  size_t have = c->cub_bytes;
  CK(sort_pairs(c->cub_temp, have, keys_in, keys_out, vals_in, vals_out, n, bits, c->stream));
  return LT_OK;
}
}  // extern C++

extern "C++" {
// The permutation of the last sort (sort_buf vals_out) applied to the rows:
// new slot start + t takes old slot start + perm[t].
static int apply_perm(lt_ctx* c, int64_t start, int64_t n) {
  uint32_t* keys_in = c->sort_buf;
  const uint32_t* vals_out = c->sort_buf + 3 * c->cap;
  const int64_t end = start + n;
  // Permute every per-particle row, kRowSet rows per launch into the pool
  // rows.  Separately allocated rows covering the whole store swap pointers
  // with their pool row (no copy back); the q block and partial ranges copy
  // the gathered slice back.
  if (int rc = ensure_pool(c)) return rc;
  const bool whole = start == 0 && end == c->cap;
  std::vector<double**> rows = {&c->time, &c->p, &c->lon, &c->lat,
                                &c->uvwp[0], &c->uvwp[1], &c->uvwp[2]};
  if (!(c->home_mask & LT_HOME_ISO)) rows.push_back(&c->iso_var);
  if (!(c->home_mask & LT_HOME_ZETA)) rows.push_back(&c->zeta);
  if (!(c->home_mask & LT_HOME_DT)) rows.push_back(&c->dt);
  for (size_t g = 0; g < rows.size(); g += kRowSet) {
    RowSet rs;
    rs.n = static_cast<int>(std::min<size_t>(kRowSet, rows.size() - g));
    for (int k = 0; k < rs.n; ++k) { rs.src[k] = *rows[g + k]; rs.dst[k] = c->pool[k]; }
    CK(launch_permute_rows(rs, vals_out, start, n, c->stream));
    for (int k = 0; k < rs.n; ++k) {
      if (whole) std::swap(*rows[g + k], c->pool[k]);
      else CK(cudaMemcpyAsync(*rows[g + k] + start, c->pool[k] + start, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  for (int g = 0; g < ((c->home_mask & LT_HOME_Q) ? 0 : c->nq); g += kRowSet) {
    RowSet rs;
    rs.n = std::min(kRowSet, c->nq - g);
    for (int k = 0; k < rs.n; ++k) { rs.src[k] = c->q + static_cast<int64_t>(g + k) * c->cap; rs.dst[k] = c->pool[k]; }
    CK(launch_permute_rows(rs, vals_out, start, n, c->stream));
    for (int k = 0; k < rs.n; ++k)
      CK(cudaMemcpyAsync(c->q + static_cast<int64_t>(g + k) * c->cap + start, c->pool[k] + start, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  }
  CK(launch_permute<uint32_t>(keys_in, c->ids, vals_out, start, n, c->stream));
  CK(cudaMemcpyAsync(c->ids + start, keys_in + start, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, c->stream));
  return LT_OK;
}

static int settle(lt_ctx* c) {
  if (!c->pending) return LT_OK;
  c->pending = false;
  return apply_perm(c, c->pend_start, c->pend_n);
}
}  // extern C++

int lt_sort_by_box(lt_ctx* c, int64_t start, int64_t end) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (!(0 <= start && start <= end && end <= c->cap))
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside ensemble of %lld particles",
                (long long)start, (long long)end, (long long)c->cap);
  if (c->use0 < 0) return fail(LT_ERR_STATE, "no met snapshots selected (lt_met_use)");
  if (n_rec(c) >= (int64_t(1) << 32)) return fail(LT_ERR_ARG, "met grid too large for 32-bit box keys");
  if ((rc = ensure_ids(c)) || (rc = ensure_scratch(c))) return rc;
  if (!c->sort_buf &&
      (rc = alloc_dev(reinterpret_cast<void**>(&c->sort_buf), 4 * sizeof(uint32_t) * c->cap, "sort keys")))
    return rc;
  if (end == start) return LT_OK;
  if (c->home_mask && end > c->home_n)
    return fail(LT_ERR_RANGE, "sort range [%lld, %lld) exceeds the home-order id range [0, %lld)",
                (long long)start, (long long)end, (long long)c->home_n);
  if (c->timing) CK(cudaEventRecord(c->ev_start, c->stream));
  rc = c->prec == LT_MET_F64 ? sort_typed<RecD>(c, start, end) : sort_typed<RecF>(c, start, end);
  if (rc) return rc;
  // With every cold row in particle order, the next production-chain step
  // can apply the permutation while it streams the hot rows (lt_run); any
  // other access settles it first.
  const uint32_t cold = LT_HOME_Q | LT_HOME_ZETA | LT_HOME_DT | LT_HOME_ISO;
  c->pend_start = start;
  c->pend_n = end - start;
  c->pending = true;
  if (!(start == 0 && end == c->cap && (c->home_mask & cold) == cold))
    if ((rc = settle(c))) return rc;
  CK(cudaEventRecord(c->compute_mark, c->stream));
  c->marked = true;
  if (c->timing) { CK(cudaEventRecord(c->ev_stop, c->stream)); c->timed_once = true; }
  return LT_OK;
}

static int ordered_copy(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt,
                        int64_t first_id, void* host, bool to_host) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (field == LT_F_ID || field == LT_F_RND_CONV || field == LT_F_RND_TURB || field == LT_F_RND_MESO)
    return fail(LT_ERR_ARG, "ordered copies apply to per-particle state fields only");
  int64_t len;
  double* p = field_ptr(c, field, row, &len, &rc);
  if (rc || (rc = slice_check(c, off, cnt, len))) return rc;
  if (!c->ids) {  // never sorted: plain copy
    return to_host ? lt_field_d2h(c, field, row, off, cnt, host)
                   : lt_field_h2d(c, field, row, off, cnt, host);
  }
  const uint32_t group = field == LT_F_Q ? LT_HOME_Q : field == LT_F_ZETA ? LT_HOME_ZETA
                         : field == LT_F_DT ? LT_HOME_DT : field == LT_F_ISO_VAR ? LT_HOME_ISO : 0u;
  if (group & c->home_mask) {  // particle order already: contiguous at id - home_base
    const int64_t at = first_id - c->home_base;
    if ((rc = slice_check(c, at, cnt, len))) return rc;
    return to_host ? lt_field_d2h(c, field, row, at, cnt, host)
                   : lt_field_h2d(c, field, row, at, cnt, host);
  }
  if ((rc = ensure_scratch(c))) return rc;
  if (cnt == 0) return LT_OK;
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  if (to_host) {
    CK(launch_unsort(c->scratch, p, c->ids, off, cnt, first_id, c->bad, 1, c->stream));
    CK(cudaMemcpyAsync(host, c->scratch, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->stream));
  } else {
    CK(cudaMemcpyAsync(c->scratch, host, sizeof(double) * cnt, cudaMemcpyHostToDevice, c->stream));
    CK(launch_resort(p, c->scratch, c->ids, off, cnt, first_id, c->bad, 1, c->stream));
  }
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (bad) return fail(LT_ERR_ARG, "particle ids of [%lld, %lld) are not a permutation of [%lld, %lld)",
                       (long long)off, (long long)(off + cnt), (long long)first_id,
                       (long long)(first_id + cnt));
  return LT_OK;
}

int lt_field_d2h_ordered(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt,
                         int64_t first_id, void* host) {
  return ordered_copy(c, field, row, off, cnt, first_id, host, true);
}

int lt_field_h2d_ordered(lt_ctx* c, int32_t field, int32_t row, int64_t off, int64_t cnt,
                         int64_t first_id, const void* host) {
  return ordered_copy(c, field, row, off, cnt, first_id, const_cast<void*>(host), false);
}

// ------------------------------------------------------------------ output statistics

int lt_grid_counts(lt_ctx* c, int32_t nx, int32_t ny, int64_t start, int64_t end, int64_t* counts) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (nx < 1 || ny < 1) return fail(LT_ERR_ARG, "grid needs nx, ny >= 1");
  if (!(0 <= start && start <= end && end <= c->cap))
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside ensemble of %lld particles",
                (long long)start, (long long)end, (long long)c->cap);
  const size_t nb = static_cast<size_t>(nx) * ny;
  unsigned long long* dev = nullptr;
  if ((rc = alloc_dev(reinterpret_cast<void**>(&dev), sizeof(unsigned long long) * nb, "grid counts")))
    return rc;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  cudaError_t e = cudaMemsetAsync(dev, 0, sizeof(unsigned long long) * nb, c->stream);
  if (e == cudaSuccess) e = launch_grid_counts(c->lon, c->lat, start, end - start, nx, ny, dev, sms, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(counts, dev, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dev);
  CK(e);
  return LT_OK;
}

int lt_group_stats(lt_ctx* c, int32_t slot, int64_t start, int64_t end, int64_t max_groups,
                   int64_t* ngroups, int64_t* gid, int64_t* count, double* mean, double* std_) {
  int rc = check_ctx(c);
  if (rc || (rc = check_particles(c))) return rc;
  if ((rc = settle(c))) return rc;
  if (slot < 0 || slot >= c->nq)
    return fail(LT_ERR_ARG, "ens_group_slot %d is not a valid quantity slot", slot);
  if (!(0 <= start && start <= end && end <= c->cap))
    return fail(LT_ERR_RANGE, "range [%lld, %lld) outside ensemble of %lld particles",
                (long long)start, (long long)end, (long long)c->cap);
  if (max_groups < 0) return fail(LT_ERR_ARG, "max_groups < 0");
  *ngroups = 0;
  const int64_t n = end - start;
  if (n == 0) return LT_OK;
  const double* qrow = c->q + static_cast<int64_t>(slot) * c->cap;
  size_t need = 0;
  int64_t ng = 0;
  std::vector<uint32_t> g32(std::max<int64_t>(max_groups, 1));
  std::vector<double> m(3 * std::max<int64_t>(max_groups, 1)), sd(m.size());
  const int64_t qbase = (c->home_mask & LT_HOME_Q) && c->ids ? c->home_base : -1;
  CK(group_stats(c->lon, c->lat, c->p, qrow, c->ids, qbase, start, n, max_groups, nullptr, 0, &need,
                 c->bad, &ng, g32.data(), count, m.data(), sd.data(), c->stream));
  void* ws = nullptr;
  if ((rc = alloc_dev(&ws, need, "group stats workspace"))) return rc;
  cudaError_t e = cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream);
  if (e == cudaSuccess)
    e = group_stats(c->lon, c->lat, c->p, qrow, c->ids, qbase, start, n, max_groups, ws, need, &need,
                    c->bad, &ng, g32.data(), count, m.data(), sd.data(), c->stream);
  int bad = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&bad, c->bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(ws);
  CK(e);
  *ngroups = ng;
  if (bad) return fail(LT_ERR_ARG, bad == 1 ? "group ids must be non-negative" : "group id exceeds 2^32");
  if (ng > max_groups)
    return fail(LT_ERR_RANGE, "%lld groups exceed max_groups %lld", (long long)ng, (long long)max_groups);
  for (int64_t g = 0; g < ng; ++g) {
    gid[g] = g32[g];
    for (int f = 0; f < 3; ++f) {
      mean[f * max_groups + g] = m[f * ng + g];
      std_[f * max_groups + g] = sd[f * ng + g];
    }
  }
  return LT_OK;
}

// ------------------------------------------------------------------ timing / host memory

int lt_sort_info(lt_ctx* c, int64_t* sorts, int64_t* sorts_with_step_keys) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  if (!sorts || !sorts_with_step_keys) return fail(LT_ERR_ARG, "null output");
  *sorts = c->n_sorts;
  *sorts_with_step_keys = c->n_sorts_fused;
  return LT_OK;
}

int lt_timing(lt_ctx* c, int32_t enable) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  c->timing = enable != 0;
  return LT_OK;
}

int lt_last_elapsed_ms(lt_ctx* c, float* ms) {
  int rc = check_ctx_keep(c);
  if (rc) return rc;
  if (!c->timed_once) return fail(LT_ERR_STATE, "no timed launch recorded");
  CK(cudaEventSynchronize(c->ev_stop));
  CK(cudaEventElapsedTime(ms, c->ev_start, c->ev_stop));
  return LT_OK;
}

int lt_host_alloc(int64_t bytes, void** out) {
  CK(cudaHostAlloc(out, static_cast<size_t>(bytes), cudaHostAllocPortable));
  return LT_OK;
}

int lt_host_free(void* p) {
  CK(cudaFreeHost(p));
  return LT_OK;
}

}  // extern "C"
