// lt_host.cpp — host-side output formatting for the drop-in.
//
// output.py:17-25 (write_atm) writes one CSV row per particle with Python's
// repr() of every double — a per-particle interpreter loop that takes hours
// at 1e8 particles.  lt_write_atm produces the same bytes from C++: the
// shortest round-trip digits (std::to_chars), laid out with CPython's
// repr rules (float_repr_style 'short': exponent form when the decimal
// exponent is < -4 or >= 16, at least two exponent digits, '.0' appended to
// integral values), formatted by worker threads chunk by chunk and written
// in order.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lagtrans_b200.h"

namespace {

thread_local std::string g_host_err;

// repr(float) of CPython (Python/pystrtod.c format_float_short, mode 'r')
size_t py_repr(double x, char* out) {
  char* o = out;
  if (std::isnan(x)) { std::memcpy(o, "nan", 3); return 3; }
  if (std::isinf(x)) {
    if (x < 0) *o++ = '-';
    std::memcpy(o, "inf", 3);
    return (o - out) + 3;
  }
  if (std::signbit(x)) { *o++ = '-'; x = -x; }
  if (x == 0.0) { std::memcpy(o, "0.0", 3); return (o - out) + 3; }
  // shortest round-trip digits in scientific form: d[.ddd]e[+-]XX
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  char* e = std::find(buf, r.ptr, 'e');
  char digits[32];
  int nd = 0;
  for (char* c = buf; c < e; ++c)
    if (*c != '.') digits[nd++] = *c;
  int exp10 = 0;
  std::from_chars(e + 1 + (e[1] == '+'), r.ptr, exp10);
  const int decpt = exp10 + 1;  // value = 0.d1d2... * 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      std::memcpy(o, digits + 1, nd - 1);
      o += nd - 1;
    }
    *o++ = 'e';
    int ex = decpt - 1;
    *o++ = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    if (ex < 10) *o++ = '0';
    o = std::to_chars(o, o + 8, ex).ptr;
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int k = 0; k < -decpt; ++k) *o++ = '0';
    std::memcpy(o, digits, nd);
    o += nd;
  } else if (decpt >= nd) {
    std::memcpy(o, digits, nd);
    o += nd;
    for (int k = 0; k < decpt - nd; ++k) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    std::memcpy(o, digits, decpt);
    o += decpt;
    *o++ = '.';
    std::memcpy(o, digits + decpt, nd - decpt);
    o += nd - decpt;
  }
  return o - out;
}

}  // namespace

extern "C" {

int lt_format_double(double x, char* out, int32_t cap, int32_t* len) {
  char buf[40];
  const size_t n = py_repr(x, buf);
  if (static_cast<int32_t>(n) + 1 > cap) return LT_ERR_ARG;
  std::memcpy(out, buf, n);
  out[n] = '\0';
  *len = static_cast<int32_t>(n);
  return LT_OK;
}

int lt_write_atm(const char* path, int64_t n, int32_t nq, const double* time, const double* p,
                 const double* zeta, const double* lon, const double* lat, const double* q,
                 int64_t q_stride, int32_t threads) {
  if (n < 0 || nq < 0 || (nq > 0 && !q) || (n > 0 && (!time || !p || !zeta || !lon || !lat)))
    return LT_ERR_ARG;
  FILE* f = std::fopen(path, "wb");
  if (!f) return LT_ERR_ARG;
  std::string head = "time,p,zeta,lon,lat";
  for (int k = 0; k < nq; ++k) head += ",q" + std::to_string(k);
  head += "\n";
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  const int64_t chunk = 1 << 16;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  int nt = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  nt = static_cast<int>(std::min<int64_t>(nt, std::max<int64_t>(nchunks, 1)));
  // ring of formatted chunks: worker w formats chunks w, w+nt, ...; the
  // calling thread writes them in order
  const int ring = 2 * nt;
  std::vector<std::string> bufs(ring);
  std::vector<int64_t> ready(ring, -1);
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<int64_t> next{0};
  int64_t written = 0;
  auto format = [&](int64_t c, std::string& s) {
    const int64_t lo = c * chunk, hi = std::min(n, lo + chunk);
    s.resize(static_cast<size_t>(hi - lo) * (5 + nq) * 25);
    char* o = s.data();
    for (int64_t i = lo; i < hi; ++i) {
      const double v[5] = {time[i], p[i], zeta[i], lon[i], lat[i]};
      for (int k = 0; k < 5; ++k) {
        o += py_repr(v[k], o);
        *o++ = ',';
      }
      for (int k = 0; k < nq; ++k) {
        o += py_repr(q[k * q_stride + i], o);
        *o++ = ',';
      }
      o[-1] = '\n';
    }
    s.resize(o - s.data());
  };
  auto worker = [&]() {
    std::string local;
    for (;;) {
      const int64_t c = next.fetch_add(1);
      if (c >= nchunks) return;
      format(c, local);
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return c - written < ring; });  // slot free
      bufs[c % ring].swap(local);
      ready[c % ring] = c;
      cv.notify_all();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
  for (int64_t c = 0; c < nchunks; ++c) {
    std::string out;
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return ready[c % ring] == c; });
      out.swap(bufs[c % ring]);
      ready[c % ring] = -1;
      written = c + 1;
      cv.notify_all();
    }
    if (ok) ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
  }
  for (auto& t : pool) t.join();
  ok = (std::fclose(f) == 0) && ok;
  return ok ? LT_OK : LT_ERR_ARG;
}

}  // extern "C"
