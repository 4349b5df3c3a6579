// Lazily built, immutable device tables (see xft_tables.h).
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/xft_b200.h"
#include "xft_tables.h"

namespace xftb {

double2 host_kernel_prefactor(int64_t n) {
  // C(n) = pi/sqrt(2n) * exp(-i pi ((n-1)^2 mod 4n) / (2n))   (xft/kernel.py:45-48)
  const long double nn = (long double)n;
  const int64_t red = (int64_t)(((__int128)(n - 1) * (n - 1)) % (4 * (__int128)n));
  const double mag = M_PI / std::sqrt(2.0 * (double)n);
  const long double th = 3.141592653589793238462643383279502884L * (long double)red / (2.0L * nn);
  return make_double2(mag * (double)cosl(th), -mag * (double)sinl(th));
}

double host_half_step(int64_t n) { return (M_PI / std::sqrt(2.0 * (double)n)) / 2.0; }

namespace {

struct Entry {
  void* tw = nullptr;
  void* ptab = nullptr;
};

std::mutex g_mu;
std::map<std::tuple<int, int64_t, int>, Entry> g_tables;

template <class T2, class R>
void fill(std::vector<T2>& tw, std::vector<T2>& pt, int64_t n) {
  const long double PI_L = 3.141592653589793238462643383279502884L;
  for (int64_t m = 0; m < n; ++m) {
    const long double th = 2.0L * PI_L * (long double)m / (long double)n;
    tw[m].x = (R)cosl(th);
    tw[m].y = (R)(-sinl(th));
    // p_k = exp(+i pi ((n-1)k mod 2n) / n)   (xft/kernel.py:51-65)
    const int64_t red = (int64_t)(((__int128)(n - 1) * m) % (2 * (__int128)n));
    const long double ph = PI_L * (long double)red / (long double)n;
    pt[m].x = (R)cosl(ph);
    pt[m].y = (R)sinl(ph);
  }
}

}  // namespace

int get_tables(int64_t n, int dtype, Tables* out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  out->cn = host_kernel_prefactor(n);
  out->half = host_half_step(n);
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, n, dtype);
  auto it = g_tables.find(key);
  if (it == g_tables.end()) {
    Entry e;
    const size_t esz = dtype == XFT_C64 ? sizeof(float2) : sizeof(double2);
    const size_t bytes = esz * (size_t)n;
    if (cudaMalloc(&e.tw, bytes) != cudaSuccess) return XFT_ECUDA;
    if (cudaMalloc(&e.ptab, bytes) != cudaSuccess) return XFT_ECUDA;
    cudaError_t r1, r2;
    if (dtype == XFT_C64) {
      std::vector<float2> tw(n), pt(n);
      fill<float2, float>(tw, pt, n);
      r1 = cudaMemcpy(e.tw, tw.data(), bytes, cudaMemcpyHostToDevice);
      r2 = cudaMemcpy(e.ptab, pt.data(), bytes, cudaMemcpyHostToDevice);
    } else {
      std::vector<double2> tw(n), pt(n);
      fill<double2, double>(tw, pt, n);
      r1 = cudaMemcpy(e.tw, tw.data(), bytes, cudaMemcpyHostToDevice);
      r2 = cudaMemcpy(e.ptab, pt.data(), bytes, cudaMemcpyHostToDevice);
    }
    if (r1 != cudaSuccess || r2 != cudaSuccess) return XFT_ECUDA;
    it = g_tables.emplace(key, e).first;
  }
  out->tw = it->second.tw;
  out->ptab = it->second.ptab;
  return XFT_OK;
}

}  // namespace xftb
