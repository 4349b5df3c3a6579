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
std::map<std::pair<int, int>, void*> g_gtab;
std::map<std::tuple<int, int64_t, int, int>, Entry> g_tables;

const long double PI_L = 3.141592653589793238462643383279502884L;

// Pass-major twiddles: for pass p >= 1 (NS = R0 E^(p-1)), entry (t-1)*NS + k
// holds e^{-2 pi i t k / (NS E)}; layout identical to PipeCfg::twoff.
template <class T2, class R>
void fill_twiddles(std::vector<T2>& tw, int64_t n, int E) {
  int l = 0, le = 0;
  while ((int64_t(1) << l) < n) ++l;
  while ((1 << le) < E) ++le;
  tw.clear();
  if (n <= E) return;  // single-pass sizes use no table
  const int npass = (l + le - 1) / le;
  const int64_t r0 = int64_t(1) << (l - (npass - 1) * le);
  int64_t ns = r0;
  for (int p = 1; p < npass; ++p, ns *= E) {
    for (int t = 1; t < E; ++t)
      for (int64_t k = 0; k < ns; ++k) {
        const long double th = 2.0L * PI_L * (long double)(t * k) / (long double)(ns * E);
        T2 w;
        w.x = (R)cosl(th);
        w.y = (R)(-sinl(th));
        tw.push_back(w);
      }
  }
}

template <class T2, class R>
void fill(std::vector<T2>& pt, int64_t n) {
  for (int64_t m = 0; m < n; ++m) {
    // p_k = exp(+i pi ((n-1)k mod 2n) / n)   (xft/kernel.py:51-65)
    const int64_t red = (int64_t)(((__int128)(n - 1) * m) % (2 * (__int128)n));
    const long double ph = PI_L * (long double)red / (long double)n;
    pt[m].x = (R)cosl(ph);
    pt[m].y = (R)sinl(ph);
  }
}

}  // namespace

int get_tables(int64_t n, int dtype, Tables* out, int radix) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  out->cn = host_kernel_prefactor(n);
  out->half = host_half_step(n);
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<int, bool> pool_kept;
  if (!pool_kept[dev]) {
    // stream-ordered scratch of the large-row / Mehler / 2-D paths comes from the
    // default pool: keep freed blocks cached instead of unmapping them at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_kept[dev] = true;
  }
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  const int E = radix > 0 ? radix : pipe_radix(dtype, l);
  auto key = std::make_tuple(dev, n, dtype, E);
  auto it = g_tables.find(key);
  if (it == g_tables.end()) {
    Entry e;
    cudaError_t r1 = cudaSuccess, r2 = cudaSuccess;
    auto upload = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
      if (bytes == 0) bytes = 16;  // keep a valid pointer for empty tables
      cudaError_t r = cudaMalloc(dst, bytes);
      if (r != cudaSuccess) return r;
      return src ? cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
    };
    if (dtype == XFT_C64) {
      std::vector<float2> tw, pt(n);
      fill_twiddles<float2, float>(tw, n, E);
      fill<float2, float>(pt, n);
      r1 = upload(&e.tw, tw.empty() ? nullptr : tw.data(), tw.size() * sizeof(float2));
      r2 = upload(&e.ptab, pt.data(), pt.size() * sizeof(float2));
    } else {
      std::vector<double2> tw, pt(n);
      fill_twiddles<double2, double>(tw, n, E);
      fill<double2, double>(pt, n);
      r1 = upload(&e.tw, tw.empty() ? nullptr : tw.data(), tw.size() * sizeof(double2));
      r2 = upload(&e.ptab, pt.data(), pt.size() * sizeof(double2));
    }
    if (r1 != cudaSuccess || r2 != cudaSuccess) return XFT_ECUDA;
    it = g_tables.emplace(key, e).first;
  }
  auto gt = g_gtab.find({dev, dtype});
  if (gt == g_gtab.end()) {
    // chirp phasor tables: c128 e^{2 pi i m/C128_TABN}, c64 e^{2 pi i m/1024}
    const int tn = dtype == XFT_C64 ? 1024 : C128_TABN;
    std::vector<double2> g(tn);
    std::vector<float2> gf(tn);
    for (int m = 0; m < tn; ++m) {
      const long double th = 2.0L * PI_L * (long double)m / (long double)tn;
      g[m] = make_double2((double)cosl(th), (double)sinl(th));
      gf[m] = make_float2((float)cosl(th), (float)sinl(th));
    }
    const size_t bytes = dtype == XFT_C64 ? tn * sizeof(float2) : tn * sizeof(double2);
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return XFT_ECUDA;
    const void* src = dtype == XFT_C64 ? (const void*)gf.data() : (const void*)g.data();
    if (cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return XFT_ECUDA;
    gt = g_gtab.emplace(std::make_pair(dev, dtype), d).first;
  }
  out->gtab = gt->second;
  out->tw = it->second.tw;
  out->ptab = it->second.ptab;
  return XFT_OK;
}

}  // namespace xftb
