// Host side of the chirp-z kernels: arbitrary-length DFT / scaled Fourier /
// LCT (xft/fftcore.py:84-100, 116-119) and the complex-z Mehler transform
// (xft/dense.py:122-151).  Plan tables are built once per (device, n, sign,
// dtype, mode) on the host in long double and cached (immutable).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <complex>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/xft_b200.h"
#include "xft_blue.cuh"
#include "xft_internal.h"
#include "xft_tables.h"

using namespace xftb;

namespace {

using cld = std::complex<long double>;
const long double PI_L = 3.141592653589793238462643383279502884L;

constexpr int MAXL_C64 = 14;   // M <= 16384 (128 KiB exchange buffer)
constexpr int MAXL_C128 = 13;  // M <= 8192

// iterative radix-2 FFT, sign s (plan-time only)
void host_fft(std::vector<cld>& a, int s) {
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  std::vector<cld> w;
  for (size_t len = 2; len <= n; len <<= 1) {
    const long double ang = s * 2.0L * PI_L / (long double)len;
    w.resize(len / 2);
    for (size_t k = 0; k < len / 2; ++k) w[k] = cld(cosl(ang * k), sinl(ang * k));  // once per stage
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const cld u = a[i + k], v = a[i + k + len / 2] * w[k];
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

struct CzPlan {
  double2* pre = nullptr;
  double2* post = nullptr;
  double2* hspec = nullptr;
  int64_t m = 0;
};

std::mutex g_mu;
std::map<std::tuple<int, int64_t, int, int>, CzPlan> g_plans;  // (dev, n, sign, mode)

int get_plan(int64_t n, int sign, int mode, CzPlan* out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, n, sign, mode);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    *out = it->second;
    return XFT_OK;
  }
  int64_t m = 1;
  while (m < 2 * n - 1) m *= 2;
  // chirp_k = exp(s i pi (k^2 mod 2n) / n)           (xft/fftcore.py:88-90)
  std::vector<cld> chirp(n), filt(m, cld(0, 0));
  for (int64_t k = 0; k < n; ++k) {
    const int64_t r = (int64_t)(((__int128)k * k) % (2 * (__int128)n));
    const long double th = sign * PI_L * (long double)r / (long double)n;
    chirp[k] = cld(cosl(th), sinl(th));
  }
  for (int64_t k = 0; k < n; ++k) filt[k] = std::conj(chirp[k]);  // xft/fftcore.py:91-93
  for (int64_t k = 1; k < n; ++k) filt[m - k] = std::conj(chirp[k]);
  host_fft(filt, -1);
  std::vector<double2> pre(n), post(n), hs(m);
  // C(n) and p_k for the scaled-Fourier / LCT wrappers (xft/kernel.py:45-65)
  const int64_t red = (int64_t)(((__int128)(n - 1) * (n - 1)) % (4 * (__int128)n));
  const cld cn = (PI_L / sqrtl(2.0L * n)) * cld(cosl(PI_L * red / (2.0L * n)), -sinl(PI_L * red / (2.0L * n)));
  for (int64_t k = 0; k < n; ++k) {
    cld a = chirp[k], b = chirp[k] / (long double)m;
    if (mode != 0) {
      const int64_t rk = (int64_t)(((__int128)(n - 1) * k) % (2 * (__int128)n));
      const cld p(cosl(PI_L * rk / (long double)n), sinl(PI_L * rk / (long double)n));
      a *= p;
      b *= p * cn;
    }
    pre[k] = make_double2((double)a.real(), (double)a.imag());
    post[k] = make_double2((double)b.real(), (double)b.imag());
  }
  for (int64_t k = 0; k < m; ++k) hs[k] = make_double2((double)filt[k].real(), (double)filt[k].imag());
  CzPlan p;
  p.m = m;
  if (cudaMalloc(&p.pre, n * sizeof(double2)) != cudaSuccess) return XFT_ECUDA;
  if (cudaMalloc(&p.post, n * sizeof(double2)) != cudaSuccess) return XFT_ECUDA;
  if (cudaMalloc(&p.hspec, m * sizeof(double2)) != cudaSuccess) return XFT_ECUDA;
  if (cudaMemcpy(p.pre, pre.data(), n * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p.post, post.data(), n * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p.hspec, hs.data(), m * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess)
    return XFT_ECUDA;
  g_plans.emplace(key, p);
  *out = p;
  return XFT_OK;
}

template <class C, int L, class Op>
int launch_blue(const void* in, void* out, long long rows, const int* rowlist, const Op& op, cudaStream_t st) {
  if constexpr (L < 2) {
    return XFT_ENOTSUP;
  } else {
    constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
    constexpr int E = blue_radix(dtype, L);
    using BC = BlueStage<C, L, E, Op>;  // (SMEM: the exchange buffer + the Mehler apply CTAs' spectrum stage)
    constexpr int TR = (1 << L) / E;
    auto kern = xft_blue_kernel<C, L, E, Op>;
    Tables tb;
    int rc = get_tables(int64_t(1) << L, dtype, &tb, E);
    if (rc) return rc;
    if (BC::SMEM > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BC::SMEM) != cudaSuccess)
      return XFT_ECUDA;
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TR, BC::SMEM);
    const long long cap = (long long)sms * (occ < 1 ? 1 : (occ > 8 ? 8 : occ));  // Mehler scratch: <= 8 rows/SM
    const long long grid = rows < cap ? rows : cap;
    kern<<<(unsigned)grid, TR, BC::SMEM, st>>>(static_cast<const C*>(in), static_cast<C*>(out), rows, rowlist, op,
                                                   static_cast<const C*>(tb.tw));
    return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
  }
}

template <class C, class Op, int... Ls>
int dispatch_blue(int l, const void* in, void* out, long long rows, const int* rowlist, const Op& op,
                  cudaStream_t st, std::integer_sequence<int, Ls...>) {
  int rc = XFT_ENOTSUP;
  ((l == Ls ? (rc = launch_blue<C, Ls, Op>(in, out, rows, rowlist, op, st), 0) : 0), ...);
  return rc;
}

template <class C, class Op>
int blue(int l, const void* in, void* out, long long rows, const int* rowlist, const Op& op, cudaStream_t st) {
  constexpr int MAXL = sizeof(C) == 8 ? MAXL_C64 : MAXL_C128;
  if (l < 2 || l > MAXL) return XFT_ENOTSUP;
  return dispatch_blue<C, Op>(l, in, out, rows, rowlist, op, st, std::make_integer_sequence<int, MAXL + 1>{});
}

int log2_ceil(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

}  // namespace

namespace xftb {

int64_t chirpz_max_m(int dtype) { return int64_t(1) << (dtype == XFT_C64 ? MAXL_C64 : MAXL_C128); }

int run_chirpz(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
               int64_t stride, const double* uni4, int flags, cudaStream_t st) {
  if (n < 2) return XFT_EINVALID_SIZE;
  int64_t m = 1;
  while (m < 2 * n - 1) m *= 2;
  CzPlan p;
  int rc = get_plan(n, mode == 0 ? sign : -1, mode == 0 ? 0 : 1, &p);
  if (rc) return rc;
  if (m > chirpz_max_m(dtype))  // beyond one CTA: the four-step convolution
    return run_large_chirpz(mode == 2, (flags & XFT_FLAG_BARE_FOURIER) ? 1 : 0, in, out, batch, n, dtype, abcd, stride,
                            uni4, p.pre, p.post, p.hspec, m, st);
  OpChirpZ op;
  op.pre = p.pre;
  op.post = p.post;
  op.hspec = p.hspec;
  op.abcd = abcd;
  op.abcd_stride = stride;
  op.uni = uni4 ? Abcd{uni4[0], uni4[1], uni4[2], uni4[3]} : Abcd{0, 0, 0, 0};
  op.half = host_half_step(n);
  op.n = (int)n;
  op.lct = mode == 2;
  op.bare = (flags & XFT_FLAG_BARE_FOURIER) ? 1 : 0;
  const int l = log2_ceil(m);
  return dtype == XFT_C64 ? blue<float2>(l, in, out, batch, nullptr, op, st)
                          : blue<double2>(l, in, out, batch, nullptr, op, st);
}

}  // namespace xftb

// ---------------------------------------------------------------------------
// Mehler (complex-z fractional transform)
// ---------------------------------------------------------------------------
namespace {

struct MehlerPlanRow {
  OpMehlerRow p;
  int l;
};

MehlerPlanRow mehler_row(std::complex<double> z, int64_t n) {
  using cd = std::complex<double>;
  const double half = host_half_step(n);
  const cd one = 1.0 - z * z;
  const cd A = std::sqrt(2.0 / one);                     // principal branch, xft/dense.py:135
  const cd Q = 2.0 * z / one;
  const int sigma = Q.real() >= 0.0 ? 1 : -1;
  // gamma' = P - sigma Q/2 in closed form (no cancellation near z = +-1)
  const cd gam = sigma > 0 ? (1.0 - z) / (2.0 * (1.0 + z)) : (1.0 + z) / (2.0 * (1.0 - z));
  const cd beta = 2.0 * (double)sigma * Q * half * half;  // h(l) = exp(-beta l^2)
  // window: keep samples with exp(-Re(gam) x^2) > 1e-20 (|x| < sqrt(46 / Re gam))
  int64_t k0 = 0;
  if (gam.real() > 0.0) {
    const double xc = std::sqrt(46.0 / gam.real());
    const double kk = std::ceil(xc / (2.0 * half)) + 1.0;
    if (kk < n / 2) k0 = n / 2 - (int64_t)kk;
  }
  const int64_t wn = n - 2 * k0;
  int64_t m = 1;
  while (m < 2 * wn - 1) m *= 2;
  if (m < 4) m = 4;
  const cd scale = (2.0 * half) * A / (double)m;
  MehlerPlanRow r;
  r.p.gam = make_double2(gam.real(), gam.imag());
  r.p.beta = make_double2(beta.real(), beta.imag());
  r.p.scale = make_double2(scale.real(), scale.imag());
  r.p.k0 = (int)k0;
  r.p.wn = (int)wn;
  r.p.sigma = sigma;
  r.p.pad = 0;
  r.l = log2_ceil(m);
  return r;
}

}  // namespace

// A Mehler "plan": the per-row parameters, size classes and row lists of one
// z array (the B200 analogue of frft_matrix_asymptotic's DenseTransform,
// xft/dense.py:139-151), built on the host once and kept on the device.  Calls
// with the same (n, z) reuse it: no host work, no copies, no synchronisation.
// Immutable once built; shared (refcounted) between the implicit cache and
// every call using it.  It also keeps the exact z values it was built from, so
// a cache hit is an exact match, never a hash match.
struct MehlerPlan {
  int dev = 0;
  int64_t batch = 0, n = 0;
  std::vector<double> z;                    // [batch][2] as used (z_stride 0 -> one row repeated)
  OpMehlerRow* rows = nullptr;              // [batch] device
  int* list = nullptr;                      // [batch] device, rows grouped by class
  std::vector<std::pair<int, long long>> classes;  // (log2 M, count) in list order
  // kernel spectra FFT(h) of every row ([class rows][M] per class, four-step classes in their
  // permuted order): functions of z alone, computed once when the plan is built
  double2* hspec = nullptr;
  std::vector<size_t> hoff;  // element offset of each class in hspec
  int maxl = 0;
  ~MehlerPlan() {
    if (rows || list || hspec) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaFree(rows);
      cudaFree(list);
      cudaFree(hspec);
      cudaSetDevice(cur);
    }
  }
};

namespace xftb {
SideStreams& side_streams(int dev, cudaStream_t caller, int count) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SideStreams*> pool;
  std::lock_guard<std::mutex> lock(mu);
  SideStreams*& p = pool[{dev, caller}];
  if (!p) {
    p = new SideStreams();
    if (cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming) != cudaSuccess) p->ok = false;
  }
  while (p->ok && (int)p->st.size() < count) {
    cudaStream_t s = nullptr;
    cudaEvent_t e = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      p->ok = false;
      break;
    }
    p->st.push_back(s);
    p->join.push_back(e);
  }
  return *p;
}
}  // namespace xftb

namespace {
// Runs `f` with this thread's stream-capture mode relaxed, so plan/scratch
// allocation (cudaMalloc, a pageable cudaMemcpy) is legal while the caller's
// stream is being captured into a CUDA graph; the mode is restored after.
template <class F>
auto relaxed_capture(F&& f) {
  cudaStreamCaptureMode m = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&m);
  auto r = f();
  cudaThreadExchangeStreamCaptureMode(&m);
  return r;
}

// Device memory that graphs captured earlier may still reference is never
// freed implicitly: superseded scratch buffers and evicted plans are retired
// here and released only by xft_release_caches() (the caller's promise that no
// pending work or live graph uses them).
struct Retired {
  std::mutex mu;
  std::vector<std::pair<int, void*>> buffers;
  std::vector<std::shared_ptr<const MehlerPlan>> plans;
};
Retired& retired() {
  static Retired* r = new Retired();  // leaked on purpose: outlives static destruction order
  return *r;
}

struct ScratchPool {
  std::mutex mu;
  std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> pool;
};
ScratchPool& scratch_pool() {
  static ScratchPool* p = new ScratchPool();
  return *p;
}

struct PlanCache {
  std::mutex mu;
  // (device, batch, n, FNV-1a of z) -> plans with that key (exact z compared on lookup)
  std::map<std::tuple<int, int64_t, int64_t, uint64_t>, std::vector<std::shared_ptr<const MehlerPlan>>> map;
  std::vector<std::shared_ptr<const MehlerPlan>> lru;  // most recently used last
};
PlanCache& plan_cache() {
  static PlanCache* c = new PlanCache();
  return *c;
}
constexpr size_t PLAN_CACHE_ENTRIES = 64;

std::vector<double> gather_z(int64_t batch, const double* z, int64_t z_stride) {
  std::vector<double> v(2 * batch);
  for (int64_t r = 0; r < batch; ++r) {
    const double* zz = z + (z_stride ? r * z_stride : 0);
    v[2 * r] = zz[0];
    v[2 * r + 1] = zz[1];
  }
  return v;
}

uint64_t fnv1a(const std::vector<double>& v) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
  for (size_t i = 0; i < v.size() * sizeof(double); ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

// builds a plan for the (already validated) z values on device `dev`
int build_mehler_plan(int dev, int64_t batch, int64_t n, std::vector<double> zv,
                      std::shared_ptr<const MehlerPlan>* out) {
  auto p = std::make_shared<MehlerPlan>();
  p->dev = dev;
  p->batch = batch;
  p->n = n;
  std::vector<OpMehlerRow> rows(batch);
  std::map<int, std::vector<int>> classes;
  for (int64_t r = 0; r < batch; ++r) {
    const MehlerPlanRow pr = mehler_row(std::complex<double>(zv[2 * r], zv[2 * r + 1]), n);
    rows[r] = pr.p;
    classes[pr.l].push_back((int)r);
  }
  std::vector<int> list;
  list.reserve(batch);
  for (auto& kv : classes) {
    list.insert(list.end(), kv.second.begin(), kv.second.end());
    p->classes.emplace_back(kv.first, (long long)kv.second.size());
    if (kv.first <= MAXL_C128) p->maxl = kv.first;
  }
  p->z = std::move(zv);
  size_t hs_elems = 0;
  for (const auto& cl : p->classes) {
    p->hoff.push_back(hs_elems);
    hs_elems += (size_t)cl.second << cl.first;
  }
  // the kernel spectra run on a private stream and are waited for here: plan creation is
  // host-synchronous (like the uploads above) and stays outside any graph being captured
  const int rc = relaxed_capture([&]() -> int {
    if (cudaMalloc(&p->rows, batch * sizeof(OpMehlerRow)) != cudaSuccess ||
        cudaMalloc(&p->list, batch * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&p->hspec, hs_elems * sizeof(double2)) != cudaSuccess ||
        cudaMemcpy(p->rows, rows.data(), batch * sizeof(OpMehlerRow), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->list, list.data(), batch * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
      return XFT_ECUDA;
    cudaStream_t ps = nullptr;
    if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) != cudaSuccess) return XFT_ECUDA;
    int r = XFT_OK;
    size_t off = 0;
    for (size_t c = 0; c < p->classes.size() && !r; ++c) {
      const auto& cl = p->classes[c];
      if (cl.first <= MAXL_C128) {
        OpMehlerSpec op;
        op.rows = p->rows;
        op.hscratch = p->hspec + p->hoff[c];
        op.half = host_half_step(n);
        op.n = (int)n;
        r = blue<double2>(cl.first, nullptr, nullptr, cl.second, p->list + off, op, ps);
      } else {
        r = large_mehler_spectrum(cl.second, p->list + off, p->rows, cl.first, p->hspec + p->hoff[c], ps);
      }
      off += (size_t)cl.second;
    }
    if (cudaStreamSynchronize(ps) != cudaSuccess && !r) r = XFT_ECUDA;
    cudaStreamDestroy(ps);
    return r;
  });
  if (rc) {
    cudaGetLastError();
    return rc;  // ~MehlerPlan frees what was allocated
  }
  *out = std::move(p);
  return XFT_OK;
}

// the implicit per-process cache behind xft_mehler: exact-z lookup, bounded LRU;
// evicted plans are retired (not freed), so graphs captured with them stay valid
int cached_mehler_plan(int dev, int64_t batch, int64_t n, const double* z, int64_t z_stride,
                       std::shared_ptr<const MehlerPlan>* out) {
  std::vector<double> zv = gather_z(batch, z, z_stride);
  const auto key = std::make_tuple(dev, batch, n, fnv1a(zv));
  PlanCache& c = plan_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (const auto& p : c.map[key]) {
    if (p->z == zv) {  // exact match of every value (a hash collision cannot alias two z arrays)
      auto pos = std::find(c.lru.begin(), c.lru.end(), p);
      if (pos != c.lru.end()) std::rotate(pos, pos + 1, c.lru.end());
      *out = p;
      return XFT_OK;
    }
  }
  std::shared_ptr<const MehlerPlan> p;
  int rc = build_mehler_plan(dev, batch, n, std::move(zv), &p);
  if (rc) return rc;
  if (c.lru.size() >= PLAN_CACHE_ENTRIES) {
    std::shared_ptr<const MehlerPlan> old = c.lru.front();
    c.lru.erase(c.lru.begin());
    auto& bucket = c.map[std::make_tuple(old->dev, old->batch, old->n, fnv1a(old->z))];
    bucket.erase(std::remove(bucket.begin(), bucket.end(), old), bucket.end());
    std::lock_guard<std::mutex> rl(retired().mu);
    retired().plans.push_back(std::move(old));
  }
  c.map[key].push_back(p);
  c.lru.push_back(p);
  *out = std::move(p);
  return XFT_OK;
}
}  // namespace

// Per-(device, stream) scratch, grown on demand and never shrunk.  Growth
// allocates a new buffer and retires the old one (work already queued, or a
// graph captured earlier, may still use it): no synchronisation, legal during
// stream capture.
void* xftb::stream_scratch(int dev, cudaStream_t st, size_t bytes) {
  ScratchPool& sp = scratch_pool();
  std::lock_guard<std::mutex> lock(sp.mu);
  auto& e = sp.pool[{dev, st}];
  if (e.second < bytes) {
    void* p = nullptr;
    if (!relaxed_capture([&]() { return cudaMalloc(&p, bytes) == cudaSuccess; })) {
      cudaGetLastError();
      return nullptr;
    }
    if (e.first) {
      std::lock_guard<std::mutex> rl(retired().mu);
      retired().buffers.emplace_back(dev, e.first);
    }
    e.first = p;
    e.second = bytes;
  }
  return e.first;
}

namespace {
// one Mehler transform with a resolved plan (stream-ordered, capturable)
int mehler_run(const void* in, void* out, const MehlerPlan& plan, void* workspace, cudaStream_t st) {
  const int dev = plan.dev;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n = plan.n;
  int rc = XFT_OK;
  // scratch: the four-step classes' data rows (count x M each); the kernel spectra are the plan's
  size_t all_bytes = 0;
  for (const auto& cl : plan.classes)
    if (cl.first > MAXL_C128) all_bytes += (size_t)cl.second * ((size_t)1 << cl.first) * 16;
  OpMehler op;
  op.rows = plan.rows;
  op.half = host_half_step(n);
  op.n = (int)n;
  if (workspace) {  // caller scratch (xft_mehler_workspace_bytes): the classes one after another
    size_t off = 0;
    for (size_t c = 0; c < plan.classes.size(); ++c) {
      const auto& cl = plan.classes[c];
      const long long cnt = cl.second;
      OpMehler oc = op;
      oc.hscratch = plan.hspec + plan.hoff[c];
      rc = cl.first <= MAXL_C128 ? blue<double2>(cl.first, in, out, cnt, plan.list + off, oc, st)
                                 : run_large_mehler(in, out, cnt, plan.list + off, plan.rows, cl.first, n, st,
                                                    workspace, plan.hspec + plan.hoff[c]);
      if (rc) return rc;
      off += cnt;
    }
    return XFT_OK;
  }
  // Size classes are disjoint row sets: each runs on its own internal stream
  // (forked from and joined back to `st`, so the call stays stream-ordered and
  // graph-capturable) with its own scratch, and the small in-CTA classes fill
  // the SMs the four-step classes' short tile kernels leave idle.
  char* base = static_cast<char*>(stream_scratch(dev, st, all_bytes > 0 ? all_bytes : 16));
  if (!base) return XFT_ECUDA;
  SideStreams& ss = side_streams(dev, st, (int)plan.classes.size());
  if (!ss.ok) return XFT_ECUDA;
  std::lock_guard<std::mutex> lock(ss.mu);
  if (cudaEventRecord(ss.fork, st) != cudaSuccess) return XFT_ECUDA;
  size_t forked = 0, off = 0, boff = 0;
  for (size_t c = 0; c < plan.classes.size() && !rc; ++c) {
    const auto& cl = plan.classes[c];
    const long long cnt = cl.second;
    cudaStream_t sc = ss.st[c];
    if (cudaStreamWaitEvent(sc, ss.fork, 0) != cudaSuccess) {
      rc = XFT_ECUDA;
      break;
    }
    forked = c + 1;
    if (cl.first <= MAXL_C128) {
      OpMehler oc = op;
      oc.hscratch = plan.hspec + plan.hoff[c];
      rc = blue<double2>(cl.first, in, out, cnt, plan.list + off, oc, sc);
    } else {
      rc = run_large_mehler(in, out, cnt, plan.list + off, plan.rows, cl.first, n, sc, base + boff,
                            plan.hspec + plan.hoff[c]);
      boff += (size_t)cnt * ((size_t)1 << cl.first) * 16;
    }
    off += cnt;
  }
  for (size_t c = 0; c < forked; ++c) {  // join every forked stream (also after an error: `st` stays consistent)
    if (cudaEventRecord(ss.join[c], ss.st[c]) != cudaSuccess || cudaStreamWaitEvent(st, ss.join[c], 0) != cudaSuccess)
      rc = rc ? rc : XFT_ECUDA;
  }
  return rc;
}
}  // namespace

extern "C" {

int64_t xft_mehler_workspace_bytes(int64_t batch, int64_t n) {
  // the four-step classes' data rows: at most every row at the largest convolution length
  int64_t m = 1;
  while (m < 2 * n - 1) m *= 2;
  return batch * m * 16 + 4096;
}

int xft_mehler(const void* in, void* out, int64_t batch, int64_t n, const double* z, int64_t z_stride,
               void* workspace, void* stream) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  int rc = xft_validate_mehler_z(z, batch, z_stride, nullptr);
  if (rc) return rc;
  if (batch == 0) return XFT_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::shared_ptr<const MehlerPlan> plan;  // held for the whole call: eviction cannot free it under us
  if ((rc = cached_mehler_plan(dev, batch, n, z, z_stride, &plan))) return rc;
  return mehler_run(in, out, *plan, workspace, static_cast<cudaStream_t>(stream));
}

int xft_mehler_plan_create(int64_t batch, int64_t n, const double* z, int64_t z_stride, void** plan) {
  if (!plan) return XFT_EPARAM;
  *plan = nullptr;
  if (n < 1 || batch < 1) return XFT_EINVALID_SIZE;
  int rc = xft_validate_mehler_z(z, batch, z_stride, nullptr);
  if (rc) return rc;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::shared_ptr<const MehlerPlan> p;
  if ((rc = build_mehler_plan(dev, batch, n, gather_z(batch, z, z_stride), &p))) return rc;
  *plan = new std::shared_ptr<const MehlerPlan>(std::move(p));
  return XFT_OK;
}

int xft_mehler_plan_destroy(void* plan) {
  delete static_cast<std::shared_ptr<const MehlerPlan>*>(plan);
  return XFT_OK;
}

int xft_mehler_planned(const void* in, void* out, const void* plan, void* workspace, void* stream) {
  if (!plan) return XFT_EPARAM;
  const auto& p = *static_cast<const std::shared_ptr<const MehlerPlan>*>(plan);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  if (dev != p->dev) return XFT_EPARAM;  // a plan lives on the device it was created on
  return mehler_run(in, out, *p, workspace, static_cast<cudaStream_t>(stream));
}

int xft_release_caches(void) {
  std::vector<std::shared_ptr<const MehlerPlan>> drop;
  {
    PlanCache& c = plan_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    drop.swap(c.lru);
    c.map.clear();
  }
  std::vector<std::pair<int, void*>> bufs;
  {
    std::lock_guard<std::mutex> rl(retired().mu);
    for (auto& p : retired().plans) drop.push_back(std::move(p));
    retired().plans.clear();
    bufs.swap(retired().buffers);
  }
  {
    ScratchPool& sp = scratch_pool();
    std::lock_guard<std::mutex> lock(sp.mu);
    for (auto& kv : sp.pool)
      if (kv.second.first) bufs.emplace_back(kv.first.first, kv.second.first);
    sp.pool.clear();
  }
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& b : bufs) {
    cudaSetDevice(b.first);
    cudaFree(b.second);
  }
  cudaSetDevice(cur);
  drop.clear();  // plans still held by a caller's handle or an in-flight call survive (refcount)
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

}  // extern "C"
