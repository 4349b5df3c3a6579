// Dense O(n^2) transforms on the GPU (SURVEY
// 8(f) item 4: the reference's correctness oracles, made fast enough to check
// full-size rows).  These are *independent* evaluations -- entry by entry from
// the closed-form kernels, no FFT, no chirp factorisation shared with K1 -- of
//   * dense_lct_matrix   L = S1 F S2            (xft/dense.py:230-249)
//   * scaled_fourier_matrix F = C(n) p_j w^{jk mod n} p_k   (xft/kernel.py:68-80)
//   * frft_matrix_asymptotic K_z(x_j, x_k) dx   (xft/dense.py:122-151)
// either applied to vectors (matrix-free, any n) or materialised (n <= 4096,
// the reference's MAX_DENSE_N).  fp64 throughout.
#include <cmath>
#include <complex>
#include <vector>

#include "../../include/xft_b200.h"
#include "xft_blue.cuh"
#include "xft_internal.h"
#include "xft_tables.h"

using namespace xftb;

namespace {

constexpr int64_t MAX_DENSE_N = 4096;  // xft/dense.py:44

__device__ __forceinline__ double2 cdiv_d(double2 a, double2 b) {  // a / b, textbook form
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
__device__ __forceinline__ double2 cexpi(double th) {
  double s, c;
  sincos(th, &s, &c);
  return make_double2(c, s);
}

// per-n / per-parameter vectors of the dense LCT, in the reference's operation order:
//   ic_k = exp((0.5j a/b) x_k^2)                                  xft/kernel.py:98-102
//   oc_j = exp((0.5j d/b) y_j^2) / sqrt(2 pi i b), y = (4b/pi) x  xft/kernel.py:105-113, lct.py:196
//   p_k  = exp(+i pi ((n-1)k mod 2n)/n)                          xft/kernel.py:51-65
struct DenseLct {
  double cin, cout, s4, half;
  double2 rnorm;  // 1 / sqrt(2 pi i b)
  double2 cn;     // C(n)
  int lct;        // 0: plain scaled Fourier matrix F
  int plain;      // 1: the bare DFT kernel e^{sign 2 pi i (jk mod n)/n} (naive_dft): no p, no chirps, C = 1
  int sign;       // DFT sign of w (the LCT / F paths use DFT_SIGN = -1)
};

__global__ void dense_vectors_kernel(DenseLct q, long long n, double2* ic, double2* oc, double2* p, double2* w) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const double x = __dmul_rn((double)(2 * k - n + 1), q.half);  // xft/hermite.py:87-89
    if (q.lct) {
      ic[k] = cexpi(__dmul_rn(q.cin, __dmul_rn(x, x)));
      const double y = __dmul_rn(q.s4, x);
      oc[k] = cmul_d(cexpi(__dmul_rn(q.cout, __dmul_rn(y, y))), q.rnorm);
    } else {
      ic[k] = make_double2(1.0, 0.0);
      oc[k] = make_double2(1.0, 0.0);
    }
    const long long red = (long long)(((__int128)(n - 1) * k) % (2 * (__int128)n));
    double s, c;
    sincospi((double)red / (double)n, &s, &c);
    p[k] = q.plain ? make_double2(1.0, 0.0) : make_double2(c, s);
    sincospi(2.0 * q.sign * (double)k / (double)n, &s, &c);  // w^m = exp(sign 2 pi i m / n)
    w[k] = make_double2(c, s);
  }
}

// out[b][j] = oc_j C p_j sum_k w[(j k) mod n] p_k ic_k in[b][k]   (matrix-free, one CTA per (j-tile, row))
template <int TJ>
__global__ void __launch_bounds__(256) dense_lct_apply_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                             long long n, const double2* __restrict__ ic,
                                                             const double2* __restrict__ oc,
                                                             const double2* __restrict__ p,
                                                             const double2* __restrict__ w, double2 cn) {
  extern __shared__ double2 su[];  // u_k = p_k ic_k in_k for a chunk of k
  const long long row = blockIdx.y;
  const long long j0 = (long long)blockIdx.x * TJ;
  const int t = threadIdx.x;
  const int lane_j = t % TJ, kslot = t / TJ;  // TJ outputs x (256/TJ) k-strides
  constexpr int KS = 256 / TJ;
  const long long j = j0 + lane_j;
  double2 acc = make_double2(0.0, 0.0);
  constexpr int CH = 2048;
  for (long long k0 = 0; k0 < n; k0 += CH) {
    const int cnt = (int)((n - k0) < CH ? (n - k0) : CH);
    __syncthreads();
    for (int i = t; i < cnt; i += 256) {
      const long long k = k0 + i;
      su[i] = cmul_d(cmul_d(p[k], ic[k]), in[row * n + k]);
    }
    __syncthreads();
    if (j < n) {
      long long m = (j * (k0 + kslot)) % n;
      const long long step = (j * KS) % n;
      for (int i = kslot; i < cnt; i += KS) {
        const double2 e = w[m];
        const double2 u = su[i];
        acc.x = fma(e.x, u.x, fma(-e.y, u.y, acc.x));
        acc.y = fma(e.x, u.y, fma(e.y, u.x, acc.y));
        m += step;
        if (m >= n) m -= n;
      }
    }
  }
  // reduce the KS partial sums of each output j
  __shared__ double2 part[256];
  part[t] = acc;
  __syncthreads();
  if (kslot == 0 && j < n) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = 0; q < KS; ++q) {
      s.x += part[q * TJ + lane_j].x;
      s.y += part[q * TJ + lane_j].y;
    }
    out[row * n + j] = cmul_d(cmul_d(cmul_d(oc[j], cn), p[j]), s);
  }
}

// K_z(x_j, x_k) dx in the reference's operation order (xft/dense.py:122-136, 145-149)
struct MehlerDense {
  double2 z, one, opz2, twoone, pref;  // z, 1 - z^2, 1 + z^2, 2(1 - z^2), sqrt(2/(1-z^2))
  double half, dx;
};

__device__ __forceinline__ double2 mehler_entry(const MehlerDense& m, double x, double y) {
  const double r2 = x * x + y * y;
  const double2 a = make_double2(m.opz2.x * r2, m.opz2.y * r2);     // (1+z^2)(x^2+y^2)
  const double xy4 = 4.0 * x * y;
  const double2 bq = make_double2(xy4 * m.z.x, xy4 * m.z.y);       // 4 x y z
  const double2 num = make_double2(-(a.x - bq.x), -(a.y - bq.y));
  const double2 ex = cdiv_d(num, m.twoone);
  const double mag = exp(ex.x);
  double s, c;
  sincos(ex.y, &s, &c);
  const double2 e = make_double2(mag * c, mag * s);
  const double2 k = cmul_d(m.pref, e);
  return make_double2(k.x * m.dx, k.y * m.dx);
}

// g[b][j] = sum_k K_z(x_j, x_k) dx f[b][k]
__global__ void __launch_bounds__(256) dense_mehler_apply_kernel(const double2* __restrict__ in,
                                                                 double2* __restrict__ out, long long n,
                                                                 const MehlerDense* __restrict__ prm,
                                                                 long long prm_stride) {
  const long long row = blockIdx.y;
  const MehlerDense m = prm[row * prm_stride];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long j = (long long)blockIdx.x * 8 + warp;  // one warp per output
  if (j >= n) return;
  const double xj = __dmul_rn((double)(2 * j - n + 1), m.half);
  double2 acc = make_double2(0.0, 0.0);
  for (long long k = lane; k < n; k += 32) {
    const double xk = __dmul_rn((double)(2 * k - n + 1), m.half);
    const double2 kk = mehler_entry(m, xj, xk);
    const double2 f = in[row * n + k];
    acc.x = fma(kk.x, f.x, fma(-kk.y, f.y, acc.x));
    acc.y = fma(kk.x, f.y, fma(kk.y, f.x, acc.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) out[row * n + j] = acc;
}

// materialised n x n entries (kind 0: F, 1: L, 2: Mehler)
__global__ void dense_entries_kernel(double2* __restrict__ out, long long n, int kind, const double2* __restrict__ ic,
                                     const double2* __restrict__ oc, const double2* __restrict__ p,
                                     const double2* __restrict__ w, double2 cn, MehlerDense m) {
  const long long total = n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / n, k = e - j * n;
    if (kind == 2) {
      const double xj = __dmul_rn((double)(2 * j - n + 1), m.half);
      const double xk = __dmul_rn((double)(2 * k - n + 1), m.half);
      out[e] = mehler_entry(m, xj, xk);
    } else {
      // kernel_prefactor * (p[:, None] * dft * p[None, :]), then chirps   (xft/kernel.py:79-80, dense.py:243-247)
      const double2 f = cmul_d(cn, cmul_d(cmul_d(p[j], w[(j * k) % n]), p[k]));
      out[e] = kind == 0 ? f : cmul_d(cmul_d(oc[j], f), ic[k]);
    }
  }
}

DenseLct dense_lct_params(int64_t n, const double* abcd) {
  DenseLct q{};
  q.half = host_half_step(n);
  q.cn = host_kernel_prefactor(n);
  q.sign = -1;
  q.lct = abcd != nullptr;
  if (abcd) {
    const double a = abcd[0], b = abcd[1], d = abcd[3];
    q.cin = (0.5 * a) / b;
    q.cout = (0.5 * d) / b;
    q.s4 = (4.0 * b) / 3.141592653589793116;
    // 1 / sqrt(2 pi i b), principal branch: e^{-i pi sgn(b)/4} / sqrt(2 pi |b|)   (xft/kernel.py:108-113)
    const long double h = 0.70710678118654752440L / sqrtl(2.0L * 3.141592653589793238462643383279502884L * fabsl(b));
    q.rnorm = make_double2((double)h, b > 0.0 ? -(double)h : (double)h);
  }
  return q;
}

MehlerDense mehler_dense_params(int64_t n, double zr, double zi) {
  MehlerDense m{};
  const std::complex<double> z(zr, zi);
  const std::complex<double> one = 1.0 - z * z;
  m.z = make_double2(zr, zi);
  m.one = make_double2(one.real(), one.imag());
  const std::complex<double> opz2 = 1.0 + z * z;
  m.opz2 = make_double2(opz2.real(), opz2.imag());
  const std::complex<double> two = 2.0 * one;
  m.twoone = make_double2(two.real(), two.imag());
  const std::complex<double> pref = std::sqrt(2.0 / one);  // principal branch
  m.pref = make_double2(pref.real(), pref.imag());
  m.half = host_half_step(n);
  m.dx = 2.0 * m.half;  // grid.spacing = pi / sqrt(2n)   (xft/hermite.py:80-84)
  return m;
}

struct Scratch {
  double2 *ic = nullptr, *oc = nullptr, *p = nullptr, *w = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  int alloc(int64_t n) {
    const size_t b = (size_t)n * sizeof(double2);
    if (cudaMallocAsync((void**)&ic, b, st) != cudaSuccess || cudaMallocAsync((void**)&oc, b, st) != cudaSuccess ||
        cudaMallocAsync((void**)&p, b, st) != cudaSuccess || cudaMallocAsync((void**)&w, b, st) != cudaSuccess)
      return XFT_ECUDA;
    return XFT_OK;
  }
  ~Scratch() {
    for (double2* q : {ic, oc, p, w})
      if (q) cudaFreeAsync(q, st);
  }
};

}  // namespace

extern "C" {

int xft_dense_lct_apply(const void* in, void* out, int64_t batch, int64_t n, const double* abcd_host, void* stream) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  if (abcd_host) {
    int rc = xft_validate_lct_params(abcd_host, 1, 0, 0, 0.0, nullptr);  // b == 0 / non-finite only
    if (rc) return rc;
  }
  if (batch == 0) return XFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  Scratch s(st);
  int rc = s.alloc(n);
  if (rc) return rc;
  const DenseLct q = dense_lct_params(n, abcd_host);
  dense_vectors_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(q, n, s.ic, s.oc, s.p, s.w);
  constexpr int TJ = 32;
  dim3 grid((unsigned)((n + TJ - 1) / TJ), (unsigned)batch);
  dense_lct_apply_kernel<TJ><<<grid, 256, 2048 * sizeof(double2), st>>>(
      static_cast<const double2*>(in), static_cast<double2*>(out), n, s.ic, s.oc, s.p, s.w, q.cn);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

int xft_naive_dft(const void* in, void* out, int64_t batch, int64_t n, int sign, void* stream) {
  if (sign != 1 && sign != -1) return XFT_EPARAM;          // xft/fftcore.py:125-126
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;        // 129-130
  if (n > MAX_DENSE_N) return XFT_EINVALID_SIZE;           // _NAIVE_CAP, 131-132
  if (batch == 0) return XFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  Scratch s(st);
  int rc = s.alloc(n);
  if (rc) return rc;
  DenseLct q = dense_lct_params(n, nullptr);
  q.plain = 1;
  q.sign = sign;
  q.cn = make_double2(1.0, 0.0);
  dense_vectors_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(q, n, s.ic, s.oc, s.p, s.w);
  constexpr int TJ = 32;
  dim3 grid((unsigned)((n + TJ - 1) / TJ), (unsigned)batch);
  dense_lct_apply_kernel<TJ><<<grid, 256, 2048 * sizeof(double2), st>>>(
      static_cast<const double2*>(in), static_cast<double2*>(out), n, s.ic, s.oc, s.p, s.w, q.cn);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

int xft_dense_mehler_apply(const void* in, void* out, int64_t batch, int64_t n, const double* z_host,
                           int64_t z_stride, void* stream) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  int rc = xft_validate_mehler_z(z_host, batch, z_stride, nullptr);
  if (rc) return rc;
  if (batch == 0) return XFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t np_ = z_stride ? batch : 1;
  std::vector<MehlerDense> h(np_);
  for (int64_t r = 0; r < np_; ++r) h[r] = mehler_dense_params(n, z_host[r * z_stride], z_host[r * z_stride + 1]);
  MehlerDense* d = nullptr;
  if (cudaMallocAsync((void**)&d, np_ * sizeof(MehlerDense), st) != cudaSuccess) return XFT_ECUDA;
  if (cudaMemcpyAsync(d, h.data(), np_ * sizeof(MehlerDense), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaFreeAsync(d, st);
    return XFT_ECUDA;
  }
  dim3 grid((unsigned)((n + 7) / 8), (unsigned)batch);
  dense_mehler_apply_kernel<<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out), n, d,
                                                 z_stride ? 1 : 0);
  rc = cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
  cudaFreeAsync(d, st);
  // (h is pageable: cudaMemcpyAsync staged it before returning)
  return rc;
}

int xft_dense_entries(void* out, int64_t n, int kind, const double* param_host, void* stream) {
  if (n < 1) return XFT_EINVALID_SIZE;
  if (n > MAX_DENSE_N) return XFT_EINVALID_SIZE;  // xft/dense.py:72-77
  if (kind < 0 || kind > 2) return XFT_EPARAM;
  if (kind == 1) {
    int rc = xft_validate_lct_params(param_host, 1, 0, 0, 0.0, nullptr);
    if (rc) return rc;
  }
  if (kind == 2) {
    int rc = xft_validate_mehler_z(param_host, 1, 0, nullptr);
    if (rc) return rc;
  }
  auto st = static_cast<cudaStream_t>(stream);
  Scratch s(st);
  int rc = s.alloc(n);
  if (rc) return rc;
  const DenseLct q = dense_lct_params(n, kind == 1 ? param_host : nullptr);
  const MehlerDense m = kind == 2 ? mehler_dense_params(n, param_host[0], param_host[1]) : MehlerDense{};
  dense_vectors_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(q, n, s.ic, s.oc, s.p, s.w);
  const long long total = n * n;
  const unsigned grid = (unsigned)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  dense_entries_kernel<<<grid, 256, 0, st>>>(static_cast<double2*>(out), n, kind, s.ic, s.oc, s.p, s.w, q.cn, m);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

}  // extern "C"
