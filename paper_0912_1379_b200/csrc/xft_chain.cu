// Composed transforms in one launch and the b = 0 branch.
//
// xft_lct_chain: L_k ... L_1 f for up to four parameter quadruples, each stage
// reading the previous stage's output as samples on the standard grid (the
// reference CLI's inverse round trip, xft/cli.py:236-253, and the semigroup
// checks of pkg/tests/test_lct.py:176-200).  The rows stay in registers and the
// exchange buffer between stages: one HBM read and one HBM write for the whole
// chain instead of one per stage.
//
// xft_lct_b_zero: values_j = sqrt(d) exp(i c d y_j^2 / 2) f(d y_j), y = x
// (xft/lct.py:236-263), for caller-supplied samples f(d y_j), batched.
#include <cmath>

#include "../../include/xft_b200.h"
#include "xft_internal.h"
#include "xft_pipe.cuh"
#include "xft_tables.h"

using namespace xftb;

namespace {

struct ChainParams {
  Abcd st[4];
  int nst;
  int reverse;
  double scale;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS)
xft_chain_kernel(const typename Cfg::C* __restrict__ in, typename Cfg::C* __restrict__ out, long long batch,
                 ChainParams cp, const typename Cfg::C* __restrict__ tw, const typename Cfg::C* __restrict__ ptab,
                 const void* __restrict__ gtab, double2 cn, RowConst kc) {
  using C = typename Cfg::C;
  using Coef = typename Cfg::Coef;
  constexpr int N = Cfg::N, ROWS = Cfg::ROWS, E = Cfg::E, TR = Cfg::TR;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ Coef cs[4];
  C* xbuf = reinterpret_cast<C*>(xft_smem);
  void* tab = xft_smem + size_t(Cfg::STAGE) * sizeof(C);
  const int tid = threadIdx.x, lrow = tid / TR, j = tid - lrow * TR;
  const ThreadConst<Cfg> tc(j);
  if constexpr (Cfg::C128) {
    double2* t = static_cast<double2*>(tab);
    const double2* g = static_cast<const double2*>(gtab);
    for (int m = tid; m < XFT_C128_TABCOPIES * C128_TABN; m += Cfg::THREADS)
      t[m] = g[XFT_C128_TABCOPIES == 8 ? m >> 3 : m];
    __syncthreads();  // make_coef reads the table
  }
  if (tid < cp.nst) make_coef(cs[tid], nullptr, cp.st[tid], kc, TR, static_cast<const double2*>(tab));
  __syncthreads();
  auto noop = []() {};
  const long long ntiles = (batch + ROWS - 1) / ROWS;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row = tile * ROWS + lrow;
    const bool active = row < batch;
    C v[E];
#pragma unroll
    for (int s = 0; s < E; ++s) v[s] = active ? in[row * N + j + s * TR] : czero<C>();
    for (int k = 0; k < cp.nst; ++k) {
      const Coef rc = cs[k];
      pre_apply<Cfg>(v, [&](int s) { return v[s]; }, j, rc, tc, kc, ptab, tab);
      pipe_passes<Cfg, 0>(v, xbuf + lrow * Cfg::NP, j, tw, noop);
      post_apply<Cfg>(v, j, rc, tc, kc, cn, ptab, tab, [&](int s, C o) { v[s] = o; });
    }
    if (active) {
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int c = j + s * TR;
        out[row * N + (cp.reverse ? N - 1 - c : c)] = cscale(v[s], (decltype(v[s].x))cp.scale);
      }
    }
  }
}

template <class C, int L>
int launch_chain(const void* in, void* out, long long batch, const ChainParams& cp, cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int E = pipe_radix(dtype, L);
  constexpr int TR = (1 << L) / E;
  constexpr int ROWS = TR >= 256 ? 1 : (256 / TR > 64 ? 64 : 256 / TR);
  using Cfg = PipeCfg<C, L, E, MODE_LCT, -1, ROWS, 1, 1>;
  auto kern = xft_chain_kernel<Cfg>;
  Tables tb;
  int rc = get_tables(int64_t(1) << L, dtype, &tb);
  if (rc) return rc;
  if (Cfg::SMEM > 48 * 1024 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM) != cudaSuccess)
    return XFT_ECUDA;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::THREADS, Cfg::SMEM);
  const long long tiles = (batch + ROWS - 1) / ROWS;
  const long long cap = (long long)sms * (occ < 1 ? 1 : occ);
  RowConst kc;
  kc.half = tb.half;
  kc.cnabs = M_PI / std::sqrt(2.0 * double(1 << L));
  kc.cnred = (long long)(((__int128)((1 << L) - 1) * ((1 << L) - 1)) % (4 * (__int128)(1 << L)));
  kc.log2n = L;
  kc.flags = 0;
  kern<<<(unsigned)(tiles < cap ? tiles : cap), Cfg::THREADS, Cfg::SMEM, st>>>(
      static_cast<const C*>(in), static_cast<C*>(out), batch, cp, static_cast<const C*>(tb.tw),
      static_cast<const C*>(tb.ptab), tb.gtab, tb.cn, kc);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

template <class C, int... Ls>
int chain_dispatch(int l, const void* in, void* out, long long batch, const ChainParams& cp, cudaStream_t st,
                   std::integer_sequence<int, Ls...>) {
  int rc = XFT_ENOTSUP;
  ((l == Ls + 5 ? (rc = launch_chain<C, Ls + 5>(in, out, batch, cp, st), 0) : 0), ...);
  return rc;
}

// b = 0 branch, elementwise: sqrt(d) e^{i fl(fl(0.5 c d) fl(y^2))} samples   (xft/lct.py:260)
template <class C>
__global__ void xft_bzero_kernel(const C* __restrict__ in, C* __restrict__ out, long long batch, long long n,
                                 const double* __restrict__ abcd, long long stride, double half) {
  const long long total = batch * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / n, k = i - r * n;
    const double* p = abcd + r * stride;
    const double c = p[2], d = p[3];
    const double y = __dmul_rn((double)(2 * k - n + 1), half);    // xft/hermite.py:87-89
    const double ph = __dmul_rn(__dmul_rn(0.5 * c, d), __dmul_rn(y, y));
    double s, co;
    sincos(ph, &s, &co);
    const double sd = sqrt(d);
    const double2 f = make_double2((double)in[i].x, (double)in[i].y);
    const double ex = __dmul_rn(sd, co), ey = __dmul_rn(sd, s);   // numpy complex multiply, no contraction
    out[i] = to_c<C>(make_double2(__dsub_rn(__dmul_rn(ex, f.x), __dmul_rn(ey, f.y)),
                                  __dadd_rn(__dmul_rn(ex, f.y), __dmul_rn(ey, f.x))));
  }
}

}  // namespace

extern "C" {

int xft_lct_chain(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd_host, int nst,
                  double scale, int reverse, void* stream) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  if (nst < 1 || nst > 4) return XFT_EPARAM;
  int rc = xft_validate_lct_params(abcd_host, nst, 4, 1, 1e-10, nullptr);
  if (rc) return rc;
  if (batch == 0) return XFT_OK;
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  if ((int64_t(1) << l) != n || l < 5 || l > (dtype == XFT_C64 ? 14 : 13)) return XFT_ENOTSUP;
  ChainParams cp{};
  for (int k = 0; k < nst; ++k)
    cp.st[k] = Abcd{abcd_host[4 * k], abcd_host[4 * k + 1], abcd_host[4 * k + 2], abcd_host[4 * k + 3]};
  cp.nst = nst;
  cp.reverse = reverse ? 1 : 0;
  cp.scale = scale;
  auto st = static_cast<cudaStream_t>(stream);
  return dtype == XFT_C64 ? chain_dispatch<float2>(l, in, out, batch, cp, st, std::make_integer_sequence<int, 10>{})
                          : chain_dispatch<double2>(l, in, out, batch, cp, st, std::make_integer_sequence<int, 9>{});
}

int xft_validate_b_zero(const double* abcd, int64_t count, int64_t stride, double tol, int64_t* bad_row) {
  const int64_t rows = stride == 0 ? (count > 0 ? 1 : 0) : count;
  for (int64_t r = 0; r < rows; ++r) {
    const double* p = abcd + r * stride;
    int st = XFT_OK;
    if (p[1] != 0.0) st = XFT_EPARAM;                                // xft/lct.py:244-245
    else if (std::fabs(p[0] * p[3] - 1.0) > tol) st = XFT_EPARAM;    // 246-249
    else if (p[3] <= 0.0) st = XFT_EBRANCH;                          // 250-253
    if (st) {
      if (bad_row) *bad_row = r;
      return st;
    }
  }
  return XFT_OK;
}

int xft_lct_b_zero(const void* samples, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                   int64_t abcd_stride, void* stream) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  if (batch == 0) return XFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const long long total = batch * n;
  const unsigned grid = (unsigned)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  const double half = host_half_step(n);
  if (dtype == XFT_C64)
    xft_bzero_kernel<float2><<<grid, 256, 0, st>>>(static_cast<const float2*>(samples), static_cast<float2*>(out),
                                                    batch, n, abcd, abcd_stride, half);
  else
    xft_bzero_kernel<double2><<<grid, 256, 0, st>>>(static_cast<const double2*>(samples), static_cast<double2*>(out),
                                                     batch, n, abcd, abcd_stride, half);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

}  // extern "C"
