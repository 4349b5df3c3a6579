// Four-step path for rows longer than one CTA (M = M1 * M2 > in-CTA limit).
//
//   X[k1 + M1 k2] = sum_m2 w_M^{k1 m2} w_M2^{k2 m2} [ sum_m1 x[m1 M2 + m2] w_M1^{k1 m1} ]
//
// pass 1 ("columns"): length-M1 DFTs down the columns of the [M1][M2] view,
//          fused with the input generator / pre-multiplier and the w_M^{k1 m2}
//          twiddle, result in place ([k1][m2]);
// pass 2 ("rows"):    length-M2 DFTs along the rows.  Its store either goes to
//          natural order (transposed, coalesced in W-wide chunks) fused with the
//          post-multiplier, or stays permuted ([k1][k2]) for a convolution.
// Convolutions (chirp-z, Mehler) keep the spectrum permuted: the row pass
// multiplies by the permuted kernel spectrum between a forward and an inverse
// FFT, applies the conjugate twiddle, and an inverse column pass returns to
// natural order fused with the post-multiplier.  Scratch lives in device
// memory (L2-resident for the configurations of BASELINE.json).
#include <cuda.h>  // CUtensorMap (the encoder is fetched with cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>

#include <cmath>
#include <complex>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/xft_b200.h"
#include "xft_blue.cuh"
#include "xft_internal.h"
#include "xft_tables.h"
#include "xft_tile.cuh"

using namespace xftb;

namespace {

const long double PI_L = 3.141592653589793238462643383279502884L;

template <class C> constexpr int tile_w() { return sizeof(C) == 8 ? 16 : 8; }    // 128-byte lines
#ifndef XFT_TILE_E7
#define XFT_TILE_E7 8
#endif
template <class C> constexpr int tile_e(int l) {
  return l >= 8 ? (sizeof(C) == 8 ? 16 : 8) : (l == 7 && sizeof(C) == 8 ? XFT_TILE_E7 : 8);
}

// natural twiddles e^{-2 pi i m / M}, m < M, per (device, M, dtype)
std::mutex g_mu;
std::map<std::tuple<int, int64_t, int>, void*> g_nat;

int natural_twiddles(int64_t M, int dtype, const void** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, M, dtype);
  auto it = g_nat.find(key);
  if (it == g_nat.end()) {
    const size_t esz = dtype == XFT_C64 ? 8 : 16;
    std::vector<double2> d(M);
    std::vector<float2> f(M);
    for (int64_t m = 0; m < M; ++m) {
      const long double th = 2.0L * PI_L * (long double)m / (long double)M;
      d[m] = make_double2((double)cosl(th), (double)-sinl(th));
      f[m] = make_float2((float)cosl(th), (float)-sinl(th));
    }
    void* p = nullptr;
    if (cudaMalloc(&p, esz * M) != cudaSuccess) return XFT_ECUDA;
    if (cudaMemcpy(p, dtype == XFT_C64 ? (const void*)f.data() : (const void*)d.data(), esz * M,
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return XFT_ECUDA;
    it = g_nat.emplace(key, p).first;
  }
  *out = it->second;
  return XFT_OK;
}

struct Shape {
  int l1, l2;  // M1 = 2^l1 (columns pass), M2 = 2^l2 (rows pass)
  long long M;
};
Shape split(int l) {
  Shape s;
  s.l1 = (l + 1) / 2;
  s.l2 = l / 2;
  s.M = 1ll << l;
  return s;
}

// ---------------------------------------------------------------------------
// generators / pre-multipliers of pass 1 (natural index m of row b)
// ---------------------------------------------------------------------------
template <class C>
struct GenLoad {  // plain input row
  const C* in;
  const int* rowlist;
  long long M;
  __device__ C operator()(long long b, long long m) const {
    const long long row = rowlist ? rowlist[b] : b;
    return in[row * M + m];
  }
};

struct RowChirp {  // exact LCT chirp coefficients + row factor (per row)
  double cin, cout, s4;
  double2 g;
  int pre, post;
  int pad[2];
};

template <class C>
struct GenLct {  // x p_k e^{i phi_k}  (pow2 n = M), or just p_k (scaled Fourier)
  const C* in;
  const RowChirp* rc;
  const double2* ptab;  // p_k, natural
  double half;
  long long n;
  int lct;
  __device__ C operator()(long long b, long long k) const {
    double2 u = cmul_d(ptab[k], to_d2(in[b * n + k]));
    if (lct && rc[b].pre) {
      const double x = __dmul_rn((double)(2 * k - n + 1), half);
      const double phi = __dmul_rn(rc[b].cin, __dmul_rn(x, x));
      double s, c;
      sincos(phi, &s, &c);
      u = cmul_d(make_double2(c, s), u);
    }
    return to_c<C>(u);
  }
};

template <class C>
struct GenChirpZ {  // chirp-z: pre[k] x [e^{i phi_k}] for k < n, zero padding beyond
  const C* in;
  const RowChirp* rc;
  const double2* pre;
  double half;
  long long n;
  int lct;
  __device__ C operator()(long long b, long long k) const {
    if (k >= n) return to_c<C>(make_double2(0.0, 0.0));
    double2 u = cmul_d(pre[k], to_d2(in[b * n + k]));
    if (lct && rc[b].pre) {
      const double x = __dmul_rn((double)(2 * k - n + 1), half);
      const double phi = __dmul_rn(rc[b].cin, __dmul_rn(x, x));
      double s, c;
      sincos(phi, &s, &c);
      u = cmul_d(make_double2(c, s), u);
    }
    return to_c<C>(u);
  }
};

struct GenMehlerH {  // kernel h(lag) = exp(-beta lag^2), circular lags
  const OpMehlerRow* rows;
  const int* rowlist;
  long long M;
  __device__ double2 operator()(long long b, long long m) const {
    const OpMehlerRow p = rows[rowlist[b]];
    const long long lag = m < p.wn ? m : (m > M - p.wn ? m - M : -(1ll << 62));
    if (lag == -(1ll << 62)) return make_double2(0.0, 0.0);
    const double l2 = (double)lag * (double)lag;
    return cexp_d(-p.beta.x * l2, -p.beta.y * l2);
  }
};

struct GenMehlerU {  // windowed input times exp(-gam x^2)
  const double2* in;
  const OpMehlerRow* rows;
  const int* rowlist;
  double half;
  long long n;
  __device__ double2 operator()(long long b, long long m) const {
    const long long row = rowlist[b];
    const OpMehlerRow p = rows[row];
    if (m >= p.wn) return make_double2(0.0, 0.0);
    const long long k = p.k0 + m;
    const long long ks = p.sigma > 0 ? k : n - 1 - k;
    const double x = (double)(2 * k - n + 1) * half;
    const double x2 = x * x;
    return cmul_d(cexp_d(-p.gam.x * x2, -p.gam.y * x2), in[row * n + ks]);
  }
};

// ---------------------------------------------------------------------------
// pass operators
// ---------------------------------------------------------------------------
template <class C, class Gen>
struct OpCols {  // pass 1: columns (generator in, twiddled permuted-column out)
  static constexpr bool MID = false;
  Gen gen;
  C* out;
  const C* twm;  // natural twiddles of length M
  int M2, W;
  long long M;
  int conj_tw;   // +1 transforms use the conjugate twiddle
  __device__ C load(long long tile, int w, int a) const {
    const int cb = M2 / W;
    const long long b = tile / cb;
    const int c = (int)(tile % cb) * W + w;
    return gen(b, (long long)a * M2 + c);
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const int cb = M2 / W;
    const long long b = tile / cb;
    const int c = (int)(tile % cb) * W + w;
    const C w8 = twm[(long long)a * c];
    out[b * M + (long long)a * M2 + c] = cmul(v, conj_tw ? cconj(w8) : w8);
  }
};

template <class C, class Post>
struct OpRowsNat {  // pass 2 of a plain FFT: rows, transposed store to natural order
  static constexpr bool MID = false;
  const C* scr;
  Post post;
  int M1, M2, W;
  long long M;
  __device__ C load(long long tile, int w, int a) const {
    const int rb = M1 / W;
    const long long b = tile / rb;
    const int k1 = (int)(tile % rb) * W + w;
    return scr[b * M + (long long)k1 * M2 + a];
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const int rb = M1 / W;
    const long long b = tile / rb;
    const int k1 = (int)(tile % rb) * W + w;
    post(b, k1 + (long long)M1 * a, v);
  }
};

template <class C>
struct OpRowsPerm {  // pass 2 kept permuted (kernel spectra)
  static constexpr bool MID = false;
  C* scr;
  int M1, M2, W;
  long long M;
  __device__ C load(long long tile, int w, int a) const {
    const long long b = tile / (M1 / W);
    const int k1 = (int)(tile % (M1 / W)) * W + w;
    return scr[b * M + (long long)k1 * M2 + a];
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const long long b = tile / (M1 / W);
    const int k1 = (int)(tile % (M1 / W)) * W + w;
    scr[b * M + (long long)k1 * M2 + a] = v;
  }
};

template <class C>
struct OpRowsConv {  // rows: forward, x spectrum, inverse, conjugate twiddle
  static constexpr bool MID = true;
  C* scr;
  const C* spec;  // permuted spectrum, row stride spec_stride (0: shared by all rows)
  long long spec_stride;
  const C* twm;
  int M1, M2, W;
  long long M;
  __device__ long long base(long long tile, int w, int& k1) const {
    const long long b = tile / (M1 / W);
    k1 = (int)(tile % (M1 / W)) * W + w;
    return b;
  }
  __device__ C load(long long tile, int w, int a) const {
    int k1;
    const long long b = base(tile, w, k1);
    return scr[b * M + (long long)k1 * M2 + a];
  }
  __device__ C mid(long long tile, int w, int a, C v) const {
    int k1;
    const long long b = base(tile, w, k1);
    return cmul(v, spec[b * spec_stride + (long long)k1 * M2 + a]);
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    int k1;
    const long long b = base(tile, w, k1);
    scr[b * M + (long long)k1 * M2 + a] = cmul(v, cconj(twm[(long long)k1 * a]));
  }
};

template <class C, class Post>
struct OpColsInv {  // inverse columns: permuted [k1][m2] -> natural m = m1 M2 + m2, fused post
  static constexpr bool MID = false;
  const C* scr;
  Post post;
  int M2, W;
  long long M;
  __device__ C load(long long tile, int w, int a) const {
    const long long b = tile / (M2 / W);
    const int c = (int)(tile % (M2 / W)) * W + w;
    return scr[b * M + (long long)a * M2 + c];
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const long long b = tile / (M2 / W);
    const int c = (int)(tile % (M2 / W)) * W + w;
    post(b, (long long)a * M2 + c, v);
  }
};

// post-multipliers (natural output index j of row b)
template <class C>
struct PostLct {
  C* out;
  const RowChirp* rc;
  const double2* post;  // C(n) p_j (LCT/scaled) or 1 (DFT): natural
  double half;
  long long n;
  int lct, plain;
  __device__ void operator()(long long b, long long j, C v) const {
    if (plain) {
      out[b * n + j] = v;
      return;
    }
    double2 o = cmul_d(post[j], to_d2(v));
    if (lct) {
      o = cmul_d(rc[b].g, o);
      if (rc[b].post) {
        const double x = __dmul_rn((double)(2 * j - n + 1), half);
        const double y = __dmul_rn(rc[b].s4, x);
        const double psi = __dmul_rn(rc[b].cout, __dmul_rn(y, y));
        double s, c;
        sincos(psi, &s, &c);
        o = cmul_d(make_double2(c, s), o);
      }
    }
    out[b * n + j] = to_c<C>(o);
  }
};

template <class C>
struct PostChirpZ {
  C* out;
  const RowChirp* rc;
  const double2* post;  // chirp_j / M [* C(n) p_j]
  double half;
  long long n;
  int lct;
  __device__ void operator()(long long b, long long j, C v) const {
    if (j >= n) return;
    double2 o = cmul_d(post[j], to_d2(v));
    if (lct) {
      o = cmul_d(rc[b].g, o);
      if (rc[b].post) {
        const double x = __dmul_rn((double)(2 * j - n + 1), half);
        const double y = __dmul_rn(rc[b].s4, x);
        const double psi = __dmul_rn(rc[b].cout, __dmul_rn(y, y));
        double s, c;
        sincos(psi, &s, &c);
        o = cmul_d(make_double2(c, s), o);
      }
    }
    out[b * n + j] = to_c<C>(o);
  }
};

struct PostMehler {
  double2* out;
  const OpMehlerRow* rows;
  const int* rowlist;
  double half;
  long long n;
  __device__ void operator()(long long b, long long m, double2 v) const {
    const long long row = rowlist[b];
    const OpMehlerRow p = rows[row];
    if (m >= p.wn) return;
    const long long k = p.k0 + m;
    const double x = (double)(2 * k - n + 1) * half;
    const double x2 = x * x;
    out[row * n + k] = cmul_d(cmul_d(p.scale, cexp_d(-p.gam.x * x2, -p.gam.y * x2)), v);
  }
};

// Mehler four-step passes with walked Gaussian chirps: in the columns pass a
// thread's samples a = j + s TR of column c sit at m = a M2 + c, so the kernel
// lags (two monotone pieces) and the grid offsets m' = 2(k0 + m) - n + 1 are
// linear in s and the values come from GaussWalk (xft_blue.cuh) instead of an
// exp + table phasor per element.
constexpr DD kInv2Pi{0.15915494309189535, -9.839338337591243e-18};

struct OpColsMehlerH : OpCols<double2, GenMehlerH> {  // kernel spectrum, pass 1
  static constexpr bool LOAD_LINE = true;
  template <int E, int TR>
  __device__ void load_line(long long tile, int w, int j, double2 (&v)[E]) const {
    const int cb = M2 / W;
    const long long b = tile / cb;
    const int c = (int)(tile % cb) * W + w;
    const OpMehlerRow p = gen.rows[gen.rowlist[b]];
    const DD db = dd_mul(DD{-p.beta.y, 0.0}, kInv2Pi);
    const double dl = (double)TR * M2;
    const double2 S = gauss_val(p.beta.x, db, 2.0 * dl * dl);
    GaussWalk wa;  // lags l = (j + s TR) M2 + c, s < E/2
    const double la = (double)j * M2 + c;
    wa.init(p.beta.x, db, la * la, dl * (2.0 * la + dl));
#pragma unroll
    for (int s = 0; s < E / 2; ++s) {
      v[s] = la + s * dl < p.wn ? wa.W : make_double2(0.0, 0.0);
      if (s < E / 2 - 1) wa.step(S);
    }
    GaussWalk wb;  // |l| = ((E - s) TR - j) M2 - c, s >= E/2 (ascending as s falls)
    const double lb = (double)(TR - j) * M2 - c;
    wb.init(p.beta.x, db, lb * lb, dl * (2.0 * lb + dl));
#pragma unroll
    for (int s = E - 1; s >= E / 2; --s) {
      v[s] = lb + (E - 1 - s) * dl < p.wn ? wb.W : make_double2(0.0, 0.0);
      if (s > E / 2) wb.step(S);
    }
  }
};

struct OpColsMehlerU : OpCols<double2, GenMehlerU> {  // windowed, weighted input, pass 1
  static constexpr bool LOAD_LINE = true;
  template <int E, int TR>
  __device__ void load_line(long long tile, int w, int j, double2 (&v)[E]) const {
    const int cb = M2 / W;
    const long long b = tile / cb;
    const int c = (int)(tile % cb) * W + w;
    const long long row = gen.rowlist[b];
    const OpMehlerRow p = gen.rows[row];
    const long long n = gen.n;
    const DD hh = dd_prod(gen.half, gen.half);
    const double ag = p.gam.x * hh.hi;
    const DD dg = dd_mul(dd_mul(hh, -p.gam.y), kInv2Pi);
    const double dm = 2.0 * TR * M2;                              // m' step
    const double mp0 = 2.0 * ((double)p.k0 + c + (double)j * M2) - (double)n + 1.0;
    GaussWalk wg;
    wg.init(ag, dg, mp0 * mp0, dm * (2.0 * mp0 + dm));
    const double2 S = gauss_val(ag, dg, 2.0 * dm * dm);
    const double2* src = gen.in + row * n;
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const long long m = (long long)(j + s * TR) * M2 + c;
      double2 u = make_double2(0.0, 0.0);
      if (m < p.wn) {
        const long long k = p.k0 + m;
        u = cmul_d(wg.W, src[p.sigma > 0 ? k : n - 1 - k]);
      }
      v[s] = u;
      if (s < E - 1) wg.step(S);
    }
  }
};

struct OpColsInvMehler : OpColsInv<double2, PostMehler> {  // inverse columns + output weights
  static constexpr bool STORE_LINE = true;
  template <int E, int TR>
  __device__ void store_line(long long tile, int w, int j, const double2 (&v)[E]) const {
    const long long b = tile / (M2 / W);
    const int c = (int)(tile % (M2 / W)) * W + w;
    const long long row = post.rowlist[b];
    const OpMehlerRow p = post.rows[row];
    const long long n = post.n;
    const DD hh = dd_prod(post.half, post.half);
    const double ag = p.gam.x * hh.hi;
    const DD dg = dd_mul(dd_mul(hh, -p.gam.y), kInv2Pi);
    const double dm = 2.0 * TR * M2;
    const double mp0 = 2.0 * ((double)p.k0 + c + (double)j * M2) - (double)n + 1.0;
    GaussWalk wg;
    wg.init(ag, dg, mp0 * mp0, dm * (2.0 * mp0 + dm));
    wg.W = cmul_d(p.scale, wg.W);
    const double2 S = gauss_val(ag, dg, 2.0 * dm * dm);
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const long long m = (long long)(j + s * TR) * M2 + c;
      if (m < p.wn) post.out[row * n + p.k0 + m] = cmul_d(wg.W, v[s]);
      if (s < E - 1) wg.step(S);
    }
  }
};

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
template <class C, int LOGL, bool LC, bool SC, int SIGN, int W, class Op>
int launch_tile(long long ntiles, const Op& op, cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int E = tile_e<C>(LOGL);
  constexpr int T = W * ((1 << LOGL) / E);
  constexpr size_t SM = tile_smem<C, LOGL, W>();
  if constexpr (T > 1024 || SM > 200 * 1024) {
    return XFT_ENOTSUP;  // tile too wide for this line length (callers fall back to narrower tiles)
  } else {
    auto kern = xft_tile_kernel<C, LOGL, E, W, LC, SC, SIGN, Op>;
    Tables tb;
    int rc = get_tables(int64_t(1) << LOGL, dtype, &tb, E);
    if (rc) return rc;
    if (SM > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM) != cudaSuccess)
      return XFT_ECUDA;
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T, SM);
    const long long cap = (long long)sms * (occ < 1 ? 1 : occ);
    kern<<<(unsigned)(ntiles < cap ? ntiles : cap), T, SM, st>>>(ntiles, op, static_cast<const C*>(tb.tw));
    return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
  }
}

constexpr int LMIN = 6, LMAX = 10;  // per-pass lengths 64 .. 1024  =>  M up to 2^20

template <class C, bool LC, bool SC, int SIGN, int W, class Op, int... Ls>
int tile_dispatch(int l, long long ntiles, const Op& op, cudaStream_t st, std::integer_sequence<int, Ls...>) {
  int rc = XFT_ENOTSUP;
  ((l == Ls + LMIN ? (rc = launch_tile<C, Ls + LMIN, LC, SC, SIGN, W, Op>(ntiles, op, st), 0) : 0), ...);
  return rc;
}

template <class C, bool LC, bool SC, int SIGN, class Op, int W = tile_w<C>()>
int tile(int l, long long ntiles, const Op& op, cudaStream_t st) {
  if (l < LMIN || l > LMAX) return XFT_ENOTSUP;
  return tile_dispatch<C, LC, SC, SIGN, W, Op>(l, ntiles, op, st, std::make_integer_sequence<int, LMAX - LMIN + 1>{});
}

// samples outside a Mehler row's window: exact zeros
__global__ void mehler_zero_kernel(double2* out, const int* rowlist, const OpMehlerRow* prm, long long n) {
  const long long row = rowlist[blockIdx.x];
  const int k0 = prm[row].k0;
  for (int k = threadIdx.x; k < k0; k += blockDim.x) {
    out[row * n + k] = make_double2(0.0, 0.0);
    out[row * n + n - 1 - k] = make_double2(0.0, 0.0);
  }
}

__global__ void row_chirp_kernel(RowChirp* out, long long rows, const double* abcd, long long stride, Abcd uni,
                                 int bare) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  OpChirpZ op{};
  op.abcd = abcd;
  op.abcd_stride = stride;
  op.uni = uni;
  op.lct = 1;
  op.bare = bare;
  const ChirpZRow c = chirpz_row(op, r);
  RowChirp o;
  o.cin = c.cin;
  o.cout = c.cout;
  o.s4 = c.s4;
  o.g = c.g;
  o.pre = c.pre;
  o.post = c.post;
  out[r] = o;
}

template <class T>
struct DevBuf {  // stream-ordered scratch
  T* p = nullptr;
  cudaStream_t st;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  int alloc(size_t count) { return cudaMallocAsync((void**)&p, count * sizeof(T), st) == cudaSuccess ? XFT_OK : XFT_ECUDA; }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

int log2_of(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

// boundary phase p_k and C(n) p_k (natural, fp64) for the large pow2 path
std::mutex g_pmu;
std::map<std::pair<int, int64_t>, std::pair<double2*, double2*>> g_ptab;
int boundary_tables(int64_t n, const double2** p, const double2** cp) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pmu);
  auto it = g_ptab.find({dev, n});
  if (it == g_ptab.end()) {
    std::vector<double2> a(n), b(n);
    const int64_t red = (int64_t)(((__int128)(n - 1) * (n - 1)) % (4 * (__int128)n));
    const std::complex<long double> cn =
        (PI_L / sqrtl(2.0L * n)) *
        std::complex<long double>(cosl(PI_L * red / (2.0L * n)), -sinl(PI_L * red / (2.0L * n)));
    for (int64_t k = 0; k < n; ++k) {
      const int64_t rk = (int64_t)(((__int128)(n - 1) * k) % (2 * (__int128)n));
      const std::complex<long double> pk(cosl(PI_L * rk / (long double)n), sinl(PI_L * rk / (long double)n));
      const std::complex<long double> q = pk * cn;
      a[k] = make_double2((double)pk.real(), (double)pk.imag());
      b[k] = make_double2((double)q.real(), (double)q.imag());
    }
    double2 *da = nullptr, *db = nullptr;
    if (cudaMalloc(&da, n * 16) != cudaSuccess || cudaMalloc(&db, n * 16) != cudaSuccess) return XFT_ECUDA;
    if (cudaMemcpy(da, a.data(), n * 16, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(db, b.data(), n * 16, cudaMemcpyHostToDevice) != cudaSuccess)
      return XFT_ECUDA;
    it = g_ptab.emplace(std::make_pair(dev, n), std::make_pair(da, db)).first;
  }
  *p = it->second.first;
  *cp = it->second.second;
  return XFT_OK;
}

template <class C>
int large_pow2(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, const double* abcd,
               int64_t stride, Abcd uni, int flags, cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int W = tile_w<C>();
  const int l = log2_of(n);
  const Shape sh = split(l);
  const int M1 = 1 << sh.l1, M2 = 1 << sh.l2;
  const void* twm = nullptr;
  int rc = natural_twiddles(sh.M, dtype, &twm);
  if (rc) return rc;
  DevBuf<C> scr(st);
  DevBuf<RowChirp> rcs(st);
  if ((rc = scr.alloc((size_t)batch * sh.M))) return rc;
  const double2 *ptab = nullptr, *cptab = nullptr;
  if (mode != MODE_DFT && (rc = boundary_tables(n, &ptab, &cptab))) return rc;
  if (mode == MODE_LCT) {
    if ((rc = rcs.alloc(batch))) return rc;
    row_chirp_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(rcs.p, batch, abcd, stride, uni,
                                                                      (flags & XFT_FLAG_BARE_FOURIER) ? 1 : 0);
  }
  const long long t1 = batch * (M2 / W), t2 = batch * (M1 / W);
  PostLct<C> post{static_cast<C*>(out), rcs.p, cptab, host_half_step(n), n, mode == MODE_LCT, mode == MODE_DFT};
  if (mode == MODE_DFT) {
    OpCols<C, GenLoad<C>> op1{GenLoad<C>{static_cast<const C*>(in), nullptr, sh.M}, scr.p,
                              static_cast<const C*>(twm), M2, W, sh.M, sign > 0};
    OpRowsNat<C, PostLct<C>> op2{scr.p, post, M1, M2, W, sh.M};
    if (sign < 0) {
      if ((rc = tile<C, true, true, -1>(sh.l1, t1, op1, st))) return rc;
      return tile<C, false, true, -1>(sh.l2, t2, op2, st);
    }
    if ((rc = tile<C, true, true, +1>(sh.l1, t1, op1, st))) return rc;
    return tile<C, false, true, +1>(sh.l2, t2, op2, st);
  }
  OpCols<C, GenLct<C>> op1{GenLct<C>{static_cast<const C*>(in), rcs.p, ptab, host_half_step(n), n, mode == MODE_LCT},
                           scr.p, static_cast<const C*>(twm), M2, W, sh.M, 0};
  OpRowsNat<C, PostLct<C>> op2{scr.p, post, M1, M2, W, sh.M};
  if ((rc = tile<C, true, true, -1>(sh.l1, t1, op1, st))) return rc;
  return tile<C, false, true, -1>(sh.l2, t2, op2, st);
}

}  // namespace

namespace xftb {

// rows longer than the in-CTA kernels: four-step path (power-of-two n)
int run_large_pow2(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, int dtype,
                   const double* abcd, int64_t stride, const double* uni4, int flags, cudaStream_t st) {
  const int l = log2_of(n);
  if ((int64_t(1) << l) != n || l > 2 * LMAX || (l + 1) / 2 < LMIN) return XFT_ENOTSUP;
  const Abcd uni = uni4 ? Abcd{uni4[0], uni4[1], uni4[2], uni4[3]} : Abcd{0, 0, 0, 0};
  return dtype == XFT_C64 ? large_pow2<float2>(mode, sign, in, out, batch, n, abcd, stride, uni, flags, st)
                          : large_pow2<double2>(mode, sign, in, out, batch, n, abcd, stride, uni, flags, st);
}

// chirp-z rows whose convolution length m exceeds the in-CTA kernels:
// u = pre x f [x e^{i phi}] zero-padded to m -> columns pass -> rows pass
// (forward, x filter spectrum, inverse) -> inverse columns with the post
// multiplier (xft/fftcore.py:84-100, 116-119; the LCT wrappers of
// xft/lct.py:204-207).  The filter spectrum is permuted once into the
// four-step order [k1][k2] = H[k1 + M1 k2] and cached per (plan, dtype).
template <class C>
__global__ void permute_spectrum_kernel(C* out, const double2* hnat, int M1, int M2) {
  const long long M = (long long)M1 * M2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
    const long long k1 = i / M2, k2 = i - k1 * M2;
    out[i] = to_c<C>(hnat[k1 + (long long)M1 * k2]);
  }
}

std::mutex g_czmu;
std::map<std::tuple<int, const void*, int>, void*> g_czperm;  // (device, plan spectrum, dtype)

template <class C>
int large_chirpz(int lct, int bare, const C* in, C* out, int64_t batch, int64_t n, const double* abcd, int64_t stride,
                 Abcd uni, const double2* pre, const double2* post, const double2* hspec, int64_t m, cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int W = tile_w<C>();
  const int l = log2_of(m);
  const Shape sh = split(l);
  if (sh.l1 < LMIN || sh.l1 > LMAX || sh.l2 < LMIN || sh.l2 > LMAX) return XFT_ENOTSUP;
  const int M1 = 1 << sh.l1, M2 = 1 << sh.l2;
  const void* twm = nullptr;
  int rc = natural_twiddles(sh.M, dtype, &twm);
  if (rc) return rc;
  C* spec = nullptr;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_czmu);
    auto key = std::make_tuple(dev, (const void*)hspec, dtype);
    auto it = g_czperm.find(key);
    if (it == g_czperm.end()) {
      void* d = nullptr;
      if (cudaMalloc(&d, sh.M * sizeof(C)) != cudaSuccess) return XFT_ECUDA;
      permute_spectrum_kernel<C><<<592, 256>>>(static_cast<C*>(d), hspec, M1, M2);  // legacy stream: before any use
      if (cudaDeviceSynchronize() != cudaSuccess) return XFT_ECUDA;
      it = g_czperm.emplace(key, d).first;
    }
    spec = static_cast<C*>(it->second);
  }
  DevBuf<C> scr(st);
  DevBuf<RowChirp> rcs(st);
  if ((rc = scr.alloc((size_t)batch * sh.M))) return rc;
  if (lct) {
    if ((rc = rcs.alloc(batch))) return rc;
    row_chirp_kernel<<<(unsigned)((batch + 127) / 128), 128, 0, st>>>(rcs.p, batch, abcd, stride, uni, bare);
  }
  const long long t1 = batch * (M2 / W), t2 = batch * (M1 / W);
  const double half = host_half_step(n);
  OpCols<C, GenChirpZ<C>> c1{GenChirpZ<C>{in, rcs.p, pre, half, n, lct}, scr.p, static_cast<const C*>(twm), M2, W,
                             sh.M, 0};
  if ((rc = tile<C, true, true, -1>(sh.l1, t1, c1, st))) return rc;
  OpRowsConv<C> c2{scr.p, spec, 0, static_cast<const C*>(twm), M1, M2, W, sh.M};
  if ((rc = tile<C, false, false, -1>(sh.l2, t2, c2, st))) return rc;
  OpColsInv<C, PostChirpZ<C>> c3{scr.p, PostChirpZ<C>{out, rcs.p, post, half, n, lct}, M2, W, sh.M};
  return tile<C, true, true, +1>(sh.l1, t1, c3, st);
}

// Mehler rows whose window needs M > in-CTA limit (complex128)
// plan time: the permuted kernel spectra of a four-step Mehler class, [rows][M] into hs
int large_mehler_spectrum(long long rows, const int* rowlist, const OpMehlerRow* prm, int l, void* hs_out,
                          cudaStream_t st) {
  using C = double2;
  constexpr int W = tile_w<C>();
  const Shape sh = split(l);
  const int M1 = 1 << sh.l1, M2 = 1 << sh.l2;
  const void* twm = nullptr;
  int rc = natural_twiddles(sh.M, XFT_C128, &twm);
  if (rc) return rc;
  C* hs = static_cast<C*>(hs_out);
  const long long t1 = rows * (M2 / W), t2 = rows * (M1 / W);
  OpColsMehlerH h1{{GenMehlerH{prm, rowlist, sh.M}, hs, static_cast<const C*>(twm), M2, W, sh.M, 0}};
  if ((rc = tile<C, true, true, -1>(sh.l1, t1, h1, st))) return rc;
  OpRowsPerm<C> h2{hs, M1, M2, W, sh.M};
  return tile<C, false, false, -1>(sh.l2, t2, h2, st);
}

// data passes of a four-step Mehler class with the plan's spectra hspec ([rows][M], permuted)
int run_large_mehler(const void* in, void* out, long long rows, const int* rowlist, const OpMehlerRow* prm,
                     int l, int64_t n, cudaStream_t st, void* scratch, const void* hspec) {
  using C = double2;
  constexpr int W = tile_w<C>();
  const Shape sh = split(l);
  const int M1 = 1 << sh.l1, M2 = 1 << sh.l2;
  const void* twm = nullptr;
  int rc = natural_twiddles(sh.M, XFT_C128, &twm);
  if (rc) return rc;
  DevBuf<C> us(st);  // caller scratch (one row x M per row) when given, else stream-ordered
  if (scratch) {
    us.p = static_cast<C*>(scratch);
    us.st = nullptr;
  } else if ((rc = us.alloc((size_t)rows * sh.M))) {
    return rc;
  }
  struct Release {  // caller scratch is not freed
    DevBuf<C>& a; bool own;
    ~Release() { if (!own) a.p = nullptr; }
  } release{us, scratch == nullptr};
  const long long t1 = rows * (M2 / W), t2 = rows * (M1 / W);
  const double half = host_half_step(n);
  // data: columns, rows (forward x H inverse), inverse columns with the output weights
  OpColsMehlerU u1{{GenMehlerU{static_cast<const C*>(in), prm, rowlist, half, n}, us.p,
                    static_cast<const C*>(twm), M2, W, sh.M, 0}};
  if ((rc = tile<C, true, true, -1>(sh.l1, t1, u1, st))) return rc;
  OpRowsConv<C> u2{us.p, static_cast<const C*>(hspec), sh.M, static_cast<const C*>(twm), M1, M2, W, sh.M};
  if ((rc = tile<C, false, false, -1>(sh.l2, t2, u2, st))) return rc;
  OpColsInvMehler u3{{us.p, PostMehler{static_cast<C*>(out), prm, rowlist, half, n}, M2, W, sh.M}};
  if ((rc = tile<C, true, true, +1>(sh.l1, t1, u3, st))) return rc;
  mehler_zero_kernel<<<(unsigned)rows, 256, 0, st>>>(static_cast<C*>(out), rowlist, prm, n);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

int run_large_chirpz(int lct, int bare, const void* in, void* out, int64_t batch, int64_t n, int dtype,
                     const double* abcd, int64_t stride, const double* uni4, const void* pre, const void* post,
                     const void* hspec, int64_t m, cudaStream_t st) {
  const Abcd uni = uni4 ? Abcd{uni4[0], uni4[1], uni4[2], uni4[3]} : Abcd{0, 0, 0, 0};
  const auto* p = static_cast<const double2*>(pre);
  const auto* q = static_cast<const double2*>(post);
  const auto* h = static_cast<const double2*>(hspec);
  return dtype == XFT_C64
             ? large_chirpz<float2>(lct, bare, static_cast<const float2*>(in), static_cast<float2*>(out), batch, n,
                                    abcd, stride, uni, p, q, h, m, st)
             : large_chirpz<double2>(lct, bare, static_cast<const double2*>(in), static_cast<double2*>(out), batch,
                                     n, abcd, stride, uni, p, q, h, m, st);
}

}  // namespace xftb

// ---------------------------------------------------------------------------
// column LCT of a [R][ncols] slab (row stride ld), one parameter quadruple:
// the second axis of the separable 2-D transform.  Lines are columns, so every
// access moves W adjacent columns; R <= 1024 in one pass, larger R by the
// four-step split R = R1 R2 (pass 1 over r1 with the twiddle, pass 2 over r2
// storing straight to the natural row index j = k1 + R1 k2).
// ---------------------------------------------------------------------------
namespace {

struct ColChirp {               // host-computed, uniform over the slab
  // c64: exact fixed-point turns (see xft_pipe.cuh)
  unsigned long long dq_in, dq_out;
  unsigned gq;
  float gabs;
  // c128: exact fp64 phase arguments
  double cin, cout, s4, half;
  double2 g;
  int pre, post, log2r;
  long long R;
};

template <class C>
struct ColPhase;

template <>
struct ColPhase<float2> {
  static __device__ __forceinline__ float2 pre(const ColChirp& k, const double2*, long long r, float2 v) {
    const int off = (int)(2 * r - k.R + 1);
    const unsigned o2 = (unsigned)(off * off);
    const unsigned bt = ((unsigned)(r & 1) << 31) - ((unsigned)r << (31 - k.log2r));
    unsigned top = bt;
    if (k.pre) top += (unsigned)(k.dq_in >> 32) * o2 + __umulhi((unsigned)k.dq_in, o2);
    return cmul(unit_turns_sfu(top, 1.0f), v);
  }
  static __device__ __forceinline__ float2 post(const ColChirp& k, const double2*, long long j, float2 v) {
    const int off = (int)(2 * j - k.R + 1);
    const unsigned o2 = (unsigned)(off * off);
    const unsigned bt = ((unsigned)(j & 1) << 31) - ((unsigned)j << (31 - k.log2r));
    unsigned top = bt + k.gq;
    if (k.post) top += (unsigned)(k.dq_out >> 32) * o2 + __umulhi((unsigned)k.dq_out, o2);
    return cmul(unit_turns_sfu(top, k.gabs), v);
  }
};

template <>
struct ColPhase<double2> {
  static __device__ __forceinline__ double2 pre(const ColChirp& k, const double2* ptab, long long r, double2 v) {
    double2 u = cmul_d(ptab[r], v);
    if (k.pre) {
      const double x = __dmul_rn((double)(2 * r - k.R + 1), k.half);
      const double phi = __dmul_rn(k.cin, __dmul_rn(x, x));
      double s, c;
      sincos(phi, &s, &c);
      u = cmul_d(make_double2(c, s), u);
    }
    return u;
  }
  static __device__ __forceinline__ double2 post(const ColChirp& k, const double2* cptab, long long j, double2 v) {
    double2 o = cmul_d(cmul_d(k.g, cptab[j]), v);
    if (k.post) {
      const double x = __dmul_rn((double)(2 * j - k.R + 1), k.half);
      const double y = __dmul_rn(k.s4, x);
      const double psi = __dmul_rn(k.cout, __dmul_rn(y, y));
      double s, c;
      sincos(psi, &s, &c);
      o = cmul_d(make_double2(c, s), o);
    }
    return o;
  }
};

template <class C>
struct OpColLctOne {  // R <= 1024
  static constexpr bool MID = false;
  const C* in;
  C* out;
  long long ld;
  int W;
  ColChirp k;
  const double2 *ptab, *cptab;
  __device__ C load(long long tile, int w, int a) const {
    const long long c = tile * W + w;
    return ColPhase<C>::pre(k, ptab, a, in[(long long)a * ld + c]);
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const long long c = tile * W + w;
    out[(long long)a * ld + c] = ColPhase<C>::post(k, cptab, a, v);
  }
};

template <class C>
struct OpColLct1 {  // four-step pass 1: DFT over r1 for the line (r2, c); twiddle w_R^{k1 r2}
  static constexpr bool MID = false;
  const C* in;
  C* scr;
  long long ld, lds;  // row strides of the slab and of the scratch
  int W, ncols, R2;
  ColChirp k;
  const double2* ptab;
  const C* twr;  // natural twiddles of length R
  __device__ C load(long long tile, int w, int a) const {
    const int cb = ncols / W;
    const long long r2 = tile / cb, c = (tile % cb) * W + w;
    const long long r = (long long)a * R2 + r2;
    return ColPhase<C>::pre(k, ptab, r, in[r * ld + c]);
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const int cb = ncols / W;
    const long long r2 = tile / cb, c = (tile % cb) * W + w;
    scr[((long long)a * R2 + r2) * lds + c] = cmul(v, twr[(long long)a * r2]);
  }
};

template <class C>
struct OpColLct2 {  // pass 2: DFT over r2 for the line (k1, c); natural row j = k1 + R1 k2
  static constexpr bool MID = false;
  const C* scr;
  C* out;
  long long ld, lds;
  int W, ncols, R1, R2;
  ColChirp k;
  const double2* cptab;
  __device__ C load(long long tile, int w, int a) const {
    const int cb = ncols / W;
    const long long k1 = tile / cb, c = (tile % cb) * W + w;
    return scr[(k1 * R2 + a) * lds + c];
  }
  __device__ void store(long long tile, int w, int a, C v) const {
    const int cb = ncols / W;
    const long long k1 = tile / cb, c = (tile % cb) * W + w;
    const long long j = k1 + (long long)R1 * a;
    out[j * ld + c] = ColPhase<C>::post(k, cptab, j, v);
  }
};

unsigned long long frac_q64_host(long double v) {
  long double f = v - floorl(v);
  if (!(f >= 0.0L && f < 1.0L)) f = 0.0L;
  return (unsigned long long)(f * 18446744073709551616.0L);
}

ColChirp col_chirp(const double* abcd, int64_t R, int bare) {
  ColChirp k{};
  const double a = abcd[0], b = abcd[1], d = abcd[3];
  k.cin = (0.5 * a) / b;  // IEEE double division: the reference's (0.5j * a / b).imag
  k.cout = (0.5 * d) / b;
  k.s4 = (4.0 * b) / 3.141592653589793116;
  k.half = host_half_step(R);
  k.pre = a != 0.0;
  k.post = d != 0.0;
  k.R = R;
  int l = 0;
  while ((int64_t(1) << l) < R) ++l;
  k.log2r = l;
  const long double h2 = (long double)k.half * k.half;
  const long double i2pi = 1.0L / (2.0L * PI_L);
  k.dq_in = frac_q64_host(k.cin * h2 * i2pi);
  k.dq_out = frac_q64_host(k.cout * (long double)k.s4 * k.s4 * h2 * i2pi);
  const int64_t red = (int64_t)(((__int128)(R - 1) * (R - 1)) % (4 * (__int128)R));
  unsigned long long gq = 0ull - ((unsigned long long)red << (62 - l));
  gq += (b > 0.0) ? (0ull - (1ull << 61)) : (1ull << 61);
  if (bare) gq += (1ull << 61);
  k.gq = (unsigned)(gq >> 32);
  const long double gabs = (PI_L / sqrtl(2.0L * R)) / sqrtl(2.0L * PI_L * fabsl((long double)b)) * (bare ? sqrtl(2.0L * PI_L) : 1.0L);
  k.gabs = (float)gabs;
  // c128 row factor e^{-i pi sgn(b)/4}/sqrt(2 pi |b|) [* sqrt(2 pi i)] (C(n) p_j is in cptab)
  const long double h = 0.70710678118654752440L / sqrtl(2.0L * PI_L * fabsl((long double)b));
  long double gx = h, gy = b > 0.0 ? -h : h;
  if (bare) {
    const long double sp = sqrtl(PI_L);
    const long double ux = (gx - gy) * sp, uy = (gx + gy) * sp;
    gx = ux;
    gy = uy;
  }
  k.g = make_double2((double)gx, (double)gy);
  return k;
}

template <class C>
int lct_cols_narrow(const void* in, void* out, void* ws, int64_t R, int64_t ncols, int64_t ld, const double* abcd,
                    int bare, cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int W = tile_w<C>();
  if (ncols % W) return XFT_ENOTSUP;
  const int l = log2_of(R);
  const ColChirp k = col_chirp(abcd, R, bare);
  const double2 *ptab = nullptr, *cptab = nullptr;
  int rc = boundary_tables(R, &ptab, &cptab);
  if (rc) return rc;
  if (l <= LMAX) {
    OpColLctOne<C> op{static_cast<const C*>(in), static_cast<C*>(out), ld, W, k, ptab, cptab};
    return tile<C, true, true, -1>(l, ncols / W, op, st);
  }
  const Shape sh = split(l);
  const int R1 = 1 << sh.l1, R2 = 1 << sh.l2;
  const void* twr = nullptr;
  if ((rc = natural_twiddles(R, dtype, &twr))) return rc;
  OpColLct1<C> op1{static_cast<const C*>(in), static_cast<C*>(ws), ld, ld, W, (int)ncols, R2, k, ptab,
                   static_cast<const C*>(twr)};
  if ((rc = tile<C, true, true, -1>(sh.l1, (long long)R2 * (ncols / W), op1, st))) return rc;
  OpColLct2<C> op2{static_cast<const C*>(ws), static_cast<C*>(out), ld, ld, W, (int)ncols, R1, R2, k, cptab};
  return tile<C, true, true, -1>(sh.l2, (long long)R1 * (ncols / W), op2, st);
}

// ---------------------------------------------------------------------------
// Column LCT in ONE HBM round trip with a thread-block cluster (R = K * L).
// The K CTAs of a cluster own W adjacent columns at a time (a "group"); CTA c
// holds rows r = c + K m (m < L) of the group in shared memory:
//   1. 3-D bulk-tensor TMA: box {W, 1, 256} over the view [R/K][K][ncols], so
//      every row segment is W contiguous samples (64 B), double-buffered
//      across groups;
//   2. pre-chirp, length-L FFT down each column in registers + the padded
//      exchange buffer (the row kernel's passes), twiddle w_R^{c k1};
//   3. cluster barrier; CTA c' gathers Y_c[k1] for its k1 slice from all K
//      CTAs through distributed shared memory, runs the length-K DFT across
//      them (X[k1 + L k2] = sum_c w_K^{c k2} Y_c[k1]), post-chirps and stores
//      row k1 + L k2 of the group: the natural-order output, 64-B segments.
// Each sample crosses HBM once in, once out (the two-pass tile path reads and
// writes it twice).  In place is safe: a group is fully read before any of it
// is written, groups are disjoint.
// ---------------------------------------------------------------------------
#ifndef XFT_CLU14
#define XFT_CLU14 0  // R = 16384: 0 = 16-CTA clusters x 1024 rows, 1 = 8-CTA clusters x 2048 rows (half-width groups)
#endif
#ifndef XFT_CLU_E10
#define XFT_CLU_E10 32  // c64 radix of the 1024-row cluster slices (32: two passes, one warp per column)
#endif
#ifndef XFT_CLU_PROMO
#define XFT_CLU_PROMO 0  // L2 promotion of the column-group TMA loads (bytes; 0 = none)
#endif
#ifndef XFT_CLU_PF
#define XFT_CLU_PF 0  // L2 prefetch of the next group at the start of each group
#endif
#ifndef XFT_CLU_NB
#define XFT_CLU_NB 1  // group buffers per CTA (2: double-buffered TMA)
#endif
#ifndef XFT_CLU_W64
#define XFT_CLU_W64 8  // c64 columns per cluster group (8: 64-byte row segments)
#endif
#ifndef XFT_CLU_MINB
#define XFT_CLU_MINB 2  // resident CTAs per SM the registers are sized for
#endif
#ifndef XFT_COLCLU
#define XFT_COLCLU 1  // 0: always use the two-pass tile path for tall columns
#endif

__device__ __forceinline__ uint32_t clu_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t clu_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t clu_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void clu_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t clu_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void clu_ld(uint32_t a, float2& v) {
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void clu_ld(uint32_t a, double2& v) {
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void clu_st(uint32_t a, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void clu_st(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
#ifndef XFT_CLU_PUSH
#define XFT_CLU_PUSH 0  // 1: cross-CTA exchange by remote stores into the owner's buffer (A/B cfg5: 3.09 vs 2.81 ms: off)
#endif

__device__ __forceinline__ void clu_sync_relaxed() {  // WAR only: the peers' DSMEM loads have been consumed
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(map), "r"(x), "r"(y), "r"(z)
               : "memory");
}

template <class C_, int K_, int LOGL_, int W_, int NBUF_, int MINB_>
struct CluCfg {
  using C = C_;
  static constexpr int K = K_, LOGL = LOGL_, W = W_, NBUF = NBUF_, MINB = MINB_;
  static constexpr int L = 1 << LOGL, E = (sizeof(C) == 8 && LOGL == 10) ? XFT_CLU_E10 : 16, TR = L / E,
                       THREADS = W * TR;
  using Fft = PipeCfg<C, LOGL, E, MODE_DFT, -1, W, 1, 1>;
  // line stride: a 128-byte wavefront covers S = 128/sizeof(C) lanes = W lines x S/W
  // consecutive positions; LS = S/W (mod S) puts them in S distinct slots
  static constexpr int S = 128 / (int)sizeof(C);
  static constexpr int LS = Fft::NP + (((S / W) - Fft::NP % S) % S + S) % S;
  static constexpr int GS = K * W + 8;  // (see PAIRS below)
  static constexpr int BUF0 = W * LS > L * W ? W * LS : L * W;
  static constexpr int BUF1 = XFT_CLU_PUSH && (L / K) * GS > BUF0 ? (L / K) * GS : BUF0;
  static constexpr int BUF = (BUF1 * (int)sizeof(C) + 127) / 128 * 128 / (int)sizeof(C);
  static constexpr size_t SMEM = NBUF * size_t(BUF) * sizeof(C);
  static constexpr int BOXM = L < 256 ? L : 256;
  static constexpr int EW = (int)sizeof(C) / 8;  // 8-byte tensor elements per sample
  static constexpr int PAIRS = (L / K) * W;      // (k1, column) pairs a CTA finishes per group
  // push layout of the gathered values in the owner's buffer: [k1 local][source CTA][column],
  // row stride GS = K W + 8 (4 k1 rows of a warp fall on the two halves of the banks)
  static_assert(THREADS <= 1024 && L % K == 0 && W <= S, "cluster column shape");
  static_assert(!XFT_CLU_PUSH || (L / K) * GS <= BUF, "push layout fits the group buffer");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
xft_colclu_kernel(const __grid_constant__ CUtensorMap map, typename Cfg::C* __restrict__ out, long long ld,
                  int ngroups, ColChirp ck, const double2* __restrict__ ptab, const double2* __restrict__ cptab,
                  const typename Cfg::C* __restrict__ tw) {
  using C = typename Cfg::C;
  constexpr int K = Cfg::K, L = Cfg::L, W = Cfg::W, E = Cfg::E, TR = Cfg::TR, T = Cfg::THREADS, NB = Cfg::NBUF;
  constexpr int LOGR = Cfg::LOGL + ilog2(K);
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t bars[2];
  C* const buf0 = reinterpret_cast<C*>(xft_smem);
  const int c = (int)clu_rank();
  const int q = (int)clu_id(), nq = (int)clu_count();
  const int t = threadIdx.x, w = t % W, j = t / W;
  auto noop = []() {};
  auto issue = [&](int g, int b) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[b], (uint32_t)(L * W * sizeof(C)));
#pragma unroll 1
    for (int m0 = 0; m0 < L; m0 += Cfg::BOXM)
      tma_load_3d(buf0 + b * Cfg::BUF + m0 * W, &map, g * W * Cfg::EW, c, m0, &bars[b]);
  };
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if (q < ngroups) issue(q, 0);
    if (NB == 2 && q + nq < ngroups) issue(q + nq, 1);
  }
  __syncthreads();
  int it = 0;
  for (int g = q; g < ngroups; g += nq, ++it) {
    const int b = NB == 2 ? (it & 1) : 0;
    C* const X = buf0 + b * Cfg::BUF;
    mbar_wait(&bars[b], (uint32_t)((NB == 2 ? it >> 1 : it) & 1));
    if (XFT_CLU_PF && t == 0 && g + NB * nq < ngroups) {
      // warm L2 with the group this buffer takes next: its TMA load (issued after
      // the gather) then streams from L2 instead of waiting on HBM
#pragma unroll 1
      for (int m0 = 0; m0 < L; m0 += Cfg::BOXM) tma_prefetch_3d(&map, (g + NB * nq) * W * Cfg::EW, c, m0);
    }
    C v[E];
    if constexpr (sizeof(C) == 8) {
      // this thread's rows r = r0 + s K TR: the chirp + boundary phase is a quadratic walk in s
      const int r0 = c + K * j;
      const uint32_t bt0 = ((uint32_t)(r0 & 1) << 31) - ((uint32_t)r0 << (31 - LOGR));
      TurnWalk wk(ck.dq_in, 2 * r0 - (1 << LOGR) + 1, 2 * K * TR, (unsigned long long)bt0 << 32,
                  (unsigned long long)(K * TR) << (63 - LOGR));
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = cmul(walk_phasor(wk.next()), X[(j + s * TR) * W + w]);
    } else {
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int m = j + s * TR;
        v[s] = ColPhase<C>::pre(ck, ptab, c + (long long)K * m, X[m * W + w]);
      }
    }
    pipe_passes<typename Cfg::Fft, 0>(v, X + w * Cfg::LS, j, tw, noop);
    const uint32_t xaddr = smem_addr(X);
    if constexpr (XFT_CLU_PUSH) {
      // every CTA of the cluster is done with its buffer: Y_c[k1][w] goes straight into the
      // buffer of the CTA that owns k1 (remote stores: no load latency on the critical path)
      clu_sync();
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k1 = j + s * TR;
        C y = v[s];
        if constexpr (sizeof(C) == 8) {  // w_R^{c k1}, exact turns
          y = cmul(walk_phasor((0u - ((uint32_t)(c * k1) << (32 - LOGR))) + ((512u - 326u) << 0)), y);
        } else {
          double sn, cs;
          sincospi(-2.0 * (double)(c * k1) / (double)(K * L), &sn, &cs);
          y = cmul(make_double2(cs, sn), y);
        }
        const int owner = k1 / (L / K), kl = k1 % (L / K);
        clu_st(clu_map(xaddr + (uint32_t)((kl * Cfg::GS + c * W + w) * sizeof(C)), owner), y);
      }
      clu_sync();  // every push into this CTA's buffer has landed
    } else {
      __syncthreads();  // the exchange buffer is dead; it now receives Y[k1][w]
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k1 = j + s * TR;
        C y = v[s];
        if constexpr (sizeof(C) == 8) {  // w_R^{c k1}, exact turns
          y = cmul(walk_phasor((0u - ((uint32_t)(c * k1) << (32 - LOGR))) + ((512u - 326u) << 0)), y);
        } else {
          double sn, cs;
          sincospi(-2.0 * (double)(c * k1) / (double)(K * L), &sn, &cs);
          y = cmul(make_double2(cs, sn), y);
        }
        X[k1 * W + w] = y;
      }
      clu_sync();
    }
#pragma unroll 1
    for (int p = t; p < Cfg::PAIRS; p += T) {
      const int pw = p % W, k1 = c * (L / K) + p / W;
      C y[K];
      if constexpr (XFT_CLU_PUSH) {
        const C* g = X + (p / W) * Cfg::GS + pw;
#pragma unroll
        for (int cc = 0; cc < K; ++cc) y[cc] = g[cc * W];
      } else {
        const uint32_t la = xaddr + (uint32_t)((k1 * W + pw) * sizeof(C));
#pragma unroll
        for (int cc = 0; cc < K; ++cc) clu_ld(clu_map(la, cc), y[cc]);
      }
      dft_r<K, -1>(y);
      C* dst = out + (long long)k1 * ld + (long long)g * W + pw;
      const long long step = (long long)L * ld;
      if constexpr (sizeof(C) == 8) {
        // output rows k1 + L k2: post-chirp + boundary + arg G walk in k2
        const uint32_t bt0 = ((uint32_t)(k1 & 1) << 31) - ((uint32_t)k1 << (31 - LOGR)) + ck.gq;
        TurnWalk wk(ck.dq_out, 2 * k1 - (1 << LOGR) + 1, 2 * L, (unsigned long long)bt0 << 32,
                    (unsigned long long)L << (63 - LOGR));
        const float2 gg = make_float2(ck.gabs, ck.gabs);
#pragma unroll
        for (int k2 = 0; k2 < K; ++k2) dst[k2 * step] = cmul(walk_phasor(wk.next()), p_mul(y[k2], gg));
      } else {
#pragma unroll
        for (int k2 = 0; k2 < K; ++k2) dst[k2 * step] = ColPhase<C>::post(ck, cptab, k1 + (long long)L * k2, y[k2]);
      }
    }
    if constexpr (XFT_CLU_PUSH) {
      __syncthreads();  // this CTA's own reads of its buffer are done (peers push only after the next A')
    } else {
      clu_sync_relaxed();  // every peer is done reading this CTA's Y
    }
    if (t == 0) {
      const int gn = g + NB * nq;
      if (gn < ngroups) issue(gn, b);
    }
  }
}

// ---------------------------------------------------------------------------
// K6b: the same cluster column transform with the cross-CTA exchange done by the
// copy engines.  Per group: TMA the column group into one of two buffers (the
// next group's load is issued while this one is exchanged), FFT, write
// Y_c[k1][w] k1-major, then ONE thread issues K bulk copies
// (cp.async.bulk.shared::cluster.shared::cta, 4 KB each) that deliver the k1
// slice owned by CTA o straight into o's receive buffer, completing on o's
// mbarrier; each CTA waits only on its own mbarrier (no cluster-wide barrier
// on the data path) and gathers locally.  The only cluster barrier is split:
// arrive after this CTA's gather, wait one group later before the next copies
// (the receive buffers are free) -- the FFT of the next group sits in between.
// One CTA per SM (two group buffers + the receive buffer: ~200 KB).
// ---------------------------------------------------------------------------
#ifndef XFT_CLU_BULK
#define XFT_CLU_BULK 0  // 1: c64 16-CTA column clusters with the copy-engine exchange (K6b). A/B cfg5:
                        // 3.35 ms (W = 8, one CTA/SM), 3.03 ms (W = 4, two/SM) vs 2.81 ms for K6: off
#endif
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
               : "memory");
}
__device__ __forceinline__ void clu_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void clu_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
xft_colclu2_kernel(const __grid_constant__ CUtensorMap map, typename Cfg::C* __restrict__ out, long long ld,
                   int ngroups, ColChirp ck, const double2* __restrict__ ptab, const double2* __restrict__ cptab,
                   const typename Cfg::C* __restrict__ tw) {
  using C = typename Cfg::C;
  static_assert(sizeof(C) == 8, "K6b is the c64 path");
  constexpr int K = Cfg::K, L = Cfg::L, W = Cfg::W, E = Cfg::E, TR = Cfg::TR, T = Cfg::THREADS;
  constexpr int LOGR = Cfg::LOGL + ilog2(K);
  constexpr int SL = (L / K) * W;  // elements of one k1 slice (the chunk one CTA sends another)
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ __align__(8) uint64_t rxbar;
  C* const buf0 = reinterpret_cast<C*>(xft_smem);
  C* const RX = buf0 + 2 * Cfg::BUF;  // [source CTA][k1 local][column]
  const int c = (int)clu_rank();
  const int q = (int)clu_id(), nq = (int)clu_count();
  const int t = threadIdx.x, w = t % W, j = t / W;
  auto noop = []() {};
  auto issue = [&](int g, int b) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[b], (uint32_t)(L * W * sizeof(C)));
#pragma unroll 1
    for (int m0 = 0; m0 < L; m0 += Cfg::BOXM)
      tma_load_3d(buf0 + b * Cfg::BUF + m0 * W, &map, g * W * Cfg::EW, c, m0, &bars[b]);
  };
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&rxbar, 1);
    fence_mbar_init();
  }
  clu_sync();  // every peer's receive mbarrier is initialised before any copy completes on it
  if (t == 0 && q < ngroups) issue(q, 0);
  const uint32_t rx_local = smem_addr(RX + c * SL), rxbar_local = smem_addr(&rxbar);
  int it = 0;
  for (int g = q; g < ngroups; g += nq, ++it) {
    const int b = it & 1;
    C* const X = buf0 + b * Cfg::BUF;
    mbar_wait(&bars[b], (uint32_t)((it >> 1) & 1));
    C v[E];
    {
      // this thread's rows r = r0 + s K TR: the chirp + boundary phase is a quadratic walk in s
      const int r0 = c + K * j;
      const uint32_t bt0 = ((uint32_t)(r0 & 1) << 31) - ((uint32_t)r0 << (31 - LOGR));
      TurnWalk wk(ck.dq_in, 2 * r0 - (1 << LOGR) + 1, 2 * K * TR, (unsigned long long)bt0 << 32,
                  (unsigned long long)(K * TR) << (63 - LOGR));
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = cmul(walk_phasor(wk.next()), X[(j + s * TR) * W + w]);
    }
    pipe_passes<typename Cfg::Fft, 0>(v, X + w * Cfg::LS, j, tw, noop);
    __syncthreads();  // the exchange buffer is dead; it now holds Y[k1][w], k1-major
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k1 = j + s * TR;
      X[k1 * W + w] = cmul(walk_phasor((0u - ((uint32_t)(c * k1) << (32 - LOGR))) + ((512u - 326u) << 0)), v[s]);
    }
    fence_proxy_async_smem();  // the copy engine reads what these threads wrote
    if (it > 0) clu_wait();    // every CTA has gathered the previous group: receive buffers are free
    __syncthreads();
    if (t == 0) {
      // the other buffer held the previous group's Y, whose copies have all landed (the wait above)
      const int gn = g + nq;
      if (gn < ngroups) issue(gn, b ^ 1);
      mbar_arrive_expect_tx(&rxbar, (uint32_t)(L * W * sizeof(C)));  // K chunks of this group
      const uint32_t src0 = smem_addr(X);
#pragma unroll 1
      for (int o = 0; o < K; ++o)
        bulk_s2c(clu_map(rx_local, o), src0 + (uint32_t)(o * SL * sizeof(C)), (uint32_t)(SL * sizeof(C)),
                 clu_map(rxbar_local, o));
    }
    mbar_wait(&rxbar, (uint32_t)(it & 1));
#pragma unroll 1
    for (int p = t; p < Cfg::PAIRS; p += T) {
      const int pw = p % W, kl = p / W, k1 = c * (L / K) + kl;
      C y[K];
#pragma unroll
      for (int cc = 0; cc < K; ++cc) y[cc] = RX[cc * SL + kl * W + pw];
      dft_r<K, -1>(y);
      C* dst = out + (long long)k1 * ld + (long long)g * W + pw;
      const long long step = (long long)L * ld;
      // output rows k1 + L k2: post-chirp + boundary + arg G walk in k2
      const uint32_t bt0 = ((uint32_t)(k1 & 1) << 31) - ((uint32_t)k1 << (31 - LOGR)) + ck.gq;
      TurnWalk wk(ck.dq_out, 2 * k1 - (1 << LOGR) + 1, 2 * L, (unsigned long long)bt0 << 32,
                  (unsigned long long)L << (63 - LOGR));
      const float2 gg = make_float2(ck.gabs, ck.gabs);
#pragma unroll
      for (int k2 = 0; k2 < K; ++k2) dst[k2 * step] = cmul(walk_phasor(wk.next()), p_mul(y[k2], gg));
    }
    clu_arrive();  // this CTA's receive buffer may be refilled
  }
  if (it > 0) clu_wait();  // pairs the last arrive; no peer touches this CTA's memory afterwards
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}


template <class C, int K, int LOGL, int W, int NBUF = 1, int MINB = 2, bool BULK = false>
int launch_colclu(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, const ColChirp& ck,
                  const double2* ptab, const double2* cptab, cudaStream_t st, int64_t ld_out = -1,
                  bool probe = false) {
  if (ld_out < 0) ld_out = ld;
  using Cfg = CluCfg<C, K, LOGL, W, NBUF, MINB>;
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  if (R != (int64_t)K * Cfg::L || ncols % W || ncols / W > INT32_MAX || ld % 2) return XFT_ENOTSUP;
  auto enc = tensor_encoder();
  if (!enc) return XFT_ENOTSUP;
  Tables tb;
  int rc = get_tables(Cfg::L, dtype, &tb, Cfg::E);
  if (rc) return rc;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)(ncols * Cfg::EW), (cuuint64_t)K, (cuuint64_t)(R / K)};
  const cuuint64_t strides[2] = {(cuuint64_t)(ld * sizeof(C)), (cuuint64_t)(K * ld * sizeof(C))};
  const cuuint32_t box[3] = {(cuuint32_t)(W * Cfg::EW), 1u, (cuuint32_t)Cfg::BOXM};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(in), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          XFT_CLU_PROMO == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
          : XFT_CLU_PROMO == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
          : XFT_CLU_PROMO == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return XFT_ENOTSUP;
  void (*kern)(const CUtensorMap, C*, long long, int, ColChirp, const double2*, const double2*, const C*);
  if constexpr (BULK) kern = xft_colclu2_kernel<Cfg>;
  else kern = xft_colclu_kernel<Cfg>;
  const size_t smem = BULK ? (2 * (size_t)Cfg::BUF + (size_t)Cfg::L * W) * sizeof(C) : Cfg::SMEM;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return XFT_ECUDA;
  if (K > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return XFT_ENOTSUP;
  }
  const int groups = (int)(ncols / W);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(K * groups));
  int maxc = 0;
  if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess || maxc < 1) {
    cudaGetLastError();
    return XFT_ENOTSUP;
  }
  if (probe) return XFT_OK;  // everything checked, nothing launched
  const int ncl = groups < maxc ? groups : maxc;
  cfg.gridDim = dim3((unsigned)(K * ncl));
  if (cudaLaunchKernelEx(&cfg, kern, map, static_cast<C*>(out), (long long)ld_out, groups, ck, ptab, cptab,
                         static_cast<const C*>(tb.tw)) != cudaSuccess)
    return XFT_ECUDA;
  return XFT_OK;
}

// tall columns through the cluster kernel: R = K * 1024 (K = 2..16), 64-byte row segments
template <class C>
int lct_cols_cluster(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, const ColChirp& ck,
                     const double2* ptab, const double2* cptab, cudaStream_t st, int64_t ld_out = -1,
                     bool probe = false) {
  constexpr int W = sizeof(C) == 8 ? XFT_CLU_W64 : 4;
  if (!XFT_COLCLU || ncols % W) return XFT_ENOTSUP;
  switch (log2_of(R)) {
#if XFT_CLU14 == 1
    case 14: return launch_colclu<C, 8, 11, W / 2, XFT_CLU_NB, XFT_CLU_MINB>(in, out, R, ncols, ld, ck, ptab, cptab, st, ld_out, probe);
#else
    case 14:
      if constexpr (sizeof(C) == 8 && XFT_CLU_BULK && (W == 8 || W == 4))
        return launch_colclu<C, 16, 10, W, 1, (W == 4 ? 2 : 1), true>(in, out, R, ncols, ld, ck, ptab, cptab, st,
                                                                        ld_out, probe);
      else
        return launch_colclu<C, 16, 10, W, XFT_CLU_NB, XFT_CLU_MINB>(in, out, R, ncols, ld, ck, ptab, cptab, st, ld_out, probe);
#endif
    case 13: return launch_colclu<C, 8, 10, W>(in, out, R, ncols, ld, ck, ptab, cptab, st, ld_out, probe);
    case 12: return launch_colclu<C, 4, 10, W>(in, out, R, ncols, ld, ck, ptab, cptab, st, ld_out, probe);
    case 11: return launch_colclu<C, 2, 10, W>(in, out, R, ncols, ld, ck, ptab, cptab, st, ld_out, probe);
    default: return XFT_ENOTSUP;
  }
}

#include "xft_colring.cuh"

#ifndef XFT_COLSLAB_MB
#define XFT_COLSLAB_MB 4096  // L2-resident scratch per column slab (4096: one slab; smaller slabs measured slower)
#endif
#ifndef XFT_COLW
#define XFT_COLW 4  // column tiles: 512 contiguous bytes per access (DRAM page locality)
#endif
template <class C>
int lct_cols(const void* in, void* out, void* ws, int64_t R, int64_t ncols, int64_t ld, const double* abcd, int bare,
             cudaStream_t st) {
  constexpr int dtype = sizeof(C) == 8 ? XFT_C64 : XFT_C128;
  constexpr int W = tile_w<C>() * XFT_COLW;
  const int l = log2_of(R);
  if (l > LMAX) {  // tall columns: one HBM round trip through a cluster when the shape allows
    const ColChirp k = col_chirp(abcd, R, bare);
    const double2 *ptab = nullptr, *cptab = nullptr;
    int rc = boundary_tables(R, &ptab, &cptab);
    if (rc) return rc;
    if constexpr (sizeof(C) == 8) {  // c64, 2^14 .. 2^16 rows: two passes through an L2-resident ring (K7)
      rc = lct_cols_ring(in, out, R, ncols, ld, ld, k, st);
      if (rc != XFT_ENOTSUP) return rc;
    }
    rc = lct_cols_cluster<C>(in, out, R, ncols, ld, k, ptab, cptab, st);
    if (rc != XFT_ENOTSUP) return rc;
  }
  // wide tiles for the two-pass (four-step) heights; one-pass heights use 128-byte tiles
  if (ncols % W || l <= LMAX) return lct_cols_narrow<C>(in, out, ws, R, ncols, ld, abcd, bare, st);
  const ColChirp k = col_chirp(abcd, R, bare);
  const double2 *ptab = nullptr, *cptab = nullptr;
  int rc = boundary_tables(R, &ptab, &cptab);
  if (rc) return rc;
  const Shape sh = split(l);
  const int R1 = 1 << sh.l1, R2 = 1 << sh.l2;
  const void* twr = nullptr;
  if ((rc = natural_twiddles(R, dtype, &twr))) return rc;
  // column slabs whose [R][slab] scratch fits in L2: the intermediate of the
  // two passes never goes to HBM, so the column transform costs one HBM round trip
  int64_t slab = ((int64_t)XFT_COLSLAB_MB << 20) / (R * (int64_t)sizeof(C));
  slab = slab < W ? W : (slab / W) * W;
  if (slab > ncols) slab = ncols;
  for (int64_t c0 = 0; c0 < ncols; c0 += slab) {
    const int64_t cw = ncols - c0 < slab ? ncols - c0 : slab;
    if (cw % W) return lct_cols_narrow<C>(static_cast<const C*>(in) + c0, static_cast<C*>(out) + c0, ws, R, cw, ld,
                                          abcd, bare, st);
    OpColLct1<C> op1{static_cast<const C*>(in) + c0, static_cast<C*>(ws), ld, cw, W, (int)cw, R2, k, ptab,
                     static_cast<const C*>(twr)};
    if ((rc = tile<C, true, true, -1, OpColLct1<C>, W>(sh.l1, (long long)R2 * (cw / W), op1, st))) return rc;
    OpColLct2<C> op2{static_cast<const C*>(ws), static_cast<C*>(out) + c0, ld, cw, W, (int)cw, R1, R2, k, cptab};
    if ((rc = tile<C, true, true, -1, OpColLct2<C>, W>(sh.l2, (long long)R1 * (cw / W), op2, st))) return rc;
  }
  return XFT_OK;
}

}  // namespace

namespace xftb {

// tall columns through the cluster kernel only, reading a [R][ncols] slab with
// row stride ld and writing rows of stride ld_out (XFT_ENOTSUP if the cluster
// path does not take this shape; nothing has been launched then)
int run_lct_cols_cluster(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, int64_t ld_out, int dtype,
                         const double* abcd_host, int flags, cudaStream_t st, bool probe) {
  const int l = log2_of(R);
  if ((int64_t(1) << l) != R || l <= LMAX || l > 14) return XFT_ENOTSUP;
  const int bare = (flags & XFT_FLAG_BARE_FOURIER) ? 1 : 0;
  const ColChirp k = col_chirp(abcd_host, R, bare);
  const double2 *ptab = nullptr, *cptab = nullptr;
  int rc = boundary_tables(R, &ptab, &cptab);
  if (rc) return rc;
  return dtype == XFT_C64 ? lct_cols_cluster<float2>(in, out, R, ncols, ld, k, ptab, cptab, st, ld_out, probe)
                          : lct_cols_cluster<double2>(in, out, R, ncols, ld, k, ptab, cptab, st, ld_out, probe);
}

// true when the L2-staged column path (K7) takes this shape on this device (nothing launched)
bool lct_cols_ring_ok(const void* in, int64_t R, int64_t ncols, int64_t ld, int dtype) {
  const int l = log2_of(R);
  if (dtype != XFT_C64 || (int64_t(1) << l) != R) return false;
  ColChirp k{};
  return lct_cols_ring(in, nullptr, R, ncols, ld, ld, k, nullptr, true) == XFT_OK;
}

// K7 schedule of tile `index` (host only): out = {pass, super-block, column block, line index, ring slot},
// info = {tiles, super-blocks, lag, slots, tiles per pass-1 / pass-2 block-phase}
int ring_schedule(int64_t R, int64_t ncols, int64_t index, int* out, int* info) {
  const int l = log2_of(R);
  int l1, l2, W;
  if ((int64_t(1) << l) != R || ncols < 1 || !ring_shape(l, &l1, &l2, &W)) return XFT_ENOTSUP;
  const RingPlan pl = ring_plan(l1, l2, W, ncols, ncols, ncols);
  if (info) {
    info[0] = (int)pl.total;
    info[1] = pl.nsb;
    info[2] = pl.lag;
    info[3] = pl.slots;
    info[4] = (int)pl.T0;
    info[5] = (int)pl.T1;
  }
  if (out) {
    if (index < 0) return XFT_EINVALID_SIZE;
    const RingTile t = ring_decode(pl, (unsigned)(index < (int64_t)pl.total ? index : pl.total));
    out[0] = t.phase;
    out[1] = t.sb;
    out[2] = t.cb;
    out[3] = t.idx;
    out[4] = t.phase == 2 ? -1 : t.sb % pl.slots;
  }
  return XFT_OK;
}

int run_lct_cols(const void* in, void* out, void* ws, int64_t R, int64_t ncols, int64_t ld, int dtype,
                 const double* abcd_host, int flags, cudaStream_t st) {
  const int l = log2_of(R);
  if ((int64_t(1) << l) != R || l < LMIN || l > 2 * LMAX) return XFT_ENOTSUP;
  const int bare = (flags & XFT_FLAG_BARE_FOURIER) ? 1 : 0;
  return dtype == XFT_C64 ? lct_cols<float2>(in, out, ws, R, ncols, ld, abcd_host, bare, st)
                          : lct_cols<double2>(in, out, ws, R, ncols, ld, abcd_host, bare, st);
}

}  // namespace xftb
