// K1/K2: batched chirp-DFT-chirp kernel over rows that fit one CTA's shared memory.
//
// One CTA owns ROWS whole rows (ROWS = 1 for n >= 256*E); each row is
// transformed by TR = n/E threads holding E complex samples in registers.
// The DFT is a Stockham autosort factorisation: a first radix-R0 pass
// (R0 = n / E^(P-1)) followed by radix-E passes, every butterfly in
// registers, the data exchanged between passes through XOR-swizzled shared
// memory (bank-conflict free for the 16-byte c128 and 8-byte c64 patterns),
// twiddles read from an L1/L2-resident table e^{-2 pi i m/n}.
//
//  * the first pass reads its inputs straight from HBM with coalesced loads
//    (thread j, register s <- element j + s*TR) and applies the pre-chirp
//    p_k * e^{i phi_k} on the fly (reference: xft/lct.py:204-205,
//    xft/kernel.py:51-65, 98-102);
//  * the last pass leaves element j + s*TR in register s, applies the
//    post-scale C(n) p_j e^{i psi_j} / sqrt(2 pi i b) and stores coalesced
//    (reference: xft/lct.py:207, xft/kernel.py:45-48, 105-113).
//
// HBM traffic is exactly one read and one write of every sample.
// The phases phi_k = fl(fl(0.5a/b) * fl(x_k^2)), x_k = fl((2k-n+1)*half),
// psi_j = fl(fl(0.5d/b) * fl(y_j^2)), y_j = fl(fl(4b/pi) * x_j) are formed
// with explicitly rounded fp64 products (no FMA contraction), i.e. the exact
// fp64 arguments the reference passes to exp.
#pragma once
#include "xft_device.cuh"

namespace xftb {

enum Mode { MODE_DFT = 0, MODE_SCALED = 1, MODE_LCT = 2 };
enum { FLAG_BARE_FOURIER = 1 };

struct Abcd {
  double a, b, c, d;
};

struct RowCoef {
  double cin, cout, s4;   // 0.5a/b, 0.5d/b, 4b/pi (each one correctly rounded op)
  double gx, gy;          // C(n) / sqrt(2 pi i b)  [* sqrt(2 pi i) for xft_fourier]
  int pre, post;          // chirps present (a != 0, d != 0)
};

__device__ __forceinline__ void make_row_coef(RowCoef& rc, const double* p, Abcd uni, double2 cn, int flags) {
  const double a = p ? p[0] : uni.a, b = p ? p[1] : uni.b, d = p ? p[3] : uni.d;
  rc.cin = __ddiv_rn(0.5 * a, b);      // (0.5j * a / b).imag   xft/kernel.py:102
  rc.cout = __ddiv_rn(0.5 * d, b);     // (0.5j * d / b).imag   xft/kernel.py:113
  rc.s4 = __ddiv_rn(4.0 * b, 3.141592653589793116);  // 4.0 * b / np.pi   xft/lct.py:196
  rc.pre = (a != 0.0);
  rc.post = (d != 0.0);
  // 1/sqrt(2 pi i b) = e^{-i pi sgn(b)/4} / sqrt(2 pi |b|)   (principal branch)
  const double inv = 1.0 / sqrt(6.283185307179586232 * fabs(b));
  const double h = 0.70710678118654752440 * inv;
  double gx = h, gy = (b > 0.0) ? -h : h;
  // times C(n)
  double tx = cn.x * gx - cn.y * gy;
  double ty = cn.x * gy + cn.y * gx;
  if (flags & FLAG_BARE_FOURIER) {  // sqrt(2 pi i) = sqrt(pi) (1 + i)
    const double sp = 1.772453850905516104;
    const double ux = (tx - ty) * sp, uy = (tx + ty) * sp;
    tx = ux;
    ty = uy;
  }
  rc.gx = tx;
  rc.gy = ty;
}

template <class C> __device__ __forceinline__ C to_c(double2 a);
template <> __device__ __forceinline__ float2 to_c<float2>(double2 a) { return make_float2((float)a.x, (float)a.y); }
template <> __device__ __forceinline__ double2 to_c<double2>(double2 a) { return a; }

// XOR swizzle of a within-row element index (bank analysis)
template <class C> __device__ __forceinline__ int swz(int p);
template <> __device__ __forceinline__ int swz<float2>(int p) { return p ^ ((p >> 4) & 15); }
template <> __device__ __forceinline__ int swz<double2>(int p) { return p ^ (((p >> 3) ^ (p >> 4)) & 7); }

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }
constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

template <class C_, int LOG2N_, int E_, int MODE_, int SIGN_>
struct RowCfg {
  using C = C_;
  static constexpr int LOG2N = LOG2N_;
  static constexpr int N = 1 << LOG2N;
  static constexpr int E = E_;
  static constexpr int MODE = MODE_;
  static constexpr int SIGN = SIGN_;
  static constexpr int TR = N / E;
  static constexpr int ROWS = TR >= 256 ? 1 : 256 / TR;
  static constexpr int THREADS = TR * ROWS;
  static constexpr int LE = ilog2(E) > 0 ? ilog2(E) : 1;
  static constexpr int NPASS = LOG2N == 0 ? 0 : (LOG2N + LE - 1) / LE;
  static constexpr int R0 = NPASS == 0 ? 1 : (1 << (LOG2N - (NPASS - 1) * LE));
  static constexpr size_t SMEM = NPASS > 1 ? size_t(ROWS) * N * sizeof(C) : 0;
  static_assert(E >= 1 && (E & (E - 1)) == 0 && E <= 32, "E");
  static_assert(THREADS <= 1024, "threads");
};

template <class Cfg, int P>
__device__ __forceinline__ void row_pass(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                         const typename Cfg::C* __restrict__ tw) {
  using C = typename Cfg::C;
  constexpr int E = Cfg::E, TR = Cfg::TR, N = Cfg::N;
  constexpr int R = (P == 0) ? Cfg::R0 : E;
  constexpr int NS = (P == 0) ? 1 : Cfg::R0 * ipow(E, P - 1);
  constexpr int NB = E / R;
  constexpr bool LAST = (P == Cfg::NPASS - 1);
  constexpr int TWSTRIDE = N / (NS * R);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int i = j + b * TR;
    const int k = i & (NS - 1);
    C u[R];
#pragma unroll
    for (int t = 0; t < R; ++t) u[t] = v[b + t * NB];
    if constexpr (NS > 1) {
#pragma unroll
      for (int t = 1; t < R; ++t) {
        C w = __ldg(&tw[t * k * TWSTRIDE]);
        if (Cfg::SIGN > 0) w = cconj(w);
        u[t] = cmul(u[t], w);
      }
    }
    dft_r<R, Cfg::SIGN>(u);
#pragma unroll
    for (int t = 0; t < R; ++t) v[b + t * NB] = u[t];
  }
  if constexpr (!LAST) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = j + b * TR;
      const int k = i & (NS - 1);
      const int base = (i - k) * R + k;
#pragma unroll
      for (int t = 0; t < R; ++t) rs[swz<C>(base + t * NS)] = v[b + t * NB];
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < E; ++s) v[s] = rs[swz<C>(j + s * TR)];
    __syncthreads();
  }
}

template <class Cfg, int P>
__device__ __forceinline__ void row_passes(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                           const typename Cfg::C* __restrict__ tw) {
  if constexpr (P < Cfg::NPASS) {
    row_pass<Cfg, P>(v, rs, j, tw);
    row_passes<Cfg, P + 1>(v, rs, j, tw);
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS)
xft_rows_kernel(const typename Cfg::C* __restrict__ in, typename Cfg::C* __restrict__ out, long long batch,
                const double* __restrict__ abcd, long long abcd_stride, Abcd uni, const typename Cfg::C* __restrict__ tw,
                const typename Cfg::C* __restrict__ ptab, double2 cn, double half, int flags) {
  using C = typename Cfg::C;
  constexpr int E = Cfg::E, TR = Cfg::TR, N = Cfg::N, ROWS = Cfg::ROWS;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ RowCoef coef[Cfg::MODE == MODE_LCT ? ROWS : 1];

  const int tid = threadIdx.x;
  const int lrow = tid / TR;
  const int j = tid - lrow * TR;
  const long long row = (long long)blockIdx.x * ROWS + lrow;
  const bool active = row < batch;
  C* rs = reinterpret_cast<C*>(xft_smem) + (size_t)lrow * N;

  if constexpr (Cfg::MODE == MODE_LCT) {
    if (j == 0 && active) make_row_coef(coef[lrow], abcd ? abcd + row * abcd_stride : nullptr, uni, cn, flags);
    __syncthreads();
  }

  // ---- load + pre-chirp (coalesced: register s <- element j + s*TR) -------
  C v[E];
  const C* src = in + row * N;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int pos = j + s * TR;
    C f = active ? src[pos] : czero<C>();
    if constexpr (Cfg::MODE == MODE_SCALED) {
      f = cmul(__ldg(&ptab[pos]), f);
    } else if constexpr (Cfg::MODE == MODE_LCT) {
      C m = __ldg(&ptab[pos]);
      if (coef[lrow].pre) {
        const double x = __dmul_rn((double)(2 * pos - N + 1), half);
        const double phi = __dmul_rn(coef[lrow].cin, __dmul_rn(x, x));
        m = cmul(m, phase_of<C>::eval(phi));
      }
      f = cmul(m, f);
    }
    v[s] = f;
  }

  row_passes<Cfg, 0>(v, rs, j, tw);

  // ---- post-scale + store (coalesced: register s -> element j + s*TR) ------
  if (!active) return;
  C* dst = out + row * N;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int pos = j + s * TR;
    C o = v[s];
    if constexpr (Cfg::MODE == MODE_SCALED) {
      o = cmul(to_c<C>(cn), cmul(__ldg(&ptab[pos]), o));
    } else if constexpr (Cfg::MODE == MODE_LCT) {
      const RowCoef& rc = coef[lrow];
      C m = cmul(to_c<C>(make_double2(rc.gx, rc.gy)), __ldg(&ptab[pos]));
      if (rc.post) {
        const double x = __dmul_rn((double)(2 * pos - N + 1), half);
        const double y = __dmul_rn(rc.s4, x);
        const double psi = __dmul_rn(rc.cout, __dmul_rn(y, y));
        m = cmul(m, phase_of<C>::eval(psi));
      }
      o = cmul(m, o);
    }
    dst[pos] = o;
  }
}

}  // namespace xftb
