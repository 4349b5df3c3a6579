// Device-side building blocks for the XFT kernels (sm_100a).
//
//  * complex helpers over float2 / double2 (c64 / c128 storage types)
//  * unit_phase(): e^{i phi} for an fp64 phase argument phi.  The phase is
//    produced bit-identically to the reference (xft/kernel.py:98-113), then
//    reduced by a two-constant Cody-Waite FMA reduction (exact to ~1e-16 rad
//    for |phi| < 2^30) and evaluated with fdlibm's published minimax
//    polynomials.  Beyond 2^30 it defers to CUDA's full-range sincos.
//  * in-register radix-2/4/8/16 DFT butterflies with a compile-time sign.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace xftb {

template <class R> struct cplx;
template <> struct cplx<float> { using T = float2; };
template <> struct cplx<double> { using T = double2; };

__device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }

template <class C> __device__ __forceinline__ C czero();
template <> __device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }

template <class C> __device__ __forceinline__ C cadd(C a, C b) { return mk(a.x + b.x, a.y + b.y); }
template <class C> __device__ __forceinline__ C csub(C a, C b) { return mk(a.x - b.x, a.y - b.y); }
template <class C> __device__ __forceinline__ C cmul(C a, C b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <class C> __device__ __forceinline__ C cconj(C a) { return mk(a.x, -a.y); }
// a * (sign * i):  sign=-1 -> multiply by -i ; sign=+1 -> multiply by +i
template <int SIGN, class C> __device__ __forceinline__ C rot(C a) {
  if (SIGN < 0) return mk(a.y, -a.x);
  return mk(-a.y, a.x);
}
template <class C, class S> __device__ __forceinline__ C cscale(C a, S s) { return mk(a.x * s, a.y * s); }

// ---------------------------------------------------------------------------
// e^{i phi}
// ---------------------------------------------------------------------------
#define XFT_TWO_OVER_PI 6.36619772367581382433e-01
#define XFT_PIO2_HI 1.57079632679489655800e+00   /* pi/2 rounded to double    */
#define XFT_PIO2_MID 6.12323399573676603587e-17  /* pi/2 - XFT_PIO2_HI        */
#define XFT_ROUND_MAGIC 6755399441055744.0        /* 1.5 * 2^52                */

// fdlibm __kernel_sin / __kernel_cos coefficients (|r| <= pi/4)
__device__ __forceinline__ void sincos_poly(double r, double& s, double& c) {
  const double z = r * r;
  double ps = 1.58969099521155010221e-10;
  ps = fma(ps, z, -2.50507602534068634195e-08);
  ps = fma(ps, z, 2.75573137070700676789e-06);
  ps = fma(ps, z, -1.98412698298579493134e-04);
  ps = fma(ps, z, 8.33333333332248946124e-03);
  ps = fma(ps, z, -1.66666666666666324348e-01);
  s = fma(r * z, ps, r);
  double pc = -1.13596475577881948265e-11;
  pc = fma(pc, z, 2.08757232129817482790e-09);
  pc = fma(pc, z, -2.75573143513906633035e-07);
  pc = fma(pc, z, 2.48015872894767294178e-05);
  pc = fma(pc, z, -1.38888888888741095749e-03);
  pc = fma(pc, z, 4.16666666666666019037e-02);
  const double w = fma(-0.5, z, 1.0);
  c = fma(z * z, pc, w);
}

__device__ __forceinline__ double2 apply_quadrant(double s, double c, int q) {
  double cs = (q & 1) ? -s : c;
  double sn = (q & 1) ? c : s;
  if (q & 2) { cs = -cs; sn = -sn; }
  return make_double2(cs, sn);
}

// e^{i phi} in fp64, |error| ~ 2e-16 absolute.
__device__ __forceinline__ double2 unit_phase(double phi) {
  if (fabs(phi) < 1.0e9) {
    const double t = fma(phi, XFT_TWO_OVER_PI, XFT_ROUND_MAGIC);
    const double qd = t - XFT_ROUND_MAGIC;
    const int q = __double2loint(t);
    double r = fma(-qd, XFT_PIO2_HI, phi);
    r = fma(-qd, XFT_PIO2_MID, r);
    double s, c;
    sincos_poly(r, s, c);
    return apply_quadrant(s, c, q);
  }
  double s, c;
  sincos(phi, &s, &c);
  return make_double2(c, s);
}

// e^{i phi} for the c64 path: fp64 reduction of the fp64 phase, fp32 polynomial.
__device__ __forceinline__ float2 unit_phase_f32(double phi) {
  if (fabs(phi) < 1.0e9) {
    const double t = fma(phi, XFT_TWO_OVER_PI, XFT_ROUND_MAGIC);
    const double qd = t - XFT_ROUND_MAGIC;
    const int q = __double2loint(t);
    const float r = (float)fma(-qd, XFT_PIO2_HI, phi);
    const float z = r * r;
    // Taylor to r^9 / r^8 on |r| <= pi/4: abs error < 4e-8
    float ps = fmaf(z, 2.7557319e-06f, -1.9841270e-04f);
    ps = fmaf(z, ps, 8.3333333e-03f);
    ps = fmaf(z, ps, -1.6666667e-01f);
    const float s = fmaf(r * z, ps, r);
    float pc = fmaf(z, 2.4801587e-05f, -1.3888889e-03f);
    pc = fmaf(z, pc, 4.1666667e-02f);
    pc = fmaf(z, pc, -0.5f);
    const float c = fmaf(z, pc, 1.0f);
    float cs = (q & 1) ? -s : c;
    float sn = (q & 1) ? c : s;
    if (q & 2) { cs = -cs; sn = -sn; }
    return make_float2(cs, sn);
  }
  double s, c;
  sincos(phi, &s, &c);
  return make_float2((float)c, (float)s);
}

template <class C> struct phase_of;
template <> struct phase_of<float2> {
  static __device__ __forceinline__ float2 eval(double phi) { return unit_phase_f32(phi); }
};
template <> struct phase_of<double2> {
  static __device__ __forceinline__ double2 eval(double phi) { return unit_phase(phi); }
};

// ---------------------------------------------------------------------------
// in-register DFT butterflies, X_t = sum_s x_s e^{SIGN 2 pi i s t / R}
// ---------------------------------------------------------------------------
template <int SIGN, class C> __device__ __forceinline__ void dft2(C& a, C& b) {
  const C t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int SIGN, class C> __device__ __forceinline__ void dft4(C& x0, C& x1, C& x2, C& x3) {
  const C t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const C t2 = cadd(x1, x3), t3 = rot<SIGN>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <class C> struct rconst;
template <> struct rconst<float2> {
  using R = float;
  static constexpr float SQRT1_2 = 0.70710678118654752440f;
  static constexpr float C16 = 0.92387953251128675613f;  // cos(pi/8)
  static constexpr float S16 = 0.38268343236508977173f;  // sin(pi/8)
};
template <> struct rconst<double2> {
  using R = double;
  static constexpr double SQRT1_2 = 0.70710678118654752440;
  static constexpr double C16 = 0.92387953251128675613;
  static constexpr double S16 = 0.38268343236508977173;
};

// multiply by w8^k = e^{SIGN 2 pi i k / 8}
template <int SIGN, int K, class C> __device__ __forceinline__ C w8(C a) {
  using RC = rconst<C>;
  constexpr int k = K & 7;
  if (k == 0) return a;
  if (k == 2) return rot<SIGN>(a);
  if (k == 4) return mk(-a.x, -a.y);
  if (k == 6) return rot<-SIGN>(a);
  // odd k: (cos, SIGN*sin) of 2pi k/8 with |cos|=|sin|=sqrt(1/2)
  const auto h = RC::SQRT1_2;
  const int cs = (k == 1 || k == 7) ? 1 : -1;
  const int sn = ((k == 1 || k == 3) ? 1 : -1) * SIGN;
  // (a.x + i a.y)(cs*h + i sn*h)
  return mk((cs * a.x - sn * a.y) * h, (cs * a.y + sn * a.x) * h);
}

template <int SIGN, class C> __device__ __forceinline__ void dft8(C* v) {
  // radix-2 split: even / odd halves then combine with w8^k
  C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<SIGN>(e0, e1, e2, e3);
  dft4<SIGN>(o0, o1, o2, o3);
  o1 = w8<SIGN, 1>(o1);
  o2 = w8<SIGN, 2>(o2);
  o3 = w8<SIGN, 3>(o3);
  v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

// multiply by w16^k = e^{SIGN 2 pi i k / 16}, k odd in {1,3,5,7}
template <int SIGN, int K, class C> __device__ __forceinline__ C w16odd(C a) {
  using RC = rconst<C>;
  // cos/sin of 2 pi k / 16 for k = 1,3,5,7
  constexpr int k = K;
  const auto c = (k == 1) ? RC::C16 : (k == 3) ? RC::S16 : (k == 5) ? -RC::S16 : -RC::C16;
  const auto s0 = (k == 1) ? RC::S16 : (k == 3) ? RC::C16 : (k == 5) ? RC::C16 : RC::S16;
  const auto s = SIGN * s0;
  return mk(a.x * c - a.y * s, a.x * s + a.y * c);
}

template <int SIGN, class C> __device__ __forceinline__ void dft16(C* v) {
  C e[8], o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
  dft8<SIGN>(e);
  dft8<SIGN>(o);
  o[1] = w16odd<SIGN, 1>(o[1]);
  o[2] = w8<SIGN, 1>(o[2]);
  o[3] = w16odd<SIGN, 3>(o[3]);
  o[4] = w8<SIGN, 2>(o[4]);
  o[5] = w16odd<SIGN, 5>(o[5]);
  o[6] = w8<SIGN, 3>(o[6]);
  o[7] = w16odd<SIGN, 7>(o[7]);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = cadd(e[i], o[i]);
    v[i + 8] = csub(e[i], o[i]);
  }
}

template <int R, int SIGN, class C> __device__ __forceinline__ void dft_r(C* v) {
  if constexpr (R == 2) dft2<SIGN>(v[0], v[1]);
  else if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<SIGN>(v);
  else if constexpr (R == 16) dft16<SIGN>(v);
}

}  // namespace xftb
