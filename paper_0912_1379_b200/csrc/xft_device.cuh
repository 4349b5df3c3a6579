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

// ---- packed fp32x2 (sm_100 FADD2/FMUL2/FFMA2): one instruction per complex add ----
// The operand swaps/broadcasts/single-lane negations below are folded by ptxas
// into the .F32x2.LO_HI / .F32 / .NP operand modifiers of the packed ops.
__device__ __forceinline__ unsigned long long pk2(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 p_add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 p_sub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 p_mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(d);
}
__device__ __forceinline__ float2 p_fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(d);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return p_add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return p_sub(a, b); }
// (a.x + i a.y)(b.x + i b.y) = b.x (a.x, a.y) + b.y (-a.y, a.x): FMUL2 + FFMA2
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return p_fma(make_float2(-a.y, a.x), make_float2(b.y, b.y), p_mul(a, make_float2(b.x, b.x)));
}

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

// x + a w (complex) as FMA chains, and 2 x - t
__device__ __forceinline__ double2 cfma(double2 a, double2 w, double2 x) {
  return make_double2(fma(a.x, w.x, fma(-a.y, w.y, x.x)), fma(a.x, w.y, fma(a.y, w.x, x.y)));
}
__device__ __forceinline__ float2 cfma(float2 a, float2 w, float2 x) {  // FFMA2 x 2
  return p_fma(make_float2(-a.y, a.x), make_float2(w.y, w.y), p_fma(a, make_float2(w.x, w.x), x));
}
__device__ __forceinline__ double2 ctwice_minus(double2 x, double2 t) {
  return make_double2(fma(2.0, x.x, -t.x), fma(2.0, x.y, -t.y));
}
__device__ __forceinline__ float2 ctwice_minus(float2 x, float2 t) {
  return p_fma(x, make_float2(2.0f, 2.0f), make_float2(-t.x, -t.y));
}

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

template <int SIGN, int K> __device__ __forceinline__ float2 w8(float2 a) {
  constexpr int k = K & 7;
  if constexpr (k == 0) return a;
  else if constexpr (k == 2) return rot<SIGN>(a);
  else if constexpr (k == 4) return make_float2(-a.x, -a.y);
  else if constexpr (k == 6) return rot<-SIGN>(a);
  else {
    const float h = 0.70710678118654752440f;
    const float cs = (k == 1 || k == 7) ? h : -h;
    const float sn = ((k == 1 || k == 3) ? h : -h) * SIGN;
    return p_fma(make_float2(-a.y, a.x), make_float2(sn, sn), p_mul(a, make_float2(cs, cs)));
  }
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

template <int SIGN, int K> __device__ __forceinline__ float2 w16odd(float2 a) {
  constexpr int k = K;
  const float c = (k == 1) ? 0.92387953251128675613f : (k == 3) ? 0.38268343236508977173f
                : (k == 5) ? -0.38268343236508977173f : -0.92387953251128675613f;
  const float s0 = (k == 1) ? 0.38268343236508977173f : (k == 3) ? 0.92387953251128675613f
                 : (k == 5) ? 0.92387953251128675613f : 0.38268343236508977173f;
  const float s = SIGN * s0;
  return p_fma(make_float2(-a.y, a.x), make_float2(s, s), p_mul(a, make_float2(c, c)));
}

#ifndef XFT_DFT16_44
#define XFT_DFT16_44 1  // radix-16 butterfly as 4 x 4 (160 real ops) instead of 2 x 8 (168)
#endif
// 16-point DFT as 4 x 4: four 4-point DFTs down the columns n2 of x[4 n1 + n2],
// the internal twiddles w16^(n2 k1), four 4-point DFTs along k1
template <int SIGN, class C> __device__ __forceinline__ void dft16_44(C* v) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<SIGN>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // v[4 k1 + n2] now holds y[n2][k1]
  v[4 + 1] = w16odd<SIGN, 1>(v[4 + 1]);    // k1=1 n2=1: w^1
  v[4 + 2] = w8<SIGN, 1>(v[4 + 2]);        // k1=1 n2=2: w^2
  v[4 + 3] = w16odd<SIGN, 3>(v[4 + 3]);    // k1=1 n2=3: w^3
  v[8 + 1] = w8<SIGN, 1>(v[8 + 1]);        // k1=2 n2=1: w^2
  v[8 + 2] = w8<SIGN, 2>(v[8 + 2]);        // k1=2 n2=2: w^4
  v[8 + 3] = w8<SIGN, 3>(v[8 + 3]);        // k1=2 n2=3: w^6
  v[12 + 1] = w16odd<SIGN, 3>(v[12 + 1]);  // k1=3 n2=1: w^3
  v[12 + 2] = w8<SIGN, 3>(v[12 + 2]);      // k1=3 n2=2: w^6
  {
    const C t = w16odd<SIGN, 1>(v[12 + 3]);  // k1=3 n2=3: w^9 = -w^1
    v[12 + 3] = mk(-t.x, -t.y);
  }
  C r[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    C a = v[4 * k1], b = v[4 * k1 + 1], c = v[4 * k1 + 2], d = v[4 * k1 + 3];
    dft4<SIGN>(a, b, c, d);
    r[k1] = a; r[k1 + 4] = b; r[k1 + 8] = c; r[k1 + 12] = d;  // X[k1 + 4 k2]
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = r[i];
}

// the second half of dft16_44: internal twiddles and the 4-point DFTs along k1
// (for callers that ran the column stage themselves)
template <int SIGN, class C> __device__ __forceinline__ void dft16_44_rows(C* v) {
  v[4 + 1] = w16odd<SIGN, 1>(v[4 + 1]);
  v[4 + 2] = w8<SIGN, 1>(v[4 + 2]);
  v[4 + 3] = w16odd<SIGN, 3>(v[4 + 3]);
  v[8 + 1] = w8<SIGN, 1>(v[8 + 1]);
  v[8 + 2] = w8<SIGN, 2>(v[8 + 2]);
  v[8 + 3] = w8<SIGN, 3>(v[8 + 3]);
  v[12 + 1] = w16odd<SIGN, 3>(v[12 + 1]);
  v[12 + 2] = w8<SIGN, 3>(v[12 + 2]);
  {
    const C t = w16odd<SIGN, 1>(v[12 + 3]);
    v[12 + 3] = mk(-t.x, -t.y);
  }
  C r[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    C a = v[4 * k1], b = v[4 * k1 + 1], c = v[4 * k1 + 2], d = v[4 * k1 + 3];
    dft4<SIGN>(a, b, c, d);
    r[k1] = a; r[k1 + 4] = b; r[k1 + 8] = c; r[k1 + 12] = d;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = r[i];
}

template <int SIGN, class C> __device__ __forceinline__ void dft16(C* v) {
  if constexpr (XFT_DFT16_44) {
    dft16_44<SIGN>(v);
  } else {
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
}

// w32^k (k = 1..15), cos and sin of 2 pi k / 32
static __constant__ const double kW32c[16] = {1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
                                       0.7071067811865476, 0.5555702330196023, 0.38268343236508984,
                                       0.19509032201612833, 0.0, -0.19509032201612833, -0.38268343236508984,
                                       -0.5555702330196023, -0.7071067811865476, -0.8314696123025452,
                                       -0.9238795325112867, -0.9807852804032304};
static __constant__ const double kW32s[16] = {0.0, 0.19509032201612825, 0.3826834323650898, 0.5555702330196022,
                                       0.7071067811865475, 0.8314696123025452, 0.9238795325112867,
                                       0.9807852804032304, 1.0, 0.9807852804032304, 0.9238795325112867,
                                       0.8314696123025452, 0.7071067811865475, 0.5555702330196022,
                                       0.3826834323650898, 0.19509032201612825};
template <int SIGN, int K> __device__ __forceinline__ double2 w32(double2 a) {
  const double c = kW32c[K], s = SIGN * kW32s[K];
  return make_double2(a.x * c - a.y * s, a.x * s + a.y * c);
}
template <int SIGN, int K> __device__ __forceinline__ float2 w32(float2 a) {
  const float c = (float)kW32c[K], s = (float)(SIGN * kW32s[K]);
  return p_fma(make_float2(-a.y, a.x), make_float2(s, s), p_mul(a, make_float2(c, c)));
}

template <int SIGN, class C> __device__ __forceinline__ void dft32(C* v) {
  C e[16], o[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { e[i] = v[2 * i]; o[i] = v[2 * i + 1]; }
  dft16<SIGN>(e);
  dft16<SIGN>(o);
  o[1] = w32<SIGN, 1>(o[1]);   o[2] = w32<SIGN, 2>(o[2]);   o[3] = w32<SIGN, 3>(o[3]);
  o[4] = w32<SIGN, 4>(o[4]);   o[5] = w32<SIGN, 5>(o[5]);   o[6] = w32<SIGN, 6>(o[6]);
  o[7] = w32<SIGN, 7>(o[7]);   o[8] = rot<SIGN>(o[8]);      o[9] = w32<SIGN, 9>(o[9]);
  o[10] = w32<SIGN, 10>(o[10]); o[11] = w32<SIGN, 11>(o[11]); o[12] = w32<SIGN, 12>(o[12]);
  o[13] = w32<SIGN, 13>(o[13]); o[14] = w32<SIGN, 14>(o[14]); o[15] = w32<SIGN, 15>(o[15]);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = cadd(e[i], o[i]);
    v[i + 16] = csub(e[i], o[i]);
  }
}

template <int R, int SIGN, class C> __device__ __forceinline__ void dft_r(C* v) {
  if constexpr (R == 2) dft2<SIGN>(v[0], v[1]);
  else if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<SIGN>(v);
  else if constexpr (R == 16) dft16<SIGN>(v);
  else if constexpr (R == 32) dft32<SIGN>(v);
}

}  // namespace xftb
