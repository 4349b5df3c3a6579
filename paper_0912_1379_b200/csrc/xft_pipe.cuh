// K1 (production path): persistent, TMA-pipelined batched chirp-DFT-chirp.
//
// Each CTA is persistent over "tiles" (ROWS consecutive rows = one contiguous
// HBM span).  A STAGES-deep ring of shared-memory tile buffers is filled by
// 1-D bulk TMA (cp.async.bulk, completion on an mbarrier) STAGES-1 tiles
// ahead of the tile being transformed, so HBM reads stay in flight while the
// SM computes.  The tile buffer doubles as the Stockham exchange buffer
// (XOR-swizzled, bank-conflict free); results leave from registers with
// coalesced streaming stores.  Every sample is read from and written to HBM
// exactly once.
//
// Per-element work (reference: xft/lct.py:204-207, xft/kernel.py:45-113):
//   pre  : f_k * p_k * e^{i phi_k}                       (a != 0)
//   post : S_j * C(n) p_j e^{i psi_j} / sqrt(2 pi i b)   (d != 0)
// with p_k = (-1)^k e^{-i pi k/n} folded into the chirp argument.
//  * c128: phi_k = fl(fl(0.5a/b) fl(x_k^2)), x_k = fl((2k-n+1) half) is formed
//    exactly as the reference forms it (bit-identical fp64 argument);
//    e^{i(phi+delta)} = T[q mod 256] e^{i r}, q = rint((phi+delta)/(2pi/256)),
//    r by a two-constant FMA Cody-Waite step (|r| <= pi/256), e^{ir} by a
//    degree-6/7 Taylor polynomial (|err| < 1e-17), T a 256-entry table in
//    shared memory (XFT_C128_TABL; 1024/2048 entries with shorter
//    polynomials measured slower).  The boundary phase's integer table steps
//    ride on q; only a per-thread residual |delta| <= U/2 enters the fp64 math.
//  * c64: the chirp phase in turns, frac(D k'^2 + boundary) with
//    D = (a/2b) half^2 / 2pi, is evaluated exactly in 64-bit fixed point
//    (wraps mod 1 turn).  Along a thread's elements the phase is a quadratic
//    in s, so it is walked with integer adds (TurnWalk), then one LEA.HI +
//    FFMA map the turn fraction to MUFU sin/cos.  No fp64 per element.
// Twiddles come from a pass-major table (entry (t-1)*NS + k of pass p holds
// w_{NS*E}^{t k}) so every warp's twiddle loads are coalesced.
#pragma once
#include <type_traits>

#include "xft_rows.cuh"
#include "xft_tables.h"

#ifndef XFT_NOMEM
#define XFT_NOMEM 0  // tuning only: a CTA re-reads / rewrites its first tile (L2-resident: compute-bound timing)
#endif
// L2 bulk prefetch (cp.async.bulk.prefetch.L2) of the tile this many tiles beyond the TMA ring, issued when a
// tile's transform starts, so the later TMA load is an L2 hit (PipeCfg::L2PF).  Measured per kernel, depth 1
// against off (A/B on one box, outputs bit-identical): c128 n = 4096 116.7 -> 115.6 us, c64 n = 16384 (one CTA
// per SM) 945 -> 900 us, c64 n = 1024 (config 4) 184.0 -> 178.3 us: on.  c64 n = 4096 / 8192 (single-stage CTAs
// at 4 / 2 per SM) +1.3-1.5%, c128 n = 2048 +2%, c128 n = 8192 and the short-row rings: no change: off.
// Depths 2 and 3 are slower everywhere (c128 n = 4096: 117.0 / 122.4 us).
#ifndef XFT_L2PF_EARLY
#define XFT_L2PF_EARLY 0  // 1: issue the prefetch before waiting for the current tile instead of after
#endif
#ifndef XFT_L2PF
#define XFT_L2PF -1  // >= 0: force this depth on every row kernel (tuning)
#endif
#ifndef XFT_C128_TABCOPIES
#define XFT_C128_TABCOPIES 1
#endif
#include "xft_tma.cuh"

#ifndef XFT_NOTW
#define XFT_NOTW 0  // tuning only: 1 = skip the inter-pass twiddles
#endif
#ifndef XFT_FUSE_TW
#define XFT_FUSE_TW 1  // c128: inter-pass twiddles fused into the first butterfly stage (FMA chains)
#endif
#ifndef XFT_FUSE_TW64
#define XFT_FUSE_TW64 1  // the same for c64 (packed FP32x2 FMA chains)
#endif
#ifndef XFT_TWBASE
#define XFT_TWBASE 1  // c128 row kernels: per-thread base twiddles held across rows (see pipe_pass)
#endif
#ifndef XFT_TWLOAD1
#define XFT_TWLOAD1 1  // c128: w^8 = (w^4)^2 too, one table load per butterfly (A/B: -0.5% n=4096, -1.5% n=8192)
#endif
#ifndef XFT_TWLOAD4
#define XFT_TWLOAD4 0  // 1: w^2 and w^4 loaded too (two loads for two multiplies)
#endif
#ifndef XFT_TWGEN
#define XFT_TWGEN 1  // LCT-mode inter-pass twiddles generated from two table entries per butterfly (0: all loaded)
#endif
#ifndef XFT_COEF_PREFETCH
#define XFT_COEF_PREFETCH 1  // prefetch the first coefficient chunk's parameter rows at kernel entry
#endif
#ifndef XFT_TW_PREFETCH
#define XFT_TW_PREFETCH 0  // (A/B: slower, off) prefetch this thread's first-row twiddle entries at kernel entry
#endif
#ifndef XFT_C128_CH
#define XFT_C128_CH 32  // coefficient chunk (rows) of the single-row c128 CTAs
#endif
#ifndef XFT_MIRROR
#define XFT_MIRROR 1  // mirror lane map + shared rounding corrections (see PipeCfg::MIRROR)
#endif
#ifndef XFT_C128_EARLY
#define XFT_C128_EARLY 0  // c128 single-stage CTAs: issue the next tile's load after the last exchange read
#endif
#ifndef XFT_SPLIT
#define XFT_SPLIT 1  // split next-row prefetch for single-row CTAs (see PipeCfg::SPLIT)
#endif
#ifndef XFT_SPLIT2
#define XFT_SPLIT2 0  // 1: also at two single-row CTAs per SM (c128 n = 4096, the spare ~36 KB per CTA): A/B 121.0 vs 119.2 us, off
#endif

// Split "buffer read" barriers (PipeCfg::XBAR).  A/B on one box (outputs bit-identical): the 512-thread,
// one-CTA-per-SM c64 row kernel (n = 16384) 1016 -> 951 us; with 2 or 4 CTAs per SM, where the other CTAs already
// fill a CTA-wide rendezvous, it LOSES: config 2 c64 52.8 -> 58.3 us, c128 117.4 -> 126.5 us (n = 8192: 296 ->
// 335 us), config 4 184.9 -> 188.2 us.  Hence: c64 at one CTA per SM only.
// Two follow-ups, both measured slower and removed: replacing only the row's last rendezvous (thread 0 waits on an
// mbarrier phase, the other warps go on) at 2-4 CTAs per SM -- c64 52.7 -> 57.1 us, c128 115.6 -> 120.8 us; and
// letting the warp that arrives last hand the stage back to the TMA instead of thread 0 waiting for the phase --
// n = 16384: 900 -> 948 us (the slowest warp gets the extra work).
#ifndef XFT_XBAR64
#define XFT_XBAR64 1      // c64 row kernels at one CTA per SM
#endif
#ifndef XFT_XBAR64_ALL
#define XFT_XBAR64_ALL 0  // every c64 row kernel
#endif
#ifndef XFT_XBAR128
#define XFT_XBAR128 0     // c128 row kernels
#endif

#ifndef XFT_SPLIT4
#define XFT_SPLIT4 0  // 1: the split next-row prefetch for c64 single-row CTAs at 2 and 4 CTAs per SM too (n = 8192, 4096)
#endif

#ifndef XFT_SKELETON
#define XFT_SKELETON 0  // tuning only: 1 = exchanges without math, 2 = pure copy
#endif

namespace xftb {

#define XFT_PI 3.141592653589793116
#define XFT_INV_2PI 0.15915494309189534561

// fp64 constants live in the constant bank so DFMA/DMUL take them as c[] operands.
// U = 2 pi / C128_TABN (the table step) in two parts, 1/U, and the Taylor
// coefficients of sin / cos on |r| <= U/2 (the terms the table size needs).
static __constant__ double kC128[8] = {
    6.283185307179586 / C128_TABN,                          // 0 U_HI
    2.4492935982947064e-16 / C128_TABN,                     // 1 U_LO (2 pi - fl(2 pi)) / TABN
    C128_TABN * 0.15915494309189535,                        // 2 1/U
    -1.6666666666666667e-01,                                // 3 sin: -1/6
    8.3333333333333333e-03,                                 // 4 sin:  1/120
    -0.5,                                                   // 5 cos: -1/2
    4.1666666666666667e-02,                                 // 6 cos:  1/24
    -1.3888888888888889e-03,                                // 7 cos: -1/720
};
// 32 pi = 4096 U in three parts, and its inverse: pre-reduction for huge phases
static __constant__ double kC128Big[4] = {100.53096491487338, 3.91886975727153e-15, -9.583263391098687e-32,
                                   0.009947183943243459};

// s * pi / 16, s = 0..15: the boundary-phase step between a thread's registers

// ---------------------------------------------------------------------------
// per-row coefficients
// ---------------------------------------------------------------------------
// Computed once per row inside the row kernel, by all threads of a CTA for
// the next CH tiles at a time, into shared memory.
struct __align__(16) Coef64 {
  unsigned long long dq_in, dq_out;  // Q0.64 turns per unit k'^2 (chirp rates)
  uint32_t gq;                       // top 32 bits of arg G in turns
  float gabs;                        // |G|
  float2 g;                          // G (used when d == 0)
  int pre, post;
  int pad[2];
};

struct __align__(16) Coef128 {
  double cin, cout, s4;  // fl(0.5a/b), fl(0.5d/b), fl(4b/pi)
  double gabs, gf;       // |G|, small part of arg G (|gf| <= U/2)
  double2 g;             // G (used when d == 0)
  // walk path: the chirp phase without the reference's roundings, in turns per
  // m^2 (m = 2k - n + 1), as double-doubles: cin half^2 / 2pi, cout s4^2 half^2 / 2pi
  double din_hi, din_lo, dout_hi, dout_lo;
  double2 sin_, sout;    // second-difference phasors e^{2 pi i D (2 TR)^2 2}
  double gturn;          // arg G in turns (exact)
  int gi;                // arg G / U rounded (table units)
  int pre, post;         // 0 none, 1 walk, 2 walk + rounding correction, 3 table, 4 table + pre-reduction
  int pad;
};
static_assert(sizeof(Coef64) % 16 == 0 && sizeof(Coef128) % 16 == 0, "bulk-copy granularity");

template <class C> struct CoefOf;
template <> struct CoefOf<float2> { using T = Coef64; };
template <> struct CoefOf<double2> { using T = Coef128; };

struct RowConst {  // per-launch constants (host computed)
  double half;      // (pi / sqrt(2n)) / 2
  double cnabs;     // |C(n)| = pi / sqrt(2n)
  long long cnred;  // (n-1)^2 mod 4n   (arg C(n) = -pi red / (2n))
  int log2n;
  int flags;
  unsigned long long* bad = nullptr;  // non-null: atomicMin'd with every row holding a non-finite input
};

// 0 iff some component of x is Inf/NaN (all-ones exponent), two integer ops per component
__device__ __forceinline__ unsigned nonfinite_key(double2 x) {
  const unsigned e = 0x7ff00000u;
  return min(~(unsigned)__double2hiint(x.x) & e, ~(unsigned)__double2hiint(x.y) & e);
}
__device__ __forceinline__ unsigned nonfinite_key(float2 x) {
  const unsigned e = 0x7f800000u;
  return min(~__float_as_uint(x.x) & e, ~__float_as_uint(x.y) & e);
}

__device__ __forceinline__ unsigned long long frac_q64(double v) {
  double f = v - floor(v);
  if (!(f >= 0.0 && f < 1.0)) f = 0.0;                 // non-finite guard
  return __double2ull_rz(f * 18446744073709551616.0);  // * 2^64
}

__device__ __forceinline__ void row_params(const double* p, const Abcd& uni, double& a, double& b, double& d) {
  if (p) { a = p[0]; b = p[1]; d = p[3]; } else { a = uni.a; b = uni.b; d = uni.d; }
}

__device__ __forceinline__ double g_abs(double b, const RowConst& k) {
  double g = k.cnabs / sqrt(6.283185307179586232 * fabs(b));
  if (k.flags & FLAG_BARE_FOURIER) g *= 2.506628274631000502;  // |sqrt(2 pi i)|
  return g;
}

__device__ __forceinline__ void make_coef(Coef64& c, const double* p, const Abcd& uni, const RowConst& k, int,
                                          const double2*) {
  double a, b, d;
  row_params(p, uni, a, b, d);
  const double cin = __ddiv_rn(0.5 * a, b), cout = __ddiv_rn(0.5 * d, b), s4 = __ddiv_rn(4.0 * b, XFT_PI);
  const double h2 = k.half * k.half;
  c.dq_in = frac_q64(cin * h2 * XFT_INV_2PI);
  c.dq_out = frac_q64(cout * s4 * s4 * h2 * XFT_INV_2PI);
  // arg G in turns (exact): -red/(4n) - sgn(b)/8 [+ 1/8 for xft_fourier]
  unsigned long long gq = 0ull - ((unsigned long long)k.cnred << (62 - k.log2n));
  gq += (b > 0.0) ? (0ull - (1ull << 61)) : (1ull << 61);
  if (k.flags & FLAG_BARE_FOURIER) gq += (1ull << 61);
  c.gq = (uint32_t)(gq >> 32);  // the low word is zero for n <= 2^30
  const double gabs = g_abs(b, k);
  c.gabs = (float)gabs;
  double s, co;
  sincospi((double)(long long)gq * 1.0842021724855044e-19, &s, &co);  // 2 * gq / 2^64
  c.g = make_float2((float)(gabs * co), (float)(gabs * s));
  c.pre = (a != 0.0);
  c.post = (d != 0.0);
}

// ---- c128 chirp walk helpers -------------------------------------------------
#ifndef XFT_C128_WALK
#define XFT_C128_WALK 1  // 0: every c128 chirp through the per-element table path (modes 3/4)
#endif
#ifndef XFT_WALK_MIN_LOG2N
#define XFT_WALK_MIN_LOG2N 11  // c128 rows shorter than 2^11 use the per-element table path (accuracy)
#endif
#ifndef XFT_WALK_SMOOTH_BELOW
#define XFT_WALK_SMOOTH_BELOW 8192.0  // rows with max |phase| below this skip the rounding corrections (max row
                                      // error 4.4e-13 in [4096, 8192) vs 1.2e-13 corrected; c128 119.3 -> 116.9 us)
#endif
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_norm(double s, double e) {  // fast two-sum, |s| >= |e|
  const double h = __dadd_rn(s, e);
  return DD{h, __dsub_rn(e, __dsub_rn(h, s))};
}
__device__ __forceinline__ DD dd_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return DD{p, fma(a, b, -p)};
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const DD p = dd_prod(a.hi, b.hi);
  return dd_norm(p.hi, fma(a.hi, b.lo, fma(a.lo, b.hi, p.lo)));
}
__device__ __forceinline__ DD dd_mul(DD a, double b) {
  const DD p = dd_prod(a.hi, b);
  return dd_norm(p.hi, fma(a.lo, b, p.lo));
}

// frac(D M) for a double-double D and an exact integer-valued M (|M| < 2^53):
// f = a - rint(a) exactly (|f| <= 1/2) and the low part lo, D M = f + lo (mod 1)
__device__ __forceinline__ void frac_dd(double dhi, double dlo, double M, double& f, double& lo) {
  const double a = __dmul_rn(dhi, M);
  lo = fma(dlo, M, fma(dhi, M, -a));
  f = __dsub_rn(a, rint(a));
}

// e^{2 pi i (f + lin + lo)} from the c128 table: f exact with |f| <= 1/2, lin a
// short multiple of 2^-16 (|lin| <= 2), lo small.  The table quantum q is taken
// out of f + lin exactly (Sterbenz) before the low part is added, so the
// argument is accurate to ~1e-18 turn whatever the magnitude of the phase was.
__device__ __forceinline__ double2 turn_phasor(double f, double lin, double lo, const double2* __restrict__ tab) {
  const double t = fma(__dadd_rn(f, lin), (double)C128_TABN, 6755399441055744.0);
  const double qd = __dsub_rn(t, 6755399441055744.0);
  const int q = __double2loint(t);
  const double g = __dadd_rn(__dadd_rn(f, fma(-qd, 1.0 / C128_TABN, lin)), lo);
  const double r = __dmul_rn(g, 6.283185307179586);
  const double z = r * r;
  const double sn = fma(r * z, fma(z, kC128[4], kC128[3]), r);
  const double cs = fma(z, fma(z, fma(z, kC128[7], kC128[6]), kC128[5]), 1.0);
  const double2 w = tab[q & (C128_TABN - 1)];
  return make_double2(w.x * cs - w.y * sn, w.x * sn + w.y * cs);
}

__device__ __forceinline__ void make_coef(Coef128& c, const double* p, const Abcd& uni, const RowConst& k, int tr,
                                          const double2* __restrict__ tab) {
  double a, b, d;
  row_params(p, uni, a, b, d);
  c.cin = __ddiv_rn(0.5 * a, b);      // (0.5j * a / b).imag     xft/kernel.py:102
  c.cout = __ddiv_rn(0.5 * d, b);     // (0.5j * d / b).imag     xft/kernel.py:113
  c.s4 = __ddiv_rn(4.0 * b, XFT_PI);  // 4.0 * b / np.pi        xft/lct.py:196
  // arg G / U, U = 2pi/T: (T/256) (-64 red / n - 32 sgn(b) [+ 32])   (exact in fp64)
  constexpr double Q = C128_TABN / 256.0;
  double v = -64.0 * Q * (double)k.cnred / (double)(1ll << k.log2n) + ((b > 0.0) ? -32.0 * Q : 32.0 * Q);
  if (k.flags & FLAG_BARE_FOURIER) v += 32.0 * Q;
  const double vi = rint(v);
  c.gi = (int)vi;
  c.gf = (v - vi) * kC128[0];
  c.gturn = v * (1.0 / C128_TABN);
  c.gabs = g_abs(b, k);
  // G = |G| e^{2 pi i v / T}: the table path (v / T is exact, |v / T| < 1/2), no libm sincospi
  const double2 eg = turn_phasor(v * (1.0 / C128_TABN), 0.0, 0.0, tab);
  c.g = make_double2(c.gabs * eg.x, c.gabs * eg.y);
  // smooth chirp rates (turns per m^2) and the walk's second-difference phasors
  const DD h2i = dd_mul(dd_prod(k.half, k.half), DD{0.15915494309189535, -9.839338337591243e-18});
  const DD din = dd_mul(h2i, c.cin);
  const DD dout = dd_mul(dd_mul(dd_prod(c.s4, c.s4), c.cout), h2i);
  c.din_hi = din.hi; c.din_lo = din.lo; c.dout_hi = dout.hi; c.dout_lo = dout.lo;
  const double m2 = 8.0 * (double)tr * (double)tr;  // (2 tr)^2 * 2, a power of two: exact scaling
  double f, lo;
  frac_dd(din.hi, din.lo, m2, f, lo);
  c.sin_ = turn_phasor(f, 0.0, lo, tab);
  frac_dd(dout.hi, dout.lo, m2, f, lo);
  c.sout = turn_phasor(f, 0.0, lo, tab);
  // largest |phase| on the row = |coef| x_max^2.  Below 2^11 rad the reference's
  // argument roundings stay under 1.1e-13 rms per row and the smooth walk is
  // used as is; below 2^24 the rounding error is re-added per element to first
  // order (|eps| < 1e-8); the table path is exact for |phi| < ~1e13, beyond
  // 1e12 the row is pre-reduced.
  const double x2 = (double)((1ll << k.log2n) - 1) * k.half;
  const double pmax_in = fabs(c.cin) * x2 * x2;
  const double y2 = fabs(c.s4) * x2;
  const double pmax_out = fabs(c.cout) * y2 * y2;
  // short rows (n < 2^XFT_WALK_MIN_LOG2N: latency-bound, never FP64-bound) take the
  // exact per-element table path: the walk's accumulated rounding (~15 products)
  // would double the reference's own error at n = 512 (its frozen figure-1
  // threshold, xft/calibration.py:17-22: 2.84e-15 walked vs 1.35e-15 tabled)
  const bool walk = XFT_C128_WALK && k.log2n >= XFT_WALK_MIN_LOG2N;
  auto mode_of = [walk](double pm) {
    if (walk && pm < XFT_WALK_SMOOTH_BELOW) return 1;
    if (walk && pm < 16777216.0) return 2;
    return pm < 1e12 ? 3 : 4;
  };
  c.pre = (a != 0.0) ? mode_of(pmax_in) : 0;
  c.post = (d != 0.0) ? mode_of(pmax_out) : 0;
#ifdef XFT_NOCHIRP  // tuning only: time the kernel with the chirps replaced by the p_k table path
  c.pre = (XFT_NOCHIRP & 1) ? 0 : c.pre;
  c.post = (XFT_NOCHIRP & 2) ? 0 : c.post;
#endif
}

// ---------------------------------------------------------------------------
// unit phasors
// ---------------------------------------------------------------------------
// e^{i (phi + add)} e^{i U qoff} in fp64 via the table tab[m] = e^{i U m}, U = 2 pi / C128_TABN.
// phi: exact fp64 chirp argument, |phi| < 1e12 (larger: prereduce first); |add| < 2 pi.
__device__ __forceinline__ double2 unit_phase_tab(double phi, double add, int qoff, const double2* __restrict__ tab) {
  const double t = fma(phi + add, kC128[2], 6755399441055744.0);
  const double qd = t - 6755399441055744.0;
  const int q = __double2loint(t) + qoff;
  double r = fma(-qd, kC128[0], phi);
  r = r + add;
  r = fma(-qd, kC128[1], r);
  const double z = r * r;
  // |r| <= pi / TABN: 256 -> sin to r^5, cos to r^6; 1024 -> cos to r^4; 2048 -> sin to r^3
  const double sn = C128_TABN >= 2048 ? fma(r * z, kC128[3], r) : fma(r * z, fma(z, kC128[4], kC128[3]), r);
  const double cs = C128_TABN >= 1024 ? fma(z, fma(z, kC128[6], kC128[5]), 1.0)
                                      : fma(z, fma(z, fma(z, kC128[7], kC128[6]), kC128[5]), 1.0);
  // XFT_C128_TABCOPIES = 8: lane l reads interleaved copy (l & 7), so the 8 lanes
  // of a quarter-warp always hit 8 different 16-byte bank groups
  const double2 w = XFT_C128_TABCOPIES == 8 ? tab[((q & (C128_TABN - 1)) << 3) | (threadIdx.x & 7)]
                                            : tab[q & (C128_TABN - 1)];
  return make_double2(w.x * cs - w.y * sn, w.x * sn + w.y * cs);
}

// hide a value from the optimiser (stops it from re-deriving per-element
// integer->fp64 conversions or hoisting per-element constants into registers)
__device__ __forceinline__ double opaque(double x) {
  double y;
  asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// phi - m * 32pi (exact multiple of 4096 table units, so the table index is
// unchanged): keeps the table reduction accurate for |phi| up to ~2e17
__device__ __forceinline__ double prereduce(double phi) {
  const double t = fma(phi, kC128Big[3], 6755399441055744.0);
  const double q = t - 6755399441055744.0;
  double r = fma(-q, kC128Big[0], phi);
  r = fma(-q, kC128Big[1], r);
  return fma(-q, kC128Big[2], r);
}

// g e^{2 pi i t / 2^32} in fp32 through the SFU (MUFU.SIN/COS): t -> signed
// turns -> radians in [-pi, pi); |err| < 2e-6 (well inside the c64 budget).
__device__ __forceinline__ float2 unit_turns_sfu(uint32_t t, float g) {
  const int fm = ((int)t + 512) >> 10;                                  // |fm| <= 2^21
  const float F = __int_as_float(0x4B400000 + fm) - 12582912.0f;       // = fm exactly
  const float th = F * 1.4980281e-06f;                                  // 2 pi / 2^22
  float s, c;
  __sincosf(th, &s, &c);
  return make_float2(c * g, s * g);
}

// e^{2 pi i t / 2^32} for a walk value t (TurnWalk below: the +512 rounding
// and the -326 magic-constant correction are already folded in):
// one LEA.HI, one FFMA, the SFU pair.  (12582912 + fm) c - K = fm c + 4.768e-7,
// and 4.768e-7 rad = 325.95 units of 2^-32 turn.
__device__ __forceinline__ float2 walk_phasor(uint32_t t) {
  const float F = __int_as_float(0x4B400000 + ((int)t >> 10));  // 12582912 + fm, exact
  const float th = fmaf(F, 1.4980281548560015e-06f, -18.84955596923828f);
  float s, c;
  __sincosf(th, &s, &c);
  return make_float2(c, s);
}

// The c64 chirp phase of element s of a thread, in 2^-32 turns:
//   t(s) = top32( dq * off_s^2 + lin0 - s * lstep )   (mod 2^64),  off_s = off0 + s * S2
// is a quadratic in s: t(s+1) = t(s) + D(s), D(s+1) = D(s) + 2 dq S2^2, with D
// carried in 64 bits (exact) and t in 32 (one dropped carry per step at most,
// < 4e-9 turn over a row).  Replaces one 64x32 multiply per element with adds.
struct TurnWalk {
  uint32_t t;
  unsigned long long d, dd;
  __device__ __forceinline__ TurnWalk(unsigned long long dq, int off0, int S2, unsigned long long lin0,
                                      unsigned long long lstep) {
    const unsigned long long o0 = (unsigned long long)((long long)off0 * off0);
    const unsigned long long b = (unsigned long long)(2ll * off0 * S2);
    const unsigned long long c = (unsigned long long)((long long)S2 * S2);
    const unsigned long long a = dq * o0 + lin0 + ((512ull - 326ull) << 32);
    t = (uint32_t)(a >> 32);
    d = dq * (b + c) - lstep;
    dd = dq * (2 * c);
  }
  __device__ __forceinline__ uint32_t next() {
    const uint32_t r = t;
    t += (uint32_t)(d >> 32);
    d += dd;
    return r;
  }
};

// The same walk with the differences rounded to 32 bits (one add each per
// element): the phase drifts by at most s^2/2 units of 2^-32 turn over s
// steps (<= 1.2e-7 turn at s = 31), far inside the c64 budget.
struct TurnWalk32 {
  uint32_t t, d, dd;
  __device__ __forceinline__ TurnWalk32(unsigned long long dq, int off0, int S2, unsigned long long lin0,
                                        unsigned long long lstep) {
    const TurnWalk w(dq, off0, S2, lin0, lstep);
    t = w.t;
    d = (uint32_t)((w.d + (1ull << 31)) >> 32);
    dd = (uint32_t)((w.dd + (1ull << 31)) >> 32);
  }
  __device__ __forceinline__ uint32_t next() {
    const uint32_t r = t;
    t += d;
    d += dd;
    return r;
  }
};
#ifndef XFT_WALK32
#define XFT_WALK32 1
#endif
using ChirpTurnWalk = std::conditional_t<XFT_WALK32 != 0, TurnWalk32, TurnWalk>;

// ---------------------------------------------------------------------------
// configuration
// ---------------------------------------------------------------------------
template <class C_, int LOG2N_, int E_, int MODE_, int SIGN_, int ROWS_, int STAGES_, int MINB_, int SPLITOK_ = 0,
          int BARTH_ = 0, int XBAR_ = -1>
struct PipeCfg {
  // threads that take part in the exchange barriers: 0 = the whole CTA (__syncthreads), else a named
  // barrier over the first BARTH threads (kernels with extra, non-computing warps)
  static constexpr int BARTH = BARTH_;
  using C = C_;
  using Coef = typename CoefOf<C>::T;
  static constexpr int LOG2N = LOG2N_, N = 1 << LOG2N, E = E_, MODE = MODE_, SIGN = SIGN_;
  static constexpr int ROWS = ROWS_, STAGES = STAGES_;
  static constexpr int TR = N / E;
  static constexpr int THREADS_C = TR * ROWS;
  static constexpr int THREADS = THREADS_C;
  static constexpr int TILE = ROWS * N;
  // exchange-buffer footprint of one row: one pad slot per 16 elements
  // (pad_idx), so every Stockham store/load offset is a compile-time immediate
  // and both sides stay bank-conflict free
  static constexpr int NP = N + N / 16;
  static constexpr int STAGE = ROWS * NP;  // a stage holds ROWS input rows (TMA, contiguous) / exchange rows
  static constexpr int LE = ilog2(E);
  static constexpr int NPASS = (LOG2N + LE - 1) / LE;
  static constexpr int R0 = 1 << (LOG2N - (NPASS - 1) * LE);
  static constexpr bool C128 = sizeof(C) == 16;
  static constexpr size_t TAB_BYTES = C128 ? XFT_C128_TABCOPIES * C128_TABN * sizeof(double2) : 0;
  // One resident single-row CTA per SM (rows of 128 KB) cannot double-buffer
  // its tile, so the spare shared memory becomes a landing region for the first
  // SPLIT samples of the next row, loaded as soon as this row's input has been
  // read (first exchange barrier); the rest of the next row lands in the stage
  // once the last exchange has been read.  SPLIT is a multiple of TR.
  // Two resident CTAs per SM (c128 n = 4096) split the SM's 228 KB: each keeps
  // its half minus the 1 KB per-CTA reservation and its static coefficient chunk.
  static constexpr size_t STATIC_EST =
      size_t(MODE == MODE_LCT ? (C128 ? XFT_C128_CH : 32) : 1) * ROWS * sizeof(Coef) + 8 * STAGES + 256;
  static constexpr size_t SMEM_MAX = MINB_ == 1 ? 232448 - 8192  // 227 KB opt-in minus static shared memory
                                                : 233472 / (MINB_ > 0 ? MINB_ : 1) - 1024 - STATIC_EST;
  static constexpr size_t MAIN = size_t(STAGES) * STAGE * sizeof(C) + TAB_BYTES;
  static constexpr int SPLIT0 = (SPLITOK_ && ROWS == 1 && STAGES == 1 &&
                                 (MINB_ == 1 || (MINB_ == 2 && XFT_SPLIT2) || (!C128 && MINB_ > 1 && XFT_SPLIT4)) &&
                                 XFT_SPLIT && SMEM_MAX > MAIN)
                                    ? int((SMEM_MAX - MAIN) / sizeof(C)) / TR * TR : 0;
  static constexpr int SPLIT = SPLIT0 < N ? SPLIT0 : 0;
  // Mirror lane map (row kernels, c128 LCT): lanes l and l^16 of a warp hold the
  // columns j and TR-1-j, whose elements k and n-1-k share x^2 (x_{n-1-k} =
  // -x_k exactly), hence the chirp-argument rounding corrections: each lane
  // computes 8 of its 16 and takes the other 8 from its partner by shuffle.
  static constexpr bool MIRROR = SPLITOK_ && C128 && MODE == MODE_LCT && TR % 32 == 0 && XFT_MIRROR;
  // (single-row CTAs only: at two CTAs/SM, n = 4096, the held registers spill and cost 6%; n = 8192 gains 4%)
  static constexpr bool TWBASE = SPLITOK_ && C128 && MODE == MODE_LCT && XFT_TWBASE && XFT_TWGEN && E == 16 &&
                                 NPASS <= E && MINB_ == 1;
  static constexpr size_t SMEM = MAIN + size_t(SPLIT) * sizeof(C);
  // Split exchange barriers (row kernels): "every thread has finished reading the buffer" is an
  // mbarrier phase -- each warp arrives right after its reads and only waits just before its next
  // exchange stores, one butterfly pass later -- instead of a CTA-wide rendezvous in front of the
  // stores; the barrier between the stores and the loads stays.  With one stage the last phase of a
  // row (last exchange read) is waited for by thread 0 alone, which then issues the next row's load.
  // XBAR_: -1 = the row kernels' choice (XFT_XBAR* above), 0 = off, 1 = on for a caller that brings its own
  // mbarriers and does not need the last exchange's phase (the column ring kernel: its `empty` barrier)
  static constexpr bool XBAR =
      XFT_SKELETON == 0 && THREADS % 32 == 0 &&
      (XBAR_ >= 0 ? XBAR_ != 0
                  : SPLITOK_ && BARTH_ == 0 &&
                        (sizeof(C_) == 16 ? XFT_XBAR128 != 0 : (XFT_XBAR64_ALL || (XFT_XBAR64 && MINB_ == 1))));
  static constexpr bool XBAR_LAST = XBAR && XBAR_ < 0 && STAGES_ == 1;
  // L2 prefetch depth of the row kernels (tiles beyond the ring; see XFT_L2PF_*)
  static constexpr int L2PF = !SPLITOK_       ? 0
                              : XFT_L2PF >= 0 ? XFT_L2PF
                              : (sizeof(C_) == 16 ? LOG2N_ == 12 : (LOG2N_ == 14 || LOG2N_ == 10)) ? 1 : 0;
  static_assert(NPASS >= 2, "pipelined kernel needs at least one exchange");
  static_assert(TR >= 2, "k & 1 == j & 1 needs an even thread stride");
  static_assert(THREADS <= 1024, "threads");
  static constexpr int ns(int p) { return p == 0 ? 1 : R0 * ipow(E, p - 1); }
  static constexpr int twoff(int p) { return p <= 1 ? 0 : twoff(p - 1) + (E - 1) * ns(p - 1); }
  static constexpr int TW_ENTRIES = twoff(NPASS);
  // resident CTAs per SM the register budget is sized for
  static constexpr int MINB = MINB_;
};

#ifndef XFT_DFT_COLTW
#define XFT_DFT_COLTW 1  // c128 plain-DFT radix-16 passes: exact twiddles applied per 4-point column
#endif
#ifndef XFT_PDL_C128
#define XFT_PDL_C128 0  // 1: c128 row kernels launched with programmatic stream serialization (griddepcontrol):
                        // no gain alone (116.6 vs 116.7 us), and the early CTAs hold SM slots the concurrent
                        // c64 batch of a config-2 step needs (step 0.159 -> 0.170 ms): off
#endif
#ifndef XFT_PDL_C64
#define XFT_PDL_C64 0   // c64: A/B 53.6 vs 52.6 us with it: off
#endif
#define XFT_PDL (XFT_PDL_C128 || XFT_PDL_C64)
__device__ __forceinline__ void griddep_launch_dependents() {
  if (XFT_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() {
  if (XFT_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// padded exchange index: element a of a row lives at a + a/16
__device__ __forceinline__ constexpr int pad_idx(int a) { return a + (a >> 4); }

// release(): runs right after the first exchange barrier (pass 0).
// FREE_EARLY: after the last exchange's reads, one more barrier and free_hook()
// -- the buffer is dead from there on, so a single-stage caller can start the
// next tile's load under the last pass and the epilogue.
#ifndef XFT_TWPRE
#define XFT_TWPRE 0  // 1: load the next pass's twiddles between the exchange stores and the barrier
#endif
template <class Cfg>
__device__ __forceinline__ void pipe_sync() {
  if constexpr (Cfg::BARTH > 0) named_sync(1, Cfg::BARTH);
  else __syncthreads();
}

// split-barrier handle of a thread: NPASS mbarriers (one arrival per warp each), barrier IDX used once per row --
// IDX = 0: the input tile has been read, IDX = p: exchange p - 1 has been read -- so the phase parity is the row
// iteration's and no per-thread phase counter is carried (registers: the c128 CTAs run at their 128-register cap)
struct XBar {
  uint64_t* bars = nullptr;
  int it = 0;
  template <int IDX>
  __device__ __forceinline__ void arrive() const {  // this warp has finished reading the buffer
    __syncwarp();
    // one elected lane arrives for the warp (elect.sync: no lane index held in a register)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n"
        "}\n" ::"r"(smem_addr(bars + IDX))
        : "memory");
  }
  template <int IDX>
  __device__ __forceinline__ void wait() const { mbar_wait(bars + IDX, (uint32_t)it & 1u); }
};

template <class Cfg, int P, bool FREE_EARLY, class Release, class Free>
__device__ __forceinline__ void pipe_pass(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                          const typename Cfg::C* __restrict__ tw, Release&& release,
                                          Free&& free_hook, typename Cfg::C (&wpre)[Cfg::E], const XBar& xb) {
  using C = typename Cfg::C;
  constexpr int E = Cfg::E, TR = Cfg::TR;
  constexpr int R = (P == 0) ? Cfg::R0 : E;
  constexpr int NS = Cfg::ns(P);
  constexpr int NB = E / R;
  constexpr bool LAST = (P == Cfg::NPASS - 1);
  // c128 LCT-mode radix-16 passes: twiddles fused into the butterfly's first stage
  constexpr bool FUSED = (Cfg::C128 ? XFT_FUSE_TW : XFT_FUSE_TW64) && R == 16 && XFT_DFT16_44 && NS > 1 &&
                         XFT_SKELETON == 0 && !XFT_NOTW && XFT_TWGEN && (!Cfg::C128 || Cfg::MODE != MODE_DFT);
  // exact-table twiddles column by column (the passes that do not generate them: c128 plain DFT)
  constexpr bool COLTW = !FUSED && XFT_DFT_COLTW && R == 16 && XFT_DFT16_44 && NS > 1 && XFT_SKELETON == 0 &&
                         !XFT_NOTW && !XFT_TWPRE && Cfg::C128 && Cfg::MODE == MODE_DFT;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int i = j + b * TR;
    const int k = i & (NS - 1);
    C u[R];
#pragma unroll
    for (int t = 0; t < R; ++t) u[t] = v[b + t * NB];
    if constexpr (NS > 1 && XFT_SKELETON == 0 && !XFT_NOTW && XFT_TWGEN && (!Cfg::C128 || Cfg::MODE != MODE_DFT) && R >= 8) {
      // w^t from w and w^{8b} (table): w^2..w^7 by a product tree of depth 3,
      // w^{8b+r} = w^{8b} w^r.  R/8 loads instead of R - 1 (fewer registers held
      // by in-flight loads; cfg4 191 -> 182 us, cfg2 c128 129.2 -> 127.6 us) and
      // short dependency chains; error <= 4 rounding steps per twiddle.
      // The plain-DFT configurations (chirp-z / Mehler convolutions, up to
      // 2^17 points) keep the exact table twiddles.
      const C* twp = tw + Cfg::twoff(P) + k;
      auto ld = [&](int t) {
        C w = __ldg(twp + (t - 1) * NS);
        return Cfg::SIGN > 0 ? cconj(w) : w;
      };
      C lo[8];
      // row kernels (c128): w^1 of every twiddled pass is a per-thread constant,
      // loaded once per kernel into wpre[P] by the caller (no load per row)
      if constexpr (Cfg::TWBASE) lo[1] = wpre[P];
      else lo[1] = ld(1);
      lo[2] = XFT_TWLOAD4 ? ld(2) : cmul(lo[1], lo[1]);
      lo[3] = cmul(lo[2], lo[1]);
      lo[4] = XFT_TWLOAD4 ? ld(4) : cmul(lo[2], lo[2]);
      lo[5] = cmul(lo[4], lo[1]);
      lo[6] = cmul(lo[4], lo[2]);
      lo[7] = cmul(lo[4], lo[3]);
      if constexpr (FUSED) {
        // twiddles folded into the first 4-point stage of the 4 x 4 butterfly:
        // x0 + w2 u2 = fma chain (no separate product), x0 - w2 u2 = 2 x0 - (x0 + w2 u2)
        const C h = (Cfg::C128 ? XFT_TWLOAD1 : 0) ? cmul(lo[4], lo[4]) : ld(8);  // c128: one table load
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) {
          const C x0 = n2 == 0 ? u[0] : cmul(u[n2], lo[n2]);
          const C x1 = cmul(u[4 + n2], lo[4 + n2]);
          const C w2 = n2 == 0 ? h : cmul(h, lo[n2]);
          const C w3 = cmul(h, lo[4 + n2]);
          const C a = u[8 + n2], b = u[12 + n2];
          const C t0 = cfma(a, w2, x0);
          const C t1 = ctwice_minus(x0, t0);
          const C t2 = cfma(b, w3, x1);
          const C t3 = rot<Cfg::SIGN>(ctwice_minus(x1, t2));
          u[n2] = cadd(t0, t2);
          u[8 + n2] = csub(t0, t2);
          u[4 + n2] = cadd(t1, t3);
          u[12 + n2] = csub(t1, t3);
        }
      } else {
#pragma unroll
        for (int t = 1; t < 8; ++t) u[t] = cmul(u[t], lo[t]);
#pragma unroll
        for (int b = 1; b < R / 8; ++b) {
          const C h = ld(8 * b);
          u[8 * b] = cmul(u[8 * b], h);
#pragma unroll
          for (int r = 1; r < 8; ++r) u[8 * b + r] = cmul(u[8 * b + r], cmul(h, lo[r]));
        }
      }
    } else if constexpr (COLTW) {
      // exact table twiddles (plain-DFT passes: chirp-z / Mehler convolutions), applied one
      // 4-point column of the 4 x 4 butterfly at a time, the column's 4-point DFT right after:
      // at most 3 twiddles are live (c128 M = 8192 Mehler rows: spills 868 -> see ptxas log)
      const C* twp = tw + Cfg::twoff(P) + k;
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int t = 4 * q + n2;
          if (t == 0) continue;
          C w = __ldg(twp + (t - 1) * NS);
          if (Cfg::SIGN > 0) w = cconj(w);
          u[t] = cmul(u[t], w);
        }
        dft4<Cfg::SIGN>(u[n2], u[4 + n2], u[8 + n2], u[12 + n2]);
      }
    } else if constexpr (NS > 1 && XFT_SKELETON == 0 && !XFT_NOTW) {
      const C* twp = tw + Cfg::twoff(P) + k;
#pragma unroll
      for (int t = 1; t < R; ++t) {
        C w;
        if constexpr (XFT_TWPRE && P >= 1 && NB == 1) w = wpre[t - 1];  // loaded under the previous barrier
        else w = __ldg(twp + (t - 1) * NS);
        if (Cfg::SIGN > 0) w = cconj(w);
        u[t] = cmul(u[t], w);
      }
    }
    if constexpr (FUSED || COLTW) dft16_44_rows<Cfg::SIGN>(u);  // first stage done above
    else if constexpr (XFT_SKELETON == 0) dft_r<R, Cfg::SIGN>(u);
#pragma unroll
    for (int t = 0; t < R; ++t) v[b + t * NB] = u[t];
  }
  if constexpr (!LAST) {
    // every thread is done reading this buffer
    if constexpr (Cfg::XBAR) xb.template wait<P>();  // (arrivals: after the pre-multiply reads / the previous exchange's loads)
    else pipe_sync<Cfg>();
    if constexpr (P == 0) release();  // (first-barrier hook)
    // Stockham store: element t of butterfly i goes to base + t NS, base =
    // (i - k) R + k.  (base mod 16) + (t NS mod 16) < 16 for every thread (NS
    // and R are powers of two, k < NS), so pad_idx(base + t NS) =
    // pad_idx(base) + t NS + (t NS) / 16: one address per butterfly.
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = j + b * TR;
      const int k = i & (NS - 1);
      C* dst = rs + pad_idx((i - k) * R + k);
#pragma unroll
      for (int t = 0; t < R; ++t) dst[t * NS + ((t * NS) >> 4)] = v[b + t * NB];
    }
    if constexpr (XFT_TWPRE && XFT_SKELETON == 0 && !XFT_NOTW) {
      // v is dead until the loads below: its registers carry the next pass's twiddles
      // across the barrier, so their L1/L2 latency overlaps the wait
      constexpr int NS1 = Cfg::ns(P + 1);
      if constexpr (NS1 > 1 && E / E == 1) {
        const C* twp = tw + Cfg::twoff(P + 1) + (j & (NS1 - 1));
#pragma unroll
        for (int t = 1; t < E; ++t) wpre[t - 1] = __ldg(twp + (t - 1) * NS1);
      }
    }
    pipe_sync<Cfg>();
    // j < TR and TR | 16 or 16 | TR: pad_idx(j + s TR) = pad_idx(j) + s TR + (s TR) / 16
    const C* src = rs + pad_idx(j);
#pragma unroll
    for (int s = 0; s < E; ++s) v[s] = src[s * TR + ((s * TR) >> 4)];
    if constexpr (Cfg::XBAR) {
      // the last exchange's phase is only needed (and only waited for, by thread 0) where the
      // buffer is handed back to the TMA right away: single-stage CTAs
      if constexpr (P < Cfg::NPASS - 2 || Cfg::XBAR_LAST) xb.template arrive<P + 1>();
      if constexpr (FREE_EARLY && P == Cfg::NPASS - 2) {
        if (threadIdx.x == 0) xb.template wait<P + 1>();
        free_hook();
      }
    } else if constexpr (FREE_EARLY && P == Cfg::NPASS - 2) {
      pipe_sync<Cfg>();
      free_hook();
    }
  }
}

template <class Cfg, int P, bool FREE_EARLY, class Release, class Free>
__device__ __forceinline__ void pipe_passes_w(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                              const typename Cfg::C* __restrict__ tw, Release&& release,
                                              Free&& free_hook, typename Cfg::C (&wpre)[Cfg::E], const XBar& xb) {
  if constexpr (P < Cfg::NPASS) {
    pipe_pass<Cfg, P, FREE_EARLY>(v, rs, j, tw, release, free_hook, wpre, xb);
    pipe_passes_w<Cfg, P + 1, FREE_EARLY>(v, rs, j, tw, release, free_hook, wpre, xb);
  }
}

template <class Cfg, int P, bool FREE_EARLY = false, class Release, class Free>
__device__ __forceinline__ void pipe_passes(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                            const typename Cfg::C* __restrict__ tw, Release&& release,
                                            Free&& free_hook) {
  typename Cfg::C wpre[Cfg::E];
  XBar none;  // (callers of this overload never set Cfg::XBAR)
  static_assert(!Cfg::XBAR, "split barriers need the caller's mbarriers");
  pipe_passes_w<Cfg, P, FREE_EARLY>(v, rs, j, tw, release, free_hook, wpre, none);
}

template <class Cfg, int P, class Release>
__device__ __forceinline__ void pipe_passes(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                            const typename Cfg::C* __restrict__ tw, Release&& release) {
  pipe_passes<Cfg, P, false>(v, rs, j, tw, release, []() {});
}

// the same with the caller's split barriers (Cfg::XBAR; the caller has arrived on barrier 0 after its own reads)
template <class Cfg, int P, class Release>
__device__ __forceinline__ void pipe_passes_x(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                              const typename Cfg::C* __restrict__ tw, Release&& release,
                                              const XBar& xb) {
  typename Cfg::C wpre[Cfg::E];
  pipe_passes_w<Cfg, P, false>(v, rs, j, tw, release, []() {}, wpre, xb);
}

// ---------------------------------------------------------------------------
// per-thread invariants (depend on j and n only; computed once per kernel)
// ---------------------------------------------------------------------------
template <class Cfg, bool IS128 = Cfg::C128>
struct ThreadConst;

template <class Cfg>
struct ThreadConst<Cfg, false> {
  int off0;      // 2j - n + 1
  uint32_t bt0;  // top word of the boundary-phase turns at k = j
  __device__ __forceinline__ explicit ThreadConst(int j) {
    off0 = 2 * j - Cfg::N + 1;
    bt0 = ((uint32_t)(j & 1) << 31) - ((uint32_t)j << (31 - Cfg::LOG2N));
  }
};

template <class Cfg>
struct ThreadConst<Cfg, true> {
  double off0;  // 2j - n + 1
  // boundary phase (-1)^k e^{-i pi k/n}, k = j + s TR, in table units U = 2 pi/T
  // (T = C128_TABN, H = T/2): H (k & 1) - H k / n = [q0 - (H/E) s] + d0 / U, the
  // integer part going to the table index (q0, and a per-s immediate), |d0| <= U/2
  static constexpr int H = C128_TABN / 2;
  double d0;
  int q0;
  // walk path: the boundary phase at k = j in turns, (n-1) j / 2n mod 1 (exact)
  double lin0;
  __device__ __forceinline__ explicit ThreadConst(int j) {
    off0 = opaque((double)(2 * j - Cfg::N + 1));
    lin0 = opaque(0.5 * (double)(j & 1) - (double)j / (double)(2 * Cfg::N));
    const int jq = (H * j + Cfg::N / 2) / Cfg::N;  // nearest integer to H j / n
    d0 = opaque(-(double)(H * j - jq * Cfg::N) * (6.283185307179586477 / (double(C128_TABN) * Cfg::N)));
    q0 = (j & 1) * H - jq;
  }
  static constexpr int qstep(int s) { return -(H / Cfg::E) * s; }
};

// c128 chirp walk over a thread's elements k = j + s TR (m = m0 + 2 TR s):
// the smooth phase D m^2 + (boundary/constant turns) is a quadratic in s, so
// W(s+1) = W(s) R(s), R(s+1) = R(s) S with W(0), R(0) from the table path
// (exact double-double arguments) and S per row.  Two complex multiplies per
// element, no table loads; |error| < ~2e-14 after 15 steps.
struct ChirpWalk {
  double2 W, R;
  template <class Cfg>
  __device__ __forceinline__ void init(double dhi, double dlo, const ThreadConst<Cfg>& tc, double lin, double mag,
                                       const double2* __restrict__ tab) {
    constexpr int TR = Cfg::TR;
    const double m0 = tc.off0;
    double f, lo;
    frac_dd(dhi, dlo, m0 * m0, f, lo);
    W = turn_phasor(f, lin, lo, tab);
    W.x *= mag;
    W.y *= mag;
    // R(0): D ((m0 + 2TR)^2 - m0^2) + one step of the boundary phase, (n-1) TR / 2n = -1/2E (mod 1)
    frac_dd(dhi, dlo, (double)(4 * TR) * (m0 + (double)TR), f, lo);
    R = turn_phasor(f, -0.5 / Cfg::E, lo, tab);
  }
  __device__ __forceinline__ void step(const double2& S, bool moveR) {
    W = make_double2(W.x * R.x - W.y * R.y, W.x * R.y + W.y * R.x);
    if (moveR) R = make_double2(R.x * S.x - R.y * S.y, R.x * S.y + R.y * S.x);
  }
};

// e^{i eps} ~ 1 + i eps applied to w: the reference's argument roundings,
// eps = fl(c fl(x^2)) - c X^2, x = fl(X), X = m half (xft/kernel.py:102, xft/hermite.py:87-89)
__device__ __forceinline__ double2 rot_eps(double2 w, double eps) {
  return make_double2(fma(-w.y, eps, w.x), fma(w.x, eps, w.y));
}
__device__ __forceinline__ double pre_eps(double m, double half, double c, double c2) {
  const double x = __dmul_rn(m, half);
  const double ex = fma(m, half, -x);   // X = x + ex
  const double x2 = __dmul_rn(x, x);
  const double e2 = fma(x, x, -x2);     // x^2 = x2 + e2
  const double ph = __dmul_rn(c, x2);   // the reference's phase
  const double ep = fma(-c, x2, ph);    // ph - c x2
  // ph - c X^2 = ep - c e2 - 2 c x ex  (- c ex^2, below 1e-25)
  return fma(c2, __dmul_rn(x, ex), fma(-c, e2, ep));
}
// output side: y = fl(s4 x), psi = fl(cout fl(y^2)) (xft/lct.py:196, xft/kernel.py:113), Y = s4 X
__device__ __forceinline__ double post_eps(double m, double half, double s4, double c, double c2) {
  const double x = __dmul_rn(m, half);
  const double ex = fma(m, half, -x);
  const double y = __dmul_rn(s4, x);
  const double dy = fma(s4, ex, fma(s4, x, -y));  // Y = y + dy
  const double y2 = __dmul_rn(y, y);
  const double e2 = fma(y, y, -y2);
  const double ps = __dmul_rn(c, y2);
  const double ep = fma(-c, y2, ps);
  return fma(c2, __dmul_rn(y, dy), fma(-c, e2, ep));
}

// ---------------------------------------------------------------------------
// pre / post multipliers over a thread's E registers (row-uniform branches
// are taken once per tile, not per element)
// ---------------------------------------------------------------------------
// v[s] = pre-multiplier(s) * ld(s): each element is fetched right where it is
// used, so the phasor chains of later elements overlap earlier loads instead of
// all E samples being held in registers before the first phasor starts
template <class Cfg, class Load>
__device__ __forceinline__ void pre_apply(typename Cfg::C (&v)[Cfg::E], Load&& ld, int j,
                                          const typename Cfg::Coef& rcs, const ThreadConst<Cfg>& tc,
                                          const RowConst& kc, const typename Cfg::C* __restrict__ ptab,
                                          const void* tabv) {
  constexpr int E = Cfg::E, TR = Cfg::TR;
  if constexpr (Cfg::MODE == MODE_DFT) {
#pragma unroll
    for (int s = 0; s < E; ++s) v[s] = ld(s);
  } else {
    int mode = 0;
    if constexpr (Cfg::MODE == MODE_LCT) mode = rcs.pre;
    if (mode == 0) {
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = cmul(__ldg(&ptab[j + s * TR]), ld(s));
      return;
    }
    if constexpr (Cfg::MODE == MODE_LCT) {
      if constexpr (!Cfg::C128) {
        // boundary phase (-1)^k e^{-i pi k/n} rides on the walk's linear term
        ChirpTurnWalk w(rcs.dq_in, tc.off0, 2 * TR, (unsigned long long)tc.bt0 << 32, 1ull << (63 - Cfg::LE));
#pragma unroll
        for (int s = 0; s < E; ++s) v[s] = cmul(walk_phasor(w.next()), ld(s));
      } else {
        const double2* tab = static_cast<const double2*>(tabv);
        const double cin = rcs.cin, half = kc.half;
        if (mode <= 2) {
          ChirpWalk w;
          w.init<Cfg>(rcs.din_hi, rcs.din_lo, tc, tc.lin0, 1.0, tab);
          const double2 S = rcs.sin_;
          if (mode == 1) {
#pragma unroll
            for (int s = 0; s < E; ++s) {
              v[s] = cmul(w.W, ld(s));
              if (s < E - 1) w.step(S, s < E - 2);
            }
          } else {
            const double c2 = -2.0 * cin;
            const double o = opaque(tc.off0);  // per tile: keeps the 16 m's from being hoisted (and spilled)
            if constexpr (Cfg::MIRROR) {
              double e[E];
#pragma unroll
              for (int s = 0; s < E / 2; ++s) e[s] = pre_eps(o + (double)(2 * s * TR), half, cin, c2);
#pragma unroll
              for (int s = E / 2; s < E; ++s) e[s] = __shfl_xor_sync(0xffffffffu, e[E - 1 - s], 16);
#pragma unroll
              for (int s = 0; s < E; ++s) {
                v[s] = cmul(rot_eps(w.W, e[s]), ld(s));
                if (s < E - 1) w.step(S, s < E - 2);
              }
            } else {
#pragma unroll
              for (int s = 0; s < E; ++s) {
                const double eps = pre_eps(o + (double)(2 * s * TR), half, cin, c2);
                v[s] = cmul(rot_eps(w.W, eps), ld(s));
                if (s < E - 1) w.step(S, s < E - 2);
              }
            }
          }
        } else if (mode == 3) {
#pragma unroll
          for (int s = 0; s < E; ++s) {
            const double x = __dmul_rn(tc.off0 + (double)(2 * s * TR), half);  // xft/hermite.py:87-89
            const double phi = __dmul_rn(cin, __dmul_rn(x, x));               // xft/kernel.py:102
            v[s] = cmul(unit_phase_tab(phi, tc.d0, tc.q0 + tc.qstep(s), tab), ld(s));
          }
        } else {
#pragma unroll
          for (int s = 0; s < E; ++s) {
            const double x = __dmul_rn(tc.off0 + (double)(2 * s * TR), half);
            const double phi = __dmul_rn(cin, __dmul_rn(x, x));
            v[s] = cmul(unit_phase_tab(prereduce(phi), tc.d0, tc.q0 + tc.qstep(s), tab), ld(s));
          }
        }
      }
    }
  }
}

template <class Cfg>
__device__ __forceinline__ void pre_multiply(typename Cfg::C (&v)[Cfg::E], const typename Cfg::C* rs, int j,
                                             const typename Cfg::Coef& rcs, const ThreadConst<Cfg>& tc,
                                             const RowConst& kc, const typename Cfg::C* __restrict__ ptab,
                                             const void* tabv) {
  pre_apply<Cfg>(v, [&](int s) { return rs[j + s * Cfg::TR]; }, j, rcs, tc, kc, ptab, tabv);
}

// output addressing of one row: natural (seg_stride == 0) or split into
// 2^segl-wide segments placed seg_stride apart (the all-to-all send layout of
// the sharded 2-D transform: segment g of row r lands at g*seg_stride + r*2^segl)
template <class C>
struct OutRow {
  C* base;  // natural: row start; segmented: out + r * 2^segl; peer: (row0 + r) * 2^segl
  long long seg_stride;
  int segl;
  void* const* peers;  // peer mode (seg_stride < 0): segment h goes to peers[h] + base offset
  __device__ __forceinline__ C* at(int c) const {
    if (seg_stride == 0) return base + c;
    if (seg_stride < 0)
      return static_cast<C*>(peers[c >> segl]) + reinterpret_cast<long long>(base) + (c & ((1 << segl) - 1));
    return base + (long long)(c >> segl) * seg_stride + (c & ((1 << segl) - 1));
  }
};

// Peer destinations of the sharded 2-D transform's row pass: segment h of
// every row is stored straight into rank h's receive slab (NVLink peer
// memory), at row row0 + r, so the all-to-all is the row kernel's own stores.
struct PeerTable {
  void* p[8];
  long long row0;
  int count;  // 0: not used
};

// post-multiplier of element s of a thread's E registers, handed to emit(s, value)
// (a streaming store in the row kernel, a register write-back in the chain kernel)
template <class Cfg, class Emit>
__device__ __forceinline__ void post_apply(typename Cfg::C (&v)[Cfg::E], int j, const typename Cfg::Coef& rcs,
                                           const ThreadConst<Cfg>& tc, const RowConst& kc, double2 cn,
                                           const typename Cfg::C* __restrict__ ptab, const void* tabv, Emit&& emit) {
  using C = typename Cfg::C;
  constexpr int E = Cfg::E, TR = Cfg::TR;
  if constexpr (Cfg::MODE == MODE_DFT) {
#pragma unroll
    for (int s = 0; s < E; ++s) emit(s, v[s]);
  } else if constexpr (Cfg::MODE == MODE_SCALED) {
    const C c = to_c<C>(cn);
#pragma unroll
    for (int s = 0; s < E; ++s) emit(s, cmul(c, cmul(__ldg(&ptab[j + s * TR]), v[s])));
  } else {
    if (rcs.post == 0) {
      const C g = rcs.g;
#pragma unroll
      for (int s = 0; s < E; ++s) emit(s, cmul(cmul(g, __ldg(&ptab[j + s * TR])), v[s]));
      return;
    }
    if constexpr (!Cfg::C128) {
      ChirpTurnWalk w(rcs.dq_out, tc.off0, 2 * TR, (unsigned long long)(tc.bt0 + rcs.gq) << 32, 1ull << (63 - Cfg::LE));
      const float2 g = make_float2(rcs.gabs, rcs.gabs);
#pragma unroll
      for (int s = 0; s < E; ++s) emit(s, cmul(walk_phasor(w.next()), p_mul(v[s], g)));
    } else {
      const double2* tab = static_cast<const double2*>(tabv);
      const double cout = rcs.cout, s4 = rcs.s4, half = kc.half, g = rcs.gabs;
      const double d0 = tc.d0 + rcs.gf;
      const int q0 = tc.q0 + rcs.gi;
      if (rcs.post <= 2) {
        ChirpWalk w;
        w.init<Cfg>(rcs.dout_hi, rcs.dout_lo, tc, tc.lin0 + rcs.gturn, g, tab);
        const double2 S = rcs.sout;
        if (rcs.post == 1) {
#pragma unroll
          for (int s = 0; s < E; ++s) {
            emit(s, cmul(w.W, v[s]));
            if (s < E - 1) w.step(S, s < E - 2);
          }
        } else {
          const double c2 = -2.0 * cout;
          const double o = opaque(tc.off0);
          if constexpr (Cfg::MIRROR) {  // y_{n-1-k} = -y_k exactly: the corrections are shared too
            double e[E];
#pragma unroll
            for (int s = 0; s < E / 2; ++s) e[s] = post_eps(o + (double)(2 * s * TR), half, s4, cout, c2);
#pragma unroll
            for (int s = E / 2; s < E; ++s) e[s] = __shfl_xor_sync(0xffffffffu, e[E - 1 - s], 16);
#pragma unroll
            for (int s = 0; s < E; ++s) {
              emit(s, cmul(rot_eps(w.W, e[s]), v[s]));
              if (s < E - 1) w.step(S, s < E - 2);
            }
          } else {
#pragma unroll
            for (int s = 0; s < E; ++s) {
              const double eps = post_eps(o + (double)(2 * s * TR), half, s4, cout, c2);
              emit(s, cmul(rot_eps(w.W, eps), v[s]));
              if (s < E - 1) w.step(S, s < E - 2);
            }
          }
        }
      } else if (rcs.post == 3) {
#pragma unroll
        for (int s = 0; s < E; ++s) {
          const double x = __dmul_rn(tc.off0 + (double)(2 * s * TR), half);
          const double y = __dmul_rn(s4, x);                    // xft/lct.py:196
          const double psi = __dmul_rn(cout, __dmul_rn(y, y));  // xft/kernel.py:113
          const double2 e = unit_phase_tab(psi, d0, q0 + tc.qstep(s), tab);
          emit(s, cmul(make_double2(e.x * g, e.y * g), v[s]));
        }
      } else {
#pragma unroll
        for (int s = 0; s < E; ++s) {
          const double x = __dmul_rn(tc.off0 + (double)(2 * s * TR), half);
          const double y = __dmul_rn(s4, x);
          const double psi = __dmul_rn(cout, __dmul_rn(y, y));
          const double2 e = unit_phase_tab(prereduce(psi), d0, q0 + tc.qstep(s), tab);
          emit(s, cmul(make_double2(e.x * g, e.y * g), v[s]));
        }
      }
    }
  }
}

template <class Cfg>
__device__ __forceinline__ void post_store(typename Cfg::C (&v)[Cfg::E], const OutRow<typename Cfg::C>& dst, int j,
                                           const typename Cfg::Coef& rcs, const ThreadConst<Cfg>& tc,
                                           const RowConst& kc, double2 cn, const typename Cfg::C* __restrict__ ptab,
                                           const void* tabv) {
  if (dst.seg_stride == 0) {  // row-uniform: one address per thread, immediate offsets
    typename Cfg::C* p = dst.base + j;
    post_apply<Cfg>(v, j, rcs, tc, kc, cn, ptab, tabv,
                    [&](int s, typename Cfg::C o) { st_stream(p + s * Cfg::TR, o); });
  } else {
    post_apply<Cfg>(v, j, rcs, tc, kc, cn, ptab, tabv,
                    [&](int s, typename Cfg::C o) { st_stream(dst.at(j + s * Cfg::TR), o); });
  }
}

// ---------------------------------------------------------------------------
// the kernel.  Thread 0 keeps STAGES-1 tile loads in flight (bulk TMA onto
// one mbarrier per stage); every thread transforms.  The next load is issued right after the first
// exchange barrier of the current tile, i.e. once every thread has finished
// the previous tile and the oldest stage is free.
// ---------------------------------------------------------------------------
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
xft_pipe_kernel(const typename Cfg::C* __restrict__ in, typename Cfg::C* __restrict__ out, long long batch,
                const double* __restrict__ abcd, long long abcd_stride, Abcd uni, const typename Cfg::C* __restrict__ tw,
                const typename Cfg::C* __restrict__ ptab, const void* __restrict__ gtab, double2 cn, RowConst kc,
                int seg_log2w, long long seg_stride, const __grid_constant__ PeerTable peers) {
  using C = typename Cfg::C;
  using Coef = typename Cfg::Coef;
  constexpr int N = Cfg::N, ROWS = Cfg::ROWS, S = Cfg::STAGES;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t bars[S];
  __shared__ __align__(8) uint64_t xbars[Cfg::NPASS];  // PipeCfg::XBAR: the "buffer read" phases, one arrival per warp
  // per-row coefficients of the next CH tiles of this CTA, computed by all
  // threads together once per CH tiles (one make_coef latency per chunk)
  constexpr int CH = Cfg::MODE == MODE_LCT ? (Cfg::C128 && ROWS == 1 ? XFT_C128_CH
                                             : ROWS >= 128 ? 1 : 128 / ROWS < 32 ? 128 / ROWS : 32) : 1;
  __shared__ Coef coeft[CH][Cfg::MODE == MODE_LCT ? ROWS : 1];

  C* stage0 = reinterpret_cast<C*>(xft_smem);
  void* tab = xft_smem + size_t(S) * Cfg::STAGE * sizeof(C);
  constexpr int SPLIT = Cfg::SPLIT;
  C* const regA = reinterpret_cast<C*>(xft_smem + Cfg::MAIN);  // samples [0, SPLIT) of the row (split mode)

  const int tid = threadIdx.x;
  const int lrow = tid / Cfg::TR;
  const int jt = tid - lrow * Cfg::TR;
  const int j = Cfg::MIRROR ? ((jt & 16) ? Cfg::TR - 1 - (((jt >> 5) << 4) | (jt & 15)) : (((jt >> 5) << 4) | (jt & 15)))
                            : jt;
  const long long ntiles = (batch + ROWS - 1) / ROWS;
  const long long G = gridDim.x;
  const ThreadConst<Cfg> tc(j);

  auto issue = [&](long long t, int st) {
    fence_proxy_async_smem();
    const long long rows = batch - t * ROWS < ROWS ? batch - t * ROWS : ROWS;
    const uint32_t bytes = (uint32_t)(rows * N * sizeof(C));
    mbar_arrive_expect_tx(&bars[st], bytes);
    tma_load_1d(stage0 + size_t(st) * Cfg::STAGE, in + (XFT_NOMEM ? (long long)blockIdx.x : t) * Cfg::TILE, bytes, &bars[st]);
  };
  // split mode (ROWS == 1): part A = samples [0, SPLIT) -> regA, part B = the rest -> the stage
  auto issue_a = [&](long long t) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[0], (uint32_t)(SPLIT * sizeof(C)));
    tma_load_1d(regA, in + (XFT_NOMEM ? (long long)blockIdx.x : t) * Cfg::TILE, (uint32_t)(SPLIT * sizeof(C)), &bars[0]);
  };
  auto issue_b = [&](long long t) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[0], (uint32_t)((N - SPLIT) * sizeof(C)));
    tma_load_1d(stage0 + SPLIT, in + (XFT_NOMEM ? (long long)blockIdx.x : t) * Cfg::TILE + SPLIT,
                (uint32_t)((N - SPLIT) * sizeof(C)), &bars[0]);
  };
  auto fill_coefs = [&](long long first_tile) {  // tiles first_tile + q*G, q < CH
    if constexpr (Cfg::MODE == MODE_LCT) {
      for (int idx = threadIdx.x; idx < CH * ROWS; idx += Cfg::THREADS) {
        const long long row = (first_tile + (long long)(idx / ROWS) * G) * ROWS + idx % ROWS;
        if (row < batch) make_coef(coeft[idx / ROWS][idx % ROWS], abcd ? abcd + row * abcd_stride : nullptr, uni, kc, Cfg::TR,
                                static_cast<const double2*>(tab));
      }
    }
  };

  // ---- prologue ----
  // Programmatic dependent launch (XFT_PDL): the next launch on this stream may
  // start its own prologue on SMs this grid frees; everything before
  // griddep_wait() below touches only library-owned constant tables.
  griddep_launch_dependents();
  if constexpr (XFT_TW_PREFETCH && Cfg::NPASS > 1) {
    // this thread's first-row twiddle entries (w and w^8 of every pass) into L1
#pragma unroll
    for (int p = 1; p < Cfg::NPASS; ++p) {
      const typename Cfg::C* tp = tw + Cfg::twoff(p) + (j & (Cfg::ns(p) - 1));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
      if (Cfg::E >= 16) asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + 7 * Cfg::ns(p)));
    }
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], SPLIT ? 2 : 1);  // split: one arrival per part
    if constexpr (Cfg::XBAR)
      for (int s = 0; s < Cfg::NPASS; ++s) mbar_init(&xbars[s], Cfg::THREADS / 32);
    fence_mbar_init();
  }
  if constexpr (Cfg::C128) {
    double2* t = static_cast<double2*>(tab);
    const double2* g = static_cast<const double2*>(gtab);
    for (int m = tid; m < XFT_C128_TABCOPIES * C128_TABN; m += Cfg::THREADS)
      t[m] = g[XFT_C128_TABCOPIES == 8 ? m >> 3 : m];
  }
  // the caller's data (in, abcd, out) only after the previous grid on the stream is complete
  griddep_wait();
  if constexpr (Cfg::MODE == MODE_LCT && XFT_COEF_PREFETCH) {
    // the first chunk's parameter rows: their global latency overlaps the barrier and first TMA issue
    if (abcd && tid < CH * ROWS) {
      const long long row = ((long long)blockIdx.x + (long long)(tid / ROWS) * G) * ROWS + tid % ROWS;
      if (row < batch) asm volatile("prefetch.global.L1 [%0];" ::"l"(abcd + row * abcd_stride));
    }
  }
  __syncthreads();
  long long tile = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S - 1; ++s)
      if (tile + s * G < ntiles) issue(tile + s * G, s);
    if (S == 1 && tile < ntiles) {
      if constexpr (SPLIT > 0) {
        issue_a(tile);
        issue_b(tile);
      } else {
        issue(tile, 0);
      }
    }
  }

  C wbase[Cfg::E];  // TWBASE: wbase[P] = w^1 of pass P for this thread (constant over rows)
  if constexpr (Cfg::TWBASE) {
#pragma unroll
    for (int p = 1; p < Cfg::NPASS; ++p) {
      const int nsp = Cfg::ns(p);
      C w = __ldg(tw + Cfg::twoff(p) + (j & (nsp - 1)));
      wbase[p] = Cfg::SIGN > 0 ? cconj(w) : w;
    }
  }
  for (int it = 0; tile < ntiles; ++it, tile += G) {
    const int st = it % S;
    if constexpr (Cfg::MODE == MODE_LCT) {
      if (it % CH == 0) {
        __syncthreads();  // the previous chunk's coefficients are no longer read
        fill_coefs(tile);
        __syncthreads();
      }
    }
    auto l2_prefetch = [&]() {
      if constexpr (Cfg::L2PF > 0 && !XFT_NOMEM) {
        // pull the tile L2PF ahead of the ring into L2 while this one is transformed
        const long long pt = tile + (long long)(S - 1 + Cfg::L2PF) * G;
        if (tid == 0 && pt < ntiles) {
          const long long rows = batch - pt * ROWS < ROWS ? batch - pt * ROWS : ROWS;
          tma_prefetch_l2(in + pt * Cfg::TILE, (uint32_t)(rows * N * sizeof(C)));
        }
      }
    };
    if constexpr (XFT_L2PF_EARLY) l2_prefetch();
    mbar_wait(&bars[st], (uint32_t)((it / S) & 1));
    if constexpr (!XFT_L2PF_EARLY) l2_prefetch();
    C* const stg = stage0 + size_t(st) * Cfg::STAGE;
    const C* rs = stg + size_t(lrow) * N;      // this row's input (TMA layout)
    C* xs = stg + size_t(lrow) * Cfg::NP;      // this row's exchange buffer (read-after-barrier)
    Coef rc;
    if constexpr (Cfg::MODE == MODE_LCT) rc = coeft[it % CH][lrow];

    C v[Cfg::E];
    if constexpr (XFT_SKELETON) {
#pragma unroll
      for (int s = 0; s < Cfg::E; ++s) v[s] = rs[j + s * Cfg::TR];
    } else if constexpr (SPLIT > 0) {
      // element s of this thread lives in part A iff s TR + j < SPLIT, i.e. s < SPLIT / TR
      pre_apply<Cfg>(v, [&](int s) { return (s < SPLIT / Cfg::TR ? regA : rs)[j + s * Cfg::TR]; }, j, rc, tc, kc,
                     ptab, tab);
    } else {
      pre_multiply<Cfg>(v, rs, j, rc, tc, kc, ptab, tab);
    }
    const XBar xb{xbars, it};
    if constexpr (Cfg::XBAR) xb.template arrive<0>();  // this warp has read its share of the input tile
    // the reference rejects non-finite samples (xft/lct.py:125-126): when the
    // caller asks (kc.bad), the pre-multiplied samples are checked right here --
    // a unit-modulus pre-multiplier keeps Inf/NaN non-finite -- two integer ops
    // per component, no extra HBM or shared-memory traffic
    if (kc.bad != nullptr) {
      unsigned fin = ~0u;
#pragma unroll
      for (int s = 0; s < Cfg::E; ++s) fin = min(fin, nonfinite_key(v[s]));
      if (fin == 0 && tile * ROWS + lrow < batch) atomicMin(kc.bad, (unsigned long long)(tile * ROWS + lrow));
    }

    // runs right after the first exchange barrier of this tile
    auto first_barrier = [&]() {
      if (S >= 2 && tid == 0) {
        const long long nt = tile + (S - 1) * G;
        if (nt < ntiles) issue(nt, (it + S - 1) % S);
      }
      if constexpr (SPLIT > 0) {  // part A of this row has been read: start the next row's part A
        if (tid == 0 && tile + G < ntiles) issue_a(tile + G);
      }
    };
    // single stage: the next tile's load starts once the last exchange has been
    // read (c64; for c128 the barrier in front of the fp64-heavy last pass
    // costs more than the earlier load gains, measured 137 -> 146 us at cfg2)
    constexpr bool EARLY = S == 1 && (!Cfg::C128 || XFT_C128_EARLY);
    auto stage_free = [&]() {
      if (tid == 0 && tile + G < ntiles) {
        if constexpr (SPLIT > 0) issue_b(tile + G);
        else issue(tile + G, 0);
      }
    };
    if constexpr (XFT_SKELETON == 2) {
      __syncthreads();
      first_barrier();
      if constexpr (EARLY) stage_free();  // (the passes that would free the stage are skipped)
    } else {
      pipe_passes_w<Cfg, 0, EARLY>(v, xs, j, tw, first_barrier, stage_free, wbase, xb);
    }
    if constexpr (S == 1 && !EARLY) {
      if constexpr (Cfg::XBAR) {  // thread 0 alone waits for the last exchange's reads
        if (tid == 0) xb.template wait<Cfg::NPASS - 1>();
      } else {
        __syncthreads();
      }
      stage_free();
    }

    const long long row = tile * ROWS + lrow;
    if constexpr (XFT_SKELETON) {
      if (row < batch)
#pragma unroll
        for (int s = 0; s < Cfg::E; ++s) st_stream(out + row * N + j + s * Cfg::TR, v[s]);
    } else {
      if (row < batch) {
        const OutRow<C> o{
            peers.count ? reinterpret_cast<C*>((peers.row0 + row) << seg_log2w)
            : seg_stride ? out + (row << seg_log2w)
                         : out + (XFT_NOMEM ? (long long)blockIdx.x * ROWS + lrow : row) * N,
            peers.count ? -1 : seg_stride, seg_log2w, peers.p};
        post_store<Cfg>(v, o, j, rc, tc, kc, cn, ptab, tab);
      }
    }
  }
}

}  // namespace xftb
