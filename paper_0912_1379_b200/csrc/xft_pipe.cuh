// K1 (production path): persistent, TMA-pipelined batched chirp-DFT-chirp.
//
// Each CTA is persistent over "tiles" (ROWS consecutive rows, one contiguous
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
//  * c128: phi_k = fl(fl(0.5a/b) fl(x_k^2)) is formed exactly as the reference
//    forms it (bit-identical fp64 argument); e^{i(phi+delta)} is evaluated as
//    T[q mod 256] * e^{i r}, q = rint((phi+delta)/(2pi/256)), r reduced with a
//    two-constant FMA Cody-Waite step, e^{ir} by degree-6/7 Taylor (|r|<=pi/256,
//    |err| < 1e-17), T a 256-entry table in shared memory.
//  * c64: the chirp phase in turns, frac(D k'^2 + boundary) with
//    D = (a/2b) half^2 / 2pi, is evaluated exactly in 64-bit fixed point
//    (integer multiply, wraps mod 1 turn), then an fp32 polynomial.
//    No fp64 and no conversions per element.
// Twiddles come from a pass-major table (entry (t-1)*NS + k of pass p holds
// w_{NS*E}^{t k}) so every warp's twiddle loads are coalesced.
#pragma once
#include "xft_rows.cuh"
#include "xft_tma.cuh"

namespace xftb {

#define XFT_PI 3.141592653589793116
#define XFT_INV_2PI 0.15915494309189534561
#define XFT_U_HI 0.02454369260617026          /* 2 pi / 256 */
#define XFT_U_LO 9.567553118338697e-19
#define XFT_INV_U 40.74366543152521

// ---------------------------------------------------------------------------
// per-row coefficients
// ---------------------------------------------------------------------------
struct Coef64 {
  unsigned long long dq_in, dq_out, gq;  // Q0.64 turns: chirp rates and arg G
  float gabs;                             // |G|
  float2 g;                               // G (used when d == 0)
  int pre, post;
};

struct Coef128 {
  double cin, cout, s4;  // fl(0.5a/b), fl(0.5d/b), fl(4b/pi)
  double gabs, gf;       // |G|, small part of arg G (|gf| <= U/2)
  double2 g;             // G (used when d == 0)
  int gi;                // arg G / U rounded (table units)
  int pre, post;
};

template <class C> struct CoefOf;
template <> struct CoefOf<float2> { using T = Coef64; };
template <> struct CoefOf<double2> { using T = Coef128; };

struct RowConst {  // per-launch constants (host computed)
  double half;         // (pi / sqrt(2n)) / 2
  double cnabs;        // |C(n)| = pi / sqrt(2n)
  long long cnred;     // (n-1)^2 mod 4n   (arg C(n) = -pi red / (2n))
  int log2n;
  int flags;
};

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

__device__ __forceinline__ void make_coef(Coef64& c, const double* p, const Abcd& uni, const RowConst& k) {
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
  c.gq = gq;
  const double gabs = g_abs(b, k);
  c.gabs = (float)gabs;
  double s, co;
  sincospi((double)(long long)gq * 1.0842021724855044e-19, &s, &co);  // 2 * gq / 2^64
  c.g = make_float2((float)(gabs * co), (float)(gabs * s));
  c.pre = (a != 0.0);
  c.post = (d != 0.0);
}

__device__ __forceinline__ void make_coef(Coef128& c, const double* p, const Abcd& uni, const RowConst& k) {
  double a, b, d;
  row_params(p, uni, a, b, d);
  c.cin = __ddiv_rn(0.5 * a, b);              // (0.5j * a / b).imag     xft/kernel.py:102
  c.cout = __ddiv_rn(0.5 * d, b);             // (0.5j * d / b).imag     xft/kernel.py:113
  c.s4 = __ddiv_rn(4.0 * b, XFT_PI);          // 4.0 * b / np.pi        xft/lct.py:196
  // arg G / U, U = 2pi/256: -64 red / n - 32 sgn(b) [+ 32]   (exact in fp64)
  double v = -64.0 * (double)k.cnred / (double)(1ll << k.log2n) + ((b > 0.0) ? -32.0 : 32.0);
  if (k.flags & FLAG_BARE_FOURIER) v += 32.0;
  const double vi = rint(v);
  c.gi = (int)vi;
  c.gf = (v - vi) * XFT_U_HI;
  c.gabs = g_abs(b, k);
  double s, co;
  sincospi(v * (1.0 / 128.0), &s, &co);
  c.g = make_double2(c.gabs * co, c.gabs * s);
  c.pre = (a != 0.0);
  c.post = (d != 0.0);
}

// ---------------------------------------------------------------------------
// unit phasors
// ---------------------------------------------------------------------------
// e^{2 pi i t / 2^32} in fp32 (t = turns in Q0.32), |err| ~ 1e-7
__device__ __forceinline__ float2 unit_from_turns(uint32_t t) {
  const uint32_t v = t + 0x20000000u;                     // + 1/8 turn
  const uint32_t quad = v >> 30;
  const int fi = (int)(v & 0x3FFFFFFFu) - 0x20000000;     // [-2^29, 2^29)
  const int fm = (fi + 64) >> 7;                          // |fm| <= 2^22
  const float r = (__int_as_float(0x4B400000 + fm) - 12582912.0f) * 1.8725351414619535e-07f;  // 2pi/2^25
  const float z = r * r;
  float ps = fmaf(z, -1.9841270e-04f, 8.3333333e-03f);
  ps = fmaf(z, ps, -1.6666667e-01f);
  const float s = fmaf(r * z, ps, r);
  float pc = fmaf(z, 2.4801587e-05f, -1.3888889e-03f);
  pc = fmaf(z, pc, 4.1666667e-02f);
  pc = fmaf(z, pc, -0.5f);
  const float c = fmaf(z, pc, 1.0f);
  float cs = (quad & 1) ? -s : c;
  float sn = (quad & 1) ? c : s;
  if (quad & 2) { cs = -cs; sn = -sn; }
  return make_float2(cs, sn);
}

// e^{i (phi + add)} * i^(2*odd) in fp64 via the 256-entry table tab[m] = e^{2 pi i m/256}.
// phi: exact fp64 chirp argument (any size up to ~1e12); add: small (|add| < 2 pi).
__device__ __forceinline__ double2 unit_phase_tab(double phi, double add, int qoff, const double2* __restrict__ tab) {
  if (fabs(phi) < 1.0e12) {
    const double t = fma(phi + add, XFT_INV_U, XFT_ROUND_MAGIC);
    const double qd = t - XFT_ROUND_MAGIC;
    const int q = __double2loint(t) + qoff;
    double r = fma(-qd, XFT_U_HI, phi);
    r = r + add;
    r = fma(-qd, XFT_U_LO, r);
    const double z = r * r;
    const double sn = fma(r * z, fma(z, 8.3333333333333333e-03, -1.6666666666666667e-01), r);
    const double cs = fma(z, fma(z, fma(z, -1.3888888888888889e-03, 4.1666666666666667e-02), -0.5), 1.0);
    const double2 w = tab[q & 255];
    return make_double2(w.x * cs - w.y * sn, w.x * sn + w.y * cs);
  }
  double s0, c0, s1, c1;
  sincos(phi, &s0, &c0);
  sincos(add, &s1, &c1);
  double2 e = make_double2(c0 * c1 - s0 * s1, s0 * c1 + c0 * s1);
  const double2 w = tab[qoff & 255];
  return make_double2(w.x * e.x - w.y * e.y, w.x * e.y + w.y * e.x);
}

// ---------------------------------------------------------------------------
// configuration
// ---------------------------------------------------------------------------
template <class C_, int LOG2N_, int E_, int MODE_, int SIGN_, int ROWS_, int STAGES_>
struct PipeCfg {
  using C = C_;
  using Coef = typename CoefOf<C>::T;
  static constexpr int LOG2N = LOG2N_, N = 1 << LOG2N, E = E_, MODE = MODE_, SIGN = SIGN_;
  static constexpr int ROWS = ROWS_, STAGES = STAGES_;
  static constexpr int TR = N / E;
  static constexpr int THREADS = TR * ROWS;
  static constexpr int TILE = ROWS * N;
  static constexpr int LE = ilog2(E);
  static constexpr int NPASS = (LOG2N + LE - 1) / LE;
  static constexpr int R0 = 1 << (LOG2N - (NPASS - 1) * LE);
  static constexpr bool C128 = sizeof(C) == 16;
  static constexpr size_t TAB_BYTES = C128 ? 256 * sizeof(double2) : 0;
  static constexpr size_t SMEM = size_t(STAGES) * TILE * sizeof(C) + TAB_BYTES;
  static_assert(NPASS >= 2, "pipelined kernel needs at least one exchange");
  static_assert(THREADS <= 1024 && THREADS % 32 == 0, "threads");
  static constexpr int ns(int p) { return p == 0 ? 1 : R0 * ipow(E, p - 1); }
  static constexpr int twoff(int p) { return p <= 1 ? 0 : twoff(p - 1) + (E - 1) * ns(p - 1); }
  static constexpr int TW_ENTRIES = twoff(NPASS);
  // resident CTAs per SM the register budget is sized for
  static constexpr int MINB = (SMEM * 2 <= 220 * 1024 && THREADS <= 512) ? 2 : 1;
};

template <class Cfg, int P, class Hook>
__device__ __forceinline__ void pipe_pass(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                          const typename Cfg::C* __restrict__ tw, Hook&& hook) {
  using C = typename Cfg::C;
  constexpr int E = Cfg::E, TR = Cfg::TR;
  constexpr int R = (P == 0) ? Cfg::R0 : E;
  constexpr int NS = Cfg::ns(P);
  constexpr int NB = E / R;
  constexpr bool LAST = (P == Cfg::NPASS - 1);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int i = j + b * TR;
    const int k = i & (NS - 1);
    C u[R];
#pragma unroll
    for (int t = 0; t < R; ++t) u[t] = v[b + t * NB];
    if constexpr (NS > 1) {
      const C* twp = tw + Cfg::twoff(P) + k;
#pragma unroll
      for (int t = 1; t < R; ++t) {
        C w = __ldg(twp + (t - 1) * NS);
        if (Cfg::SIGN > 0) w = cconj(w);
        u[t] = cmul(u[t], w);
      }
    }
    dft_r<R, Cfg::SIGN>(u);
#pragma unroll
    for (int t = 0; t < R; ++t) v[b + t * NB] = u[t];
  }
  if constexpr (!LAST) {
    __syncthreads();  // every thread is done reading this buffer
    if constexpr (P == 0) hook();
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
  }
}

template <class Cfg, int P, class Hook>
__device__ __forceinline__ void pipe_passes(typename Cfg::C (&v)[Cfg::E], typename Cfg::C* rs, int j,
                                            const typename Cfg::C* __restrict__ tw, Hook&& hook) {
  if constexpr (P < Cfg::NPASS) {
    pipe_pass<Cfg, P>(v, rs, j, tw, hook);
    pipe_passes<Cfg, P + 1>(v, rs, j, tw, hook);
  }
}

// ---------------------------------------------------------------------------
// pre / post multipliers
// ---------------------------------------------------------------------------
template <class Cfg, bool IS128 = Cfg::C128>
struct Chirp;

template <class Cfg>
struct Chirp<Cfg, false> {
  using C = float2;
  // f * p_k e^{i phi_k}
  static __device__ __forceinline__ C pre(C f, int k, const Coef64& rc, const RowConst& kc, const C* __restrict__ ptab,
                                          const double2*) {
    if constexpr (Cfg::MODE == MODE_DFT) return f;
    if (Cfg::MODE == MODE_LCT && rc.pre) {
      const int off = 2 * k - Cfg::N + 1;
      const unsigned long long bt = ((unsigned long long)(k & 1) << 63) - ((unsigned long long)k << (63 - Cfg::LOG2N));
      const unsigned long long u = rc.dq_in * (unsigned long long)(unsigned)(off * off) + bt;
      return cmul(unit_from_turns((uint32_t)(u >> 32)), f);
    }
    return cmul(__ldg(&ptab[k]), f);
  }
  static __device__ __forceinline__ C post(C S, int jj, const Coef64& rc, const RowConst& kc, double2 cn,
                                           const C* __restrict__ ptab, const double2*) {
    if constexpr (Cfg::MODE == MODE_DFT) return S;
    if constexpr (Cfg::MODE == MODE_SCALED) return cmul(make_float2((float)cn.x, (float)cn.y), cmul(__ldg(&ptab[jj]), S));
    if (rc.post) {
      const int off = 2 * jj - Cfg::N + 1;
      const unsigned long long bt = ((unsigned long long)(jj & 1) << 63) - ((unsigned long long)jj << (63 - Cfg::LOG2N));
      const unsigned long long u = rc.dq_out * (unsigned long long)(unsigned)(off * off) + bt + rc.gq;
      const float2 e = unit_from_turns((uint32_t)(u >> 32));
      return cmul(make_float2(e.x * rc.gabs, e.y * rc.gabs), S);
    }
    return cmul(cmul(rc.g, __ldg(&ptab[jj])), S);
  }
};

template <class Cfg>
struct Chirp<Cfg, true> {
  using C = double2;
  static __device__ __forceinline__ C pre(C f, int k, const Coef128& rc, const RowConst& kc,
                                          const C* __restrict__ ptab, const double2* tab) {
    if constexpr (Cfg::MODE == MODE_DFT) return f;
    if (Cfg::MODE == MODE_LCT && rc.pre) {
      const double x = __dmul_rn((double)(2 * k - Cfg::N + 1), kc.half);        // xft/hermite.py:87-89
      const double phi = __dmul_rn(rc.cin, __dmul_rn(x, x));                     // xft/kernel.py:102
      const double add = -(XFT_PI / Cfg::N) * (double)k;                         // p_k = (-1)^k e^{-i pi k/n}
      return cmul(unit_phase_tab(phi, add, (k & 1) << 7, tab), f);
    }
    return cmul(__ldg(&ptab[k]), f);
  }
  static __device__ __forceinline__ C post(C S, int jj, const Coef128& rc, const RowConst& kc, double2 cn,
                                           const C* __restrict__ ptab, const double2* tab) {
    if constexpr (Cfg::MODE == MODE_DFT) return S;
    if constexpr (Cfg::MODE == MODE_SCALED) return cmul(cn, cmul(__ldg(&ptab[jj]), S));
    if (rc.post) {
      const double x = __dmul_rn((double)(2 * jj - Cfg::N + 1), kc.half);
      const double y = __dmul_rn(rc.s4, x);                                       // xft/lct.py:196
      const double psi = __dmul_rn(rc.cout, __dmul_rn(y, y));                     // xft/kernel.py:113
      const double add = rc.gf - (XFT_PI / Cfg::N) * (double)jj;
      const double2 e = unit_phase_tab(psi, add, rc.gi + ((jj & 1) << 7), tab);
      return cmul(make_double2(e.x * rc.gabs, e.y * rc.gabs), S);
    }
    return cmul(cmul(rc.g, __ldg(&ptab[jj])), S);
  }
};

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
xft_pipe_kernel(const typename Cfg::C* __restrict__ in, typename Cfg::C* __restrict__ out, long long batch,
                const double* __restrict__ abcd, long long abcd_stride, Abcd uni, const typename Cfg::C* __restrict__ tw,
                const typename Cfg::C* __restrict__ ptab, const double2* __restrict__ gtab, double2 cn, RowConst kc) {
  using C = typename Cfg::C;
  using Coef = typename Cfg::Coef;
  constexpr int E = Cfg::E, TR = Cfg::TR, N = Cfg::N, ROWS = Cfg::ROWS, S = Cfg::STAGES;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t bars[S];
  __shared__ Coef coef[2][ROWS];

  C* stage0 = reinterpret_cast<C*>(xft_smem);
  double2* tab = reinterpret_cast<double2*>(xft_smem + size_t(S) * Cfg::TILE * sizeof(C));

  const int tid = threadIdx.x;
  const int lrow = tid / TR;
  const int j = tid - lrow * TR;
  const long long ntiles = (batch + ROWS - 1) / ROWS;
  const long long G = gridDim.x;

  auto tile_bytes = [&](long long t) -> uint32_t {
    const long long rows = batch - t * ROWS < ROWS ? batch - t * ROWS : ROWS;
    return (uint32_t)(rows * N * sizeof(C));
  };
  auto issue = [&](long long t, int st) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[st], tile_bytes(t));
    tma_load_1d(stage0 + size_t(st) * Cfg::TILE, in + t * Cfg::TILE, tile_bytes(t), &bars[st]);
  };
  auto coefs = [&](long long t, int slot) {
    if constexpr (Cfg::MODE == MODE_LCT) {
      if (tid < 32) {
        for (int r = tid; r < ROWS; r += 32) {
          const long long row = t * ROWS + r;
          if (row < batch) make_coef(coef[slot][r], abcd ? abcd + row * abcd_stride : nullptr, uni, kc);
        }
      }
    }
  };

  // ---- prologue ----
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if constexpr (Cfg::C128) {
    for (int m = tid; m < 256; m += Cfg::THREADS) tab[m] = gtab[m];
  }
  __syncthreads();
  long long tile = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S - 1; ++s)
      if (tile + s * G < ntiles) issue(tile + s * G, s);
    if (S == 1 && tile < ntiles) issue(tile, 0);
  }
  coefs(tile, 0);
  __syncthreads();

  for (int it = 0; tile < ntiles; ++it, tile += G) {
    const int st = it % S;
    mbar_wait(&bars[st], (uint32_t)((it / S) & 1));
    C* rs = stage0 + size_t(st) * Cfg::TILE + size_t(lrow) * N;
    const Coef& rc = coef[it & 1][lrow];

    C v[E];
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const int k = j + s * TR;
      v[s] = Chirp<Cfg>::pre(rs[k], k, rc, kc, ptab, tab);
    }

    auto hook = [&]() {
      if (S >= 2 && tid == 0) {
        const long long nt = tile + (S - 1) * G;
        if (nt < ntiles) issue(nt, (it + S - 1) % S);
      }
      coefs(tile + G, (it + 1) & 1);
    };
    pipe_passes<Cfg, 0>(v, rs, j, tw, hook);
    if constexpr (S == 1) {
      __syncthreads();
      if (tid == 0 && tile + G < ntiles) issue(tile + G, 0);
    }

    const long long row = tile * ROWS + lrow;
    if (row < batch) {
      C* dst = out + row * N;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int jj = j + s * TR;
        st_stream(dst + jj, Chirp<Cfg>::post(v[s], jj, rc, kc, cn, ptab, tab));
      }
    }
  }
}

}  // namespace xftb
