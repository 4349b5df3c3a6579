// Immutable per-(device, n, dtype) device tables -- the B200 analogue of an
// xft DftPlan (xft/fftcore.py:57-105): built once on the host, uploaded once,
// shared read-only by every launch and every host thread.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace xftb {

// Radix (elements per thread) of the pipelined kernel for (dtype, log2 n);
// shared by the host table builder and the kernel instantiation.
#ifndef XFT_C64_E10
#define XFT_C64_E10 32  // radix of the n = 512, 1024 c64 rows: 32 = two passes, one exchange (cfg4 232 -> 191 us)
#endif
#ifndef XFT_C64_E14
#define XFT_C64_E14 32  // radix of the n = 16384 c64 rows (16: 1024 threads, 4 passes)
#endif
#ifndef XFT_C128_E
#define XFT_C128_E 16
#endif
// log2 of the c128 chirp phasor table size (tab[m] = e^{2 pi i m / 2^TABL})
#ifndef XFT_C128_TABL
#define XFT_C128_TABL 8
#endif
constexpr int C128_TABN = 1 << XFT_C128_TABL;
constexpr int pipe_radix(int dtype, int l) {
  return dtype == 0 ? (l >= 14 ? XFT_C64_E14 : (l == 9 || l == 10) ? XFT_C64_E10 : 16) : (l >= 13 ? 16 : XFT_C128_E);
}

struct Tables {
  const void* tw = nullptr;    // pass-major twiddles of the pipelined kernel (see xft_pipe.cuh)
  const void* ptab = nullptr;  // n entries p_k = e^{i pi ((n-1)k mod 2n)/n}  (xft/kernel.py:51-65)
  const void* gtab = nullptr;  // C128_TABN entries e^{2 pi i m/C128_TABN} (c128 chirp table)
  double2 cn{0.0, 0.0};        // C(n)                                    (xft/kernel.py:45-48)
  double half = 0.0;           // (pi / sqrt(2n)) / 2                     (xft/hermite.py:74-89)
};

// Returns 0 and fills *out, or an XFT_E* status.  Thread-safe.
int get_tables(int64_t n, int dtype, Tables* out, int radix = -1);

// radix of the in-CTA chirp-z kernels for an FFT of length 2^l
#ifndef XFT_BLUE_E13
#define XFT_BLUE_E13 16  // radix of the c128 M = 8192 chirp-z / Mehler CTA (32: 256 threads)
#endif
#ifndef XFT_BLUE_E12
#define XFT_BLUE_E12 8  // radix of the c128 M = 4096 chirp-z / Mehler CTA (8: 512 threads, no spills; cfg3 0.344 -> 0.338 ms)
#endif
constexpr int blue_radix(int dtype, int l) {
  return (dtype == 1 && l == 13) ? XFT_BLUE_E13
         : (dtype == 1 && l == 12) ? XFT_BLUE_E12
         : pipe_radix(dtype, l) < (1 << (l - 1)) ? pipe_radix(dtype, l) : (1 << (l - 1));
}

// Host formulas shared with the C-ABI.
double2 host_kernel_prefactor(int64_t n);
double host_half_step(int64_t n);

}  // namespace xftb
