// C-ABI entry points (include/xft_b200.h) for the 1-D row transforms,
// validation, the host end-to-end pipeline, the transpose and the 2-D pass.
#include <array>
#include <cmath>
#include <cstdlib>
#include <map>
#include <atomic>
#include <mutex>
#include <cstring>
#include <utility>
#include <vector>

#include "../../include/xft_b200.h"
#include "xft_pipe.cuh"
#include "xft_internal.h"
#include "xft_tables.h"

using namespace xftb;

#ifndef XFT_LCT2D_LANES
#define XFT_LCT2D_LANES 4  // internal streams for the 8 slab column passes (1 = in order on the caller stream)
#endif
#ifndef XFT_LCT2D_SLABS
#define XFT_LCT2D_SLABS 1  // single-GPU 2-D: row pass into 8 column slabs, cluster columns slab -> natural
#endif

namespace {

constexpr int MAXLOG_C64 = 14;   // 16384 x 8 B = 128 KiB per row in shared memory
constexpr int MAXLOG_C128 = 13;  //  8192 x 16 B = 128 KiB

struct LaunchArgs {
  const void* in;
  void* out;
  long long batch;
  const double* abcd;
  long long stride;
  Abcd uni;
  Tables tb;
  int flags;
  cudaStream_t st;
  int seg_log2w = 0;        // segmented (all-to-all send) output layout
  long long seg_stride = 0;  // 0: natural rows
  PeerTable peers{};         // peer-store output (count > 0)
  unsigned long long* bad = nullptr;  // non-finite input report (xft_lct_checked)
};

// smallest row index holding a non-finite sample -> atomicMin(*bad): the
// stand-alone check for the row paths whose kernels do not fuse it (short rows,
// chirp-z, four-step); the pipelined row kernel checks inside its loads
template <class C>
__global__ void __launch_bounds__(256) nonfinite_rows_kernel(const C* __restrict__ in, long long batch, long long n,
                                                            unsigned long long* bad) {
  const long long total = batch * n;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    if (nonfinite_key(in[i]) == 0) atomicMin(bad, (unsigned long long)(i / n));
  }
}

int scan_nonfinite(const void* in, long long batch, long long n, int dtype, unsigned long long* bad, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (batch * n + 255) / 256;
  const unsigned grid = (unsigned)(want < 8ll * sms ? (want < 1 ? 1 : want) : 8ll * sms);
  if (dtype == XFT_C64)
    nonfinite_rows_kernel<float2><<<grid, 256, 0, st>>>(static_cast<const float2*>(in), batch, n, bad);
  else
    nonfinite_rows_kernel<double2><<<grid, 256, 0, st>>>(static_cast<const double2*>(in), batch, n, bad);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

using LaunchFn = int (*)(const LaunchArgs&);

// single-pass sizes (n <= radix): one register DFT per thread, no exchange
template <class C, int L, int MODE, int SIGN>
int launch_small(const LaunchArgs& a) {
  if (a.bad) {
    int rc = scan_nonfinite(a.in, a.batch, 1 << L, sizeof(C) == 8 ? XFT_C64 : XFT_C128, a.bad, a.st);
    if (rc) return rc;
  }
  using Cfg = RowCfg<C, L, (1 << L), MODE, SIGN>;
  auto kern = xft_rows_kernel<Cfg>;
  const long long grid = (a.batch + Cfg::ROWS - 1) / Cfg::ROWS;
  kern<<<(unsigned)grid, Cfg::THREADS, 0, a.st>>>(
      static_cast<const C*>(a.in), static_cast<C*>(a.out), a.batch, a.abcd, a.stride, a.uni,
      static_cast<const C*>(a.tb.tw), static_cast<const C*>(a.tb.ptab), a.tb.cn, a.tb.half, a.flags);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

// Shape of the pipelined kernel per (dtype, n): threads per CTA, resident CTAs
// per SM (register budget), ring depth.  Overridable at build time for tuning.
#ifndef XFT_C64_TARGET
#define XFT_C64_TARGET 256
#endif
#ifndef XFT_C64_MINB
#define XFT_C64_MINB 4
#endif
#ifndef XFT_C64_MAXST
#define XFT_C64_MAXST 1
#endif
#ifndef XFT_C128_TARGET
#define XFT_C128_TARGET 256
#endif
#ifndef XFT_C128_MINB
#define XFT_C128_MINB 2
#endif
#ifndef XFT_C128_MAXST
#define XFT_C128_MAXST 1
#endif
template <class C, int L>
struct PipeShape {
  static constexpr bool C64 = sizeof(C) == 8;
  static constexpr int E = pipe_radix(C64 ? XFT_C64 : XFT_C128, L);
  static constexpr int TR = (1 << L) / E;
  static constexpr int TARGET = C64 ? XFT_C64_TARGET : XFT_C128_TARGET;  // threads per CTA
  static constexpr int ROWS = TR >= TARGET ? 1 : (TARGET / TR > 64 ? 64 : TARGET / TR);
  // c64 rows up to 1024: two resident CTAs with a 3-deep ring measured best (cfg4); longer rows: 4 CTAs
  static constexpr int MINB0 = C64 ? (L <= 10 ? 2 : XFT_C64_MINB) : XFT_C128_MINB;
  static constexpr size_t TILE_BYTES = size_t(ROWS) * ((size_t(1) << L) + (size_t(1) << L) / 16) * sizeof(C);
  static constexpr size_t STATIC =
      (C64 ? (ROWS >= 128 ? ROWS : 128) * sizeof(Coef64)
           : (ROWS == 1 ? XFT_C128_CH : (ROWS >= 128 ? ROWS : 128)) * sizeof(Coef128)) + 256;
  static constexpr size_t TAB = C64 ? 0 : XFT_C128_TABCOPIES * C128_TABN * 16;
  // resident CTAs per SM: requested, capped by threads (2048/SM) and by one stage of smem
  static constexpr int MINB_T = 65536 / (TR * ROWS * 64);  // keep >= 64 registers per thread
  static constexpr int MINB_S = int((226 * 1024) / (TILE_BYTES + TAB + STATIC + 1024));
  static constexpr int MINB1 = MINB0 < MINB_T ? MINB0 : MINB_T;
  static constexpr int MINB = (MINB1 < MINB_S ? MINB1 : MINB_S) < 1 ? 1 : (MINB1 < MINB_S ? MINB1 : MINB_S);
  static constexpr size_t BUDGET = (226 * 1024) / MINB - 1024 - STATIC - TAB;
  static constexpr int MAXST = C64 ? (L <= 10 ? 3 : XFT_C64_MAXST) : XFT_C128_MAXST;
  static constexpr int STAGES = BUDGET / TILE_BYTES >= MAXST ? MAXST : (BUDGET / TILE_BYTES >= 2 ? 2 : 1);
};

template <class C, int L, int MODE, int SIGN>
int launch_pipe(const LaunchArgs& a) {
  using SH = PipeShape<C, L>;
  using Cfg = PipeCfg<C, L, SH::E, MODE, SIGN, SH::ROWS, SH::STAGES, SH::MINB, 1>;
  auto kern = xft_pipe_kernel<Cfg>;
  static std::atomic<int> occ_cache[64];  // resident CTAs x SMs per device (0 = not yet queried)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM) != cudaSuccess)
    return XFT_ECUDA;
#ifdef XFT_CARVEOUT
  {
    // smallest shared-memory carveout that holds MINB CTAs: the rest of the
    // 256 KB stays L1 for the (re-read every tile) twiddle table
    const int pct = XFT_CARVEOUT > 0 ? XFT_CARVEOUT
                                     : (int)((SH::MINB * (Cfg::SMEM + 4096) * 100 + 228 * 1024 - 1) / (228 * 1024));
    if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct > 100 ? 100 : pct) !=
        cudaSuccess)
      return XFT_ECUDA;
  }
#endif
  int occ = occ_cache[dev & 63].load(std::memory_order_relaxed);
  if (occ == 0) {  // idempotent: concurrent first calls compute and store the same value
    int o = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cfg::THREADS, Cfg::SMEM) != cudaSuccess)
      return XFT_ECUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return XFT_ECUDA;
    occ = (o < 1 ? 1 : o) * sms;
    occ_cache[dev & 63].store(occ, std::memory_order_relaxed);
  }
  const long long tiles = (a.batch + Cfg::ROWS - 1) / Cfg::ROWS;
  long long cap = occ;
#ifdef XFT_GRID_CAP_ENV  // tuning only: XFT_GRID_CAP[64|128]=<ctas> caps the persistent grid
  if (const char* e = getenv("XFT_GRID_CAP")) cap = atoll(e) < cap ? atoll(e) : cap;
  if (const char* e = getenv(sizeof(C) == 8 ? "XFT_GRID_CAP64" : "XFT_GRID_CAP128")) cap = atoll(e) < cap ? atoll(e) : cap;
#endif
  const long long grid = tiles < cap ? tiles : cap;
  RowConst kc;
  kc.half = a.tb.half;
  kc.cnabs = M_PI / std::sqrt(2.0 * double(1 << L));
  kc.cnred = (long long)(((__int128)((1 << L) - 1) * ((1 << L) - 1)) % (4 * (__int128)(1 << L)));
  kc.log2n = L;
  kc.flags = a.flags;
  kc.bad = a.bad;
  // programmatic stream serialization: the next launch's CTAs may start their
  // prologue while this grid's tail runs (the kernel waits before touching data)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = a.st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (sizeof(C) == 16 ? XFT_PDL_C128 : XFT_PDL_C64) ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<const C*>(a.in), static_cast<C*>(a.out), a.batch,
                                           a.abcd, (long long)a.stride, a.uni, static_cast<const C*>(a.tb.tw),
                                           static_cast<const C*>(a.tb.ptab), a.tb.gtab, a.tb.cn, kc, a.seg_log2w,
                                           a.seg_stride, a.peers);
  return e == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

template <class C, int L, int MODE, int SIGN>
int launch_rows(const LaunchArgs& a) {
  if constexpr ((1 << L) <= pipe_radix(sizeof(C) == 8 ? XFT_C64 : XFT_C128, L))
    return launch_small<C, L, MODE, SIGN>(a);
  else
    return launch_pipe<C, L, MODE, SIGN>(a);
}

template <class C, int MODE, int SIGN, int... Ls>
constexpr auto make_table(std::integer_sequence<int, Ls...>) {
  return std::array<LaunchFn, sizeof...(Ls)>{&launch_rows<C, Ls, MODE, SIGN>...};
}

template <class C, int MODE, int SIGN, int MAXL>
LaunchFn pick(int l) {
  static const auto tab = make_table<C, MODE, SIGN>(std::make_integer_sequence<int, MAXL + 1>{});
  return (l >= 0 && l <= MAXL) ? tab[l] : nullptr;
}

int log2_exact(int64_t n) {
  if (n < 1 || (n & (n - 1))) return -1;
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}

int run_rows(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, int dtype,
             const double* abcd, int64_t stride, Abcd uni, int flags, cudaStream_t st, int seg_log2w = 0,
             long long seg_stride = 0, const PeerTable* peers = nullptr, unsigned long long* bad = nullptr) {
  if (n < 1) return XFT_EINVALID_SIZE;
  if (batch < 0) return XFT_EINVALID_SIZE;
  if (dtype != XFT_C64 && dtype != XFT_C128) return XFT_EPARAM;
  if (batch == 0) return XFT_OK;
  const int l = log2_exact(n);
  if (bad && (l < 0 || l > (dtype == XFT_C64 ? MAXLOG_C64 : MAXLOG_C128))) {
    const int rc = scan_nonfinite(in, batch, n, dtype, bad, st);
    if (rc) return rc;
  }
  if (l < 0) {  // not a power of two: chirp-z route (xft/fftcore.py:84-100)
    const double u4[4] = {uni.a, uni.b, uni.c, uni.d};
    return run_chirpz(mode, sign, in, out, batch, n, dtype, abcd, stride, u4, flags, st);
  }
  if (l > (dtype == XFT_C64 ? MAXLOG_C64 : MAXLOG_C128)) {  // longer than one CTA: four-step path
    const double u4[4] = {uni.a, uni.b, uni.c, uni.d};
    return run_large_pow2(mode, sign, in, out, batch, n, dtype, abcd, stride, u4, flags, st);
  }
  if ((seg_stride || peers) && (1 << l) <= pipe_radix(dtype, l))
    return XFT_ENOTSUP;  // segmented / peer epilogues live in the pipelined row kernel
  LaunchArgs a{in, out, (long long)batch, abcd, (long long)stride, uni, {}, flags, st};
  a.bad = bad;
  a.seg_log2w = seg_log2w;
  a.seg_stride = seg_stride;
  if (seg_stride && (seg_log2w < 0 || seg_log2w > l || mode != MODE_LCT)) return XFT_EPARAM;
  if (peers) {
    if (mode != MODE_LCT || peers->count < 1 || peers->count > 8 || (int64_t(peers->count) << seg_log2w) != n)
      return XFT_EPARAM;
    a.peers = *peers;
  }
  int rc = get_tables(n, dtype, &a.tb);
  if (rc) return rc;
  LaunchFn fn = nullptr;
  if (dtype == XFT_C64) {
    if (mode == MODE_LCT) fn = pick<float2, MODE_LCT, -1, MAXLOG_C64>(l);
    else if (mode == MODE_SCALED) fn = pick<float2, MODE_SCALED, -1, MAXLOG_C64>(l);
    else fn = sign < 0 ? pick<float2, MODE_DFT, -1, MAXLOG_C64>(l) : pick<float2, MODE_DFT, 1, MAXLOG_C64>(l);
  } else {
    if (mode == MODE_LCT) fn = pick<double2, MODE_LCT, -1, MAXLOG_C128>(l);
    else if (mode == MODE_SCALED) fn = pick<double2, MODE_SCALED, -1, MAXLOG_C128>(l);
    else fn = sign < 0 ? pick<double2, MODE_DFT, -1, MAXLOG_C128>(l) : pick<double2, MODE_DFT, 1, MAXLOG_C128>(l);
  }
  if (!fn) return XFT_ENOTSUP;
  return fn(a);
}

// ---------------------------------------------------------------------------
// tiled transpose: out[c * ld_out + r] = in[r * ld_in + c]
// ---------------------------------------------------------------------------
template <class C, int TILE>
__global__ void __launch_bounds__(TILE * 8) transpose_kernel(const C* __restrict__ in, C* __restrict__ out,
                                                           long long rows, long long cols, long long ld_in,
                                                           long long ld_out) {
  __shared__ C tile[TILE][TILE + 1];
  const long long r0 = (long long)blockIdx.y * TILE, c0 = (long long)blockIdx.x * TILE;
  const int tx = threadIdx.x % TILE, ty = threadIdx.x / TILE;
#pragma unroll
  for (int k = ty; k < TILE; k += 8) {
    const long long r = r0 + k, c = c0 + tx;
    if (r < rows && c < cols) tile[k][tx] = in[r * ld_in + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = ty; k < TILE; k += 8) {
    const long long c = c0 + k, r = r0 + tx;
    if (r < rows && c < cols) out[c * ld_out + r] = tile[tx][k];
  }
}

template <class C>
int launch_transpose(const void* in, void* out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
                     cudaStream_t st) {
  constexpr int TILE = 32;
  dim3 grid((unsigned)((cols + TILE - 1) / TILE), (unsigned)((rows + TILE - 1) / TILE));
  transpose_kernel<C, TILE><<<grid, TILE * 8, 0, st>>>(static_cast<const C*>(in), static_cast<C*>(out), rows,
                                                      cols, ld_in, ld_out);
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

}  // namespace

#ifndef XFT_HOST_CHUNK_MB
#define XFT_HOST_CHUNK_MB 32  // host-path chunk (H2D / kernel / D2H pipeline granularity; A/B config-2 e2e step:
                              // 4: 11.9, 8: 10.1, 16: 9.7, 32: 9.4, 48: 9.6, 64: 10.1 ms)
#endif
namespace {
// persistent resources of the host-buffer path (xft_lct_host), one per device
struct HostPipe {
  static constexpr int NSLOT = 3;
  std::mutex mu;
  cudaStream_t st[NSLOT] = {};
  void* buf[NSLOT][2] = {};
  void* par[NSLOT] = {};
  size_t cap = 0, pcap = 0;
  int reserve(size_t bytes, size_t pbytes) {
    for (int s = 0; s < NSLOT; ++s)
      if (!st[s] && cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking) != cudaSuccess) return XFT_ECUDA;
    if (bytes > cap) {
      for (int s = 0; s < NSLOT; ++s) {
        if (cudaStreamSynchronize(st[s]) != cudaSuccess) return XFT_ECUDA;
        for (int h = 0; h < 2; ++h) {
          if (buf[s][h]) cudaFree(buf[s][h]);
          buf[s][h] = nullptr;
          if (cudaMalloc(&buf[s][h], bytes) != cudaSuccess) return XFT_ECUDA;
        }
      }
      cap = bytes;
    }
    if (pbytes > pcap) {
      for (int s = 0; s < NSLOT; ++s) {
        if (par[s]) cudaFree(par[s]);
        par[s] = nullptr;
        if (cudaMalloc(&par[s], pbytes) != cudaSuccess) return XFT_ECUDA;
      }
      pcap = pbytes;
    }
    return XFT_OK;
  }
};
// a pool of pipelines per device: concurrent host-buffer calls (e.g. a c64 and
// a c128 batch from two threads) each take their own streams and staging, so
// their PCIe transfers interleave instead of queueing behind one lock
struct PipeLease {
  HostPipe* p;
  std::unique_lock<std::mutex> lock;
};
PipeLease host_pipe(int dev) {
  static std::mutex m;
  static std::map<int, std::vector<HostPipe*>> pools;
  std::lock_guard<std::mutex> guard(m);
  auto& pool = pools[dev];
  for (HostPipe* p : pool) {
    std::unique_lock<std::mutex> l(p->mu, std::try_to_lock);
    if (l.owns_lock()) return PipeLease{p, std::move(l)};
  }
  pool.push_back(new HostPipe());
  return PipeLease{pool.back(), std::unique_lock<std::mutex>(pool.back()->mu)};
}
}  // namespace

extern "C" {

int xft_version(void) { return 100; }

int64_t xft_max_n(int dtype) { return int64_t(1) << 20; }  // four-step path beyond the in-CTA sizes

int xft_prepare(int64_t n, int dtype) {
  if (n < 1) return XFT_EINVALID_SIZE;
  if (log2_exact(n) < 0) return XFT_OK;  // chirp-z plans are built on first use
  if (n > xft_max_n(dtype)) return XFT_ENOTSUP;
  if (n > (int64_t(1) << (dtype == XFT_C64 ? MAXLOG_C64 : MAXLOG_C128))) return XFT_OK;  // four-step: built on use
  Tables tb;
  return get_tables(n, dtype, &tb);
}

int xft_validate_lct_params(const double* abcd, int64_t count, int64_t stride, int check_unimodular, double tol,
                            int64_t* bad_row) {
  const int64_t rows = stride == 0 ? (count > 0 ? 1 : 0) : count;
  for (int64_t r = 0; r < rows; ++r) {
    const double* p = abcd + r * stride;
    if (p[1] == 0.0) {  // xft/lct.py:187-190
      if (bad_row) *bad_row = r;
      return XFT_EDEGENERATE;
    }
  }
  if (check_unimodular) {
    for (int64_t r = 0; r < rows; ++r) {
      const double* p = abcd + r * stride;
      const double det = p[0] * p[3] - p[1] * p[2];  // LctParams.det, xft/lct.py:60-64
      if (!(std::fabs(det - 1.0) <= tol)) {          // xft/lct.py:66-71
        if (bad_row) *bad_row = r;
        return XFT_EPARAM;
      }
    }
  }
  return XFT_OK;
}

int xft_lct(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd, int64_t abcd_stride,
            int flags, void* stream) {
  return run_rows(MODE_LCT, -1, in, out, batch, n, dtype, abcd, abcd_stride, Abcd{0, 0, 0, 0}, flags,
                  static_cast<cudaStream_t>(stream));
}

int xft_lct_checked(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                    int64_t abcd_stride, int flags, int64_t* bad_row, void* stream) {
  if (!bad_row) return XFT_EPARAM;
  auto st = static_cast<cudaStream_t>(stream);
  // sentinel: INT64_MAX (no offending row); the kernels atomicMin row indices into it
  if (cudaMemsetAsync(bad_row, 0xff, sizeof(int64_t), st) != cudaSuccess) return XFT_ECUDA;
  if (cudaMemsetAsync(reinterpret_cast<char*>(bad_row) + 7, 0x7f, 1, st) != cudaSuccess) return XFT_ECUDA;
  return run_rows(MODE_LCT, -1, in, out, batch, n, dtype, abcd, abcd_stride, Abcd{0, 0, 0, 0}, flags, st, 0, 0,
                  nullptr, reinterpret_cast<unsigned long long*>(bad_row));
}

int xft_dft(const void* in, void* out, int64_t batch, int64_t n, int sign, int dtype, void* stream) {
  if (sign != 1 && sign != -1) return XFT_EPARAM;
  return run_rows(MODE_DFT, sign, in, out, batch, n, dtype, nullptr, 0, Abcd{0, 0, 0, 0}, 0,
                  static_cast<cudaStream_t>(stream));
}

int xft_scaled_fourier(const void* in, void* out, int64_t batch, int64_t n, int dtype, void* stream) {
  return run_rows(MODE_SCALED, -1, in, out, batch, n, dtype, nullptr, 0, Abcd{0, 0, 0, 0}, 0,
                  static_cast<cudaStream_t>(stream));
}

int xft_transpose(const void* in, void* out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out, int dtype,
                  void* stream) {
  if (rows < 0 || cols < 0) return XFT_EINVALID_SIZE;
  if (rows == 0 || cols == 0) return XFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  return dtype == XFT_C64 ? launch_transpose<float2>(in, out, rows, cols, ld_in, ld_out, st)
                          : launch_transpose<double2>(in, out, rows, cols, ld_in, ld_out, st);
}

int xft_lct2d(const void* in, void* out, int64_t n_rows, int64_t n_cols, int dtype, const double* abcd_row,
              const double* abcd_col, void* workspace, void* stream) {
  if (n_rows < 1 || n_cols < 1) return XFT_EINVALID_SIZE;
  int rc = xft_validate_lct_params(abcd_row, 1, 0, 1, 1e-10, nullptr);
  if (!rc) rc = xft_validate_lct_params(abcd_col, 1, 0, 1, 1e-10, nullptr);
  if (rc) return rc;
  auto st = static_cast<cudaStream_t>(stream);
  const Abcd ur{abcd_row[0], abcd_row[1], abcd_row[2], abcd_row[3]};
  const Abcd uc{abcd_col[0], abcd_col[1], abcd_col[2], abcd_col[3]};
  const size_t esz = dtype == XFT_C64 ? 8 : 16;
  // tall power-of-two fields: the row pass writes 8 column slabs [n_rows][n_cols/8]
  // (the sharded layout; 2 KB+ row segments) into the workspace, and the
  // cluster column kernel reads each narrow slab and writes its columns straight
  // into `out` (column kernel 1.99 -> 1.82 ms at 16384^2 c64: shorter rows)
  const int lr = log2_exact(n_rows), lc = log2_exact(n_cols);
  const int64_t nc = n_cols / 8;
  // (only where the cluster column kernel runs on this device: probed first, nothing launched)
  // (c64 fields 16384 .. 65536 rows high skip this: their columns run in place through the L2-staged path)
  if (workspace && XFT_LCT2D_SLABS && !lct_cols_ring_ok(out, n_rows, n_cols, n_cols, dtype) && lr >= 11 && lr <= 14 && lc >= 0 && lc <= (dtype == XFT_C64 ? MAXLOG_C64 : MAXLOG_C128) &&
      nc >= 256 && nc % 8 == 0 &&
      run_lct_cols_cluster(workspace, out, n_rows, nc, nc, n_cols, dtype, abcd_col, 0, st, true) == XFT_OK) {
    const int segl = log2_exact(nc);
    rc = run_rows(MODE_LCT, -1, in, workspace, n_rows, n_cols, dtype, nullptr, 0, ur, 0, st, segl, n_rows * nc);
    if (rc) return rc;
    // the 8 slabs are independent: internal streams (forked from / joined to
    // `st`) so one slab's column kernel starts on the SMs another's tail frees
    int dev = 0;
    cudaGetDevice(&dev);
    SideStreams& ss = side_streams(dev, st, XFT_LCT2D_LANES);
    if (!ss.ok) return XFT_ECUDA;
    std::lock_guard<std::mutex> lock(ss.mu);
    if (cudaEventRecord(ss.fork, st) != cudaSuccess) return XFT_ECUDA;
    int forked = 0;
    for (; forked < XFT_LCT2D_LANES; ++forked)
      if (cudaStreamWaitEvent(ss.st[forked], ss.fork, 0) != cudaSuccess) {
        rc = XFT_ECUDA;
        break;
      }
    for (int h = 0; h < 8 && !rc; ++h) {
      cudaStream_t sh = ss.st[h % XFT_LCT2D_LANES];
      const char* slab = static_cast<const char*>(workspace) + esz * (size_t)h * n_rows * nc;
      char* dst = static_cast<char*>(out) + esz * (size_t)h * nc;
      rc = run_lct_cols_cluster(slab, dst, n_rows, nc, nc, n_cols, dtype, abcd_col, 0, sh);
      if (rc == XFT_ENOTSUP) {
        // no cluster path on this device/shape (e.g. MIG/MPS, no 16-CTA clusters): the
        // two-pass column transform on the slab with its own [n_rows][nc] scratch (per
        // lane stream), then place the slab's columns into `out`
        void* cs = stream_scratch(dev, sh, esz * (size_t)n_rows * nc);
        rc = cs ? run_lct_cols(slab, const_cast<char*>(slab), cs, n_rows, nc, nc, dtype, abcd_col, 0, sh) : XFT_ECUDA;
        if (!rc && cudaMemcpy2DAsync(dst, esz * n_cols, slab, esz * nc, esz * nc, n_rows, cudaMemcpyDeviceToDevice,
                                     sh) != cudaSuccess)
          rc = XFT_ECUDA;
      }
    }
    for (int q = 0; q < forked; ++q)  // join every forked lane, also after an error (`st` stays consistent)
      if (cudaEventRecord(ss.join[q], ss.st[q]) != cudaSuccess || cudaStreamWaitEvent(st, ss.join[q], 0) != cudaSuccess)
        rc = rc ? rc : XFT_ECUDA;
    return rc;
  }
  // axis 1: rows (in -> out); axis 0: columns in place on `out` (workspace = four-step scratch)
  rc = run_rows(MODE_LCT, -1, in, out, n_rows, n_cols, dtype, nullptr, 0, ur, 0, st);
  if (rc) return rc;
  rc = run_lct_cols(out, out, workspace, n_rows, n_cols, n_cols, dtype, abcd_col, 0, st);
  if (rc != XFT_ENOTSUP) return rc;
  // other shapes: transpose, transform the (former) columns as rows, transpose back
  rc = xft_transpose(out, workspace, n_rows, n_cols, n_cols, n_rows, dtype, stream);
  if (!rc) rc = run_rows(MODE_LCT, -1, workspace, out, n_cols, n_rows, dtype, nullptr, 0, uc, 0, st);
  if (!rc) rc = xft_transpose(out, workspace, n_cols, n_rows, n_rows, n_cols, dtype, stream);
  if (!rc) {
    if (cudaMemcpyAsync(out, workspace, esz * n_rows * n_cols, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rc = XFT_ECUDA;
  }
  return rc;
}

int xft_lct_columns(const void* in, void* out, int64_t n_rows, int64_t n_cols, int64_t ld, int dtype,
                    const double* abcd_host, void* workspace, void* stream) {
  if (n_rows < 1 || n_cols < 1 || ld < n_cols) return XFT_EINVALID_SIZE;
  int rc = xft_validate_lct_params(abcd_host, 1, 0, 1, 1e-10, nullptr);
  if (rc) return rc;
  return run_lct_cols(in, out, workspace, n_rows, n_cols, ld, dtype, abcd_host, 0, static_cast<cudaStream_t>(stream));
}

int xft_column_schedule(int64_t n_rows, int64_t n_cols, int64_t index, int* tile, int* info) {
  return ring_schedule(n_rows, n_cols, index, tile, info);
}

int xft_lct_rows_packed(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd_host,
                        int seg_log2w, int64_t seg_stride, void* stream) {
  int rc = xft_validate_lct_params(abcd_host, 1, 0, 1, 1e-10, nullptr);
  if (rc) return rc;
  if (seg_log2w < 0 || seg_stride < (int64_t)batch << seg_log2w) return XFT_ESHAPE;
  const Abcd u{abcd_host[0], abcd_host[1], abcd_host[2], abcd_host[3]};
  return run_rows(MODE_LCT, -1, in, out, batch, n, dtype, nullptr, 0, u, 0, static_cast<cudaStream_t>(stream),
                  seg_log2w, seg_stride);
}

int xft_lct_rows_peers(const void* in, const uint64_t* peer_ptrs, int npeers, int64_t row0, int64_t batch, int64_t n,
                       int dtype, const double* abcd_host, void* stream) {
  int rc = xft_validate_lct_params(abcd_host, 1, 0, 1, 1e-10, nullptr);
  if (rc) return rc;
  if (npeers < 1 || npeers > 8 || n % npeers || row0 < 0) return XFT_ESHAPE;
  const int64_t nc = n / npeers;
  const int segl = log2_exact(nc);
  if (segl < 0) return XFT_ESHAPE;
  const int l = log2_exact(n);
  if (l < 0 || l > (dtype == XFT_C64 ? MAXLOG_C64 : MAXLOG_C128) || (1 << l) <= pipe_radix(dtype, l))
    return XFT_ENOTSUP;  // the peer epilogue lives in the pipelined row kernel
  PeerTable pt{};
  for (int h = 0; h < npeers; ++h) pt.p[h] = reinterpret_cast<void*>(static_cast<uintptr_t>(peer_ptrs[h]));
  pt.row0 = row0;
  pt.count = npeers;
  const Abcd u{abcd_host[0], abcd_host[1], abcd_host[2], abcd_host[3]};
  return run_rows(MODE_LCT, -1, in, nullptr, batch, n, dtype, nullptr, 0, u, 0, static_cast<cudaStream_t>(stream),
                  segl, 0, &pt);
}

int xft_lct_host(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                 int64_t abcd_stride, int flags, int check_unimodular, double tol) {
  if (n < 1 || batch < 0) return XFT_EINVALID_SIZE;
  if (dtype != XFT_C64 && dtype != XFT_C128) return XFT_EPARAM;
  if (log2_exact(n) >= 0 && n > xft_max_n(dtype)) return XFT_ENOTSUP;
  int rc = xft_validate_lct_params(abcd, batch, abcd_stride, check_unimodular, tol, nullptr);
  if (rc) return rc;
  if (batch == 0) return XFT_OK;
  rc = xft_prepare(n, dtype);
  if (rc) return rc;
  const size_t esz = dtype == XFT_C64 ? 8 : 16;
  const size_t row_bytes = esz * (size_t)n;
  // chunk ~ XFT_HOST_CHUNK_MB, at least one row; 3 slots rotate over 3 streams so the
  // H2D of chunk c+1, the kernel of chunk c and the D2H of chunk c-1 overlap.
  int64_t chunk = (int64_t)(((size_t)XFT_HOST_CHUNK_MB << 20) / row_bytes);
  if (chunk < 1) chunk = 1;
  if (chunk > batch) chunk = batch;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  // per-device persistent streams and staging buffers (grown on demand, never
  // freed): no allocation, stream creation or pool trimming inside the call
  PipeLease lease = host_pipe(dev);  // held for the call
  HostPipe& hp = *lease.p;
  rc = hp.reserve(row_bytes * (size_t)chunk, abcd_stride ? sizeof(double) * abcd_stride * (size_t)chunk : 0);
  if (rc) return rc;
  const Abcd uni = abcd_stride ? Abcd{0, 0, 0, 0} : Abcd{abcd[0], abcd[1], abcd[2], abcd[3]};
  for (int64_t r0 = 0, c = 0; r0 < batch && !rc; r0 += chunk, ++c) {
    const int s = (int)(c % HostPipe::NSLOT);
    const int64_t rows = (batch - r0 < chunk) ? batch - r0 : chunk;
    const char* hin = static_cast<const char*>(in) + row_bytes * r0;
    char* hout = static_cast<char*>(out) + row_bytes * r0;
    cudaStream_t st = hp.st[s];
    if (cudaMemcpyAsync(hp.buf[s][0], hin, row_bytes * rows, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      rc = XFT_ECUDA;
      break;
    }
    const double* dp = nullptr;
    if (abcd_stride) {
      if (cudaMemcpyAsync(hp.par[s], abcd + abcd_stride * r0, sizeof(double) * abcd_stride * rows,
                          cudaMemcpyHostToDevice, st) != cudaSuccess) {
        rc = XFT_ECUDA;
        break;
      }
      dp = static_cast<const double*>(hp.par[s]);
    }
    rc = run_rows(MODE_LCT, -1, hp.buf[s][0], hp.buf[s][1], rows, n, dtype, dp, abcd_stride, uni, flags, st);
    if (rc) break;
    if (cudaMemcpyAsync(hout, hp.buf[s][1], row_bytes * rows, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = XFT_ECUDA;
  }
  for (int s = 0; s < HostPipe::NSLOT; ++s)
    if (cudaStreamSynchronize(hp.st[s]) != cudaSuccess && !rc) rc = XFT_ECUDA;
  return rc;
}


int xft_validate_mehler_z(const double* z, int64_t count, int64_t stride, int64_t* bad_row) {
  const int64_t rows = stride == 0 ? (count > 0 ? 1 : 0) : count;
  for (int64_t r = 0; r < rows; ++r) {
    const double zr = z[r * stride], zi = z[r * stride + 1];
    if (std::hypot(zr, zi) > 1.0 + 1e-12) {  // FrftOrder, xft/dense.py:57-58
      if (bad_row) *bad_row = r;
      return XFT_EPARAM;
    }
    if (std::hypot(zr - 1.0, zi) < 1e-14 || std::hypot(zr + 1.0, zi) < 1e-14) {  // xft/dense.py:129-130
      if (bad_row) *bad_row = r;
      return XFT_ESINGULAR;
    }
  }
  return XFT_OK;
}


}  // extern "C"
