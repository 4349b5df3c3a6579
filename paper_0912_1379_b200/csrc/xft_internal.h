// Internal entry points shared between the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <vector>

namespace xftb {

struct Abcd;

// internal streams of a call on caller stream `caller` (fork/join events),
// created once per (device, caller stream) and grown to `count`; independent
// pieces of one call run concurrently and are joined back before it returns
struct SideStreams {
  std::mutex mu;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> join;
  cudaEvent_t fork = nullptr;
  bool ok = true;
};
SideStreams& side_streams(int dev, cudaStream_t caller, int count);

// per-(device, stream) scratch of at least `bytes`, grown on demand; superseded
// buffers are retired (kept alive until xft_release_caches), never freed under
// queued work; legal during stream capture.  nullptr on allocation failure.
void* stream_scratch(int dev, cudaStream_t st, size_t bytes);

// chirp-z route for lengths that are not powers of two (xft_bluestein.cu);
// mode: 0 DFT (sign), 1 scaled Fourier, 2 LCT.  abcd: device, stride 0|4.
int run_chirpz(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
               int64_t stride, const double* uni4, int flags, cudaStream_t st);

// largest M (power of two) the in-CTA chirp-z kernel handles for dtype
int64_t chirpz_max_m(int dtype);

// four-step path (xft_large.cu) for rows longer than the in-CTA kernels
int run_large_pow2(int mode, int sign, const void* in, void* out, int64_t batch, int64_t n, int dtype,
                   const double* abcd, int64_t stride, const double* uni4, int flags, cudaStream_t st);
// chirp-z route beyond the in-CTA sizes (xft_large.cu): the same convolution as
// run_chirpz (pre/post multipliers and the natural-order filter spectrum of
// its plan, convolution length m = 2^l) through the four-step tile passes
int run_large_chirpz(int lct, int bare, const void* in, void* out, int64_t batch, int64_t n, int dtype,
                     const double* abcd, int64_t stride, const double* uni4, const void* pre, const void* post,
                     const void* hspec, int64_t m, cudaStream_t st);
struct OpMehlerRow;
int run_large_mehler(const void* in, void* out, long long rows, const int* rowlist, const OpMehlerRow* prm, int l,
                     int64_t n, cudaStream_t st, void* scratch, const void* hspec);
// plan time: the permuted kernel spectra of a four-step Mehler class ([rows][2^l] double2)
int large_mehler_spectrum(long long rows, const int* rowlist, const OpMehlerRow* prm, int l, void* hs_out,
                          cudaStream_t st);

// column LCT of a [R][ncols] slab with row stride ld (xft_large.cu); abcd on the host.
// ws: scratch of R*ld elements when R > 1024.
int run_lct_cols(const void* in, void* out, void* ws, int64_t R, int64_t ncols, int64_t ld, int dtype,
                 const double* abcd_host, int flags, cudaStream_t st);
// true when run_lct_cols takes the L2-staged one-round-trip path (K7, xft_colring.cuh) for this shape
bool lct_cols_ring_ok(const void* in, int64_t R, int64_t ncols, int64_t ld, int dtype);
// the K7 tile schedule, host side (xft_column_schedule)
int ring_schedule(int64_t R, int64_t ncols, int64_t index, int* out, int* info);
// the cluster (one HBM round trip) column kernel alone, with a separate output row stride;
// probe = true checks that the kernel can run this shape on this device (cluster
// occupancy, tensor-map encoding) and launches nothing
int run_lct_cols_cluster(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, int64_t ld_out, int dtype,
                         const double* abcd_host, int flags, cudaStream_t st, bool probe = false);

}  // namespace xftb
