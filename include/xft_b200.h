/* xft_b200.h -- C ABI of the B200-native XFT fast linear canonical transform.
 *
 * Drop-in boundary for the reference's hot path (reference = the pure-Python
 * `xft` package, /root/reference/pkg/src/xft).  Every entry point takes plain
 * pointers and sizes; no torch / CUDA C++ types cross the boundary (streams
 * are passed as `void*` = cudaStream_t, NULL = legacy default stream).
 *
 * Conventions (all fixed by the reference):
 *   grid      x_k = (2k - n + 1) * pi / (2 sqrt(2n))          xft/hermite.py:80-89
 *   DFT       out[j] = sum_k e^{sign 2 pi i jk/n} in[k]        xft/fftcore.py:1-8
 *   LCT       out[j] = C(n) p_j e^{i psi_j}/sqrt(2 pi i b) DFT(p_k e^{i phi_k} in[k])[j]
 *             with DFT_SIGN = -1                                xft/lct.py:168-208
 *   output nodes y_j = 4 b x_j / pi (not materialised; see xft_output_nodes)
 *
 * Layout: `batch` contiguous rows of `n` complex samples, interleaved
 * (re, im) pairs -- complex64 = 2 x float32, complex128 = 2 x float64 --
 * i.e. the memory layout of numpy/torch complex arrays.  Out-of-place; the
 * input is never written (reference contract xft/fftcore.py:113).
 *
 * Alignment: device (and host) data pointers must be 16-byte aligned (the row
 * kernels move rows with cp.async.bulk); the Python layer copies misaligned
 * views to an aligned buffer before calling.
 *
 * Status codes mirror the reference exception classes (xft/errors.py:4-49).
 * Device entry points are stream-ordered and never synchronise the host;
 * parameters passed through device memory are assumed pre-validated (call
 * xft_validate_lct_params on the host copy, as the Python layer does).
 *
 * Threading (reference contract: xft/fftcore.py:8-11, pkg/tests/test_fftcore.py:
 * 97-148): all entry points are thread-safe and reentrant; identical inputs give
 * bit-identical outputs on any thread.  Global state, all behind locks:
 *   - immutable per-(device, n, dtype) twiddle/phase tables and chirp-z plans,
 *     built once on first use and kept for the process lifetime;
 *   - the implicit Mehler plan cache of xft_mehler (exact-z keyed, LRU of 64;
 *     evicted plans are retired, not freed) and per-(device, stream) scratch
 *     (growth retires the old buffer).  Retired memory may still be referenced
 *     by a CUDA graph captured earlier, so it is released only by
 *     xft_release_caches().  Callers that capture graphs around xft_mehler can
 *     instead own their plan (xft_mehler_plan_create / _destroy).
 * CUDA-graph capture: every device entry point is capturable once its tables
 * exist (call it once, or xft_prepare, before capture).
 */
#ifndef XFT_B200_H
#define XFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception class in brackets) ---------------- */
#define XFT_OK 0
#define XFT_EINVALID_SIZE 1  /* [InvalidSizeError]        xft/errors.py:8   */
#define XFT_EPARAM 2         /* [ParameterError]          xft/errors.py:12  */
#define XFT_ESINGULAR 3      /* [SingularParameterError]  xft/errors.py:16  */
#define XFT_EDEGENERATE 4    /* [DegenerateParameterError] xft/errors.py:20 */
#define XFT_EBRANCH 5        /* [UnsupportedBranchError]  xft/errors.py:25  */
#define XFT_ESHAPE 6         /* [ShapeError]              xft/errors.py:29  */
#define XFT_EGRID 7          /* [GridMismatchError]       xft/errors.py:33  */
#define XFT_ECUDA 8          /* CUDA runtime failure (no reference analogue) */
#define XFT_ENOTSUP 9        /* size/dtype combination not built           */

/* ---- element types ----------------------------------------------------------- */
#define XFT_C64 0   /* complex64: float32 (re, im)  */
#define XFT_C128 1  /* complex128: float64 (re, im) */

/* ---- flags --------------------------------------------------------------------- */
#define XFT_FLAG_BARE_FOURIER 1 /* multiply by sqrt(2 pi i): xft_fourier, xft/lct.py:211-223 */

/* Library version (major*10000 + minor*100 + patch). */
int xft_version(void);

/* Largest power-of-two row length the row entry points accept for dtype
 * (2^20: in-CTA kernels up to 2^14 c64 / 2^13 c128, four-step tile passes
 * beyond).  Other lengths take the chirp-z route (xft/fftcore.py:84-100) up to
 * a convolution length of 2^20, i.e. n <= 524288. */
int64_t xft_max_n(int dtype);

/* Build (once) the immutable tables for (current device, n, dtype).  Must be
 * called outside CUDA-graph capture; the transform entry points call it
 * lazily otherwise.  Replaces the plan construction of DftPlan.__init__ /
 * plan_dft (xft/fftcore.py:73-105). */
int xft_prepare(int64_t n, int dtype);

/* Host-side validation of LCT parameters in the reference's order:
 *   b == 0                        -> XFT_EDEGENERATE   (xft/lct.py:187-190)
 *   |ad - bc - 1| > tol (check=1) -> XFT_EPARAM        (xft/lct.py:191-192, 66-71)
 * abcd: host array of `count` rows of 4 doubles with row stride `stride`
 * (0 = one quadruple shared by all rows).  On failure *bad_row (if non-NULL)
 * receives the first offending row. */
int xft_validate_lct_params(const double* abcd, int64_t count, int64_t stride, int check_unimodular,
                            double tol, int64_t* bad_row);

/* Batched fast LCT (device pointers).  Replaces fast_lct (xft/lct.py:168-208),
 * fast_frft (226-233) and, with XFT_FLAG_BARE_FOURIER, xft_fourier (211-223).
 *   in, out   : device, batch x n complex (dtype)
 *   abcd      : device, per-row (a,b,c,d) doubles, row stride abcd_stride
 *               (4 = per-row parameters, 0 = one quadruple for all rows)
 *   stream    : cudaStream_t */
int xft_lct(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
            int64_t abcd_stride, int flags, void* stream);

/* xft_lct plus the reference's finite-input check (Signal, xft/lct.py:125-126) fused
 * into the row kernel's loads (no extra HBM pass on the pipelined path; the short-row,
 * chirp-z and four-step paths scan first): *bad_row (DEVICE int64) receives the
 * smallest row index holding an Inf/NaN sample, or INT64_MAX if every row is finite.
 * Stream-ordered: read it after the stream has reached this point.  The transform
 * itself runs either way (rows with non-finite input give non-finite output). */
int xft_lct_checked(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                    int64_t abcd_stride, int flags, int64_t* bad_row, void* stream);

/* Batched unnormalised DFT, sign = +1 or -1 (device pointers).
 * Replaces apply_dft(plan_dft(n, sign), v) (xft/fftcore.py:103-119). */
int xft_dft(const void* in, void* out, int64_t batch, int64_t n, int sign, int dtype, void* stream);

/* Batched scaled Fourier kernel F v = C(n) p * DFT(p * v) (device pointers).
 * Replaces apply_scaled_fourier (xft/kernel.py:83-95). */
int xft_scaled_fourier(const void* in, void* out, int64_t batch, int64_t n, int dtype, void* stream);

/* End-to-end LCT on HOST buffers: validates abcd (host, reference order),
 * streams the batch through the device in chunks (H2D / kernel / D2H
 * overlapped on the library's own streams) and returns when `out` holds
 * the result.  Pinned host buffers give full link bandwidth; pageable
 * buffers work but stage through the driver.  The call a reference-side
 * ctypes/cffi binding makes. */
int xft_lct_host(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                 int64_t abcd_stride, int flags, int check_unimodular, double tol);

/* Complex-z fractional transform through the Mehler kernel (in/out: device):
 *   out_j = dx sqrt(2/(1-z^2)) sum_k exp(-((1+z^2)(x_j^2+x_k^2) - 4 x_j x_k z) / (2(1-z^2))) in_k
 * i.e. frft_matrix_asymptotic(n, FrftOrder(z)).apply(in) (xft/dense.py:122-151,
 * 76-80) evaluated in O(n log n) as a windowed Bluestein convolution.
 * z: HOST array of batch (re, im) pairs (z_stride 2) or one pair (z_stride 0);
 * it is validated here (|z| <= 1 + 1e-12, |z -+ 1| >= 1e-14: XFT_EPARAM /
 * XFT_ESINGULAR, as FrftOrder / mehler_kernel).  complex128 only (the 1e-12
 * tolerance needs fp64).  `workspace`: device scratch of
 * xft_mehler_workspace_bytes(batch, n) bytes, or NULL to allocate on `stream`. */
int64_t xft_mehler_workspace_bytes(int64_t batch, int64_t n);
int xft_mehler(const void* in, void* out, int64_t batch, int64_t n, const double* z, int64_t z_stride,
               void* workspace, void* stream);
/* Host check of z values (FrftOrder / mehler_kernel, xft/dense.py:49-59, 127-130). */
int xft_validate_mehler_z(const double* z, int64_t count, int64_t stride, int64_t* bad_row);

/* Caller-owned Mehler plan for one z array on the current device (the
 * analogue of holding frft_matrix_asymptotic's DenseTransform,
 * xft/dense.py:139-151): per-row parameters, size classes, row lists and every
 * row's kernel spectrum FFT(h) (a function of z alone; sum over rows of M * 16
 * bytes, M = the row's windowed convolution length <= 2^ceil(log2(2n-1))),
 * built once on a private stream (validated like xft_mehler).  xft_mehler_planned applies it to a
 * [batch][n] complex128 batch (workspace as xft_mehler).  A plan is immutable and
 * may be used from several threads/streams at once; destroy it only when no
 * pending work or live CUDA graph uses it. */
int xft_mehler_plan_create(int64_t batch, int64_t n, const double* z, int64_t z_stride, void** plan);
int xft_mehler_planned(const void* in, void* out, const void* plan, void* workspace, void* stream);
int xft_mehler_plan_destroy(void* plan);

/* Releases the implicit Mehler plan cache, retired plans and the internal
 * per-stream scratch buffers.  The caller guarantees that no pending work and
 * no live CUDA graph references them (e.g. after cudaDeviceSynchronize and
 * destroying graphs captured around xft_mehler / xft_lct2d). */
int xft_release_caches(void);

/* Separable 2-D LCT on one device: fast LCT along rows (abcd_row, host) then
 * along columns (abcd_col, host) of an n_rows x n_cols field (device in/out).
 * `workspace`: device scratch of n_rows*n_cols complex elements (dtype).
 * Composition of fast_lct along axis 1 then axis 0 (no reference symbol;
 * SURVEY 8(a) last row). */
int xft_lct2d(const void* in, void* out, int64_t n_rows, int64_t n_cols, int dtype, const double* abcd_row,
              const double* abcd_col, void* workspace, void* stream);

/* Sharded separable 2-D LCT over NCCL: the calling rank holds rows
 * [g n/G, (g+1) n/G) of an n x n field (`local`, device, rows_local = n/G rows).  Row LCT
 * into the all-to-all send layout (`send`: device [G][rows_local][n/G]), one all-to-all
 * over the caller's NCCL communicator (`nccl_comm` = an ncclComm_t; grouped
 * ncclSend/ncclRecv on `stream`), then the column LCT of the received row-major
 * [n][n/G] slab in place (`slab`, device; `workspace`: n*n/G elements or NULL).
 * The result stays column-sharded: `slab` holds columns [g n/G, (g+1) n/G) of the
 * 2-D transform.  nccl_comm == NULL: one rank, no exchange (send unused).  n/G a power of two.
 * NCCL is resolved at run time from the caller's process (no link dependency).
 * Composition of fast_lct (xft/lct.py:168-208) along both axes. */
int xft_lct2d_sharded(const void* local, void* slab, void* send, int64_t rows_local, int64_t n, int dtype,
                      const double* abcd_row, const double* abcd_col, void* nccl_comm, void* workspace,
                      void* stream);
/* The NCCL library xft_lct2d_sharded resolved in this process: its file path
 * (path_len bytes incl. NUL) and ncclGetVersion code.  XFT_ENOTSUP: none loaded. */
int xft_nccl_info(char* path, int path_len, int* version);

/* Column LCT of a [n_rows][n_cols] slab with row stride ld (device in/out,
 * abcd on the host): the second axis of the separable 2-D LCT and the receive
 * side of the sharded 2-D transform.  In place allowed.  `workspace`: n_rows*ld
 * elements (used when n_rows > 1024).  n_rows: power of two >= 64. */
int xft_lct_columns(const void* in, void* out, int64_t n_rows, int64_t n_cols, int64_t ld, int dtype,
                    const double* abcd_host, void* workspace, void* stream);

/* Diagnostics (host only, no device work): the tile schedule of the c64 column kernel that
 * xft_lct_columns / xft_lct2d use for 16384 <= n_rows <= 65536 (two four-step passes through a
 * scratch ring that stays in L2).  tile (5 ints, may be NULL) = {pass 0|1 (2: past the end),
 * super-block, column block, line index inside the pass, ring slot} of tile `index`;
 * info (6 ints, may be NULL) = {tiles, super-blocks, lag, ring slots, tiles per pass-1 and per
 * pass-2 block-phase}.  A tile may only depend on tiles with a smaller index: pass 2 of a
 * super-block on all of its pass-1 tiles, pass 1 of super-block s on all pass-2 tiles of
 * s - slots (the ring slot it overwrites); tests/test_native_cpu.py checks exactly that.
 * XFT_ENOTSUP for shapes the kernel does not take. */
int xft_column_schedule(int64_t n_rows, int64_t n_cols, int64_t index, int* tile, int* info);

/* Row LCT (one quadruple, host) written in the all-to-all send layout of the
 * sharded 2-D transform: segment g (2^seg_log2w samples) of row r is stored at
 * out + g*seg_stride + r*2^seg_log2w (seg_stride >= batch * 2^seg_log2w). */
int xft_lct_rows_packed(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd_host,
                        int seg_log2w, int64_t seg_stride, void* stream);

/* Row LCT (one quadruple, host) whose epilogue stores segment h (n/npeers
 * samples) of local row r straight into peer buffer h at row row0 + r, i.e.
 * peer_ptrs[h] + (row0 + r) * n/npeers: the all-to-all of the sharded 2-D
 * transform done by the row kernel's own stores over NVLink (peer_ptrs: device
 * addresses valid in this process, e.g. symmetric-memory / IPC mappings; host
 * array of npeers <= 8).  The caller synchronises the ranks before reading the
 * peer buffers.  n a power of two, 32 <= n <= in-CTA limit, npeers | n. */
int xft_lct_rows_peers(const void* in, const uint64_t* peer_ptrs, int npeers, int64_t row0, int64_t batch, int64_t n,
                       int dtype, const double* abcd_host, void* stream);

/* Composed transform in one launch (device in/out, parameters on the host):
 * out = scale * R(L_{nst} ... L_2 L_1 in), 1 <= nst <= 4, each stage reading the
 * previous stage's output as samples on the standard grid; R reverses the
 * sample order when `reverse`.  The CLI inverse round trip of the reference
 * (xft/cli.py:236-253) is nst = 2 with the scale-adjusted inverse, scale =
 * sqrt(4b/pi), reverse = 1.  Power-of-two n, 32 <= n <= in-CTA limit. */
int xft_lct_chain(const void* in, void* out, int64_t batch, int64_t n, int dtype, const double* abcd_host, int nst,
                  double scale, int reverse, void* stream);

/* b = 0 branch (xft/lct.py:236-263), batched: out = sqrt(d) exp(i c d y^2/2) samples,
 * y the grid nodes, samples = f(d y) supplied by the caller (device), abcd device
 * (stride 0|4).  Host validation (b = 0, ad = 1, d > 0) in xft_validate_b_zero. */
int xft_lct_b_zero(const void* samples, void* out, int64_t batch, int64_t n, int dtype, const double* abcd,
                   int64_t abcd_stride, void* stream);
int xft_validate_b_zero(const double* abcd, int64_t count, int64_t stride, double tol, int64_t* bad_row);

/* ---- dense O(n^2) oracles on the GPU, complex128 only ----
 * Independent, entry-by-entry evaluations of the reference's dense matrices
 * (no FFT): applied matrix-free to [batch][n] vectors (any n), or materialised
 * as [n][n] row-major (n <= 4096, xft/dense.py:44 MAX_DENSE_N). */
/* out = L in, L = dense_lct_matrix(n, abcd) (xft/dense.py:230-249); abcd == NULL: the
 * scaled Fourier matrix F (xft/kernel.py:68-80).  abcd on the host. */
int xft_dense_lct_apply(const void* in, void* out, int64_t batch, int64_t n, const double* abcd_host, void* stream);
/* out[j] = sum_k e^{sign 2 pi i (jk mod n)/n} in[k], the quadratic-time DFT oracle; replaces
 * naive_dft (xft/fftcore.py:122-137): sign +-1 (else XFT_EPARAM), 1 <= n <= 4096 (else
 * XFT_EINVALID_SIZE, the reference's _NAIVE_CAP). */
int xft_naive_dft(const void* in, void* out, int64_t batch, int64_t n, int sign, void* stream);
/* out = (K_z(x_j, x_k) dx) in, frft_matrix_asymptotic (xft/dense.py:122-151); z host (stride 0|2). */
int xft_dense_mehler_apply(const void* in, void* out, int64_t batch, int64_t n, const double* z_host,
                           int64_t z_stride, void* stream);
/* [n][n] entries: kind 0 = F, 1 = L (param = abcd), 2 = Mehler (param = z re, im). */
int xft_dense_entries(void* out, int64_t n, int kind, const double* param_host, void* stream);

/* Tiled transpose used by the 2-D pass and the sharded all-to-all layout:
 * out[c * ld_out + r] = in[r * ld_in + c] for r < rows, c < cols. */
int xft_transpose(const void* in, void* out, int64_t rows, int64_t cols, int64_t ld_in, int64_t ld_out,
                  int dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XFT_B200_H */
