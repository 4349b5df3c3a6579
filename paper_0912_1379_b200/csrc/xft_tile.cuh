// Tiled strided FFT kernel: the building block of the four-step path for rows
// longer than one CTA's shared memory (M = M1 * M2 > in-CTA limit).
//
// A tile is W "lines" of length L = 2^LOGL.  A line is either a row segment
// (elements contiguous, lines L apart: LOAD/STORE_COL = false) or a column of
// a [M1][M2] row-major matrix (elements M2 apart, lines adjacent: *_COL = true),
// so every warp access moves W (column) or 32 (row) contiguous elements.  The
// FFT of each line runs in registers + the swizzled exchange buffer exactly as
// in the row kernels; when the load and store layouts differ the results are
// re-staged through shared memory so both sides stay coalesced.
//
// The operator supplies the addressing and the fused elementwise work:
//   C    Op::load (tile, line, a)          input sample a of the line (pre-multiplied)
//   void Op::store(tile, line, a, C v)     output sample a of the line
//   C    Op::mid  (tile, line, a, C v)     optional: between a forward and an
//                                          inverse FFT (Op::MID = true)
#pragma once
#include <type_traits>

#include "xft_pipe.cuh"

#ifndef XFT_TILE_PREFETCH
#define XFT_TILE_PREFETCH 0
#endif

namespace xftb {

// optional whole-line hooks of an operator: op.load_line<E, TR>(tile, w, j, v)
// (Op::LOAD_LINE) / op.store_line<E, TR>(tile, w, j, v) (Op::STORE_LINE) see all
// E samples j + s TR of a thread at once (generators that walk a quadratic
// phase across s)
template <class Op, class = void>
struct HasLoadLine : std::false_type {};
template <class Op>
struct HasLoadLine<Op, std::void_t<decltype(Op::LOAD_LINE)>> : std::bool_constant<Op::LOAD_LINE> {};
template <class Op, class = void>
struct HasStoreLine : std::false_type {};
template <class Op>
struct HasStoreLine<Op, std::void_t<decltype(Op::STORE_LINE)>> : std::bool_constant<Op::STORE_LINE> {};

template <class C, int LOGL, int E, int W, bool LOAD_COL, bool STORE_COL, int SIGN, class Op>
__global__ void __launch_bounds__(W*((1 << LOGL) / E))
xft_tile_kernel(long long ntiles, Op op, const C* __restrict__ tw) {
  constexpr int L = 1 << LOGL, TR = L / E;
  using Fwd = PipeCfg<C, LOGL, E, MODE_DFT, SIGN, W, 1, 1>;
  using Inv = PipeCfg<C, LOGL, E, MODE_DFT, -SIGN, W, 1, 1>;
  constexpr int LS = Fwd::NP + 1;  // odd line stride: adjacent lines start in different banks
  extern __shared__ __align__(128) unsigned char xft_smem[];
  C* smem = reinterpret_cast<C*>(xft_smem);
  const int t = threadIdx.x;
  // compute mapping (matches the load layout so loads coalesce)
  const int w = LOAD_COL ? t % W : t / TR;
  const int j = LOAD_COL ? t / W : t % TR;
  auto noop = []() {};
  C nxt[XFT_TILE_PREFETCH ? E : 1];
  if constexpr (XFT_TILE_PREFETCH) {
    if (blockIdx.x < ntiles)
#pragma unroll
      for (int s = 0; s < E; ++s) nxt[s] = op.load(blockIdx.x, w, j + s * TR);
  }
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    C v[E];
    if constexpr (XFT_TILE_PREFETCH) {
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = nxt[s];
      // software pipelining: the next tile's loads are in flight during this tile's FFT and stores
      if (tile + gridDim.x < ntiles)
#pragma unroll
        for (int s = 0; s < E; ++s) nxt[s] = op.load(tile + gridDim.x, w, j + s * TR);
    } else if constexpr (HasLoadLine<Op>::value) {
      op.template load_line<E, TR>(tile, w, j, v);
    } else {
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = op.load(tile, w, j + s * TR);
    }
    pipe_passes<Fwd, 0>(v, smem + w * LS, j, tw, noop);
    if constexpr (Op::MID) {
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = op.mid(tile, w, j + s * TR, v[s]);
      pipe_passes<Inv, 0>(v, smem + w * LS, j, tw, noop);
    }
    if constexpr (LOAD_COL == STORE_COL && HasStoreLine<Op>::value) {
      op.template store_line<E, TR>(tile, w, j, v);
    } else if constexpr (LOAD_COL == STORE_COL) {
#pragma unroll
      for (int s = 0; s < E; ++s) op.store(tile, w, j + s * TR, v[s]);
    } else {
      __syncthreads();
#pragma unroll
      for (int s = 0; s < E; ++s) smem[w * LS + j + s * TR] = v[s];
      __syncthreads();
      const int w2 = STORE_COL ? t % W : t / TR;
      const int j2 = STORE_COL ? t / W : t % TR;
#pragma unroll
      for (int s = 0; s < E; ++s) op.store(tile, w2, j2 + s * TR, smem[w2 * LS + j2 + s * TR]);
    }
  }
}

template <class C, int LOGL, int W>
constexpr size_t tile_smem() {
  return size_t(W) * ((1 << LOGL) + (1 << LOGL) / 16 + 1) * sizeof(C);
}

}  // namespace xftb
