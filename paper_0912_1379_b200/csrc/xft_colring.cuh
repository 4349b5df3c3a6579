// K7: tall column LCTs in ONE HBM round trip, the four-step intermediate kept in L2.
//
// A column of height R = R1 R2 (r = a R2 + r2) is transformed in two passes
// (as OpColLct1/OpColLct2): pass 1 = pre-chirp, length-R1 DFT over a, twiddle
// w_R^{k1 r2}; pass 2 = length-R2 DFT over r2, post-chirp, natural row
// j = k1 + R1 k2.  Run as two kernels the [R][ncols] intermediate crosses HBM
// twice more.  Here ONE persistent kernel runs both passes over a stream of
// W-column "blocks" (W = 64: 512-byte row segments): the pass-1 tiles of a
// block write one slot of a small ring of scratch (5 slots x 8 MB at R = 16384:
// it lives in the 126 MB L2), and the pass-2 tiles of the same block follow a
// few blocks later, once every pass-1 tile of the block has signalled
// (per-block completion counters, release/acquire at GPU scope).  The slot is
// reused once its pass-2 tiles have signalled.
//
// Schedule.  Tiles are numbered so that every tile depends only on tiles with
// smaller numbers (ring_decode: LAG pass-1 block-phases ahead, then alternating
// pass-1 / pass-2 block-phases).  CTA b owns tiles b, b + grid, b + 2 grid, ...
// in that order; the launch is cooperative, so every CTA is resident and the
// lowest unfinished tile can always run: no deadlock.  (A global ticket
// counter, XFT_RING_STATIC = 0, needs no residency guarantee but costs one
// same-address atomic per tile.)  A dependency that never completes would be a
// bug in the schedule: the issuer traps after 4 s instead of hanging the device.
//
// Data path of a tile (W columns x L rows):
//   TMA (3-D tensor box over the view [R1][R2][ncols] for pass 1, one 1-D bulk
//   copy of the contiguous [r2][w] scratch tile for pass 2; the tile's chirp /
//   twiddle table rows ride on the same mbarrier) into a 3-deep stage ring ->
//   registers (L/8 samples per thread, 8 threads per column) -> FFT passes of
//   the row kernels, exchanging through the tile's own stage -> plain coalesced
//   stores (evict_last into the ring, streaming for the output).
// Every global read is an async bulk copy issued by a helper warp tiles ahead;
// the compute warps wait on shared-memory mbarriers only.
//
// Measured (16384^2 c64, B200): 1.26 ms for the column axis (the 16-CTA cluster
// kernel K6: 1.80 ms), DRAM traffic 2.15 GB read + 2.7-2.9 GB written (4.29 GB
// algorithmic: part of the ring still leaks to HBM).  Experiments kept as
// compile-time switches (XFT_RING_ABL): the bare schedule costs 0.20 ms per
// pass, the FFT arithmetic alone 0.45 ms per pass -- the kernel is bound by
// FP32 issue + shared-memory instructions at 16 compute warps per SM, not by HBM.
#pragma once

#ifndef XFT_RING_SB
#define XFT_RING_SB 1      // column blocks per super-block (the unit of the ring and of the counters)
#endif
#ifndef XFT_RING_LAG
#define XFT_RING_LAG 2     // super-blocks between a block's pass 1 and its pass 2
#endif
#ifndef XFT_RING_SLOTS
#define XFT_RING_SLOTS 5   // ring slots (super-blocks of scratch)
#endif
#ifndef XFT_RING_STAGES
#define XFT_RING_STAGES 3  // TMA stages per CTA
#endif
#ifndef XFT_RING_W
#define XFT_RING_W 64      // columns per tile up to 128 rows a pass (512-byte row segments); a quarter of it beyond
#endif
#ifndef XFT_RING_TR
#define XFT_RING_TR 8      // threads per column (each holds L / TR samples)
#endif
#ifndef XFT_RING_MINB
#define XFT_RING_MINB (64 / XFT_RING_W)  // resident CTAs per SM the registers are sized for (full-width tiles)
#endif
#ifndef XFT_RING_STATIC
#define XFT_RING_STATIC 1  // 1: CTA b takes tiles b, b + grid, ... (cooperative launch: every CTA is resident);
#endif                     // 0: a global ticket counter (one same-address atomic per tile: measured the bottleneck)
#ifndef XFT_RING_QUEUE
#define XFT_RING_QUEUE 2   // tiles a CTA looks ahead beyond its unsignalled ones
#endif
#ifndef XFT_RING_NSUB
#define XFT_RING_NSUB 8    // completion sub-counters per (pass, super-block), 256 B apart (different L2 slices)
#endif
#ifndef XFT_RING_DONE
#define XFT_RING_DONE 8    // completion barriers per CTA: tiles computed but not yet signalled
#endif
#ifndef XFT_RING_ABL
#define XFT_RING_ABL 0     // timing experiments only (wrong results), bits: 1 = pass 1 alone, 2 = pass 2 alone (no
#endif                     // waits), 4 = no FFT passes, 8 = relaxed signals, 32 = consecutive-row tiles, 64 = no stores,
                           // 128 = no loads
#ifndef XFT_COLRING
#define XFT_COLRING 1      // 0: never take the L2-staged column path
#endif
#ifndef XFT_RING_PERSIST_MB
#define XFT_RING_PERSIST_MB 0  // > 0: set the device's persisting-L2 set-aside once (48: the ring stops leaking to HBM,
#endif                         // 2.9 -> 2.1 GB written, but the kernel slows 1.26 -> 1.40 ms: less L2 for the streams)
#ifndef XFT_RING_PF
#define XFT_RING_PF 0      // > 0: the issuer pulls the pass-1 input tiles of its next XFT_RING_PF decoded-but-unissued
#endif                     // tiles into L2 (bulk tensor prefetch).  A/B, 16384^2: 1.311 (1), 1.32 (2) vs 1.257 ms: off
#ifndef XFT_RING_XBAR
#define XFT_RING_XBAR 0    // 1: the "tile has been read" barrier of the compute warps is a split mbarrier phase
                           // (PipeCfg::XBAR).  A/B, 16384^2: 1.272 vs 1.257 ms: off
#endif
#ifndef XFT_RING_HINT
#define XFT_RING_HINT 1    // L2 eviction hints: input evict_first, scratch evict_last
#endif

struct RingPlan {
  int R1, R2, nblocks, SB, nsb, lag, slots;
  unsigned T0, T1;        // tiles per super-block: pass 1 (SB R2), pass 2 (SB R1)
  unsigned tA, tB, total; // ticket regions: leading pass-1 only, interleaved, trailing pass-2 only
  int l0, l1, lsb;        // log2 of T0, T1, SB (all powers of two: the decode below uses shifts only)
  long long ld_in, ld_out;
  int ncols;
};

struct RingTile {
  int phase;  // 0 = pass 1, 1 = pass 2, 2 = no more work
  int sb, cb, idx;
};

__host__ __device__ __forceinline__ RingTile ring_decode(const RingPlan& p, unsigned tk) {
  RingTile t;
  if (tk >= p.total) {
    t.phase = 2;
    t.sb = t.cb = t.idx = 0;
    return t;
  }
  unsigned off;
  if (XFT_RING_ABL & 3) {  // one pass alone over every block
    const int l = (XFT_RING_ABL & 1) ? p.l0 : p.l1;
    t.phase = (XFT_RING_ABL & 1) ? 0 : 1;
    t.sb = (int)(tk >> l);
    off = tk & ((1u << l) - 1);
    t.idx = (int)(off >> p.lsb);
    t.cb = (t.sb << p.lsb) + (int)(off & ((1u << p.lsb) - 1));
    return t;
  }
  if (tk < p.tA) {
    t.phase = 0;
    t.sb = (int)(tk >> p.l0);
    off = tk & (p.T0 - 1);
  } else if (tk < p.tA + p.tB) {
    // one pass-1 block-phase (T0 tiles) then one pass-2 block-phase (T1 = T0 or 2 T0 tiles)
    const unsigned u = tk - p.tA;
    const unsigned m = p.l1 == p.l0 ? u >> (p.l0 + 1) : (u >> p.l0) / 3u;
    off = u - m * (p.T0 + p.T1);
    if (off < p.T0) {
      t.phase = 0;
      t.sb = p.lag + (int)m;
    } else {
      t.phase = 1;
      t.sb = (int)m;
      off -= p.T0;
    }
  } else {
    const unsigned u = tk - p.tA - p.tB;
    t.phase = 1;
    t.sb = p.nsb - p.lag + (int)(u >> p.l1);
    off = u & (p.T1 - 1);
  }
  t.idx = (int)(off >> p.lsb);
  t.cb = (t.sb << p.lsb) + (int)(off & ((1u << p.lsb) - 1));
  return t;
}

constexpr int RING_CSTRIDE = 64;  // words between sub-counters (256 B: the L2 slice hash granularity)
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// every sub-counter of a (pass, super-block) has reached `want`: relaxed loads in flight together,
// then one acquire fence
__device__ __forceinline__ bool ring_complete(const unsigned* ctr, unsigned want) {
  unsigned v[XFT_RING_NSUB];
#pragma unroll
  for (int u = 0; u < XFT_RING_NSUB; ++u) v[u] = ld_relaxed_gpu(ctr + u * RING_CSTRIDE);
  bool ok = true;
#pragma unroll
  for (int u = 0; u < XFT_RING_NSUB; ++u) ok = ok && v[u] >= want;
  if (ok) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  return ok;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

template <int LOG1_, int LOG2_>
struct RingCfg {
  using C = float2;
  static constexpr int LOG1 = LOG1_, LOG2 = LOG2_, R1 = 1 << LOG1, R2 = 1 << LOG2;
  static constexpr int LMAXR = R1 > R2 ? R1 : R2;
  static constexpr int W = LMAXR <= 128 ? XFT_RING_W : XFT_RING_W / 4, TR = XFT_RING_TR, THREADS = W * TR;
  static constexpr int MINB = LMAXR <= 128 ? XFT_RING_MINB : (XFT_RING_W >= 64 ? 2 : 1);
  static constexpr int E1 = R1 / TR, E2 = R2 / TR;
  // exchange barriers: the compute warps only; XFT_RING_XBAR: "tile read" is an mbarrier phase (PipeCfg::XBAR)
  using Fft1 = PipeCfg<C, LOG1, E1, MODE_DFT, -1, W, 1, 1, 0, THREADS, XFT_RING_XBAR>;
  using Fft2 = PipeCfg<C, LOG2, E2, MODE_DFT, -1, W, 1, 1, 0, THREADS, XFT_RING_XBAR>;
  static constexpr int XB = Fft1::NPASS > Fft2::NPASS ? Fft1::NPASS : Fft2::NPASS;  // split barriers per stage
  static constexpr int NPMAX = LMAXR + LMAXR / 16;
  static constexpr int LS = NPMAX + (((1 - NPMAX % 16) % 16) + 16) % 16;  // == 1 (mod 16): W lines x 1 slot per wavefront
  // stages; completion barriers (tiles whose stores may still be unsignalled); tile-info slots
  static constexpr int NS = XFT_RING_STAGES, ND = XFT_RING_DONE, NI = ND + XFT_RING_QUEUE;
  // stage: [L][W] tile, then two table rows of L entries; later the tile's padded exchange buffer [W][LS]
  static constexpr int STAGE0 = LMAXR * W + 2 * LMAXR > W * LS ? LMAXR * W + 2 * LMAXR : W * LS;
  static constexpr int STAGE = (STAGE0 + 15) / 16 * 16;
  static constexpr size_t SMEM = size_t(NS) * STAGE * sizeof(C);
};

// table rows + counters for one call (stream scratch), written by ring_setup_kernel:
//   pre [r2][a]  = pre-chirp of row a R2 + r2            post[k1][k2] = post-chirp of row k1 + R1 k2
struct RingBufs {
  float2* ring;
  const float2* pre;
  const float2* post;
  const float2* twr;    // [r2][k1] = w_R^{k1 r2} (per device and R)
  unsigned* ticket;     // the ticket counter (XFT_RING_STATIC = 0), 256 B before the completion counters
  unsigned* done1;      // [nsb][NSUB] sub-counters, RING_CSTRIDE words apart; tile idx counts on idx % NSUB
  unsigned* done2;
};

// Table rows are stored in the order the threads read them: entry j E + s of a row belongs to
// sample j + TR s (thread j's register s), so a thread fetches its E entries as E/2 16-byte loads.
__global__ void ring_setup_kernel(float2* pre, float2* post, unsigned* counters, int ncounters, ColChirp ck, int R1,
                                  int R2, int TR) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ncounters) counters[i] = 0u;
  const long long R = (long long)R1 * R2;
  if (i >= R) return;
  const int lr = ck.log2r;
  {  // pre[r2][a], r = a R2 + r2
    const int r2 = i / R1, e = R1 / TR, a = (i % R1) / e + TR * ((i % R1) % e);
    const long long r = (long long)a * R2 + r2;
    const long long off = 2 * r - R + 1;
    unsigned long long ph = ((unsigned long long)(r & 1) << 63) - ((unsigned long long)r << (63 - lr));
    if (ck.pre) ph += ck.dq_in * (unsigned long long)(off * off);
    double s, c;
    sincospi(2.0 * ((double)(long long)ph * 5.42101086242752217e-20), &s, &c);
    pre[i] = make_float2((float)c, (float)s);
  }
  {  // post[k1][k2], j = k1 + R1 k2
    const int k1 = i / R2, e = R2 / TR, k2 = (i % R2) / e + TR * ((i % R2) % e);
    const long long j = k1 + (long long)R1 * k2;
    const long long off = 2 * j - R + 1;
    unsigned long long ph = ((unsigned long long)(j & 1) << 63) - ((unsigned long long)j << (63 - lr)) +
                            ((unsigned long long)ck.gq << 32);
    if (ck.post) ph += ck.dq_out * (unsigned long long)(off * off);
    double s, c;
    sincospi(2.0 * ((double)(long long)ph * 5.42101086242752217e-20), &s, &c);
    post[i] = make_float2((float)(c * (double)ck.gabs), (float)(s * (double)ck.gabs));
  }
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p) {
  if (XFT_RING_ABL & 8) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
  else asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// Warp roles: THREADS compute threads, one issuer warp, one signaller warp (lane 0 of each).
//   issuer     decodes its next tiles ahead (XFT_RING_QUEUE beyond the unsignalled ones), checks each tile's
//              dependency counter ahead of time, and issues the tile's bulk copies as soon as its
//              stage is free -- nothing with a global round trip sits between "stage free" and
//              the TMA issue;
//   signaller  waits for done[s] of sequence q and publishes the tile's completion (one
//              red.release at GPU scope), then advances `nsig` (shared);
//   compute    waits on full[s], transforms, stores, arrives on done[s].
// Barriers:  full[s]   issuer -> compute: the tile (or the end marker) of sequence q, s = q % NS, has landed
//            empty[s]  compute -> issuer: the last shared-memory read of the tile is done (before its stores)
//            done[d]   compute -> signaller: every compute thread has issued the tile's stores, d = q % ND
// Sequence q is issued only once q - NS has released its stage and q - ND has been signalled, so
// stages, barriers and info slots are reused strictly one phase at a time, while a stage is NOT
// held for the store-drain and signal latencies of its tile.  Neither helper blocks on a dependency: a tile
// whose counter is not yet complete stays pending while completions keep being published, which
// (with the ticket order) rules out deadlock.
// The Stockham exchange of a tile runs inside its own stage (the tile and its table rows are in
// registers by then), so a CTA needs NS x 18.5 KB of shared memory.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 64, Cfg::MINB)
xft_colring_kernel(const __grid_constant__ CUtensorMap map, float2* __restrict__ out, RingPlan pl, RingBufs bf,
                   const float2* __restrict__ tw1, const float2* __restrict__ tw2) {
  using C = float2;
  constexpr int W = Cfg::W, TR = Cfg::TR, NS = Cfg::NS, ND = Cfg::ND, NI = Cfg::NI, R1 = Cfg::R1, R2 = Cfg::R2;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ __align__(8) uint64_t done[ND];
  __shared__ __align__(8) uint64_t rdbar[NS][Cfg::XB];  // XFT_RING_XBAR: the stage's tile / exchanges have been read
  __shared__ RingTile info[NI];
  __shared__ volatile int nsig;  // sequences signalled so far (signaller -> issuer)
  C* const stages = reinterpret_cast<C*>(xft_smem);
  const int t = threadIdx.x;
  const long long R = (long long)R1 * R2;
  auto slot_base = [&](const RingTile& ti) -> C* {
    const int slot = ti.sb % pl.slots;
    return bf.ring + ((long long)(slot * pl.SB + (ti.cb - ti.sb * pl.SB)) * R) * W;
  };
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::THREADS);
      for (int x = 0; x < Cfg::XB; ++x) mbar_init(&rdbar[s][x], Cfg::THREADS / 32);
    }
#pragma unroll
    for (int s = 0; s < ND; ++s) mbar_init(&done[s], Cfg::THREADS);
    nsig = 0;
    fence_mbar_init();
  }
  __syncthreads();

  if (t >= Cfg::THREADS + 32) {
    // ------------------------------ signaller ------------------------------
    if (t != Cfg::THREADS + 32) return;
    for (int q = 0;; ++q) {
      mbar_wait(&done[q % ND], (uint32_t)((q / ND) & 1));
      const RingTile ti = info[q % NI];
      if (ti.phase == 2) break;
      red_release_gpu((ti.phase == 0 ? bf.done1 : bf.done2) +
                      ((long long)ti.sb * XFT_RING_NSUB + ti.idx % XFT_RING_NSUB) * RING_CSTRIDE);
      nsig = q + 1;
    }
    return;
  }
  if (t >= Cfg::THREADS) {
    // ------------------------------ issuer ------------------------------
    if (t != Cfg::THREADS) return;
    const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
    // tickets fetched; dependencies verified; tiles issued (incl. the end marker); stage releases observed
    int nf = 0, nd = 0, ni = 0, nrel = 0;
    int npf = 0;  // XFT_RING_PF: tiles whose input has been prefetched into L2 (or skipped)
    bool ended = false;
    const unsigned* ok_ctr = nullptr;  // the last dependency counter seen complete
    unsigned long long idle_since = 0;
    while (true) {
      bool progress = false;
      const int sg = nsig;
      if (!ended && nf < sg + NI) {
        const unsigned tk = XFT_RING_STATIC ? blockIdx.x + (unsigned)nf * gridDim.x : atomicAdd(bf.ticket, 1u);
        const RingTile ti = ring_decode(pl, tk);
        info[nf % NI] = ti;
        if (ti.phase == 2) ended = true;
        ++nf;
        progress = true;
      }
      if (nd < nf) {  // the oldest tile whose dependency is still unverified
        const RingTile ti = info[nd % NI];
        const unsigned* ctr = nullptr;
        unsigned want = 0;
        if (ti.phase == 0) {
          if (ti.sb >= pl.slots) {
            ctr = bf.done2 + (long long)(ti.sb - pl.slots) * XFT_RING_NSUB * RING_CSTRIDE;
            want = pl.T1 / XFT_RING_NSUB;
          }
        } else if (ti.phase == 1) {
          ctr = bf.done1 + (long long)ti.sb * XFT_RING_NSUB * RING_CSTRIDE;
          want = pl.T0 / XFT_RING_NSUB;
        }
        if (XFT_RING_ABL & 3) ctr = nullptr;
        if (ctr == nullptr || ctr == ok_ctr) {
          ++nd;
          progress = true;
        } else if (ring_complete(ctr, want)) {
          ok_ctr = ctr;
          fence_proxy_async_all();  // the acquired generic-proxy stores (scratch) are read by bulk copies
          ++nd;
          progress = true;
        }
      }
      if constexpr (XFT_RING_PF > 0) {
        if (npf < ni) npf = ni;  // already issued: nothing to prefetch
        if (npf < nf && npf < ni + XFT_RING_PF) {
          const RingTile tp = info[npf % NI];
          if (tp.phase == 0) tma_prefetch_3d(&map, tp.cb * W, tp.idx, 0);
          ++npf;
          progress = true;
        }
      }
      if (nrel < ni && mbar_test(&empty[nrel % NS], (uint32_t)((nrel / NS) & 1))) {
        ++nrel;  // the compute warps have read the last shared-memory word of sequence nrel's stage
        progress = true;
      }
      if (ni < nd && ni < nrel + NS && ni < sg + ND) {
        const int st = ni % NS;
        const RingTile ti = info[ni % NI];
        C* const S = stages + st * Cfg::STAGE;
        if (ti.phase == 2 || (XFT_RING_ABL & 128)) {
          mbar_arrive(&full[st]);  // end marker: the compute warps wake up, read it and leave
        } else if (ti.phase == 0) {
          mbar_arrive_expect_tx(&full[st], (uint32_t)((R1 * W + 2 * R1) * sizeof(C)));
          if (XFT_RING_HINT) tma_load_3d_hint(S, &map, ti.cb * W, ti.idx, 0, &full[st], pol_first);
          else tma_load_3d(S, &map, ti.cb * W, ti.idx, 0, &full[st]);
          tma_load_1d(S + Cfg::LMAXR * W, bf.pre + (long long)ti.idx * R1, R1 * sizeof(C), &full[st]);
          tma_load_1d(S + Cfg::LMAXR * W + Cfg::LMAXR, bf.twr + (long long)ti.idx * R1, R1 * sizeof(C), &full[st]);
        } else {
          mbar_arrive_expect_tx(&full[st], (uint32_t)((R2 * W + R2) * sizeof(C)));
          const C* src = slot_base(ti) + (long long)ti.idx * R2 * W;
          if (XFT_RING_HINT) tma_load_1d_hint(S, src, R2 * W * sizeof(C), &full[st], pol_last);
          else tma_load_1d(S, src, R2 * W * sizeof(C), &full[st]);
          tma_load_1d(S + Cfg::LMAXR * W, bf.post + (long long)ti.idx * R2, R2 * sizeof(C), &full[st]);
        }
        ++ni;
        progress = true;
        if (ti.phase == 2) break;
      }
      if (progress) {
        idle_since = 0;
      } else {
        // nothing moved: a dependency or a completion is outstanding.  A schedule that never
        // advances is a bug: trap (a loud launch failure) rather than hang the device.
        const unsigned long long now = global_ns();
        if (idle_since == 0) idle_since = now;
        else if (now - idle_since > 4000000000ull) __trap();
        __nanosleep(64);
      }
    }
    return;
  }

  // ------------------------------ compute warps ------------------------------
  const int w = t % W, j = t / W;
  const uint64_t pol_last = l2_policy_evict_last();
  auto noop = []() {};
  for (int i = 0;; ++i) {
    const int st = i % NS;
    mbar_wait(&full[st], (uint32_t)((i / NS) & 1));
    const RingTile ti = info[i % NI];
    if (ti.phase == 2) {
      mbar_arrive(&done[i % ND]);  // lets the signaller see the end marker
      break;
    }
    C* const S = stages + st * Cfg::STAGE;
    const int col = ti.cb * W + w;
    const XBar xb{rdbar[st], i / NS};
    if (ti.phase == 0) {
      constexpr int E = Cfg::E1;
      C v[E], tq[E];
      const C* pre = S + Cfg::LMAXR * W;
      const C* twr = pre + Cfg::LMAXR;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int a = j + s * TR;
        v[s] = S[a * W + w];
      }
      {
        const float4* p4 = reinterpret_cast<const float4*>(pre + j * E);
        const float4* t4 = reinterpret_cast<const float4*>(twr + j * E);
#pragma unroll
        for (int s = 0; s < E; s += 2) {
          const float4 p = p4[s / 2], q = t4[s / 2];
          v[s] = cmul(make_float2(p.x, p.y), v[s]);
          v[s + 1] = cmul(make_float2(p.z, p.w), v[s + 1]);
          tq[s] = make_float2(q.x, q.y);
          tq[s + 1] = make_float2(q.z, q.w);
        }
      }
      if constexpr (Cfg::Fft1::XBAR) {
        xb.template arrive<0>();  // this warp has read its part of the tile and of the table rows
        pipe_passes_x<typename Cfg::Fft1, 0>(v, S + w * Cfg::LS, j, tw1, noop, xb);
      } else if (!(XFT_RING_ABL & 4)) {
        pipe_passes<typename Cfg::Fft1, 0>(v, S + w * Cfg::LS, j, tw1, noop);
      }
      mbar_arrive(&empty[st]);  // this thread is done with the stage
      C* dst = slot_base(ti) + (long long)ti.idx * W + w;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k1 = j + s * TR;
        const C y = cmul(v[s], tq[s]);
        if ((XFT_RING_ABL & 64) && y.x != 123.f) continue;
        if (XFT_RING_HINT) st_hint(dst + (long long)k1 * R2 * W, y, pol_last);
        else dst[(long long)k1 * R2 * W] = y;
      }
      fence_proxy_async_global();  // these stores are read by another CTA's bulk copy
    } else {
      constexpr int E = Cfg::E2;
      C v[E], pq[E];
      const C* post = S + Cfg::LMAXR * W;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int a = j + s * TR;
        v[s] = S[a * W + w];
      }
      {
        const float4* p4 = reinterpret_cast<const float4*>(post + j * E);
#pragma unroll
        for (int s = 0; s < E; s += 2) {
          const float4 p = p4[s / 2];
          pq[s] = make_float2(p.x, p.y);
          pq[s + 1] = make_float2(p.z, p.w);
        }
      }
      if constexpr (Cfg::Fft2::XBAR) {
        xb.template arrive<0>();
        pipe_passes_x<typename Cfg::Fft2, 0>(v, S + w * Cfg::LS, j, tw2, noop, xb);
      } else if (!(XFT_RING_ABL & 4)) {
        pipe_passes<typename Cfg::Fft2, 0>(v, S + w * Cfg::LS, j, tw2, noop);
      }
      mbar_arrive(&empty[st]);
      if (col < pl.ncols) {
        C* dst = out + (long long)ti.idx * pl.ld_out + col;
#pragma unroll
        for (int s = 0; s < E; ++s) {
          const int k2 = j + s * TR;
          if ((XFT_RING_ABL & 64) && v[s].x != 123.f) continue;
          st_stream(dst + (long long)k2 * R1 * pl.ld_out, cmul(v[s], pq[s]));
        }
      }
    }
    mbar_arrive(&done[i % ND]);
  }
}

// (device, R) -> [r2][k1] twiddles w_R^{k1 r2}, R = R1 R2
std::mutex g_ring_mu;
std::map<std::tuple<int, int, int, int>, float2*> g_ring_tw;
int ring_twiddles(int l1, int l2, int TR, const float2** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  auto key = std::make_tuple(dev, l1, l2, TR);
  auto it = g_ring_tw.find(key);
  if (it == g_ring_tw.end()) {
    const int R1 = 1 << l1, R2 = 1 << l2;
    const long long R = (long long)R1 * R2;
    std::vector<float2> h((size_t)R);
    const int e = R1 / TR;  // thread order within a row: entry j e + s is k1 = j + TR s
    for (int r2 = 0; r2 < R2; ++r2)
      for (int k1 = 0; k1 < R1; ++k1) {
        const long long m = ((long long)k1 * r2) % R;
        const long double th = 2.0L * PI_L * (long double)m / (long double)R;
        h[(size_t)r2 * R1 + (k1 % TR) * e + k1 / TR] = make_float2((float)cosl(th), (float)-sinl(th));
      }
    float2* p = nullptr;
    if (cudaMalloc(&p, sizeof(float2) * R) != cudaSuccess) return XFT_ECUDA;
    if (cudaMemcpy(p, h.data(), sizeof(float2) * R, cudaMemcpyHostToDevice) != cudaSuccess) return XFT_ECUDA;
    it = g_ring_tw.emplace(key, p).first;
  }
  *out = it->second;
  return XFT_OK;
}

// the schedule of a [2^(log1+log2)][ncols] column transform with W-column tiles (host side)
inline RingPlan ring_plan(int log1, int log2, int W, int64_t ncols, int64_t ld, int64_t ld_out) {
  RingPlan pl{};
  pl.R1 = 1 << log1;
  pl.R2 = 1 << log2;
  pl.nblocks = (int)((ncols + W - 1) / W);
  pl.SB = XFT_RING_SB;
  while (pl.nblocks % pl.SB) pl.SB /= 2;
  pl.nsb = pl.nblocks / pl.SB;
  pl.lag = pl.nsb < XFT_RING_LAG ? pl.nsb : XFT_RING_LAG;
  pl.slots = pl.nsb < XFT_RING_SLOTS ? pl.nsb : XFT_RING_SLOTS;
  pl.T0 = (unsigned)(pl.SB * pl.R2);
  pl.T1 = (unsigned)(pl.SB * pl.R1);
  pl.lsb = log2_of(pl.SB);
  pl.l0 = pl.lsb + log2;
  pl.l1 = pl.lsb + log1;  // log1 == log2 or log2 + 1: pass-2 block-phases are 1x or 2x the pass-1 ones
  pl.tA = (unsigned)pl.lag * pl.T0;
  pl.tB = (unsigned)(pl.nsb - pl.lag) * (pl.T0 + pl.T1);
  pl.total = pl.tA + pl.tB + (unsigned)pl.lag * pl.T1;
  if (XFT_RING_ABL & 3) pl.total = (unsigned)pl.nsb * ((XFT_RING_ABL & 1) ? pl.T0 : pl.T1);
  pl.ld_in = ld;
  pl.ld_out = ld_out;
  pl.ncols = (int)ncols;
  return pl;
}

template <int LOG1, int LOG2>
int launch_colring(const void* in, void* out, int64_t ncols, int64_t ld, int64_t ld_out, const ColChirp& ck,
                   cudaStream_t st, bool probe) {
  using Cfg = RingCfg<LOG1, LOG2>;
  constexpr int W = Cfg::W, R1 = Cfg::R1, R2 = Cfg::R2;
  constexpr long long R = (long long)R1 * R2;
  if (ld % 2 || (reinterpret_cast<uintptr_t>(in) & 15) || ncols < 1 || ncols > (1ll << 24)) return XFT_ENOTSUP;
  auto enc = tensor_encoder();
  if (!enc) return XFT_ENOTSUP;
  auto kern = xft_colring_kernel<Cfg>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM) != cudaSuccess) {
    cudaGetLastError();
    return XFT_ENOTSUP;
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::THREADS + 64, Cfg::SMEM) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return XFT_ENOTSUP;
  }
  if (probe) return XFT_OK;
  if (XFT_RING_PERSIST_MB > 0) {
    static std::once_flag once;
    std::call_once(once, []() { cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)XFT_RING_PERSIST_MB << 20); });
  }
  const RingPlan pl = ring_plan(LOG1, LOG2, W, ncols, ld, ld_out);
  // scratch: ring, pre/post table rows, counters
  const size_t ring_bytes = (size_t)pl.slots * pl.SB * R * W * sizeof(float2);
  const size_t tab_bytes = (size_t)R * sizeof(float2);
  const int ncounters = RING_CSTRIDE * (1 + 2 * pl.nsb * XFT_RING_NSUB);
  const size_t ctr_bytes = (size_t)ncounters * 4;
  char* base = static_cast<char*>(stream_scratch(dev, st, ring_bytes + 2 * tab_bytes + ctr_bytes));
  if (!base) return XFT_ECUDA;
  RingBufs bf{};
  bf.ring = reinterpret_cast<float2*>(base);
  float2* pre = reinterpret_cast<float2*>(base + ring_bytes);
  float2* post = reinterpret_cast<float2*>(base + ring_bytes + tab_bytes);
  bf.pre = pre;
  bf.post = post;
  bf.ticket = reinterpret_cast<unsigned*>(base + ring_bytes + 2 * tab_bytes);
  bf.done1 = bf.ticket + RING_CSTRIDE;
  bf.done2 = bf.done1 + (size_t)pl.nsb * XFT_RING_NSUB * RING_CSTRIDE;
  int rc = ring_twiddles(LOG1, LOG2, Cfg::TR, &bf.twr);
  if (rc) return rc;
  Tables t1, t2;
  if ((rc = get_tables(R1, XFT_C64, &t1, Cfg::E1))) return rc;
  if ((rc = get_tables(R2, XFT_C64, &t2, Cfg::E2))) return rc;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)ncols, (cuuint64_t)R2, (cuuint64_t)R1};
  // (XFT_RING_ABL & 32: a tile = R1 CONSECUTIVE rows -- wrong rows, the access-pattern experiment)
  const cuuint64_t strides[2] = {(cuuint64_t)(((XFT_RING_ABL & 32) ? R1 : 1) * ld * sizeof(float2)),
                                 (cuuint64_t)(((XFT_RING_ABL & 32) ? 1 : R2) * ld * sizeof(float2))};
  const cuuint32_t box[3] = {(cuuint32_t)W, 1u, (cuuint32_t)R1};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(in), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return XFT_ENOTSUP;
  const int nset = (int)((R > ncounters ? R : ncounters) + 255) / 256;
  ring_setup_kernel<<<nset, 256, 0, st>>>(pre, post, bf.ticket, ncounters, ck, R1, R2, Cfg::TR);
  const long long cap = (long long)sms * occ;
  const unsigned grid = (unsigned)(pl.total < cap ? pl.total : cap);
  // cooperative launch: the runtime refuses a grid whose CTAs cannot all be resident, which the
  // static tile assignment relies on (a non-resident CTA would own tiles others wait for)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = XFT_RING_STATIC;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::THREADS + 64);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, map, static_cast<float2*>(out), pl, bf, static_cast<const float2*>(t1.tw),
                         static_cast<const float2*>(t2.tw)) != cudaSuccess) {
    cudaGetLastError();
    return XFT_ENOTSUP;  // e.g. a cooperative grid the device cannot hold right now (MPS/MIG): the caller's other paths
  }
  return XFT_OK;
}

// shape of the K7 tiles for a column height 2^l (14 <= l <= 16): pass lengths and tile width
inline bool ring_shape(int l, int* log1, int* log2, int* W) {
  if (l < 14 || l > 16) return false;
  *log1 = (l + 1) / 2;
  *log2 = l / 2;
  *W = *log1 <= 7 ? XFT_RING_W : XFT_RING_W / 4;
  return true;
}

// c64 columns of height 2^14 .. 2^16 (R1 x R2 = 128x128 .. 256x256); anything else: XFT_ENOTSUP, nothing launched.
// (Measured on 4096- and 8192-row fields the cluster kernel K6 is faster -- 0.10 vs 0.15 ms at 4096^2, 0.39 vs
// 0.43 ms at 8192^2: shorter passes leave less work per tile handshake -- so those heights stay with K6.)
inline int lct_cols_ring(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, int64_t ld_out,
                         const ColChirp& ck, cudaStream_t st, bool probe = false) {
  if (!XFT_COLRING) return XFT_ENOTSUP;
  switch (log2_of(R)) {
    case 14: return launch_colring<7, 7>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 15: return launch_colring<8, 7>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 16: return launch_colring<8, 8>(in, out, ncols, ld, ld_out, ck, st, probe);
    default: return XFT_ENOTSUP;
  }
}
