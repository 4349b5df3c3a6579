// K7: tall column LCTs in ONE HBM round trip, the four-step intermediate kept in L2.
//
// A column of height R = R1 R2 (r = a R2 + r2) is transformed in two passes
// (as OpColLct1/OpColLct2): pass 1 = pre-chirp, length-R1 DFT over a, twiddle
// w_R^{k1 r2}; pass 2 = length-R2 DFT over r2, post-chirp, natural row
// j = k1 + R1 k2.  Run as two kernels the [R][ncols] intermediate crosses HBM
// twice more.  Here ONE persistent kernel runs both passes over a stream of
// 16-column "blocks": the pass-1 tiles of a block write a 2 MB slot of a small
// ring of scratch (tens of MB: it lives in the 126 MB L2), and the pass-2 tiles
// of the same block are handed out a few blocks later, when every pass-1 tile
// of the block has signalled (a per-block counter, release/acquire at GPU
// scope).  The slot is reused once its pass-2 tiles have signalled.  Tiles are
// handed out by a global ticket in an order in which every tile depends only on
// tiles with smaller tickets, and a CTA only ever blocks when all its earlier
// tiles are complete, so the schedule cannot deadlock whatever the residency.
//
// Data path of a tile (W = 16 columns x L rows, 128-byte row segments):
//   TMA (3-D tensor box over the view [R1][R2][ncols] for pass 1, one 1-D bulk
//   copy of the contiguous [r2][w] scratch tile for pass 2; the tile's chirp /
//   twiddle table rows ride on the same mbarrier) into a 2-deep stage ring ->
//   registers (L/8 samples per thread, 8 threads per column) -> FFT passes of
//   the row kernels -> plain coalesced stores (streaming for the output).
// Every global read is an async bulk copy issued one or two tiles ahead.
#pragma once

#ifndef XFT_RING_SB
#define XFT_RING_SB 2      // column blocks handed out side by side (SB x 128 B contiguous per row)
#endif
#ifndef XFT_RING_LAG
#define XFT_RING_LAG 4     // super-blocks between a block's pass 1 and its pass 2
#endif
#ifndef XFT_RING_SLOTS
#define XFT_RING_SLOTS 8   // ring slots (super-blocks of scratch)
#endif
#ifndef XFT_RING_STAGES
#define XFT_RING_STAGES 2  // TMA stages per CTA
#endif
#ifndef XFT_RING_MINB
#define XFT_RING_MINB 4    // resident CTAs per SM the registers are sized for
#endif
#ifndef XFT_COLRING
#define XFT_COLRING 1      // 0: never take the L2-staged column path
#endif
#ifndef XFT_RING_HINT
#define XFT_RING_HINT 1    // L2 eviction hints: input evict_first, scratch evict_last
#endif

struct RingPlan {
  int R1, R2, nblocks, SB, nsb, lag, slots;
  unsigned T0, T1;        // tiles per super-block: pass 1 (SB R2), pass 2 (SB R1)
  unsigned tA, tB, total; // ticket regions: leading pass-1 only, interleaved, trailing pass-2 only
  long long ld_in, ld_out;
  int ncols;
};

struct RingTile {
  int phase;  // 0 = pass 1, 1 = pass 2, 2 = no more work
  int sb, cb, idx;
};

__device__ __forceinline__ RingTile ring_decode(const RingPlan& p, unsigned tk) {
  RingTile t;
  if (tk >= p.total) {
    t.phase = 2;
    t.sb = t.cb = t.idx = 0;
    return t;
  }
  unsigned off;
  if (tk < p.tA) {
    t.phase = 0;
    t.sb = (int)(tk / p.T0);
    off = tk % p.T0;
  } else if (tk < p.tA + p.tB) {
    const unsigned u = tk - p.tA, per = p.T0 + p.T1;
    const int m = (int)(u / per);
    off = u % per;
    if (off < p.T0) {
      t.phase = 0;
      t.sb = p.lag + m;
    } else {
      t.phase = 1;
      t.sb = m;
      off -= p.T0;
    }
  } else {
    const unsigned u = tk - p.tA - p.tB;
    t.phase = 1;
    t.sb = p.nsb - p.lag + (int)(u / p.T1);
    off = u % p.T1;
  }
  t.idx = (int)(off / p.SB);
  t.cb = t.sb * p.SB + (int)(off % p.SB);
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
  static constexpr int W = 16, TR = 8, THREADS = W * TR;
  static constexpr int E1 = R1 / TR, E2 = R2 / TR;
  using Fft1 = PipeCfg<C, LOG1, E1, MODE_DFT, -1, W, 1, 1, 0, THREADS>;  // exchange barriers: the compute warps only
  using Fft2 = PipeCfg<C, LOG2, E2, MODE_DFT, -1, W, 1, 1, 0, THREADS>;
  static constexpr int LMAXR = R1 > R2 ? R1 : R2;
  static constexpr int NPMAX = LMAXR + LMAXR / 16;
  static constexpr int LS = NPMAX + (((1 - NPMAX % 16) % 16) + 16) % 16;  // == 1 (mod 16): W lines x 1 slot per wavefront
  static constexpr int NS = XFT_RING_STAGES;
  // stage: [L][W] tile, then two table rows of L entries
  static constexpr int STAGE = LMAXR * W + 2 * LMAXR;
  static constexpr size_t SMEM = (size_t(NS) * STAGE + size_t(W) * LS) * sizeof(C);
};

// table rows + counters for one call (stream scratch), written by ring_setup_kernel:
//   pre [r2][a]  = pre-chirp of row a R2 + r2            post[k1][k2] = post-chirp of row k1 + R1 k2
struct RingBufs {
  float2* ring;
  const float2* pre;
  const float2* post;
  const float2* twr;    // [r2][k1] = w_R^{k1 r2} (per device and R)
  unsigned* ticket;     // [0] = ticket, then done1[nsb], done2[nsb]
  unsigned* done1;
  unsigned* done2;
};

__global__ void ring_setup_kernel(float2* pre, float2* post, unsigned* counters, int ncounters, ColChirp ck, int R1,
                                  int R2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ncounters) counters[i] = 0u;
  const long long R = (long long)R1 * R2;
  if (i >= R) return;
  const int lr = ck.log2r;
  {  // pre[r2][a], r = a R2 + r2
    const int r2 = i / R1, a = i % R1;
    const long long r = (long long)a * R2 + r2;
    const long long off = 2 * r - R + 1;
    unsigned long long ph = ((unsigned long long)(r & 1) << 63) - ((unsigned long long)r << (63 - lr));
    if (ck.pre) ph += ck.dq_in * (unsigned long long)(off * off);
    double s, c;
    sincospi(2.0 * ((double)(long long)ph * 5.42101086242752217e-20), &s, &c);
    pre[i] = make_float2((float)c, (float)s);
  }
  {  // post[k1][k2], j = k1 + R1 k2
    const int k1 = i / R2, k2 = i % R2;
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
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

// One scheduler warp (lane 0) + THREADS compute threads.  The scheduler takes tickets, checks the
// tile's dependency counter, issues the tile's bulk copies and publishes completion counters; the
// compute warps only ever wait on shared-memory mbarriers:
//   full[s]  scheduler -> compute: tile (or the end marker) of sequence number q, s = q % NS, has landed
//   done[s]  compute -> scheduler: every compute thread has issued the tile's stores
// Sequence q + NS is fetched and issued only after q has been signalled, so a stage, its info
// slot and both barriers are reused strictly one phase at a time.  The scheduler never blocks: a
// tile whose dependency is not yet satisfied just stays pending while completions are published,
// which (with the ticket order) rules out deadlock.
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 32, XFT_RING_MINB)
xft_colring_kernel(const __grid_constant__ CUtensorMap map, float2* __restrict__ out, RingPlan pl, RingBufs bf,
                   const float2* __restrict__ tw1, const float2* __restrict__ tw2) {
  using C = float2;
  constexpr int W = Cfg::W, TR = Cfg::TR, NS = Cfg::NS, R1 = Cfg::R1, R2 = Cfg::R2;
  extern __shared__ __align__(128) unsigned char xft_smem[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t done[NS];
  __shared__ RingTile info[NS];
  C* const stages = reinterpret_cast<C*>(xft_smem);
  C* const xbuf = stages + NS * Cfg::STAGE;
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
      mbar_init(&done[s], Cfg::THREADS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (t >= Cfg::THREADS) {
    // ------------------------------ scheduler ------------------------------
    if (t != Cfg::THREADS) return;
    const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
    int nf = 0, ni = 0, nsg = 0, nreal = 0x7fffffff;
    bool ended = false;
    const unsigned* ok_ctr = nullptr;  // the last dependency counter seen satisfied (acquired once per CTA)
    unsigned long long idle_since = 0;
    while (true) {
      bool progress = false;
      if (nsg < ni && nsg < nreal && mbar_test(&done[nsg % NS], (uint32_t)((nsg / NS) & 1))) {
        const RingTile ti = info[nsg % NS];
        red_release_gpu((ti.phase == 0 ? bf.done1 : bf.done2) + ti.sb);
        ++nsg;
        progress = true;
      }
      if (!ended && nf < nsg + NS) {
        const unsigned tk = atomicAdd(bf.ticket, 1u);
        const RingTile ti = ring_decode(pl, tk);
        info[nf % NS] = ti;
        if (ti.phase == 2) {
          ended = true;
          nreal = nf;
        }
        ++nf;
        progress = true;
      }
      if (ni < nf) {
        const int st = ni % NS;
        const RingTile ti = info[st];
        if (ti.phase == 2) {
          mbar_arrive(&full[st]);  // end marker: the compute warps wake up, read it and leave
          ++ni;
          progress = true;
        } else {
          const unsigned* ctr = nullptr;
          unsigned want = 0;
          if (ti.phase == 0) {
            if (ti.sb >= pl.slots) {
              ctr = bf.done2 + (ti.sb - pl.slots);
              want = pl.T1;
            }
          } else {
            ctr = bf.done1 + ti.sb;
            want = pl.T0;
          }
          if (ctr == nullptr || ctr == ok_ctr || ld_acquire_gpu(ctr) >= want) {
            if (ctr) ok_ctr = ctr;
            C* const S = stages + st * Cfg::STAGE;
            fence_proxy_async_all();  // the stage's generic-proxy reads; (pass 2) the acquired scratch stores
            if (ti.phase == 0) {
              mbar_arrive_expect_tx(&full[st], (uint32_t)((R1 * W + 2 * R1) * sizeof(C)));
              if (XFT_RING_HINT) tma_load_3d_hint(S, &map, ti.cb * W, ti.idx, 0, &full[st], pol_first);
              else tma_load_3d(S, &map, ti.cb * W, ti.idx, 0, &full[st]);
              tma_load_1d(S + Cfg::LMAXR * W, bf.pre + (long long)ti.idx * R1, R1 * sizeof(C), &full[st]);
              tma_load_1d(S + Cfg::LMAXR * W + Cfg::LMAXR, bf.twr + (long long)ti.idx * R1, R1 * sizeof(C),
                          &full[st]);
            } else {
              mbar_arrive_expect_tx(&full[st], (uint32_t)((R2 * W + R2) * sizeof(C)));
              const C* src = slot_base(ti) + (long long)ti.idx * R2 * W;
              if (XFT_RING_HINT) tma_load_1d_hint(S, src, R2 * W * sizeof(C), &full[st], pol_last);
              else tma_load_1d(S, src, R2 * W * sizeof(C), &full[st]);
              tma_load_1d(S + Cfg::LMAXR * W, bf.post + (long long)ti.idx * R2, R2 * sizeof(C), &full[st]);
            }
            ++ni;
            progress = true;
          }
        }
      }
      if (ended && ni == nf && nsg >= nreal) break;
      if (progress) {
        idle_since = 0;
      } else {
        // nothing moved: a dependency or a completion is outstanding.  A schedule that never
        // advances is a bug: trap (a loud launch failure) rather than hang the device.
        const unsigned long long now = global_ns();
        if (idle_since == 0) idle_since = now;
        else if (now - idle_since > 4000000000ull) __trap();
        __nanosleep(40);
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
    const RingTile ti = info[st];
    if (ti.phase == 2) break;
    C* const S = stages + st * Cfg::STAGE;
    const int col = ti.cb * W + w;
    if (ti.phase == 0) {
      constexpr int E = Cfg::E1;
      C v[E], tq[E];
      const C* pre = S + Cfg::LMAXR * W;
      const C* twr = pre + Cfg::LMAXR;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int a = j + s * TR;
        v[s] = cmul(pre[a], S[a * W + w]);
        tq[s] = twr[a];
      }
      pipe_passes<typename Cfg::Fft1, 0>(v, xbuf + w * Cfg::LS, j, tw1, noop);
      C* dst = slot_base(ti) + (long long)ti.idx * W + w;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k1 = j + s * TR;
        const C y = cmul(v[s], tq[s]);
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
        pq[s] = post[a];
      }
      pipe_passes<typename Cfg::Fft2, 0>(v, xbuf + w * Cfg::LS, j, tw2, noop);
      if (col < pl.ncols) {
        C* dst = out + (long long)ti.idx * pl.ld_out + col;
#pragma unroll
        for (int s = 0; s < E; ++s) {
          const int k2 = j + s * TR;
          st_stream(dst + (long long)k2 * R1 * pl.ld_out, cmul(v[s], pq[s]));
        }
      }
    }
    mbar_arrive(&done[st]);
  }
}

// (device, R) -> [r2][k1] twiddles w_R^{k1 r2}, R = R1 R2
std::mutex g_ring_mu;
std::map<std::tuple<int, int, int>, float2*> g_ring_tw;
int ring_twiddles(int l1, int l2, const float2** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return XFT_ECUDA;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  auto key = std::make_tuple(dev, l1, l2);
  auto it = g_ring_tw.find(key);
  if (it == g_ring_tw.end()) {
    const int R1 = 1 << l1, R2 = 1 << l2;
    const long long R = (long long)R1 * R2;
    std::vector<float2> h((size_t)R);
    for (int r2 = 0; r2 < R2; ++r2)
      for (int k1 = 0; k1 < R1; ++k1) {
        const long long m = ((long long)k1 * r2) % R;
        const long double th = 2.0L * PI_L * (long double)m / (long double)R;
        h[(size_t)r2 * R1 + k1] = make_float2((float)cosl(th), (float)-sinl(th));
      }
    float2* p = nullptr;
    if (cudaMalloc(&p, sizeof(float2) * R) != cudaSuccess) return XFT_ECUDA;
    if (cudaMemcpy(p, h.data(), sizeof(float2) * R, cudaMemcpyHostToDevice) != cudaSuccess) return XFT_ECUDA;
    it = g_ring_tw.emplace(key, p).first;
  }
  *out = it->second;
  return XFT_OK;
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
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::THREADS + 32, Cfg::SMEM) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    return XFT_ENOTSUP;
  }
  if (probe) return XFT_OK;
  RingPlan pl{};
  pl.R1 = R1;
  pl.R2 = R2;
  pl.nblocks = (int)((ncols + W - 1) / W);
  pl.SB = XFT_RING_SB;
  while (pl.nblocks % pl.SB) pl.SB /= 2;
  pl.nsb = pl.nblocks / pl.SB;
  pl.lag = pl.nsb < XFT_RING_LAG ? pl.nsb : XFT_RING_LAG;
  pl.slots = pl.nsb < XFT_RING_SLOTS ? pl.nsb : XFT_RING_SLOTS;
  pl.T0 = (unsigned)(pl.SB * R2);
  pl.T1 = (unsigned)(pl.SB * R1);
  pl.tA = (unsigned)pl.lag * pl.T0;
  pl.tB = (unsigned)(pl.nsb - pl.lag) * (pl.T0 + pl.T1);
  pl.total = pl.tA + pl.tB + (unsigned)pl.lag * pl.T1;
  pl.ld_in = ld;
  pl.ld_out = ld_out;
  pl.ncols = (int)ncols;
  // scratch: ring, pre/post table rows, counters
  const size_t ring_bytes = (size_t)pl.slots * pl.SB * R * W * sizeof(float2);
  const size_t tab_bytes = (size_t)R * sizeof(float2);
  const int ncounters = 1 + 2 * pl.nsb;
  const size_t ctr_bytes = ((size_t)ncounters * 4 + 255) / 256 * 256;
  char* base = static_cast<char*>(stream_scratch(dev, st, ring_bytes + 2 * tab_bytes + ctr_bytes));
  if (!base) return XFT_ECUDA;
  RingBufs bf{};
  bf.ring = reinterpret_cast<float2*>(base);
  float2* pre = reinterpret_cast<float2*>(base + ring_bytes);
  float2* post = reinterpret_cast<float2*>(base + ring_bytes + tab_bytes);
  bf.pre = pre;
  bf.post = post;
  bf.ticket = reinterpret_cast<unsigned*>(base + ring_bytes + 2 * tab_bytes);
  bf.done1 = bf.ticket + 1;
  bf.done2 = bf.done1 + pl.nsb;
  int rc = ring_twiddles(LOG1, LOG2, &bf.twr);
  if (rc) return rc;
  Tables t1, t2;
  if ((rc = get_tables(R1, XFT_C64, &t1, Cfg::E1))) return rc;
  if ((rc = get_tables(R2, XFT_C64, &t2, Cfg::E2))) return rc;
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)ncols, (cuuint64_t)R2, (cuuint64_t)R1};
  const cuuint64_t strides[2] = {(cuuint64_t)(ld * sizeof(float2)), (cuuint64_t)(R2 * ld * sizeof(float2))};
  const cuuint32_t box[3] = {(cuuint32_t)W, 1u, (cuuint32_t)R1};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(in), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return XFT_ENOTSUP;
  const int nset = (int)((R > ncounters ? R : ncounters) + 255) / 256;
  ring_setup_kernel<<<nset, 256, 0, st>>>(pre, post, bf.ticket, ncounters, ck, R1, R2);
  const long long cap = (long long)sms * occ;
  const unsigned grid = (unsigned)(pl.total < cap ? pl.total : cap);
  kern<<<grid, Cfg::THREADS + 32, Cfg::SMEM, st>>>(map, static_cast<float2*>(out), pl, bf, static_cast<const float2*>(t1.tw),
                                              static_cast<const float2*>(t2.tw));
  return cudaGetLastError() == cudaSuccess ? XFT_OK : XFT_ECUDA;
}

// c64 columns of height 2^12 .. 2^16 (R1 x R2 = 64x64 .. 256x256); anything else: XFT_ENOTSUP, nothing launched
inline int lct_cols_ring(const void* in, void* out, int64_t R, int64_t ncols, int64_t ld, int64_t ld_out,
                         const ColChirp& ck, cudaStream_t st, bool probe = false) {
  if (!XFT_COLRING) return XFT_ENOTSUP;
  switch (log2_of(R)) {
    case 12: return launch_colring<6, 6>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 13: return launch_colring<7, 6>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 14: return launch_colring<7, 7>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 15: return launch_colring<8, 7>(in, out, ncols, ld, ld_out, ck, st, probe);
    case 16: return launch_colring<8, 8>(in, out, ncols, ld, ld_out, ck, st, probe);
    default: return XFT_ENOTSUP;
  }
}
