// Sharded separable 2-D LCT over NCCL (SURVEY 8(b) "xft_lct2d(..., ncclComm_t, stream)",
// 8(e) steps 1-4): the C-ABI route for callers that hold their own NCCL
// communicator (no torch).  Rank g owns rows [g n/G, (g+1) n/G) of the field:
//   1. row LCT of the local rows, written straight into the all-to-all send
//      layout [G][rl][n/G] by the row kernel's segmented epilogue;
//   2. one all-to-all over NVLink (grouped ncclSend/ncclRecv, byte counts);
//      the receive buffer IS the row-major [n][n/G] column slab of rank g;
//   3. column LCT of that slab in place (cluster kernel for tall columns).
// The result stays column-sharded (8(e) step 4).  NCCL is resolved at run time
// from the caller's process (the library has no link-time NCCL dependency):
// the communicator's own library is already loaded when a caller passes one.
#include <dlfcn.h>

#include <mutex>

#include "../../include/xft_b200.h"
#include "xft_internal.h"

using namespace xftb;

namespace {

typedef int (*NcclGroupFn)();
typedef int (*NcclP2PFn)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*NcclRecvFn)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*NcclCommIntFn)(const void*, int*);
typedef int (*NcclVersionFn)(int*);

struct Nccl {
  NcclGroupFn group_start = nullptr, group_end = nullptr;
  NcclP2PFn send = nullptr;
  NcclRecvFn recv = nullptr;
  NcclCommIntFn count = nullptr, rank = nullptr;
  NcclVersionFn version = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, []() {
    void* h = RTLD_DEFAULT;
    if (!dlsym(h, "ncclSend")) {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy the caller already loaded
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    }
    if (!h) return;
    n.group_start = reinterpret_cast<NcclGroupFn>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<NcclGroupFn>(dlsym(h, "ncclGroupEnd"));
    n.send = reinterpret_cast<NcclP2PFn>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<NcclRecvFn>(dlsym(h, "ncclRecv"));
    n.count = reinterpret_cast<NcclCommIntFn>(dlsym(h, "ncclCommCount"));
    n.rank = reinterpret_cast<NcclCommIntFn>(dlsym(h, "ncclCommUserRank"));
    n.version = reinterpret_cast<NcclVersionFn>(dlsym(h, "ncclGetVersion"));
    n.ok = n.group_start && n.group_end && n.send && n.recv && n.count && n.rank;
  });
  return n;
}

constexpr int NCCL_UINT8 = 1;  // ncclUint8: the exchange moves bytes, no arithmetic

int log2_pow2(int64_t v) {
  if (v < 1 || (v & (v - 1))) return -1;
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

}  // namespace

extern "C" {

int xft_nccl_info(char* path, int path_len, int* version) {
  const Nccl& nc = nccl();
  if (!nc.ok) return XFT_ENOTSUP;
  if (version) {
    *version = 0;
    if (nc.version) nc.version(version);
  }
  if (path && path_len > 0) {
    Dl_info info{};
    path[0] = 0;
    if (dladdr(reinterpret_cast<void*>(nc.send), &info) && info.dli_fname) {
      int i = 0;
      for (; info.dli_fname[i] && i < path_len - 1; ++i) path[i] = info.dli_fname[i];
      path[i] = 0;
    }
  }
  return XFT_OK;
}

int xft_lct2d_sharded(const void* local, void* slab, void* send, int64_t rows_local, int64_t n, int dtype,
                      const double* abcd_row, const double* abcd_col, void* nccl_comm, void* workspace,
                      void* stream) {
  if (n < 1 || rows_local < 1) return XFT_EINVALID_SIZE;
  if (dtype != XFT_C64 && dtype != XFT_C128) return XFT_EPARAM;
  int rc = xft_validate_lct_params(abcd_row, 1, 0, 1, 1e-10, nullptr);
  if (!rc) rc = xft_validate_lct_params(abcd_col, 1, 0, 1, 1e-10, nullptr);
  if (rc) return rc;
  int world = 1, me = 0;
  const Nccl* nc = nullptr;
  if (nccl_comm) {
    nc = &nccl();
    if (!nc->ok) return XFT_ENOTSUP;
    if (nc->count(nccl_comm, &world) != 0 || nc->rank(nccl_comm, &me) != 0) return XFT_ECUDA;
  }
  if (rows_local * world != n) return XFT_ESHAPE;  // the ranks' row blocks must tile the field
  const int64_t ncol = n / world;
  const int segl = log2_pow2(ncol);
  if (segl < 0 || ncol * world != n) return XFT_ESHAPE;
  auto st = static_cast<cudaStream_t>(stream);
  const size_t esz = dtype == XFT_C64 ? 8 : 16;
  (void)me;
  // 1. row pass into the send layout (no communicator: straight into the slab)
  void* rows_out = nccl_comm ? send : slab;
  if (!rows_out) return XFT_EPARAM;
  rc = xft_lct_rows_packed(local, rows_out, rows_local, n, dtype, abcd_row, segl, rows_local * ncol, stream);
  if (rc) return rc;
  // 2. all-to-all: block h of the send buffer -> rank h, rank g's block lands at rows [g rl, (g+1) rl)
  if (nccl_comm) {  // (a one-rank communicator exchanges with itself)
    const size_t bytes = esz * (size_t)rows_local * ncol;
    if (nc->group_start() != 0) return XFT_ECUDA;
    int bad = 0;
    for (int h = 0; h < world; ++h) {
      bad |= nc->send(static_cast<const char*>(send) + h * bytes, bytes, NCCL_UINT8, h, nccl_comm, st);
      bad |= nc->recv(static_cast<char*>(slab) + h * bytes, bytes, NCCL_UINT8, h, nccl_comm, st);
    }
    if (nc->group_end() != 0 || bad) return XFT_ECUDA;
  }
  // 3. column pass on the [n][n/G] slab, in place
  return xft_lct_columns(slab, slab, n, ncol, ncol, dtype, abcd_col, workspace, stream);
}

}  // extern "C"
