"""GPU parity for the separable 2-D LCT (BASELINE config 5) and its sharded building blocks."""
import math

import numpy as np
import pytest

from oracle import xft_oracle as O
from tests.conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    if not _t.cuda.is_available():
        pytest.skip("no CUDA device")
    return _t


@pytest.fixture(scope="module")
def L2():
    from paper_0912_1379_b200 import lct2d

    return lct2d


ABCD5 = (1.0, 0.25, 0.0, 1.0)


@pytest.mark.parametrize("shape,dtype,tol", [((64, 64), np.complex128, 1e-12), ((2048, 256), np.complex128, 1e-12),
                                             ((256, 2048), np.complex64, 2e-5), ((4096, 64), np.complex64, 2e-5),
                                             ((100, 48), np.complex128, 1e-12),
                                             # slab route (row pass into 8 column slabs, cluster columns)
                                             ((2048, 2048), np.complex128, 1e-12), ((4096, 2048), np.complex64, 2e-5),
                                             ((4096, 1024), np.complex64, 2e-5), ((8192, 528), np.complex64, 2e-5),
                                             # L2-staged columns (K7): several super-blocks, ring slots reused,
                                             # a ragged last block
                                             ((16384, 528), np.complex64, 2e-5)])
def test_lct2d_vs_oracle(torch, L2, shape, dtype, tol):
    rng = np.random.default_rng(5)
    f = (rng.normal(size=shape) + 1j * rng.normal(size=shape)).astype(dtype)
    pr, pc = ABCD5, (0.5, 1.5, -0.5, 0.5)
    got = L2.lct2d(torch.from_numpy(f).cuda(), pr, pc).cpu().numpy()
    ref = O.lct2d(pr, pc, f.astype(complex))
    assert rel_l2(got, ref) <= tol


@pytest.mark.parametrize("n,G", [(1024, 4), (4096, 4)])
def test_packed_rows_and_columns_emulate_shards(torch, L2, n, G):
    """G virtual shards on one GPU: packed row pass per shard, the all-to-all as a copy, column pass per slab."""
    rng = np.random.default_rng(9)
    f = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)
    ft = torch.from_numpy(f).cuda()
    rl, nc = n // G, n // G
    sends = [L2.rows_packed(ft[g * rl:(g + 1) * rl], ABCD5, G) for g in range(G)]
    full = L2.lct2d(ft, ABCD5, ABCD5)
    for h in range(G):  # rank h receives block h of every source, stacked by source rank
        slab = torch.cat([sends[g][h] for g in range(G)], dim=0).contiguous()
        L2.columns_inplace(slab, ABCD5)
        assert rel_l2(slab.cpu().numpy(), full[:, h * nc:(h + 1) * nc].cpu().numpy()) <= 1e-6


def test_config5_full(torch, L2):
    """Config 5 at full size (16384^2 c64, 2 GiB): norm identity + sampled rows/columns against the oracle."""
    from paper_0912_1379_b200 import ops, workloads

    n = 16384
    field = workloads.config5_field(n)
    ft = torch.from_numpy(field).cuda()
    out = L2.lct2d(ft, ABCD5, ABCD5)
    # ||G||^2 = (pi / (4 |b|))^2 ||f||^2  (unitary up to the kernel scale on each axis)
    lhs = float((out.to(torch.complex128).abs() ** 2).sum())
    rhs = (math.pi / (4 * 0.25)) ** 2 * float((ft.to(torch.complex128).abs() ** 2).sum())
    assert abs(lhs / rhs - 1) <= 1e-4
    # intermediate rows (axis 1) checked against the oracle on sampled rows ...
    rows = ops.lct_rows(ft, ABCD5)
    for r in (0, 4321, n // 2, n - 1):
        _, ref = O.fast_lct_rows(ABCD5, field[r].astype(complex))
        assert rel_l2(rows[r].cpu().numpy(), ref) <= 2e-5
    # ... and sampled output columns = oracle column LCT of the (verified) row pass
    rows_h = rows.cpu().numpy()
    outh = out.cpu().numpy()
    for c in (0, 777, n // 2, n - 1):
        _, ref = O.fast_lct_rows(ABCD5, rows_h[:, c].astype(complex))
        assert rel_l2(outh[:, c], ref) <= 2e-5


@pytest.mark.parametrize("R", [2048, 4096, 8192, 16384, 32768, 65536])
@pytest.mark.parametrize("dtype,tol", [(np.complex64, 2e-5), (np.complex128, 1e-12)])
@pytest.mark.parametrize("inplace", [True, False])
def test_columns_tall(torch, L2, R, dtype, tol, inplace):
    """Tall column LCTs (the cluster path: K CTAs x 1024 rows share a column group through DSMEM).

    Strided slab (row stride ld > n_cols), in place and out of place, against the
    oracle's per-column fast_lct (xft/lct.py:168-208 down each column).
    """
    from paper_0912_1379_b200 import _native, ops

    if R > 16384 and dtype == np.complex128:
        pytest.skip("c128 columns above 16384 rows: not a path of the 2-D transform (xft_lct2d transposes instead)")
    nc, ld = (24, 40) if dtype == np.complex64 else (12, 20)
    rng = np.random.default_rng(R + nc)
    full = (rng.normal(size=(R, ld)) + 1j * rng.normal(size=(R, ld))).astype(dtype)
    src = torch.from_numpy(full).cuda()
    dst = src if inplace else torch.zeros_like(src)
    ws = torch.empty_like(src)
    p = np.array((0.5, 1.5, -0.5, 0.5))
    _native.call("xft_lct_columns", src.data_ptr(), dst.data_ptr(), R, nc, ld, ops._dtype_code(src), p.ctypes.data,
                 ws.data_ptr(), ops._stream_ptr(src.device))
    got = dst.cpu().numpy()
    _, ref = O.fast_lct_rows(tuple(p), full[:, :nc].T.astype(complex))
    assert rel_l2(got[:, :nc], ref.T) <= tol
    if not inplace:
        assert np.all(got[:, nc:] == 0)  # columns outside the slab untouched
    else:
        assert np.array_equal(got[:, nc:], full[:, nc:])


@pytest.mark.parametrize("n,dtype,tol", [(2048, np.complex64, 1e-6), (512, np.complex128, 1e-13)])
@pytest.mark.parametrize("transport", ["nccl", "capi"])
def test_sharded_over_nccl_world1(torch, L2, tmp_path, n, dtype, tol, transport):
    """lct2d_sharded through a real NCCL process group (one rank: the only GPU of this box):
    packed row pass -> ncclAllToAll (all_to_all_single) -> column pass on the received slab."""
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group is already active")
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(17)
        f = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(dtype)
        ft = torch.from_numpy(f).cuda()
        got = L2.lct2d_sharded(ft, ABCD5, (0.5, 1.5, -0.5, 0.5), transport=transport)
        torch.cuda.synchronize()
        ref = L2.lct2d(ft, ABCD5, (0.5, 1.5, -0.5, 0.5))
        assert got.shape == (n, n)
        assert rel_l2(got.cpu().numpy(), ref.cpu().numpy()) <= tol
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,dtype,tol", [(4, np.complex64, 1e-6), (2, np.complex128, 1e-13), (8, np.complex64, 1e-6)])
def test_peer_store_rows_emulate_shards(torch, L2, G, dtype, tol):
    """xft_lct_rows_peers with G virtual ranks on one GPU: each 'rank' stores its row segments straight
    into the G receive slabs (the NVLink peer-store all-to-all); the slabs then hold the column blocks."""
    n = 1024
    rng = np.random.default_rng(21)
    f = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(dtype)
    ft = torch.from_numpy(f).cuda()
    rl, nc = n // G, n // G
    slabs = [torch.full((n, nc), float("nan"), dtype=ft.dtype, device=ft.device) for _ in range(G)]
    ptrs = [s.data_ptr() for s in slabs]
    for g in range(G):
        L2.rows_to_peers(ft[g * rl:(g + 1) * rl], ABCD5, ptrs, g * rl)
    full = L2.lct2d(ft, ABCD5, ABCD5)
    for h in range(G):
        L2.columns_inplace(slabs[h], ABCD5)
        assert rel_l2(slabs[h].cpu().numpy(), full[:, h * nc:(h + 1) * nc].cpu().numpy()) <= tol


def test_sharded_p2p_symmetric_memory_world1(torch, L2, tmp_path):
    """lct2d_sharded(transport="p2p") through torch symmetric memory (one rank on this box's one GPU)."""
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group is already active")
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 2048
        rng = np.random.default_rng(23)
        f = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)
        ft = torch.from_numpy(f).cuda()
        try:
            got = L2.lct2d_sharded(ft, ABCD5, (0.5, 1.5, -0.5, 0.5), transport="p2p").clone()
        except (RuntimeError, NotImplementedError) as e:  # no symmetric-memory backend on this box
            pytest.skip(f"symmetric memory unavailable: {e}")
        ref = L2.lct2d(ft, ABCD5, (0.5, 1.5, -0.5, 0.5))
        assert rel_l2(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-6
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_slab_route_without_cluster_kernel(torch):
    """The single-GPU 2-D slab route on a build without the cluster column kernel (XFT_COLCLU=0,
    the path MIG/MPS devices take when no 16-CTA cluster fits) gives the default build's result."""
    import os
    import subprocess

    from paper_0912_1379_b200 import _native, lct2d

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = os.path.join(root, "tune", "libxft_noclu.so")
    if not os.path.exists(so):
        subprocess.run(["bash", os.path.join(root, "tools", "build_variant.sh"), "noclu", "-DXFT_COLCLU=0"],
                       check=True, timeout=900)
    rng = np.random.default_rng(21)
    n = 2048
    f = torch.from_numpy((rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)).cuda()
    p = (1.0, 0.25, 0.0, 1.0)
    ref = lct2d.lct2d(f, p, p)
    saved = _native.lib()
    try:
        _native._lib = _native.load_library(so)
        got = lct2d.lct2d(f, p, p)
        torch.cuda.synchronize()
    finally:
        _native._lib = saved
    err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert err <= 2e-6, err


def test_capi_sharded_on_a_caller_owned_nccl_comm(torch, L2):
    """xft_lct2d_sharded driven the way a non-torch caller drives it: its own ncclComm_t
    (ncclGetUniqueId + ncclCommInitRank through ctypes, one rank), raw device pointers."""
    import ctypes
    import os

    import nvidia.nccl

    from paper_0912_1379_b200 import _native

    nccl = ctypes.CDLL(os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2"))

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]

    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    try:
        n = 2048
        rng = np.random.default_rng(23)
        f = torch.from_numpy((rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)).cuda()
        send, slab, ws = torch.empty_like(f), torch.empty_like(f), torch.empty_like(f)
        pr = np.array(ABCD5, dtype=np.float64)
        pc = np.array((0.5, 1.5, -0.5, 0.5), dtype=np.float64)
        s = torch.cuda.current_stream().cuda_stream
        _native.call("xft_lct2d_sharded", f.data_ptr(), slab.data_ptr(), send.data_ptr(), n, n, _native.C64,
                     pr.ctypes.data, pc.ctypes.data, comm.value, ws.data_ptr(), s)
        torch.cuda.synchronize()
        ref = L2.lct2d(f, ABCD5, (0.5, 1.5, -0.5, 0.5))
        assert rel_l2(slab.cpu().numpy(), ref.cpu().numpy()) <= 1e-6
        # shape contract: rows_local * world must tile n
        from paper_0912_1379_b200.errors import ShapeError

        with pytest.raises(ShapeError):
            _native.call("xft_lct2d_sharded", f.data_ptr(), slab.data_ptr(), send.data_ptr(), n // 2, n,
                         _native.C64, pr.ctypes.data, pc.ctypes.data, comm.value, ws.data_ptr(), s)
    finally:
        nccl.ncclCommDestroy(comm)


@pytest.mark.slow
def test_config5_256_rows_and_256_columns_independent(torch, L2):
    """Config 5 at full size: 256 output columns and 256 output rows against an oracle that shares
    nothing with the GPU path.  Output column c = fast_lct(F L[c, :]^T) and output row r =
    fast_lct(L[r, :] F): the dense LCT rows L[j, :] restate xft/dense.py:162-171 exactly
    (oracle.dense_lct_rows, pinned bit for bit to the reference's matrix), the contraction with the
    c64-rounded field runs in complex128 (a plain ZGEMM), the final 1-D transform is the oracle's
    fast_lct.  Tolerance: the complex64 bar (2e-5 per line)."""
    from paper_0912_1379_b200 import workloads

    n = 16384
    field = workloads.config5_field(n)
    ft = torch.from_numpy(field).cuda()
    out = L2.lct2d(ft, ABCD5, ABCD5).cpu().numpy()
    f128 = ft.to(torch.complex128)
    del ft
    rng = np.random.default_rng(55)
    idx = np.unique(np.concatenate([[0, n // 2, n - 1], rng.choice(n, 253, replace=False)]))[:256]
    Lsel = torch.from_numpy(O.dense_lct_rows(ABCD5, n, idx)).cuda()   # [256, n] rows of L
    cols_in = (f128 @ Lsel.T).T.contiguous().cpu().numpy()             # [256, n]: F L[c, :]^T
    rows_in = (Lsel @ f128).cpu().numpy()                              # [256, n]: L[r, :] F
    del f128
    _, want_cols = O.fast_lct_rows(ABCD5, cols_in)
    _, want_rows = O.fast_lct_rows(ABCD5, rows_in)
    for i, c in enumerate(idx):
        assert rel_l2(out[:, c], want_cols[i]) <= 2e-5, ("column", c)
        assert rel_l2(out[c, :], want_rows[i]) <= 2e-5, ("row", c)


def test_config5_every_element_two_routes(torch, L2):
    """Config 5 at full size, every one of the 2^28 outputs: the 2-D transform (row kernel, then the L2-staged
    column kernel) against the same transform done with the row kernel alone on both axes (rows, transpose,
    rows, transpose) -- the 1-D row kernel is what the golden vectors, the full config-2/4 batches and the
    random sweep pin to the oracle.  Two independent c64 roundings: per-column relative L2 <= 2e-5."""
    from paper_0912_1379_b200 import ops, workloads

    n = 16384
    ft = torch.from_numpy(workloads.config5_field(n)).cuda()
    out = L2.lct2d(ft, ABCD5, ABCD5)
    rows = ops.lct_rows(ft, ABCD5)
    # 512 rows of the row pass, and below 512 of the transposed pass, against the oracle itself
    pick = np.unique(np.concatenate([[0, n // 2, n - 1], np.random.default_rng(5).choice(n, 509, replace=False)]))
    _, want = O.fast_lct_rows(ABCD5, ft[pick].cpu().numpy().astype(np.complex128))
    got = rows[pick].cpu().numpy()
    assert max(rel_l2(got[i], want[i]) for i in range(len(pick))) <= 2e-5
    del ft
    rt = rows.T.contiguous()
    del rows
    ref_t = ops.lct_rows(rt, ABCD5)  # [column, row]: the column LCTs as rows of the transposed field
    _, want = O.fast_lct_rows(ABCD5, rt[pick].cpu().numpy().astype(np.complex128))
    got = ref_t[pick].cpu().numpy()
    assert max(rel_l2(got[i], want[i]) for i in range(len(pick))) <= 2e-5
    del rt
    num = torch.zeros(n, dtype=torch.float64, device="cuda")
    den = torch.zeros(n, dtype=torch.float64, device="cuda")
    for c0 in range(0, n, 2048):  # per output column, in slabs (bounded temporaries)
        a = out[:, c0:c0 + 2048].to(torch.complex128)
        b = ref_t[c0:c0 + 2048, :].T.to(torch.complex128)
        num[c0:c0 + 2048] = ((a - b).abs() ** 2).sum(dim=0)
        den[c0:c0 + 2048] = (b.abs() ** 2).sum(dim=0)
    err = float(torch.sqrt(num / den).max())
    assert err <= 2e-5, err


@pytest.mark.parametrize("nc,ld", [(64, 64), (65, 66), (200, 256), (1000, 1024)])
def test_ring_columns_ragged_and_repeatable(torch, L2, nc, ld):
    """The L2-staged column kernel (16384 rows, c64) on ragged slabs: partial last 64-column block, row
    stride > width.  In place == out of place bit for bit, repeated runs identical (the schedule has no
    data-dependent order), columns beyond the slab untouched, sampled columns against the oracle."""
    from paper_0912_1379_b200 import _native, ops

    R = 16384
    rng = np.random.default_rng(nc)
    full = (rng.normal(size=(R, ld)) + 1j * rng.normal(size=(R, ld))).astype(np.complex64)
    p = np.array((0.5, 1.5, -0.5, 0.5))
    src = torch.from_numpy(full).cuda()
    ws = torch.empty_like(src)

    def run(dst):
        _native.call("xft_lct_columns", src.data_ptr() if dst is not src else dst.data_ptr(), dst.data_ptr(), R, nc, ld,
                     ops._dtype_code(src), p.ctypes.data, ws.data_ptr(), ops._stream_ptr(src.device))
        return dst.cpu().numpy()

    a = run(torch.full_like(src, 7.0))
    b = run(torch.full_like(src, 7.0))
    assert np.array_equal(a, b)
    if ld > nc:
        assert np.all(a[:, nc:] == 7.0)
    c = run(src)  # in place (src is overwritten: last)
    assert np.array_equal(c[:, :nc], a[:, :nc])
    if ld > nc:
        assert np.array_equal(c[:, nc:], full[:, nc:])
    for col in sorted({0, nc // 2, nc - 1}):
        _, ref = O.fast_lct_rows(tuple(p), full[:, col].astype(complex))
        assert rel_l2(a[:, col], ref) <= 2e-5
