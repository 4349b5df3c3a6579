"""Separable 2-D LCT: fast LCT along axis 1 (rows), then along axis 0 (columns).

No reference symbol exists; the transform is defined as the composition of
the reference 1-D ``fast_lct`` (xft/lct.py:168-208) along both axes
(last row).

* ``lct2d`` -- one GPU: row kernel, then the column kernels (``xft_lct2d``).
* ``lct2d_sharded`` -- G ranks (one process per GPU, torch.distributed/NCCL):
  rank g holds rows [g n/G, (g+1) n/G).  The row kernel writes its output
  directly in the all-to-all send layout (segment h of every row goes to the
  block for rank h), one ``all_to_all_single`` over NVLink delivers to every
  rank the full height of its n/G columns as a row-major [n, n/G] slab, and the
  column kernels transform that slab in place.  The result stays column-sharded:
  rank g returns columns [g n/G, (g+1) n/G) of the 2-D transform.
"""
from __future__ import annotations

import numpy as np

from . import _native, ops
from .errors import ShapeError


def _abcd4(p):
    a = np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(4))
    return a


def lct2d(field, abcd_row, abcd_col=None, *, out=None, workspace=None):
    """2-D LCT of a [n_rows, n_cols] complex CUDA tensor on one GPU."""
    torch = ops._torch()
    if abcd_col is None:
        abcd_col = abcd_row
    if field.dim() != 2 or not field.is_cuda:
        raise ShapeError("lct2d needs a 2-D CUDA tensor")
    f = ops.aligned(field)
    r, c = f.shape
    pr, pc = _abcd4(abcd_row), _abcd4(abcd_col)
    out = ops.check_out(out, f)
    workspace = ops.check_out(workspace, f)
    with torch.cuda.device(f.device):
        _native.call("xft_lct2d", f.data_ptr(), out.data_ptr(), r, c, ops._dtype_code(f),
                     pr.ctypes.data, pc.ctypes.data, workspace.data_ptr(), ops._stream_ptr(f.device))
    return out


# ---- device building blocks of the sharded transform ------------------------
def rows_packed(local, abcd_row, world: int, out=None):
    """Row LCT of the local [rl, n] rows written as the all-to-all send buffer [world, rl, n/world]."""
    torch = ops._torch()
    rl, n = local.shape
    nc = n // world
    if nc * world != n or nc & (nc - 1):
        raise ShapeError(f"n = {n} must split into {world} power-of-two column blocks")
    local = ops.aligned(local)
    out = ops.check_out(out, local, (world, rl, nc))
    p = _abcd4(abcd_row)
    with torch.cuda.device(local.device):
        _native.call("xft_lct_rows_packed", local.data_ptr(), out.data_ptr(), rl, n, ops._dtype_code(local),
                     p.ctypes.data, int(nc).bit_length() - 1, rl * nc, ops._stream_ptr(local.device))
    return out


def rows_to_peers(local, abcd_row, peer_ptrs, row0: int):
    """Row LCT of the local [rl, n] rows whose epilogue stores segment h of row r
    straight into peer slab h ([n, n/G] row-major, device pointer peer_ptrs[h]) at
    row row0 + r: the all-to-all of the sharded transform done by the row kernel's
    own NVLink stores (``xft_lct_rows_peers``).  The caller synchronises the ranks
    before the column pass reads its slab."""
    import ctypes

    rl, n = local.shape
    G = len(peer_ptrs)
    if not 1 <= G <= 8 or n % G:
        raise ShapeError(f"{G} peers do not split n = {n}")
    ptrs = (ctypes.c_uint64 * G)(*[int(p) for p in peer_ptrs])
    p = _abcd4(abcd_row)
    torch = ops._torch()
    with torch.cuda.device(local.device):
        _native.call("xft_lct_rows_peers", local.data_ptr(), ctypes.addressof(ptrs), G, int(row0), rl, n,
                     ops._dtype_code(local), p.ctypes.data, ops._stream_ptr(local.device))


def columns_inplace(slab, abcd_col, workspace=None):
    """Column LCT of a row-major [n, nc] slab, in place."""
    torch = ops._torch()
    n, nc = slab.shape
    if not slab.is_contiguous() or slab.data_ptr() % ops.ALIGN:
        raise ShapeError("the column slab is transformed in place: it must be contiguous and 16-byte aligned")
    p = _abcd4(abcd_col)
    if n > 1024:
        workspace = ops.check_out(workspace, slab)
    with torch.cuda.device(slab.device):
        _native.call("xft_lct_columns", slab.data_ptr(), slab.data_ptr(), n, nc, nc, ops._dtype_code(slab),
                     p.ctypes.data, 0 if workspace is None else workspace.data_ptr(), ops._stream_ptr(slab.device))
    return slab


_P2P = {}  # (group, n, dtype, device) -> (symmetric receive slab, its rendezvous handle)
_COMMS = {}  # (group, device) -> ncclComm_t of the "capi" transport


def _capi_comm(group, device):
    """An NCCL communicator of our own over ``group``'s ranks, made the way a non-torch caller makes
    one (ncclGetUniqueId on rank 0, broadcast, ncclCommInitRank), for ``xft_lct2d_sharded``."""
    import ctypes
    import os

    import nvidia.nccl
    import torch
    import torch.distributed as dist

    key = (id(group), str(device))
    if key not in _COMMS:
        nccl = ctypes.CDLL(os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2"))

        class UniqueId(ctypes.Structure):
            _fields_ = [("internal", ctypes.c_char * 128)]

        uid = UniqueId()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if rank == 0 and nccl.ncclGetUniqueId(ctypes.byref(uid)) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        box = [bytes(uid.internal) if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid.internal = box[0]
        comm = ctypes.c_void_p()
        with torch.cuda.device(device):
            if nccl.ncclCommInitRank(ctypes.byref(comm), world, uid, rank) != 0:
                raise RuntimeError("ncclCommInitRank failed")
        _COMMS[key] = comm.value
    return _COMMS[key]


def _p2p_slab(group, n, nc, dtype, device):
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    key = (dist.get_group_rank(group, dist.get_rank()) if group is not None else dist.get_rank(),
           id(group), n, dtype, str(device))
    if key not in _P2P:
        slab = symm.empty((n, nc), dtype=dtype, device=device)
        _P2P[key] = (slab, symm.rendezvous(slab, group if group is not None else dist.group.WORLD))
    return _P2P[key]


def lct2d_sharded(local, abcd_row, abcd_col=None, *, group=None, row_fn=None, col_fn=None, buffers=None,
                  transport="nccl"):
    """Sharded 2-D LCT over the ranks of ``group``.

    ``local``: this rank's [n/G, n] rows.  Returns this rank's [n, n/G] column
    slab of the result.  ``row_fn(local, abcd, world) -> send[world, rl, nc]``
    and ``col_fn(slab, abcd) -> slab`` default to the CUDA kernels; tests on
    CPU (gloo) substitute the CPU oracle to check the orchestration/layout.
    ``buffers``: optional preallocated (send, recv) of shape [world, rl, nc].

    ``transport``: "nccl" -- packed row pass, ``all_to_all_single``, column pass;
    "p2p" -- the row kernel stores every segment straight into the owning
    rank's symmetric-memory receive slab over NVLink (no separate collective,
    ``xft_lct_rows_peers``), two device-side barriers, column pass in place.
    The p2p result is that persistent slab: the next p2p call of the same shape
    overwrites it.  "capi" -- the whole sharded transform through the C ABI
    (``xft_lct2d_sharded``) on an NCCL communicator of its own over the group's
    ranks (made with the plain NCCL API): the route a non-torch caller takes
    with its ncclComm_t.
    """
    import torch
    import torch.distributed as dist

    if abcd_col is None:
        abcd_col = abcd_row
    world = dist.get_world_size(group)
    rl, n = local.shape
    if rl * world != n:
        raise ShapeError(f"{world} ranks x {rl} rows do not tile an n = {n} field")
    nc = n // world
    if transport == "p2p":
        rank = dist.get_rank(group)
        slab, hdl = _p2p_slab(group, n, nc, local.dtype, local.device)
        hdl.barrier()  # every rank's slab is free (previous column pass done)
        rows_to_peers(local, abcd_row, list(hdl.buffer_ptrs), rank * rl)
        hdl.barrier()  # every rank's stores into this slab have landed
        return (col_fn or columns_inplace)(slab, abcd_col)
    if transport == "capi":
        comm = _capi_comm(group, local.device)
        local = ops.aligned(local)
        send = ops.check_out(None if buffers is None else buffers[0], local, (world, rl, nc))
        slab = ops.check_out(None if buffers is None else buffers[1].view(n, nc), local, (n, nc))
        ws = torch.empty((n, nc), dtype=local.dtype, device=local.device) if n > 1024 else None
        pr, pc = _abcd4(abcd_row), _abcd4(abcd_col)  # held: the call reads them through raw pointers
        with torch.cuda.device(local.device):
            _native.call("xft_lct2d_sharded", local.data_ptr(), slab.data_ptr(), send.data_ptr(), rl, n,
                         ops._dtype_code(local), pr.ctypes.data, pc.ctypes.data,
                         int(comm), None if ws is None else ws.data_ptr(), ops._stream_ptr(local.device))
        return slab
    if transport != "nccl":
        raise ValueError(f"transport must be 'nccl', 'p2p' or 'capi', got {transport!r}")
    row_fn = row_fn or (lambda x, p, w: rows_packed(x, p, w, out=None if buffers is None else buffers[0]))
    col_fn = col_fn or columns_inplace
    send = row_fn(local, abcd_row, world)
    recv = torch.empty_like(send) if buffers is None else buffers[1]
    dist.all_to_all_single(recv.view(-1), send.view(-1), group=group)
    return col_fn(recv.view(n, nc), abcd_col)
