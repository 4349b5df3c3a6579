"""Sharded 2-D LCT orchestration on CPU: world_size 2 over gloo.

The row/column transforms are the CPU oracle here (the CUDA kernels cannot run
without a GPU); what is under test is the sharded layout contract -- the row
pass writes segment h of every local row into the send block of rank h, one
all_to_all_single delivers a row-major [n, n/G] column slab, the column pass
runs on it -- against the oracle's full 2-D transform.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import xft_oracle as O

ABCD_R = (1.0, 0.25, 0.0, 1.0)
ABCD_C = (0.5, 1.5, -0.5, 0.5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_rows(local, abcd, world):
    # oracle row LCT, then the send layout [world, rl, nc] (segment h of row r -> block h)
    _, v = O.fast_lct_rows(abcd, local.numpy())
    rl, n = v.shape
    nc = n // world
    return torch.from_numpy(np.ascontiguousarray(v.reshape(rl, world, nc).transpose(1, 0, 2)))


def _cpu_cols(slab, abcd):
    _, v = O.fast_lct_rows(abcd, np.ascontiguousarray(slab.numpy().T))
    slab.copy_(torch.from_numpy(np.ascontiguousarray(v.T)))
    return slab


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_0912_1379_b200.lct2d import lct2d_sharded

        rng = np.random.default_rng(11)
        field = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        rl = n // world
        local = torch.from_numpy(field[rank * rl:(rank + 1) * rl].copy())
        slab = lct2d_sharded(local, ABCD_R, ABCD_C, row_fn=_cpu_rows, col_fn=_cpu_cols)
        q.put((rank, slab.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 16), (2, 64)])
def test_sharded_2d_matches_oracle(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r] for r in range(world)], axis=1)  # column-sharded result
    rng = np.random.default_rng(11)
    field = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    ref = O.lct2d(ABCD_R, ABCD_C, field)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
