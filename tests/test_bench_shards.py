"""bench.py's multi-GPU work split and its CPU reference harness, checked on CPU.

* Strong scaling (configs 2/3/4): under world_size 2 (gloo, two processes)
  every rank builds its own row block with ``bench.make_workload``; the blocks
  gathered over the process group must tile the one seeded batch exactly --
  no row missing, none duplicated, same per-row parameters (the reference
  makes rows independent).
* The CPU arm (oracle/cpu_ref.py) returns the reference's own per-row outputs
  (bit-identical to the oracle port, which tests/test_oracle.py pins to the
  reference's golden vectors).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, rows, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench

        work, _ = bench.make_workload(name, rows, rank, world)
        local = [(it.tag, torch.from_numpy(np.ascontiguousarray(it.values)),
                  torch.from_numpy(np.ascontiguousarray(np.atleast_2d(it.params if it.kind != "mehler"
                                                                      else np.stack([it.params.real,
                                                                                     it.params.imag], 1)))))
                 for it in work]
        gathered = [None] * world
        dist.all_gather_object(gathered, [(t, v.numpy(), p.numpy()) for t, v, p in local])
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,rows", [("cfg2", 64), ("cfg3", 6), ("cfg4", 40)])
def test_strong_scaling_shards_tile_the_batch(name, rows):
    sys.path.insert(0, ROOT)
    import bench

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full, _ = bench.make_workload(name, rows, 0, 1)
    for k, it in enumerate(full):
        vals = np.concatenate([g[k][1] for g in gathered], axis=0)
        assert vals.shape == it.values.shape
        assert np.array_equal(vals, it.values)
        if it.kind == "mehler":
            z = np.concatenate([g[k][2][:, 0] + 1j * g[k][2][:, 1] for g in gathered])
            assert np.array_equal(z, it.params)
        elif np.asarray(it.params).ndim == 2:
            assert np.array_equal(np.concatenate([g[k][2] for g in gathered]), it.params)
    # shard sizes differ by at most one row
    sizes = [g[0][1].shape[0] for g in gathered]
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == full[0].values.shape[0]


def test_shard_bounds_cover_every_row():
    sys.path.insert(0, ROOT)
    import bench

    for total in (1, 7, 1024, 4096, 65536):
        for world in (1, 2, 3, 4, 8):
            b = [bench.shard(total, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == total
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_cpu_arm_runs_the_reference_per_row():
    sys.path.insert(0, ROOT)
    from oracle import cpu_ref, xft_oracle
    from paper_0912_1379_b200 import workloads as W

    c2 = W.config2(rows=6, n=256, dtype=np.complex64)
    with cpu_ref.CpuArm("lct", c2.values, 6, 2, params=c2.abcd, alpha=c2.extra["alpha"]) as arm:
        s, dt = arm.run()
        out = arm.output()
    assert s == 6 * 256 and dt > 0
    _, ref = xft_oracle.fast_lct_rows(c2.abcd, c2.values.astype(np.complex128))
    assert np.array_equal(out, ref)  # the reference == the port, bit for bit


def test_cpu_arm_mehler_outputs_match_dense_oracle():
    sys.path.insert(0, ROOT)
    from oracle import cpu_ref, xft_oracle

    rng = np.random.default_rng(5)
    n = 512
    f = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    z = np.array([0.6 * np.exp(0.3j), 0.8 * np.exp(2.1j)])
    with cpu_ref.CpuArm("mehler", f, 2, 1, z=z, outs_per_row=32) as arm:
        arm.run()
        out = arm.output()
    outs = np.unique(np.linspace(0, n - 1, 32).astype(np.int64))
    for i in range(2):
        ref = xft_oracle.mehler_apply(z[i], f[i], rows_out=outs)
        assert np.allclose(out[i], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_cpu_measure_reports_one_and_p_cores():
    sys.path.insert(0, ROOT)
    from oracle import cpu_ref
    from paper_0912_1379_b200 import workloads as W

    c4 = W.config4(rows=64, n=1024)
    r = cpu_ref.measure("lct", c4.values, target_s=0.2, target_1core_s=0.1, procs=2, params=c4.abcd)
    assert r["kind"] == ("reference" if cpu_ref.reference_available() else "port")
    assert r["cores"] == 2 and r["cores_P"]["cores"] == 2 and r["cores_1"]["cores"] == 1
    assert r["value"] > 0 and r["cores_1"]["value"] > 0
