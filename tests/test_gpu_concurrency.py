"""Thread-safety and reentrancy of the GPU path (the reference's concurrency contract).

Reference: plans own no scratch and one plan may serve many threads at once
(xft/fftcore.py:8-11, pkg/README.md:66-70); pkg/tests/test_fftcore.py:112-148
runs 8 threads on one shared plan and two plans in parallel and requires
bit-identical results.  Here every thread also drives its own CUDA stream, so
the library's lazily built tables, chirp-z plans, Mehler plan cache, scratch
and side streams are exercised from concurrent first calls (cold caches).
"""
import threading

import numpy as np
import pytest

from tests.conftest import max_row_rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _run_threads(fns):
    results, errs = [None] * len(fns), []

    def wrap(i, f):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                r = f()
                s.synchronize()
            results[i] = r
        except Exception as e:  # re-raised in the main thread
            errs.append(e)

    ths = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return results


def test_shared_plan_parallel_applies_cold():
    """8 threads on one plan, first use of this length in the process (pkg/tests/test_fftcore.py:115-131)."""
    from paper_0912_1379_b200.fft import apply_dft, plan_dft

    rng = np.random.default_rng(11)
    n = 600 + 6  # a chirp-z length no other test builds first
    plan = plan_dft(n, 1)
    vs = [rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(8)]
    got = _run_threads([lambda v=v: apply_dft(plan, v) for v in vs])
    expected = [apply_dft(plan, v) for v in vs]
    for g, e in zip(got, expected):
        assert np.array_equal(g, e)


def test_two_plans_in_parallel():
    """pkg/tests/test_fftcore.py:133-148."""
    from paper_0912_1379_b200.fft import apply_dft, plan_dft

    rng = np.random.default_rng(12)
    n = 256
    p1, p2 = plan_dft(n, 1), plan_dft(n, -1)
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    got = _run_threads([lambda: apply_dft(p1, v), lambda: apply_dft(p2, v)])
    assert np.array_equal(got[0], apply_dft(p1, v))
    assert np.array_equal(got[1], apply_dft(p2, v))


@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
def test_batched_rows_from_8_threads_cold_sizes(dtype):
    """8 threads x (cold sizes, per-row parameters) on their own streams == sequential, bit for bit."""
    from paper_0912_1379_b200 import ops
    from paper_0912_1379_b200.workloads import frft_abcd

    rng = np.random.default_rng(7)
    sizes = [128, 512, 2048, 4096, 640, 3000, 8192, 96]  # radix-2 and chirp-z, several cold
    jobs = []
    for n in sizes:
        x = torch.from_numpy(rng.normal(size=(17, n)) + 1j * rng.normal(size=(17, n))).to(dtype).cuda()
        p = np.array([frft_abcd(a) for a in rng.uniform(0.1, 3.0, 17)])
        jobs.append((x, p))
    got = _run_threads([lambda x=x, p=p: ops.lct_rows(x, p).cpu() for x, p in jobs] * 2)
    for k, (x, p) in enumerate(jobs):
        ref = ops.lct_rows(x, p).cpu()
        assert torch.equal(got[k], ref) and torch.equal(got[k + len(jobs)], ref)


def test_mehler_two_threads_different_z():
    """Two threads, two z arrays of the same (batch, n): each gets its own plan, results == sequential."""
    from paper_0912_1379_b200 import mehler

    rng = np.random.default_rng(3)
    n, B = 2048, 6
    f = torch.from_numpy(rng.normal(size=(B, n)) + 1j * rng.normal(size=(B, n))).cuda()
    za = 0.7 * np.exp(1j * rng.uniform(0, 2 * np.pi, B))
    zb = 0.9 * np.exp(1j * rng.uniform(0, 2 * np.pi, B))
    got = _run_threads([lambda z=z: [mehler.mehler_rows(f, z).cpu() for _ in range(5)] for z in (za, zb, za, zb)])
    ra, rb = mehler.mehler_rows(f, za).cpu(), mehler.mehler_rows(f, zb).cpu()
    for k, r in enumerate((ra, rb, ra, rb)):
        for g in got[k]:
            assert torch.equal(g, r)


def test_mehler_cache_is_exact_not_hashed():
    """z arrays one ulp apart are different plans (the cache compares every z value)."""
    from oracle import xft_oracle as O
    from paper_0912_1379_b200 import mehler

    rng = np.random.default_rng(4)
    n = 1024
    f = rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n))
    z1 = np.array([0.6 + 0.2j, -0.3 + 0.5j])
    z2 = z1.copy()
    z2[1] = complex(np.nextafter(z1[1].real, 1.0), z1[1].imag)
    t = torch.from_numpy(f).cuda()
    g1 = mehler.mehler_rows(t, z1).cpu().numpy()
    g2 = mehler.mehler_rows(t, z2).cpu().numpy()
    for z, g in ((z1, g1), (z2, g2)):
        ref = np.stack([O.mehler_apply(z[i], f[i]) for i in range(2)])
        assert max_row_rel_l2(g, ref) <= 1e-12


def test_mehler_lru_eviction_keeps_captured_graph_valid():
    """A graph captured with a cached plan still replays correctly after > 64 other z arrays evicted it."""
    from paper_0912_1379_b200 import mehler

    rng = np.random.default_rng(5)
    n, B = 1024, 3
    f = torch.from_numpy(rng.normal(size=(B, n)) + 1j * rng.normal(size=(B, n))).cuda()
    z0 = 0.8 * np.exp(1j * np.array([0.3, 1.9, 4.0]))
    out = torch.empty_like(f)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        mehler.mehler_rows(f, z0, out=out)  # plan + scratch built outside capture
        s.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            mehler.mehler_rows(f, z0, out=out)
    for k in range(70):  # evict z0's plan from the implicit cache (LRU of 64)
        mehler.mehler_rows(f, z0 * (0.999 - 1e-3 * k))
    torch.cuda.synchronize()
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # and the evicted z array is rebuilt correctly on its next direct call
    assert torch.equal(mehler.mehler_rows(f, z0), ref)


def test_caller_owned_plan_matches_implicit_cache_and_survives_release():
    from paper_0912_1379_b200 import mehler

    rng = np.random.default_rng(6)
    n, B = 4096, 4
    f = torch.from_numpy(rng.normal(size=(B, n)) + 1j * rng.normal(size=(B, n))).cuda()
    z = 0.75 * np.exp(1j * np.array([0.1, 1.2, 2.5, 5.5]))
    plan = mehler.MehlerPlan(n, z)
    a = plan.apply(f)
    b = mehler.mehler_rows(f, z)
    assert torch.equal(a, b)
    torch.cuda.synchronize()
    mehler.release_caches()  # drops the implicit cache; the caller's plan keeps its own reference
    assert torch.equal(plan.apply(f), b)
    assert torch.equal(mehler.mehler_rows(f, z), b)  # rebuilt after the release
    got = _run_threads([lambda: plan.apply(f).cpu() for _ in range(4)])
    for g in got:
        assert torch.equal(g, b.cpu())
    plan.close()
    with pytest.raises(Exception):
        plan.apply(f)


def test_out_argument_is_checked():
    from paper_0912_1379_b200 import ops
    from paper_0912_1379_b200.errors import ParameterError, ShapeError

    x = torch.randn(4, 256, dtype=torch.complex64, device="cuda")
    with pytest.raises(ShapeError):
        ops.lct_rows(x, (0.0, 1.0, -1.0, 0.0), out=torch.empty(4, 128, dtype=torch.complex64, device="cuda"))
    with pytest.raises(ParameterError):
        ops.lct_rows(x, (0.0, 1.0, -1.0, 0.0), out=torch.empty(4, 256, dtype=torch.complex128, device="cuda"))
    with pytest.raises(ShapeError):
        ops.lct_rows(x, (0.0, 1.0, -1.0, 0.0), out=torch.empty(256, 4, dtype=torch.complex64, device="cuda").T)
    with pytest.raises(ShapeError):
        ops.dft_rows(x, -1, out=torch.empty(4, 256, dtype=torch.complex64))  # host tensor
    big = torch.empty(4 * 256 + 1, dtype=torch.complex64, device="cuda")
    with pytest.raises(ShapeError):  # 8-byte offset: not 16-byte aligned
        ops.lct_rows(x, (0.0, 1.0, -1.0, 0.0), out=big[1:].view(4, 256))


def test_misaligned_input_view_is_copied_not_faulted():
    """A contiguous c64 view at an odd element offset (8-byte aligned only) gives the aligned result."""
    from paper_0912_1379_b200 import ops

    base = torch.randn(1 + 8 * 512, dtype=torch.complex64, device="cuda")
    view = base[1:].view(8, 512)
    assert view.data_ptr() % 16 == 8
    ref = ops.lct_rows(view.clone(), (0.5, 1.5, -0.5, 0.5))
    assert torch.equal(ops.lct_rows(view, (0.5, 1.5, -0.5, 0.5)), ref)
    assert torch.equal(ops.dft_rows(view, 1), ops.dft_rows(view.clone(), 1))


def test_host_path_from_two_threads_matches_device_path():
    """xft_lct_host from two host threads (own pipelines) == the device path, bit for bit."""
    from paper_0912_1379_b200 import ops
    from paper_0912_1379_b200.workloads import config2

    a = config2(rows=64, n=4096, dtype=np.complex64)
    b = config2(rows=64, n=4096, dtype=np.complex128)
    got = _run_threads([lambda: ops.lct_host(a.values, a.abcd), lambda: ops.lct_host(b.values, b.abcd)])
    assert np.array_equal(got[0], ops.lct_rows(torch.from_numpy(a.values).cuda(), a.abcd).cpu().numpy())
    assert np.array_equal(got[1], ops.lct_rows(torch.from_numpy(b.values).cuda(), b.abcd).cpu().numpy())


def test_lct2d_from_four_threads_matches_serial():
    """The 2-D transform's L2-staged column kernel (K7) launched from four threads at once, each on
    its own stream: every launch is a cooperative, GPU-filling persistent grid with its own scratch
    ring and counters (per-stream scratch), so concurrent calls must queue, not interfere."""
    from paper_0912_1379_b200 import lct2d

    rng = np.random.default_rng(77)
    p = (1.0, 0.25, 0.0, 1.0)
    fields = [torch.from_numpy((rng.normal(size=(16384, 256)) + 1j * rng.normal(size=(16384, 256))).astype(np.complex64)).cuda()
              for _ in range(4)]
    serial = [lct2d.lct2d(f, p, p).cpu().numpy() for f in fields]
    torch.cuda.synchronize()

    def job(f):
        def run():
            out = None
            for _ in range(3):
                out = lct2d.lct2d(f, p, p)
            return out.cpu().numpy()
        return run

    got = _run_threads([job(f) for f in fields])
    for g, s in zip(got, serial):
        assert np.array_equal(g, s)
