"""CPU timing harness for bench.py's reference arm and ``cpu_baseline`` -- BENCH INFRASTRUCTURE ONLY.

Times the reference's OWN CPU implementation of the hot path on the host's
cores: the ``xft`` package installed from ``/root/reference/pkg`` into
``oracle/_ref/`` by ``oracle/build_ref.sh`` (git-ignored, shipped to the GPU
box with the snapshot).  Only ``bench.py`` imports this module; the product
package never does.  If ``oracle/_ref`` is missing the harness falls back to
the NumPy restatement ``oracle/xft_oracle.py`` and says so (``kind: "port"``).

What is timed, per workload kind (SURVEY.md 8(d) "CPU baseline timing"):

* ``lct``   -- one reference call per row, exactly as a reference user would
  batch it: ``fast_frft(alpha_i, Signal(grid, row))`` for FrFT rows
  (xft/lct.py:226-233), ``fast_lct(LctParams(a,b,c,d), Signal(grid, row))``
  otherwise (xft/lct.py:168-208).  One sample = one output value.
* ``mehler`` -- the reference's only CPU path for complex z is the dense
  kernel ``mehler_kernel(FrftOrder(z), x_j, x_k) * spacing @ f``
  (xft/dense.py:122-151; ``frft_matrix_asymptotic`` refuses n > 4096, so its
  entries are formed block by block of output rows through the same
  ``mehler_kernel``).  A bounded set of output samples per row is computed;
  one sample = one output value.
* ``lct2d`` -- the separable 2-D transform is ``fast_lct`` along every row then
  every column; each line costs one 1-D call, every output sample needs two
  line transforms, so samples/s = (lines/s) * n / 2.

Process model: a pool of P worker processes (P = the host threads available),
``OMP/OPENBLAS/MKL_NUM_THREADS=1`` in the workers.  The sampled input rows
live in one ``multiprocessing.shared_memory`` block, outputs are written into
another, so the timed region ships only (start, stop) index pairs -- nothing
is pickled per row.  Worker start-up, imports, grid and plan caches are warmed
before timing.
"""
from __future__ import annotations

import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from multiprocessing import get_context, shared_memory

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "xft"))


def _import_reference():
    """The installed reference package (kind "reference"), else None."""
    if not reference_available():
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import xft  # noqa: F401  (oracle/_ref/xft)

    return xft


# ---------------------------------------------------------------------------
# worker side
# ---------------------------------------------------------------------------
_W = {}


def _worker_init(spec):
    """Attach the shared input/output blocks and warm the reference's caches."""
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    shm_in = shared_memory.SharedMemory(name=spec["in_name"])
    shm_out = shared_memory.SharedMemory(name=spec["out_name"])
    vin = np.ndarray(spec["shape"], dtype=np.dtype(spec["dtype"]), buffer=shm_in.buf)
    vout = np.ndarray(spec["out_shape"], dtype=np.complex128, buffer=shm_out.buf)
    xft = None if spec["force_port"] else _import_reference()
    _W.update(spec=spec, shm=(shm_in, shm_out), vin=vin, vout=vout, xft=xft)
    n = spec["shape"][1]
    if xft is not None:
        _W["grid"] = xft.asymptotic_zeros(n)
    else:
        sys.path.insert(0, os.path.dirname(HERE))
        from oracle import xft_oracle

        _W["port"] = xft_oracle


def _row_params(i):
    p = _W["spec"]["params"]
    return p if p.ndim == 1 else p[i]


def _run_block(bounds):
    """Transforms rows [s, e) of the shared sample into the shared output."""
    s, e = bounds
    spec, vin, vout, xft = _W["spec"], _W["vin"], _W["vout"], _W["xft"]
    kind = spec["kind"]
    if xft is not None:
        grid = _W["grid"]
        if kind in ("lct", "lct2d"):
            alpha = spec.get("alpha")
            for i in range(s, e):
                sig = xft.Signal(grid, vin[i])
                if alpha is not None:
                    vout[i] = xft.fast_frft(float(alpha[i]), sig).values
                else:
                    a, b, c, d = (float(t) for t in _row_params(i))
                    vout[i] = xft.fast_lct(xft.LctParams(a, b, c, d), sig).values
        else:  # mehler: dense kernel rows, the reference's only complex-z path
            x = grid.nodes
            outs = spec["outs"]
            for i in range(s, e):
                order = xft.FrftOrder(complex(spec["z"][i]))
                f = np.asarray(vin[i], dtype=complex)
                for c0 in range(0, outs.size, 64):
                    sel = outs[c0:c0 + 64]
                    blk = xft.mehler_kernel(order, x[sel, None], x[None, :]) * grid.spacing
                    vout[i, c0:c0 + sel.size] = blk @ f
    else:
        port = _W["port"]
        if kind in ("lct", "lct2d"):
            p = spec["params"]
            pp = p if p.ndim == 1 else p[s:e]
            vout[s:e] = port.fast_lct_rows(pp, vin[s:e].astype(np.complex128))[1]
        else:
            outs = spec["outs"]
            for i in range(s, e):
                vout[i, :outs.size] = port.mehler_apply(complex(spec["z"][i]), vin[i].astype(np.complex128),
                                                        rows_out=outs, chunk=64)
    return e - s


# ---------------------------------------------------------------------------
# parent side
# ---------------------------------------------------------------------------
class CpuArm:
    """A warmed process pool over a shared-memory sample of one workload item.

    ``kind`` in {lct, mehler, lct2d}; ``values`` [B, n]; ``params`` [B, 4] or
    [4] (lct), ``z`` [B] complex (mehler); ``alpha`` [B] routes FrFT rows
    through ``fast_frft``.  ``rows`` sampled rows are copied once into shared
    memory (outside any timed region).
    """

    def __init__(self, kind, values, rows, procs, params=None, alpha=None, z=None, outs_per_row=256,
                 force_port=False):
        self.kind, self.procs = kind, max(1, int(procs))
        rows = max(1, int(rows))
        self.rows, self.n = rows, values.shape[1]
        # rows beyond the batch (e.g. config 1's single row) repeat the batch's rows in order
        idx = np.arange(rows) % values.shape[0]
        sample = np.ascontiguousarray(values[idx])
        self.kind_label = "port" if (force_port or not reference_available()) else "reference"
        self._in = shared_memory.SharedMemory(create=True, size=max(1, sample.nbytes))
        np.ndarray(sample.shape, sample.dtype, buffer=self._in.buf)[...] = sample
        if kind == "mehler":
            outs = np.unique(np.linspace(0, self.n - 1, min(outs_per_row, self.n)).astype(np.int64))
            out_shape = (rows, outs.size)
        else:
            outs = None
            out_shape = (rows, self.n)
        self.outs_per_row = None if outs is None else int(outs.size)
        self._out = shared_memory.SharedMemory(create=True, size=int(np.prod(out_shape)) * 16)
        spec = {"kind": kind, "in_name": self._in.name, "out_name": self._out.name, "shape": sample.shape,
                "dtype": sample.dtype.str, "out_shape": out_shape, "force_port": force_port,
                "params": None if params is None else np.asarray(params, dtype=np.float64),
                "alpha": None if alpha is None else np.asarray(alpha, dtype=np.float64)[idx],
                "z": None if z is None else np.asarray(z, dtype=np.complex128)[idx], "outs": outs}
        if spec["params"] is not None and spec["params"].ndim == 2:
            spec["params"] = spec["params"][idx]
        self._pool = ProcessPoolExecutor(self.procs, mp_context=get_context("fork"),
                                         initializer=_worker_init, initargs=(spec,))
        # warm-up: every worker imports, builds the grid / plan caches
        list(self._pool.map(_run_block, [(i % rows, i % rows + 1) for i in range(self.procs)]))

    def samples_per_row(self):
        if self.kind == "mehler":
            return self.outs_per_row
        if self.kind == "lct2d":
            return self.n / 2.0  # each output sample needs a row and a column line transform
        return self.n

    def run(self, rows=None):
        """Times one pass over the first ``rows`` sampled rows; returns (samples, seconds)."""
        rows = self.rows if rows is None else max(1, min(rows, self.rows))
        blk = max(1, rows // (self.procs * 4))
        bounds = [(s, min(rows, s + blk)) for s in range(0, rows, blk)]
        t0 = time.perf_counter()
        done = sum(self._pool.map(_run_block, bounds))
        dt = time.perf_counter() - t0
        assert done == rows
        return rows * self.samples_per_row(), dt

    def output(self):
        shape = (self.rows, self.outs_per_row if self.kind == "mehler" else self.n)
        return np.ndarray(shape, np.complex128, buffer=self._out.buf).copy()

    def close(self):
        self._pool.shutdown()
        for s in (self._in, self._out):
            s.close()
            s.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


def per_row_seconds(kind, values, **kw) -> float:
    """One-core cost of one row (two rows timed after a warm row)."""
    with CpuArm(kind, values, 3, 1, **kw) as arm:
        arm.run(1)
        s, dt = arm.run(2)
    return dt / 2


def measure(kind, values, target_s=4.0, target_1core_s=2.0, procs=None, **kw):
    """cpu_baseline entry: P-core and 1-core figures on bounded row samples.

    The sample sizes are chosen from a one-core per-row cost so the P-core
    pass takes about ``target_s`` and the 1-core pass about ``target_1core_s``.
    Returns a dict in bench.py's ``cpu_baseline`` shape.
    """
    procs = procs or host_threads()
    t_row = max(per_row_seconds(kind, values, **kw), 1e-6)
    # at most the whole batch per pass (tiled when the batch has fewer rows than processes);
    # passes repeat until the timed pool time reaches the target
    cap = max(values.shape[0], procs * 4)
    rows_p = int(min(cap, max(procs, round(target_s * procs / t_row))))
    rows_1 = int(min(cap, max(1, round(target_1core_s / t_row))))

    def passes(arm, target):
        s = t = 0.0
        k = 0
        while k == 0 or (t < target and k < 32):
            ds, dt = arm.run()
            s, t, k = s + ds, t + dt, k + 1
        return s, t, k

    with CpuArm(kind, values, rows_p, procs, **kw) as arm:
        sp, dtp, kp = passes(arm, target_s)
        label, opr = arm.kind_label, arm.outs_per_row
    with CpuArm(kind, values, rows_1, 1, **kw) as arm:
        s1, dt1, k1 = passes(arm, target_1core_s)
    what = {"lct": "one reference fast_lct/fast_frft call per row",
            "mehler": f"dense reference mehler_kernel rows ({opr} output samples per row)",
            "lct2d": "one reference fast_lct call per line (2 lines per output sample)"}[kind]
    src = "oracle/_ref (xft from /root/reference/pkg)" if label == "reference" else "oracle/xft_oracle.py (port)"
    return {"value": sp / dtp / 1e6, "unit": "Msamples/s", "cores": procs, "kind": label,
            "sample": f"{kp} pass(es) over {rows_p} rows x {values.shape[1]} of the same seeded batch, {what}; "
                      f"{src}; {procs}-process pool over shared memory",
            "cores_P": {"cores": procs, "value": sp / dtp / 1e6, "rows": rows_p, "passes": kp, "seconds": dtp},
            "cores_1": {"cores": 1, "value": s1 / dt1 / 1e6, "rows": rows_1, "passes": k1, "seconds": dt1}}
