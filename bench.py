"""Benchmark of the batched XFT fast LCT (BASELINE.json metric).

Default workload = BASELINE config 2: 4096 rows x N=4096, per-row FrFT angle
alpha ~ U(0, pi) (seed 1), rows i.i.d. CN(0,1); one step = the whole batch
transformed in complex64 AND in complex128 (metric "batched LCT Msamples/s at
N=4096 c64/c128").  `value` is whole-job throughput with inputs resident in
HBM (CUDA events on the launching stream, max over ranks); `e2e` is the same
metric through the public host-buffer API (ops.lct_host -> xft_lct_host:
pinned host in, H2D + kernel + D2H, host out).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg4|...]
  python bench.py --impl reference ...   # CPU reference path (oracle port), rank 0 only

Multi-GPU (torchrun): rows are independent, so every rank transforms its own
full batch with no collective (weak scaling); value = N x per-rank samples /
max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML poller)
# ---------------------------------------------------------------------------
_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def _clock_worker(index, period, stop, out):
    """Child process: samples NVML SM clocks and throttle reasons until `stop` is set
    (a separate process, so the GIL held by blocking graph launches cannot starve it)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        samples = []
        while not stop.is_set():
            try:
                samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(period)
        out.put((samples, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))
    except Exception:
        out.put(None)


class ClockSampler:
    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.max_mhz, self.ok = [], 0, None, False

    def __enter__(self):
        import multiprocessing as mp

        ctx = mp.get_context("fork")
        self._stop, self._q = ctx.Event(), ctx.Queue()
        self._p = ctx.Process(target=_clock_worker, args=(self.index, self.period, self._stop, self._q), daemon=True)
        self._p.start()
        time.sleep(0.05)  # the child is sampling before the timed region starts
        self._t0 = time.perf_counter()
        return self

    def __exit__(self, *a):
        t1 = time.perf_counter()
        self._stop.set()
        try:
            res = self._q.get(timeout=10)
        except Exception:
            res = None
        self._p.join(timeout=10)
        if res is not None:
            rows, self.max_mhz = res
            inside = [r for r in rows if self._t0 <= r[0] <= t1]  # the timed region only
            self.samples = [r[1] for r in inside]
            for r in inside:
                self.reasons |= r[2]
            self.ok = True

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [v for k, v in _REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workloads: each item is one transform launched once per step
# ---------------------------------------------------------------------------
class Item:
    """tag, host input, parameters, kind in {lct, mehler, lct2d}; alg_bytes = HBM bytes the op must move."""

    def __init__(self, tag, kind, values, params, samples=None, alg_bytes=None, extra=None):
        self.tag, self.kind, self.values, self.params = tag, kind, values, params
        self.samples = values.size if samples is None else samples
        self.alg_bytes = values.nbytes * 2 if alg_bytes is None else alg_bytes
        self.extra = extra or {}


def make_workload(name: str, rows_override=None, rank=0, world=1):
    from paper_0912_1379_b200 import workloads as W

    if name == "cfg2":
        rows = rows_override or 4096
        c64 = W.config2(rows=rows, n=4096, dtype=np.complex64)
        c128 = W.config2(rows=rows, n=4096, dtype=np.complex128)
        return [Item("c64", "lct", c64.values, c64.abcd), Item("c128", "lct", c128.values, c128.abcd)], \
            {"workload": f"cfg2 batched FrFT {rows}x4096 c64+c128, per-row alpha~U(0,pi) seed 1",
             "rows": rows, "n": 4096}
    if name == "cfg4":
        c4 = W.config4(rows=rows_override or 65536)
        return [Item("c64", "lct", c4.values, c4.abcd)], \
            {"workload": f"cfg4 Fourier (0,1,-1,0) {c4.values.shape[0]}x1024 c64, Hermite mixtures seed 3",
             "rows": c4.values.shape[0], "n": 1024}
    if name == "cfg1":
        c1 = W.config1()
        return [Item("c128", "lct", c1.values, c1.abcd)], {"workload": "cfg1 single LCT 1x1024 c128 (2,1,1,1)",
                                                           "rows": 1, "n": 1024}
    if name == "cfg3":
        c3 = W.config3(rows=rows_override or 1024)
        return [Item("c128", "mehler", c3.values, c3.extra["z"])], \
            {"workload": f"cfg3 complex-z Mehler FrFT {c3.values.shape[0]}x16384 c128, r~U(.5,.99) seed 2",
             "rows": c3.values.shape[0], "n": 16384}
    if name == "cfg5":
        n = rows_override or 16384
        rl = n // world
        field = W.config5_field(n=n, rows=rl, row_start=rank * rl)
        # HBM: row pass read+write + column passes (2 round trips of the slab by the roofline model of
        # 32 n^2 / G bytes per GPU); NVLink: 8 n^2 (G-1)/G^2 per GPU per direction
        return [Item("c64", "lct2d", field, W.CONFIG5_ABCD, samples=n * n // world,
                     alg_bytes=32 * n * n // world, extra={"n": n, "nvl_bytes": 8 * n * n * (world - 1) // world ** 2})], \
            {"workload": f"cfg5 2-D Fresnel LCT {n}x{n} c64 (1,0.25,0,1) both axes, disk aperture seed 4",
             "rows": n, "n": n}
    raise SystemExit(f"unknown config {name}")


def samples_of(work):
    return sum(it.samples for it in work)


def bytes_of(work):
    return sum(it.alg_bytes for it in work)


# ---------------------------------------------------------------------------
# CPU reference (oracle port) timing
# ---------------------------------------------------------------------------
def _cpu_worker(args):
    kind, p, vals = args
    from oracle import xft_oracle

    t0 = time.perf_counter()
    if kind == "mehler":  # the reference's only CPU path: the dense kernel matrix apply (512 outputs per row)
        for z, f in zip(p, vals):
            xft_oracle.mehler_apply(z, f.astype(np.complex128), rows_out=np.arange(0, f.shape[0], f.shape[0] // 512),
                                    chunk=128)
    else:  # 1-D rows (the 2-D transform is rows then columns of the same kernel)
        xft_oracle.fast_lct_rows(p, vals.astype(np.complex128))
    return time.perf_counter() - t0


def cpu_reference(work, sample_rows: int, procs: int, pool=None):
    """Oracle port of the reference fast_lct over a bounded row sample, process pool of `procs`."""
    from concurrent.futures import ProcessPoolExecutor

    tasks = []
    total = 0
    for it in work:
        v, p = it.values, np.asarray(it.params)
        rows = min(sample_rows if it.kind != "mehler" else max(procs, sample_rows // 32), v.shape[0])
        block = max(1, rows // (procs * 4))
        for s in range(0, rows, block):
            e = min(rows, s + block)
            tasks.append((it.kind, p if p.ndim <= 1 and it.kind != "mehler" else p[s:e], v[s:e]))
        total += rows * (v.shape[1] if it.kind != "mehler" else 512)
    ex = pool if pool is not None else ProcessPoolExecutor(procs)
    try:
        if pool is None:
            list(ex.map(_cpu_worker, tasks[:procs]))  # warm the workers (imports)
        t0 = time.perf_counter()
        list(ex.map(_cpu_worker, tasks))
        dt = time.perf_counter() - t0
    finally:
        if pool is None:
            ex.shutdown()
    return total / dt / 1e6, total, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    work, cfg = make_workload(args.config, args.rows)
    from concurrent.futures import ProcessPoolExecutor

    procs = len(os.sched_getaffinity(0))
    # bounded per-step sample so the whole --steps run stays within a few minutes
    sample_rows = max(procs, min(args.cpu_rows or 512, 32768 // max(1, args.steps)))
    vals = []
    with ProcessPoolExecutor(procs) as pool:
        for _ in range(max(1, args.warmup)):
            cpu_reference(work, procs, procs, pool)
        for _ in range(args.steps):
            v, total, dt = cpu_reference(work, sample_rows, procs, pool)
            vals.append(v)
    value = statistics.median(vals)
    sample = f"{sample_rows} rows per dtype of {cfg['workload']} ({total} samples/step)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Msamples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_OF(work), "data": "synthetic (seeded)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "Msamples/s", "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "Msamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "batched LCT Msamples/s at N=4096 c64/c128"


def DTYPE_OF(work):
    return "+".join(sorted({it.tag for it in work}))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch

    from paper_0912_1379_b200 import lct2d as L2
    from paper_0912_1379_b200 import mehler, ops

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    work, cfg = make_workload(args.config, args.rows, rank, world)
    nsets = 3  # rotate 3 input/output sets: every launch reads cold data (inputs > L2 for cfg2..5)
    stream = torch.cuda.Stream(dev)

    # validate once (reference order) outside the timed region
    for it in work:
        if it.kind == "lct":
            ops.validate_abcd_host(it.params)

    class State:
        pass

    def make_state(it):
        st = State()
        st.vin = torch.from_numpy(it.values).to(dev)
        st.vout = torch.empty_like(st.vin)
        st.p = torch.from_numpy(np.ascontiguousarray(it.params)).to(dev) if it.kind == "lct" else it.params
        if it.kind == "lct2d":
            if world == 1:
                st.ws = torch.empty_like(st.vin)
            else:
                rl, n = st.vin.shape
                st.bufs = (torch.empty((world, rl, n // world), dtype=st.vin.dtype, device=dev),
                           torch.empty((world, rl, n // world), dtype=st.vin.dtype, device=dev))
        return st

    def launch(it, st):
        """Launches one transform; returns the tensor holding its result."""
        if it.kind == "lct":
            return ops.lct_rows(st.vin, st.p, out=st.vout, validate=False)
        elif it.kind == "mehler":
            return mehler.mehler_rows(st.vin, st.p, out=st.vout)
        elif world == 1:
            return L2.lct2d(st.vin, st.p, st.p, out=st.vout, workspace=st.ws)
        else:
            if args.transport == "p2p":
                try:  # row kernel stores straight into the peers' symmetric-memory slabs
                    return L2.lct2d_sharded(st.vin, st.p, st.p, transport="p2p")
                except (RuntimeError, NotImplementedError) as e:
                    print(f"p2p transport unavailable ({e}); falling back to NCCL all_to_all", file=sys.stderr)
                    args.transport = "nccl"
            return L2.lct2d_sharded(st.vin, st.p, st.p, buffers=st.bufs)

    sets = [[make_state(it) for it in work] for _ in range(nsets)]
    # The sharded 2-D pass calls NCCL through torch.distributed: it is launched
    # directly; everything else (incl. the Mehler path, whose per-row plans are
    # built and cached on the device by the warm-up call before capture) is
    # captured as CUDA graphs so the timed loop has no host launch overhead.
    capturable = all(it.kind in ("lct", "mehler") or (it.kind == "lct2d" and world == 1) for it in work)
    chunk = max(1, min(10, args.steps))

    def runner(item_idx):
        """callable(n_steps) that launches n steps on `stream` (all items, or one item)."""
        idx = range(len(work)) if item_idx is None else [item_idx]
        if not capturable:
            def run(nsteps):
                for i in range(nsteps):
                    for k in idx:
                        launch(work[k], sets[i % nsets][k])
            return run
        graphs = {}
        per_set = [[(work[k], sets[i][k]) for k in idx] for i in range(nsets)]
        # --lane-priority: the heaviest item's lane (the c128 batch) gets the higher priority, so
        # freed SM slots go to it first and the lighter batch fills what remains
        heavy = max(idx, key=lambda k: work[k].values.itemsize) if len(idx) > 1 else None
        lanes = [torch.cuda.Stream(dev, priority=(-1 if (args.lane_priority and k == heavy) else 0)) for k in idx]

        def graph(reps):
            if reps not in graphs:
                with torch.cuda.stream(stream):
                    for i in range(nsets):
                        for it, st in per_set[i]:
                            launch(it, st)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    if len(idx) > 1 and args.overlap:
                        # the step's batches are independent: each item's launches are chained
                        # on its own stream (fork/join around the whole graph, or around every
                        # step with --overlap 2), so the batches share the SMs
                        for lane in lanes:
                            lane.wait_stream(stream)
                        for r in range(reps):
                            for lane, (it, st) in zip(lanes, per_set[r % nsets]):
                                with torch.cuda.stream(lane):
                                    launch(it, st)
                            if args.overlap == 2:
                                for lane in lanes:
                                    stream.wait_stream(lane)
                                for lane in lanes:
                                    lane.wait_stream(stream)
                        for lane in lanes:
                            stream.wait_stream(lane)
                    else:
                        for r in range(reps):
                            for it, st in per_set[r % nsets]:
                                launch(it, st)
                graphs[reps] = g
            return graphs[reps]

        graph(chunk)
        if args.steps % chunk:
            graph(args.steps % chunk)

        def run(nsteps):
            for _ in range(nsteps // chunk):
                graph(chunk).replay()
            if nsteps % chunk:
                graph(nsteps % chunk).replay()
        return run

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def timed(run, n):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        run(n)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1)

    with torch.cuda.stream(stream):
        step_run = runner(None)
        kern_runs = [runner(k) for k in range(len(work))]
        step_run(max(args.warmup, 3))  # warm-up (graphs for the remainder are captured here too)
        torch.cuda.synchronize()
        kern_ms = [timed(kern_runs[k], args.steps) / args.steps for k in range(len(work))]
        with ClockSampler(local_rank) as clk:
            total_ms = timed(step_run, args.steps)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    samples = samples_of(work)
    value = world * samples / (ms_per_step * 1e-3) / 1e6
    # our kernels per step (ncu launch lists, profiles/r1/final/launches_*.txt): a row batch is one
    # xft_pipe_kernel; config 3's Mehler step is 2 xft_blue_kernel + 10 xft_tile_kernel + 2 zero-fill
    # kernels; the single-GPU 2-D step is 1 row kernel + 8 cluster column kernels (one per slab),
    # the sharded one 1 row kernel + 1 column kernel per rank
    launches_per_step = sum({"lct": 1, "mehler": 14, "lct2d": 9 if world == 1 else 2}[it.kind] for it in work)

    # end-to-end through the public host-buffer API: pinned host in, result back on the host
    e2e_steps = max(2, min(args.steps, args.e2e_steps))
    pinned = []
    for it in work:
        hin = torch.from_numpy(it.values).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        pinned.append((it, hin, hout))

    def e2e_once():
        if args.overlap and len(pinned) > 1 and all(it.kind == "lct" for it, _, _ in pinned):
            # independent batches from two host threads: each call takes its own host pipeline
            # (streams + staging), so one batch's H2D fills the other's D2H-only drain
            import threading

            errs = []

            def one(it, hin, hout):
                try:
                    ops.lct_host(hin.numpy(), it.params, out=hout.numpy())
                except Exception as e:  # surfaced below
                    errs.append(e)

            ths = [threading.Thread(target=one, args=x) for x in pinned]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            if errs:
                raise errs[0]
            return
        for it, hin, hout in pinned:
            if it.kind == "lct":
                ops.lct_host(hin.numpy(), it.params, out=hout.numpy())  # xft_lct_host: chunked H2D/kernel/D2H
            else:
                st = sets[0][work.index(it)]
                st.vin.copy_(hin, non_blocking=True)
                with torch.cuda.stream(torch.cuda.current_stream(dev)):
                    res = launch(it, st)
                hout.view(-1)[:res.numel()].copy_(res.view(-1), non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()

    e2e_once()
    barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    e2e_dt = time.perf_counter() - te
    if world > 1:
        t = torch.tensor([e2e_dt], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_dt = float(t.item())
    e2e_value = world * samples * e2e_steps / e2e_dt / 1e6
    h2d = sum(h.nbytes for _, h, _ in pinned) + sum(np.asarray(it.params).nbytes for it in work)
    d2h = sum(o.nbytes for _, _, o in pinned)

    if rank != 0:
        return
    peak, peak_kind = load_peaks()
    traffic = load_traffic()
    per = {}
    for k, it in enumerate(work):
        ach = it.alg_bytes / (kern_ms[k] * 1e-3) / 1e9
        per[it.tag] = {"kernel_ms": kern_ms[k], "Msamples_per_s": it.samples / (kern_ms[k] * 1e-3) / 1e6,
                       "achieved_GBps": ach, "frac": ach / peak, "alg_bytes_per_launch": it.alg_bytes,
                       "traffic": traffic.get(f"{args.config}_{it.tag}")}
        if "nvl_bytes" in it.extra and world > 1:
            t_roof = it.alg_bytes / (peak * 1e9) + it.extra["nvl_bytes"] / 900e9
            per[it.tag]["hbm_nvlink_serial_roofline_ms"] = t_roof * 1e3
            per[it.tag]["frac_of_hbm_nvlink_roofline"] = t_roof * 1e3 / kern_ms[k]
    dom = max(per, key=lambda t: per[t]["kernel_ms"])
    kname = {"lct": "xft_pipe_kernel", "mehler": "xft_blue_kernel + xft_tile_kernel",
             "lct2d": "xft_pipe_kernel + xft_colclu_kernel"}[work[[it.tag for it in work].index(dom)].kind]
    roof = {"bound": "hbm", "achieved": per[dom]["achieved_GBps"], "peak": peak, "unit": "GB/s",
            "frac": per[dom]["frac"], "traffic": per[dom]["traffic"], "kernel": f"{kname} {dom}",
            "peak_source": peak_kind,
            "measured": "each kernel alone: K graph-replayed launches on its stream, CUDA events; "
                        "step_achieved = all items' algorithmic bytes / step time (items on their own streams)",
            "step_achieved": bytes_of(work) / (ms_per_step * 1e-3) / 1e9}

    cpu = None
    if world == 1 and not args.no_cpu:
        from concurrent.futures import ProcessPoolExecutor

        procs = len(os.sched_getaffinity(0))
        # bounded sample of the same workload: whole rows of every item (the full batch for the 1-D
        # configs), repeated until >= 10 s of CPU work (core-seconds), at most 4 passes
        rows = args.cpu_rows or max(it.values.shape[0] for it in work)
        vals, core_s, passes, total = [], 0.0, 0, 0
        with ProcessPoolExecutor(procs) as pool:
            cpu_reference(work, procs, procs, pool)  # warm the workers (imports)
            while passes < 4 and (core_s < 10.0 or passes == 0):
                v, total, dt = cpu_reference(work, rows, procs, pool)
                vals.append(v)
                core_s += dt * procs
                passes += 1
        cpu = {"value": statistics.median(vals), "unit": "Msamples/s", "cores": procs, "kind": "port",
               "sample": f"{rows} rows per item of the same batch ({total} samples per pass, {passes} passes, "
                         f"{core_s:.0f} core-s), oracle/xft_oracle.py in a {procs}-process pool"}
    line = {
        "metric": METRIC, "value": value, "unit": "Msamples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE_OF(work), "data": "synthetic (seeded, BASELINE config draw order)",
        "config": dict(cfg, l2="3 rotating input/output sets; each launch streams >= 2x L2 of cold data",
                       parallelism=(f"batch-sharded x{world}, no collective" if args.config != "cfg5"
                                    else f"row-sharded x{world}, " + ("row-kernel NVLink peer stores (symmetric memory)"
                                                                     if args.transport == "p2p" and world > 1
                                                                     else "one NCCL all_to_all_single")),
                       timing=("CUDA graphs" if capturable else "direct launches")
                       + (", step items on independent streams" if capturable and args.overlap and len(work) > 1
                          else "")),
        "roofline": roof, "per_dtype": per, "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "Msamples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "api": "ops.lct_host -> xft_lct_host" if work[0].kind == "lct"
                else "pinned H2D + public op + D2H"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=None, help="CPU baseline rows per item (default: full batch)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--overlap", type=int, default=1,
                    help="1: the step's independent batches (c64, c128) on their own streams inside the graph")
    ap.add_argument("--lane-priority", type=int, default=0, help="1: higher stream priority for the c128 lane")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="cfg5 under torchrun: row-kernel NVLink peer stores (p2p) or NCCL all_to_all")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
