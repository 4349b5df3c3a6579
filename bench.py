"""Benchmark of the batched XFT fast LCT (BASELINE.json metric).

Default workload = BASELINE config 2: 4096 rows x N=4096, per-row FrFT angle
alpha ~ U(0, pi) (seed 1), rows i.i.d. CN(0,1); one step = the whole batch
transformed in complex64 AND in complex128 (metric "batched LCT Msamples/s at
N=4096 c64/c128").  `value` is whole-job throughput with inputs resident in
HBM (CUDA events on the launching stream, max over ranks); `e2e` is the same
metric through the public host-buffer API (ops.lct_host -> xft_lct_host:
pinned host in, H2D + kernel + D2H, host out).  The default line also carries
`configs`: configs 1, 3, 4 and 5 measured the same way (GPU value, kernel
times, roofline fraction, ncu traffic, CPU reference baseline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg4|...]
  python bench.py --impl reference ...   # the reference's own CPU path, rank 0 only

Multi-GPU: `--gpus N` without torchrun re-launches itself under
`torch.distributed.run` with N ranks.  Rows are independent,
so configs 2/3/4 are STRONG-scaled: rank r transforms rows [rB/N, (r+1)B/N)
of the one seeded batch, no collective; `weak_scaling` adds the per-rank
full-batch figure.  Config 5 shards rows and exchanges once (row-kernel
NVLink peer stores into symmetric memory, NCCL all_to_all fallback).

CPU arms (oracle/cpu_ref.py): the reference package itself, installed into
oracle/_ref by oracle/build_ref.sh, one fast_lct/fast_frft call per row in a
process pool fed through shared memory (1-core and P-core figures).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0
METRIC = "batched LCT Msamples/s at N=4096 c64/c128"
EXTRA_CONFIGS = ("cfg1", "cfg3", "cfg4", "cfg5")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_profile_table():
    """ncu-derived per-launch DRAM traffic and FP64 op counts (profiles/ncu_traffic.json)."""
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
    """NVML SM clocks and throttle reasons sampled by a child process every `period_s` during the
    timed region.  A short region (the driver's 20-step runs last ~3 ms) may see no sample at all:
    the summary then uses the samples nearest to it (within `window_s`) and says so."""

    def __init__(self, index: int, period_s: float = 0.002, window_s: float = 0.25):
        self.index, self.period, self.window = index, period_s, window_s
        self.samples, self.reasons, self.max_mhz, self.ok, self.where = [], 0, None, False, "inside"
        self.probed = []

    def __enter__(self):
        import multiprocessing as mp

        ctx = mp.get_context("fork")
        self._stop, self._q = ctx.Event(), ctx.Queue()
        self._p = ctx.Process(target=_clock_worker, args=(self.index, self.period, self._stop, self._q), daemon=True)
        self._p.start()
        time.sleep(0.25)  # the child is sampling before the timed region starts
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
            inside += [(t1, c, why) for c, why in self.probed]  # taken while the timed work ran
            if not inside:  # region shorter than the sampling period: the nearest samples
                inside = [r for r in rows if self._t0 - self.window <= r[0] <= t1 + self.window]
                self.where = f"nearest (within {self.window * 1e3:.0f} ms of a {1e3 * (t1 - self._t0):.1f} ms region)"
            self.samples = [r[1] for r in inside]
            for r in inside:
                self.reasons |= r[2]
            self.ok = True

    def probe(self, count=2):
        """In-process samples taken while the timed work is still running on the GPU (the graph
        launches return immediately; called between the end event and the synchronize)."""
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            for _ in range(count):
                self.probed.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:
            pass

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [v for k, v in _REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples), "window": self.where}


# ---------------------------------------------------------------------------
# workloads: each item is one transform launched once per step
# ---------------------------------------------------------------------------
class Item:
    """tag, host input, parameters, kind in {lct, mehler, lct2d}; alg_bytes = HBM bytes the op must move.

    ``ref`` holds what the CPU reference arm needs (per-row FrFT angles, z, ...)."""

    def __init__(self, tag, kind, values, params, samples=None, alg_bytes=None, extra=None, ref=None):
        self.tag, self.kind, self.values, self.params = tag, kind, values, params
        self.samples = values.size if samples is None else samples
        self.alg_bytes = values.nbytes * 2 if alg_bytes is None else alg_bytes
        self.extra = extra or {}
        self.ref = ref or {}


def shard(total: int, rank: int, world: int):
    """Contiguous row block of rank ``rank`` (strong scaling of a fixed batch)."""
    return total * rank // world, total * (rank + 1) // world


def make_workload(name: str, rows_override=None, rank=0, world=1, replicate=False):
    """The config's items for this rank: rows [rB/W, (r+1)B/W) of the seeded batch (or all of it
    with ``replicate``, the weak-scaling figure).  cfg5 always shards rows (one exchange)."""
    from paper_0912_1379_b200 import workloads as W

    def rows_of(total):
        return (0, total) if replicate else shard(total, rank, world)

    if name == "cfg2":
        rows = rows_override or 4096
        s, e = rows_of(rows)
        c64 = W.config2(rows=rows, n=4096, dtype=np.complex64)
        c128 = W.config2(rows=rows, n=4096, dtype=np.complex128)
        alpha = c64.extra["alpha"][s:e]
        return [Item("c64", "lct", c64.values[s:e], c64.abcd[s:e], ref={"alpha": alpha}),
                Item("c128", "lct", c128.values[s:e], c128.abcd[s:e], ref={"alpha": alpha})], \
            {"workload": f"cfg2 batched FrFT {rows}x4096 c64+c128, per-row alpha~U(0,pi) seed 1",
             "rows": rows, "n": 4096}
    if name == "cfg4":
        c4 = W.config4(rows=rows_override or 65536)
        s, e = rows_of(c4.values.shape[0])
        return [Item("c64", "lct", c4.values[s:e], c4.abcd)], \
            {"workload": f"cfg4 Fourier (0,1,-1,0) {c4.values.shape[0]}x1024 c64, Hermite mixtures seed 3",
             "rows": c4.values.shape[0], "n": 1024}
    if name == "cfg1":
        c1 = W.config1()
        return [Item("c128", "lct", c1.values, c1.abcd)], {"workload": "cfg1 single LCT 1x1024 c128 (2,1,1,1)",
                                                           "rows": 1, "n": 1024}
    if name == "cfg3":
        c3 = W.config3(rows=rows_override or 1024)
        s, e = rows_of(c3.values.shape[0])
        z = c3.extra["z"][s:e]
        return [Item("c128", "mehler", c3.values[s:e], z, ref={"z": z})], \
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


def workload_config(cfg):
    """The line's `config`: the workload and its size (same dict on both arms)."""
    return dict(cfg, l2="inputs and outputs exceed L2 (126 MB) for configs 2-5; the GPU arm also rotates "
                        "3 input/output sets")


def samples_of(work):
    return sum(it.samples for it in work)


def bytes_of(work):
    return sum(it.alg_bytes for it in work)


def DTYPE_OF(work):
    return "+".join(sorted({it.tag for it in work}))


# ---------------------------------------------------------------------------
# CPU reference (oracle/cpu_ref.py: the reference package itself, shared-memory process pool)
# ---------------------------------------------------------------------------
def _arm_kwargs(it):
    if it.kind == "mehler":
        return {"z": it.ref["z"]}
    return {"params": np.asarray(it.params, dtype=np.float64), "alpha": it.ref.get("alpha")}


def cpu_baseline_for(work, target_s=4.0, target_1core_s=2.0):
    """P-core and 1-core reference figures over bounded samples of every item of the workload."""
    from oracle import cpu_ref

    parts = [cpu_ref.measure(it.kind, it.values, target_s=target_s, target_1core_s=target_1core_s,
                             **_arm_kwargs(it)) for it in work]
    if len(parts) == 1:
        return parts[0]

    def comb(key):  # the step's items back to back: total samples / total seconds
        s = sum(p[key]["value"] * p[key]["seconds"] for p in parts)
        t = sum(p[key]["seconds"] for p in parts)
        return {"cores": parts[0][key]["cores"], "value": s / t, "rows": [p[key]["rows"] for p in parts],
                "seconds": t}

    cp, c1 = comb("cores_P"), comb("cores_1")
    return {"value": cp["value"], "unit": "Msamples/s", "cores": cp["cores"], "kind": parts[0]["kind"],
            "sample": " | ".join(f"{it.tag}: {p['sample']}" for it, p in zip(work, parts)),
            "cores_P": cp, "cores_1": c1}


def run_reference(args, rank, world):
    """The reference arm: rank 0 times the reference's own CPU implementation; other ranks exit."""
    if rank != 0:
        return
    from oracle import cpu_ref

    work, cfg = make_workload(args.config, args.rows)
    procs = cpu_ref.host_threads()
    arms = []
    try:
        for it in work:
            t_row = max(cpu_ref.per_row_seconds(it.kind, it.values, **_arm_kwargs(it)), 1e-6)
            # bounded per-step sample: ~2 s of pool time per item, at least one row per process
            rows = args.cpu_rows or int(max(procs, min(it.values.shape[0], round(2.0 * procs / t_row))))
            arms.append(cpu_ref.CpuArm(it.kind, it.values, rows, procs, **_arm_kwargs(it)))
        for _ in range(max(1, args.warmup)):
            for a in arms:
                a.run(procs)
        vals = []
        for _ in range(args.steps):
            s = t = 0.0
            for a in arms:
                ds, dt = a.run()
                s, t = s + ds, t + dt
            vals.append(s / t / 1e6)
        kind = arms[0].kind_label
        sample = "; ".join(f"{it.tag}: {a.rows} rows of {it.values.shape[1]} per step" for it, a in zip(work, arms))
    finally:
        for a in arms:
            a.close()
    value = statistics.median(vals)
    src = "oracle/_ref (the reference xft package), one fast_lct/fast_frft call per row" if kind == "reference" \
        else "oracle/xft_oracle.py port (oracle/_ref missing)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Msamples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE_OF(work),
        "data": "synthetic (seeded, BASELINE config draw order)", "config": workload_config(cfg),
        "cpu_baseline": {"value": value, "unit": "Msamples/s", "cores": procs, "kind": kind,
                         "sample": f"{sample}; {src}; {procs}-process pool over shared memory"},
        "e2e": {"value": value, "unit": "Msamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# FP64 peak probe (tools/libxft_probe.so: a DFMA-chain kernel), for the FP64 roofline
# ---------------------------------------------------------------------------
def fp64_peak_tflops(dev_index):
    import ctypes

    path = os.path.join(ROOT, "tools", "libxft_probe.so")
    try:
        lib = ctypes.CDLL(path)
        lib.xft_probe_fp64_tflops.restype = ctypes.c_double
        lib.xft_probe_fp64_tflops.argtypes = [ctypes.c_int]
        v = float(lib.xft_probe_fp64_tflops(dev_index))
        return v if v > 0 else None
    except OSError:
        return None


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
LAUNCHES = {"lct": 1, "mehler": 14, "lct2d1": 9, "lct2dN": 2}


def measure_config(name, args, rank, world, local_rank, steps, replicate=False, e2e=True, clocks=True):
    """Times `steps` steps of config `name` on this rank; returns the rank-0 record (None elsewhere)."""
    import torch

    from paper_0912_1379_b200 import lct2d as L2
    from paper_0912_1379_b200 import mehler, ops

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    work, cfg = make_workload(name, args.rows if name == args.config else None, rank, world, replicate)
    nsets = 3  # rotate 3 input/output sets: every launch reads cold data (inputs > L2 for cfg2..5)
    stream = torch.cuda.Stream(dev)

    for it in work:  # validate once (reference order) outside the timed region
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

    transport = [args.transport]

    def launch(it, st):
        """Launches one transform; returns the tensor holding its result."""
        if it.kind == "lct":
            return ops.lct_rows(st.vin, st.p, out=st.vout, validate=False)
        elif it.kind == "mehler":
            return mehler.mehler_rows(st.vin, st.p, out=st.vout)
        elif world == 1:
            return L2.lct2d(st.vin, st.p, st.p, out=st.vout, workspace=st.ws)
        if transport[0] == "p2p":
            try:  # row kernel stores straight into the peers' symmetric-memory slabs
                return L2.lct2d_sharded(st.vin, st.p, st.p, transport="p2p")
            except (RuntimeError, NotImplementedError) as e:
                print(f"p2p transport unavailable ({e}); falling back to NCCL all_to_all", file=sys.stderr)
                transport[0] = "nccl"
        return L2.lct2d_sharded(st.vin, st.p, st.p, buffers=st.bufs)

    sets = [[make_state(it) for it in work] for _ in range(nsets)]
    # The sharded 2-D pass synchronises ranks through torch.distributed: it is launched directly;
    # everything else (incl. the Mehler path, whose per-row plans are built and cached on the
    # device by the warm-up call before capture) is captured as CUDA graphs.
    capturable = all(it.kind in ("lct", "mehler") or (it.kind == "lct2d" and world == 1) for it in work)
    chunk = max(1, min(10, steps))

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
        lanes = [torch.cuda.Stream(dev) for _ in idx]

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
                        # the step's batches are independent: each item's launches are chained on
                        # its own stream (fork/join around the whole graph): the batches share the SMs
                        for lane in lanes:
                            lane.wait_stream(stream)
                        for r in range(reps):
                            for lane, (it, st) in zip(lanes, per_set[r % nsets]):
                                with torch.cuda.stream(lane):
                                    launch(it, st)
                        for lane in lanes:
                            stream.wait_stream(lane)
                    else:
                        for r in range(reps):
                            for it, st in per_set[r % nsets]:
                                launch(it, st)
                graphs[reps] = g
            return graphs[reps]

        graph(chunk)
        if steps % chunk:
            graph(steps % chunk)

        def run(nsteps):
            for _ in range(nsteps // chunk):
                graph(chunk).replay()
            if nsteps % chunk:
                graph(nsteps % chunk).replay()
        return run

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def timed(run, n, during=None):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        run(n)
        e1.record(stream)
        if during is not None:  # host-side work while the GPU is still executing the timed steps
            during()
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        step_run = runner(None)
        kern_runs = [runner(k) for k in range(len(work))] if len(work) > 1 else [step_run]
        step_run(max(args.warmup, 3))  # warm-up (graphs for the remainder are captured here too)
        torch.cuda.synchronize()
        # each item alone (the roofline's per-kernel time): median of 3 timed runs of `steps` launches
        kern_ms = [statistics.median(max_over_ranks(timed(kern_runs[k], steps)) / steps for _ in range(3))
                   for k in range(len(work))] if len(work) > 1 else None
        if clocks:
            with ClockSampler(local_rank, period_s=args.clock_period) as clk:
                total_ms = timed(step_run, steps, during=clk.probe if args.clock_probe else None)
        else:
            clk = None
            total_ms = timed(step_run, steps)
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / steps
    if kern_ms is None:
        kern_ms = [ms_per_step]
    # whole-job samples: every rank's shard (configs 2-4 strong-scaled: the shards add up to the batch)
    samples_job = samples_of(work)
    if world > 1:
        t = torch.tensor([float(samples_job)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t)
        samples_job = int(t.item())
    value = samples_job / (ms_per_step * 1e-3) / 1e6
    launches_per_step = sum(LAUNCHES[it.kind if it.kind != "lct2d" else ("lct2d1" if world == 1 else "lct2dN")]
                            for it in work)

    e2e_rec = None
    if e2e:
        e2e_rec = measure_e2e(work, sets, launch, dev, args, world, samples_job, barrier, max_over_ranks)

    rec = {"value": value, "ms_per_step": ms_per_step, "steps": steps, "config": cfg, "work": work,
           "kern_ms": kern_ms, "samples_job": samples_job, "capturable": capturable,
           "launches": launches_per_step * steps, "clocks": clk.summary() if clk else None, "e2e": e2e_rec,
           "transport": transport[0]}
    del sets
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


def measure_e2e(work, sets, launch, dev, args, world, samples_job, barrier, max_over_ranks):
    """End to end through the public host-buffer API: pinned host in, result back on the host."""
    import threading

    import torch

    from paper_0912_1379_b200 import ops

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
            errs = []

            def one(it, hin, hout):
                try:
                    torch.cuda.set_device(dev)  # the CUDA current device is per host thread
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
    e2e_dt = max_over_ranks(time.perf_counter() - te)
    h2d = sum(h.nbytes for _, h, _ in pinned) + sum(np.asarray(it.params).nbytes for it in work)
    d2h = sum(o.nbytes for _, _, o in pinned)
    return {"value": samples_job * e2e_steps / e2e_dt / 1e6, "unit": "Msamples/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": e2e_steps,
            "api": "ops.lct_host -> xft_lct_host" if work[0].kind == "lct" else "pinned H2D + public op + D2H"}


FP64_ALG_FLOPS = {  # nominal fp64 flops per output sample of a c128 row
    # fast LCT: one length-n FFT (5 n log2 n) + the two chirp products (6 + 6)
    "lct": lambda n: 5.0 * np.log2(n) + 12.0,
    # Mehler apply (the kernel spectrum is part of the plan): two length-2n FFTs per row
    # (2 x 5 (2n) log2(2n) / n) + input weight, spectrum and output weight products (6 + 12 + 6);
    # the per-row windows make the true M smaller on most rows, so this overstates the work
    "mehler": lambda n: 20.0 * np.log2(2 * n) + 24.0,
}


def roofline_of(name, rec, world, peak, peak_src, fp64_peak):
    """Per-item kernel figures and the dominant item's roofline object."""
    prof = load_profile_table()
    work = rec["work"]
    per = {}
    for k, it in enumerate(work):
        ms = rec["kern_ms"][k]
        ach = it.alg_bytes / (ms * 1e-3) / 1e9
        tr = prof.get(f"{name}_{it.tag}")
        per[it.tag] = {"kernel_ms": ms, "Msamples_per_s": it.samples / (ms * 1e-3) / 1e6,
                       "achieved_GBps": ach, "frac": ach / peak, "alg_bytes_per_launch": it.alg_bytes,
                       "traffic": tr}
        if it.tag == "c128" and fp64_peak and it.kind in FP64_ALG_FLOPS:
            n = it.values.shape[1]
            fl = FP64_ALG_FLOPS[it.kind](n) * it.samples
            issued = prof.get(f"{name}_{it.tag}_fp64_ops_per_sample")
            f64 = {"algorithmic_flops_per_launch": fl, "achieved_TFLOPs": fl / (ms * 1e-3) / 1e12,
                   "peak_TFLOPs": fp64_peak, "frac": fl / (ms * 1e-3) / 1e12 / fp64_peak,
                   "peak_source": "measured DFMA chain (tools/xft_probe.cu), 2 flops per DFMA"}
            if issued:  # the FP64 pipe's load: issued fp64 lane-ops (ncu) vs the DFMA lane rate
                f64["issued_ops_per_sample"] = issued
                f64["pipe_frac"] = issued * it.samples / (ms * 1e-3) / (fp64_peak * 1e12 / 2)
            per[it.tag]["fp64"] = f64
        if "nvl_bytes" in it.extra and world > 1:
            t_roof = it.alg_bytes / (peak * 1e9) + it.extra["nvl_bytes"] / 900e9
            per[it.tag]["hbm_nvlink_serial_roofline_ms"] = t_roof * 1e3
            per[it.tag]["frac_of_hbm_nvlink_roofline"] = t_roof * 1e3 / ms
    dom = max(per, key=lambda t: per[t]["kernel_ms"])
    kind = work[[it.tag for it in work].index(dom)].kind
    kname = {"lct": "xft_pipe_kernel", "mehler": "xft_blue_kernel + xft_tile_kernel",
             "lct2d": "xft_pipe_kernel + xft_colring_kernel"}[kind]
    roof = {"bound": "hbm", "achieved": per[dom]["achieved_GBps"], "peak": peak, "unit": "GB/s",
            "frac": per[dom]["frac"], "traffic": per[dom]["traffic"], "kernel": f"{kname} {dom}",
            "peak_source": peak_src,
            "measured": "each item alone: K graph-replayed launches on its stream, CUDA events, median of 3 "
                        "runs; step_achieved = all items' algorithmic bytes / step time",
            "step_achieved": bytes_of(work) / (rec["ms_per_step"] * 1e-3) / 1e9}
    if "fp64" in per[dom]:
        roof["fp64"] = per[dom]["fp64"]
    return per, roof


def run_ours(args, rank, world, local_rank):
    import torch

    peak, peak_src = load_peaks()
    fp64_peak = fp64_peak_tflops(local_rank) if rank == 0 else None
    head = measure_config(args.config, args, rank, world, local_rank, args.steps)
    extras = {}
    if args.config == "cfg2" and not args.no_extras:
        for c in EXTRA_CONFIGS:
            extras[c] = measure_config(c, args, rank, world, local_rank, min(args.steps, args.extra_steps),
                                       e2e=False, clocks=False)
    weak = None
    if world > 1 and args.config in ("cfg2", "cfg3", "cfg4"):
        weak = measure_config(args.config, args, rank, world, local_rank, min(args.steps, args.extra_steps),
                              replicate=True, e2e=False, clocks=False)
    if rank != 0:
        return
    work = head["work"]
    per, roof = roofline_of(args.config, head, world, peak, peak_src, fp64_peak)
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline_for(work)
    cfgs = {}
    for c, rec in extras.items():
        p, r = roofline_of(c, rec, world, peak, peak_src, fp64_peak)
        cfgs[c] = {"workload": rec["config"]["workload"], "value": rec["value"], "unit": "Msamples/s",
                   "ms_per_step": rec["ms_per_step"], "steps": rec["steps"], "dtype": DTYPE_OF(rec["work"]),
                   "roofline": r, "per_dtype": p, "gpu_launches": rec["launches"],
                   "cpu_baseline": (cpu_baseline_for(rec["work"], 3.0, 1.5)
                                    if world == 1 and not args.no_cpu else None)}
        if c == "cfg5":
            cfgs[c]["transport"] = rec["transport"] if world > 1 else "single GPU (row pass, then columns in place through the L2-resident ring: K7)"
    strong = args.config in ("cfg2", "cfg3", "cfg4") and world > 1
    # `config` names the workload only (identical on the reference arm's line); how it ran is beside it
    line = {
        "metric": METRIC, "value": head["value"], "unit": "Msamples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if args.config in ("cfg2", "cfg3", "cfg4") else "weak",
        "vs_baseline": None, "dtype": DTYPE_OF(work), "data": "synthetic (seeded, BASELINE config draw order)",
        "config": workload_config(head["config"]),
        "parallelism": (f"rows sharded over {world} GPU(s) (rank r: rows [rB/N,(r+1)B/N)), no collective"
                        if args.config != "cfg5"
                        else f"row-sharded x{world}, " + ("row-kernel NVLink peer stores" if head["transport"] == "p2p"
                                                           and world > 1 else ("NCCL all_to_all_single" if world > 1
                                                                               else "single GPU"))),
        "timing": ("CUDA graphs" if head["capturable"] else "direct launches")
        + (", step items on independent streams" if head["capturable"] and args.overlap and len(work) > 1 else "")
        + "; 3 rotating input/output sets",
        "roofline": roof, "per_dtype": per, "cpu_baseline": cpu, "e2e": head["e2e"],
        "gpu_launches": head["launches"], "clocks": head["clocks"],
    }
    if strong:
        line["shard_rows_per_rank"] = head["work"][0].values.shape[0]
    if cfgs:
        line["configs"] = cfgs
    if weak is not None:
        line["weak_scaling"] = {"value": weak["value"], "unit": "Msamples/s", "ms_per_step": weak["ms_per_step"],
                                "what": f"every rank transforms the full {args.config} batch (replicated rows)"}
    print(json.dumps(line), flush=True)
    del torch


def relaunch_under_torchrun(n):
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=20)  # the driver's own K; long runs (1000 steps) meet sw_power_cap
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=None, help="reference arm: rows per item per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--extra-steps", type=int, default=200, help="steps for the per-config extras")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--clock-period", type=float, default=0.002, help="NVML clock sampling period (s)")
    ap.add_argument("--clock-probe", type=int, default=1, help="1: in-process clock probes while the steps run")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--overlap", type=int, default=1,
                    help="1: the step's independent batches (c64, c128) on their own streams inside the graph")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="cfg5 with N>1: row-kernel NVLink peer stores (p2p) or NCCL all_to_all")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
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
