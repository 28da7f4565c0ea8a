#!/usr/bin/env python3
"""Benchmark of the B200 Store-zechin engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference] [--no-suite]

A "step" is one pass of the hot path over one batch of the config's synthetic
input. The headline workload is BASELINE.json configs[1] = C2 (100,000
boson-sampling 5x5 complex128 submatrices); the same JSON line carries a
"suite" object with every config (C1..C5) measured the same way, so the
layer kernel (C4/C5) numbers are visible next to the batched ones.

  value  device-resident inputs (in HBM before the timed region), device
         compute only, CUDA events on the launching stream, L2 flushed
         between steps (inputs are < L2), max over ranks;
  e2e    the public API call with pinned HOST buffers: H2D of the inputs,
         compute, D2H of the results, all inside the timed region;
  roofline  algorithmic bytes per launch of the dominant kernel (DESIGN.md
         section 4) / its average CUDA-event duration, against the measured
         HBM copy bandwidth in MEASURED_PEAKS.json;
  cpu_baseline  the reference engine itself (oracle/_ref, compiled from the
         reference sources) on a bounded sample, all host threads.

Multi-GPU (torchrun): batches shard by matrix with no collective, each rank a
full batch (weak scaling); C4/C5 in the suite run one matrix on all ranks
(sharded.py, strong scaling): top-column blocks with point-to-point exchange
for power-of-two worlds, equal slices with an all-gather otherwise.

--impl reference times the reference's own CPU path (oracle/_ref; the oracle
port for C5, which the reference cannot run) on this config with all host
threads; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic bytes / ops per unit.
ELEM = {"int64": 8, "float64": 8, "complex128": 16}
DT_SHORT = {"int64": "int64", "float64": "f64", "complex128": "c128"}


def layer_dp_bytes(n: int, s: int) -> int:
    """Compulsory traffic of the layer DP: every stored layer 2..n-1 written once
    and read once (C(n,2) + sum_{k=3}^{n-1} (C(n,k-1) + C(n,k)) + C(n,n-1))."""
    b = math.comb(n, 2)
    for k in range(3, n):
        b += math.comb(n, k - 1) + math.comb(n, k)
    b += math.comb(n, n - 1)
    return b * s


def algorithmic_bytes_per_perm(n: int, s: int) -> int:
    if n <= 16:  # batched kernels: the matrix in, one value out
        return n * n * s + s
    return layer_dp_bytes(n, s)


def flops_per_perm(n: int, dtype: str) -> int:
    if n == 1:
        return 0
    if n == 2:
        m, a = 2, 1
    else:
        m, a = n * 2 ** (n - 1) - n, n * 2 ** (n - 1) - 2 ** n + 1
    return 6 * m + 2 * a if dtype == "complex128" else m + a


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return {}
    return {}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling through NVML."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- workloads

def _configs_module():
    """paper_1802_02779_b200/configs.py loaded by path: the seeded generators
    only (libpermlab_gen.so), never the engine's libpermlab_b200.so -- the
    reference arm must not map the product library."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("permlab_bench_configs", ROOT / "paper_1802_02779_b200" / "configs.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def workload(name: str):
    configs = _configs_module()
    spec = configs.CONFIGS[name]
    a = configs.generate(name)
    return spec, a


def config_spec(name: str):
    return _configs_module().CONFIGS[name]


def config_dict(name: str, world: int, fma: bool) -> dict:
    """The `config` object of both arms' JSON lines (identical for the same
    workload, so the driver can pair them)."""
    spec = config_spec(name)
    batched = spec["n"] <= 16
    if batched:
        l2 = "inputs from HBM every step: rotating device copies of the batch (>= 320 MiB > L2), K steps in one CUDA graph"
        if os.environ.get("PL_BENCH_INPUT_READY", "1") != "0" and (spec["n"] <= 5 or name == "c3"):
            l2 += "; steps launched with PL_FLAG_INPUT_READY (static inputs: a step's loads overlap the previous step's tail)"
        par = f"dp{world} (batch by matrix, no collective)"
    else:
        l2 = "L2 flushed between timed steps (256 MiB write, then 256 MiB read), one event pair per step"
        par = "1 GPU" if world == 1 else f"layer DP sharded over {world} GPUs"
    return {"workload": f"{name}: {spec['desc']}", "n": spec["n"], "count": spec["count"],
            "per_rank_count": spec["count"], "l2": l2,
            "arith": "fma" if fma else "reference rounding order (no FMA)", "parallelism": par}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_reference_time(name: str, a: np.ndarray, budget_s: float, threads: int):
    """Time the reference's own CPU path on a bounded sample: returns
    (permanents/s, sample description, kind, cores)."""
    from oracle import oracle as O

    n = a.shape[1]
    if name == "c5" or not O.ref_available():
        # order 32 is beyond the reference (mask cap 31, 128 GiB memo): the
        # oracle port (restated layer DP, all threads) stands in.
        t = time.perf_counter()
        O.sz_batch(a[:1], nthreads=threads)
        dt = time.perf_counter() - t
        return 1.0 / dt, f"1 matrix n={n} via oracle port ({threads} threads)", "port", threads
    if n >= 20:  # single large matrix: the reference engine is single-threaded
        t = time.perf_counter()
        O.ref_sz_batch(a[:1], nthreads=1, memo_budget_bytes=8 << 30)
        dt = time.perf_counter() - t
        return 1.0 / dt, f"1 matrix n={n}, reference engine (single-threaded by design)", "reference", 1
    # contiguous chunks of the batch (one contiguous slice per thread inside
    # ref_sz_batch), growing until one takes >= 0.25 s, repeated to budget_s
    done, t0 = 0, time.perf_counter()
    size, pos = min(a.shape[0], 256 * threads), 0
    while True:
        if pos + size > a.shape[0]:
            pos = 0
        t1 = time.perf_counter()
        O.ref_sz_batch(a[pos:pos + size], nthreads=threads)
        pos += size
        done += size
        now = time.perf_counter()
        if now - t0 >= budget_s:
            break
        if now - t1 < 0.25:
            size = min(a.shape[0], size * 2)
    el = time.perf_counter() - t0
    return done / el, f"{done} matrices n={n} ({el:.1f} s wall, {threads} threads, contiguous chunks)", \
        "reference", threads


CPU_LARGE = ROOT / "profiles" / "cpu_large.json"


def measure_cpu_large() -> dict:
    """The single large matrices on the host: C4 through the reference engine
    itself (oracle/_ref, single-threaded as it is written, ~1 min) and C5
    through the oracle port (the reference cannot run n = 32; all threads,
    ~19 GB of host memory). Written to profiles/cpu_large.json by
    `bench.py --cpu-large-only` on the GPU box's host, read by the suite."""
    out = {"cpu_model": cpu_model(), "nproc": os.cpu_count(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    for name in ("c4", "c5"):
        _, a = workload(name)
        threads = 1 if name == "c4" else (os.cpu_count() or 1)
        try:
            import psutil

            if name == "c5" and psutil.virtual_memory().available < (40 << 30):
                out[name] = {"error": "less than 40 GB of host memory available for the n = 32 port"}
                continue
        except ImportError:
            pass
        v, sample, kind, cores = cpu_reference_time(name, a, 0.0, threads)
        out[name] = {"value": v, "unit": "permanents/s", "seconds_per_permanent": 1.0 / v, "cores": cores,
                     "kind": kind, "sample": sample}
    return out


def suite_cpu_baseline(name: str, a: np.ndarray, budget_s: float, live_large: bool):
    """cpu_baseline of one suite entry: batched configs at all host threads
    (the value) and at one thread; the single large matrices from
    profiles/cpu_large.json (measured on a GPU box's host, provenance inside)
    unless --cpu-large re-measures them here."""
    threads = os.cpu_count() or 1
    spec = config_spec(name)
    if spec["n"] >= 20:
        if live_large:
            d = measure_cpu_large()
            src = "measured in this run"
        elif CPU_LARGE.exists():
            d = json.loads(CPU_LARGE.read_text())
            src = f"profiles/cpu_large.json ({d.get('when', '?')}, bench.py --cpu-large-only on a GPU box host)"
        else:
            return None
        e = dict(d.get(name) or {})
        if not e or "error" in e:
            return e or None
        e.update({"cpu_model": d.get("cpu_model"), "nproc": d.get("nproc"), "source": src})
        return e
    v, sample, kind, cores = cpu_reference_time(name, a, budget_s, threads)
    v1, sample1, _, _ = cpu_reference_time(name, a, budget_s, 1)
    return {"value": v, "unit": "permanents/s", "cores": cores, "kind": kind, "sample": sample,
            "single_thread": {"value": v1, "cores": 1, "sample": sample1}, "cpu_model": cpu_model(),
            "nproc": os.cpu_count()}


def suite_cpu_baseline_batch(a: np.ndarray, budget_s: float):
    """The reference engine on a bounded sample of the batch_n16 matrices
    (contiguous chunks over all host threads)."""
    from oracle import oracle as O

    if not O.ref_available():
        return {"error": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    done, t0, pos = 0, time.perf_counter(), 0
    while time.perf_counter() - t0 < budget_s:
        size = min(threads * 4, a.shape[0] - pos) or threads * 4
        if pos + size > a.shape[0]:
            pos = 0
        O.ref_sz_batch(a[pos:pos + size], nthreads=threads)
        pos += size
        done += size
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "permanents/s", "cores": threads, "kind": "reference",
            "sample": f"{done} matrices n={a.shape[1]} ({el:.1f} s wall, {threads} threads)", "cpu_model": cpu_model()}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    name = args.config
    spec, a = workload(name)
    threads = os.cpu_count() or 1
    n, count = spec["n"], spec["count"]
    per_step = []
    kind, cores, sample = None, None, None
    for i in range(args.warmup + args.steps):
        budget = 2.0 if i >= args.warmup else 0.5
        v, sample, kind, cores = cpu_reference_time(name, a, budget, threads)
        if i >= args.warmup:
            per_step.append(v)
    value = statistics.mean(per_step)
    line = {
        "impl": "reference",
        "metric": f"permanents/s ({name.upper()}: {spec['desc']})",
        "value": value, "unit": "permanents/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * count / value, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DT_SHORT[spec["dtype"]], "data": "synthetic (seeded generators following BASELINE.json recipes; no public dataset)",
        "config": config_dict(name, args.gpus, args.fma),
        "cpu_baseline": {"value": value, "unit": "permanents/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "permanents/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- device measurement

def measure_config(name, steps, warmup, rank, world, device, flush_buf, fma=False):
    import torch
    import torch.distributed as dist

    import paper_1802_02779_b200 as pl

    spec, a = workload(name)
    n, count = spec["n"], spec["count"]
    s = ELEM[spec["dtype"]]
    stream = torch.cuda.current_stream(device)
    a_host = torch.from_numpy(a).pin_memory()
    a_dev = a_host.to(device)
    status = torch.zeros(1, dtype=torch.int32, device=device)
    out = torch.empty(count, dtype=a_dev.dtype, device=device)
    sharded = world > 1 and n >= 20
    launches_per_step = 1 if n <= 16 else (n - 1)

    def step():
        if sharded:
            from paper_1802_02779_b200.sharded import sharded_permanent

            return sharded_permanent(a_dev[0], fma=fma)
        return pl.store_zechin_permanent_batch(a_dev, out=out, fma=fma, status=status, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    for _ in range(warmup):
        step()
    barrier()
    if not sharded and n <= 16:
        # Batches: the K steps read R device copies of the batch in rotation (R x input
        # > 2.5 x the 126 MB L2, so every step's input comes from HBM), captured once in
        # a CUDA graph and replayed between one event pair: whole-job throughput of a
        # stream of batches, with no flush kernels or per-step event gaps inside.
        in_bytes = a_dev.numel() * a_dev.element_size()
        reps = max(3, -(-(320 << 20) // in_bytes))
        bufs = [a_dev] + [a_dev.clone() for _ in range(reps - 1)]
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device)
        cap.wait_stream(stream)
        # the rotating copies were written long before the graph runs: PL_FLAG_INPUT_READY lets a
        # step's loads start while the previous step's kernel drains (its stores still wait)
        ready = os.environ.get("PL_BENCH_INPUT_READY", "1") != "0"
        with torch.cuda.stream(cap):
            for i in range(2):  # the API's lazy setup (kernel attributes) outside the capture
                pl.store_zechin_permanent_batch(bufs[i % reps], out=out, fma=fma, status=status, stream=cap,
                                                input_ready=ready)
        torch.cuda.synchronize(device)
        with torch.cuda.graph(graph, stream=cap):
            for i in range(steps):
                pl.store_zechin_permanent_batch(bufs[i % reps], out=out, fma=fma, status=status, stream=cap,
                                                input_ready=ready)
        for _ in range(2):
            graph.replay()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        barrier()
        times = [e0.elapsed_time(e1)]
        timing = f"{reps} rotating device copies of the batch ({reps * in_bytes / 2**20:.0f} MiB > L2), " \
                 f"{steps} steps in one CUDA graph between one event pair" \
                 + ("; PL_FLAG_INPUT_READY (a step's loads overlap the previous step's tail)" if ready and (n <= 5 or name == "c3") else "")
        del bufs
    else:
        evs = []
        for _ in range(steps):
            # evict the (< L2) inputs between timed steps, outside the event pair: write a
            # 256 MiB buffer, then read a second one so that the write's dirty lines are
            # written back before the timed step rather than during it
            flush_buf[0].add_(1)
            flush_buf[1].sum(dtype=torch.float32)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()  # asynchronous: the host runs ahead, the device never waits on it
            e1.record(stream)
            evs.append((e0, e1))
        barrier()
        times = [e0.elapsed_time(e1) for e0, e1 in evs]
        timing = "L2 flushed between timed steps (256 MiB write, then 256 MiB read), one event pair per step"
    if int(status.item()) != 0:
        raise RuntimeError(f"{name}: device status {int(status.item())}")
    t_local = sum(times) / 1000.0
    t = torch.tensor([t_local], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    units = count * steps * (world if not sharded else 1)
    value = units / t_max
    ms_step = 1000.0 * t_max / steps

    # e2e through the public API with pinned host buffers (H2D + compute + D2H inside)
    out_host = torch.empty(count, dtype=a_dev.dtype).pin_memory()
    # short host calls (batched configs: < 1 ms each) are sampled at least 30 times: one
    # host-scheduling hiccup of ~1 ms in a 10-call sample moved C3's e2e by 3x on the boxes
    e2e_steps = max(1, min(steps, 5)) if n >= 26 else (max(steps, 30) if n <= 16 else steps)
    for _ in range(2 if n >= 26 else warmup):  # warm the host path (pool growth, pinned staging)
        if sharded:
            from paper_1802_02779_b200.sharded import sharded_permanent

            sharded_permanent(a_host.to(device)[0], fma=fma)
        else:
            pl.store_zechin_permanent_batch(a_host, out=out_host, fma=fma, stream=stream)
    barrier()
    e2e_times = []
    for _ in range(e2e_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if sharded:
            from paper_1802_02779_b200.sharded import sharded_permanent

            ad = a_host.to(device, non_blocking=True)
            v = sharded_permanent(ad[0], fma=fma)
            out_host[0] = v
        else:
            pl.store_zechin_permanent_batch(a_host, out=out_host, fma=fma, stream=stream)
        e1.record(stream)
        e1.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
    te = torch.tensor([sum(e2e_times) / 1000.0], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = count * e2e_steps * (world if not sharded else 1) / float(te.item())

    bytes_per_launch = algorithmic_bytes_per_perm(n, s) * count
    per_launch_s = t_local / steps
    return {
        "name": name, "spec": spec, "value": value, "ms_per_step": ms_step, "t_max": t_max,
        "e2e": {"value": e2e_value, "unit": "permanents/s", "h2d_bytes_per_step": count * n * n * s,
                "d2h_bytes_per_step": count * s},
        "algorithmic_bytes_per_step": bytes_per_launch, "per_step_s": per_launch_s,
        "launches_per_step": launches_per_step, "flops_per_step": flops_per_perm(n, spec["dtype"]) * count,
        "sharded": sharded, "timing": timing, "fma": fma,
    }


BOSON = dict(m=25, modes=[0, 1, 2, 3, 4], seed=2,
             desc="full outcome distribution of 5 photons in Haar(25) seed 2, input modes 0..4 "
                  "(118,755 patterns; the collision-aware form of C2's submatrices)")
BOSON_LARGE = dict(m=40, modes=[0, 1, 2, 3, 4, 5], seed=6,
                   desc="full outcome distribution of 6 photons in Haar(40) seed 6, input modes 0..5 "
                        "(8,145,060 patterns: a launch long enough to reach the FP64 roofline)")
FP64_PEAK = (18.518, "measured DMUL/DADD rate x 1 flop (profiles/microbench_b200.json; the non-FMA reference "
                     "rounding mode issues no DFMA)")


def boson_flops_per_pattern(n: int) -> int:
    return flops_per_perm(n, "complex128") + 3  # + |z|^2 (2 mul, 1 add); the divide not counted


def measure_boson(steps, warmup, rank, world, device, flush_buf, fma=False, spec=None):
    """The boson driver's fused kernel (pl_boson_distribution): every pattern
    of the distribution enumerated, gathered, evaluated and normalised on the
    device. value: device buffers, asynchronous calls, events; e2e: the
    public host call (H2D of U, D2H of the probabilities)."""
    import torch
    import torch.distributed as dist

    from paper_1802_02779_b200 import boson as B

    spec = spec or BOSON
    itf = B.haar_unitary(spec["m"], spec["seed"])
    modes = spec["modes"]
    count = B.pattern_count(spec["m"], len(modes))
    stream = torch.cuda.current_stream(device)
    out = torch.empty(count, dtype=torch.float64, device=device)
    status = torch.zeros(1, dtype=torch.int32, device=device)

    def step():
        B.distribution_probabilities(itf, modes, out=out, stream=stream, status=status, fma=fma)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    for _ in range(warmup):
        step()
    barrier()
    # the kernel reads only U (10 KB): K steps captured in one CUDA graph, one event pair
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(device)
    cap.wait_stream(stream)
    ready = os.environ.get("PL_BENCH_INPUT_READY", "1") != "0"  # U is static: steps may overlap (PL_FLAG_INPUT_READY)
    with torch.cuda.graph(graph, stream=cap):
        for _ in range(steps):
            B.distribution_probabilities(itf, modes, out=out, stream=cap, status=status, fma=fma, input_ready=ready)
    for _ in range(2):
        graph.replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    graph.replay()
    e1.record(stream)
    barrier()
    t_local = e0.elapsed_time(e1) / 1000.0
    t = torch.tensor([t_local], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = count * steps * world / float(t.item())
    host = np.empty(count)
    for _ in range(warmup):
        B.distribution_probabilities(itf, modes, out=host, fma=fma)
    barrier()
    te = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        B.distribution_probabilities(itf, modes, out=host, fma=fma)
        e1.record(stream)
        e1.synchronize()
        te.append(e0.elapsed_time(e1) / 1000.0)
    tt = torch.tensor([sum(te)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = count * steps * world / float(tt.item())
    per_step = t_local / steps
    achieved = boson_flops_per_pattern(len(modes)) * count / per_step / 1e12
    return {
        "value": value, "unit": "probabilities/s", "ms_per_step": 1000.0 * float(t.item()) / steps, "steps": steps,
        "workload": spec["desc"], "patterns": count,
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK[0], "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK[0], "peak_source": FP64_PEAK[1],
                     "kernel": f"sz_boson_kernel<RC128,{len(modes)},VS=1> (enumerate + gather + DP + |per|^2/prod occ!)",
                     "hbm_bytes_per_pattern": 8},
        "e2e": {"value": e2e, "unit": "probabilities/s", "h2d_bytes_per_step": spec["m"] ** 2 * 16,
                "d2h_bytes_per_step": count * 8},
    }


def boson_cpu_reference(budget_s: float):
    """The reference's own full_distribution (oracle/_ref), single-threaded as
    the reference is; bounded by repeating it until budget_s."""
    from oracle import oracle as O

    from paper_1802_02779_b200 import boson as B

    if not O.ref_available():
        return None
    u = B.haar_unitary(BOSON["m"], BOSON["seed"]).unitary()
    done, t0 = 0, time.perf_counter()
    while True:
        _, p = O.ref_full_distribution(u, BOSON["modes"], enumeration_cap=10 ** 6)
        done += p.shape[0]
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": done / el, "unit": "probabilities/s", "cores": 1, "kind": "reference",
            "sample": f"{done} patterns ({done // p.shape[0]} x full_distribution, {el:.1f} s, 1 thread)"}


DFMA_PEAK = (33.40, "measured DFMA rate x 2 flop (profiles/microbench_b200.json: 16.7 T DFMA/s)")


FP32_PEAK = (74.4, "nominal FFMA rate x 2 flop (148 SMs x 128 FFMA/clk x 1.965 GHz)")


def kernel_name(n: int, dtype: str = "") -> str:
    if n <= 5:
        return "sz_batch_tma_kernel"
    if 10 <= n <= 14 and dtype == "int64":
        return "sz_batch_f32_pack_kernel (four matrices per CTA, exact integers on the FP32 pipe)"
    if n <= 14:
        return "sz_batch_smem_pack_kernel (8-byte) / sz_batch_smem_kernel (complex)"
    return "sz_ws_kernel (middle layers) + sz_lean_kernel (layers <= 24 MB), all layers of one step"


def roofline_of(res, peak, peak_src, traffic):
    """The dominant kernel's roofline on its binding resource: HBM for the
    streaming batches (n <= 5) and the layer DP (compulsory layer traffic);
    the FP64 pipe for the shared-memory batch kernels (n = 6..14), whose
    input is a few KB per matrix against ~10^4-10^5 DFMA (C3: 45,045 exact
    integer ops per permanent executed as DFMA on exact doubles)."""
    n = res["spec"]["n"]
    dtype = res["spec"]["dtype"]
    tr = traffic.get(res["name"])
    fp = res["flops_per_step"] / res["per_step_s"] / 1e12
    if 10 <= n <= 14 and dtype == "int64":
        return {"bound": "fp32", "achieved": fp, "peak": FP32_PEAK[0], "unit": "TFLOP/s", "frac": fp / FP32_PEAK[0],
                "peak_source": FP32_PEAK[1], "traffic": tr, "kernel": kernel_name(n, dtype),
                "hbm_gbs": res["algorithmic_bytes_per_step"] / res["per_step_s"] / 1e9,
                "fp64_equivalent_frac": fp / DFMA_PEAK[0],
                "note": "exact integers on the FP32 pipe (every value provably < 2^24); co-limited by the "
                        "L1TEX/shared-memory data pipe (74 % busy: a 16-byte operand pack per term; the coefficient "
                        "pack is one word of four bytes) and instruction issue (69 %), profiles/r2c/"
                        "full_c3_byte_coef.md -- not by the FFMA rate"}
    if 6 <= n <= 14:
        return {"bound": "fp64", "achieved": fp, "peak": DFMA_PEAK[0], "unit": "TFLOP/s", "frac": fp / DFMA_PEAK[0],
                "peak_source": DFMA_PEAK[1], "traffic": tr, "kernel": kernel_name(n, dtype),
                "hbm_gbs": res["algorithmic_bytes_per_step"] / res["per_step_s"] / 1e9,
                "note": "bytes are ~1 KB per 45 k ops: neither HBM nor L2 binds; the FP64 pipe is the ceiling "
                        "(shared-memory operand loads are the measured limiter, DESIGN.md section 4)"}
    achieved = res["algorithmic_bytes_per_step"] / res["per_step_s"] / 1e9
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": tr, "peak_source": peak_src, "kernel": kernel_name(n, dtype), "fp_rate_tflops": fp}
    if n >= 20:
        fpk = FP64_PEAK if not res.get("fma") else DFMA_PEAK
        out["fp64_frac"] = fp / fpk[0]
        out["fp64_peak_source"] = fpk[1]
    return out


def cold_call(name: str, fma: bool) -> dict:
    """First call of the public API in a fresh process (library load, module
    load, tables and schedules, scratch allocation, H2D, compute, D2H), after
    the CUDA context exists: what a one-matrix-per-process caller (the
    reference CLI `perm`) pays. Run as `bench.py --cold-call NAME`."""
    import torch

    torch.cuda.init()
    torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    _, a = workload(name)
    t0 = time.perf_counter()
    import paper_1802_02779_b200 as pl

    t1 = time.perf_counter()
    v = pl.store_zechin_permanent_batch(a, fma=fma)
    t2 = time.perf_counter()
    pl.store_zechin_permanent_batch(a, fma=fma)
    t3 = time.perf_counter()
    return {"config": name, "first_call_ms": 1e3 * (t2 - t0), "import_ms": 1e3 * (t1 - t0),
            "second_call_ms": 1e3 * (t3 - t2), "value_ok": bool(np.all(np.isfinite(np.asarray(v).view(np.float64))))}


def measure_cold(name: str, fma: bool):
    import subprocess

    cmd = [sys.executable, str(ROOT / "bench.py"), "--cold-call", name] + (["--fma"] if fma else [])
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)[:200]}


def suite_entry(r, name, steps, peak, peak_src, traffic, world):
    from paper_1802_02779_b200.sharded import block_plan_applies

    return {"value": r["value"], "unit": "permanents/s", "ms_per_step": r["ms_per_step"], "steps": steps,
            "time_to_permanent_ms": r["ms_per_step"] if r["spec"]["count"] == 1 else None,
            "arith": "fma" if r["fma"] else "reference rounding order (no FMA)",
            "roofline": roofline_of(r, peak, peak_src, traffic), "e2e": r["e2e"], "timing": r["timing"],
            "sharded": (("top-column blocks, point-to-point" if block_plan_applies(r["spec"]["n"], world)
                         else "equal slices, all-gather") if r["sharded"] else None)}


BATCH16 = {"n": 16, "count": 2000, "seed": 16,
           "desc": "2,000 x 16x16 complex128 (standard complex Gaussian, seed 16): a batch of large orders, "
                   "every layer of the batch in one lean launch"}
RYSER = {"n": 22, "seed": 22, "cpu_n": 18,
         "desc": "Ryser engine (pl_ryser_permanent), single 22x22 float64 matrix, uniform [-1, 1] (seed 22); "
                 "bitwise the reference's visit-order fold"}


BIGINT = {"n": 24, "seed": 24,
          "desc": "exact Int beyond int64: single 24x24 integer matrix, entries uniform in [0, 3] (seed 24), "
                  "permanent ~2^93; int64 attempt (overflow reported) + residue passes modulo 31-bit primes + CRT"}


def bigint_matrix():
    return np.random.default_rng(BIGINT["seed"]).integers(0, 4, (BIGINT["n"], BIGINT["n"]), dtype=np.int64)


def measure_bigint(steps, warmup):
    """The public call on a matrix whose permanent leaves int64 (reference ring.hpp:29-31: Int is
    arbitrary precision). Host call, H2D/D2H and the host-side CRT inside the timed region."""
    import paper_1802_02779_b200 as pl

    a = bigint_matrix()
    for _ in range(warmup):
        v = pl.store_zechin_permanent(a).value
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        v = pl.store_zechin_permanent(a).value
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    bound_bits = sum(int(r.sum()).bit_length() for r in a)
    return {"value": 1.0 / t, "unit": "permanents/s", "time_to_permanent_ms": 1e3 * t, "steps": steps,
            "workload": BIGINT["desc"], "result_bits": int(v).bit_length(),
            "residue_passes": max(1, (bound_bits + 2 + 29) // 30), "result": str(v)}


def bigint_cpu_reference(device_result):
    from oracle import oracle as O

    if not O.ref_available():
        return {"error": "oracle/_ref not built"}
    a = bigint_matrix()
    t0 = time.perf_counter()
    v, _ = O.ref_sz_int(a, memo_budget_bytes=1 << 36)  # its 2^24-slot memo table exceeds the default budget
    t = time.perf_counter() - t0
    return {"value": 1.0 / t, "unit": "permanents/s", "cores": 1, "kind": "reference",
            "sample": f"reference store_zechin_permanent on the same matrix ({t:.2f} s, 1 thread; the engine is "
                      "single-threaded)", "equal_to_device_result": str(v) == device_result}


def measure_batch16(steps, warmup, device):
    """Batched large orders (callers looping store_zechin_permanent at 15 <= n <= 20):
    value device-resident, events around K back-to-back calls; CPU baseline the reference engine."""
    import torch

    import paper_1802_02779_b200 as pl

    n, cnt = BATCH16["n"], BATCH16["count"]
    rng = np.random.default_rng(BATCH16["seed"])
    a_np = rng.standard_normal((cnt, n, n)) + 1j * rng.standard_normal((cnt, n, n))
    a = torch.from_numpy(a_np).to(device)
    out = torch.empty(cnt, dtype=torch.complex128, device=device)
    st = torch.zeros(1, dtype=torch.int32, device=device)
    for _ in range(warmup):
        pl.store_zechin_permanent_batch(a, out=out, status=st)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pl.store_zechin_permanent_batch(a, out=out, status=st)
    e1.record()
    torch.cuda.synchronize(device)
    t = e0.elapsed_time(e1) / 1000.0 / steps
    flops = flops_per_perm(n, "complex128") * cnt
    res = {"value": cnt / t, "unit": "permanents/s", "ms_per_step": 1e3 * t, "steps": steps,
           "workload": BATCH16["desc"],
           "roofline": {"bound": "fp64", "achieved": flops / t / 1e12, "peak": FP64_PEAK[0], "unit": "TFLOP/s",
                        "frac": flops / t / 1e12 / FP64_PEAK[0], "peak_source": FP64_PEAK[1],
                        "kernel": "sz_lean_kernel (batched: tiles of all matrices per launch)"},
           "per_matrix_path_ms": None}
    t0 = time.perf_counter()
    host = pl.store_zechin_permanent_batch(a_np)
    res["e2e"] = {"value": cnt / (time.perf_counter() - t0), "unit": "permanents/s",
                  "h2d_bytes_per_step": int(a_np.nbytes), "d2h_bytes_per_step": int(host.nbytes)}
    return res, a_np


def measure_ryser(steps, warmup):
    import torch

    import paper_1802_02779_b200 as pl

    a = np.random.default_rng(RYSER["seed"]).uniform(-1, 1, (RYSER["n"], RYSER["n"]))
    for _ in range(warmup):
        pl.ryser_permanent(a)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        pl.ryser_permanent(a)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return {"value": 1.0 / t, "unit": "permanents/s", "time_to_permanent_ms": 1e3 * t, "steps": steps,
            "workload": RYSER["desc"],
            "note": "host call incl. H2D/D2H; the visit-order fold of 2^22 - 1 terms is one sequential chain "
                    "(bitwise the reference), so the device time is latency-bound by design"}


def ryser_cpu_reference():
    from oracle import oracle as O

    if not O.ref_available():
        return {"error": "oracle/_ref not built"}
    n = RYSER["cpu_n"]
    a = np.random.default_rng(RYSER["seed"]).uniform(-1, 1, (n, n)).astype(np.complex128)
    t0 = time.perf_counter()
    O.ref_ryser_c128(a)
    t = time.perf_counter() - t0
    scale = (RYSER["n"] * 2 ** RYSER["n"]) / (n * 2 ** n)
    return {"value": 1.0 / (t * scale), "unit": "permanents/s", "cores": 1, "kind": "reference",
            "sample": f"reference ryser_permanent at n={n} ({t:.2f} s, 1 thread), scaled by n*2^n to n={RYSER['n']}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-large", action="store_true", help="re-measure the C4/C5 CPU baselines in this run (~2 min)")
    ap.add_argument("--cpu-large-only", action="store_true", help="print the C4/C5 CPU baselines as JSON and exit")
    ap.add_argument("--cold-call", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--fma", action="store_true", help="allow FMA contraction (not the reference rounding order)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return run_reference_arm(args)
    if args.cpu_large_only:
        print(json.dumps(measure_cpu_large(), indent=1), flush=True)
        return 0
    if args.cold_call:
        print(json.dumps(cold_call(args.cold_call, args.fma)), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import datetime

        # a finite timeout: a stuck collective in the sharded suite entries errors out
        # (and is reported in the suite) instead of hanging the job
        dist.init_process_group("nccl", device_id=device, timeout=datetime.timedelta(seconds=300))

    flush_buf = torch.zeros(2, 64 * 1024 * 1024, dtype=torch.float32, device=device)  # 2 x 256 MiB > 126 MB L2
    peak, peak_src = load_peaks()
    traffic = load_traffic()
    cpu_on = rank == 0 and world == 1 and not args.no_cpu

    with ClockSampler(local) as clocks:
        head = measure_config(args.config, args.steps, args.warmup, rank, world, device, flush_buf, args.fma)
        suite = {}
        if not args.no_suite:
            plan = [("c1", False), ("c2", False), ("c3", False), ("c4", False), ("c4_fma", True), ("c5", False),
                    ("c5_fma", True)]
            for key, fma in plan:
                name = key.split("_")[0]
                # batched configs: a replayed graph of 40 steps (5-70 us each), so that the first step,
                # which has no predecessor to overlap with, weighs little
                k = {"c1": 40, "c2": 40, "c3": 40, "c4": 5, "c5": 2}[name]
                try:
                    same = name == args.config and fma == args.fma
                    r = head if same else measure_config(name, k, 3, rank, world, device, flush_buf, fma)
                except Exception as e:  # e.g. the sharded large-order path on a multi-GPU run
                    print(f"bench: suite entry {key} failed: {e!r}", file=sys.stderr, flush=True)
                    suite[key] = {"error": repr(e)[:300]}
                    continue
                suite[key] = suite_entry(r, name, args.steps if same else k, peak, peak_src, traffic, world)
            if world == 1:
                try:
                    suite["batch_n16"], a16 = measure_batch16(5, 2, device)
                except Exception as e:  # noqa: BLE001
                    print(f"bench: suite entry batch_n16 failed: {e!r}", file=sys.stderr, flush=True)
                    suite["batch_n16"], a16 = {"error": repr(e)[:300]}, None
                try:
                    suite["ryser"] = measure_ryser(5, 2)
                except Exception as e:  # noqa: BLE001
                    suite["ryser"] = {"error": repr(e)[:300]}
                try:
                    suite["bigint"] = measure_bigint(5, 2)
                except Exception as e:  # noqa: BLE001
                    suite["bigint"] = {"error": repr(e)[:300]}
            for key, steps_b, spec_b in (("boson", 10, BOSON), ("boson_large", 3, BOSON_LARGE)):
                try:
                    suite[key] = measure_boson(steps_b, 3, rank, world, device, flush_buf, args.fma, spec_b)
                except Exception as e:
                    print(f"bench: suite entry {key} failed: {e!r}", file=sys.stderr, flush=True)
                    suite[key] = {"error": repr(e)[:300]}

    if not args.no_suite and rank == 0 and world == 1:
        # cold first calls (fresh processes), outside the clock-sampled region
        for key in ("c4", "c5"):
            if key in suite and "error" not in suite[key]:
                suite[key]["cold_call"] = measure_cold(key, False)
    if cpu_on and not args.no_suite:
        for key in ("c1", "c2", "c3", "c4", "c5"):
            if key in suite and "error" not in suite[key]:
                _, a = workload(key)
                try:
                    suite[key]["cpu_baseline"] = suite_cpu_baseline(key, a, 3.0, args.cpu_large)
                except Exception as e:  # noqa: BLE001
                    suite[key]["cpu_baseline"] = {"error": repr(e)[:200]}
        if "error" not in suite.get("boson", {"error": 1}):
            suite["boson"]["cpu_baseline"] = boson_cpu_reference(5.0)
        if "error" not in suite.get("batch_n16", {"error": 1}) and a16 is not None:
            try:
                suite["batch_n16"]["cpu_baseline"] = suite_cpu_baseline_batch(a16, 5.0)
            except Exception as e:  # noqa: BLE001
                suite["batch_n16"]["cpu_baseline"] = {"error": repr(e)[:200]}
        if "error" not in suite.get("ryser", {"error": 1}):
            suite["ryser"]["cpu_baseline"] = ryser_cpu_reference()
        if "error" not in suite.get("bigint", {"error": 1}):
            try:
                suite["bigint"]["cpu_baseline"] = bigint_cpu_reference(suite["bigint"]["result"])
            except Exception as e:  # noqa: BLE001
                suite["bigint"]["cpu_baseline"] = {"error": repr(e)[:200]}

    cpu = None
    if cpu_on:
        if not args.no_suite and args.config in suite and suite[args.config].get("cpu_baseline"):
            cpu = dict(suite[args.config]["cpu_baseline"])
        else:
            _, a = workload(args.config)
            cpu = suite_cpu_baseline(args.config, a, 10.0, args.cpu_large)

    if rank == 0:
        spec = head["spec"]
        line = {
            "metric": f"permanents/s ({args.config.upper()}: {spec['desc']})",
            "value": head["value"], "unit": "permanents/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "weak" if not head["sharded"] else "strong", "vs_baseline": None,
            "dtype": DT_SHORT[spec["dtype"]],
            "data": "synthetic (seeded generators following BASELINE.json recipes; no public dataset)",
            "config": config_dict(args.config, world, args.fma),
            "roofline": roofline_of(head, peak, peak_src, traffic),
            "cpu_baseline": cpu,
            "e2e": head["e2e"],
            "clocks": clocks.summary(),
            "gpu_launches": head["launches_per_step"] * args.steps,
            "suite": suite,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        try:
            dist.barrier()
            dist.destroy_process_group()
        except Exception as e:  # the JSON line is already out
            print(f"bench: teardown: {e!r}", file=sys.stderr, flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
