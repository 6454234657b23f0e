#!/usr/bin/env python
"""Benchmark of the α-DFT / α-FFT hot path (BASELINE.json metric:
"α-FFT complex points/sec & % of HBM roofline at 1/2/4/8 B200 vs CPU oracle").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--method auto]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference      # the reference's own CPU path on host cores

Workload: BASELINE config 4 by default (65536 signals x N=8192 complex64,
α = 1/8, M = N), the config the metric is quoted on at 1/2/4/8 GPUs; the
batch is split into contiguous shards, one per rank, with no communication in
the timed region (strong scaling of a fixed total batch).  A step is one
transform of the rank's whole shard.  Rank 0 prints ONE JSON line.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL); under torchrun
the world size must equal N.  After the timed region every rank checks ALL
of its shard's bins against the complex128 GPU path (a different algorithm)
on the same inputs and the per-signal max|ΔX|/max|X| is all-reduced (MAX)
into the line's ``parity`` field.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="4", help="BASELINE config key: 0, 1a, 1b, 3, 4")
    ap.add_argument("--method", default="auto", choices=["auto", "fft", "chirp", "direct"])
    ap.add_argument("--impl", default="asx", choices=["asx", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override total batch (testing)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the non-production methods")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the side measurements of configs 1a, 1b and 3 (not part of value)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target busy seconds per host core for the CPU baseline sample")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N > 1 (gloo lets several ranks share one GPU in tests)")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-run parity check")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0,
                    help="--impl reference: target wall seconds of one step (a bounded sample)")
    return ap.parse_args()


def maybe_self_launch(args) -> None:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run, N ranks."""
    if "WORLD_SIZE" in os.environ:
        ws = int(os.environ["WORLD_SIZE"])
        if ws != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank per GPU")
        return
    if args.gpus <= 1:
        return
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


from paper_2403_16665_b200.dist import barrier as dist_barrier  # noqa: E402
from paper_2403_16665_b200.dist import gather_checksums, max_over_ranks, shard_range, sum_over_ranks  # noqa: E402
from paper_2403_16665_b200.dist import world as dist_env  # noqa: E402


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def tensor_peak():
    """Dense fp16/bf16 tensor-core peak (TFLOP/s): MEASURED_PEAKS.json's cuBLAS bf16 burst figure."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"]), "measured bf16_tflops (MEASURED_PEAKS.json)"
    except Exception:
        return 2250.0, "nominal dense bf16/fp16"


def tensor_peak_sustained():
    """cuBLAS bf16 back to back for seconds (MEASURED_PEAKS.json bf16_tflops_sustained): the rate the
    chip holds under its power cap (SM clock ~1.3-1.5 GHz), which a kernel timed over many launches meets."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops_sustained"])
    except Exception:
        return None


def fp_peak(dtype: str):
    """Measured FFMA / DFMA peak (TFLOP/s) of a pool B200 (scripts/fp_peaks.cu -> profiles/fp_peaks.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "fp_peaks.json")) as fh:
            d = json.load(fh)
        return float(d["fp32_tflops" if dtype == "complex64" else "fp64_tflops"]), "measured (profiles/fp_peaks.json)"
    except Exception:
        return (74.4 if dtype == "complex64" else 37.2), "nominal 148 SMs x 1.965 GHz"


def pcie_duplex(dev, mib=512, reps=5):
    """Concurrent H2D + D2H bandwidth from pinned memory (GB/s per direction): the e2e roofline.
    Both copies start from one common event (so they truly overlap); best of `reps`."""
    import torch

    n = mib << 20
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.zeros(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    best_h2d = best_d2h = 0.0
    for _ in range(reps + 1):
        torch.cuda.synchronize(dev)
        go = torch.cuda.Event()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        evs[0].record(s1)
        go.record(s1)
        s2.wait_event(go)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        evs[1].record(s1)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        evs[2].record(s2)
        torch.cuda.synchronize(dev)
        best_h2d = max(best_h2d, n / (evs[0].elapsed_time(evs[1]) / 1e3) / 1e9)
        best_d2h = max(best_d2h, n / (evs[0].elapsed_time(evs[2]) / 1e3) / 1e9)
    return best_h2d, best_d2h


def launched_kernel(method: str) -> str:
    """Name of the kernel the last execute launched (asx_last_launch variant bits)."""
    import ctypes

    from paper_2403_16665_b200 import _lib

    v = [ctypes.c_int() for _ in range(4)]
    _lib.lib().asx_last_launch(*[ctypes.byref(c) for c in v])
    variant = v[3].value >> 1
    if method == "chirp" and variant == 14:
        return "k_chirp_r32<float> (32 values per thread, 4 exchanges per signal, csrc/asx_chirp_r32.cuh)"
    if method == "chirp" and variant == 2:
        return "k_chirp_local<float> (group-local exchanges, csrc/asx_chirp_local.cuh)"
    if method == "fft" and variant == 4:
        return "k_afft_local<double> (group-local alpha-FFT, csrc/asx_afft_local.cuh)"
    if method == "chirp" and variant == 6:
        return "k_chirp_local128<double> (group-local chirp-z, csrc/asx_chirp_local128.cuh)"
    if method == "direct" and variant == 8:
        return "k_direct_tc (tcgen05.mma kind::f16, fp16 hi/lo split, TMEM accumulators, csrc/asx_direct_tc.cuh)"
    if method == "direct":
        return "k_direct"
    kind = "afft" if method == "fft" else "chirp"
    return f"k_fft_persist<{kind}{', TMEM tables' if variant == 1 else ''}>"


def profiled_traffic(config_key: str, method: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(f"{config_key}:{method}")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU reference
#
# The reference package, installed unmodified into baseline/_ref (DESIGN.md
# §6: pip install --no-index --no-deps --target baseline/_ref), timed through
# its own public API: fastpath.transform_samples with a pre-built plan, one
# signal per call as the reference's batching is a Python loop
# (ref/fastpath.py:162-181; plan construction untimed, ref/bench.py:14-16).
# Configs the reference cannot run (config 3: alpha*N not an integer; config
# 1b: alpha_ref = 10 has no power-of-two plan, its route is naive_forward)
# use the reference's naive_forward when it accepts the pair, else the CPU
# oracle port (kind "port").

REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _ref_module():
    if os.path.isdir(os.path.join(REF_DIR, "alpha_spectra")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import alpha_spectra

        return alpha_spectra
    return None


def _ref_callable(key: str):
    """(kind, fn(row) -> bins[:M]) of the reference's CPU path for a workload."""
    from paper_2403_16665_b200.signals import WORKLOADS

    w = WORKLOADS[key]
    a, d = w.alpha.numerator, w.alpha.denominator  # BASELINE alpha = a/d = 1 / DenseFactor(d, a)
    ref = _ref_module()
    if ref is not None and (w.n * d) % a == 0:
        from alpha_spectra import fastpath, oracle
        from alpha_spectra.core import DenseFactor, Signal

        density = DenseFactor(d, a)
        try:
            pl = fastpath.plan(w.n, density)  # untimed, as the reference's bench
            return "reference", "alpha_spectra.fastpath.transform_samples", \
                lambda row: fastpath.transform_samples(row, pl)[: w.m]
        except ValueError:
            return "reference", "alpha_spectra.oracle.naive_forward", \
                lambda row: oracle.naive_forward(Signal(row), density).bins[: w.m]
    from oracle import alpha_oracle as orc  # CPU baseline leg only: the port, when the reference cannot run

    if a == 1 and (w.n & (w.n - 1)) == 0:
        return "port", "oracle/alpha_oracle.py alpha_fft (restated transform_samples)", \
            lambda row: orc.alpha_fft(row[None], a, d, w.m)[0]
    return "port", "oracle/alpha_oracle.py direct (restated naive_forward, generalised alpha)", \
        lambda row: orc.direct(row[None], a, d, w.m)[0]


_POOL_STATE = {}


def _pool_init(key, lo_hi):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import numpy as np

    from paper_2403_16665_b200.signals import WORKLOADS, generate

    _POOL_STATE["fn"] = _ref_callable(key)[2]
    _POOL_STATE["key"] = key
    _POOL_STATE["np"] = np
    _POOL_STATE["gen"] = lambda lo, hi: generate(WORKLOADS[key], lo, hi - lo, threads=1).astype(np.complex128)


def _pool_step(lo_hi):
    """One worker's share of a step: its signals, one reference call each; busy seconds."""
    lo, hi = lo_hi
    x = _POOL_STATE.get(("x", lo, hi))
    if x is None:
        x = _POOL_STATE["gen"](lo, hi)  # generated once per worker slice, untimed
        _POOL_STATE[("x", lo, hi)] = x
    fn = _POOL_STATE["fn"]
    t0 = time.perf_counter()
    for row in x:
        fn(row)
    return time.perf_counter() - t0


class RefPool:
    """All host cores, one process each (OPENBLAS_NUM_THREADS=1), each looping the
    reference over its contiguous slice of a bounded sample."""

    def __init__(self, key: str, step_seconds: float):
        import multiprocessing as mp

        from paper_2403_16665_b200.signals import WORKLOADS

        self.key = key
        self.w = WORKLOADS[key]
        self.kind, self.api, fn = _ref_callable(key)
        self.cores = len(os.sched_getaffinity(0))
        # calibrate one core on 2 signals, then size a step to ~step_seconds
        import numpy as np

        from paper_2403_16665_b200.signals import generate

        x = generate(self.w, 0, 2, threads=1).astype(np.complex128)
        fn(x[0])
        t0 = time.perf_counter()
        fn(x[1])
        self.per_signal = max(time.perf_counter() - t0, 1e-6)
        per_core = max(1, int(step_seconds / self.per_signal))
        self.sample = min(self.w.batch, per_core * self.cores)
        self.sample = max(1, self.sample)
        nproc = min(self.cores, self.sample)
        self.slices = [(i * self.sample // nproc, (i + 1) * self.sample // nproc) for i in range(nproc)]
        self.pool = mp.get_context("fork").Pool(nproc, initializer=_pool_init, initargs=(key, None))
        self.pool.map(_pool_step, self.slices)  # generate the slices (untimed) and warm up

    def step(self) -> float:
        """Seconds of one step: the busiest worker's time on its slice."""
        return max(self.pool.map(_pool_step, self.slices))

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, busy: float) -> dict:
        return {"value": self.sample * self.w.m / busy, "unit": "complex points/s", "cores": len(self.slices),
                "kind": self.kind,
                "sample": f"{self.sample} of {self.w.batch} signals of config {self.key} per step "
                          f"({len(self.slices)} processes x ~{self.sample // len(self.slices)} signals, one "
                          f"{self.api} call per signal, {busy:.2f} s for the busiest process; "
                          f"{'baseline/_ref, unmodified' if self.kind == 'reference' else 'CPU restatement'})"}


def cpu_reference(key: str, target_seconds: float):
    """cpu_baseline of the GPU arm: one bounded step of the reference on all host cores."""
    pool = RefPool(key, target_seconds)
    try:
        busy = min(pool.step() for _ in range(2))
    finally:
        pool.close()
    return pool.describe(busy)


# ----------------------------------------------------------------- GPU arm

def side_config(key, dev, stream, peak, reps=20):
    """Device time of another BASELINE config (method auto) with CUDA events on
    the launch stream, after warm-up; inputs exceed L2."""
    import torch

    import paper_2403_16665_b200 as asx
    from paper_2403_16665_b200.signals import WORKLOADS, generate_device

    w = WORKLOADS[key]
    x = generate_device(w, 0, w.batch, device=dev)
    p = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method="auto", real_input=w.real, device=dev.index)
    out = torch.empty((w.batch, w.m), dtype=getattr(torch, w.dtype), device=dev)
    for _ in range(3):
        p.execute(x, out=out)
    torch.cuda.synchronize()
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_.record(stream)
    for _ in range(reps):
        p.execute(x, out=out)
    e_.record(stream)
    torch.cuda.synchronize()
    ms = s_.elapsed_time(e_) / reps
    kern = launched_kernel(p.method)
    if p.fft_size > 16384:  # past one CTA: the four-step path (asx_last_launch reports its last pass only)
        kern = ("k_large_cols + k_large_rows_local + k_large_cols (four-step chirp-z, 3 launches, csrc/asx_large.cuh)"
                if p.method == "chirp" else "k_large_cols + k_large_rows per residue (four-step alpha-FFT, csrc/asx_large.cuh)")
    gbs = w.bytes_alg(w.batch) / (ms / 1e3) / 1e9
    res = {"workload": f"config {w.key}: batch {w.batch} x N={w.n} {w.dtype}, alpha={w.alpha}, M={w.m}",
           "method": p.method, "kernel": kern, "ms_per_step": ms, "value": w.batch * w.m / (ms / 1e3),
           "unit": "complex points/s", "hbm_gbs": gbs, "hbm_frac": gbs / peak, "reps": reps,
           "traffic": profiled_traffic(key, p.method), "bytes_alg": w.bytes_alg(w.batch)}
    if kern.startswith("k_direct_tc"):
        # direct form: 8 M N flops per signal; the tensor cores execute 3x that
        # (A_hi B_hi + A_hi B_lo + A_lo B_hi per real product)
        flops = 8.0 * w.m * w.n * w.batch
        tp, src = tensor_peak()
        res["tensor"] = {"alg_tflops": flops / (ms / 1e3) / 1e12,
                         "executed_tflops": 3 * flops / (ms / 1e3) / 1e12, "peak_tflops": tp,
                         "frac": 3 * flops / (ms / 1e3) / 1e12 / tp, "peak_source": src,
                         "flops": "8 M N per signal (direct form); executed = 3x (fp16 hi/lo split)"}
        tps = tensor_peak_sustained()
        if tps:
            # the kernel is power-limited like cuBLAS run back to back (profiles/r2_c3_direct_tc_waits.txt:
            # SM clock ~1.45-1.55 GHz under it), so the sustained cuBLAS rate is the fair yardstick
            res["tensor"]["sustained_peak_tflops"] = tps
            res["tensor"]["frac_of_sustained"] = res["tensor"]["executed_tflops"] / tps
    del x, out
    torch.cuda.empty_cache()
    return res


def workload_config(w, total, world, big_inputs) -> dict:
    """The config dict both arms print (same keys and values for the same run)."""
    return {"workload": f"config {w.key}: batch {total} x N={w.n} {w.dtype}, alpha={w.alpha}, M={w.m}",
            "batch": total, "n": w.n, "m": w.m, "alpha": str(w.alpha), "dtype": w.dtype,
            "parallelism": f"dp{world} (batch shards, no data-path collective)",
            "l2": "inputs larger than L2 (no flush)" if big_inputs else "L2 flushed between steps"}


def executed_flops(w, plan, nloc, launch_s, peak):
    """Textbook flop count of the algorithm the kernel actually runs (radix-2
    count 5 P log2 P per complex P-point FFT, 6 flops per complex product),
    against the measured FP peak -- beside the reference op-count credit."""
    P = max(plan.fft_size, 1)
    lg = max(1, (P - 1).bit_length())
    if plan.method == "chirp":
        per, how = 2 * 5 * P * lg + 6 * 3 * P, "chirp-z: 2 P-point FFTs + 3 complex products per point"
    elif plan.method == "fft":
        r = max(1, w.alpha.denominator // max(1, w.alpha.numerator))
        per, how = r * (5 * P * lg + 6 * P), "alpha-FFT: r P-point FFTs + r pre-twiddles per point"
    else:
        per, how = 8 * w.m * w.n, "direct: 8 M N"
    tf = per * nloc / launch_s / 1e12
    return {"flops_per_signal": per, "how": how, "achieved_tflops": tf, "frac": tf / peak}


def shard_parity(asx, w, x, out, dev, chunk=2048):
    """Per-signal max|ΔX|/max|X| (ref/verify.py:75-77) of a rank's whole output
    shard against the complex128 GPU path on the same inputs: the FP64 α-FFT
    recursion where the plan allows it, else chirp-z / direct -- always a
    different algorithm or precision from the production plan."""
    import torch

    tol = 2e-5 if w.dtype == "complex64" else 1e-10
    ref = None
    for meth in ("fft", "chirp", "direct"):
        if w.dtype == "complex128" and meth == out_method(out):
            continue
        try:
            ref = asx.plan(w.n, w.density, m=w.m, dtype="complex128", method=meth, real_input=w.real,
                           device=dev.index)
            break
        except Exception:
            continue
    worst, nsig = 0.0, 0
    for b0 in range(0, x.shape[0], chunk):
        xi = x[b0:b0 + chunk]
        xi = xi.to(torch.float64 if w.real else torch.complex128)
        want = ref.execute(xi)
        got = out[b0:b0 + chunk].to(torch.complex128)
        den = want.abs().amax(dim=1).clamp_min(1e-300)
        worst = max(worst, float(((got - want).abs().amax(dim=1) / den).max()))
        nsig += xi.shape[0]
    return {"max_rel_err": worst, "tolerance": tol, "signals_checked": nsig,
            "reference": f"complex128 GPU plan, method {ref.method} (fft_size {ref.fft_size}), same inputs",
            "metric": "per-signal max|dX| / max|X| (ref/verify.py:75-77), MAX over all signals and ranks"}


_OUT_METHOD = {}


def out_method(out):
    return _OUT_METHOD.get(id(out))


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2403_16665_b200 as asx
    from paper_2403_16665_b200.signals import WORKLOADS, generate_device

    world, rank, local = dist_env()
    ndev = torch.cuda.device_count()
    if ndev < 1:
        sys.exit("bench.py: no CUDA device (libasx has no CPU fallback)")
    if args.dist_backend == "nccl" and world > ndev:
        sys.exit(f"bench.py: {world} ranks but {ndev} GPU(s); NCCL needs one GPU per rank")
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    barrier = dist_barrier

    w = WORKLOADS[args.config]
    total = args.batch or w.batch
    lo, hi = shard_range(total, world, rank)
    nloc = hi - lo
    x = generate_device(w, lo, nloc, device=dev)
    plan = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=args.method, real_input=w.real,
                    device=dev.index)
    out = torch.empty((nloc, w.m), dtype=getattr(torch, w.dtype), device=dev)
    _OUT_METHOD[id(out)] = plan.method
    stream = torch.cuda.current_stream(dev)
    bytes_step = w.bytes_alg(nloc)
    flush = None
    if bytes_step < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        plan.execute(x, out=out)
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(dev.index)
    barrier()
    torch.cuda.synchronize()
    with clocks:
        for s, e in evs:
            if flush is not None:
                flush.zero_()
            s.record(stream)
            plan.execute(x, out=out)
            e.record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in evs]
    tot_ms = sum(step_ms)
    tot_ms_max = max_over_ranks(tot_ms, device=dev)
    ms_per_step = tot_ms_max / args.steps
    value = total * w.m / (ms_per_step / 1e3)
    # roofline of the dominant (only) kernel: algorithmic bytes per launch / avg launch duration
    avg_launch_s = (tot_ms / args.steps) / 1e3
    kernel_name = launched_kernel(plan.method)  # before other methods / the host path launch
    peak, peak_kind = measured_peaks()
    fpk, fpk_src = fp_peak(w.dtype)
    achieved = bytes_step / avg_launch_s / 1e9
    flops = w.flops_alg(nloc)

    # the other method(s) on the same shard, for reference (the α-FFT recursion
    # is the paper's algorithm; `auto` picks the cheapest for the config)
    alt = {}
    if not args.no_alt:
        for meth in ("fft", "chirp", "direct"):
            if meth == plan.method:
                continue
            try:
                q = asx.plan(w.n, w.density, m=w.m, dtype=w.dtype, method=meth, real_input=w.real,
                             device=dev.index)
            except Exception:
                continue
            if meth == "direct" and w.n * w.m * nloc > 2e12:
                continue
            q.execute(x, out=out)
            torch.cuda.synchronize()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, min(args.steps, 10))
            s_.record(stream)
            for _ in range(reps):
                q.execute(x, out=out)
            e_.record(stream)
            torch.cuda.synchronize()
            alt[meth] = {"ms_per_step": s_.elapsed_time(e_) / reps, "fft_size": q.fft_size}
        plan.execute(x, out=out)  # leave the production result in `out`
        torch.cuda.synchronize()

    # e2e through the C ABI with host buffers (H2D + transform + D2H inside)
    e2e = None
    if not args.no_e2e:
        hx = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        hx.copy_(x)
        hX = torch.empty((nloc, w.m), dtype=out.dtype, pin_memory=True)
        hxn, hXn = hx.numpy(), hX.numpy()
        plan.execute_host(hxn, out=hXn)  # warm-up (allocates the staging ring)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.execute_host(hxn, out=hXn)
        el = time.perf_counter() - t0
        barrier()
        e2e_s = max_over_ranks(el, device=dev) / args.e2e_steps
        elem_in = x.element_size()
        e2e = {"value": total * w.m / e2e_s, "unit": "complex points/s",
               "h2d_bytes_per_step": nloc * w.n * elem_in, "d2h_bytes_per_step": nloc * w.m * out.element_size(),
               "ms_per_step": e2e_s * 1e3, "path": "asx_execute_host (C ABI, pinned host buffers)"}
        # cross-check the host-path result against the device-path result (untimed)
        same = torch.equal(hX.to(dev), out)
        e2e["matches_device_path"] = bool(same)
        # e2e roofline: both directions of the PCIe link at once (the ring overlaps them)
        h2d_gbs, d2h_gbs = pcie_duplex(dev)
        bound_s = max(e2e["h2d_bytes_per_step"] / (h2d_gbs * 1e9), e2e["d2h_bytes_per_step"] / (d2h_gbs * 1e9))
        e2e["roofline"] = {"bound": "pcie", "h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs,
                           "how": "concurrent pinned 512 MiB copies on two streams from one start event, best of 5",
                           "bound_ms": bound_s * 1e3, "frac": bound_s / e2e_s}

    # parity of the whole shard vs the complex128 GPU path (untimed), MAX over ranks
    parity = None
    if not args.no_parity:
        parity = shard_parity(asx, w, x, out, dev)
        parity["max_rel_err"] = max_over_ranks(parity["max_rel_err"], device=dev)
        parity["signals_checked"] = int(sum_over_ranks(parity["signals_checked"], device=dev))
        parity["pass"] = parity["max_rel_err"] <= parity["tolerance"]

    # side measurements (world 1 only, not part of `value`): the other BASELINE
    # configs -- 1a (the α-FFT recursion itself, the one config whose op count
    # lets it approach the HBM roofline), 1b, 3 and the two
    # single-signal configs 0 and 2, so one line covers all five
    other = {}
    if world == 1 and not args.no_other_configs:
        for key in ("1a", "1b", "3", "0", "2"):
            if key != args.config:
                other[key] = side_config(key, dev, stream, peak)
                if key in ("0", "2"):  # single signals: launch latency, not throughput; config 0 sits in L2
                    other[key]["note"] = "single signal (replicas only): device time per transform, launch-latency bound"

    # untimed verification collective: per-rank checksums gathered over NCCL
    checks = gather_checksums(out, device=dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(args.config, min(args.cpu_seconds, 4.0))

    if rank == 0:
        dtype_arith = "f32" if w.dtype == "complex64" else "f64"
        line = {
            "metric": "alpha-FFT complex output points/sec",
            "value": value,
            "unit": "complex points/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": dtype_arith,
            "data": "synthetic (BASELINE config tones+noise, numpy PCG64 per-signal seeds, tones synthesised on GPU)",
            "config": workload_config(w, total, world, flush is None),
            "impl_detail": {"method": plan.method, "fft_size": plan.fft_size, "kernel": kernel_name,
                            "shard": f"contiguous {nloc} signals/rank (rank 0)",
                            "collectives": f"{args.dist_backend if world > 1 else 'none'}; none in the timed region"},
            "parity": parity,
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": profiled_traffic(args.config, plan.method),
                "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)" if peak_kind == "measured"
                else "fallback 6650 GB/s (B200_PROFILING.md)",
                "bytes_alg_per_launch": bytes_step,
                "flops_alg_per_launch": flops, "achieved_alg_tflops": flops / avg_launch_s / 1e12,
                "kernel": kernel_name,
                # the FP-side roofline of the same launches (configs 1b-4 are FP-bound)
                "compute": {"pipe": "fp32" if w.dtype == "complex64" else "fp64",
                            "achieved_tflops": flops / avg_launch_s / 1e12, "peak_tflops": fpk,
                            "frac": flops / avg_launch_s / 1e12 / fpk, "peak_source": fpk_src,
                            "flops": "8*M*N per signal (direct form: alpha has no dyadic alpha-FFT count)"
                            if (w.n * w.alpha.denominator) % w.alpha.numerator
                            else "reference alpha-FFT op count 6*mults+2*adds per signal (fastpath.py:113-127): "
                                 "an op-count credit, not what the kernel executes",
                            "executed": executed_flops(w, plan, nloc, avg_launch_s, fpk)},
            },
            "other_methods": alt,
            "other_configs": other,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * int(plan.info.kernels_per_execute),
            "clocks": clocks.summary(),
            "checksums": checks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    """--impl reference: the reference's own CPU path on all host cores.

    Each step is one bounded sample of the workload (about --ref-step-seconds
    of wall time, all cores busy); W warm-up and K timed steps are run and
    their real count, sample size and per-step time are what the line reports.
    Under torchrun only rank 0 works; the other ranks exit at once."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2403_16665_b200.signals import WORKLOADS

    w = WORKLOADS[args.config]
    step_s = args.ref_step_seconds
    # keep the whole run (W + K steps) within ~4 minutes
    step_s = max(0.05, min(step_s, 240.0 / max(1, args.steps + args.warmup)))
    pool = RefPool(args.config, step_s)
    t_run = time.perf_counter()
    try:
        for _ in range(args.warmup):
            pool.step()
        times = [pool.step() for _ in range(args.steps)]
    finally:
        pool.close()
    run_s = time.perf_counter() - t_run
    ms_per_step = 1e3 * sum(times) / len(times)
    value = pool.sample * w.m / (ms_per_step / 1e3)
    cpu = pool.describe(ms_per_step / 1e3)
    cpu["value"] = value
    line = {
        "impl": "reference",
        "metric": "alpha-FFT complex output points/sec",
        "value": value,
        "unit": "complex points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (same generator and config as the GPU arm)",
        "config": workload_config(w, w.batch, world, True),
        "impl_detail": {"step": f"one bounded sample of {pool.sample} signals (not the whole batch of "
                                f"{w.batch}); value = sample * M / mean step time",
                        "api": pool.api, "kind": pool.kind, "wall_s_all_steps": run_s,
                        "min_step_ms": 1e3 * min(times), "max_step_ms": 1e3 * max(times)},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "complex points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    maybe_self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
