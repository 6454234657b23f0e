"""bench.py on the GPU: the multi-rank path a plain `bench.py --gpus N` takes
(self-launch under torch.distributed.run), here with 2 ranks sharing the one
GPU of the test box and gloo for the collectives (NCCL refuses two ranks on
one device).  Every rank transforms its own shard; the line must report the
world size, the whole batch, and the parity of ALL signals of both shards
against the complex128 GPU path."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


QUICK = ("--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-other-configs", "--no-alt")


def test_two_ranks_self_launch_and_parity():
    line = _run("--gpus", "2", "--batch", "256", "--dist-backend", "gloo", *QUICK)
    assert line["n_gpus"] == 2
    assert line["config"]["batch"] == 256 and line["config"]["parallelism"].startswith("dp2")
    par = line["parity"]
    assert par["signals_checked"] == 256
    assert par["pass"] and par["max_rel_err"] <= 2e-5
    assert line["gpu_launches"] == 3
    assert len(line["checksums"]) == 2


def test_single_rank_line_has_parity_and_executed_flops():
    line = _run("--batch", "512", *QUICK)
    assert line["n_gpus"] == 1
    assert line["parity"]["signals_checked"] == 512 and line["parity"]["pass"]
    ex = line["roofline"]["compute"]["executed"]
    assert 0 < ex["frac"] < 1.5
