"""bench.py contract checks that need no GPU: the reference arm (the
unmodified reference package from baseline/_ref, or the oracle port when it
is absent) prints one JSON line whose steps / sample / time agree, with the
same config dict the GPU arm prints; a torchrun world that disagrees with
--gpus is refused."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=REPO)


def test_reference_arm_line_is_consistent():
    r = _bench("--impl", "reference", "--config", "1a", "--steps", "2", "--warmup", "1", "--ref-step-seconds", "0.3")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["config"]["workload"].startswith("config 1a:")
    assert set(line["config"]) == {"workload", "batch", "n", "m", "alpha", "dtype", "parallelism", "l2"}
    # the line's value is its own sample over its own step time
    sample = int(line["impl_detail"]["step"].split("sample of ")[1].split()[0])
    assert abs(line["value"] - sample * 4096 / (line["ms_per_step"] / 1e3)) <= 1e-6 * line["value"]
    # every step really ran: K steps of ms_per_step fit inside the measured wall time
    assert line["steps"] * line["ms_per_step"] / 1e3 <= line["impl_detail"]["wall_s_all_steps"]
    kind = line["cpu_baseline"]["kind"]
    if os.path.isdir(os.path.join(REPO, "baseline", "_ref", "alpha_spectra")):
        assert kind == "reference" and "transform_samples" in line["impl_detail"]["api"]
    else:
        assert kind == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_must_match_gpus():
    r = _bench("--gpus", "4", "--steps", "1", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr
