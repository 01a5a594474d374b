"""The bench.py JSON contract the driver reads (one line, fixed keys)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    """--impl reference: the reference algorithm (oracle/, CPU) on a bounded sample."""
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert d["config"]["workload"].startswith("cfg1")


@pytest.mark.gpu
def test_our_arm_contract(cuda):
    d = _run(["--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-extras"], 900)
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]


def test_gpus_flag_spawns_ranks():
    """--gpus N without torchrun launches N ranks (torch.distributed.run on
    127.0.0.1); the launcher hook checks the rendezvous and the max-over-ranks
    reduction on gloo (no GPU needed)."""
    d = _run(["--gpus", "2", "--launcher-dry-run"], 600)
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2 and d["max_over_ranks"] == 2.0


def test_gpus_flag_fails_loudly_without_gpus():
    """Asking for more GPUs than are visible is an error, not a silent 1-GPU run."""
    import torch

    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(max(n, 2)),
                          "--config", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode != 0 and "visible" in out.stdout
