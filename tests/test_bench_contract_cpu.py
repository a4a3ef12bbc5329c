"""bench.py JSON contract: the reference arm (CPU only: the oracle port on the host
threads; rank != 0 under torchrun prints nothing) and, on a GPU, our own arm."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-sample", "65536"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, check=True)
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["unit"] == "params/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert "workload" in d["config"] and "model" not in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # measured, not extrapolated: the claimed timed work fits inside the run
    assert d["ms_per_step"] * d["steps"] / 1e3 <= cb["wall_s"] + 1e-6
    assert abs(d["value"] - d["config"]["groups"] * 65536 / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    assert cb["single_thread"]["cores"] == 1 and cb["single_thread"]["value"] > 0
    # the same config object our arm prints (bench.workload_config)
    assert {"params", "params_padded", "groups", "bucket_elems", "reduce", "schedule", "l2"} <= set(d["config"])


def test_reference_arm_groups_follow_gpus():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--steps", "1", "--warmup", "3", "--ref-sample", "65536"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT, check=True)
    d = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][0])
    assert d["n_gpus"] == 4 and d["config"]["groups"] == 4 and d["config"]["reduce"] == "p2p"


def test_gpus_n_without_a_launcher_starts_n_ranks():
    """`python bench.py --gpus 2` re-execs under torch.distributed.run with 2 ranks on
    127.0.0.1 (the launcher path of the scaling run, exercised without a GPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr
    rows = sorted((json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")), key=lambda d: d["rank"])
    assert [(d["rank"], d["world"], d["master"]) for d in rows] == [(0, 2, "127.0.0.1"), (1, 2, "127.0.0.1")]


def test_our_arm_refuses_a_world_size_mismatch():
    """`--gpus N` under a launcher with another WORLD_SIZE fails loudly (no silent 1-GPU line)."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr, out.stderr
    assert not [x for x in out.stdout.splitlines() if x.startswith("{")]


OURS_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
             "outer_step", "step_roofline"}


@pytest.mark.gpu
def test_our_arm_json_contract():
    """bench.py's own arm on one GPU (GPT-2 small, short): the driver's keys,
    roofline and cpu_baseline objects, e2e through the host-buffer API."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--steps", "3",
                          "--warmup", "3", "--breakdown-steps", "1", "--cpu-sample", "1048576", "--cpu-reps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, check=True)
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert OURS_KEYS <= set(d), OURS_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["higher_is_better"] is True and d["scaling"] == "weak" and d["value"] > 0
    assert d["gpu_launches"] == 2 * d["steps"]                  # K4a + K5 per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.3 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] == 1 and cb["value"] > 0
    assert d["clocks"]["samples"] >= 0 and "workload" in d["config"]
