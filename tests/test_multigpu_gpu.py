"""Multi-GPU (NCCL, one group per GPU) parity: runs tests/mp_outer_check.py
under torchrun on every visible GPU pair/quad (skipped with < 2 GPUs).  The
same checks run on one GPU through VirtualGroups in test_virtual_groups_gpu.py."""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT
from group_checks import assert_outer, assert_topology

pytestmark = pytest.mark.gpu


def _run(world: int, bucket: int, tmp_path):
    out = tmp_path / f"mp_{world}_{bucket}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + bucket % 97),
           os.path.join(ROOT, "tests", "mp_outer_check.py"), str(out), str(bucket)]
    subprocess.run(cmd, check=True, timeout=600, cwd=ROOT)
    keep = os.environ.get("PIER_TEST_OUT")  # optional: keep the per-run parity numbers
    if keep:
        os.makedirs(keep, exist_ok=True)
        (open(os.path.join(keep, out.name), "w")).write(out.read_text())
    return json.loads(out.read_text())


def test_dp_and_tp_layouts(tmp_path):
    """groups x dp x tp: 2x2x1 and 2x1x2 on 4 GPUs."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    out = tmp_path / "topo.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", "29577",
           os.path.join(ROOT, "tests", "mp_topology_check.py"), str(out)]
    subprocess.run(cmd, check=True, timeout=900, cwd=ROOT)
    res = json.loads(out.read_text())
    keep = os.environ.get("PIER_TEST_OUT")
    if keep:
        os.makedirs(keep, exist_ok=True)
        open(os.path.join(keep, "topo.json"), "w").write(out.read_text())
    assert_topology(res, ("dp2", "tp2"))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("bucket", [64, 1024])
def test_nccl_outer_step_open_loop(world, bucket, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    res = _run(world, bucket, tmp_path)
    assert_outer(res)
