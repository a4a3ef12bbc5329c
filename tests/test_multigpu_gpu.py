"""Multi-GPU (NCCL, one group per GPU) parity: runs tests/mp_outer_check.py
under torchrun on every visible GPU pair/quad (skipped with < 2 GPUs)."""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

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
    for name in ("dp2", "tp2"):
        assert res[f"{name}_open_loop"]["theta_bitwise"] and res[f"{name}_open_loop"]["mom_bitwise"], res
        r = res[f"{name}_closed_noclip"]
        assert r["theta_bitwise"] and r["mom_bitwise"], (name, r)
        r = res[f"{name}_closed_clip"]
        assert r["clipped_last"] and r["sqnorm_relerr"] < 1e-12, (name, r)
        assert r["theta_maxrel"] <= 1e-5 and r["mom_maxrel"] <= 1e-5, (name, r)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("bucket", [64, 1024])
def test_nccl_outer_step_open_loop(world, bucket, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    res = _run(world, bucket, tmp_path)
    for tag in ("p2p_resident", "p2p_offload", "nccl_resident", "nccl_offload", "nvls_resident"):
        key = f"open_loop_{tag}"
        if key not in res:
            continue  # no golden for this group count
        r = res[key]
        kinds = [k for _, k, _, _ in r["records"]]
        assert kinds.count("fold") == 2 and kinds.count("outer") == 18
        if world == 2 or tag.startswith("p2p"):
            # the fused kernel folds ranks in ascending order: bitwise at every n
            assert r["theta_bitwise"] and r["mom_bitwise"], (tag, r)
        # params within the north_star fp32 tolerance (max-rel and l2-rel <= 1e-5)
        assert r["theta_rel"][0] <= 1e-5 and r["theta_rel"][1] <= 1e-5, (tag, r)
        # the NCCL ring sums theta in ring order; after 18 open-loop rounds the
        # momentum (a sum of small deltas) drifts further (measured 7.2e-5 max-rel
        # at n=4) -- the reason the fused p2p path (bitwise) is the default
        mom_tol = 1e-5 if tag.startswith("p2p") or world == 2 else 2e-4
        assert r["mom_rel"][0] <= mom_tol and r["mom_rel"][1] <= mom_tol / 2, (tag, r)
    for tag in ("p2p_fused_persistent", "p2p_fused_streams", "p2p_unfused", "nccl_unfused",
                "nvls_fused",
                "nvls_unfused"):
        r = res[f"closed_{tag}"]
        assert not r["clipped"]
        if tag.startswith("p2p") or world == 2:
            assert r["theta_bitwise"] and r["mom_bitwise"], (tag, r)
        assert r["theta_rel"][0] <= 1e-5 and r["mom_rel"][0] <= 2e-4, (tag, r)
    assert all(res["step_host"].values()), res["step_host"]
    r = res["replicas_agree_after_outer"]          # test_driver.py:249-258
    assert r["all"] and r["boundaries"] == 3, r
    if world == 2:                                  # test_driver.py:229-241
        assert res["two_groups_identical_data_params_bitwise"]
    r = res["lazy_prefix_equals_adamw_baseline"]   # acceptance criterion 2, test_driver.py:165-172
    assert r["all_bitwise"] and r["iterations"] == 30 and r["folds"] == 3, r
    r = res["bf16_round_fused_vs_unfused"]   # 7B recipe: fused bf16-gradient round == unfused path
    assert r["bitwise"] and r["offload_bitwise"] and r["records_equal"], r
    assert r["outer_steps"] == 3 and r["clipped_steps"] > 0, r
    if world == 2:  # BASELINE config 1 closed loop on the real 2-GPU engine
        for tag in ("fused", "unfused"):
            r = res[f"tiny_gpt_{tag}"]
            assert r["train_loss_max_abs_diff"] <= 1e-4, r
            assert r["folds"] == 2 and r["outer"] == list(range(24, 161, 8))
    assert res["grad_mean"]["rel"][0] <= 1e-6
    if world == 2:
        assert res["grad_mean"]["bitwise"]
    assert res["grad_mean_p2p"]["bitwise"], res["grad_mean_p2p"]
    r = res["grad_mean_norm_p2p"]   # lazy phase: mean + clip norm in one pass
    assert r["bitwise"] and r["same_on_all_ranks"] and r["sqnorm_relerr"] < 1e-12 and r["clipped"], r
    assert r["scale_equals_k4a"], r
