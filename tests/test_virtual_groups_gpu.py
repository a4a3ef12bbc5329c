"""Every multi-rank path of the engine on ONE GPU.

A ``VirtualGroup`` runs n Pier ranks on one device, one host thread per rank,
through the same ``PierEngine`` / ``GroupComm`` calls and the same kernels as
the one-process-per-GPU build: the P2P exchanges read and write the other
ranks' buffers, the persistent round is ONE cooperative launch over all ranks
(k_round_multi), and the collectives' ordering barriers are host rendezvous
with CUDA events.  So the driver's single-GPU ``pytest -m gpu`` checks, bitwise
against the reference (golden open-loop fixtures of the reference ENGINE) and
the oracle:

* n = 2, 3, 4, 8 groups: open loop (resident + offload), closed inner+outer
  loops (persistent round, two-stream round, unfused), lazy-phase prefix ==
  AdamW baseline, replica agreement, the bf16 7B recipe (config 5 at 8 groups
  with offload) vs an oracle replay, step_host, the f32 / fused-norm / bf16
  lazy-phase gradient means (driver.py:372-443, topology.py:104-122);
* groups x dp x tp layouts 2x2x1, 2x1x2 and 2x2x2 (topology.py:31-92,
  driver.py:372-378, test_driver.py:296-301);
* failure propagation: a failing rank aborts the others' collectives
  (driver.py:494-501);
* the round kernel's timeout record (a rank that never arrives).
"""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT
from group_checks import assert_outer, assert_topology, outer_checks, topology_checks

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2511_17849_b200")


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _keep(name, res):
    keep = os.environ.get("PIER_TEST_OUT")
    if keep:
        os.makedirs(keep, exist_ok=True)
        with open(os.path.join(keep, name), "w") as fh:
            json.dump(res, fh)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_virtual_group_engine_bitwise(n):
    with P.VirtualGroup(n) as vg:
        res = vg.run(outer_checks, 1024)
    _keep(f"virtual_outer_n{n}.json", res[0])
    for r in res:                       # every rank's view of the same run
        assert_outer(r)
    assert "open_loop_p2p_offload" in res[0] and "bf16_vs_oracle" in res[0] and "grad_mean_p2p_bf16" in res[0]


def test_virtual_group_small_spans():
    """64-element slices: hundreds of spans per round through the signal counters."""
    with P.VirtualGroup(4) as vg:
        res = vg.run(outer_checks, 64, ("open_loop", "closed", "agree"))
    for r in res:
        assert_outer(r)


@pytest.mark.parametrize("names,n", [(("dp2", "tp2"), 4), (("dp2tp2",), 8)], ids=["2x2x1+2x1x2", "2x2x2"])
def test_virtual_group_layouts(names, n):
    with P.VirtualGroup(n) as vg:
        res = vg.run(topology_checks, names)
    _keep(f"virtual_topology_n{n}.json", res[0])
    for r in res:
        assert_topology(r, names)


def test_virtual_group_failure_aborts_collectives():
    """A rank that raises aborts the group: the ranks blocked in a collective get
    GroupAborted and run() re-raises the failing rank's exception (driver.py:494-501)."""
    from paper_2511_17849_b200._lib import GroupAborted

    seen = {}

    def fn(comm):
        eng = P.PierEngine(4099, P.ScheduleConfig(total_iters=60, lazy_fraction=0.5, sync_interval=10),
                           comm=comm, bucket_elems=1024)
        if comm.rank == 1:
            raise ValueError("rank 1 failed")
        try:
            for t in range(1, 3):
                eng.step(t)              # lazy phase: a gradient mean every iteration
            torch.cuda.synchronize()
        except GroupAborted as exc:
            seen[comm.rank] = str(exc)
            raise

    vg = P.VirtualGroup(3)
    with pytest.raises(ValueError, match="rank 1 failed"):
        vg.run(fn)
    assert set(seen) == {0, 2}, seen


def test_round_timeout_is_recorded(tmp_path):
    """A rank that never releases its span: the round's waits time out after
    PIER_ROUND_TIMEOUT_S, record which rank / counter / target in the host-mapped
    slot and trap; pier_last_error of the next failing call names them.  Runs in
    a subprocess (the trap ends that process's CUDA context)."""
    script = tmp_path / "timeout.py"
    script.write_text(f"""
import ctypes as C, json, os, sys
sys.path.insert(0, {ROOT!r})
import torch
import paper_2511_17849_b200 as P
from paper_2511_17849_b200._lib import lib, last_error
n, n_pad, B = 2, 4096, 512
f = lambda: torch.zeros(n_pad, device="cuda")
th, g, m, v = [f() for _ in range(n)], [f() for _ in range(n)], [f() for _ in range(n)], [f() for _ in range(n)]
an, mo = [f()[: n_pad // n] for _ in range(n)], [f()[: n_pad // n] for _ in range(n)]
sig = [torch.zeros(lib.pier_round_sig_bytes() // 4, dtype=torch.int32, device="cuda") for _ in range(n)]
sig[1][4096 + 64] = 1000   # rank 1 believes span 0 was released 1000 times before: a target nobody reaches
ws = [P.norm_workspace() for _ in range(n)]
hp = P.AdamWConfig().hyper(1e-3, 1)
ptrs = lambda ts: (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
torch.cuda.synchronize()
rc = lib.pier_round_virtual_f32(n, ptrs(th), ptrs(g), ptrs(m), ptrs(v), ptrs(an), ptrs(mo), ptrs(sig), n_pad, B,
                                C.byref(hp), ptrs(ws), 1.1, 0.9, 4, 2, (C.c_void_p * n)(0, 0))
rc2 = lib.pier_device_sync()
print(json.dumps({{"launch_rc": rc, "sync_rc": rc2, "error": last_error()}}))
""")
    env = dict(os.environ, PIER_ROUND_TIMEOUT_S="0.5")
    out = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300, env=env)
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert line, out.stdout + out.stderr
    res = json.loads(line[-1])
    assert res["launch_rc"] == 0 and res["sync_rc"] != 0, res
    assert "round wait timed out" in res["error"] and "target" in res["error"], res
