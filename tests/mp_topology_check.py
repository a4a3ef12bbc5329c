"""Multi-GPU worker for groups x dp x tp layouts,
launched by tests/test_multigpu_gpu.py under torchrun with 4 ranks.

  layout A: groups=2, dp_per_group=2, tp=1 -- intra-group gradient mean after
            lazy start (driver.py:372-393), outer mean over all 4 replicas
  layout B: groups=2, dp_per_group=1, tp=2 -- each rank holds a tensor shard
            (shard_offsets, topology.py:146-160); outer sync per shard over the
            groups (outer_participant_ranks, topology.py:81-92); the clip norm is
            global over each replica's two shards

Checks (rank 0 writes JSON): open loop vs the reference ENGINE's fixtures
(A: open_loop_T200_r10_g2_dp2, B: open_loop_T200_r10_g2 -- TP does not change the
arithmetic, test_driver.py:296-301) and closed inner+outer loops vs an oracle
replay, bitwise; plus the TP-global norm.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_17849_b200 as P  # noqa: E402
from oracle import pier_oracle as O  # noqa: E402


def gather_full(eng, vec_fn, topo, n_full):
    """Full-model vector from every rank's shard (TP) -- reporting only."""
    shard = vec_fn(eng).contiguous()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, shard.cpu().numpy())
    if topo.tp_size == 1:
        return parts[0]
    offs = P.shard_offsets(n_full, topo.tp_size)
    full = np.empty(n_full, np.float32)
    for t, (a, b) in enumerate(offs):
        full[a:b] = parts[topo.rank(0, 0, t)]
    return full


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    res = {}
    for name, topo in (("dp2", P.Topology(groups=2, dp_per_group=2, tp_size=1)),
                       ("tp2", P.Topology(groups=2, dp_per_group=1, tp_size=2))):
        g, d, tp = topo.coords(rank)
        # ---- open loop vs the reference engine
        f = np.load(os.path.join(ROOT, "tests", "golden",
                                 "open_loop_T200_r10_g2_dp2.npz" if name == "dp2" else "open_loop_T200_r10_g2.npz"))
        n_full = f["theta0"].shape[0]
        lo, hi = P.shard_offsets(n_full, topo.tp_size)[tp]
        sched = P.ScheduleConfig(total_iters=200, lazy_fraction=0.1, sync_interval=10)
        eng = P.PierEngine(hi - lo, sched, comm=comm, topology=topo, bucket_elems=64, model_params=n_full,
                           theta0=torch.from_numpy(f["theta0"][lo:hi].copy()).to(dev))
        k = 0
        for t in range(1, 201):
            if not eng.is_boundary(t):
                continue
            anchor = gather_full(eng, lambda e: e.snapshot(), topo, n_full)
            grp = 0 if t <= sched.lazy_end else g
            x = O.open_loop_inputs(0, k, grp, anchor)
            eng.theta[: hi - lo].copy_(torch.from_numpy(x[lo:hi]).to(dev))
            k += 1
            eng.boundary(t)
        th = gather_full(eng, lambda e: e.params(), topo, n_full)
        mo = gather_full(eng, lambda e: e.outer_momentum(), topo, n_full)
        res[f"{name}_open_loop"] = {
            "theta_bitwise": bool(np.array_equal(th.view(np.uint32), f["anchor"].view(np.uint32))),
            "mom_bitwise": bool(np.array_equal(mo.view(np.uint32), f["momentum"].view(np.uint32)))}
        del eng

        # ---- closed inner+outer loop vs an oracle replay (every replica on full vectors)
        n_full = 40_000
        lo, hi = P.shard_offsets(n_full, topo.tp_size)[tp]
        T = 60
        theta0 = (np.random.default_rng(3).standard_normal(n_full) * 0.02).astype(np.float32)
        osch = O.Sched(total_iters=T, lazy_fraction=0.5, sync_interval=10)
        evs = {e.t: e for e in O.boundary_events(osch, "pier")}
        R = topo.num_replicas
        rep = topo.replica_index(g, d)

        def grads_at(t, scale):
            return [(np.random.default_rng([t, q]).standard_normal(n_full) * scale).astype(np.float32)
                    for q in range(R)]

        for clipped in (False, True):
            scale = 0.05 if clipped else 1e-5     # |g| ~ 10 vs ~0.002: clip path on / off
            ths = [theta0.copy() for _ in range(R)]
            ms = [np.zeros(n_full, np.float32) for _ in range(R)]
            vs = [np.zeros(n_full, np.float32) for _ in range(R)]
            an, mom = theta0.copy(), np.zeros(n_full, np.float32)
            eng = P.PierEngine(hi - lo, P.ScheduleConfig(total_iters=T, lazy_fraction=0.5, sync_interval=10),
                               comm=comm, topology=topo, bucket_elems=1024, model_params=n_full,
                               theta0=torch.from_numpy(theta0[lo:hi].copy()).to(dev))
            norm_err = 0.0
            for t in range(1, T + 1):
                gs = grads_at(t, scale)
                eng.grad[: hi - lo].copy_(torch.from_numpy(gs[rep][lo:hi]).to(dev))
                eng.step(t)
                # oracle: driver.py:372-399 per replica, then the boundary
                if t <= osch.lazy_end:
                    mean = O.mean_left_fold(gs)
                    gs = [mean] * R
                elif topo.dp_per_group > 1:
                    for gg in range(topo.groups):
                        idx = [topo.replica_index(gg, dd) for dd in range(topo.dp_per_group)]
                        mean = O.mean_left_fold([gs[i] for i in idx])
                        for i in idx:
                            gs[i] = mean
                clip = eng.last_clip()
                exact = float(np.dot(gs[rep].astype(np.float64), gs[rep].astype(np.float64)))
                norm_err = max(norm_err, abs(clip.sqnorm - exact) / exact)
                for q in range(R):
                    gq = gs[q]
                    if clipped:  # the same global-norm formula as the kernel (fp64 sum -> fp32 sqrt)
                        nrm = float(np.sqrt(np.float32(np.dot(gq.astype(np.float64), gq.astype(np.float64)))))
                        gq = gq * np.float32(1.0 / nrm) if nrm > 1.0 else gq
                    ths[q], ms[q], vs[q], _ = O.adamw(ths[q], gq, ms[q], vs[q], t - 1, O.inner_lr(t, osch))
                e = evs.get(t)
                if e is not None and e.kind == "fold":
                    mom, an = O.warmup_fold(ths[0], an, mom, e.mu)
                elif e is not None:
                    new, mom = O.outer_anchor_form(O.mean_left_fold(ths), an, mom, e.lr, e.mu)
                    an = new.copy()
                    ths = [new.copy() for _ in range(R)]
            got = gather_full(eng, lambda e: e.params(), topo, n_full)
            gm = gather_full(eng, lambda e: e.outer_momentum(), topo, n_full)
            # (the oracle's clip scale from the fp64 full-vector sum can differ from the
            # kernel's shard-wise fp64 sum in the last fp64 bit: compare with a tolerance
            # when the clip is active, bitwise otherwise)
            res[f"{name}_closed_{'clip' if clipped else 'noclip'}"] = {
                "theta_bitwise": bool(np.array_equal(got.view(np.uint32), ths[0].view(np.uint32))),
                "mom_bitwise": bool(np.array_equal(gm.view(np.uint32), mom.view(np.uint32))),
                "theta_maxrel": float(np.max(np.abs(got - ths[0])) / np.max(np.abs(ths[0]))),
                "mom_maxrel": float(np.max(np.abs(gm - mom)) / max(np.max(np.abs(mom)), 1e-30)),
                "sqnorm_relerr": norm_err, "clipped_last": bool(clip.clipped),
                "inner_events": eng.commstats.inner_events}
            del eng
    torch.cuda.synchronize()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
