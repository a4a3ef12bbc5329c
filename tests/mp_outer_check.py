"""Multi-GPU parity worker (launched by tests/test_multigpu_gpu.py under torchrun):
one Pier group per GPU, NCCL outer step through PierEngine.

Checks, on every rank, written as JSON by rank 0:
  1. open loop, T=200 r=10, groups = world: the engine driven through the
     whole schedule reproduces the reference ENGINE's final anchor and outer
     momentum (golden open_loop_T200_r10_g{world}.npz): bitwise at 2 ranks
     (a two-term sum is order-free), <= 1e-5 max-rel otherwise (NCCL order);
  2. lazy-phase gradient mean (NCCL avg) vs the reference left fold.
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


def rel(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)), \
        float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30))


def main():
    out_path = sys.argv[1]
    bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world)
    res = {"world": world, "bucket": bucket}

    gold = os.path.join(ROOT, "tests", "golden", f"open_loop_T200_r10_g{world}.npz")
    if os.path.exists(gold):
        f = np.load(gold)
        n = f["theta0"].shape[0]
        sched = P.ScheduleConfig(total_iters=200, lazy_fraction=0.1, sync_interval=10)
        for reduce, offload in (("p2p", False), ("p2p", True), ("nccl", False), ("nccl", True), ("nvls", False)):
            eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(f["theta0"]).to(dev),
                               bucket_elems=bucket, offload=offload, reduce=reduce)
            k = 0
            for t in range(1, 201):
                if not eng.is_boundary(t):
                    continue
                anchor = eng.snapshot().cpu().numpy()
                lazy = t <= sched.lazy_end
                g = 0 if lazy else rank  # lazy phase: replicas identical (driver.py:412)
                eng.theta[:n].copy_(torch.from_numpy(O.open_loop_inputs(0, k, g, anchor)).to(dev))
                k += 1
                eng.boundary(t)
            th = eng.params().cpu().numpy()
            mo = eng.outer_momentum().cpu().numpy()
            tag = f"{reduce}_{'offload' if offload else 'resident'}"
            res[f"open_loop_{tag}"] = {
                "theta_bitwise": bool(np.array_equal(th.view(np.uint32), f["anchor"].view(np.uint32))),
                "mom_bitwise": bool(np.array_equal(mo.view(np.uint32), f["momentum"].view(np.uint32))),
                "theta_rel": rel(th, f["anchor"]), "mom_rel": rel(mo, f["momentum"]),
                "records": [(r.iteration, r.kind, r.mu, r.outer_lr) for r in eng.records],
                "counters": eng.host.counters(),
            }

    # closed inner+outer loop (T=60, r=10, lazy 0.5): lazy-phase gradient mean,
    # folds at 10..30, outer steps at 40..60; fused and unfused engine steps vs
    # an oracle replay of every group (no clipping: |g| << 1, so bitwise)
    n = 4099
    T = 60
    theta0 = (np.random.default_rng(9).standard_normal(n) * 0.02).astype(np.float32)
    osch = O.Sched(total_iters=T, lazy_fraction=0.5, sync_interval=10)
    evs = {e.t: e for e in O.boundary_events(osch, "pier")}

    def grads_at(t):
        return [(np.random.default_rng([t, g]).standard_normal(n) * 1e-5).astype(np.float32) for g in range(world)]

    ths = [theta0.copy() for _ in range(world)]
    ms = [np.zeros(n, np.float32) for _ in range(world)]
    vs = [np.zeros(n, np.float32) for _ in range(world)]
    anchor, mom = theta0.copy(), np.zeros(n, np.float32)
    for t in range(1, T + 1):
        gs = grads_at(t)
        if t <= osch.lazy_end:
            gm = O.mean_left_fold(gs)
            gs = [gm] * world
        for g in range(world):
            ths[g], ms[g], vs[g], _ = O.adamw(ths[g], gs[g], ms[g], vs[g], t - 1, O.inner_lr(t, osch))
        e = evs.get(t)
        if e is not None and e.kind == "fold":
            mom, anchor = O.warmup_fold(ths[0], anchor, mom, e.mu)
        elif e is not None:
            new, mom = O.outer_anchor_form(O.mean_left_fold(ths), anchor, mom, e.lr, e.mu)
            anchor = new.copy()
            ths = [new.copy() for _ in range(world)]
    sched = P.ScheduleConfig(total_iters=T, lazy_fraction=0.5, sync_interval=10)
    for reduce, fuse, impl in (("p2p", True, "persistent"), ("p2p", True, "streams"),
                               ("p2p", False, ""),
                               ("nccl", False, ""), ("nvls", True, ""), ("nvls", False, "")):
        eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket,
                           reduce=reduce)
        if impl:
            eng.round_impl = impl
        for t in range(1, T + 1):
            eng.grad[:n].copy_(torch.from_numpy(grads_at(t)[rank]).to(dev))
            eng.step(t, fuse=fuse)
        got = eng.params().cpu().numpy()
        gm = eng.outer_momentum().cpu().numpy()
        res[f"closed_{reduce}_{'fused' if fuse else 'unfused'}{'_' + impl if impl else ''}"] = {
            "theta_bitwise": bool(np.array_equal(got.view(np.uint32), ths[rank].view(np.uint32))),
            "mom_bitwise": bool(np.array_equal(gm.view(np.uint32), mom.view(np.uint32))),
            "theta_rel": rel(got, ths[rank]), "mom_rel": rel(gm, mom),
            "clipped": bool(eng.last_clip().clipped)}
        del eng

    # acceptance criterion 2 (test_driver.py:165-172): through the lazy phase the
    # Pier run's params equal the synchronous AdamW baseline's bitwise at every
    # iteration (warmup folds touch only the anchor and momentum)
    lazy_eq = []
    engs = {m: P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket,
                            mode=m) for m in ("pier", "adamw_baseline")}
    for t in range(1, sched.lazy_end + 1):
        g = torch.from_numpy(grads_at(t)[rank]).to(dev)
        for e in engs.values():
            e.grad[:n].copy_(g)
            e.step(t)
        lazy_eq.append(torch.equal(engs["pier"].params(), engs["adamw_baseline"].params()))
    res["lazy_prefix_equals_adamw_baseline"] = {"all_bitwise": all(lazy_eq), "iterations": len(lazy_eq),
                                                "folds": engs["pier"].warmup_folds}
    del engs

    # test_driver.py:249-258: every replica holds the same params after every outer
    # boundary (different gradients per group); test_driver.py:229-241: two groups
    # on identical data match one group bitwise ((x + x) / 2 == x exactly)
    eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket)
    agree = []
    for t in range(1, T + 1):
        eng.grad[:n].copy_(torch.from_numpy(grads_at(t)[rank]).to(dev))
        rec = eng.step(t)
        if rec is not None and rec.kind == "outer":
            mine = eng.params().contiguous()
            allp = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allp, mine)
            agree.append(all(torch.equal(allp[0], x) for x in allp[1:]))
    res["replicas_agree_after_outer"] = {"all": all(agree), "boundaries": len(agree)}
    del eng
    if world == 2:
        two = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket)
        one = P.PierEngine(n, sched, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket)
        for t in range(1, T + 1):
            g = torch.from_numpy(grads_at(t)[0]).to(dev)     # the same data on both groups
            for e in (two, one):
                e.grad[:n].copy_(g)
                e.step(t)
        res["two_groups_identical_data_params_bitwise"] = bool(torch.equal(two.params(), one.params()))
        del two, one

    # 7B recipe (bf16 live params and grads, fp32 master/m/v/anchor/momentum): the
    # fused persistent round with bf16 gradients (pier_round_fused_bf16_f32 + the
    # bf16 refresh) == the unfused path (AdamW-bf16, P2P outer step, cast), bitwise,
    # with the clip active (grads x 1e4: |g| ~ 6)
    bres = {}
    for fuse, offload in ((True, False), (False, False), (True, True)):
        eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket,
                           bf16_params=True, offload=offload)
        clips = []
        for t in range(1, T + 1):
            eng.grad[:n].copy_(torch.from_numpy(grads_at(t)[rank] * np.float32(1e4)).to(dev).to(torch.bfloat16))
            eng.step(t, fuse=fuse)
            clips.append(bool(eng.last_clip().clipped))
        bres[(fuse, offload)] = ([eng.theta[:n].cpu(), eng.theta_bf16[:n].cpu(), eng.m[:n].cpu(),
                                  eng.v[:n].cpu(), eng.outer_momentum().cpu(), eng.snapshot().cpu()],
                                 [(r.iteration, r.kind) for r in eng.records], clips)
        del eng
    fz, un, fo = bres[(True, False)], bres[(False, False)], bres[(True, True)]
    res["bf16_round_fused_vs_unfused"] = {
        "bitwise": all(torch.equal(a, b) for a, b in zip(fz[0], un[0])),
        "offload_bitwise": all(torch.equal(a, b) for a, b in zip(fo[0], un[0])),
        "records_equal": fz[1] == un[1] == fo[1],
        "outer_steps": sum(1 for _, k in fz[1] if k == "outer"),
        "clipped_steps": sum(fz[2])}

    # host-buffer call (e2e path) == device-resident steps, bitwise, several groups
    dev_eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket)
    host_eng = P.PierEngine(n, sched, comm=comm, theta0=torch.from_numpy(theta0).to(dev), bucket_elems=bucket)
    host_eng.host_chunk = 1024
    vs = host_eng._valid_shard()
    pin = dict(dtype=torch.float32, pin_memory=True)
    hs = {"theta": torch.from_numpy(theta0.copy()).pin_memory(), "grad": torch.empty(n, **pin),
          "m": torch.zeros(n, **pin), "v": torch.zeros(n, **pin), "anchor": torch.empty(vs, **pin),
          "mom": torch.zeros(vs, **pin)}
    hs["anchor"].copy_(host_eng.anchor[:vs])
    for t in range(1, T + 1):
        g = torch.from_numpy(grads_at(t)[rank])
        dev_eng.grad[:n].copy_(g.to(dev))
        dev_eng.step(t)
        hs["grad"].copy_(g)
        host_eng.step_host(t, hs)
    res["step_host"] = {
        "theta_bitwise": bool(torch.equal(hs["theta"], dev_eng.params().cpu())),
        "mv_bitwise": bool(torch.equal(hs["m"], dev_eng.m[:n].cpu()) and torch.equal(hs["v"], dev_eng.v[:n].cpu())),
        "shard_bitwise": bool(torch.equal(hs["mom"], dev_eng.mom[:vs].cpu())
                              and torch.equal(hs["anchor"], dev_eng.anchor[:vs].cpu()))}
    del dev_eng, host_eng

    # BASELINE config 1 on the real multi-GPU engine: tiny GPT, 2 groups (one per
    # GPU), r=8, T=160, closed loop; loss curve vs the reference within 1e-4
    if world == 2:
        from paper_2511_17849_b200 import tinygpt as TG

        torch.backends.cuda.matmul.allow_tf32 = False
        tg = np.load(os.path.join(ROOT, "tests", "golden", "tiny_gpt.npz"))
        cfg = dict(vocab=256, d=128, heads=4, layers=2, seq=64)
        sched = P.ScheduleConfig(total_iters=160, sync_interval=8, lazy_fraction=0.1)
        for fuse in (True, False):
            eng = P.PierEngine(tg["theta0"].shape[0], sched, comm=comm,
                               theta0=torch.from_numpy(tg["theta0"]).to(dev), bucket_elems=bucket)
            batches = torch.from_numpy(tg["batches"].astype(np.int64)).to(dev)
            per = batches.shape[1] // world
            curve = []
            nparam = tg["theta0"].shape[0]
            for t in range(1, 161):
                loss = TG.loss_and_grad(eng.params(), batches[t - 1, rank * per:(rank + 1) * per], cfg,
                                        eng.grad[:nparam])
                eng.step(t, fuse=fuse)
                lt = torch.tensor([loss], device=dev, dtype=torch.float64)
                allv = [torch.zeros_like(lt) for _ in range(world)]
                dist.all_gather(allv, lt)
                curve.append(sum(float(x.item()) for x in allv) / world)
            err = float(np.max(np.abs(np.array(curve) - tg["train_loss"][1:])))
            res[f"tiny_gpt_{'fused' if fuse else 'unfused'}"] = {
                "train_loss_max_abs_diff": err,
                "outer": [rec.iteration for rec in eng.records if rec.kind == "outer"],
                "folds": eng.warmup_folds}
            del eng

    # lazy-phase gradient mean vs the reference left fold
    n = 1_000_003
    grads = [np.random.default_rng([5, r]).standard_normal(n).astype(np.float32) for r in range(world)]
    buf = torch.from_numpy(grads[rank]).to(dev)
    comm.allreduce_mean_(buf, 1 << 18)
    want = O.mean_left_fold(grads)
    got = buf.cpu().numpy()
    res["grad_mean"] = {"bitwise": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
                        "rel": rel(got, want)}
    npad = P.padded_len(n, world)
    sbuf, sid = comm.alloc_shared(npad)
    sbuf[:n].copy_(torch.from_numpy(grads[rank]).to(dev))
    comm.allreduce_mean_p2p_(sid, npad)
    got = sbuf[:n].cpu().numpy()
    res["grad_mean_p2p"] = {"bitwise": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
                            "rel": rel(got, want)}
    # the same mean fused with the clip norm of its result (lazy phase, one pass)
    sbuf[:n].copy_(torch.from_numpy(grads[rank]).to(dev))
    ws = P.norm_workspace()
    comm.allreduce_mean_norm_p2p_(sid, npad, 1.0, ws)
    got = sbuf[:n].cpu().numpy()
    rec = P.read_clip(ws)
    ws2 = P.norm_workspace()
    P.grad_sqnorm_(sbuf, 1.0, ws2)               # K4a over the averaged buffer
    rec2 = P.read_clip(ws2)
    exact = float(np.dot(want.astype(np.float64), want.astype(np.float64)))
    allsq = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(allsq, torch.tensor([rec.sqnorm], dtype=torch.float64, device=dev))
    res["grad_mean_norm_p2p"] = {
        "bitwise": bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
        "sqnorm_relerr": abs(rec.sqnorm - exact) / exact,
        "same_on_all_ranks": len({float(x.item()) for x in allsq}) == 1,
        "scale_equals_k4a": rec.scale == rec2.scale and rec.clipped == rec2.clipped,
        "clipped": bool(rec.clipped)}
    torch.cuda.synchronize()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
