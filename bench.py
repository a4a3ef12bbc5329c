#!/usr/bin/env python
"""bench.py -- Pier round throughput on B200 (BASELINE.json metric).

A "step" is one Pier round per group at an outer boundary: the global-norm
clip (K4a) + AdamW inner step and the outer step (mean of the groups, Nesterov
update with the scheduled mu / outer lr, re-anchor) -- one fused K5 pass at one
group, one persistent kernel per GPU at n > 1 (AdamW overlapped with the NVLink
pull-fold-update-push exchange; --reduce nccl / nvls for the alternatives),
over a synthetic GPT-2-XL-shaped flat fp32 parameter set (1,557,611,200
params; every array 6.2 GB >> 126 MB L2, so no L2 flush is needed).  One
group per GPU; per-GPU work is fixed as N grows ("weak" scaling); ``value`` =
groups x params / s for the whole job.  At n > 1 the line also reports the
lazy-phase iteration (the sharded step: reduce-scatter + norm, AdamW on the
rank's shard, all-gather) beside the replicated variant.

  python bench.py [--gpus N --steps K --warmup W --config xl]   # N > 1: starts its own N ranks
  torchrun --nproc-per-node N bench.py --gpus N ...
  python bench.py --impl reference ...    # the reference algorithm on the host CPU
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # SURVEY.md §8a sizes
    "tiny": 306_176,
    "small": 124_439_808,
    "medium": 354_823_168,
    "xl": 1_557_611_200,
    "7b": 6_658_596_864,
}
METRIC = "Pier outer-step params/s & %HBM/NVLink roofline, GPT-2 XL, 1/2/4/8 B200"
UNIT = "params/s"
NVLINK_GBS = 900.0   # nominal per direction per GPU (BASELINE.md roofline); measured peer ~770
NVLINK_MEASURED_GBS = 770.0   # B200_PROFILING.md peer copy per direction (profiles/r01_nvlink_probe.json: 771)
NVLINK_ALLTOALL_GBS = 678.0   # SM-driven all-to-all pull+push at n=4, tools/nvl_mix_probe.cu (context only)
# T = 100,000, r = 50 (Table I); t = 50,000 + 50k is on the 1.1 plateau, mu 0.9
T_TOTAL, R_SYNC, T0 = 100_000, 50, 50_000


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a while to start: wait for its first sample, then keep
            # only the samples taken inside the timed region (a 0.4 s region at n = 4
            # otherwise ended before the first one)
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.rows.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on the host
# ---------------------------------------------------------------------------

class CpuRound:
    """Pier round on the host with the oracle port (the reference's algorithm):
    per group clip + AdamW, then the left-fold mean of the groups + delta +
    anchor-form outer step (driver.py:395-440), on `sample` params per group
    (default: the whole GPT-2-small-sized set of BASELINE config 2), chunked
    over `threads` (bitwise = unchunked).  Inputs are built once."""

    def __init__(self, sample: int, groups: int, threads: int):
        import numpy as np

        from oracle import pier_oracle as O

        self.O, self.np = O, np
        f32 = np.float32
        rng = np.random.default_rng(0)
        base = 1 << 22  # draw one block and tile it: input generation stays cheap
        tile = lambda scale: np.resize(rng.standard_normal(min(sample, base), dtype=f32) * f32(scale), sample)  # noqa: E731
        self.anchor = tile(0.02)
        self.thetas = [self.anchor + tile(1e-3) for _ in range(groups)]
        self.mom, self.g, self.m = tile(1e-3), tile(1e-4), tile(1e-4)
        self.v = self.m * self.m + f32(1e-12)
        s = O.Sched(total_iters=T_TOTAL, sync_interval=R_SYNC)
        self.lr_in, self.mu, self.lr = O.inner_lr(T0, s), O.momentum_mu(T0, T_TOTAL), O.outer_lr(T0, s)
        self.sample, self.groups, self.threads = sample, groups, threads
        self.ck = max(1 << 16, sample // (4 * threads))

    def run(self) -> float:
        """One round; returns seconds."""
        O, np, f32 = self.O, self.np, self.np.float32

        def par(fn, arrays):
            return O.chunked(fn, arrays, self.threads, self.ck)

        t0 = time.perf_counter()
        new = []
        for th in self.thetas:
            g = self.g
            nrm = float(np.sqrt(np.dot(g, g)))  # optim.py:76 (OpenBLAS sdot, its own threads)
            gc = g if nrm <= 1.0 else par(lambda x: (x * f32(1.0 / nrm),), [g])[0]
            out = par(lambda a, b, c, d: O.adamw(a, b, c, d, 10, self.lr_in)[:3], [th, gc, self.m, self.v])
            new.append(out[0])
        avg = par(lambda *xs: (O.mean_left_fold(list(xs)),), new)[0]
        par(lambda a, b, c: O.outer_anchor_form(a, b, c, self.lr, self.mu), [avg, self.anchor, self.mom])
        return time.perf_counter() - t0


def cpu_round_rate(sample: int, groups: int, threads: int, reps: int = 2):
    """(group-params/s, best seconds per round) of CpuRound over `reps` rounds."""
    cr = CpuRound(sample, groups, threads)
    best = min(cr.run() for _ in range(reps))
    return groups * sample / best, best


CPU_SAMPLE_DOC = ("one whole Pier round per step on the full GPT-2-small-sized parameter set (BASELINE "
                  "config 2: {sample} params per group, x {groups} groups): per group clip + AdamW, left-fold "
                  "mean, delta, anchor-form outer step (oracle/pier_oracle.py = optim.py:70-103, "
                  "topology.py:104-122, optim.py:248-276); measured, not extrapolated")


def run_reference(args):
    """The reference's CPU algorithm (the oracle port of optim.py / topology.py;
    the reference package cannot travel to the GPU box) on the host cores, for
    the same metric and config as our arm.  Each step is one measured round on
    the full small-config arrays per group (the XL arrays of n groups do not
    fit a few-minute run: ~35 s of single-core AdamW per XL group)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    groups = args.gpus
    threads = len(os.sched_getaffinity(0))
    sample = args.ref_sample
    cr = CpuRound(sample, groups, threads)
    for _ in range(args.warmup):
        cr.run()
    t_all = time.perf_counter()
    secs = [cr.run() for _ in range(args.steps)]
    wall = time.perf_counter() - t_all
    value = groups * sample * len(secs) / sum(secs)
    # context: the reference's own execution model (single-threaded NumPy), one round
    one = CpuRound(sample, 1, 1)
    s1 = one.run()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, groups),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": CPU_SAMPLE_DOC.format(sample=sample, groups=groups)
                         + f"; chunked over {threads} host threads",
                         "cpu": _cpu_model(), "cpu_count": os.cpu_count(), "affinity": threads,
                         "timed_s": sum(secs), "wall_s": wall,
                         "single_thread": {"value": sample / s1, "unit": UNIT, "cores": 1, "groups": 1,
                                           "round_s": s1}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def bucket_elems_for(args, world: int) -> int:
    # p2p round: 32 MB slices at n <= 2, 8 MB above (r02 sweep, profiles/r02_round_sweep_buckets.log:
    # n=2 16 MB 12.49 -> 32 MB 12.27 ms; n=4 8 MB 14.93 vs 16 MB 15.11); the bucketed NCCL path
    # needs large buckets (256 MB: n=2 outer step 17.0 -> 15.0 ms, tools/exp/README.md: nccl_sweep)
    bucket_mb = args.bucket_mb or (256 if args.reduce == "nccl" else 32 if world <= 2 else 8)
    return bucket_mb * (1 << 20) // 4


def workload_config(args, world: int) -> dict:
    """The `config` object both arms print (the same workload)."""
    n = CONFIGS[args.config]
    q = world * 64                                   # topology.padded_len (ALIGN = 64 elements)
    return {"workload": f"gpt2-{args.config} pier round (clip+AdamW inner step + outer step), "
                        f"one group per GPU", "params": n, "params_padded": (n + q - 1) // q * q, "groups": world,
            "bucket_elems": bucket_elems_for(args, world), "reduce": args.reduce if world > 1 else "none",
            "schedule": f"T={T_TOTAL} r={R_SYNC} t={T0}+{R_SYNC}k (mu 0.9, lr 1.1)",
            "l2": "inputs larger than L2 (each array 4*N bytes >> 126 MB); no flush"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2511_17849_b200 as P
    from paper_2511_17849_b200._lib import lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = P.GroupComm(rank, world) if world > 1 else None
    n = CONFIGS[args.config]
    sched = P.ScheduleConfig(total_iters=T_TOTAL, sync_interval=R_SYNC)
    bucket = bucket_elems_for(args, world)

    # synthetic state (BASELINE.md inputs): anchor ~ N(0,.02^2) shared; theta_g = anchor + N(0,1e-3^2)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    theta0 = torch.randn(n, device=dev, generator=gen).mul_(0.02)
    eng = P.PierEngine(n, sched, comm=comm, bucket_elems=bucket, theta0=theta0, reduce=args.reduce)
    del theta0
    gen.manual_seed(1000 + rank)
    eng.theta[:n].add_(torch.randn(n, device=dev, generator=gen).mul_(1e-3))
    eng.mom.normal_(0.0, 1e-3, generator=gen)
    eng.grad[:n].normal_(0.0, 1e-4, generator=gen)          # XL: |g| ~ 3.9 > clip 1.0
    eng.m[:n].normal_(0.0, 1e-4, generator=gen)
    torch.mul(eng.m, eng.m, out=eng.v).add_(1e-12)
    eng.opt_step = 10
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    fuse = not args.no_fuse

    def one(k, marks=None):
        # engine.step: K4a norm, then (fused) AdamW + outer step of a boundary iteration
        eng.step(T0 + R_SYNC * (k % 500), mark=(marks[1].record if marks else None), fuse=fuse)

    for k in range(args.warmup):
        one(k)
    barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = int(lib.pier_launch_count())
    with ClockSampler(local) as clk:
        barrier()
        start.record()
        for k in range(args.steps):
            ev[k][0].record()
            one(args.warmup + k, ev[k])
            ev[k][3].record()
        stop.record()
        barrier()
    launches = int(lib.pier_launch_count()) - launches0
    ms = start.elapsed_time(stop)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    t_norm = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    t_rest = statistics.mean(e[1].elapsed_time(e[3]) for e in ev)
    value = world * n / (ms_step / 1e3)

    # per-kernel breakdown on the UNFUSED path (norm | AdamW | outer step), timed live
    bd = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.breakdown_steps)]
    barrier()
    for k, e in enumerate(bd):
        t = T0 + R_SYNC * ((args.warmup + args.steps + k) % 500)
        e[0].record()
        eng.inner_step(t, mark=e[1].record)
        e[2].record()
        eng.boundary(t)
        e[3].record()
    barrier()
    adam_each = [e[1].elapsed_time(e[2]) for e in bd]
    outer_each = [e[2].elapsed_time(e[3]) for e in bd]
    t_adam, t_outer = statistics.median(adam_each), statistics.median(outer_each)

    # lazy phase: every iteration averages the gradients over
    # all groups (bitwise left fold over NVLink) before clip + AdamW (driver.py:372-399).
    # Default: sharded -- reduce-scatter + norm of the mean, AdamW on this rank's 1/n,
    # all-gather of theta (pier_lazy_step_p2p_f32); the replicated variant (all-reduce +
    # norm, then AdamW over the whole buffer on every rank) is timed beside it.
    lazy = None
    if world > 1:
        t_lazy = sched.lazy_end // 2

        def lazy_ms():
            le = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.breakdown_steps)]
            barrier()
            for e in le:
                e[0].record()
                eng.inner_step(t_lazy)
                e[1].record()
            barrier()
            return statistics.mean(e[0].elapsed_time(e[1]) for e in le)

        t_it = lazy_ms()
        sharded = eng.lazy_sharded
        eng.gather_moments()
        eng.lazy_sharded = False
        t_rep = lazy_ms()
        eng.lazy_sharded = sharded
        wire = 2.0 * (world - 1) / world * 4.0 * npad_of(eng)
        lazy = {"iteration_ms": t_it, "t": t_lazy,
                "what": ("sharded: gradient reduce-scatter (P2P left fold) fused with K4a (norm of the mean), "
                         "AdamW on this rank's shard (its slice of every span), all-gather of the params" if sharded else
                         "gradient mean over groups (P2P left fold) fused with K4a (norm of the mean), then K4b"),
                "replicated_iteration_ms": t_rep,
                "replicated_what": "all-reduce (P2P left fold) + K4a fused, then K4b over the whole buffer",
                "grad_mean_wire_bytes_per_direction": wire,
                "wire_floor_ms_at_770": wire / (NVLINK_MEASURED_GBS * 1e9) * 1e3,
                "adamw_floor_ms": 28.0 * npad_of(eng) / (peaks()[0] * 1e9) * 1e3,
                # sharded: the wire (reduce-scatter then all-gather, serialised by the norm) is the floor;
                # replicated: wire + the whole-buffer AdamW pass after it
                "frac_of_floor": (wire / (NVLINK_MEASURED_GBS * 1e9) * 1e3) / t_it if sharded else None}

    hbm, hbm_src = peaks()
    npad = eng.n_pad
    first = secondary = None
    bound, unit, peak, peak_src = "hbm", "GB/s", hbm, hbm_src
    if world == 1 and fuse:
        # dominant kernel of the fused step: K5 k_adamw_outer, one pass for AdamW + outer step
        dom, dom_bytes, dom_ms = "k_adamw_outer (K5 fused clip+AdamW+outer step)", 44.0 * npad, t_rest
        traffic = _profiled_traffic("k_adamw_outer", npad)
    elif fuse and args.reduce == "p2p":
        # dominant kernel of the fused step at n > 1: the persistent round k_round.
        # HBM per param: AdamW 28 + own slice 4/n + peers' pulls of our slices
        # 4(n-1)/n + anchor/M read+write 16/n + incoming results 4 = 36 + 16/n;
        # NVLink per direction 2(n-1)/n * 4 (pulls served + results pushed).
        # The binding resource is the one with the longer time at its peak.
        hbm_b = (36.0 + 16.0 / world) * npad
        nvl_b = 2.0 * (world - 1) / world * 4.0 * npad
        t_h, t_n = hbm_b / (hbm * 1e9), nvl_b / (NVLINK_MEASURED_GBS * 1e9)
        dom, dom_ms = "k_round (persistent AdamW || NVLink pull-fold-update-push)", t_rest
        # per-GPU DRAM bytes of the same kernel body at this group count, measured by ncu on one
        # GPU through a VirtualGroup (k_round_multi: every rank's HBM traffic on the one device / n,
        # profiles/r02_round_virtual_ncu.txt); ncu cannot replay one rank of a multi-process round
        traffic = _profiled_traffic(f"k_round_n{world}", npad)
        h = {"bound": "hbm", "achieved": hbm_b / (t_rest / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
             "algorithmic_bytes_per_launch": hbm_b, "peak_source": hbm_src}
        v = {"bound": "nvlink", "achieved": nvl_b / (t_rest / 1e3) / 1e9, "peak": NVLINK_MEASURED_GBS,
             "unit": "GB/s", "algorithmic_bytes_per_launch": nvl_b,
             "peak_source": "measured peer copy per direction (B200_PROFILING.md 770; r01_nvlink_probe 771)"}
        for d in (h, v):
            d["frac"] = d["achieved"] / d["peak"]
        v["frac_of_900_nominal"] = v["achieved"] / NVLINK_GBS   # north_star's 900 GB/s per direction
        h["traffic"] = traffic
        # context: the round's own link pattern (all-to-all pulls + pushes at once, SM-driven)
        # measured alone tops out near 678 GB/s per direction (profiles/r01_nvl_mix_probe_n4.jsonl)
        v["alltoall_pull_push_ceiling"] = NVLINK_ALLTOALL_GBS
        v["frac_of_alltoall_ceiling"] = v["achieved"] / NVLINK_ALLTOALL_GBS
        first, secondary = (h, v) if t_h >= t_n else (v, h)
        dom_bytes, bound, unit, peak, peak_src = (first["algorithmic_bytes_per_launch"], first["bound"],
                                                  first["unit"], first["peak"], first["peak_source"])
    else:
        # AdamW: read theta,g,m,v + write theta,m,v (32 B incl. the norm's 4)
        dom, dom_bytes, dom_ms = "k_adamw (K4b fused clip+AdamW)", 28.0 * npad, t_adam
        traffic = _profiled_traffic("k_adamw", npad)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    t_roof = (32.0 * n / (hbm * 1e9) + max(24.0 * n / (world * hbm * 1e9),
                                            2.0 * (world - 1) / world * 4.0 * n / (NVLINK_GBS * 1e9))) * 1e3

    # end to end through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = e2e_res = None
    if not args.no_e2e:
        e2e = run_e2e(eng, n, args, world, dev)
        e2e_res = run_e2e_resident(eng, n, args, world, dev)
        if "skipped" in e2e:
            # the host cannot hold every rank's optimizer state (8 XL groups: ~300 GB of
            # arrays on a 196 GB host): the end-to-end number is the engine API from host
            # buffers with the state resident on the GPUs (gradient in, params out)
            e2e = dict(e2e_res, full_host_state=e2e["skipped"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's execution model: single-threaded NumPy (the value), plus
        # the same round chunked over every host thread (context; = --impl reference)
        cr = CpuRound(args.cpu_sample, 1, 1)
        secs = [cr.run() for _ in range(args.cpu_reps)]
        threads = len(os.sched_getaffinity(0))
        crt = CpuRound(args.cpu_sample, 1, threads)
        tsecs = [crt.run() for _ in range(2)]
        del cr, crt
        cpu = {"value": args.cpu_sample / min(secs), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": CPU_SAMPLE_DOC.format(sample=args.cpu_sample, groups=1)
               + f"; best of {args.cpu_reps} single-threaded rounds ({sum(secs):.1f} s of CPU work)",
               "cpu": _cpu_model(), "cpu_count": os.cpu_count(), "affinity": threads,
               "all_threads": {"value": args.cpu_sample / min(tsecs), "unit": UNIT, "cores": threads}}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "kernels_ms": {"timed_step": {"grad_sqnorm(K4a)": t_norm,
                                      ("adamw+outer fused" if fuse else "adamw+outer"): t_rest},
                       "unfused_breakdown": {"adamw(K4b)": t_adam, "outer_step": t_outer,
                                             "steps": args.breakdown_steps, "stat": "median",
                                             "adamw_each": adam_each, "outer_each": outer_each}},
        "roofline": {"bound": bound, "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": unit, "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom_bytes, "peak_source": peak_src,
                     **({k: first[k] for k in ("alltoall_pull_push_ceiling", "frac_of_alltoall_ceiling",
                                               "frac_of_900_nominal")
                         if first and k in first}),
                     **({"other_resource": secondary} if secondary else {})},
        # the outer step alone (mean of the groups + Nesterov + re-anchor, unfused launch;
        # SURVEY §8d "also report the outer step alone"), whole-job params/s
        "outer_step": {"ms": t_outer, "params_per_s": world * n / (t_outer / 1e3),
                       "what": "K3 at one group; the P2P pull-fold-update-push exchange at n > 1"
                       if args.reduce == "p2p" or world == 1 else f"the {args.reduce} exchange + K3"},
        "step_roofline": {"t_roof_ms": t_roof, "frac": t_roof / ms_step,
                          "formula": "32N/BW_hbm + max(24N/(n BW_hbm), 2(n-1)/n 4N/BW_nvl), BW_nvl 900 GB/s"},
        **({"lazy_phase": lazy} if lazy else {}),
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        **({"e2e_resident_state": e2e_res} if e2e_res else {}),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def _mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def run_e2e(eng, n, args, world, dev):
    """Same metric through PierEngine.step_host: per step the whole state the
    reference keeps on the host goes H2D, the round runs, results go D2H."""
    import torch

    vs = eng._valid_shard()
    need = (4 * n + 2 * vs) * 4 * world          # pinned bytes of all ranks on this host
    avail = _mem_available()
    if world > 1:
        # one decision for all ranks (their MemAvailable readings can differ; a rank
        # that skipped while the others entered step_host would hang the exchange)
        import torch.distributed as dist
        a = torch.tensor([avail if avail is not None else -1], dtype=torch.float64, device=dev)
        dist.all_reduce(a, op=dist.ReduceOp.MIN)
        avail = None if a.item() < 0 else int(a.item())
    if avail is not None and need > 0.6 * avail:
        return {"skipped": f"host state of {world} groups needs {need / 1e9:.0f} GB pinned, "
                           f"{avail / 1e9:.0f} GB available"}
    pin = dict(dtype=torch.float32, pin_memory=True)
    host = {k: torch.empty(n, **pin) for k in ("theta", "grad", "m", "v")}
    host["anchor"] = torch.empty(vs, **pin)
    host["mom"] = torch.empty(vs, **pin)
    for k, src in (("theta", eng.theta), ("grad", eng.grad), ("m", eng.m), ("v", eng.v)):
        host[k].copy_(src[:n])
    host["anchor"].copy_(eng.anchor[:vs])
    host["mom"].copy_(eng.mom[:vs])
    torch.cuda.synchronize()
    h2d = sum(host[k].numel() * 4 for k in host)
    d2h = h2d - host["grad"].numel() * 4
    steps = max(1, min(args.steps, 5))
    for k in range(2):
        eng.step_host(T0 + R_SYNC * (400 + k), host)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        eng.step_host(T0 + R_SYNC * (450 + k), host)
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([sec], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sec = float(tt.item())
    return {"value": world * n / sec, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": sec * 1e3, "steps": steps,
            "api": "PierEngine.step_host (pinned host theta/grad/m/v + outer-state shard, in place)"}


def npad_of(eng) -> int:
    return eng.n_pad


def run_e2e_resident(eng, n, args, world, dev):
    """The engine API from host buffers: the optimizer state stays on the GPU
    (PierEngine), every step the gradient comes up from pinned host memory and
    the new parameters go back down (what a host-side model would do)."""
    import torch

    pin = dict(dtype=torch.float32, pin_memory=True)
    g_host = torch.empty(n, **pin)
    th_host = torch.empty(n, **pin)
    g_host.copy_(eng.grad[:n])
    steps = max(1, min(args.steps, 10))

    def one(t):
        eng.grad[:n].copy_(g_host, non_blocking=True)
        eng.step(t)
        th_host.copy_(eng.theta[:n], non_blocking=True)

    for k in range(2):
        one(T0 + R_SYNC * (470 + k))
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        one(T0 + R_SYNC * (475 + k))
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([sec], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sec = float(tt.item())
    return {"value": world * n / sec, "unit": UNIT, "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
            "ms_per_step": sec * 1e3, "steps": steps,
            "api": "PierEngine.step with the state resident on the GPU: gradient H2D, new params D2H (pinned)"}


def _profiled_traffic(kernel: str, npad: int):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d[kernel]
        return e["dram_bytes_per_param"] * npad
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="xl")
    ap.add_argument("--bucket-mb", type=int, default=0,
                    help="per-rank slice of one span in MB; 0 = auto: 32 at n <= 2, 8 at n >= 4 "
                         "(tools/exp/README.md: round_l2), 256 for --reduce nccl (tools/exp/README.md: nccl_sweep)")
    ap.add_argument("--reduce", choices=("p2p", "nvls", "nccl"), default="p2p")
    ap.add_argument("--no-fuse", action="store_true", help="time the unfused inner step + boundary stage")
    ap.add_argument("--breakdown-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=CONFIGS["small"])
    ap.add_argument("--cpu-reps", type=int, default=2)
    ap.add_argument("--ref-sample", type=int, default=CONFIGS["small"])
    ap.add_argument("--launch-check", action="store_true",
                    help="print this rank's launcher environment and exit (tests the N-rank self-launch on CPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)      # rank 0 only, on the host: no launcher needed
        return
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        relaunch(args.gpus)      # one process per GPU; does not return
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or drop the launcher and let bench.py start them")
    if args.launch_check:
        line = json.dumps({"rank": int(os.environ.get("RANK", "0")), "world": int(world or 1),
                           "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
                           "master": os.environ.get("MASTER_ADDR")}) + "\n"
        os.write(1, line.encode())   # one write(2) per rank: the ranks share the pipe
        return
    run_ours(args)


def relaunch(n: int) -> None:
    """`python bench.py --gpus N` without a launcher: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1, a free port)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: starting {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


if __name__ == "__main__":
    main()
