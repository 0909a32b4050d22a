#!/usr/bin/env python
"""bench.py — one simulated FedAvg round per step on N B200s (BASELINE.json metric:
client-updates/s and FedAvg round time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C3|...]

Workload: at every N, BASELINE configs[2] = C3, the north-star round (1,000
of 10,000 CIFAR-shaped clients, log-normal sizes 10..2000, McMahan CNN, E=2, B=32), placed
across the N GPUs by the library (strong scaling; one NCCL allreduce of [S‖N] per round at
N>1).  At N=1 the line also carries configs[1] (C2: 100 clients, E=1) as its `c2` object.
A step = one whole round (place -> pack -> local SGD of every client -> fused FedAvg
accumulation -> allreduce -> finalize), inputs resident in HBM.  The per-round working
set (client models K x 8.6 MB + activations) exceeds the 126 MB L2, so no flush is
needed between steps.  For N>1 launch with torchrun (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "client-updates/s (FedAvg round throughput)"
UNIT = "client-updates/s"
FLOPS_PER_SAMPLE_EPOCH = {"cnn": 101_087_232.0, "speech": 337_250_000.0, "logreg": 31_360.0}


def workload(world: int, name: str | None):
    """(Workload, description, scaling).  Default at every N: BASELINE configs[2] = C3, the
    north-star round (1,000 of 10,000 CIFAR-shaped clients, E = 2, B = 32) whose metric is
    quoted at 1/2/4/8 GPUs -- strong scaling: the same round on N GPUs, so the driver's
    per-N values form one curve.  configs[1] (C2, the single-GPU config) is measured beside
    it at N = 1 (the `c2` object of the line) and with --config C2."""
    name = name or "C3"
    wl = synth.preset(name)
    desc = {"C1": "C1: 10 logreg clients, 784-dim, sizes 5-50, E=1, B=5",
            "C2": "C2: 100 CIFAR-shaped clients, log-normal sizes 10-2000, McMahan CNN, E=1, B=32",
            "C3": "C3: 1,000 of 10,000 CIFAR-shaped clients, log-normal sizes 10-2000, McMahan CNN, E=2, B=32",
            "C4": "C4: 2,000 speech-shaped clients (1x40x98), log-normal sizes 5-5000, conv+MLP, E=1, B=20",
            "C5": "C5: 700 Shakespeare-shaped clients, log-normal sizes 4-4000, char-LSTM, E=1, B=4"}[name]
    return wl, desc, ("strong" if world > 1 else "weak")


def run_config(wl, desc, cohort, sizes, world, agg="nccl"):
    """The `config` object of both arms' JSON lines (identical for ours and --impl reference)."""
    return {"workload": desc, "clients": int(len(cohort)), "samples": int(sizes.sum()), "B": wl.B, "E": wl.E,
            "lr": wl.lr, "parallelism": f"clients x{world}", "aggregation": agg,
            "l2": "per-round working set >> 126 MB L2 (no flush needed)"}


def pop_for(wl):
    """Sizes of the whole population, the cohort, and data for the cohort's clients only,
    re-indexed so the library's population = the cohort's clients (ids 0..K-1)."""
    sizes_all = synth.client_sizes(wl)
    cohort = synth.cohort(wl)
    ids = np.sort(cohort)
    sizes = sizes_all[ids]
    _, x, y = synth.population(wl, sizes_all, clients=ids)
    return sizes, x, y, np.arange(len(ids), dtype=np.int64)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md).

    The sampler is started before the region and waits for its first sample (nvidia-smi takes
    ~100 ms to start); samples carry a timestamp and only those inside [mark_start, mark_end]
    are summarised (the nearest ones if the region is shorter than the 20 ms interval)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", ",".join(map(str, self.gpus))],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            deadline = time.time() + 5.0
            while time.time() < deadline and os.path.getsize(self.path) == 0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    @staticmethod
    def _ts(field):
        import datetime
        try:
            return datetime.datetime.strptime(field.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 10 and p[2].replace(".", "").isdigit():
                rows.append((self._ts(p[0]), p[1:]))
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        inside = [r for t, r in rows if t is not None and self.t0 is not None and self.t1 is not None
                  and self.t0 - 0.025 <= t <= self.t1 + 0.025]
        sel = inside or [r for _, r in rows]
        sm = [float(r[1]) for r in sel]
        mx = max(float(r[2]) for r in sel)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in sel for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons, "samples": len(sel),
                "samples_in_timed_region": len(inside),
                "power_w_max": max((float(r[3]) for r in sel if r[3].replace(".", "").isdigit()), default=None)}


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


# Kernel classes that run on the tensor cores when math = 0 (tcgen05 kind::tf32).
TC_KINDS = {"conv1_fwd", "conv2_fwd", "conv2_dx", "conv2_dw", "conv1_dw", "fc1_fwd", "fc1_dx", "fc1_dw_sgd"}
TF32_PER_BF16 = 1.1 / 2.25   # nominal dense tf32 / bf16 (B200_PROFILING.md table)


def kernel_roofline(name, k, math, mp):
    """One kernel class against its own roofline.

    bound = the resource its ALGORITHMIC intensity (flops / bytes) saturates first:
    tensor (TF32 peak = measured bf16 sustained x nominal tf32/bf16), HBM (measured
    copy bandwidth), or, for FP32 CUDA-core GEMMs (math = 1), the FFMA rate."""
    per_launch_s = k["ms"] / k["launches"] * 1e-3
    hbm = mp["hbm_gbs"]
    tensor = k["flops"] > 0 and name in TC_KINDS and math == 0
    if tensor:
        peak_f = mp.get("bf16_tflops_sustained", mp["bf16_tflops"]) * TF32_PER_BF16
        src_f = "measured bf16_tflops_sustained x 1.1/2.25 (tf32/bf16 nominal)"
    else:
        peak_f = 148 * 128 * 2 * mp.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        src_f = "FP32 FFMA: 148 SM x 128 lanes x 2 x sm_max_mhz"
    ridge = peak_f * 1e12 / (hbm * 1e9)
    if k["flops"] == 0 or k["flops"] / max(k["bytes"], 1.0) < ridge:
        achieved = k["bytes"] / k["launches"] / per_launch_s / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
               "peak_source": "measured hbm_gbs (copy)"}
    else:
        achieved = k["flops"] / k["launches"] / per_launch_s / 1e12
        out = {"bound": "tensor" if tensor else "alu", "achieved": achieved, "peak": peak_f, "unit": "TFLOP/s",
               "peak_source": src_f}
    out["frac"] = out["achieved"] / out["peak"]
    return out


def roofline(kstats, math, total_ms):
    """Dominant kernel class by device time, against its roofline."""
    mp, src = peaks()
    name, k = max(kstats.items(), key=lambda kv: kv[1]["ms"])
    out = kernel_roofline(name, k, math, mp)
    out["peak_source"] = f"{src}: {out['peak_source']}"
    out["kernel"] = name
    out["share_of_round"] = k["ms"] / total_ms if total_ms else None
    out["launches_per_round"] = k["launches"]
    out["traffic"], out["traffic_source"] = ncu_traffic(name)
    return out


def kernel_table(kstats, math):
    mp, _ = peaks()
    tab = {}
    for name, k in sorted(kstats.items(), key=lambda kv: -kv[1]["ms"]):
        r = kernel_roofline(name, k, math, mp)
        tab[name] = {"ms": round(k["ms"], 4), "launches": k["launches"], "bound": r["bound"],
                     "achieved": round(r["achieved"], 2), "unit": r["unit"], "frac": round(r["frac"], 4)}
    return tab


def ncu_traffic(kernel_class):
    """DRAM bytes per launch of this class (dram__bytes_read.sum + dram__bytes_write.sum) from the
    committed ncu --set full capture of that kernel (profiles/ncu_traffic.json records which
    capture); None if the class was not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
    except Exception:
        return None, None
    v = d.get(kernel_class)
    return v, (d.get("_source") if v is not None else None)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(wl, sizes, x, y, theta, max_client=64, threads=0, seed=1):
    """The oracle, as it stands, on a bounded random sample of the workload's clients.

    The fp64 oracle trains ~8 sample-steps per second per host thread on the CIFAR CNN, so one
    average C3 client (~480 sample-steps) alone is about a minute of one core.  To keep a step at
    ~10 s of wall time on all cores the sample is `threads` random clients of the cohort among
    those with n <= max_client samples (one OpenMP task per client, largest first), and
    client-updates/s = (sample-steps/s) / (mean sample-steps of a client of the whole workload):
    the oracle's cost per sample-step does not depend on the client's size.  `cores` = the
    threads that had a client.  A second, single-thread timing of one client is reported as
    `single_thread`."""
    import oracle
    threads = threads or cpu_threads()
    rng = np.random.default_rng(seed)
    order = [int(c) for c in rng.permutation(len(sizes)) if sizes[c] <= max_client]
    if not order:
        order = [int(np.argmin(sizes))]
    pick = sorted(order[:threads], key=lambda c: -int(sizes[c]))
    tot = int(sizes[pick].sum())
    pop_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    mean_client = float(np.mean(sizes)) * wl.E
    t0 = time.perf_counter()
    _, used = oracle.train_clients(wl.model, theta, x, y, pop_off, np.array(pick), wl.B, wl.E, wl.lr, threads=threads)
    dt = time.perf_counter() - t0
    value = tot * wl.E / dt / mean_client
    small = pick[-1]
    t1 = time.perf_counter()
    oracle.train_clients(wl.model, theta, x, y, pop_off, np.array([small]), wl.B, wl.E, wl.lr, threads=1)
    dt1 = time.perf_counter() - t1
    cores = int(min(used, len(pick)))
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{len(pick)} random clients of the cohort with n <= {max_client} ({tot} samples x E={wl.E}), "
                      f"largest first, trained by the fp64 oracle on {cores} host threads in {dt:.1f} s; "
                      f"client-updates/s = sample-steps/s / mean sample-steps of a workload client ({mean_client:.1f})",
            "seconds": dt, "host_threads": int(threads),
            "single_thread": {"value": int(sizes[small]) * wl.E / dt1 / mean_client, "unit": UNIT, "cores": 1,
                              "sample": f"1 client ({int(sizes[small])} samples x E={wl.E}) in {dt1:.2f} s"}}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def allmax(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allmax_list(vs, world):
    if world == 1:
        return list(vs)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in vs], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def pct(v, q):
    return float(np.percentile(np.asarray(v, dtype=np.float64), q))


def run_reference(args, world, rank):
    """The oracle (the only reference this tier has) on the host cores; rank 0 only."""
    if rank != 0:
        return
    wl, desc, scaling = workload(args.gpus, args.config)
    sizes, x, y, cohort = pop_for(wl)
    theta = synth.init_params(wl.model)
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(wl, sizes, x, y, theta, max_client=args.ref_max_client, seed=1 + i)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.median(c["value"] for c in vals)
    ms = len(cohort) / v * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8d laws)",
            "config": run_config(wl, desc, cohort, sizes, world, args.agg),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[-1]["cores"], "kind": "oracle",
                             "sample": vals[-1]["sample"] + f"; median of {args.steps} such samples"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
            "note": "each step trains a bounded random sample of the cohort's clients on the host cores and "
                    "converts samples/s to client-updates/s; ms_per_step is the implied whole-round time"}
    print(json.dumps(line), flush=True)


def peer_connect(ctx, world, max_clients):
    """Exchange the ranks' peer blobs (CUDA IPC handles) over torch.distributed and connect."""
    blob = ctx.fl_peer_export(max_clients if ctx.cfg.rank == 0 else 0)
    if world == 1:
        ctx.fl_peer_connect([blob])
        return
    import torch.distributed as dist
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    ctx.fl_peer_connect(blobs)


def timed_rounds(ctx, cohort, steps, rnd, world, stream, clk=None):
    """K rounds queued back to back on the ctx stream, bracketed by barrier + synchronize;
    one CUDA event between consecutive rounds gives the per-round device times.  Returns
    (total ms max over ranks, per-round ms max over ranks, next round index)."""
    import torch
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    barrier(world)
    torch.cuda.synchronize()
    if clk:
        clk.mark_start()
    evs[0].record(stream)
    for i in range(steps):
        ctx.fl_round(cohort, round_index=rnd, stats=False)
        rnd += 1
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.mark_end()
    barrier(world)
    per = allmax_list([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)], world)
    total = allmax(evs[0].elapsed_time(evs[-1]), world)
    return total, per, rnd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="C1..C5 (default C3, BASELINE configs[2])")
    ap.add_argument("--math", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the configs[1] (C2) measurement at N = 1")
    ap.add_argument("--cpu-max-client", type=int, default=64,
                    help="cpu_baseline samples clients with at most this many samples (~10 s per step)")
    ap.add_argument("--ref-max-client", type=int, default=48,
                    help="--impl reference: the same, per step (K + W steps must end within minutes)")
    ap.add_argument("--agg", default="nccl", choices=["nccl", "peer", "unaggregated"],
                    help="cross-rank aggregation (include/fl.h agg_mode): NCCL allreduce of partials, one "
                         "peer-memory kernel, or the unaggregated ablation (all client models to rank 0)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import paper_2306_17453_b200 as fl
    torch.cuda.set_device(local)
    wl, desc, scaling = workload(world, args.config)
    sizes, x, y, cohort = pop_for(wl)
    theta = synth.init_params(wl.model)
    def new_uid():
        """A fresh NCCL unique id from rank 0 (one per communicator: an id is not reused)."""
        if world == 1 or args.agg != "nccl":
            return None
        import torch.distributed as dist
        obj = [fl.fl_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    uid = new_uid()
    cfg = fl.Config(model=wl.model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, shuffle=wl.shuffle, seed=wl.seed,
                    rank=rank, world_size=world, device=local, nccl_unique_id=uid, math=args.math,
                    agg_mode=args.agg)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    ctx = fl.fl_round_init(cfg, sizes, xd, yd, theta)
    if args.agg != "nccl":
        peer_connect(ctx, world, len(cohort))
    stream = torch.cuda.ExternalStream(ctx.stream)
    rnd = 0
    for _ in range(args.warmup):
        ctx.fl_round(cohort, round_index=rnd, stats=False)
        rnd += 1
    torch.cuda.synchronize()
    with ClockSampler(list(range(world)) if rank == 0 else [local]) as clk:
        ms_total, per_step, rnd = timed_rounds(ctx, cohort, args.steps, rnd, world, stream, clk)
    clocks = clk.summary()
    # one more round with stats: max-over-ranks round time and "timedelta workers"
    st = ctx.fl_round(cohort, round_index=rnd)
    rnd += 1
    ms_step = ms_total / args.steps
    value = len(cohort) * args.steps / (ms_total * 1e-3)
    # per-kernel device time of one extra (profiled, serialised) round, for the roofline
    ctx.fl_set_profiling(True)
    st_p = ctx.fl_round(cohort, round_index=rnd)
    rnd += 1
    kstats = ctx.fl_get_kernel_stats()
    ctx.fl_set_profiling(False)
    roof = roofline(kstats, args.math, st_p["round_ms"])
    ctx.close()
    del xd, yd
    torch.cuda.empty_cache()
    # e2e: the public API with HOST buffers; H2D of this rank's cohort rows and D2H of θ_new per step
    e2e = None
    if not args.no_e2e:
        cfg.nccl_unique_id = new_uid()
        ctx2 = fl.fl_round_init(cfg, sizes, x, y, theta, on_device=False)
        if args.agg != "nccl":
            peer_connect(ctx2, world, len(cohort))
        # one page-locked θ_new buffer per step: every step's result is copied back and kept
        outs = [torch.empty(ctx2.P, dtype=torch.float32, pin_memory=True) for _ in range(args.steps)]
        for _ in range(2):
            ctx2.fl_place(cohort)
            ctx2.fl_train_clients(0)
            ctx2.fl_aggregate_async(outs[0])
        ctx2.fl_synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for i in range(args.steps):
            # rounds are stream-ordered on the device, so the host places and issues round i+1
            # while round i runs; each round's θ_new is copied to its own pinned buffer
            ctx2.fl_place(cohort)
            ctx2.fl_train_clients(i)
            ctx2.fl_aggregate_async(outs[i])
        ctx2.fl_synchronize()  # every step's D2H has landed
        t_e2e = allmax((time.perf_counter() - t0) * 1e3, world)
        assert np.array_equal(outs[-1].numpy(), ctx2.fl_get_global_params())
        s2 = ctx2.fl_get_stats()
        e2e = {"value": len(cohort) * args.steps / (t_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(s2["h2d_bytes"]), "d2h_bytes_per_step": int(4 * ctx2.P),
               "ms_per_step": t_e2e / args.steps, "timer": "host wall clock around the public API calls",
               "pipelined": "fl_aggregate_async into one pinned buffer per step; fl_synchronize before the clock stops"}
        ctx2.close()
    # configs[1] (C2, 100 clients, single GPU) beside the C3 line at N = 1
    c2 = None
    if world == 1 and args.config is None and not args.no_c2:
        wl2 = synth.preset("C2")
        s2z, x2, y2, co2 = pop_for(wl2)
        th2 = synth.init_params("cnn")
        cfg2 = fl.Config(model="cnn", batch_size=wl2.B, local_epochs=wl2.E, lr=wl2.lr, device=local, math=args.math)
        x2d, y2d = torch.from_numpy(x2).cuda(), torch.from_numpy(y2).cuda()
        ctx3 = fl.fl_round_init(cfg2, s2z, x2d, y2d, th2)
        r2 = 0
        for _ in range(args.warmup):
            ctx3.fl_round(co2, round_index=r2, stats=False)
            r2 += 1
        tot2, per2, r2 = timed_rounds(ctx3, co2, max(args.steps, 10), r2, 1, torch.cuda.ExternalStream(ctx3.stream))
        k2 = max(args.steps, 10)
        c2 = {"workload": "C2 (BASELINE configs[1]): 100 CIFAR-shaped clients, log-normal sizes 10-2000, E=1, B=32",
              "value": len(co2) * k2 / (tot2 * 1e-3), "unit": UNIT, "ms_per_step": tot2 / k2,
              "step_ms": {"median": statistics.median(per2), "p10": pct(per2, 10), "p90": pct(per2, 90)},
              "steps": k2}
        ctx3.close()
        del x2d, y2d
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(wl, sizes, x, y, theta, args.cpu_max_client)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None,
                "step_ms": {"median": statistics.median(per_step), "p10": pct(per_step, 10),
                            "p90": pct(per_step, 90), "max_over_ranks": True},
                # speech and LSTM run FP32 SIMT kernels; CNN GEMMs TF32
                # logreg and math = 1 run FP32 CUDA-core kernels; the CNNs' and the LSTM's GEMMs run
                # on tcgen05 with TF32 operands (the LSTM recurrences stay FP32, R15)
                "dtype": "f32" if (args.math == 1 or wl.model == "logreg") else "tf32",
                "precision_note": ("FP32 CUDA-core kernels; fp64 FedAvg accumulation" if (args.math == 1 or
                                   wl.model == "logreg") else
                                   "tensor-core GEMM operands tf32, fp32 accumulate; fp32 master weights, SGD, "
                                   "softmax-CE" + ("; LSTM recurrences fp32" if wl.model == "lstm" else "") +
                                   "; fp64 FedAvg accumulation"),
                "data": "synthetic (seeded, SURVEY §8d laws), device-resident",
                "config": run_config(wl, desc, cohort, sizes, world, args.agg),
                "round_stats": {k: st[k] for k in ["round_ms", "round_ms_max", "place_ms", "stage_ms", "train_ms",
                                                   "train_end_ms_min", "train_end_ms_max", "timedelta_ms",
                                                   "agg_ms", "allreduce_ms", "waves", "steps_local",
                                                   "clients_local", "kernels", "xfer_bytes", "sm_count"]},
                "kernels": kernel_table(kstats, args.math),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "c2": c2,
                "gpu_launches": int(st["kernels"]) * args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
