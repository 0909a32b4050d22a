#!/usr/bin/env python
"""bench.py — one simulated FedAvg round per step on N B200s (BASELINE.json metric:
client-updates/s and FedAvg round time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C3|...]

Workload: N=1 -> BASELINE configs[1] (C2: 100 CIFAR-shaped
clients, log-normal sizes 10..2000, McMahan CNN, E=1, B=32).  N>1 -> weak scaling: a
cohort of 100·N clients drawn from a 10,000-client population with the same size law
(C2's per-GPU load on every GPU, C3's population), one NCCL allreduce per round.
A step = one whole round (place -> pack -> local SGD of every client -> fused FedAvg
accumulation -> allreduce -> finalize), inputs resident in HBM.  The per-round working
set (client models 100 x 8.6 MB + activations) exceeds the 126 MB L2, so no flush is
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
    if name:
        wl = synth.preset(name)
        if name == "C3":
            return wl, "C3: 1,000 of 10,000 CIFAR-shaped clients, McMahan CNN, E=2, B=32 (strong scaling)", "strong"
        return wl, f"{name}", "weak" if world == 1 else "strong"
    if world == 1:
        return synth.preset("C2"), "C2: 100 CIFAR-shaped clients, log-normal sizes 10-2000, McMahan CNN, E=1, B=32", "weak"
    wl = synth.preset("C3", n_cohort=100 * world, E=1)
    return wl, (f"C2-per-GPU weak scaling: {100 * world} of 10,000 CIFAR-shaped clients (C3 population), "
                f"McMahan CNN, E=1, B=32"), "weak"


def run_config(wl, desc, cohort, sizes, world):
    """The `config` object of both arms' JSON lines (identical for ours and --impl reference)."""
    return {"workload": desc, "clients": int(len(cohort)), "samples": int(sizes.sum()), "B": wl.B, "E": wl.E,
            "lr": wl.lr, "parallelism": f"clients x{world}",
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
    out["traffic"] = ncu_traffic(name)
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
    """dram bytes per launch of this class from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(kernel_class)
    except Exception:
        return None


def cpu_baseline(wl, sizes, x, y, theta, budget_samples, threads=0):
    """The oracle, as it stands, on a bounded random sample of the workload's clients:
    samples/s of local SGD, converted to client-updates/s with the workload's mean
    client size (aggregation cost is negligible next to training on the CPU)."""
    import oracle
    rng = np.random.default_rng(1)
    order = rng.permutation(len(sizes))
    pick, tot = [], 0
    for c in order:
        if tot >= budget_samples:
            break
        pick.append(int(c))
        tot += int(sizes[c])
    pop_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    t0 = time.perf_counter()
    _, used = oracle.train_clients(wl.model, theta, x, y, pop_off, np.array(pick), wl.B, wl.E, wl.lr, threads=threads)
    dt = time.perf_counter() - t0
    samples_per_s = tot * wl.E / dt
    mean_client = float(np.mean(sizes)) * wl.E
    return {"value": samples_per_s / mean_client, "unit": UNIT, "cores": int(used), "kind": "oracle",
            "sample": f"{len(pick)} random clients of the cohort ({tot} samples x E={wl.E}) trained by the fp64 "
                      f"oracle in {dt:.1f} s; client-updates/s = samples/s / mean client size ({mean_client:.1f})",
            "seconds": dt}


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


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args, world, rank):
    """The oracle (the only reference this tier has) on the host cores."""
    if rank != 0:
        return
    wl, desc, scaling = workload(args.gpus, args.config)
    sizes, x, y, cohort = pop_for(wl)
    theta = synth.init_params(wl.model)
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(wl, sizes, x, y, theta, budget_samples=args.ref_samples)
        if i >= args.warmup:
            vals.append(cb)
    v = statistics.median(c["value"] for c in vals)
    ms = len(cohort) / v * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8d laws)",
            "config": run_config(wl, desc, cohort, sizes, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[-1]["cores"], "kind": "oracle",
                             "sample": vals[-1]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--math", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=400)
    ap.add_argument("--ref-samples", type=int, default=200)
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
    uid = None
    if world > 1:
        import torch.distributed as dist
        obj = [fl.fl_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = fl.Config(model=wl.model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, shuffle=wl.shuffle, seed=wl.seed,
                    rank=rank, world_size=world, device=local, nccl_unique_id=uid, math=args.math)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    ctx = fl.fl_round_init(cfg, sizes, xd, yd, theta)
    stream = torch.cuda.ExternalStream(ctx.stream)
    rnd = 0
    for _ in range(args.warmup):
        ctx.fl_round(cohort, round_index=rnd, stats=False)
        rnd += 1
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(list(range(world)) if rank == 0 else [local]) as clk:
        barrier(world)
        torch.cuda.synchronize()
        clk.mark_start()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.fl_round(cohort, round_index=rnd, stats=False)
            rnd += 1
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
        barrier(world)
    ms_total = allmax(e0.elapsed_time(e1), world)
    st = ctx.fl_get_stats()
    # "timedelta workers": slowest minus fastest rank's training time of the last round
    timedelta = allmax(st["train_ms"], world) + allmax(-st["train_ms"], world)
    ms_step = ms_total / args.steps
    value = len(cohort) * args.steps / (ms_total * 1e-3)
    clocks = clk.summary()
    # per-kernel device time of one extra (profiled) round, for the roofline
    ctx.fl_set_profiling(True)
    st_p = ctx.fl_round(cohort, round_index=rnd)
    rnd += 1
    kstats = ctx.fl_get_kernel_stats()
    ctx.fl_set_profiling(False)
    roof = roofline(kstats, args.math, st_p["round_ms"])
    ctx.close()  # the e2e context below needs the memory (C4: ~60 GB of activations per context)
    del xd, yd
    torch.cuda.empty_cache()
    # e2e: the public API with HOST buffers; H2D of this rank's cohort rows and D2H of θ_new per step
    e2e = None
    if not args.no_e2e:
        ctx2 = fl.fl_round_init(cfg if world == 1 else cfg, sizes, x, y, theta, on_device=False)
        for _ in range(2):
            ctx2.fl_place(cohort)
            ctx2.fl_train_clients(0)
            ctx2.fl_aggregate(want_params=True)
        barrier(world)
        t0 = time.perf_counter()
        h2d = 0
        for i in range(args.steps):
            ctx2.fl_place(cohort)
            ctx2.fl_train_clients(i)
            ctx2.fl_aggregate(want_params=True)  # synchronous D2H of θ_new
        t_e2e = allmax((time.perf_counter() - t0) * 1e3, world)
        s2 = ctx2.fl_get_stats()
        e2e = {"value": len(cohort) * args.steps / (t_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(s2["h2d_bytes"]), "d2h_bytes_per_step": int(4 * ctx2.P),
               "ms_per_step": t_e2e / args.steps, "timer": "host wall clock around the public API calls"}
        ctx2.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(wl, sizes, x, y, theta, args.cpu_samples)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None,
                # speech and LSTM run FP32 SIMT kernels; CNN/logreg GEMMs TF32
                "dtype": "f32" if (args.math == 1 or wl.model in ("lstm", "speech")) else "tf32",
                "precision_note": "tensor-core GEMM operands tf32, fp32 accumulate; fp32 master weights, SGD, "
                                  "softmax-CE; fp64 FedAvg accumulation",
                "data": "synthetic (seeded, SURVEY §8d laws), device-resident",
                "config": run_config(wl, desc, cohort, sizes, world),
                "round_stats": dict({k: st[k] for k in ["round_ms", "place_ms", "stage_ms", "train_ms", "agg_ms",
                                                        "allreduce_ms", "waves", "steps_local", "kernels"]},
                                    timedelta_ms=timedelta),
                "kernels": kernel_table(kstats, args.math),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "gpu_launches": int(st["kernels"]) * args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
