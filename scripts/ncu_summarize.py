"""Summarise the gpu_evidence.sh ncu outputs into profiles/<round>/ and profiles/ncu_traffic.json.

usage: python scripts/ncu_summarize.py gpurun_out profiles/r01
  launches.csv -> <out>/launches_c2_round.csv (copy) + per-kernel table (markdown, stdout)
  traffic.csv  -> profiles/ncu_traffic.json: mean DRAM bytes (read + write) per launch of each
                  bench kernel class (bench.py `roofline.traffic`), and a per-class table
"""
import collections
import csv
import json
import os
import re
import shutil
import sys

CLASS = [  # (kernel-name regex, bench class); first match wins
    (r"k_fc1_bwd_tc", "fc1_dw_sgd"), (r"k_fc1_dw_tc", "fc1_dw_sgd"), (r"k_fc1_dx_tc", "fc1_dx"),
    (r"k_fc1_fwd", "fc1_fwd"), (r"k_conv5_tc<64", "conv2_fwd"), (r"k_conv5_tc<32", "conv2_dx"),
    (r"k_conv2_dw_tc", "conv2_dw"), (r"k_dw2_reduce_sgd|k_dw_reduce2_sgd", "conv2_dw_reduce_sgd"), (r"k_conv1_dw_tc", "conv1_dw"),
    (r"k_dw_reduce_sgd", "conv1_dw_reduce_sgd"), (r"k_conv1_fwd_tc", "conv1_fwd"), (r"k_head", "head_fc2_ce"),
    (r"k_pack|k_c1wt|k_gather", "pack"), (r"k_fedavg|k_finalize", "fedavg_accum"),
]
PER_WAVE = {"fc1_dw_sgd", "fc1_dx", "fc1_fwd", "conv2_fwd", "conv2_dx", "conv2_dw", "conv2_dw_reduce_sgd", "conv1_dw",
            "conv1_dw_reduce_sgd", "conv1_fwd", "head_fc2_ce"}


def rows(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def kclass(name):
    for rx, c in CLASS:
        if re.search(rx, name):
            return c
    return None


def short(name):
    m = re.search(r"(k_[A-Za-z0-9_]+(<[^>]*>)?)", name)
    return m.group(1) if m else name[:40]


def main():
    src, out = sys.argv[1], sys.argv[2]
    os.makedirs(out, exist_ok=True)
    # launch list
    L = rows(os.path.join(src, "launches.csv"))
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(out, "launches_bench_round.csv"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in L:
        us = float(d["Metric Value"].replace(",", "")) / (1e3 if d["Metric Unit"] == "ns" else 1.0)
        k = short(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | device ms | mean us | share |\n|---|---|---|---|---|")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {us / 1e3:.3f} | {us / n:.1f} | {100 * us / tot:.1f}% |")
    print(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e3:.3f} | | |\n")
    # traffic
    T = rows(os.path.join(src, "traffic.csv"))
    per = collections.defaultdict(lambda: {"read": 0.0, "write": 0.0, "us": 0.0, "ids": set()})
    waves = set()
    for d in T:
        c = kclass(d["Kernel Name"])
        if c is None:
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
                 "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1.0)
        p = per[c]
        p["ids"].add(d["ID"])
        if d["Metric Name"] == "dram__bytes_read.sum":
            p["read"] += v * scale
        elif d["Metric Name"] == "dram__bytes_write.sum":
            p["write"] += v * scale
        elif d["Metric Name"] == "gpu__time_duration.sum":
            p["us"] += v * scale
    n_waves = max(len(per[c]["ids"]) for c in ("conv2_dx", "conv2_fwd") if c in per)
    res = {}
    print("| class | kernel launches | class launches | DRAM read MB | DRAM write MB | bytes / class launch |\n"
          "|---|---|---|---|---|---|")
    for c, p in sorted(per.items(), key=lambda kv: -(kv[1]["read"] + kv[1]["write"])):
        nl = n_waves if c in PER_WAVE else 1
        b = (p["read"] + p["write"]) / nl
        res[c] = b
        print(f"| {c} | {len(p['ids'])} | {nl} | {p['read'] / 1e6:.1f} | {p['write'] / 1e6:.1f} | {b / 1e6:.3f} MB |")
    res["_note"] = ("mean dram__bytes_read.sum + dram__bytes_write.sum per bench kernel-class launch (one per wave "
                    "for per-wave classes), ncu over one timed round of bench.py's default workload (C3); "
                    "scripts/gpu_evidence.sh")
    res["_source"] = f"{out}: ncu dram__bytes_read.sum + dram__bytes_write.sum over one timed bench round"
    json.dump(res, open(os.path.join(os.path.dirname(out.rstrip("/")), "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
