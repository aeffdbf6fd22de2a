#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/ (runs here, without a GPU).

    python tools/ncu_summary.py launches gpurun_out/r1b_launches.csv      # per-kernel share of a step
    python tools/ncu_summary.py report gpurun_out/r1b_prof_expert_fwd.ncu-rep [algorithmic_flops] [algorithmic_bytes]
    python tools/ncu_summary.py traffic <workload> gpurun_out/<tag>_prof_*.ncu-rep   # -> profiles/ncu_traffic.json
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0].replace("void ", "").strip()
        tot[name] += v * scale
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.1f} {100 * v / s:6.1f}%")
    print(f"{'total':70s} {sum(cnt.values()):8d} {s:10.1f}")


def _rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (vals[i], units[i]) for i, h in enumerate(hdr)} for vals in rows[2:] if len(vals) == len(hdr)]


def report(path, flops=None, nbytes=None):
    """Key metrics of every kernel launch captured in one report."""
    for d in _rows(path):
        print("kernel:", d.get("Kernel Name", ("?",))[0][:160])
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k][0]} {d[k][1]}")
        t = float(d["gpu__time_duration.sum"][0]) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(d["gpu__time_duration.sum"][1], 1)
        if flops:
            print(f"  algorithmic {float(flops) / 1e9:.1f} GFLOP -> {float(flops) / t / 1e12:.1f} TFLOP/s (cold, serialised)")
        if nbytes:
            print(f"  algorithmic {float(nbytes) / 1e6:.1f} MB -> {float(nbytes) / t / 1e9:.1f} GB/s")


SPAN_OF = {"expert_bwd_h": "B5_expert_bwd_dx", "expert_dw_kernel": "B5_expert_bwd_dw",
           # the opt-in fused backward (MHL_FLAG_BWD_FUSED) runs under the same span name; its traffic
           # is keyed separately and bench.py picks it when the dX GEMM span is absent
           "expert_bwd_fused": "B5_expert_bwd_dx@fused",
           "expert_fwd_sm100": "F5_expert_fwd", "expert_dx_gemm": "B5_expert_dx_gemm",
           "router_sm100": "F3_router_topk", "router_bwd_sm100": "B3_router_bwd", "scatter_kernel": "F4_cluster",
           # the same combine kernel serves F6 and then B6 within one step (capture order)
           "combine_kernel": ("F6_combine", "B6_combine_bwd")}


def traffic(workload, paths):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of each captured kernel,
    keyed by the bench span it is timed under -> profiles/ncu_traffic.json (read by bench.py)."""
    import json
    import os
    out = {"_workload": workload, "_source": "ncu --set full --clock-control none, one launch each"}
    seen = {}
    for path in paths:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for d in _rows(path):
            b = sum(float(d[k][0].replace(",", "")) * scale.get(d[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            name = d["Kernel Name"][0]
            key = next((k for k in SPAN_OF if k in name), None)
            if key is None:
                continue
            span = SPAN_OF[key]
            if isinstance(span, tuple):
                span = span[min(seen.get(key, 0), len(span) - 1)]
            seen[key] = seen.get(key, 0) + 1
            if span not in out:
                out[span] = {"kernel": name.split("(")[0][:120], "dram_bytes_per_launch": b,
                             "report": os.path.basename(path)}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    json.dump(out, open(os.path.join(root, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], *(sys.argv[3:5]))
