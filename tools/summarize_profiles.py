"""Summarise gpurun_out/ ncu captures into a committed markdown file.

usage: python tools/summarize_profiles.py <tag>   (reads gpurun_out/launches_<tag>.csv,
       gpurun_out/attn_<tag>.ncu-rep, gpurun_out/gemm_<tag>.ncu-rep, gpurun_out/kbench_<tag>.jsonl)
writes profiles/<tag>_summary.md
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
       "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_wait"]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "second": 1e6, "s": 1e6}.get(unit, 1.0)
        name = d["Kernel Name"].split("(")[0].replace("smo::", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = ["| kernel | launches | total µs | share | avg µs |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k[:70]}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0]:.1f} |")
    out.append(f"| **total (device, serialised under ncu)** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% | |")
    return "\n".join(out)


def raw_table(rep):
    txt = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return "(no data)"
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m in RAW if m in hdr}
    kname = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(m.replace("smsp__pcsamp_warps_issue_stalled_", "stall:") for m in idx) + " |",
           "|---|" + "---|" * len(idx)]
    out.append("| (unit) | " + " | ".join(units[i] for i in idx.values()) + " |")
    for r in rows[2:]:
        out.append(f"| `{r[kname].split('(')[0][-40:]}` | " + " | ".join(r[i] for i in idx.values()) + " |")
    return "\n".join(out)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    go = os.path.join(ROOT, "gpurun_out")
    parts = [f"# ncu summary — {tag}", "",
             "Captured with `tools/gpu.sh {} launches` under gpurun on one B200 (`--clock-control none`).".format(tag),
             "Launch-list times are cold-cache and serialised: compare shares, not absolutes.", ""]
    lp = os.path.join(go, f"launches_{tag}.csv")
    if os.path.exists(lp):
        parts += ["## Launch list of one timed verify step (Mixtral-8x7B, b=32, k=8)", "", launch_table(lp), ""]
    for nm in ("attn", "gemm"):
        rp = os.path.join(go, f"{nm}_{tag}.ncu-rep")
        if os.path.exists(rp):
            parts += [f"## `--set full` capture: {nm}", "", raw_table(rp), ""]
    kp = os.path.join(go, f"kbench_{tag}.jsonl")
    if os.path.exists(kp):
        parts += ["## Kernel microbench (CUDA events, L2 flushed; GB/s vs measured HBM 6555.5 GB/s)", "",
                  "| kernel | shape | µs | GB/s | frac of HBM | TFLOP/s |", "|---|---|---|---|---|---|"]
        for line in open(kp):
            try:
                d = json.loads(line)
            except Exception:
                continue
            shape = ", ".join(f"{k}={d[k]}" for k in ("b", "n", "s", "T", "K", "N", "E") if k in d)
            parts.append(f"| {d['kernel']} | {shape} | {d['us']} | {d['GBs']} | {d['frac']} | {d['TFLOPs']} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    out = os.path.join(ROOT, "profiles", f"{tag}_summary.md")
    open(out, "w").write("\n".join(parts) + "\n")
    print(out)


if __name__ == "__main__":
    main()
