"""Summarize ncu outputs from gpurun_out/ into profiles/ (committed evidence).

    python tools/summarize_ncu.py TAG

Reads gpurun_out/launches_TAG.csv (gpu__time_duration per launch) and
gpurun_out/prof_{gemm,gemv}_TAG.ncu-rep (--set full), writes
profiles/TAG_launches.csv (copy), profiles/TAG_summary.md and updates
profiles/traffic.json with the per-launch DRAM bytes of each captured kernel.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "HMMA pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "SMEM LSU wavefronts %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw_metrics_all(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        res.append({h: (vals[i], units[i]) for i, h in enumerate(hdr) if i < len(vals)})
    return res


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, h in enumerate(hdr):
        d[h] = (vals[i], units[i])
    return d


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * mult


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary — {tag}", ""]
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    reps = []
    for name in ("gemm", "gemv", "aux"):
        rep = os.path.join(OUT, f"prof_{name}_{tag}.ncu-rep")
        if os.path.exists(rep):
            reps += [(name, d) for d in raw_metrics_all(rep)]
    for name, d in reps:
        kname = d.get("Kernel Name", ("?", ""))[0]
        lines += [f"## {name}: `{kname}`", "", "| metric | value | unit |", "|---|---|---|"]
        for key, label in KEYS:
            if key in d:
                lines.append(f"| {label} (`{key}`) | {d[key][0]} | {d[key][1]} |")
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            tb = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
            key = kname.split("<")[0].split("(")[0].replace("void ", "").replace("fn::", "").strip()
            traffic[key] = tb
            lines.append(f"| DRAM traffic per launch (read+write) | {tb:.4g} | byte |")
        lines.append("")
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(PROF, f"{tag}_launches.csv"))
        rows = [r for r in csv.reader(open(lpath)) if len(r) > 10]
        hdr = rows[0]
        try:
            ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
            agg = {}
            for r in rows[1:]:
                k = r[ik].split("(")[0]
                agg.setdefault(k, []).append(float(r[iv].replace(",", "")))
            tot = sum(sum(v) for v in agg.values())
            lines += ["## launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
                      "| kernel | launches | total us | share |", "|---|---|---|---|"]
            for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
                lines.append(f"| `{k[:80]}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
        except ValueError:
            pass
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if reps:
        traffic["source"] = f"profiles/{tag}_summary.md (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
