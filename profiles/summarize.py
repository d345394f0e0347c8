"""Summarise ncu captures into profiles/ (run in the dev container):

    python profiles/summarize.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep [tag]

Writes profiles/ncu_summary.json (per-kernel duration, DRAM bytes, pipe
utilisation -- bench.py reads dram_bytes_per_launch from it as `traffic`) and
profiles/<tag>_launches.md (share of each kernel in one step)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

OUT = Path(__file__).resolve().parent
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "ns": 1e-9, "nsecond": 1e-9, "msecond": 1e-3}


def short(name):
    return name.split("(")[0].replace("void ", "").replace("lss::", "").split("<")[0]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1e-9) * 1e3
        tot[short(d["Kernel Name"])] += v
        cnt[short(d["Kernel Name"])] += 1
    T = sum(tot.values())
    lines = [f"# {tag}: ncu launch list (cold-cache, serialised; compare shares)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
    (OUT / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    summary = {"tag": tag, "source": str(rep), "kernels": {}}
    for d in data:
        name = short(d[h.index("Kernel Name")])
        ent = {}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    val = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                ent[key] = val * SCALE.get(units[i], 1) if key in ("duration", "dram_read", "dram_write") else val
        if "dram_read" in ent and "dram_write" in ent:
            ent["dram_bytes_per_launch"] = ent["dram_read"] + ent["dram_write"]
        summary["kernels"][name] = ent
    p = OUT / "ncu_summary.json"
    old = json.loads(p.read_text()) if p.exists() else {"kernels": {}}
    old["kernels"].update(summary["kernels"])
    old["tag"], old["source"] = tag, str(rep)
    p.write_text(json.dumps(old, indent=1) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    tag = sys.argv[3] if len(sys.argv) > 3 else "r01"
    if sys.argv[1] != "-":
        launches(sys.argv[1], tag)
    if len(sys.argv) > 2:
        full(sys.argv[2], tag)
