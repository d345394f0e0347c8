"""Warp-state breakdown of one ncu --set full --import-source capture, by warp role.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [kernel-regex] > profiles/<tag>_ncu.md

Splits the SASS of a warp-specialised kernel at its USETMAXREG instructions
(control warps / elementwise warps / drain warps of attn_bwd_tc_kernel), sums the
warp-stall samples per role and reason, lists the hottest instructions, and
prints the pipe utilisations of the raw page."""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum"]


KFILTER = []


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *KFILTER, *args, "--csv"], capture_output=True, text=True,
                          check=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"# ncu --set full: {vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else rep}\n")
    print("| metric | value |\n|---|---|")
    for m in RAW:
        if m in hdr:
            i = hdr.index(m)
            print(f"| `{m}` | {vals[i]} {units[i]} |")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--print-source", "sass"))))
    hdr, data = rows[1], []
    for r in rows[2:]:  # the first function's block only (a capture of several kernels repeats the header)
        if r == hdr or (r and r[0] == hdr[0]):
            break
        if len(r) == len(hdr):
            data.append(r)
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    cuts = [k for k, r in enumerate(data) if "USETMAXREG" in r[ix["Source"]]] + [len(data)]
    roles = [("prologue", 0, cuts[0])]
    names = ["control (TMA / MMA / TMEM alloc)", "elementwise", "drain"]
    for n, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        roles.append((names[n] if n < len(names) else f"section {n}", a, b))
    num = lambda r, c: int(r[ix[c]] or 0)  # noqa: E731
    print("\n## warp-state samples by role\n\n| role | samples | top reasons |\n|---|---|---|")
    for name, a, b in roles:
        tot = {s: sum(num(r, s) for r in data[a:b]) for s in stalls}
        n = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data[a:b])
        top = ", ".join(f"{k[6:]} {v / max(n, 1):.0%}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:6])
        print(f"| {name} | {n} | {top} |")
    print("\n## hottest instructions (samples, SASS index, dominant reason)\n\n| samples | # | instruction | reason |\n"
          "|---|---|---|---|")
    hot = sorted(range(len(data)), key=lambda k: -num(data[k], "Warp Stall Sampling (All Samples)"))[:25]
    for k in hot:
        r = data[k]
        why = max(stalls, key=lambda s: num(r, s))
        print(f"| {num(r, 'Warp Stall Sampling (All Samples)')} | {k} | `{r[ix['Source']].strip()[:60]}` | {why[6:]} |")


if __name__ == "__main__":
    if len(sys.argv) > 2:
        KFILTER[:] = ["-k", "regex:" + sys.argv[2]]
    main(sys.argv[1])
