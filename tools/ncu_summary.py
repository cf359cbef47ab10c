"""Summarise ncu artefacts into profiles/: the launch list (per-kernel device
time and share of the step) and the key metrics of a --set full capture.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN/launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rNN/<kernel>.md
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0][:80]
            ns = float(d["Metric Value"])
            n, t = agg.get(name, (0, 0.0))
            agg[name] = (n + 1, t + ns)
    total = sum(t for _, t in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{name}` | {n} | {t / 1e6:.3f} | {100 * t / total:.1f}% |")
    print("\n".join(out))


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## {d.get('Kernel Name', '?')[:120]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        print()
        stalls = []
        for k, v in d.items():
            if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        if stalls:
            print("warp stall reasons (cycles per issued instruction): " +
                  ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]) + "\n")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2 and "Source" in srows[1]:
        h = srows[1]
        iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in srows[2:]:
            try:
                data.append((int(r[iW]), r[iS].strip()))
            except (ValueError, IndexError):
                pass
        tot = sum(w for w, _ in data) or 1
        print("hottest SASS (share of warp stall samples):\n```")
        for w, line in sorted(data, reverse=True)[:12]:
            print(f"{100 * w / tot:5.1f}%  {line[:100]}")
        print("```")
    det = subprocess.run(["ncu", "-i", path, "--page", "details"], capture_output=True, text=True).stdout
    print("```")
    for line in det.splitlines():
        if any(s in line for s in ("Duration", "Registers Per", "Achieved Occupancy", "Theoretical Occupancy",
                                   "Issue Slots Busy", "Eligible Warps", "Warp Cycles Per Issued", "L1/TEX Hit",
                                   "L2 Hit", "Block Limit", "Executed Ipc")):
            print(line.rstrip())
    print("```")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
