"""Summarise an ncu report for profiles/ (reads the .ncu-rep with the local ncu CLI).

    python scripts/ncu_summarize.py gpurun_out/prof.ncu-rep profiles/r01_batched.txt [title]

Writes the headline SOL/occupancy numbers, DRAM bytes, pipe utilisation, warp-stall
breakdown and the hottest SASS lines (stall samples) -- the evidence the DESIGN.md
performance notes cite.
"""
import csv
import re
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    lines = [f"# {title}", f"# source: {rep} (ncu --set full --clock-control none --import-source on)", ""]
    det = list(csv.reader(ncu(rep, "--page", "details", "--csv").splitlines()))
    if det:
        hdr = det[0]
        keep = ["Kernel Name", "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput",
                "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
                "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
                "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
                "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
                "L2 Hit Rate"]
        seen = set()
        for row in det[1:]:
            d = dict(zip(hdr, row))
            name = d.get("Metric Name")
            if name in keep and name not in seen:
                seen.add(name)
                lines.append(f"{name:40s} {d.get('Metric Value')} {d.get('Metric Unit')}")
        if det[1:]:
            lines.insert(3, "kernel: " + dict(zip(hdr, det[1])).get("Kernel Name", "?"))
    raw = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    if len(raw) >= 3:
        lines.append("")
        pat = re.compile(r"dram__bytes_(read|write)\.sum$|sm__inst_executed_pipe_(alu|fma|lsu|uniform|xu|tma)"
                         r"\.avg\.pct_of_peak_sustained_active$|smsp__average_warps_issue_stalled_"
                         r"(long_scoreboard|short_scoreboard|barrier|wait|math_pipe_throttle|not_selected|"
                         r"dispatch_stall|mio_throttle|selected)_per_issue_active\.ratio$|"
                         r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_(ld|st|atom)\.sum$")
        for h, u, v in zip(raw[0], raw[1], raw[2]):
            if pat.search(h):
                lines.append(f"{h:82s} {v} {u}")
    src = list(csv.reader(ncu(rep, "--page", "source", "--csv", "--print-source", "sass").splitlines()))
    if len(src) > 2:
        hdr = src[1]
        ix = {h: i for i, h in enumerate(hdr)}

        def g(r, k):
            try:
                return int(r[ix[k]] or 0)
            except (KeyError, ValueError, IndexError):
                return 0
        data = src[2:]
        tot = sum(g(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
        lines += ["", f"hottest SASS lines (share of {tot} warp-stall samples):"]
        for r in sorted(data, key=lambda r: -g(r, "Warp Stall Sampling (All Samples)"))[:25]:
            smp = g(r, "Warp Stall Sampling (All Samples)")
            lines.append(f"  {100.0 * smp / tot:5.1f}%  exec {g(r, 'Instructions Executed'):>10d}  "
                         f"{r[ix['Source']].strip()[:70]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
