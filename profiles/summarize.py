"""Summarise an ncu report (.ncu-rep) into the metrics DESIGN.md / bench.py cite.

    python profiles/summarize.py gpurun_out/prof_bwd.ncu-rep > profiles/rNN_bwd_summary.txt
"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__waves_per_multiprocessor",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"kernel: {vals[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:60s} {vals[i]:>20s} {u[i]}")
        rd = float(vals[h.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(vals[h.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[u[h.index("dram__bytes_read.sum")]]
        wr *= scale[u[h.index("dram__bytes_write.sum")]]
        print(f"  traffic (dram read + write) bytes/launch            {rd + wr:20.4e}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and \
                    k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(vals[i].replace(",", "")), k[34:-23]))
                except ValueError:
                    pass
        print("  warp stall reasons (warps per issue-active cycle, >= 0.05):")
        for v, k in sorted(stalls, reverse=True):
            if v >= 0.05:
                print(f"    {k:28s} {v:6.3f}")
    # stall reasons: top SASS lines by warp-stall samples
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                          "sass"))))
    hh = src[1]
    si, ie, ws = hh.index("Source"), hh.index("Instructions Executed"), \
        hh.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in src[2:]:
        try:
            lines.append((r[si].strip(), int(r[ie]), int(r[ws])))
        except (ValueError, IndexError):
            pass
    tot_s = sum(x[2] for x in lines) or 1
    print(f"  SASS lines: {len(lines)}; warp-stall samples: {tot_s}")
    ops = Counter()
    for s, e, _ in lines:
        tok = s.split()
        if not tok:
            continue
        op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
        ops[op.split(".")[0]] += e
    tot_i = sum(ops.values()) or 1
    print("  executed warp-instructions by opcode (share):")
    for op, n in ops.most_common(16):
        print(f"    {op:10s} {n / tot_i:6.3f}")
    print("  top stall lines (samples share, executed, SASS):")
    for s, e, w in sorted(lines, key=lambda x: -x[2])[:12]:
        print(f"    {w / tot_s:6.3f} {e:>12d}  {s[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
