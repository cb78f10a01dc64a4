"""Summarise an ncu report (.ncu-rep) into the metrics DESIGN.md / bench.py cite.

    python profiles/summarize.py gpurun_out/prof_bwd.ncu-rep > profiles/rNN_bwd_summary.txt
    python profiles/summarize.py gpurun_out/prof.ncu-rep --json profiles/ncu_metrics.json \
        --units 6e8 --tag fused   # + the per-kernel figures bench.py's roofline reads
"""
import csv
import io
import json
import os
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


def _num(vals, h, u, key):
    if key not in h:
        return None
    i = h.index(key)
    try:
        x = float(vals[i].replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1,
             "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,
             "s": 1e9}.get(u[i], 1)
    return x * scale


def main(rep, json_out=None, units=None, tag=""):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = rows[0], rows[1]
    summary = {}
    for vals in rows[2:]:
        kname = vals[h.index('Kernel Name')]
        print(f"kernel: {kname}")
        short = kname.split("<")[0].split("(")[0].split("::")[-1].split()[-1]
        rec = {
            "kernel": kname, "source": f"{os.path.basename(rep)} ({tag})",
            "duration_ns": _num(vals, h, u, "gpu__time_duration.sum"),
            "dram_bytes": (_num(vals, h, u, "dram__bytes_read.sum") or 0) +
                          (_num(vals, h, u, "dram__bytes_write.sum") or 0),
            "issue_active_pct": _num(vals, h, u,
                                     "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": _num(vals, h, u,
                                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "xu_pipe_pct": _num(vals, h, u,
                                "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": _num(vals, h, u,
                                 "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "dram_pct": _num(vals, h, u, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers": _num(vals, h, u, "launch__registers_per_thread"),
            "warp_instr": _num(vals, h, u, "smsp__inst_executed.sum"),
        }
        if units and rec["warp_instr"]:
            rec["warp_instr_per_unit"] = rec["warp_instr"] * 32 / units
            rec["dram_bytes_per_unit"] = rec["dram_bytes"] / units
        summary.setdefault(f"{short}", rec)
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


    if json_out:
        old = {}
        if os.path.exists(json_out):
            with open(json_out) as f:
                old = json.load(f)
        for k, v in summary.items():
            old[f"{tag}_{k}" if tag and tag != "fused" else k] = v
        with open(json_out, "w") as f:
            json.dump(old, f, indent=1)


if __name__ == "__main__":
    a = sys.argv[1:]
    js = a[a.index("--json") + 1] if "--json" in a else None
    un = float(a[a.index("--units") + 1]) if "--units" in a else None
    tg = a[a.index("--tag") + 1] if "--tag" in a else ""
    main(a[0], js, un, tg)
