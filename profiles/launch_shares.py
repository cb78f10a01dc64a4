"""Per-kernel shares of the timed steps in an ncu launch list (gpu__time_duration.sum, cold
cache, serialised): compare the SHARES with bench.py's CUDA-event kernel_ms, not the absolutes.

    python profiles/launch_shares.py gpurun_out/rNN_launches.csv > profiles/rNN_launch_shares.txt
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("<")[0].split("(")[0].split()[-1].split("::")[-1]
        rows.append((short, name, float(r["Metric Value"].replace(",", ""))))
    ours = {"fwd_kernel", "bwd_kernel", "loss_kernel", "reduce_kernel", "adam_kernel",
            "validate_kernel", "fit_kernel", "vl_fwd_kernel", "vl_bwd_kernel", "adam_free_kernel",
            "state_from_obs_kernel", "fit_long_kernel"}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for short, name, ns in rows:
        tot[short] += ns
        cnt[short] += 1
    print(f"{len(rows)} launches in {path}")
    print(f"{'kernel':24s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s}  library")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k:24s} {cnt[k]:8d} {tot[k] / 1e6:10.3f} {tot[k] / cnt[k] / 1e3:10.1f}  "
              f"{'ours' if k in ours else 'torch/other'}")
    # the fused iteration's kernels in the bench's timed-step pattern: fwd_kernel<..., 1, ...>
    fused = [(s, n, t) for s, n, t in rows if s in ("fwd_kernel", "bwd_kernel") and
             ("true, 4, 1," in n or "1, 4, 1" in n or ", 1, 4, true, 2>" in n or
              "1, 0, 1, 4, 1" in n)]
    if fused:
        f = sum(t for s, _, t in fused if s == "fwd_kernel")
        b = sum(t for s, _, t in fused if s == "bwd_kernel")
        print(f"fused iteration kernels: fwd {f / 1e6:.3f} ms, bwd {b / 1e6:.3f} ms over "
              f"{len(fused)} launches; shares fwd {f / (f + b):.3f}, bwd {b / (f + b):.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
