"""Print registers / spills / smem per kernel from the last build's ptxas -v log."""
import os
import re
import subprocess

LOG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build.log")


def report(log=LOG):
    cur = None
    out = []
    names = {}
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
        if m and cur:
            names[cur] = {"stack": int(m.group(1)), "spill": int(m.group(2))}
        m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line) or \
            re.search(r"Used (\d+) registers", line)
        if m and cur:
            d = names.setdefault(cur, {})
            d["regs"] = int(m.group(1))
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.split("\n")
    for (k, v), d in zip(names.items(), dem):
        out.append(f"{v.get('regs', '?'):>4} regs  spill {v.get('spill', 0):>3}  {d}")
    return "\n".join(sorted(out, key=lambda x: x.split("  ")[-1]))


if __name__ == "__main__":
    print(report())
