"""Dynamic opcode histogram of one kernel from an ncu report (SASS view):
warp-level instructions executed per opcode, and the top SASS instructions.

    python tools/ncu_opcodes.py gpurun_out/prof.ncu-rep [top_n]
"""
import csv
import collections
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    ops = collections.Counter()
    total = 0
    for r in rows:
        if not r:
            continue
        if "Source" in r and "Instructions Executed" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            n = int(d["Instructions Executed"] or 0)
        except ValueError:
            continue
        toks = d["Source"].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += n
        total += n
    print(f"warp instructions executed: {total}")
    for op, n in ops.most_common(top):
        print(f"  {op:12s} {n:12d}  {100.0 * n / max(total, 1):5.1f}%")


if __name__ == "__main__":
    main()
