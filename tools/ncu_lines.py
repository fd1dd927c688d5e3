"""Summarise an ncu report per CUDA source line (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top_n]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    path = None
    hdr = None
    lines = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            execd = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        stalls = sorted(((int(v or 0), k) for k, v in d.items()
                         if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()),
                        reverse=True)[:2]
        lines.append((samples, execd, f"{path}:{r[0]}", r[1].strip()[:70], stalls))
    tot = sum(x[0] for x in lines) or 1
    tote = sum(x[1] for x in lines) or 1
    print(f"total samples {tot}, instructions {tote}")
    for s, e, loc, src, st in sorted(lines, key=lambda x: x[1 if __import__("os").environ.get("BY_INST") else 0], reverse=True)[:top]:
        print(f"{100*s/tot:5.1f}% {100*e/tote:5.1f}%i {loc:22s} {src:70s} {[(k[6:], v) for v, k in st]}")


if __name__ == "__main__":
    main()
