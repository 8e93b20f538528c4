"""Executed-instruction mix of a kernel from an ncu capture's SASS source page.

    python tools/sass_mix.py capture.ncu-rep [top]

Aggregates "Instructions Executed" (warp-level) per opcode and prints the
share of each, plus the stall samples per opcode (where the warps wait).
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    rd = csv.reader(io.StringIO("\n".join(lines[1:])))
    header = next(rd)
    ie = header.index("Instructions Executed")
    src = header.index("Source")
    st = header.index("Warp Stall Sampling (All Samples)")
    count, stall = Counter(), Counter()
    for row in rd:
        if len(row) <= ie:
            continue
        op = row[src].strip().split()
        if not op:
            continue
        opcode = op[0] if not op[0].startswith("@") else op[1]
        opcode = opcode.split(".")[0]
        try:
            count[opcode] += int(row[ie] or 0)
            stall[opcode] += int(row[st] or 0)
        except ValueError:
            pass
    total = sum(count.values())
    tst = sum(stall.values()) or 1
    print(f"{'opcode':12s} {'warp insts':>14s} {'share':>7s} {'stall share':>11s}")
    for opc, n in count.most_common(top):
        print(f"{opc:12s} {n:14d} {100 * n / total:6.2f}% {100 * stall[opc] / tst:10.2f}%")
    print(f"{'total':12s} {total:14d}")


if __name__ == "__main__":
    main()
