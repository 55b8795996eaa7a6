"""Instruction mix of one kernel from `ncu --page source --csv --print-source sass` output:
executed warp-instructions and stall samples per opcode (for profiles/ notes)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ii, si, ni = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    stalls = collections.Counter()
    total = 0
    for r in rows[2:]:
        if len(r) <= ii or not r[ii]:
            continue
        try:
            n = float(r[ii].replace(",", ""))
        except ValueError:
            continue
        op = r[si].split()[0] if r[si].split() else "?"
        if op.startswith("@"):
            op = r[si].split()[1]
        op = op.split(".")[0]
        ops[op] += n
        stalls[op] += float(r[ni].replace(",", "") or 0)
        total += n
    st = sum(stalls.values())
    print(f"total warp-instructions {total:.4g}")
    for op, n in ops.most_common(top):
        print(f"  {op:10s} {n:12.4g} {100 * n / total:5.1f}%   stall samples {100 * stalls[op] / max(st, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
