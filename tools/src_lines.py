"""Per-source-line share of executed warp-instructions and stall samples of one kernel, from
`ncu -i rep --page source --csv -k <kernel> --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    his = [i for i, r in enumerate(rows) if "Instructions Executed" in r]
    res = []
    for bi, h in enumerate(his):
        hdr = rows[h]
        ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        end = his[bi + 1] - 1 if bi + 1 < len(his) else len(rows)
        for r in rows[h + 1:end]:
            if len(r) > ii and r[0]:
                try:
                    n, st = float(r[ii].replace(",", "")), float(r[si].replace(",", "") or 0)
                except ValueError:
                    continue
                res.append((n, st, r[0], r[1][:120]))
    tot = sum(x[0] for x in res) or 1
    tst = sum(x[1] for x in res) or 1
    res.sort(reverse=True)
    for n, st, ln, s in res[:top]:
        print(f"{100 * n / tot:5.1f}% stall{100 * st / tst:5.1f}%  L{ln}: {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
