"""Print the SASS of one kernel from an ncu source export (--print-source sass --csv) with
executed-instruction counts and stall samples, keeping only instructions executed at least
`min_frac` of the hottest one: python scripts/sass_hot.py export.csv [min_frac]"""
import csv
import sys


def main(path, min_frac=0.02):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc, iex, ismp = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[iex].isdigit()]
    tot = sum(int(r[iex]) for r in body)
    smp = sum(int(r[ismp]) for r in body)
    top = max(int(r[iex]) for r in body)
    print(f"total inst {tot:.4g}  samples {smp}")
    for r in body:
        ex = int(r[iex])
        if ex >= min_frac * top:
            print(f"{r[ia][-5:]} {ex:>11d} {100.0 * ex / tot:5.2f}% s{int(r[ismp]):>5d}  {r[isrc].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.02)
