"""Stall samples by opcode and the hottest SASS lines from an ncu source export:
ncu -i rep --page source --csv --print-source sass --kernel-name regex:K > f.csv;
python scripts/sass_stalls.py f.csv [top]"""
import csv
import sys
from collections import Counter


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_src, i_s, i_e = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[i_e].strip().isdigit()]
    tot = sum(int(r[i_s]) for r in body)
    c, ce = Counter(), Counter()
    for r in body:
        parts = r[i_src].split()
        op = (parts[1] if parts[0].startswith("@") else parts[0]).split(".")[0]
        c[op] += int(r[i_s])
        ce[op] += int(r[i_e])
    print("samples", tot, "instructions", sum(ce.values()))
    for op, v in c.most_common(15):
        print(f"  {op:10s} {v:7d} {100 * v / tot:5.1f}%  executed {ce[op]}")
    for r in sorted(body, key=lambda r: -int(r[i_s]))[:int(top)]:
        print(f"  {r[0][-5:]} {int(r[i_s]):6d}  {r[i_src][:80]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
