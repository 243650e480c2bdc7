"""Per-basic-block instruction counts from an ncu source page (SASS), to see where a
kernel's issued instructions go.  usage: ncu_blocks.py report.ncu-rep kernel_regex"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
at = hdr.index("Avg. Threads Executed")
data = [r for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot = sum(int(r[ie]) for r in data)
print(f"total warp instructions {tot}")
blocks, cur = [], None
for i, r in enumerate(data):
    n = int(r[ie])
    op = r[src].strip().split()
    op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")).split(".")[0]
    if cur and cur[1] == n:
        cur[2] += 1
        cur[3].append(op)
    else:
        cur = [i, n, 1, [op], r[at]]
        blocks.append(cur)
for b in blocks:
    if b[1] * b[2] > tot * 0.01:
        ops = {}
        for o in b[3]:
            ops[o] = ops.get(o, 0) + 1
        desc = " ".join(f"{k}x{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1]))[:100]
        print(f"@{b[0]:4d} n={b[1]:10d} len={b[2]:3d} {100 * b[1] * b[2] / tot:5.1f}% thr={b[4]:>5s}  {desc}")
