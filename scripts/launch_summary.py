"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import io
import re
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def short(name):
    if "Onesweep" in name:
        return "cub::DeviceRadixSortOnesweep"
    for k in ("Histogram", "ExclusiveSum", "SingleTile", "DeviceScanInit", "DeviceScanKernel", "DeviceCompact"):
        if k in name:
            return "cub::" + k
    s = re.sub(r"\(.*", "", name).replace("void ", "")
    return re.sub(r"<.*", "", s)


def main(path):
    rows = load(path)
    agg = collections.OrderedDict()
    for r in rows:
        a = agg.setdefault(short(r["Kernel Name"]), [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(rows)}  total {tot:.1f} us (serialised, cold-cache ncu replay)")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:52s} {n:5d} {us:10.1f} us {100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
