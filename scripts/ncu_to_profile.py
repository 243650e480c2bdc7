"""Extract the per-launch figures bench.py cites from an ncu --set full capture of the two
compositing kernels: python scripts/ncu_to_profile.py gpurun_out/prof_composite.ncu-rep
-> profiles/ncu_composite.json (DRAM bytes, executed warp instructions, issue activity)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

NCU = "/usr/local/cuda/bin/ncu"
NAMES = {"composite_fwd2_kernel": "vegs_composite_forward", "composite_bwd4_kernel": "vegs_composite_backward"}


def main(rep, out="profiles/ncu_composite.json", suffix="", instances=None, merge=False):
    """suffix: appended to the keys (e.g. "_c3" for the config-3 render capture);
    instances: the capture's tile-instance count (bench scales per-launch figures by it);
    merge: update an existing json instead of replacing it."""
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]

    def val(r, k):
        return float(r[hdr.index(k)].replace(",", ""))

    res = {}
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")]
        key = next((v for k, v in NAMES.items() if k in kname), None)
        if key is None:
            continue
        res[key + suffix] = {
            "dram_bytes": val(r, "dram__bytes_read.sum") * 1e6 + val(r, "dram__bytes_write.sum") * 1e6
            if "Mbyte" in rows[1][hdr.index("dram__bytes_read.sum")] else
            val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
            "warp_instructions": val(r, "smsp__inst_executed.sum"),
            "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "ncu_duration_us": val(r, "gpu__time_duration.sum") * (1e3 if rows[1][hdr.index("gpu__time_duration.sum")] == "ms" else 1.0),
            "registers": val(r, "launch__registers_per_thread"),
        }
        if instances:
            res[key + suffix]["instances"] = float(instances)
    src = f"ncu --set full --clock-control none ({Path(rep).name}); per launch"
    if merge and Path(out).exists():
        old = json.loads(Path(out).read_text())
        old.update({k: v for k, v in res.items()})
        old["_source" + suffix] = src
        res = old
    else:
        res["_source" + suffix] = src
    Path(out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out", default="profiles/ncu_composite.json")
    ap.add_argument("--suffix", default="")
    ap.add_argument("--instances", type=float, default=None)
    ap.add_argument("--merge", action="store_true")
    a = ap.parse_args()
    main(a.rep, a.out, a.suffix, a.instances, a.merge)
