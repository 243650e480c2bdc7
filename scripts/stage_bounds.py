"""Stage-bound table from an ncu --page raw --csv export: per kernel the duration, DRAM bytes
and their rate against the measured HBM peak, issue activity, the busiest pipe and the top
pc-sampled stall reasons: python scripts/stage_bounds.py raw.csv [hbm_gbs]"""
import csv
import sys


def main(path, hbm=6551.4):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]

    def col(r, k):
        try:
            v = float(r[hdr.index(k)].replace(",", ""))
        except (ValueError, IndexError):
            return 0.0
        u = units[hdr.index(k)]
        return v * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}.get(u, 1.0)

    pipes = [h for h in hdr if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active")]
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    print(f"{'kernel':34s} {'us':>8s} {'DRAM MB':>8s} {'HBM %':>6s} {'issue%':>6s} {'warps%':>6s}  busiest pipe     top stalls (share of samples)")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace("void ", "").replace("vegs::", "").split("(")[0][:34]
        us = col(r, "gpu__time_duration.sum")
        dram = col(r, "dram__bytes_read.sum") + col(r, "dram__bytes_write.sum")
        frac = dram / (us * 1e-6) / (hbm * 1e9) * 100 if us else 0.0
        pipe = max(pipes, key=lambda h: col(r, h))
        tot = sum(col(r, h) for h in stalls) or 1.0
        top = sorted(((col(r, h) / tot, h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stalls),
                     reverse=True)[:3]
        print(f"{name:34s} {us:8.1f} {dram / 1e6:8.1f} {frac:6.1f} {col(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{col(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f}  "
              f"{pipe.replace('sm__inst_executed_pipe_', '').split('.')[0]:5s} {col(r, pipe):5.1f}%  "
              + ", ".join(f"{b} {100 * a:.0f}%" for a, b in top))


if __name__ == "__main__":
    main(sys.argv[1], *(float(x) for x in sys.argv[2:]))
