"""Summarise an ncu --set full report: headline metrics and pipe utilisation per kernel."""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:90])
        for i, h in enumerate(hdr):
            pipe = h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active")
            if h in KEYS or pipe:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if pipe and v < 1.0:
                    continue
                print(f"   {h:70s} {v:16.3f} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or (
                    h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct")):
                try:
                    stalls.append((float(r[i].replace(",", "")), h))
                except ValueError:
                    pass
        for v, h in sorted(stalls, reverse=True)[:8]:
            print(f"   stall {h:64s} {v:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
