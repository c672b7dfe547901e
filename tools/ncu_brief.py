"""Key metrics of a one-kernel ncu report (raw page, CSV): time, DRAM,
occupancy, pipes and the top stall reasons."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(units, val)))
    print(path, d.get("Kernel Name", ("", ""))[1][:60])
    for k in KEYS:
        if k in d:
            print(f"  {k:75s} {d[k][1]:>14s} {d[k][0]}")
    st = [(h, float(v)) for h, (u, v) in d.items()
          if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio") and v]
    st.sort(key=lambda x: -x[1])
    print("  stalls/issue:", ", ".join(f"{h[34:-23]} {v:.2f}" for h, v in st[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
