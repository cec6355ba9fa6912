"""Key metrics of an ncu --set full report (read with ncu -i, no GPU)."""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed_pipe_fp64.sum", "lts__t_sector_hit_rate.pct",
       "launch__grid_size", "launch__block_size"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        lines.append(f"kernel {name}")
        for k in RAW:
            if k in h:
                i = h.index(k)
                lines.append(f"  {k:60s} {r[i]:>16s} {units[i]}")
        try:
            rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * mult[units[h.index("dram__bytes_read.sum")]] + wr * mult[units[h.index("dram__bytes_write.sum")]]
            lines.append(f"  dram traffic (read+write) per launch: {tot / 1e6:.1f} MB")
        except Exception:
            pass
    return "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"# {rep}")
        print(summary(rep))
