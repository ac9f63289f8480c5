"""Per-kernel summary of an ncu --set full report (for profiles/): duration, SM / tensor-pipe
activity, DRAM bytes, L2 throughput, achieved occupancy.
usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__grid_size", "launch__block_size"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {rep}: ncu --set full (--clock-control none), one line per profiled launch")
    print("# time_us  sm%  tensor_pipe%  dram_rd  dram_wr  dram%  l2%  warps%  grid x block  kernel")
    for r in rows[2:]:
        g = {k: r[h.index(k)] if k in h else "?" for k in M}
        u = {k: units[h.index(k)] if k in h else "" for k in M}
        name = r[h.index("Kernel Name")].split("(")[0][:110]
        print(f"{g[M[0]]:>8} {g[M[1]]:>6} {g[M[2]]:>6} {g[M[3]]:>9}{u[M[3]][:2]} {g[M[4]]:>9}{u[M[4]][:2]} "
              f"{g[M[5]]:>6} {g[M[6]]:>6} {g[M[7]]:>6} {g[M[8]]:>5}x{g[M[9]]:<4} {name}")


if __name__ == "__main__":
    main(sys.argv[1])
