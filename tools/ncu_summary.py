"""Per-kernel summary of an ncu --set full report (for profiles/): duration, SM / tensor-pipe
activity, DRAM bytes, L2 throughput, achieved occupancy.
usage: python tools/ncu_summary.py report.ncu-rep|raw.csv > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__grid_size", "launch__block_size"]
# tcgen05 (UTCHMMA) activity: math ops of the bf16 tensor path, and the A-operand shared-memory wavefronts
TC = ["sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum",
      "l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum",
      "l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_b_scope_1cta.sum"]
EXTRA = ",".join(TC + ["sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed"])


def main(rep):
    if rep.endswith(".csv"):  # an exported raw page (tools/ncu_deep.sh)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {rep}: ncu --set full (--clock-control none), one line per profiled launch")
    print("# time_us  sm%  tensor_pipe%(hmma/utchmma subpipe)  dram_rd  dram_wr  dram%  l2%  warps%  grid x block"
          "  | tcgen05 bf16 TFLOP/s by counter (2 x UTCHMMA ops / time)  A-fetch smem wavefronts  kernel")
    for r in rows[2:]:
        g = {k: r[h.index(k)] if k in h else "?" for k in M + TC}
        u = {k: units[h.index(k)] if k in h else "" for k in M + TC}
        name = r[h.index("Kernel Name")].split("(")[0][:110]
        try:
            t_s = float(g[M[0]].replace(",", "")) * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u[M[0]], 1e-9)
            ops = float(g[TC[0]].replace(",", ""))
            tf = f"{2 * ops / t_s / 1e12:8.1f}" if ops > 0 else "       -"
        except (ValueError, ZeroDivisionError):
            tf = "       ?"
        print(f"{g[M[0]]:>8} {g[M[1]]:>6} {g[M[2]]:>6} {g[M[3]]:>9}{u[M[3]][:2]} {g[M[4]]:>9}{u[M[4]][:2]} "
              f"{g[M[5]]:>6} {g[M[6]]:>6} {g[M[7]]:>6} {g[M[8]]:>5}x{g[M[9]]:<4} | {tf} {g[TC[1]]:>10}  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
