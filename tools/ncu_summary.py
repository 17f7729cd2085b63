"""Summarise an ncu report: per kernel duration, DRAM bytes, throughputs, occupancy, stalls.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "inst",
    "sm__inst_executed_pipe_fp64.sum": "inst_fp64",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
    # the on-chip bound of the DST passes: shared-memory wavefronts (128 B each,
    # one per SM per clock at peak) and their share of that peak
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pct",
}
STALLS = ["barrier", "wait", "short_scoreboard", "long_scoreboard", "not_selected",
          "no_instruction", "math_pipe_throttle", "dispatch_stall", "mio_throttle"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70]
        vals = []
        for m, short in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{short}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
        print(name)
        print("   " + "  ".join(vals))
        st = []
        for k in STALLS:
            m = f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio"
            if m in hdr and r[hdr.index(m)]:
                st.append(f"{k}={float(r[hdr.index(m)]):.2f}")
        if st:
            print("   stalls/issue: " + "  ".join(st))


if __name__ == "__main__":
    main(sys.argv[1])
