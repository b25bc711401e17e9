"""One line per profiled launch of an ncu report: the metrics DESIGN.md and the
bench quote (duration, DRAM bytes, DMMA / FP64 pipe use, occupancy, L2 hit rate).

    python tools/ncu_summary.py gpurun_out/X.ncu-rep > profiles/rN_X_summary.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("kernel", "Kernel Name"),
    ("time_ms", "gpu__time_duration.sum"),
    ("dram_read_GB", "dram__bytes_read.sum"),
    ("dram_write_GB", "dram__bytes_write.sum"),
    ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dmma_inst_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    ("tensor_active_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("fp64_inst_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("regs", "launch__registers_per_thread"),
    ("smem_per_block", "launch__shared_mem_per_block_dynamic"),
]


def main(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = csv.writer(sys.stdout)
    out.writerow([k for k, _ in METRICS] + ["units"])
    for r in rows[2:]:
        vals, us = [], []
        for k, m in METRICS:
            if m in head:
                i = head.index(m)
                vals.append(r[i])
                us.append(f"{k}={units[i]}" if units[i] else "")
            else:
                vals.append("")
        out.writerow(vals + [";".join(u for u in us if u)])


if __name__ == "__main__":
    main(sys.argv[1])
