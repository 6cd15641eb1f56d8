"""Print the headline ncu metrics of every kernel in a report (stall breakdown, pipes, memory).
    python scripts/ncu_metrics.py gpurun_out/prof.ncu-rep [substring]"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__warps_eligible.avg.per_cycle_active"]
rows = list(csv.reader(subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if sub not in name:
        continue
    print("==", name[:110])
    for k in KEYS:
        if k in hdr:
            print(f"  {k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
    st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and
          h.endswith("_per_issue_active.ratio")]
    st = sorted(((float(v.replace(",", "")), h) for h, v in st if v), reverse=True)[:10]
    print("  stalls per issue:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st))
