"""Key metrics of each kernel in an ncu --set full report (raw page csv).
  ncu -i rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv "title" """
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg"]
stalls = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
print(sys.argv[2] if len(sys.argv) > 2 else "")
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")])
    for w in want:
        if w in h:
            print(f"  {w} = {r[h.index(w)]} {units[h.index(w)]}")
    st = sorted(((int(float(r[h.index(c)] or 0)), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in stalls), reverse=True)[:8]
    print("  top stall samples: " + ", ".join(f"{n}={v}" for v, n in st))
