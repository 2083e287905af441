"""Dev tool: one-screen summary of an ncu --set full report (pipes, DRAM, stalls)."""
import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:80])
    want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
            'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
            'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed',
            'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
            'smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__registers_per_thread','launch__occupancy_limit_registers','sm__cycles_elapsed.avg.per_second','smsp__inst_executed.sum',
            'launch__grid_size','launch__block_size']
    for w in want:
        if w in d: print(f"  {w} = {d[w]} {units[h.index(w)]}")
    st = [(k, float(d[k])) for k in h if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio') and d[k] not in ('', 'n/a')]
    st.sort(key=lambda t: -t[1])
    print("  stalls/issue:", ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={x:.2f}" for k, x in st[:8]))
