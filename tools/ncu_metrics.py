"""Print the key metrics of one kernel from an ncu report (ncu -i REP --page raw --csv)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x"]
STALL = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    d = dict(zip(hdr, r))
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k]} {units[hdr.index(k)]}")
    st = sorted(((float(d[k].replace(',', '') or 0), k) for k in hdr if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")), reverse=True)
    for v, k in st[:8]:
        print(f"  stall {k[len(STALL):-len('_per_issue_active.ratio')]:30s} {v:.3f}")
    # busiest pipes (any pipe metric reported as % of peak)
    pipes = []
    for k in hdr:
        if (k.startswith("sm__pipe_") or k.startswith("sm__inst_executed_pipe_")) and "pct_of_peak" in k:
            try:
                pipes.append((float(d[k].replace(',', '')), k))
            except ValueError:
                pass
    for v, k in sorted(pipes, reverse=True)[:10]:
        print(f"  pipe {k:76s} {v:.1f}")
