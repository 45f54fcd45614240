import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active",
        "smsp__average_warps_issue_stalled_wait_per_issue_active",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active"]
idx = [h.index(k) for k in want if k in h]
for r in rows[2:]:
    print("----")
    for i in idx:
        print(f"  {h[i][:75]:75s} {r[i][:60]}")
