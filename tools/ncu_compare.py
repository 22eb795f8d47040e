import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
 "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
 "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__block_size",
 "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
 "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
 "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
 "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
 "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
 "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
 "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]
def load(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        d = {}
        for h, v in zip(hdr, r):
            k = h.split(".", 2)[-1] if h.startswith(("TPC.", "SM_C.")) else h
            d[k] = v
        out.append(d)
    return out
reps = [load(r) for r in sys.argv[1:]]
n = len(reps[0])
for i in range(n):
    print("launch", i, [r[i].get("Kernel Name","")[:40] for r in reps])
    for k in KEYS:
        print(f"  {k[:75]:75s}", "  ".join(f"{r[i].get(k,'-'):>14s}" for r in reps))
