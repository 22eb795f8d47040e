"""Summarise an ncu --set full report of the SpMM kernel into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_<tag> --alg-bytes B
Writes <out>.txt (key counters) and <out>.json (traffic for bench.py's roofline)."""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "sm__cycles_elapsed.avg",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__warps_active.avg.per_cycle_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("out")
ap.add_argument("--alg-bytes", type=float, default=0.0)
ap.add_argument("--cell", default="")
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
got = {}
for h, u, v in zip(hdr, units, vals):
    k = h.split(".", 2)[-1] if h.startswith(("TPC.", "SM_C.")) else h  # section-prefixed names
    if k in KEYS:
        got[k] = (v, u)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def nbytes(k):
    v, u = got.get(k, ("0", "byte"))
    return float(v.replace(",", "")) * scale.get(u, 1)
traffic = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
with open(a.out + ".txt", "w") as f:
    f.write(f"ncu --set full summary of {a.rep} ({a.cell})\n")
    for k in KEYS:
        if k in got:
            f.write(f"{k} = {got[k][0]} {got[k][1]}\n")
    f.write(f"dram traffic per launch = {traffic:.0f} B; algorithmic bytes = {a.alg_bytes:.0f} B;"
            f" ratio = {traffic / a.alg_bytes if a.alg_bytes else 0:.3f}\n")
with open(a.out + ".json", "w") as f:
    json.dump({"cell": a.cell, "dram_bytes_per_launch": traffic, "alg_bytes_per_launch": a.alg_bytes,
               "duration_us_under_ncu": float(got.get("gpu__time_duration.sum", ("0", ""))[0].replace(",", ""))}, f,
              indent=1)
print(open(a.out + ".txt").read())
