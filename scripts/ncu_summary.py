"""Summarise an ncu --set full capture into profiles/ (JSON + details CSV).
usage: python scripts/ncu_summary.py gpurun_out/walk_r01.ncu-rep profiles/r01_walk_C3 [config-key] [patterns]"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
key = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sass__inst_executed_local_loads", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"]
res = {"kernel": None}
for i, h in enumerate(hdr):
    if h in want:
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            v = vals[i]
        res[h] = {"value": v, "unit": units[i]}
    if h == "Kernel Name":
        res["kernel"] = vals[i]
def tobytes(m):
    u = m["unit"].lower()
    f = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)
    return m["value"] * f
rd = tobytes(res["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in res else None
wr = tobytes(res["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in res else None
res["dram_bytes_per_launch"] = (rd or 0) + (wr or 0)
with open(out + ".json", "w") as f:
    json.dump(res, f, indent=1)
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
with open(out + "_details.csv", "w") as f:
    f.write(det)
print(json.dumps({k: (v["value"] if isinstance(v, dict) else v) for k, v in res.items()}, indent=1))
