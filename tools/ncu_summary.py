"""Summarise an ncu --set full report (raw page) for the lane kernel."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
def g(k):
    v = d.get(k, ("", ""))[0].replace(",", "")
    try: return float(v)
    except ValueError: return v
keys = [k for k in hdr if "pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued")]
tot = sum(g(k) or 0 for k in keys)
print("stall samples (top):")
for v, k in sorted(((g(k) or 0, k) for k in keys), reverse=True)[:10]:
    print(f"  {100*v/tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_','')}")
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
          "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
          "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
          "smsp__sass_inst_executed_op_shared_ld.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
          "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]:
    if k in d:
        print(f"  {k} = {d[k][0]} {d[k][1]}")
