"""Summarise an ncu --set full report of the NTT-domain mask kernel (NEXT #4) into profiles/."""
import csv, io, json, subprocess, sys

rep, out_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
out = {h[i]: {"value": v[i], "unit": u[i]} for i in range(len(h)) if h[i] in want}
st = {h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[i].replace(",", "") or 0)
      for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")}
tot = sum(st.values()) or 1.0
out["stall_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x / tot > 0.005}
json.dump(out, open(out_json, "w"), indent=1)
print(json.dumps(out, indent=1))
