"""Summarise an ncu --set full report of the mask kernel into profiles/ (json + text)."""
import csv, io, json, subprocess, sys

rep, out_json, tag = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__cluster_dim_x", "smsp__inst_executed.sum"]
d = {}
for i, name in enumerate(h):
    if name in want:
        d[name] = (v[i], u[i])
def num(k, scale=1.0):
    val, unit = d[k]
    f = float(val.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}.get(unit, 1)
    return f * mult
summary = {k: {"value": d[k][0], "unit": d[k][1]} for k in d}
traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
summary["_traffic_bytes_per_launch"] = traffic
json.dump(summary, open(out_json, "w"), indent=1)
print(json.dumps({k: v["value"] + " " + v["unit"] for k, v in summary.items() if isinstance(v, dict)}, indent=1))
print("traffic bytes/launch:", traffic)
