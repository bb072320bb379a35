"""Pipe utilization of the M4RM kernel from ncu --set full reports -> profiles/<tag>_pipes.json.

python tools/pipes_from_ncu.py TAG "CONFIG NAME::report.ncu-rep" ...
(the ALU pipe and the shared-memory wavefront pipe are the two resources the kernel can be bound
by; bench.py reports them next to the algorithmic roofline)"""
import csv
import io
import json
import subprocess
import sys

M = {
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_wavefronts_ld": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_wavefronts_st": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts_ld": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smem_bank_conflicts_st": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "alu_inst_executed": "smsp__inst_executed_pipe_alu.sum",
    "duration_us": "gpu__time_duration.sum",
}
tag = sys.argv[1]
out = {"_source": f"profiles/{tag}_pipes.json from ncu --set full captures of the M4RM kernel"}
for arg in sys.argv[2:]:
    name, rep = arg.split("::", 1)
    raw = (open(rep).read() if rep.endswith(".csv") else  # a saved `--page raw --csv` export
           subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    out[name] = {k: float(d[v].replace(",", "")) for k, v in M.items() if v in d and d[v]}
    out[name]["kernel"] = d.get("Kernel Name", "")[:80]
with open(f"profiles/{tag}_pipes.json", "w") as f:
    json.dump(out, f, indent=1)
print(out)
