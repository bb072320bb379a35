"""Summarize an ncu report: key throughput, pipe and stall metrics (python tools/ncu_summary.py REP)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smem wavefronts % (elapsed)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg", "cycles elapsed"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def main(path):
    raw = (open(path).read() if path.endswith(".csv") else  # a saved `--page raw --csv` export
           subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "")[:90])
        for k, name in KEYS:
            if k in d:
                print(f"  {name:32s} {d[k]} {u.get(k, '')}")
        st = sorted(((float(d[k]), k[len(STALLS):].replace("_per_issue_active.ratio", ""))
                     for k in d if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio") and d[k]),
                    reverse=True)
        print("  stalls per issue:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
