"""Extract per-launch DRAM traffic of the M4RM kernel from ncu reports into profiles/<tag>_traffic.json.

python tools/traffic_from_ncu.py TAG "CONFIG NAME::report.ncu-rep" ..."""
import csv
import io
import json
import subprocess
import sys

tag = sys.argv[1]
out = {"_source": f"profiles/{tag}_traffic.json from ncu --set full captures of the M4RM kernel"}
for arg in sys.argv[2:]:
    name, rep = arg.split("::", 1)
    raw = (open(rep).read() if rep.endswith(".csv") else  # a saved `--page raw --csv` export
           subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[k].replace(",", "")) * scale[u[k]]
    out[name] = tot
json.dump(out, open(f"profiles/{tag}_traffic.json", "w"), indent=1)
print(out)
