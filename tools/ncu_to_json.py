"""Write profiles/<round>/ncu_summary.json from an ncu --set full report: per kernel the
duration and DRAM bytes (read + write) of one launch, for bench.py's roofline 'traffic'."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}
res = {"report": rep, "dram_bytes_per_launch": {}, "duration_s": {}}
for row in r[2:]:
    name = row[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0].replace("k_", "")
    def val(k, tab):
        i = hdr.index(k)
        return float(row[i].replace(",", "")) * tab.get(units[i], 1.0)
    b = val("dram__bytes_read.sum", scale) + val("dram__bytes_write.sum", scale)
    res["dram_bytes_per_launch"][name] = b
    res["duration_s"][name] = val("gpu__time_duration.sum", tscale)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
