"""Executed FP32 work per kernel from an ncu report: thread-level
FFMA x 2 + FADD + FMUL (+ the packed f32x2 forms x 2) from the SASS source page, divided by the
kernel duration, against the 74.4 TFLOP/s FP32 peak.  Counts every executed lane,
including work on skin / sentinel entries, so it is an upper bound of the algorithmic rate."""
import csv
import io
import subprocess
import sys

PEAK = 148 * 128 * 2 * 1.965e9 / 1e12
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}
dur = {}
for row in r[2:]:
    name = row[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
    i = hdr.index("gpu__time_duration.sum")
    dur.setdefault(name, float(row[i].replace(",", "")) * tscale.get(units[i], 1e-9))
for k in sys.argv[2:] or ["k_density", "k_gradient", "k_force"]:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", k, "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) < 3 or k not in dur:
        continue
    h, data = rows[1], rows[2:]
    s, te = h.index("Source"), h.index("Predicated-On Thread Instructions Executed")
    fl = 0.0
    for row in data:
        if len(row) != len(h):  # (the next launch's table: count the first launch only)
            break
        t = row[s].strip()
        op = (t.split()[1] if t.startswith("@") else t.split()[0]) if t else ""
        n = float(row[te] or 0)
        if op.startswith("FFMA2"):
            fl += 4 * n
        elif op.startswith(("FADD2", "FMUL2")):
            fl += 2 * n
        elif op.startswith("FFMA"):
            fl += 2 * n
        elif op.startswith(("FADD", "FMUL")):
            fl += n
    tf = fl / dur[k] / 1e12
    print(f"{k}: executed FP32 {fl:.4g} flop in {dur[k] * 1e3:.3f} ms = {tf:.2f} TFLOP/s = {tf / PEAK:.3f} of peak")
