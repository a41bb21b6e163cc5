"""SASS of one kernel in address order with stall samples and execution counts
(ncu --page source --csv), to attribute time to code regions."""
import csv
import io
import subprocess
import sys

rep, kfilter = sys.argv[1], sys.argv[2]
minpct = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kfilter],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
start = [i for i, ln in enumerate(lines) if ln.startswith('"Kernel Name"')][0]
r = list(csv.reader(io.StringIO("\n".join(lines[start + 1:]))))
hdr = r[0]
ia, isrc = hdr.index("Address"), hdr.index("Source")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex, ith = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
rows = []
for row in r[1:]:
    if len(row) != len(hdr) or row[0].startswith('"Kernel'):
        break
    try:
        rows.append((row[ia], float(row[isamp] or 0), float(row[iex] or 0), float(row[ith] or 0), row[isrc]))
    except ValueError:
        break
tot = sum(x[1] for x in rows)
cum = 0.0
for i, (a, s, e, th, src) in enumerate(rows):
    cum += s
    if 100 * s / tot >= minpct or "BRA" in src[:12] or "EXIT" in src:
        print(f"{i:5d} {a[-5:]} {100*s/tot:5.2f}% cum {100*cum/tot:5.1f}% ex={e:9.3e} thr={th/max(e,1):4.1f} {src[:70]}")
