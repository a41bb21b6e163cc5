"""Top SASS instructions of an ncu report by stall samples (ncu --page source --csv)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + (["-k", kfilter] if kfilter else []),
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
# the csv has a kernel-name line before each table
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur:
    blocks.append(cur)
for b in blocks:
    name = b[0]
    r = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = r[0]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    ith = hdr.index("Thread Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    rows = []
    tot_s = tot_e = 0
    for row in r[1:]:
        try:
            s = float(row[isamp] or 0)
            e = float(row[iex] or 0)
        except ValueError:
            continue
        tot_s += s
        tot_e += e
        rows.append((s, e, row))
    print(name[:120], f"total samples {tot_s:.0f} inst {tot_e:.3e}")
    rows.sort(key=lambda x: -x[0])
    for s, e, row in rows[:top]:
        st = sorted(((float(row[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        th = float(row[ith] or 0)
        print(f"{row[ia]:>6} {100*s/tot_s:5.1f}% ex={e:9.3e} thr={th/max(e,1):4.1f} {row[isrc][:60]:60s} "
              + " ".join(f"{n}:{v:.0f}" for v, n in st))
