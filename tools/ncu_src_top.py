"""Per-SASS-instruction hot spots of one kernel from an ncu report: the instructions with the
most excess shared-memory wavefronts (bank conflicts) and the most warp-stall samples.
usage: python tools/ncu_src_top.py REPORT KERNEL_NAME [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[hi + 1:]:
    if len(r) != len(h):
        break
    data.append(r)


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (KeyError, ValueError):
        return 0.0


tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"{len(data)} SASS lines, {tot_s:.0f} stall samples")
ex = sorted(data, key=lambda r: -(f(r, "L1 Wavefronts Shared") - f(r, "L1 Wavefronts Shared Ideal")))
print("-- excess shared wavefronts")
for r in ex[:n]:
    w, wi = f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Ideal")
    if w <= wi:
        break
    print(f"{r[ix['Address']]} {w:.3g} ideal {wi:.3g}  {r[ix['Source']]}")
print("-- stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{r[ix['Address']]} {100 * f(r, 'Warp Stall Sampling (All Samples)') / max(tot_s, 1):5.2f}%  {r[ix['Source']]}")
