"""Per kernel: shared-memory wavefronts vs ideal of the hot LDS.128 gathers (bank conflicts),
from an ncu --set full report (ncu --page source --csv per kernel)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
for k in sys.argv[2:] or ["k_density", "k_gradient", "k_force", "k_lists"]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", k, "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, data = rows[1], rows[2:]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    wf, wfi = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
    hot = [r for r in data if "LDS.128" in r[src] and int(r[ie] or 0) > 1_000_000]
    a = sum(int(r[wf] or 0) for r in hot)
    b = sum(int(r[wfi] or 0) for r in hot)
    print(f"{k}: hot LDS.128 wavefronts {a:.4g} ideal {b:.4g} ratio {a / max(b, 1):.2f}")
