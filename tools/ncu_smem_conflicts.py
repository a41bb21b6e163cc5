"""Shared-memory wavefronts vs ideal per SASS instruction (bank conflicts) from an ncu report."""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO("\n".join(raw.splitlines()[1:]))))
hdr = r[0]
ix = {h: i for i, h in enumerate(hdr)}
tw = ti = 0
lds_w = lds_i = 0
for row in r[1:]:
    src = row[ix["Source"]]
    if any(op in src for op in ("LDS", "STS", "ATOMS", "LDGSTS")):
        w = float(row[ix["L1 Wavefronts Shared"]] or 0)
        wi = float(row[ix["L1 Wavefronts Shared Ideal"]] or 0)
        tw += w
        ti += wi
        if "LDS" in src:
            lds_w += w
            lds_i += wi
print(f"all smem ops: wavefronts {tw:.3e} ideal {ti:.3e} ratio {tw / max(ti, 1):.2f}")
print(f"LDS only:     wavefronts {lds_w:.3e} ideal {lds_i:.3e} ratio {lds_w / max(lds_i, 1):.2f}")
