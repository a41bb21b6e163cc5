"""Coarse code regions of one kernel (ncu --page source): warp-stall samples and executed
instructions per block of SASS lines, with the branches / shared loads / barriers in each."""
import csv, io, subprocess, sys
import numpy as np
rep, k = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu","-i",rep,"--page","source","--csv","-k",k],capture_output=True,text=True).stdout
lines = raw.splitlines()
start=[i for i,l in enumerate(lines) if l.startswith('"Kernel Name"')][0]
r=list(csv.reader(io.StringIO("\n".join(lines[start+1:]))))
h=r[0]
isamp=h.index("Warp Stall Sampling (All Samples)"); iex=h.index("Instructions Executed"); ith=h.index("Thread Instructions Executed")
rows=[]
for row in r[1:]:
    if len(row)!=len(h): break
    try: rows.append((float(row[isamp] or 0), float(row[iex] or 0), float(row[ith] or 0), row[h.index("Source")]))
    except: break
S=np.array([x[0] for x in rows]); E=np.array([x[1] for x in rows]); T=np.array([x[2] for x in rows])
# print coarse blocks of 40 lines
step=int(sys.argv[3]) if len(sys.argv)>3 else 50
for a in range(0,len(rows),step):
    b=min(a+step,len(rows))
    src=[x[3].strip()[:40] for x in rows[a:b] if ('BRA' in x[3] or 'LDS' in x[3] or 'BAR' in x[3] or 'SYNCS' in x[3] or 'RED' in x[3] or 'UBLKCP' in x[3])][:3]
    print(f"{a:5d} samp {100*S[a:b].sum()/S.sum():5.1f}% inst {100*E[a:b].sum()/E.sum():5.1f}% maxex {E[a:b].max():.2e}", src)
