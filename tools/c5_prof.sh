#!/bin/bash
# C5s (clustered 128^3): debug grid line, bench line and the launch list summed per kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SPH_DEBUG=1 timeout 600 python bench.py --workload C5s --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c5dbg.json 2> gpurun_out/c5d.err
grep "sph rank\|rebuild ms" gpurun_out/c5d.err | tail -3 | cut -c1-300
timeout 600 python bench.py --workload C5s --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/c5d.json 2> gpurun_out/c5.err
python -c "
import json; d=json.loads(open('gpurun_out/c5d.json').read().strip().splitlines()[-1]); print('ms/step', round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python bench.py --workload C5s --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/c5n.log 2>&1; echo ncu rc=$?
python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/c5_launches.csv')))
hdr=[r for r in rows if r and r[0]=='ID'][0]; i=rows.index(hdr)
ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value'); iu=hdr.index('Metric Unit')
tot=collections.Counter(); n=collections.Counter()
for r in rows[i+1:]:
    if len(r)<len(hdr): continue
    v=float(r[iv].replace(',','')); u=r[iu]
    v*= {'nsecond':1e-6,'ns':1e-6,'usecond':1e-3,'us':1e-3,'msecond':1,'ms':1}[u]
    k=r[ik].split('(')[0].split('::')[-1][:40]; tot[k]+=v; n[k]+=1
for k,v in tot.most_common(18): print(f"{k:40s} {v:9.2f} ms {n[k]:4d}")
PY
fi
