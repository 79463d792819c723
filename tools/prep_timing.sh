# per-phase prep wall times of the cfg3 bench (TSG_PREP_TIMING=1)
mkdir -p gpurun_out/prep
TSG_PREP_TIMING=1 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/prep/cfg3.json 2> gpurun_out/prep/cfg3.err
grep "tsg " gpurun_out/prep/cfg3.err
python -c "import json; d=json.load(open('gpurun_out/prep/cfg3.json')); print(d['prep_split'])"
python - <<'PY'
import time, numpy as np, paper_1502_00355_b200 as ts
from paper_1502_00355_b200 import capi
xy, tri = ts.graded_arrays(16_000_000, 1, 1e-3, 1024)
ctx = capi.Context(0)
for k in range(2):
    t=time.time(); o = ctx.hilbert_order(xy); t1=time.time()-t
    t=time.time(); topo = ctx.topology(len(xy), tri); t2=time.time()-t
    print("hilbert", round(t1,3), "topology", round(t2,3))
PY
