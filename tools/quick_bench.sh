#!/bin/bash
# 3 short bench runs (device-resident value only), one summary line each
for r in 1 2 3; do
  timeout 300 python bench.py --steps ${STEPS:-100} --warmup 10 --no-cpu ${@} > gpurun_out/qb_$r.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/qb_$r.log').read().strip().splitlines()[-1]); print('run $r', round(d['ms_per_step']*1e3,1), 'us', round(d['value']/1e9,2), 'Gcu/s frac', round(d['roofline']['step']['frac'],3), {k: round(v*1e3,1) for k,v in d['roofline']['kernels_ms'].items()})"
done
