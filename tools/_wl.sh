# one quick line per workload: WLS="a b" bash tools/_wl.sh
for w in ${WLS:-512x512x8_f32}; do
  timeout 300 python bench.py --workload $w --steps ${STEPS:-300} --warmup 10 --no-cpu > gpurun_out/wl_$w.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/wl_$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,3), 'Gcu/s', {k: round(v*1e3,1) for k,v in d['roofline']['kernels_ms'].items()})"
done
