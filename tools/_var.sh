# A/B timing of library variants / env settings: VARS="default pb224" ENVS="X=1" bash tools/_var.sh
for v in ${VARS:-default}; do
  if [ $v = default ]; then unset MMB_LIB; else export MMB_LIB=$PWD/build/var_$v/libmmb.so; fi
  for r in 1 2; do
  timeout 300 env $ENVS python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/v_${v}${ENVS//[=]/_}_$r.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v_${v}${ENVS//[=]/_}_$r.log').read().strip().splitlines()[-1]); print('$v $ENVS', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['roofline']['kernels_ms'].items()})"
  done
done 2>&1 | grep -v "^+"
