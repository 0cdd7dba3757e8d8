# A/B timing of library variants / env settings:
#   VARS="default pb224" ENVS="X=1" WL=512x512x8_f32 STEPS=200 bash tools/_var.sh
for v in ${VARS:-default}; do
  if [ $v = default ]; then unset MMB_LIB; else export MMB_LIB=$PWD/build/var_$v/libmmb.so; fi
  for r in 1 2; do
  f=gpurun_out/v_${WL:-512x512x8_f32}_${v}${ENVS//[=]/_}_$r.log
  timeout 300 env $ENVS python bench.py --workload ${WL:-512x512x8_f32} --steps ${STEPS:-200} --warmup 10 --no-cpu > $f 2>&1
  python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('${WL:-512x512x8_f32} $v $ENVS', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['roofline'].get('kernels_ms', {}).items()})"
  done
done 2>&1 | grep -v "^+"
