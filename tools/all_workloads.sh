# one bench line per workload (device-resident value, no CPU baseline) -> gpurun_out/all_<w>.json
for w in 512x512x8_f32 1024x1024x32_f32 2048x2048x64_f32 256x256x1_f32 256x256x1_f64 sp4_128x32x1_f64 sp3_64_f32 sp3_64_f64 sp3_128_f32; do
  s=200; [ $w = 2048x2048x64_f32 ] && s=10; [ $w = 1024x1024x32_f32 ] && s=50
  case $w in 256*|sp4*|sp3_64*) s=1000;; esac
  timeout 600 python bench.py --workload $w --steps $s --warmup 10 --no-cpu 2>/dev/null | tail -1 > gpurun_out/all_$w.json
  python -c "
import json; d=json.load(open('gpurun_out/all_$w.json')); r=d['roofline']
st=r.get('step', {}).get('frac', r.get('frac'))
print('%-18s %10.2f us  %7.3f Gcu/s  step-roofline %.3f  e2e %.3f Gcu/s' % ('$w', d['ms_per_step']*1e3, d['value']/1e9, st, d['e2e']['value']/1e9))"
done
