#!/bin/bash
# One bench line per workload (device-resident value, per-kernel split), appended to $OUT
OUT=${OUT:-gpurun_out/all_workloads.jsonl}
: > $OUT
for w in 512x512x8_f32 256x256x1_f32 256x256x1_f64 sp4_128x32x1_f64 1024x1024x32_f32 sp3_64_f32 sp3_64_f64 sp3_128_f32 2048x2048x64_f32; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-100} --warmup 10 --no-cpu 2>/dev/null | tail -1 >> $OUT
done
python - "$OUT" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    print(f"{d['config']['workload']:20s} {d['ms_per_step']*1e3:10.2f} us  {d['value']/1e9:7.3f} Gcu/s  "
          f"step frac {d['roofline'].get('step', {}).get('frac', d['roofline'].get('frac')):.3f}")
PY
