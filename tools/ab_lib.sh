# usage: bash /tmp/ab.sh OUTDIR  (A/B of libmmb.so vs libmmb_prev.so)
D=$1; mkdir -p $D
(timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_production.py -m gpu -x -q 2>&1 | tail -4) > $D/tests.log
for v in libmmb.so libmmb_prev.so libmmb.so libmmb_prev.so; do MMB_LIB=paper_1501_07293_b200/$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v\", round(d[\"ms_per_step\"]*1e3,2), {k: round(v*1e3,2) for k,v in d[\"roofline\"][\"kernels_ms\"].items()})" >> $D/ab.log; done
for w in 256x256x1_f32 256x256x1_f64 1024x1024x32_f32 sp3_128_f32; do for v in libmmb.so libmmb_prev.so; do MMB_LIB=paper_1501_07293_b200/$v timeout 300 python bench.py --workload $w --steps 100 --warmup 10 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$w $v\", round(d[\"ms_per_step\"]*1e3,2))" >> $D/ab.log; done; done
cat $D/tests.log $D/ab.log
