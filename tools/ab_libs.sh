# A/B bench of in-tree library variants: bash tools/ab_libs.sh OUTDIR WORKLOAD STEPS lib1 lib2 ...
D=$1; W=$2; S=$3; shift 3; mkdir -p $D
for rep in 1 2; do for v in "$@"; do MMB_LIB=paper_1501_07293_b200/$v timeout 300 python bench.py --workload $W --steps $S --warmup 10 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$W $v\", round(d[\"ms_per_step\"]*1e3,2), {k: round(v*1e3,2) for k,v in d[\"roofline\"][\"kernels_ms\"].items()})" >> $D/ab.log; done; done
cat $D/ab.log
