# A/B bench with environment settings: bash tools/ab_env.sh OUTDIR WORKLOAD STEPS "ENV1" "ENV2" ...
# (each ENV is a space-separated list of VAR=value, e.g. "MMB_LIB=paper_1501_07293_b200/libmmb_v2.so MMB_YZ_SPLIT=0")
D=$1; W=$2; S=$3; shift 3; mkdir -p $D
for rep in 1 2; do for e in "$@"; do env $e timeout 300 python bench.py --workload $W --steps $S --warmup 10 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$W [$e]\", round(d[\"ms_per_step\"]*1e3,2), {k: round(v*1e3,2) for k,v in d[\"roofline\"][\"kernels_ms\"].items()})" >> $D/ab.log; done; done
cat $D/ab.log
