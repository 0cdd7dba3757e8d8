set -x
D=gpurun_out/fin; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 600 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 600 $D/bench.json
timeout 600 python bench.py --steps 20 --warmup 5 > $D/bench20.json 2> $D/bench20.err; tail -c 300 $D/bench20.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $D/bench_ref.json 2> $D/bench_ref.err; tail -c 300 $D/bench_ref.json
OUT=$D/all_workloads.jsonl bash tools/all_workloads.sh > $D/all.log 2>&1; cat $D/all.log
python tools/profile_step.py --steps 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_yz|k_xstep" -s 2 -c 2 -o $D/prof_512 python tools/profile_step.py --steps 3 > $D/ncu.log 2>&1; tail -1 $D/ncu.log
