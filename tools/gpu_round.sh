# one GPU session: parity tests, bench lines for every workload, ncu launch list of the default bench
set -x
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/tests_gpu.log 2>&1; tail -8 gpurun_out/tests_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
for w in c1 c3 c4 c2c c5s; do python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; cat gpurun_out/bench_$w.json; done
timeout 600 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo done
