# one GPU session: parity tests, smoke, bench lines for every workload, ncu launch lists (small outputs only:
# gpurun brings back at most 64 MiB; full ncu captures go through tools/gpu_ncu.sh)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/tests_gpu.log 2>&1; tail -3 gpurun_out/tests_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 c2c c5s; do python bench.py --workload $w --no-cpu-baseline --steps 5 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --workload c4 --share-of 8 --no-cpu-baseline --steps 5 > gpurun_out/bench_c4s8.json 2>gpurun_out/bench_c4s8.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_c2.json 2>gpurun_out/bench_reference.err
N="ncu --clock-control none --target-processes application-only"
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_c2c.csv python bench.py --workload c2c --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
python tools/climb_rate.py > gpurun_out/climb_rate_c4.json 2>&1
python tools/climb_rate.py --seeds 16 > gpurun_out/climb_rate_c4_share8.json 2>&1
python bench.py --workload c5 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err
