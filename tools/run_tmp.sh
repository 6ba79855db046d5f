mkdir -p gpurun_out
bash tools/sanitize.sh
bash tools/ab.sh "x" c2 2>/dev/null; python bench.py --workload c2 --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('c2', round(d['ms_per_step'],3), 'gen', round(k['k1g_generate'],3), 'chain', round(k['chain'],3))"
