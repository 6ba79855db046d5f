# A/B of the static-batching generation policies (inline K1 vs split K1g + K1s) on every static workload
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random_small or edge_cases or c1_full" > gpurun_out/t_split.log 2>&1; tail -3 gpurun_out/t_split.log
for g in ${GENS:-1 2}; do
 for w in ${WLS:-c2 c4 c1 c3 c5s}; do python bench.py --workload $w --no-cpu-baseline --steps 5 --gen-policy $g 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('gen$g $w', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'gen', round(k['k1g_generate'],3), 'chain', round(k['chain'],3), 'k1b', round(k['k1b_select'],3))"; done
 python bench.py --workload c4 --no-cpu-baseline --steps 5 --gen-policy $g --share-of 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('gen$g c4/8', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'gen', round(k['k1g_generate'],3), 'chain', round(k['chain'],3), 'k1b', round(k['k1b_select'],3))"
done
