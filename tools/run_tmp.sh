SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_s2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random_small and split" 2>&1 | tail -1
for v in s1 s2; do for g in "" "--no-graph"; do SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_$v.so python bench.py --workload c1 --no-cpu-baseline --steps 10 $g 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$v c1 $g', round(d['ms_per_step'],4), 'chain', round(k['chain'],4), 'e2e', round(2000/d['e2e']['value']*1e3,4), d['config']['cuda_graph'])"; done; done
bash tools/ab.sh "s1 s2" c4 "--share-of 8"
bash tools/ab.sh "s1 s2" c4
bash tools/ab.sh "s1 s2" c2
