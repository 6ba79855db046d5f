# usage: bash tools/ab.sh "v1 v2" [workload] [extra bench args] — bench each in-tree build libslosim_<v>.so
for v in $1; do
SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_$v.so python bench.py --no-cpu-baseline --steps 3 --warmup 2 --workload ${2:-c2} $3 2>/tmp/ab_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$v ${2:-c2}', round(d['value']/1e9,3), round(d['ms_per_step'],3), 'gen', round(k['k1g_generate'],3), 'chain', round(k['chain'],3), 'k1b', round(k['k1b_select'],3))" || tail -5 /tmp/ab_err.txt
done
