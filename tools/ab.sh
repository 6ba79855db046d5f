# usage: bash tools/ab.sh "b1 b2" [workload]  — bench each in-tree experimental build libslosim_<v>.so
for v in $1; do
SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_$v.so python bench.py --no-cpu-baseline --steps 3 --warmup 2 --workload ${2:-c2} 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,3), round(d['k1_ms_per_step'],2), d['config']['launch'])"
done
