# usage: bash tools/sweep_regs.sh "r80 r96" "1 4"
for v in $1; do for w in $2; do
SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_$v.so python bench.py --no-cpu-baseline --steps 3 --warmup 2 --warps-per-block $w ${3:-} 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $w, round(d['value']/1e9,3), round(d['k1_ms_per_step'],2), d['config']['launch'])"
done; done
