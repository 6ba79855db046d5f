set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slo_sim_kernel_t -s 3 -c 1 -o gpurun_out/k1s_c4s8 python bench.py --workload c4 --eager-climb --share-of 8 --gen-policy 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slo_sim_kernel_t|slo_gen_kernel" -s 6 -c 2 -o gpurun_out/k1s_c2 python bench.py --workload c2 --gen-policy 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
