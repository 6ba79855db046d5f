bash tools/gpu_round.sh
N="ncu --clock-control none --target-processes application-only --set full --import-source on"
timeout 900 $N -k regex:slo_serve -s 3 -c 1 -o /tmp/k1s_c2 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/k1s_c2.ncu-rep gpurun_out/r02b_k1s_c2_ncu.json > /dev/null
python tools/ncu_lines.py /tmp/k1s_c2.ncu-rep 40 > gpurun_out/r02b_k1s_c2_lines.txt
ncu -i /tmp/k1s_c2.ncu-rep --page raw --csv > /tmp/k1s_raw.csv 2>/dev/null; python tools/ncu_stalls.py /tmp/k1s_raw.csv >> gpurun_out/r02b_k1s_c2_lines.txt
