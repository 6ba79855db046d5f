# full ncu captures of the hot kernels, summarised on the box (tools/ncu_summary.py, ncu_lines.py) so only small
# JSON / text files come back; usage: bash tools/gpu_ncu.sh TAG  (writes gpurun_out/TAG_*)
set -x
T=${1:-r02}
mkdir -p gpurun_out
N="ncu --clock-control none --target-processes application-only --set full --import-source on"
cap() {  # name, kernel regex, skip, bench args
  timeout 900 $N -k regex:$2 -s $3 -c 1 -o /tmp/$1 python bench.py --no-cpu-baseline $4 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/$1.ncu-rep gpurun_out/${T}_$1_ncu.json > /dev/null
  python tools/ncu_lines.py /tmp/$1.ncu-rep 40 > gpurun_out/${T}_$1_lines.txt
  ncu -i /tmp/$1.ncu-rep --page raw --csv > /tmp/$1_raw.csv 2>/dev/null; python tools/ncu_stalls.py /tmp/$1_raw.csv >> gpurun_out/${T}_$1_lines.txt
}
cap k1g_c2 slo_gen_kernel 3 "--steps 1 --warmup 3"
cap k1s_c2 slo_serve 3 "--steps 1 --warmup 3"
cap k1c_c2c slo_sim_cont 1 "--workload c2c --steps 1 --warmup 1"
cap k1s_c4s8 slo_serve 5 "--workload c4 --share-of 8 --eager-climb --steps 1 --warmup 3"
cap k1s_c1 slo_serve 5 "--workload c1 --steps 1 --warmup 3"
cap k1b_c2 slo_select 3 "--steps 1 --warmup 3"
ls -la gpurun_out
