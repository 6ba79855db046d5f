# usage: bash tools/build_variant.sh NAME "-DFLAG=V ..."  -> paper_2603_11340_b200/libslosim_NAME.so (for tools/ab.sh)
cd "$(dirname "$0")/.." && C=paper_2603_11340_b200/csrc && \
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -diag-suppress 20281 -Xcompiler -fPIC -shared $2 \
  -o paper_2603_11340_b200/libslosim_$1.so $C/slo_abi.cu $C/slo_sim_kernel.cu $C/slo_climb.cu $C/slo_pareto.cu $C/slo_selftest.cu
