SLO_SIM_LIB=$PWD/paper_2603_11340_b200/libslosim_cg4.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "continuous" 2>&1 | tail -1
bash tools/ab.sh "cg4 nocg4" c2c
