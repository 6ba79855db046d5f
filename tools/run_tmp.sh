timeout 600 python -m pytest tests/test_gpu_exhaustive.py -m gpu -q -x -k noise 2>&1 | tail -1
bash tools/ab.sh "base dp c80 c88" c2c
bash tools/ab.sh "base dp" c2
