timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/tests_gpu.log 2>&1; tail -3 gpurun_out/tests_gpu.log
for w in c2 c3 c5s c4; do bash tools/ab.sh "g4 nog4" $w; done
