timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/tests_gpu.log 2>&1; tail -5 gpurun_out/tests_gpu.log
