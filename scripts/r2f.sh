mkdir -p gpurun_out/r2f
python scripts/ab.py ab/compact ab/redratio -- cfg2:50000 cfg10:50000 cfg2r:20000 cfg2s:20000 cfg9:50000 cfg1m:1000000 > gpurun_out/r2f/ab.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_tiny.py tests/test_gpu_configs.py -x -q > gpurun_out/r2f/tests.txt 2>&1
