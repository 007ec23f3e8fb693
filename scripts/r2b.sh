mkdir -p gpurun_out/r2b
python scripts/ab.py ab/base ab/sigma -- cfg2:50000 cfg10:50000 cfg2r:20000 > gpurun_out/r2b/ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "R or cfg2 or reg" > gpurun_out/r2b/tests.txt 2>&1
