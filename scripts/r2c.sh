mkdir -p gpurun_out/r2c
python scripts/ab.py ab/base ab/compact -- cfg3:2000 cfg3s:2000 cfg8:200 cfg6:1000 > gpurun_out/r2c/ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_dist.py tests/test_gpu_configs.py -x -q > gpurun_out/r2c/tests.txt 2>&1
python scripts/timeline.py cfg2 cfg5 > gpurun_out/r2c/timeline.txt 2>&1
timeout 600 python bench.py --config cfg3 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/r2c/b_cfg3.json 2>&1
