set -x
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/gputests.txt 2>&1
echo "rc=$?" >> gpurun_out/r2a/gputests.txt
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-chunks1 > gpurun_out/r2a/b_cfg2.json 2> gpurun_out/r2a/b_cfg2.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-hint --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2a/b_cfg2_nohint.json 2>&1
