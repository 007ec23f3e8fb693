TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py --config cfg2 --e2e-chunks1 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
for cf in cfg2s cfg2r cfg10; do
  timeout 900 python bench.py --config $cf > $OUT/bench_$cf.json 2> $OUT/bench_$cf.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv \
    python bench.py --config cfg2 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simplex_reg -c 1 -o $OUT/full_cfg2 \
  python bench.py --config cfg2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
