#!/bin/bash
# Runs on the GPU box: gpu tests, smoke, bench lines for every config + ncu evidence (launch
# lists, full captures of the dominant kernels).  Usage: bash scripts/profile_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
# the whole cfg3 batch against the oracle (~6 min of oracle time on the box's cores)
LPB_SLOW=1 timeout 1500 python -m pytest tests/test_gpu_configs.py -k cfg3_full -s -q > $OUT/cfg3_full.txt 2>&1
for cf in cfg2 cfg5; do  # with the n_chunks = 1 (no overlap) e2e control
  timeout 900 python bench.py --config $cf --e2e-chunks1 > $OUT/bench_$cf.json 2> $OUT/bench_$cf.err
done
for cf in cfg1 cfg1m cfg4 cfg2s cfg2r cfg9 cfg10; do
  timeout 900 python bench.py --config $cf > $OUT/bench_$cf.json 2> $OUT/bench_$cf.err
done
# strong scaling line at N = 1 (the fixed cfg5 batch) and CUDA-graph replay of small solves
timeout 900 python bench.py --config cfg5 --scaling strong --no-cpu-baseline > $OUT/bench_cfg5_strong.json 2>&1
timeout 900 python bench.py --config cfg4 --graph --no-cpu-baseline > $OUT/bench_cfg4_graph.json 2>&1
timeout 900 python bench.py --config cfg1 --graph --no-cpu-baseline > $OUT/bench_cfg1_graph.json 2>&1
# host pipeline: per-chunk event timeline (10 vs 1 chunks) and ASan/UBSan of the host code
timeout 900 python scripts/timeline.py cfg2 cfg5 > $OUT/timeline.txt 2>&1
timeout 1200 bash scripts/sanitize_host.sh $OUT > /dev/null 2>&1
for cf in cfg3 cfg3s; do
  timeout 900 python bench.py --config $cf --steps 3 --warmup 3 --e2e-steps 1 > $OUT/bench_$cf.json 2> $OUT/bench_$cf.err
done
for cf in cfg6 cfg8 cfg7; do
  timeout 900 python bench.py --config $cf --steps 3 --warmup 3 --e2e-steps 1 > $OUT/bench_$cf.json 2> $OUT/bench_$cf.err
done
timeout 300 python bench.py --impl reference --config cfg2 --steps 3 --warmup 1 > $OUT/ref_cfg2.json 2>&1
# launch lists (cold-cache, serialised: compare shares, not absolutes)
for cf in cfg2 cfg5 cfg1 cfg1m; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cf.csv \
    python bench.py --config $cf --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
# full captures of the dominant kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simplex_reg -c 1 -o $OUT/full_cfg2 \
  python bench.py --config cfg2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hyperbox -c 1 -o $OUT/full_cfg5 \
  python bench.py --config cfg5 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simplex_tiny -c 1 -o $OUT/full_cfg1m \
  python bench.py --config cfg1m --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simplex_block -c 1 -o $OUT/full_cfg3 \
  python scripts/prof_one.py cfg3:444 1 > /dev/null 2>&1
ls -la $OUT
