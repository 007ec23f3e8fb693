#!/bin/bash
# quick GPU A/B: R-class parity subset + cfg2 timing (runs on the GPU box)
OUT=${1:-gpurun_out/rt}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "R and (random or golden or klee or shared)" > $OUT/pytest.txt 2>&1
tail -1 $OUT/pytest.txt
timeout 300 python scripts/quick_time.py cfg2:50000:R cfg2:50000:R > $OUT/time.txt 2>&1
cat $OUT/time.txt
