#!/bin/bash
# quick GPU A/B for the M/L classes: parity subset + cfg3 / big-cluster timing
OUT=${1:-gpurun_out/lt}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -x -q -k "L or M" > $OUT/pytest.txt 2>&1
tail -1 $OUT/pytest.txt
timeout 600 python scripts/quick_time.py cfg3:2000 cfg8:300 cfg7:100 > $OUT/time.txt 2>&1
cat $OUT/time.txt
