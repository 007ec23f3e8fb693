mkdir -p gpurun_out/r2e
python scripts/ab.py ab/compact ab/tinyp ab/tinyp4 ab/tinyp5 -- cfg1m:1000000 cfg1m:1000000:S cfg1:1000 cfg9:50000 > gpurun_out/r2e/ab.txt 2>&1
python scripts/phase_prof.py cfg2:50000 > gpurun_out/r2e/phase_cfg2.txt 2>&1
python scripts/phase_prof.py cfg2:296 > gpurun_out/r2e/phase_cfg2_alone.txt 2>&1
