mkdir -p gpurun_out/r2d
python scripts/ab.py ab/compact ab/cl4 -- cfg3:2000 cfg3:2000::4 cfg3s:2000::4 cfg6:1000 cfg6:1000::8 cfg8:200 > gpurun_out/r2d/ab.txt 2>&1
