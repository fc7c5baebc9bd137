#!/bin/bash
# Launch list + one full ncu capture of the top GEMM for the C2 bench (1 GPU).
set -x
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 4 -o gpurun_out/prof_c2 -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
