#!/bin/bash
# Per-round profile capture (1 GPU, under gpurun):
#   bench lines for every config, and for each config the ncu launch list of
#   the K timed steps only (NVTX range "timed" pushed by bench.py).  The bench
#   run records its autotuning decisions (BE_TUNE_FILE) and the profiled run
#   replays them: under ncu every launch is serialised and replayed, which
#   would distort the tuner's timings and change the kernels chosen.
# usage: tools/prof_round.sh r01 "c2 c4 c3 c5 c1"
R=${1:-r01}
CFGS=${2:-"c2 c4 c3 c5 c1"}
mkdir -p gpurun_out
for c in $CFGS; do
  TF=/tmp/be_tune_${R}_${c}.txt
  rm -f $TF
  BE_TUNE_FILE=$TF python bench.py --config $c --steps 30 --warmup 5 --cpu-budget 10 > gpurun_out/${R}_${c}_bench.json 2> gpurun_out/${R}_${c}_bench.err
  BE_TUNE_FILE=$TF ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${R}_${c}_launches.csv \
      python bench.py --config $c --steps 2 --warmup 3 --tune-steps 24 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out
