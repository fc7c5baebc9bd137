#!/bin/bash
# Round evidence (1 GPU, under gpurun): GPU tests, bench lines + launch lists for
# every config (tools/prof_round.sh), the C4 tensor-pipe table (tools/ncu_class.py,
# replaying the unprofiled run's autotuning decisions), allocator-poison parity.
set -x
mkdir -p gpurun_out
T=${1:-r02f}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputest.log 2>&1
tail -2 gpurun_out/${T}_gputest.log
bash tools/prof_round.sh $T "${2:-c4 c2 c3 c5 c6 c7 c1}" > /dev/null 2>&1
BE_TUNE_FILE=/tmp/be_tune_${T}_c4.txt ncu --nvtx --nvtx-include "timed/" -k regex:"gemm_tc|conv_" --clock-control none --csv \
  --log-file gpurun_out/${T}_c4_tensor_ncu.csv \
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  python tools/ncu_class.py run c4 gpurun_out/${T}_c4_tensor_prof.json > gpurun_out/${T}_ncu_class_run.log 2>&1
BE_ALLOC_POISON=1 timeout 1500 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_mlp.py tests/test_gpu_mobile.py tests/test_gpu_sparse.py -q -x > gpurun_out/${T}_poison.txt 2>&1
tail -1 gpurun_out/${T}_poison.txt
for c in ${2:-c4 c2 c3 c5 c6 c7 c1}; do python -c "import json; d=json.loads(open('gpurun_out/${T}_'+'$c'+'_bench.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])"; done
