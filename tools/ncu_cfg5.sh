#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, one GPU): launch list of set_rhs + 1 V-cycle + norm,
# then one --set full capture each of the level-4 sweep, fused residual + restriction and thin ghost kernel.
# Usage: bash tools/ncu_cfg5.sh <tag>   ->  gpurun_out/<tag>_{launches.csv,sweep4,rr2_4,thin4}.ncu-rep
set -x
T=${1:-cfg5}
python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/${T}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/${T}_l.log 2>&1
for k in k_rb_pencil:sweep4 k_rr2_pencil:rr2_4 k_c2f_thin:thin4; do
  ncu --set full --clock-control none --import-source on -k regex:${k%%:*} -s ${2:-0} -c 1 -f -o gpurun_out/${T}_${k##*:} python tools/prof_vcycle.py --cfg cfg5 --cycles 1 > gpurun_out/${T}_${k##*:}.log 2>&1
done
ls -la gpurun_out/${T}_*.ncu-rep
