#!/bin/bash
# ncu --set full of one mid-LDLT certified-rounding launch (dev): $1 = config, $2 = launches to skip
mkdir -p gpurun_out
cfg=${1:-c3}; skip=${2:-100}
timeout 300 python tools/one_run.py $cfg 1 > gpurun_out/plain_$cfg.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ItemTcRound" -s $skip -c 1 -o gpurun_out/prof_round_$cfg python tools/one_run.py $cfg 1 > gpurun_out/ncu_round_$cfg.log 2>&1
echo done
