#!/bin/bash
# ncu --set full of one mid-LDLT k_tc_bulk launch (dev): $1 = config, $2 = launches to skip
mkdir -p gpurun_out
cfg=${1:-c3}; skip=${2:-100}
timeout 300 python tools/one_run.py $cfg 1 > gpurun_out/plain_tcb_$cfg.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_tc_bulk" -s $skip -c 1 -o gpurun_out/prof_tcb_$cfg python tools/one_run.py $cfg 1 > gpurun_out/ncu_tcb_$cfg.log 2>&1
echo done
