#!/bin/bash
# TC-path launch lists (c2 with HK_TC=1, c3) + the c4 golden parity test; run under gpurun.
mkdir -p gpurun_out
HK_TC=1 timeout 900 python -m pytest tests -m gpu -q -x -k c4 > gpurun_out/c4_test.log 2>&1; echo "rc=$?" >> gpurun_out/c4_test.log
for cfg in c2 c3; do
  HK_TC=1 timeout 600 python tools/one_run.py $cfg 2 > gpurun_out/one_$cfg.log 2>&1 && \
  HK_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
     --log-file gpurun_out/launches_tc_$cfg.csv python tools/one_run.py $cfg 1 > gpurun_out/ncu_$cfg.log 2>&1
done
echo done
