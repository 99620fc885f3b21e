#!/bin/bash
# default-policy GPU tests + forced-TC tests + timings + launch lists (c2, c3); run under gpurun.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
HK_TC=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in c1 c2 c3; do timeout 900 python tools/gpu_timing.py $cfg 2>&1 | head -2; done
for cfg in c2 c3; do
  timeout 600 python tools/one_run.py $cfg 2 > gpurun_out/one_$cfg.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
     --log-file gpurun_out/launches_tc_$cfg.csv python tools/one_run.py $cfg 1 > gpurun_out/ncu_$cfg.log 2>&1
done
echo done
