#!/bin/bash
# ncu launch lists (gpu__time_duration) of the bench command at C4 / C2 / C1 — each after its own plain run exited 0
tag=${1:-r02s}
mkdir -p gpurun_out
for cfg in c1 c2 c4; do
  n=6000; [ $cfg = c2 ] && n=4000; [ $cfg = c1 ] && n=400
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_plain_$cfg.json 2> gpurun_out/${tag}_plain_$cfg.err || { echo "$cfg plain run failed"; continue; }
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c $n \
    --log-file gpurun_out/${tag}_launches_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_launches_$cfg.log 2>&1; echo "$cfg launches rc=$?"
done
