#!/bin/bash
# dev: fix counts and what-if timings of the fused product kernel (results wrong with knobs)
for c in c2 c3 c4; do echo "$c"; python tools/one_run.py $c 1 2>&1 | tail -1; done
for spec in "HK_DEV_TCB=256" "HK_DEV_TCB=768" "HK_DEV_TCB=784"; do
  echo "== $spec"; env $spec timeout 600 python tools/one_run.py c4 2 2>&1 | tail -1
done
