#!/bin/bash
# dev: what-if timings of the fused product kernel at C4 (results wrong with knobs 1/2/16; 256 keeps every step running)
for spec in "HK_TC_PAIR=0" "HK_TC_PAIR=0 HK_DEV_TCB=256" "HK_TC_PAIR=0 HK_DEV_TCB=272" "HK_TC_PAIR=0 HK_DEV_TCB=259" "HK_TC_PAIR=0 HK_DEV_TCB=275" "HK_TC_PAIR=1 HK_DEV_TCB=272"; do
  echo "== $spec"; env $spec timeout 600 python tools/one_run.py c4 2 2>&1 | tail -1
done
