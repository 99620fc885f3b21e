#!/bin/bash
# dev: what-if timings of the fused product kernel at C4 (results wrong; 256|512 keep every step running, no fix-up storm)
for spec in "HK_DEV_TCB=768" "HK_DEV_TCB=784" "HK_DEV_TCB=800" "HK_DEV_TCB=1792" "HK_DEV_TCB=1824" "HK_DEV_TCB=771"; do
  echo "== $spec"; env HK_TC_PAIR=0 $spec timeout 600 python tools/one_run.py c4 2 2>&1 | tail -1
done
