#!/bin/bash
# dev: pair kernel occupancy + issuer wait profile at C4 (full stderr)
for spec in "HK_TC_PAIR=1 HK_DEV_TCB=192" "HK_TC_PAIR=1 HK_TC_PAIR_STAGES=4" "HK_TC_PAIR=1 HK_TC_PAIR_STAGES=6" "HK_TC_PAIR=0"; do
  echo "== $spec"; env $spec timeout 600 python tools/one_run.py c4 2 2>&1 | tail -3
done
