#!/bin/bash
# dev: pair kernel occupancy + issuer wait profile at C4 (full stderr)
for spec in "HK_TC_PAIR=1 HK_DEV_TCB=192" "HK_TC_PAIR=0 HK_DEV_TCB=64"; do
  echo "== $spec"; env $spec HK_INV_FLOW=1 timeout 600 python tools/one_run.py c4 1 2>&1 | tail -4
done
