#!/bin/bash
# dev: is the fused epilogue's cost its uncoalesced row accesses? (results wrong; 768 = ignore pivots, no fix list)
for spec in "HK_DEV_TCB=768" "HK_DEV_TCB=2816" "HK_DEV_TCB=784" "HK_DEV_TCB=768"; do
  echo "== $spec $(env $spec timeout 600 python tools/one_run.py c4 2 2>&1 | tail -1)"
done
