#!/bin/bash
# Dev: time one config under several env settings (last of 3 reps each).
#   tools/env_sweep.sh c4 "HK_TC_FUSE=0" "HK_TC_FUSE=1" "HK_TC_FUSE=1 HK_TC_SLEEP=100" ...
cfg=$1; shift
for spec in "$@"; do
  line=$(env $spec timeout 600 python tools/one_run.py $cfg 3 2>&1 | tail -2 | tr "\n" " ")
  echo "$cfg [$spec] $line"
done
