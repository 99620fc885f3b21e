#!/bin/bash
# dev: A/B of build/ab/libhankel_old.so vs the current library on one box (alternating)
for cfg in ${*:-c4}; do
  for r in 1 2; do
    echo "$cfg old: $(HK_LIB_PATH=build/ab/libhankel_old.so python tools/one_run.py $cfg 2 2>&1 | tail -1)"
    echo "$cfg new: $(python tools/one_run.py $cfg 2 2>&1 | tail -1)"
  done
done
