#!/bin/bash
# ncu --set full captures of the TC bulk kernel and the rounding pass (c3, early LDLT steps).
mkdir -p gpurun_out
timeout 600 python tools/one_run.py c3 1 > gpurun_out/plain_c3.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_tc_bulk|ItemTcRound" -s 30 -c 3 -o gpurun_out/prof_tc_c3 python tools/one_run.py c3 1 > gpurun_out/ncu_full_c3.log 2>&1
echo done
