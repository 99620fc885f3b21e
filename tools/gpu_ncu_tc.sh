#!/bin/bash
# ncu --set full captures of the TC bulk kernel and the rounding pass (c3 step 20, c2 step 20).
mkdir -p gpurun_out
HK_TC=1 timeout 600 python tools/one_run.py c3 1 > gpurun_out/plain_c3.log 2>&1 || exit 1
HK_TC=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_tc_bulk|ItemTcRound" -s 40 -c 2 -o gpurun_out/prof_tc_c3 python tools/one_run.py c3 1 > gpurun_out/ncu_full_c3.log 2>&1
HK_TC=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_tc_bulk|ItemTcRound|CItemRecip" -s 60 -c 3 -o gpurun_out/prof_tc_c2 python tools/one_run.py c2 1 > gpurun_out/ncu_full_c2.log 2>&1
echo done
