#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/one_run.py c2 1 > gpurun_out/plain_c2.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ItemTcRound" -s 20 -c 1 -o gpurun_out/prof_round_c2 python tools/one_run.py c2 1 > gpurun_out/ncu_round.log 2>&1
echo done
