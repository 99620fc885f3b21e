#!/bin/bash
# ncu --set full of the dataflow L^-1 kernel at C2 (dev)
mkdir -p gpurun_out
timeout 300 python tools/one_run.py c2 1 > gpurun_out/plain_flow.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_inv_flow" -c 1 -o gpurun_out/prof_flow_c2 python tools/one_run.py c2 1 > gpurun_out/ncu_flow.log 2>&1
echo done
