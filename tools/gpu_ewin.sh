#!/bin/bash
mkdir -p gpurun_out
HK_TC=1 HK_TC_EWIN=1 timeout 900 python -m pytest tests -m gpu -q -x -k "not table2" 2>&1 | tail -2
for e in 0 1; do echo "EWIN=$e"; HK_TC_EWIN=$e timeout 300 python tools/gpu_timing.py c3 | head -2; done
HK_TC_EWIN=1 timeout 300 python tools/gpu_timing.py c2 | head -1
timeout 900 python -m pytest tests/test_gpu_table2.py -q -x 2>&1 | tail -3
timeout 1500 python tools/c5_run.py > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 rc=$?"; cat gpurun_out/c5.json; tail -3 gpurun_out/c5.err
