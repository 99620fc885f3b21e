#!/bin/bash
# dataflow L^-1 timing sweep (dev)
for f in 2 1 0; do for s in 0 100; do echo "flow=$f sleep=$s"; HK_INV_FLOW=$f HK_FLOW_SLEEP=$s timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -1; done; done
for f in 2 0; do HK_INV_FLOW=$f timeout 200 python tools/gpu_timing.py c1 2>/dev/null | head -1; done
