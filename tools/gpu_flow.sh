#!/bin/bash
for t in 96 128 160 192; do echo "threads=$t"; HK_FLOW_THREADS=$t timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -1; done
