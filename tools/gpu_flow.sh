#!/bin/bash
for t in 64 128 256; do echo "threads=$t"; HK_FLOW_THREADS=$t timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -1; HK_FLOW_THREADS=$t timeout 200 python tools/gpu_timing.py c1 2>/dev/null | head -1; done
