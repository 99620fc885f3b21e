#!/bin/bash
# LDLT chunk-group sweep (dev)
for g in 1 2 3; do echo "G=$g"; HK_TC_GROUPS=$g timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -2; done
echo "G=auto"; timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -2
timeout 200 python tools/gpu_timing.py c3 2>/dev/null | head -1
