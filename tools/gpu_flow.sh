#!/bin/bash
for p in 0 1; do echo "PDL=$p"; for c in c3 c4; do HK_PDL=$p timeout 300 python tools/gpu_timing.py $c 2>/dev/null | head -1; done; done
