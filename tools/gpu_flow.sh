#!/bin/bash
for c in c1 c2 c3; do timeout 300 python tools/gpu_timing.py $c 2>/dev/null | head -1; done
