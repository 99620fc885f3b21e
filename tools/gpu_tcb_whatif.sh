#!/bin/bash
for c in c2 c3 c4; do timeout 300 python tools/gpu_timing.py $c 2>/dev/null | head -2; done
