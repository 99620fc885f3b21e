#!/bin/bash
for t in 128 192 256; do echo "cta threads=$t"; HK_CTA_THREADS=$t timeout 200 python tools/gpu_timing.py c2 2>/dev/null | head -1; HK_CTA_THREADS=$t timeout 200 python tools/gpu_timing.py c3 2>/dev/null | head -1; done
