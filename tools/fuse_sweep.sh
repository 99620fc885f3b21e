#!/bin/bash
# dev: fused vs separate rounding pass, same box
for c in c2 c3 c4; do tools/env_sweep.sh $c "HK_TC_FUSE=0" "HK_TC_FUSE=1"; done
