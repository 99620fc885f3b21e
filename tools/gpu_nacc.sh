timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for n in 1 2; do echo "NACC=$n"; HK_TC_NACC=$n timeout 300 python tools/gpu_timing.py c2 | head -2; done
HK_TC_NACC=1 timeout 300 python tools/gpu_timing.py c3 | head -1
