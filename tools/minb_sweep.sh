for mb in 3 4; do
  sed -i "s/-DHK_TRAILING2_MINB=[0-9]/-DHK_TRAILING2_MINB=$mb/" Makefile; touch paper_1810_01478_b200/csrc/hk_api.cu
  make -j8 > /dev/null 2>&1
  echo "== minb=$mb"; python tools/gpu_timing.py c2 2>&1 | head -2; python tools/gpu_timing.py c3 2>&1 | head -2
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
