#!/bin/bash
mkdir -p gpurun_out
{
for v in "HK_LDLT_FLOW=1" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_WARPOPS=128" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_WARPOPS=128 HK_LDLT_FLOW_THREADS=64" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_WARPOPS=128 HK_LDLT_FLOW_THREADS=256"; do
  echo "== c1 $v"; env $v timeout 120 python tools/one_run.py c1 4 2>&1 | tail -2
done
for shape in "1,1,128,64,8" "1,2,128,120,8" "1,2,32,24,8"; do
  for v in "HK_LDLT_FLOW=0" "HK_LDLT_FLOW=1" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_WARPOPS=128"; do
    echo "== shape $shape $v"; env $v timeout 120 python tools/one_shape.py $shape 3 2>&1 | tail -1
  done
done
} > gpurun_out/lflow_times2.txt 2>&1
HK_LDLT_FLOW_WARPOPS=128 timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -x -q -k "dataflow or path_bit_exact or precision" > gpurun_out/lflow_tests2.log 2>&1; echo "tests rc=$?"
