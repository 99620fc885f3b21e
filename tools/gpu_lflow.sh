#!/bin/bash
# dev: the dataflow LDLT (k_ldlt_flow): tests under a timeout, then C1 and other
# small-p timings with the flow kernel on / off and several CTA sizes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py -x -q -k "dataflow or timing" > gpurun_out/lflow_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "path_bit_exact or precision or small_cases or deterministic or c1_parity" >> gpurun_out/lflow_tests.log 2>&1; echo "tests2 rc=$?"
{
for cfg in c1; do
  for v in "HK_LDLT_FLOW=0" "HK_LDLT_FLOW=1" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_THREADS=64" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_THREADS=96" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_THREADS=192" "HK_LDLT_FLOW=1 HK_LDLT_FLOW_THREADS=256" "HK_LDLT_FLOW=1 HK_FLOW_SLEEP=20" "HK_LDLT_FLOW=1 HK_FLOW_SLEEP=400"; do
    echo "== $cfg $v"; env $v timeout 120 python tools/one_run.py $cfg 4 2>&1 | tail -2
  done
done
for shape in "1,1,128,64,8" "1,1,256,96,8" "1,2,128,120,8" "1,2,200,100,8" "1,1,256,120,8"; do
  for v in "HK_LDLT_FLOW=0" "HK_LDLT_FLOW=1"; do
    echo "== shape $shape $v"; env $v timeout 120 python tools/one_shape.py $shape 3 2>&1 | tail -1
  done
done
} > gpurun_out/lflow_times.txt 2>&1
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/lflow_bench_c1.json 2> gpurun_out/lflow_bench_c1.err; echo "c1 bench rc=$?"
