#!/bin/bash
# dev: the on-device moment generator (tests, sanitizer on a small case, C2/C4 bench lines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py -q -k "moments" > gpurun_out/mom_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python -m pytest tests/test_cpp_facade.py tests/test_gpu_table2.py -m gpu -q > gpurun_out/mom_facade.log 2>&1; echo "facade rc=$?"
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_api.py -q -k "moments and (beta0-64 or beta8 or beta10)" > gpurun_out/mom_race.log 2>&1; echo "race rc=$?"
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mom_bench_c2.json 2> gpurun_out/mom_bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mom_bench_c4.json 2> gpurun_out/mom_bench_c4.err; echo "c4 rc=$?"
