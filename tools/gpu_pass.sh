#!/bin/bash
# One GPU pass (dev): GPU tests, the default bench (C4), C2 bench, ncu of the
# product / rounding kernels at C4, and the reference arm at C4.
#   tools/gpu_pass.sh TAG [tests] [bench] [c2] [ncu] [ref]
tag=${1:-r02}; shift
what=${*:-tests bench c2 ncu ref}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
nproc > gpurun_out/${tag}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${tag}_nproc.txt
for w in $what; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "tests rc=$?";;
    bench) timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "bench rc=$?";;
    c2) timeout 300 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; echo "c2 rc=$?";;
    c1) timeout 300 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/${tag}_bench_c1.json 2> gpurun_out/${tag}_bench_c1.err; echo "c1 rc=$?";;
    ncuflow)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ldlt_flow -s 2 -c 1 \
        -o gpurun_out/${tag}_prof_lflow_c1 -f python tools/one_run.py c1 4 > gpurun_out/${tag}_ncu_lflow_c1.log 2>&1; echo "ncu lflow rc=$?"
      ;;
    c3) timeout 300 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/${tag}_bench_c3.json 2> gpurun_out/${tag}_bench_c3.err; echo "c3 rc=$?";;
    ncu)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_bulk -s 300 -c 1 \
        -o gpurun_out/${tag}_prof_tcb_c4 -f python tools/one_run.py c4 1 > gpurun_out/${tag}_ncu_tcb_c4.log 2>&1; echo "ncu tcb rc=$?"
      ;;
    launches)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 6000 \
        --log-file gpurun_out/${tag}_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_launches_c4.log 2>&1; echo "launches rc=$?";;
    sweep) tools/env_sweep.sh c4 "HK_TC_FUSE=0" "HK_TC_FUSE=1" "HK_TC_FUSE=1 HK_TC_SLEEP=64" "HK_TC_FUSE=1 HK_TC_SLEEP=256" "HK_TC_FUSE=0 HK_TC_SLEEP=128" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    c5pin) timeout 1500 python tools/c5_pin.py > gpurun_out/${tag}_c5pin.json 2> gpurun_out/${tag}_c5pin.err; echo "c5pin rc=$?";;
    fusedtests) timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -x -q -k "fused or tc or c4 or c2" > gpurun_out/${tag}_gputests.log 2>&1; echo "fusedtests rc=$?";;
    sweep3) tools/env_sweep.sh c4 "HK_TC_FUSE=0" "HK_TC_FUSE=0 HK_TC_STAGES=3" "HK_TC_FUSE=1" "HK_TC_FUSE=1 HK_DEV_TCB=16" "HK_TC_FUSE=1 HK_TC_STAGES=2" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    sweep4) tools/env_sweep.sh c4 "HK_TC_FUSE=0 HK_DEV_TCB=64" "HK_TC_FUSE=1 HK_DEV_TCB=64" "HK_TC_FUSE=1" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    c5) timeout 900 python tools/one_run.py c5 1 > gpurun_out/${tag}_c5.txt 2>&1; echo "c5 rc=$?";;
    steps) timeout 600 python tools/step_profile.py c4 > gpurun_out/${tag}_steps_c4.json 2>&1; echo "steps rc=$?";;
    pairtests) timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -k "fused or tc or c4 or c2 or c3 or path" > gpurun_out/${tag}_gputests.log 2>&1; echo "pairtests rc=$?";;
    sweep5) tools/env_sweep.sh c4 "HK_TC_PAIR=0" "HK_TC_PAIR=1" "HK_TC_PAIR=1 HK_TC_STAGES=2" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    sweep6) tools/env_sweep.sh c4 "HK_TC_PAIR=1 HK_DEV_TCB=192" "HK_TC_PAIR=0 HK_DEV_TCB=64" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    sweep2) tools/env_sweep.sh c4 "HK_TC_FUSE=0" "HK_TC_FUSE=1" > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?";;
    ref) timeout 1500 python bench.py --impl reference --steps 1 --warmup 0 --ref-golden-precision > gpurun_out/${tag}_ref_c4.json 2> gpurun_out/${tag}_ref_c4.err; echo "ref rc=$?";;
  esac
done
