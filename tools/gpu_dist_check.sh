#!/bin/bash
# NCCL sharded path through bench.py on one GPU (torchrun, world 1, forced sharded).
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --sharded --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err
echo "sharded bench rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_torchrun.json 2>&1
echo "ref torchrun rc=$?"
