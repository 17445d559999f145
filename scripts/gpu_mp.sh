#!/bin/bash
# Multi-process (one process per stage) checks on ONE GPU: every rank on cuda:0.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pt_mp.log 2>&1; echo "exit $?" >> gpurun_out/pt_mp.log
export TDPIPE_SAME_DEVICE=1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --config C1 --model tiny --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mp_c1.log 2>&1; echo "exit $?" >> gpurun_out/bench_mp_c1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --steps 1 --warmup 3 --kv-blocks 4096 --no-cpu-baseline > gpurun_out/bench_mp_c2.log 2>&1; echo "exit $?" >> gpurun_out/bench_mp_c2.log
