#!/bin/bash
# Round-end evidence on one B200: full GPU test suite, smoke, bench (+ oracle
# baseline), ncu launch windows + `--set full` summaries (scripts/gpu_evidence.sh),
# multi-process bench on one GPU.  Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
bash scripts/gpu_evidence.sh
TDPIPE_SAME_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --config C1 --model tiny --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mp_c1.log 2>&1; echo "exit $?" >> gpurun_out/bench_mp_c1.log
