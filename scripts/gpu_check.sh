# tests + attention sweep + bench (1 GPU).  Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "exit $?" >> gpurun_out/pt.log
timeout 200 python scripts/attn_sweep.py ${TAG:-v1} > gpurun_out/attn_sweep.txt 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
