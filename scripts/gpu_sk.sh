mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k stream_k > gpurun_out/pt_sk.log 2>&1; echo "exit $?" >> gpurun_out/pt_sk.log
timeout 300 python scripts/gemm_sk_sweep.py > gpurun_out/gemm_sk_sweep.txt 2>&1
