# tests of the new paths + A/B of the split-K CTA target.  Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "exit $?" >> gpurun_out/pt.log
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab_bench_$tag.log 2>&1
}
run t288 TDPIPE_SPLIT_TARGET=288
run t148 TDPIPE_SPLIT_TARGET=148
run t444 TDPIPE_SPLIT_TARGET=444
run t592 TDPIPE_SPLIT_TARGET=592
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --policy pphb > gpurun_out/ab_bench_pphb.log 2>&1
timeout 300 python scripts/attn_sweep.py gqa8 > gpurun_out/attn_sweep_gqa8.txt 2>&1
