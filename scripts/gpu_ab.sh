# A/B of env knobs: attention sweep + bench per setting.  Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "exit $?" >> gpurun_out/pt.log
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 200 python scripts/attn_sweep.py $tag > gpurun_out/ab_attn_$tag.txt 2>&1
  env "$@" timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab_bench_$tag.log 2>&1
}
run bal TDPIPE_ATTN_BAL=1
run nobal TDPIPE_ATTN_BAL=0
