# A/B of env knobs: attention sweep + bench per setting.  Outputs -> gpurun_out/
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 200 python scripts/attn_sweep.py $tag > gpurun_out/ab_attn_$tag.txt 2>&1
  env "$@" timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab_bench_$tag.log 2>&1
}
run base TDPIPE_X=0
run cps16 TDPIPE_ATTN_CPS=16
run qkv1 TDPIPE_QKV_SPLIT1=1
