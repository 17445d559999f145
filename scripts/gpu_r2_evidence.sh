# Round-2 evidence on one B200 (outputs -> gpurun_out/):
#  1. compute-sanitizer memcheck/racecheck/synccheck on the tiny + GQA parity
#     tests (the tensor-core decode-attention pipeline included)
#  2. ncu DRAM traffic of the bench job's OWN decode_attn launches
#     (scripts/traffic_job.py: one C2 td_run) -> profiles/rN/traffic_decode_attn.json
#  3. ncu --set full of one GQA-8 tensor-core attention launch and one decode GEMM
#  4. the §4.4 ablations (measured C2-cap on one stage; projections) + trace
set -u
mkdir -p gpurun_out/sanitizer
python -m paper_2506_10470_b200.build -j 16 > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
if [ "${SKIP_SAN:-0}" != 1 ]; then
SEL="test_td_run_c1_teacher_forced or test_stage_forward_prefill_then_decode or test_gqa_small_batch_32_token_splits or test_decode_attention_long_context or test_td_run_trace"
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/summary.txt
done
fi
if [ "${SKIP_TRAFFIC:-0}" != 1 ]; then
# windows of the job's 32,736 decode_attn launches: the b = 256 start, the middle, the small-batch tail
W=""
for SK in 0 14000 28000; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:decode_attn -s $SK -c 1500 \
    --clock-control none --csv --log-file gpurun_out/traffic_w$SK.csv python scripts/traffic_job.py decode_attn \
    > gpurun_out/traffic_job_$SK.json 2> gpurun_out/traffic_job_$SK.err
  W="$W $SK:gpurun_out/traffic_w$SK.csv"
done
python scripts/traffic_windows.py gpurun_out/traffic_decode_attn.json $W > gpurun_out/traffic_summary.log 2>&1
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
cat > /tmp/one_attn.py <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from paper_2506_10470_b200.tdpipe import td_bench_attn
rng = np.random.default_rng(0)
ctx = np.clip(rng.lognormal(6.3, 0.8, 256), 32, 4000).astype(np.int32)
print(td_bench_attn(ctx, 64, 8, 128, iters=3))
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn_tc -s 4 -c 1 \
  -o gpurun_out/ncu_attn_gqa8_tc python /tmp/one_attn.py > gpurun_out/ncu_attn.log 2>&1
ncu -i gpurun_out/ncu_attn_gqa8_tc.ncu-rep --page details --csv > gpurun_out/ncu_attn_gqa8_tc.csv 2>/dev/null
fi
if [ "${SKIP_ABL:-0}" != 1 ]; then
timeout 1500 python scripts/ablations.py AB > gpurun_out/ablations.log 2>&1
fi
cat gpurun_out/sanitizer/summary.txt 2>/dev/null
