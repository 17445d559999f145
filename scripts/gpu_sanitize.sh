# compute-sanitizer racecheck / synccheck / memcheck on the tiny parity tests
# (C1 end to end, tiny GQA / GQA-8 stage forward).  Logs -> gpurun_out/sanitizer/
set -u
mkdir -p gpurun_out/sanitizer
python -m paper_2506_10470_b200.build -j 16 > gpurun_out/sanitizer/build.log 2>&1 || { echo build failed; exit 1; }
SEL="test_td_run_c1_teacher_forced or test_stage_forward_prefill_then_decode or test_gqa_small_batch_32_token_splits or test_decode_attention_long_context"
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer/summary.txt
done
cat gpurun_out/sanitizer/summary.txt
