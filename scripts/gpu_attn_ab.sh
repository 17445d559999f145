#!/bin/bash
# decode-attention variant A/B: parity tests, isolated sweep, decode-step times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/pt.log 2>&1; echo "exit $?" >> gpurun_out/pt.log
timeout 300 python scripts/attn_sweep.py ${TAG_A:-new} > gpurun_out/attn_sweep_a.txt 2>&1
env ${ENV_B} timeout 300 python scripts/attn_sweep.py ${TAG_B:-old} > gpurun_out/attn_sweep_b.txt 2>&1
out=gpurun_out/step_ab.jsonl; : > $out
run() { tag=$1; shift; env TAG=$tag "$@" timeout 300 python scripts/step_ab.py >> $out 2>> gpurun_out/step_ab.err; }
run ${TAG_A:-new}; run ${TAG_B:-old} ${ENV_B}; run ${TAG_A:-new}2; run ${TAG_B:-old}2 ${ENV_B}
