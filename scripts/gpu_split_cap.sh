#!/bin/bash
O=gpurun_out
for r in 1 2; do
for v in 8 4 6; do
  TDP_NVCC_DEFINES="-DTDP_RESID_MAX_SPLITS=$v" python -m paper_2506_10470_b200.build -j 32 --force > /dev/null 2>&1
  echo "cap=$v $(timeout 300 python scripts/kernel_timeline.py --b 1 4 8 16 2>/dev/null | python -c '
import json,sys
print([(d["b"], d["step_us"], d["classes"]["gemm_o"]["marginal_us_per_step"], d["classes"]["gemm_down"]["marginal_us_per_step"], d["classes"]["resid_norm_cluster"]["marginal_us_per_step"]) for d in map(json.loads, sys.stdin)])')" >> $O/split_cap.txt
done; done
