#!/bin/bash
# decode-attention launch-plan sweep: CTA target per SM x largest split
mkdir -p gpurun_out; out=gpurun_out/attn_plan.txt; : > $out
for tgt in 8 4 2 1; do for mx in 512 1024 4096; do
  TDPIPE_ATTN_TARGET=$tgt TDPIPE_ATTN_MAXSPLIT=$mx timeout 200 python scripts/attn_sweep.py t${tgt}_m${mx} >> $out 2>&1
done; done
