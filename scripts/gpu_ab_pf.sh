#!/bin/bash
# A/B: decode attention warming L2 with the O-projection weights (default build)
# vs without (-DTDP_NO_ATTN_PF); chain on/off.  -> gpurun_out/ab_pf.jsonl
O=gpurun_out
for c in 0 1; do TAG=pf timeout 300 python scripts/step_ab.py --chain $c >> $O/ab_pf.jsonl 2>>$O/ab_pf.err; done
TDP_NVCC_DEFINES=-DTDP_NO_ATTN_PF python -m paper_2506_10470_b200.build -j 32 --force > /dev/null 2>&1
for c in 0 1; do TAG=nopf timeout 300 python scripts/step_ab.py --chain $c >> $O/ab_pf.jsonl 2>>$O/ab_pf.err; done
