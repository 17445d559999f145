#!/bin/bash
mkdir -p gpurun_out
TDPIPE_MC=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc" -c 4 -o gpurun_out/prof_prefill_mc0 python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/prof_p1.log 2>&1
TDPIPE_MC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc" -c 4 -o gpurun_out/prof_prefill_mc1 python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/prof_p2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_attn" -c 3 -o gpurun_out/prof_dattn_b8 python scripts/profile_decode.py --layers 1 --b 8 --ctx 800 --steps 1 --no-prefill > gpurun_out/prof_p3.log 2>&1
