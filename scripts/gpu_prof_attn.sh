#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_attn" -c 2 -o gpurun_out/attn_b8 python scripts/profile_decode.py --layers 1 --b 8 --ctx 800 --steps 2 --no-prefill > gpurun_out/pa1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_attn" -c 2 -o gpurun_out/attn_b24 python scripts/profile_decode.py --layers 1 --b 24 --ctx 1000 --steps 2 --no-prefill > gpurun_out/pa2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc" -s 4 -c 8 -o gpurun_out/gemm_b64 python scripts/profile_decode.py --layers 1 --b 64 --ctx 500 --steps 3 --no-prefill > gpurun_out/pa3.log 2>&1
