#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc" -c 4 -o gpurun_out/prof_prefill python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/prof_p1.log 2>&1
