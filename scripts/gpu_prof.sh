#!/bin/bash
# ncu captures for the decode kernels (1 GPU).  Outputs -> gpurun_out/
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_decode.csv python scripts/profile_decode.py --layers 2 --b 256 --ctx 300 --steps 3 --no-prefill > gpurun_out/prof_run1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_decode_b32.csv python scripts/profile_decode.py --layers 2 --b 32 --ctx 600 --steps 3 --no-prefill > gpurun_out/prof_run2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|decode_attn" -c 6 -o gpurun_out/prof_decode python scripts/profile_decode.py --layers 1 --b 256 --ctx 300 --steps 1 --no-prefill > gpurun_out/prof_run3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|decode_attn" -c 6 -o gpurun_out/prof_decode_b32 python scripts/profile_decode.py --layers 1 --b 32 --ctx 600 --steps 1 --no-prefill > gpurun_out/prof_run4.log 2>&1
