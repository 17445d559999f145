#!/bin/bash
# ncu evidence for profiles/: bench launch-list windows + full captures of the top kernels.  1 GPU.
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 1200 ncu --metrics $M --clock-control none -s 48000 -c 4000 --csv --log-file gpurun_out/launches_bench_prefill.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-timing > gpurun_out/ev1.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -s 150000 -c 4000 --csv --log-file gpurun_out/launches_bench_decode.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-timing > gpurun_out/ev2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_attn|gemm_tc" -c 6 -o gpurun_out/ncu_decode_b256 python scripts/profile_decode.py --layers 1 --b 256 --ctx 300 --steps 1 --no-prefill > gpurun_out/ev3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_attn|gemm_tc" -c 6 -o gpurun_out/ncu_decode_b8 python scripts/profile_decode.py --layers 1 --b 8 --ctx 800 --steps 1 --no-prefill > gpurun_out/ev4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tn|flash_prefill" -c 6 -o gpurun_out/ncu_prefill python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/ev5.log 2>&1
timeout 600 python scripts/gemm_sweep.py > gpurun_out/sweep.log 2>&1
timeout 300 python scripts/gemm_prefill.py > gpurun_out/gemm_prefill.txt 2>&1
