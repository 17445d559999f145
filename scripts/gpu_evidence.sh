#!/bin/bash
# Evidence for profiles/: the bench line, ncu launch-list windows of one bench
# step, and `ncu --set full` summaries of the top kernels.  1 GPU.  Reports are
# summarised on the box (scripts/summarize.py, scripts/ncu_summary.py) and the
# large .ncu-rep files are dropped.  Outputs -> gpurun_out/
mkdir -p gpurun_out /tmp/ev
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_final.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 1200 ncu --metrics $M --clock-control none -s 48000 -c 4000 --csv --log-file /tmp/ev/launches_bench_prefill.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-timing > gpurun_out/ev1.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -s 150000 -c 4000 --csv --log-file /tmp/ev/launches_bench_decode.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-timing > gpurun_out/ev2.log 2>&1
python scripts/summarize.py /tmp/ev/launches_bench_prefill.csv /tmp/ev/launches_bench_decode.csv > gpurun_out/launches_bench_windows.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_attn|gemm_tc" -c 6 -o /tmp/ev/ncu_decode_b256 python scripts/profile_decode.py --layers 1 --b 256 --ctx 300 --steps 1 --no-prefill > gpurun_out/ev3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_attn|gemm_tc" -c 6 -o /tmp/ev/ncu_decode_b8 python scripts/profile_decode.py --layers 1 --b 8 --ctx 800 --steps 1 --no-prefill > gpurun_out/ev4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tn|flash_prefill" -c 6 -o /tmp/ev/ncu_prefill python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/ev5.log 2>&1
for r in ncu_decode_b256 ncu_decode_b8 ncu_prefill; do
  python scripts/ncu_summary.py /tmp/ev/$r.ncu-rep > gpurun_out/$r.txt 2>&1
done
