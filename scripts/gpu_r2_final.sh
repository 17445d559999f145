# Round-2 final evidence (1 GPU; outputs -> gpurun_out/):
#  1. bench.py (defaults) -> bench_final.log
#  2. ncu launch-list windows of the same bench command (gpu__time_duration, DRAM bytes):
#     the prefill phase and the small-batch decode tail -> launches_bench_windows.txt
#  3. ncu --set full: MHA SIMT decode attention at a small batch, GQA-8 tensor-core
#     attention, a small-batch decode GEMM and a prefill GEMM -> ncu_*.txt summaries
set -u
mkdir -p gpurun_out /tmp/ev
python -m paper_2506_10470_b200.build -j 16 > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
if [ "${SKIP_BENCH:-0}" != 1 ]; then
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_final.log
fi
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-timing --no-c5-stage"
timeout 1200 ncu --metrics $M --clock-control none -s 48000 -c 3000 --csv --log-file /tmp/ev/launches_bench_prefill.csv $B > gpurun_out/ev1.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -s 150000 -c 3000 --csv --log-file /tmp/ev/launches_bench_decode.csv $B > gpurun_out/ev2.log 2>&1
python scripts/summarize.py /tmp/ev/launches_bench_prefill.csv /tmp/ev/launches_bench_decode.csv > gpurun_out/launches_bench_windows.txt 2>&1
cat > /tmp/one_attn.py <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from paper_2506_10470_b200.tdpipe import td_bench_attn
n, H, Hkv, impl = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rng = np.random.default_rng(0)
ctx = np.clip(rng.lognormal(6.3, 0.8, n), 32, 4000).astype(np.int32)
print(td_bench_attn(ctx, H, Hkv, 128, iters=3, impl=impl))
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn -s 3 -c 1 \
  -o /tmp/ev/ncu_attn_mha_b4 python /tmp/one_attn.py 4 32 32 1 > gpurun_out/ev3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_attn -s 3 -c 1 \
  -o /tmp/ev/ncu_attn_gqa8_b256 python /tmp/one_attn.py 256 64 8 0 > gpurun_out/ev4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|gemm_tnp" -c 8 \
  -o /tmp/ev/ncu_decode_b8 python scripts/profile_decode.py --layers 1 --b 8 --ctx 800 --steps 1 --no-prefill > gpurun_out/ev5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gemm_tnp|flash_prefill" -c 6 \
  -o /tmp/ev/ncu_prefill python scripts/profile_decode.py --layers 1 --b 7 --ctx 292 --steps 0 --prefill-only > gpurun_out/ev6.log 2>&1
for r in ncu_attn_mha_b4 ncu_attn_gqa8_b256 ncu_decode_b8 ncu_prefill; do
  python scripts/ncu_summary.py /tmp/ev/$r.ncu-rep > gpurun_out/$r.txt 2>&1
  ncu -i /tmp/ev/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
done
