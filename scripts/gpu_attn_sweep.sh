mkdir -p gpurun_out
rm -f gpurun_out/attn_sweep3.txt
echo "== v1" >> gpurun_out/attn_sweep3.txt
TDPIPE_ATTN_RING=0 timeout 200 python scripts/attn_sweep.py 3 >> gpurun_out/attn_sweep3.txt 2>&1
for c in 592 1184 2368; do
  echo "== sk$c" >> gpurun_out/attn_sweep3.txt
  TDPIPE_SK_CTAS=$c TDPIPE_SK_MIN=64 timeout 200 python scripts/attn_sweep.py 2 >> gpurun_out/attn_sweep3.txt 2>&1
done
echo "== v2" >> gpurun_out/attn_sweep3.txt
TDPIPE_ATTN_V2=1 timeout 200 python scripts/attn_sweep.py 1 >> gpurun_out/attn_sweep3.txt 2>&1
