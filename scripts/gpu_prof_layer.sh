mkdir -p gpurun_out
for spec in "8 1000" "64 600" "256 300"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/layer_b$1.csv python scripts/profile_decode.py --layers 2 --b $1 --ctx $2 --steps 2 > gpurun_out/layer_b$1.log 2>&1
done
