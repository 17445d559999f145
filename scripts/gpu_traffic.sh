# DRAM traffic of decode_attn launches (engine path) for bench.py's roofline.traffic.  1 GPU.
mkdir -p gpurun_out
A=""
for B in 4 32 256; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:decode_attn --clock-control none --csv --log-file gpurun_out/traffic_b$B.csv python scripts/traffic_attn.py $B 2 > gpurun_out/traffic_b$B.json 2> gpurun_out/traffic_b$B.err
  A="$A gpurun_out/traffic_b$B.csv gpurun_out/traffic_b$B.json"
done
python scripts/traffic_summary.py gpurun_out/traffic_decode_attn.json $A > gpurun_out/traffic_summary.log 2>&1
