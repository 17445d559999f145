# A/B: decode attention as a PDL dependent for small batches (compile-time
# TDP_ATTN_PDL_MAXN = 0 / 8 / 32), C2 bench, no cpu baseline / c5 stage.
set -u
mkdir -p gpurun_out
for MX in 0 8 32; do
  TDP_NVCC_DEFINES="-DTDP_ATTN_PDL_MAXN=$MX" python -m paper_2506_10470_b200.build -j 16 --force > gpurun_out/build_pdl$MX.log 2>&1
  timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-c5-stage > gpurun_out/bench_pdl$MX.log 2>&1
done
python - <<'PY'
import json
for mx in (0, 8, 32):
    l = [x for x in open(f"gpurun_out/bench_pdl{mx}.log") if x.startswith("{")]
    if not l:
        print(mx, "no line"); continue
    d = json.loads(l[-1]); k = d["kernels"]
    print(mx, round(d["value"], 1), {b: (k[b]["ms"], k[b]["hbm_frac"]) for b in ["decode_attn@b1-8", "decode_attn@b9-32", "gemm_dec@b1-8", "gemm_dec@b9-32"]})
PY
