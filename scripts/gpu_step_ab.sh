#!/bin/bash
# A/B of engine knobs on the per-step time of an 8-layer 7B-shaped stage.
mkdir -p gpurun_out
out=gpurun_out/step_ab.jsonl; : > $out
run() { tag=$1; shift; env TAG=$tag "$@" timeout 300 python scripts/step_ab.py ${ARGS} >> $out 2>> gpurun_out/step_ab.err; }
for v in ${VARIANTS:-base}; do
  case $v in
    base) run base ;;
    nopdl) run nopdl TDPIPE_PDL=0 ;;
    qkv2) run qkv2 TDPIPE_SPLITS_QKV=2 ;;
    *) run $v ;;
  esac
done
