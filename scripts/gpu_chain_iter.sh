#!/bin/bash
# One GPU iteration on the decode chain: kernel tests, engine parity (chain on/off),
# step A/B, then a TDP_CHAIN_TRACE build + per-op trace.  Output: gpurun_out/iter_*.
set -u
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k chain > $O/iter_kern.log 2>&1; tail -1 $O/iter_kern.log
timeout 300 python scripts/dbg_chain.py > $O/iter_dbg.log 2>&1; cat $O/iter_dbg.log
for c in ${CHAINS:-0 1}; do timeout 300 python scripts/step_ab.py --chain $c ${STEP_ARGS:-} >> $O/iter_step.jsonl 2>> $O/iter_step.err; done
tail -2 $O/iter_step.jsonl
if [ -z "${NO_TRACE:-}" ]; then
  TDP_NVCC_DEFINES=-DTDP_CHAIN_TRACE python -m paper_2506_10470_b200.build -j 32 --force > /dev/null 2>&1
  timeout 300 python scripts/chain_trace.py ${TRACE_ARGS:-} > $O/iter_trace.txt 2>&1
fi
