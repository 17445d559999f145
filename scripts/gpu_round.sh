#!/bin/bash
# One GPU session: tests, smoke, bench.  Outputs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for f in ${TESTS:-tests}; do
  n=$(basename $f .py)
  timeout ${TEST_TIMEOUT:-900} python -m pytest $f -m gpu -q -p no:cacheprovider --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_$n.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$n.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
fi
