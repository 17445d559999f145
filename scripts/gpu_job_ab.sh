#!/bin/bash
# same-box job A/B: this build vs -D overrides (OLD_DEFS), C2 bench + c5_stage
O=$PWD/gpurun_out
B="python bench.py --no-cpu-baseline --steps 2"
timeout 900 $B > $O/jab2_new1.json 2>/dev/null
TDP_NVCC_DEFINES="$OLD_DEFS" python -m paper_2506_10470_b200.build -j 32 --force > /dev/null 2>&1
timeout 900 $B > $O/jab2_old.json 2>/dev/null
python -m paper_2506_10470_b200.build -j 32 --force > /dev/null 2>&1
timeout 900 $B > $O/jab2_new2.json 2>/dev/null
