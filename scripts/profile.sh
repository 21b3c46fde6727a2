#!/bin/bash
# ncu full capture of the streaming traversal kernel on CONFIG (default C2)
TAG=${1:-r1b}; CFG=${2:-C2}; KER=${3:-stream_kernel}
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on --replay-mode application \
    -k regex:$KER -s 1 -c 1 -o gpurun_out/prof_${KER}_${TAG}_${CFG} -f \
    python scripts/probe.py --config $CFG --reps 2 > gpurun_out/ncu_${KER}_${TAG}_${CFG}.log 2>&1
tail -5 gpurun_out/ncu_${KER}_${TAG}_${CFG}.log
