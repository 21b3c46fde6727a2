#!/bin/bash
# quick GPU iteration: parity tests (threshold schedule) + probe timings + C2 group trace
# usage: scripts/quick.sh TAG [configs...]
TAG=${1:-q}; shift
CFGS=${@:-C2 C3 C4 C5}
mkdir -p gpurun_out
python -c "from paper_2007_00840_b200.build import build; build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; tail -3 gpurun_out/${TAG}_tests.log
for c in $CFGS; do timeout 300 python scripts/probe.py --config $c --reps 2; done > gpurun_out/${TAG}_probe.log 2>&1
grep -v "^  " gpurun_out/${TAG}_probe.log
GSOFA_GROUP_TRACE=/tmp/tr.bin timeout 300 python scripts/probe.py --config C2 --reps 1 2>&1 | head -8
