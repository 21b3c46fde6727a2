#!/bin/bash
# One measurement pass on the GPU box: smoke, bench JSON, ncu launch list,
# ncu full capture of the solo traversal kernel.  Usage: scripts/measure.sh TAG [CONFIG]
TAG=${1:-r1}; CFG=${2:-C2}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1
python bench.py --config $CFG --steps 5 --warmup 3 > $OUT/bench_${TAG}_${CFG}.json 2> $OUT/bench_${TAG}_${CFG}.log
tail -c 3000 $OUT/bench_${TAG}_${CFG}.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_bench_${TAG}.log 2>&1
for K in solo_kernel stream_kernel; do
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:$K -s 1 -c 1 -o $OUT/prof_${K}_${TAG}_${CFG} -f \
    python scripts/probe.py --config $CFG --reps 2 > $OUT/ncu_full_${K}_${TAG}.log 2>&1
done
ls -la $OUT
