#!/bin/bash
# One measurement pass on the GPU box: smoke, bench JSON, ncu launch list of
# the bench command, ncu --set full captures of the traversal kernels folded
# into profiles/traffic.json.  Usage: scripts/measure.sh TAG [CONFIG]
TAG=${1:-r2}; CFG=${2:-C5}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1
python bench.py --config $CFG --steps 5 --warmup 3 > $OUT/bench_${TAG}_${CFG}.json 2> $OUT/bench_${TAG}_${CFG}.log
tail -c 3000 $OUT/bench_${TAG}_${CFG}.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_${TAG}_${CFG}.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_bench_${TAG}.log 2>&1
REPS=""
for K in solo_kernel stream_kernel; do
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:$K -s 1 -c 1 -o $OUT/prof_${K}_${TAG}_${CFG} -f \
    python scripts/probe.py --config $CFG --reps 2 > $OUT/ncu_full_${K}_${TAG}.log 2>&1
REPS="$REPS $OUT/prof_${K}_${TAG}_${CFG}.ncu-rep"
done
python scripts/ncu_traffic.py $CFG threshold $OUT/ncu_full_${TAG}_${CFG}.txt $REPS > /dev/null 2>&1
cp profiles/traffic.json $OUT/traffic_${TAG}.json
ls -la $OUT
