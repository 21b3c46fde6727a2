# round-2 measurement pass: C5 (default bench config) through scripts/measure.sh,
# bench lines of C2/C3/C4, FIFO budget sweep with external-frontier counts
bash scripts/measure.sh r2 C5
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_r2_$c.json 2> gpurun_out/bench_r2_$c.log; tail -c 600 gpurun_out/bench_r2_$c.json; echo; done
timeout 900 python scripts/budget_sweep.py --config C3 --schedule fifo --budgets-gb 0.25 1 5 16 0 --chunks 128 --out gpurun_out/budget_fifo_C3.json 2>&1 | tail -8
