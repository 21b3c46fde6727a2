set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p1_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/p1_tests.log 2>&1; tail -5 gpurun_out/p1_tests.log
for c in C2 C3 C4 C5; do timeout 600 python scripts/probe.py --config $c --reps 2; done > gpurun_out/p1_probe.log 2>&1
cat gpurun_out/p1_probe.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p1_bench.json 2> gpurun_out/p1_bench.log; tail -c 4000 gpurun_out/p1_bench.json
for c in C5 C4 C2; do timeout 1200 python scripts/scaling_emulation.py --config $c --gpus 2 4 8 --out gpurun_out/p1_scal_$c.json; done > gpurun_out/p1_scal.log 2>&1
cat gpurun_out/p1_scal.log
