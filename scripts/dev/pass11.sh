python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p11_smoke.log 2>&1; tail -1 gpurun_out/p11_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/p11_tests.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/p11_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p11_bench.json 2> gpurun_out/p11_bench.log; python -c "
import json; d=json.load(open('gpurun_out/p11_bench.json')); print('bench C5', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ncu']['kernels']['solo_kernel']['dram_gbs'], d['clocks'])"
timeout 600 python bench.py --gpus 2 --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p11_n2_ranges.json 2> gpurun_out/p11_n2_ranges.log; tail -c 400 gpurun_out/p11_n2_ranges.json
timeout 600 python bench.py --gpus 2 --config C2 --steps 2 --warmup 3 --no-cpu-baseline --layout interleave --unit 32 > gpurun_out/p11_n2_il.json 2> gpurun_out/p11_n2_il.log; tail -c 400 gpurun_out/p11_n2_il.json
