# final verification of the round's code: build + smoke, full GPU suite, default bench, reference arm
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p19_smoke.log 2>&1; tail -1 gpurun_out/p19_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/p19_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p19_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p19_bench.json 2> gpurun_out/p19_bench.log; python -c "
import json; d=json.load(open('gpurun_out/p19_bench.json')); r=d['roofline']
print('bench', d['config']['workload'][:20], '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%r['frac'], 'ncu_dram_frac %.4f'%r.get('ncu_dram_frac', -1), 'atomic %.3f'%r['atomic']['frac'], d['clocks'], 'launches', d['gpu_launches'])"
time (timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/p19_ref.json 2> gpurun_out/p19_ref.log); tail -c 300 gpurun_out/p19_ref.json
