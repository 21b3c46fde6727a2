python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "interleave or cap_only or external or etree" > gpurun_out/p3_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p3_tests.log
for c in C2 C5; do GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config $c --reps 2 2>&1 | tail -22; done > gpurun_out/p3_probe.log 2>&1
grep "^rep" gpurun_out/p3_probe.log
timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 --out gpurun_out/p3_scal_C5_ranges.json 2>&1 | tail -8
timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode interleave --unit 128 --out gpurun_out/p3_scal_C5_il128.json 2>&1 | tail -4
timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode interleave --unit 32 --out gpurun_out/p3_scal_C5_il32.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C4 --gpus 8 --out gpurun_out/p3_scal_C4_ranges.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C4 --gpus 8 --mode interleave --unit 128 --out gpurun_out/p3_scal_C4_il128.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C2 --gpus 8 --out gpurun_out/p3_scal_C2_ranges.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C2 --gpus 8 --mode interleave --unit 128 --out gpurun_out/p3_scal_C2_il128.json 2>&1 | tail -4
