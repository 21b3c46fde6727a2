python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
echo "== C4 auto"; timeout 120 python scripts/probe.py --config C4 --reps 2 2>&1 | tail -2
timeout 2700 python -m pytest tests -m gpu -q -x --durations=50 > gpurun_out/p2_tests.log 2>&1; echo "pytest rc=$?"
tail -75 gpurun_out/p2_tests.log
