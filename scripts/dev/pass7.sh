python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "ell or random_graphs or full_config_exact" > gpurun_out/p7_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p7_tests.log
for e in 0 1; do for c in C5 C2; do
  r=$(GSOFA_ELL=$e timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
  echo "ELL=$e $c $r"
done; done
echo "== top range ELL=1"; GSOFA_SRC_TRACE=/tmp/st2.bin timeout 300 python scripts/probe.py --config C5 --reps 2 --rows 2092230:2097152 2>&1 | grep -A4 "^rep 1\|top sources"
timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 --out gpurun_out/p7_scal_C5.json 2>&1 | tail -3
