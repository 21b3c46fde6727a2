python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "team or overflow or auto_threshold_order or solo_shapes or stream_paths" > gpurun_out/p9_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/p9_tests.log
for tr in 0 448 1024 2048; do
  r=$(GSOFA_TEAM_ROWS=$tr timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
  echo "C4 team_rows=$tr $r"
done
for c in C5 C2; do r=$(timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "$c $r"; done
timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 2 4 8 --out gpurun_out/p9_scal_C4.json 2>&1 | tail -8
