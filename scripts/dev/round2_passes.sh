#!/bin/bash
# Round-2 GPU passes, one function per pass (usage: bash scripts/dev/round2_passes.sh N);
# README.md maps each pass to the numbers it produced.  Run through gpurun from the repo root.
set -u

pass1() {
  set -x
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p1_smoke.log 2>&1
  timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/p1_tests.log 2>&1; tail -5 gpurun_out/p1_tests.log
  for c in C2 C3 C4 C5; do timeout 600 python scripts/probe.py --config $c --reps 2; done > gpurun_out/p1_probe.log 2>&1
  cat gpurun_out/p1_probe.log
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p1_bench.json 2> gpurun_out/p1_bench.log; tail -c 4000 gpurun_out/p1_bench.json
  for c in C5 C4 C2; do timeout 1200 python scripts/scaling_emulation.py --config $c --gpus 2 4 8 --out gpurun_out/p1_scal_$c.json; done > gpurun_out/p1_scal.log 2>&1
  cat gpurun_out/p1_scal.log
}

pass2() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  echo "== C4 auto"; timeout 120 python scripts/probe.py --config C4 --reps 2 2>&1 | tail -2
  timeout 2700 python -m pytest tests -m gpu -q -x --durations=50 > gpurun_out/p2_tests.log 2>&1; echo "pytest rc=$?"
  tail -75 gpurun_out/p2_tests.log
}

pass3() {
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
}

pass4() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for a in 0.85 0.90 0.97; do echo "== alpha $a"; GSOFA_PART_ALPHA=$a timeout 600 python scripts/scaling_emulation.py --config C5 --gpus 8 --reps 1 2>&1 | tail -3; done
  echo "== wide all ranks"; GSOFA_SOLO_WIDE=1 timeout 600 python scripts/scaling_emulation.py --config C5 --gpus 8 --reps 1 2>&1 | tail -3
  echo "== src trace C5 full"; GSOFA_SRC_TRACE=/tmp/st.bin timeout 300 python scripts/probe.py --config C5 --reps 1 2>&1 | tail -16
  echo "== src trace C5 top range"; GSOFA_SRC_TRACE=/tmp/st2.bin timeout 300 python scripts/probe.py --config C5 --reps 1 --rows 2092230:2097152 2>&1 | tail -16
}

pass5() {
  # A/B of builds on one box (old trees built in-tree under ab_*/), then one
  # ncu --set full capture of the solo kernel on C5's top range (chain-bound)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for t in ab_a4fd076 ab_fe8ee4c .; do
    for c in C5 C2 C3; do
      echo "== $t $c"; (cd $t && timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2")
    done
  done
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:solo_kernel -c 1 \
    -o gpurun_out/prof_solo_C5top_r2 -f python scripts/probe.py --config C5 --reps 1 --rows 2092230:2097152 > gpurun_out/ncu_solo_top.log 2>&1
  echo "ncu rc=$?"; tail -3 gpurun_out/ncu_solo_top.log
}

pass6() {
  # bisect the C5/C2 regression since round 1: each tree is an in-place git
  # archive with its own build and probe (one box, same clocks)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for t in ab_a4fd076 ab_e866041 ab_07bd247 ab_fe8ee4c ab_e49e006 ab_b88768e ab_0524b72 ab_90ed60b ab_6e59a6b ab_89c6d7c ab_17e566f . ab_a4fd076; do
    for c in C5 C2; do
      r=$(cd $t && timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
      echo "$t $c $r"
    done
  done
}

pass7() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 600 python -m pytest tests -m gpu -q -x -k "ell or random_graphs or full_config_exact" > gpurun_out/p7_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p7_tests.log
  for e in 0 1; do for c in C5 C2; do
    r=$(GSOFA_ELL=$e timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "ELL=$e $c $r"
  done; done
  echo "== top range ELL=1"; GSOFA_SRC_TRACE=/tmp/st2.bin timeout 300 python scripts/probe.py --config C5 --reps 2 --rows 2092230:2097152 2>&1 | grep -A4 "^rep 1\|top sources"
  timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 --out gpurun_out/p7_scal_C5.json 2>&1 | tail -3
}

pass8() {
  # round-2 measurement pass: C5 (default bench config) through scripts/measure.sh,
  # bench lines of C2/C3/C4, FIFO budget sweep with external-frontier counts
  bash scripts/measure.sh r2 C5
  for c in C2 C3 C4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_r2_$c.json 2> gpurun_out/bench_r2_$c.log; tail -c 600 gpurun_out/bench_r2_$c.json; echo; done
  timeout 900 python scripts/budget_sweep.py --config C3 --schedule fifo --budgets-gb 0.25 1 5 16 0 --chunks 128 --out gpurun_out/budget_fifo_C3.json 2>&1 | tail -8
}

pass9() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 900 python -m pytest tests -m gpu -q -x -k "team or overflow or auto_threshold_order or solo_shapes or stream_paths" > gpurun_out/p9_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/p9_tests.log
  for tr in 0 448 1024 2048; do
    r=$(GSOFA_TEAM_ROWS=$tr timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C4 team_rows=$tr $r"
  done
  for c in C5 C2; do r=$(timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "$c $r"; done
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 2 4 8 --out gpurun_out/p9_scal_C4.json 2>&1 | tail -8
}

pass10() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for tr in 0 448 1024; do
    r=$(GSOFA_TEAM_ROWS=$tr timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C4 team_rows=$tr $r"
  done
  timeout 600 python -m pytest tests -m gpu -q -x -k "team" 2>&1 | tail -2
}

pass11() {
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p11_smoke.log 2>&1; tail -1 gpurun_out/p11_smoke.log
  timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/p11_tests.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/p11_tests.log
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p11_bench.json 2> gpurun_out/p11_bench.log; python -c "
  import json; d=json.load(open('gpurun_out/p11_bench.json')); print('bench C5', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ncu']['kernels']['solo_kernel']['dram_gbs'], d['clocks'])"
  timeout 600 python bench.py --gpus 2 --config C2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p11_n2_ranges.json 2> gpurun_out/p11_n2_ranges.log; tail -c 400 gpurun_out/p11_n2_ranges.json
  timeout 600 python bench.py --gpus 2 --config C2 --steps 2 --warmup 3 --no-cpu-baseline --layout interleave --unit 32 > gpurun_out/p11_n2_il.json 2> gpurun_out/p11_n2_il.log; tail -c 400 gpurun_out/p11_n2_il.json
}

pass12() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for v in 0 1 0 1; do for c in C5 C2; do
    r=$(GSOFA_ID_R1=$v timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "ID_R1=$v $c $r"
  done; done
  for v in 0 1; do r=$(GSOFA_ID_R1=$v timeout 300 python scripts/probe.py --config C5 --reps 3 --rows 2092230:2097152 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "ID_R1=$v C5top $r"; done
  GSOFA_ID_R1=1 timeout 600 python -m pytest tests -m gpu -q -x -k "random_graphs and threshold or full_config_exact or overflow" 2>&1 | tail -2
}

pass13() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for c in C5 C4 C2 C3; do timeout 1200 python scripts/scaling_emulation.py --config $c --gpus 2 4 8 --out gpurun_out/p13_scal_$c.json 2>&1 | tail -7; done
  bash scripts/measure.sh r2 C2 > gpurun_out/p13_measure_C2.log 2>&1; tail -3 gpurun_out/p13_measure_C2.log
  cat profiles/traffic.json
}

pass14() {
  # per-chain time of C5 top-separator sources: narrow (48 w/SM, 1 batch) vs wide (32 w/SM, 4 batches)
  # with the range small enough for one wave of the wide shape (4736 slots)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for rows in 2092230:2097152 2093056:2097152 2094080:2097152 2095104:2097152; do for w in 0 1; do
    r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C5 --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "rows $rows wide=$w $r"
  done; done
}

pass15() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1200 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode steal --blocks-per-rank 4 --out gpurun_out/p15_steal_C5_4.json 2>&1 | tail -4
  timeout 1200 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode steal --blocks-per-rank 2 --out gpurun_out/p15_steal_C5_2.json 2>&1 | tail -4
  timeout 600 python scripts/scaling_emulation.py --config C4 --gpus 8 --mode steal --out gpurun_out/p15_steal_C4.json 2>&1 | tail -4
  timeout 600 python scripts/scaling_emulation.py --config C2 --gpus 8 --mode steal --out gpurun_out/p15_steal_C2.json 2>&1 | tail -4
}

pass17() {
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for l in default 592 296 148; do for c in C5 C2 C4; do
    if [ "$l" = "default" ]; then unset GSOFA_LIGHT_CTAS; else export GSOFA_LIGHT_CTAS=$l; fi
    r=$(timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "light=$l $c $r"
  done; done
}

pass18() {
  # reached-word cache (GSOFA_RCACHE=1) A/B and parity
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  GSOFA_RCACHE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "random_graphs or full_config_exact or overflow or config_shapes or stream_paths" 2>&1 | tail -2
  for v in 0 1 0 1; do for c in C5 C2; do
    r=$(GSOFA_RCACHE=$v timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*edges \([0-9.e+]*\).*/dev \1 trav \2/')
    echo "RCACHE=$v $c $r"
  done; done
  for v in 0 1; do r=$(GSOFA_RCACHE=$v timeout 300 python scripts/probe.py --config C5 --reps 3 --rows 2092230:2097152 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "RCACHE=$v C5top $r"; done
}

pass19() {
  # final verification of the round's code: build + smoke, full GPU suite, default bench, reference arm
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p19_smoke.log 2>&1; tail -1 gpurun_out/p19_smoke.log
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/p19_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p19_tests.log
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p19_bench.json 2> gpurun_out/p19_bench.log; python -c "
  import json; d=json.load(open('gpurun_out/p19_bench.json')); r=d['roofline']
  print('bench', d['config']['workload'][:20], '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%r['frac'], 'ncu_dram_frac %.4f'%r.get('ncu_dram_frac', -1), 'atomic %.3f'%r['atomic']['frac'], d['clocks'], 'launches', d['gpu_launches'])"
  time (timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/p19_ref.json 2> gpurun_out/p19_ref.log); tail -c 300 gpurun_out/p19_ref.json
}

pass21() {
  # (the team-kernel reruns of this pass were green twice; that kernel is removed since)
  # the suite; parallel host height order (C4 timeline, 1 vs all host threads, hub rank)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  nproc
  timeout 2400 python -m pytest tests -m gpu -q -k "not team_kernel" > gpurun_out/p21_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/p21_tests.log
  for t in 1 0; do
    if [ "$t" = "0" ]; then unset GSOFA_HOST_THREADS; else export GSOFA_HOST_THREADS=$t; fi
    echo "== C4 host threads=$t"; GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep\|height order" | tail -3
    echo "== C4 hub rank host threads=$t"; timeout 300 python scripts/probe.py --config C4 --reps 3 --rows 1584915:1585478 2>&1 | grep "^rep 2"
  done
  unset GSOFA_HOST_THREADS
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 8 --out gpurun_out/p21_scal_C4.json 2>&1 | tail -3
}

pass22() {
  # chain shape (kB = 8, 16 warps/SM): parity, then A/B against the latency shape on the
  # chain-bound ranges (C4 hub rank and its neighbours, C5 top range), full C4, C4 8-way
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1200 python -m pytest tests -m gpu -q -x -k "solo_shapes or auto_chain or auto_threshold" 2>&1 | tail -2
  for rows in 1584915:1585478 1584351:1584915 1583754:1584351; do for w in 1 2; do
    r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C4 --reps 3 --rows $rows 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C4 rows $rows wide=$w $r"
  done; done
  for rows in 2092230:2097152 2087297:2092230; do for w in 0 1 2; do
    r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C5 --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 rows $rows wide=$w $r"
  done; done
  echo "== C4 full auto"; timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2"
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 8 --out gpurun_out/p22_scal_C4.json 2>&1 | tail -3
}

pass23() {
  # C5 8-way with the top separator (the last 16,384 rows) split into four 4,096-row ranks:
  # each fits one wave of the latency shape (32 warps x 148 SMs = 4,736 slots); bulk ranges
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for rows in 2080768:2084864 2084864:2088960 2088960:2093056 2093056:2097152; do for w in 0 1; do
    r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C5 --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 rows $rows wide=$w $r"
  done; done
  for rows in 0:781266 781266:1045051 1045051:1562531 1045051:1600000 1045051:1650000 1562531:2080768 1600000:2080768 1650000:2080768; do
    r=$(timeout 300 python scripts/probe.py --config C5 --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 rows $rows auto $r"
  done
}

pass24() {
  # latency shape for calls with few rows (<= one wave of its 4,736 slots): C2's chain-bound
  # ranks of the 2/4/8-way splits, throughput vs latency shape
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for rows in 256702:258564 258564:259763 259763:260956 260956:262144 257226:259905 259905:262144 257226:262144; do for w in 0 1; do
    r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C2 --reps 3 --rows $rows 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C2 rows $rows wide=$w $r"
  done; done
}

pass25() {
  # AUTO latency shape for one-wave calls: smoke, full suite, C2/C5 emulation, bench (C5) +
  # reference arm + ncu launch list of the bench command
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p25_smoke.log 2>&1; tail -1 gpurun_out/p25_smoke.log
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/p25_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p25_tests.log
  timeout 900 python scripts/scaling_emulation.py --config C2 --gpus 2 4 8 --out gpurun_out/p25_scal_C2.json 2>&1 | tail -7
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p25_bench.json 2> gpurun_out/p25_bench.log; tail -c 600 gpurun_out/p25_bench.json
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/p25_ref.json 2> gpurun_out/p25_ref.log; tail -c 300 gpurun_out/p25_ref.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p25_launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p25_ncu_bench.log 2>&1; echo "ncu rc=$?"
  timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 --out gpurun_out/p25_scal_C5.json 2>&1 | tail -7
}

pass26() {
  # height order in the lockstep kernel (union of the group's same-height thresholds per
  # step; no solo kernel): parity, then C4 A/B against the solo kernel's height order
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1500 python -m pytest tests -m gpu -q -x -k "height or random_graphs or config_shapes or paper_example or solo_shapes or auto_threshold or auto_schedule" 2>&1 | tail -3
  for hs in 0 1; do
    if [ "$hs" = "1" ]; then export GSOFA_HEIGHT_SOLO=1; else unset GSOFA_HEIGHT_SOLO; fi
    echo "== C4 full height_solo=$hs"; GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep" | tail -2
    for rows in 1584915:1585478 1584351:1584915 1583754:1584351 1532558:1583754; do
      r=$(timeout 300 python scripts/probe.py --config C4 --reps 3 --rows $rows 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
      echo "C4 rows $rows height_solo=$hs $r"
    done
  done
  unset GSOFA_HEIGHT_SOLO
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 2 4 8 --out gpurun_out/p26_scal_C4.json 2>&1 | tail -7
}

pass27() {
  # lockstep height order with 16 / 32 warps per CTA (a hub group is one CTA's work)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_height or height_order_hub or auto_threshold" 2>&1 | tail -2
  GSOFA_LOCK_WARPS=32 timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_height" 2>&1 | tail -2
  for lw in 16 32; do
    export GSOFA_LOCK_WARPS=$lw
    echo "== C4 full lock_warps=$lw"; timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2"
    for rows in 1584915:1585478 1584351:1584915 1583754:1584351 1532558:1583754 0:438521; do
      r=$(timeout 300 python scripts/probe.py --config C4 --reps 3 --rows $rows 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
      echo "C4 rows $rows lock_warps=$lw $r"
    done
  done
  unset GSOFA_LOCK_WARPS
}

pass28() {
  # lockstep height order by default (warps per CTA by call size): full suite, C4 timeline, C4 emulation
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p28_smoke.log 2>&1; tail -1 gpurun_out/p28_smoke.log
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/p28_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p28_tests.log
  echo "== C4 full"; GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2\|height order" | tail -2
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 2 4 8 --out gpurun_out/p28_scal_C4.json 2>&1 | tail -7
}

pass29() {
  # lockstep height order on the grids (explicit schedule=height): C5/C2 full and chain-bound ranks
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for rows in 2092230:2097152 2087297:2092230 2082353:2087297 2074239:2082353; do
    r=$(GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config C5 --schedule height --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*rounds \([0-9]*\).*/dev \1 trav \2 rounds \3/')
    echo "C5 rows $rows height $r"
  done
  for rows in 256702:258564 260956:262144 0:97268; do
    r=$(timeout 300 python scripts/probe.py --config C2 --schedule height --reps 3 --rows $rows 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C2 rows $rows height $r"
  done
  echo "== C2 full height"; timeout 300 python scripts/probe.py --config C2 --schedule height --reps 3 2>&1 | grep "^rep 2"
  echo "== C5 full height"; timeout 600 python scripts/probe.py --config C5 --schedule height --reps 2 2>&1 | grep "^rep 1"
}

pass30() {
  # AUTO height order (lockstep) for n >= 2^20: C5 full-size parity, bench, 8-way emulation
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1500 python -m pytest tests -m gpu -q -x -k "full_C5 or full_config or auto_threshold or auto_schedule or l_csc_C5" 2>&1 | tail -3
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p30_bench.json 2> gpurun_out/p30_bench.log; python -c "
import json; d=json.load(open('gpurun_out/p30_bench.json')); r=d['roofline']
print('bench', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%r['frac'], r.get('ncu_dram_frac'), d['config'].get('schedule'), d['clocks'], d['gpu_launches'])"
  timeout 1500 python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 --out gpurun_out/p30_scal_C5.json 2>&1 | tail -7
}

pass31() {
  # measurement of the lockstep height order on C5 (the bench default): ncu launch list of the
  # bench command, ncu --set full of stream_kernel (second launch of a probe), folded into
  # profiles/traffic.json as C5/height; bench lines C4 and C2
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p31_launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p31_ncu_bench.log 2>&1; echo "ncu list rc=$?"
  timeout 2400 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 \
    -o gpurun_out/prof_stream_h_C5 -f python scripts/probe.py --config C5 --reps 2 > gpurun_out/p31_ncu_full.log 2>&1; echo "ncu full rc=$?"
  python scripts/ncu_traffic.py C5 height gpurun_out/ncu_full_r2_C5_height.txt gpurun_out/prof_stream_h_C5.ncu-rep > gpurun_out/p31_traffic.log 2>&1; echo "traffic rc=$?"
  cp profiles/traffic.json gpurun_out/traffic_p31.json
  for c in C4 C2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/p31_bench_$c.json 2> gpurun_out/p31_bench_$c.log; tail -c 300 gpurun_out/p31_bench_$c.json; echo; done
  timeout 1500 python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 --out gpurun_out/p31_scal_C5.json 2>&1 | tail -7
}

pass32() {
  # lockstep height order: warps per CTA on the grids (C5 whole: AUTO; C2: schedule=height)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for lw in 4 16 32; do
    r=$(GSOFA_LOCK_WARPS=$lw timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 lock_warps=$lw $r"
    r=$(GSOFA_LOCK_WARPS=$lw timeout 300 python scripts/probe.py --config C2 --schedule height --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C2 height lock_warps=$lw $r"
  done
}

pass33() {
  # one barrier per lockstep level (three rotating item counts): parity and timings
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1500 python -m pytest tests -m gpu -q -x -k "lockstep_height or height_order_hub or random_graphs or config_shapes or full_config or stream_paths or overflow or budget" 2>&1 | tail -2
  echo "== C5"; timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1"
  echo "== C4"; timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2"
  echo "== C2"; timeout 300 python scripts/probe.py --config C2 --reps 3 2>&1 | grep "^rep 2"
  echo "== C2 height"; timeout 300 python scripts/probe.py --config C2 --schedule height --reps 3 2>&1 | grep "^rep 2"
  r=$(timeout 300 python scripts/probe.py --config C4 --reps 3 --rows 1584915:1585478 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "C4 hub rank $r"
}

pass34() {
  # lockstep height order, 8 vs 16 warps per CTA on C5 (whole) and C4
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for lw in 8 16; do
    r=$(GSOFA_LOCK_WARPS=$lw timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 lock_warps=$lw $r"
    r=$(GSOFA_LOCK_WARPS=$lw timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C4 lock_warps=$lw $r"
  done
  GSOFA_LOCK_WARPS=8 timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_height" 2>&1 | tail -1
}

pass35() {
  # final verification: smoke, full suite, bench (C5) + reference arm, ncu launch list, ncu --set full
  # of the dominant kernel folded into profiles/traffic.json, C4 bench line, C5/C4 emulation
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p35_smoke.log 2>&1; tail -1 gpurun_out/p35_smoke.log
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/p35_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p35_tests.log
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p35_bench.json 2> gpurun_out/p35_bench.log; tail -c 400 gpurun_out/p35_bench.json; echo
  timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/p35_ref.json 2> gpurun_out/p35_ref.log; tail -c 200 gpurun_out/p35_ref.json; echo
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p35_launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p35_ncu_bench.log 2>&1; echo "ncu list rc=$?"
  timeout 2400 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 \
    -o gpurun_out/prof_stream_h8_C5 -f python scripts/probe.py --config C5 --reps 2 > gpurun_out/p35_ncu_full.log 2>&1; echo "ncu full rc=$?"
  python scripts/ncu_traffic.py C5 height gpurun_out/ncu_full_r2_C5_height8.txt gpurun_out/prof_stream_h8_C5.ncu-rep > gpurun_out/p35_traffic.log 2>&1; echo "traffic rc=$?"
  cp profiles/traffic.json gpurun_out/traffic_p35.json
  timeout 900 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/p35_bench_C4.json 2> gpurun_out/p35_bench_C4.log; tail -c 200 gpurun_out/p35_bench_C4.json; echo
  timeout 1500 python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 --out gpurun_out/p35_scal_C5.json 2>&1 | tail -7
  timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 2 4 8 --out gpurun_out/p35_scal_C4.json 2>&1 | tail -7
}

pass36() {
  # dev A/B: the heaviest groups on a 16-warp lockstep kernel, the rest on 4-warp CTAs (C5 whole)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  GSOFA_SPLIT_TOP=5 timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_height" 2>&1 | tail -1
  for k in 148 296 592; do
    r=$(GSOFA_SPLIT_TOP=$k timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 split_top=$k $r"
  done
  r=$(timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "C5 default $r"
}

pass37() {
  # height order (lockstep, 8-warp CTAs / 32 when groups <= SMs) on every rank range of the
  # C5 2/4/8-way splits, against the id order
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for rows in 0:781266 781266:1045051 1045051:1562531 1562531:2074239 2074239:2082353 2082353:2087297 2087297:2092230 2092230:2097152 \
              0:1046157 1046157:2076464 2076464:2087915 2087915:2097152 0:2076464 2076464:2097152; do
    r=$(timeout 600 python scripts/probe.py --config C5 --schedule height --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 rows $rows height $r"
  done
}

pass38() {
  # lockstep height order on C2 / C3 with the final CTA rule (8 warps), and CTA sizes
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for c in C2 C3; do
    for lw in 8 16; do
      r=$(GSOFA_LOCK_WARPS=$lw timeout 300 python scripts/probe.py --config $c --schedule height --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
      echo "$c height lock_warps=$lw $r"
    done
    r=$(timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*\[\([a-z]*\)\].*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/\1 dev \2 trav \3/')
    echo "$c auto $r"
  done
}

pass39() {
  # dev A/B: the heaviest groups on a 16-warp lockstep kernel, the rest on 8-warp CTAs (C5 whole)
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  GSOFA_SPLIT_TOP=5 timeout 900 python -m pytest tests -m gpu -q -x -k "lockstep_height" 2>&1 | tail -1
  for k in 148 296 512; do
    r=$(GSOFA_SPLIT_TOP=$k timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "C5 split_top=$k (16w top, 8w bulk) $r"
  done
  r=$(timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "C5 default $r"
}

pass40() {
  # HEAD check: smoke, full GPU suite, default bench line
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/p40_smoke.log 2>&1; tail -1 gpurun_out/p40_smoke.log
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/p40_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p40_tests.log
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/p40_bench.json 2> gpurun_out/p40_bench.log; tail -c 300 gpurun_out/p40_bench.json; echo
}

pass41() {
  # lockstep height: the next step's record prefetched by the scanning (last) warp, one barrier
  # less per step: parity and timings
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  timeout 1500 python -m pytest tests -m gpu -q -x -k "lockstep_height or height_order_hub or auto_threshold or full_C5 or random_graphs" 2>&1 | tail -1
  for i in 1 2; do
    echo "== C5"; timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1"
    echo "== C4"; timeout 300 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2"
  done
  r=$(timeout 300 python scripts/probe.py --config C4 --reps 3 --rows 1584915:1585478 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "C4 hub rank $r"
}

pass42() {
  # 8-warp lockstep CTAs at 3 per SM (no register spills) vs 4 per SM: C5 whole
  python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
  for i in 1 2; do echo "== C5"; timeout 600 python scripts/probe.py --config C5 --reps 2 2>&1 | grep "^rep 1"; done
}

case "${1:-}" in
  1) pass1 ;;
  2) pass2 ;;
  3) pass3 ;;
  4) pass4 ;;
  5) pass5 ;;
  6) pass6 ;;
  7) pass7 ;;
  8) pass8 ;;
  9) pass9 ;;
  10) pass10 ;;
  11) pass11 ;;
  12) pass12 ;;
  13) pass13 ;;
  14) pass14 ;;
  15) pass15 ;;
  17) pass17 ;;
  18) pass18 ;;
  19) pass19 ;;
  21) pass21 ;;
  22) pass22 ;;
  23) pass23 ;;
  24) pass24 ;;
  25) pass25 ;;
  26) pass26 ;;
  27) pass27 ;;
  28) pass28 ;;
  29) pass29 ;;
  30) pass30 ;;
  31) pass31 ;;
  32) pass32 ;;
  33) pass33 ;;
  34) pass34 ;;
  35) pass35 ;;
  36) pass36 ;;
  37) pass37 ;;
  38) pass38 ;;
  39) pass39 ;;
  40) pass40 ;;
  41) pass41 ;;
  42) pass42 ;;
  *) echo "usage: $0 PASS_NUMBER"; exit 2 ;;
esac
