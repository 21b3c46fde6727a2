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
