python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
mkdir -p gpurun_out
for v in old new; do
  lib=$L/libgsofa.so; [ $v = old ] && lib=$L/libgsofa_old.so
  GSOFA_LIB=$lib timeout 900 ncu --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis \
     --section SourceCounters --section LaunchStats --section Occupancy --clock-control none --import-source on \
     -k regex:solo_kernel -c 1 -o gpurun_out/solo_$v -f python scripts/probe.py --config C2 --reps 1 > gpurun_out/ncu_solo_$v.log 2>&1
  tail -2 gpurun_out/ncu_solo_$v.log
done
