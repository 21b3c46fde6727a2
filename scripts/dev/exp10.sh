python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
for v in base m2; do
  lib=$L/libgsofa.so; [ $v = m2 ] && lib=$L/libgsofa_m2.so
  for sc in 16 36 71; do
  echo "== $v rows 258777:259905 solo ctas $sc"; GSOFA_LIB=$lib GSOFA_SOLO_CTAS=$sc timeout 120 python scripts/probe.py --config C2 --reps 2 --rows 258777:259905 | tail -1
  done
done
git -C . status > /dev/null 2>&1
GSOFA_LIB=$L/libgsofa_old.so timeout 120 python scripts/probe.py --config C2 --reps 2 --rows 258777:259905 | tail -1
