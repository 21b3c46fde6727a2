python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
for l in default 592 296 148; do for c in C5 C2 C4; do
  if [ "$l" = "default" ]; then unset GSOFA_LIGHT_CTAS; else export GSOFA_LIGHT_CTAS=$l; fi
  r=$(timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
  echo "light=$l $c $r"
done; done
