# bisect the C5/C2 regression since round 1: each tree is an in-place git
# archive with its own build and probe (one box, same clocks)
python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
for t in ab_a4fd076 ab_e866041 ab_07bd247 ab_fe8ee4c ab_e49e006 ab_b88768e ab_0524b72 ab_90ed60b ab_6e59a6b ab_89c6d7c ab_17e566f . ab_a4fd076; do
  for c in C5 C2; do
    r=$(cd $t && timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
    echo "$t $c $r"
  done
done
