# per-chain time of C5 top-separator sources: narrow (48 w/SM, 1 batch) vs wide (32 w/SM, 4 batches)
# with the range small enough for one wave of the wide shape (4736 slots)
python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
for rows in 2092230:2097152 2093056:2097152 2094080:2097152 2095104:2097152; do for w in 0 1; do
  r=$(GSOFA_SOLO_WIDE=$w timeout 300 python scripts/probe.py --config C5 --reps 2 --rows $rows 2>&1 | grep "^rep 1" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
  echo "rows $rows wide=$w $r"
done; done
