python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
timeout 400 python -m pytest tests -m gpu -q -x -k "team" 2>&1 | tail -3
for tr in 0 448 1024; do
  r=$(GSOFA_TEAM_DEBUG=1 GSOFA_TEAM_ROWS=$tr timeout 200 python scripts/probe.py --config C4 --reps 3 2>&1 | grep "^rep 2\|team" | tail -2 | tr '\n' ' ' | sed 's/rep 2.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/')
  echo "C4 team_rows=$tr $r"
done
for tr in 0 448; do r=$(GSOFA_TEAM_DEBUG=1 GSOFA_TEAM_ROWS=$tr timeout 200 python scripts/probe.py --config C4 --reps 3 --rows 1584915:1585478 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "C4 hub rank team_rows=$tr $r"; done
