# reached-word cache (GSOFA_RCACHE=1) A/B and parity
python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
GSOFA_RCACHE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "random_graphs or full_config_exact or overflow or config_shapes or stream_paths" 2>&1 | tail -2
for v in 0 1 0 1; do for c in C5 C2; do
  r=$(GSOFA_RCACHE=$v timeout 300 python scripts/probe.py --config $c --reps 3 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*edges \([0-9.e+]*\).*/dev \1 trav \2/')
  echo "RCACHE=$v $c $r"
done; done
for v in 0 1; do r=$(GSOFA_RCACHE=$v timeout 300 python scripts/probe.py --config C5 --reps 3 --rows 2092230:2097152 2>&1 | grep "^rep 2" | sed 's/.*dev \([0-9.]*\) ms  trav \([0-9.]*\).*/dev \1 trav \2/'); echo "RCACHE=$v C5top $r"; done
