python -c "from paper_2007_00840_b200.build import build; build()"
W1=paper_2007_00840_b200/libgsofa_w1.so
for c in C2 C3 C5; do
echo "== $c default"; python scripts/probe.py --config $c --reps 2 | tail -1
echo "== $c w1 no solo"; GSOFA_LIB=$W1 GSOFA_SOLO_CTAS=0 python scripts/probe.py --config $c --reps 2 | tail -1
echo "== $c w4 no solo"; GSOFA_SOLO_CTAS=0 python scripts/probe.py --config $c --reps 2 | tail -1
done
echo "== C2 w1 trace"; GSOFA_LIB=$W1 GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/t.bin python scripts/probe.py --config C2 --reps 1 | head -8
