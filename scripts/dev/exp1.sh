python -c "from paper_2007_00840_b200.build import build; build()"
echo "== top group alone"; python scripts/probe.py --config C2 --reps 2 --rows 262112:262144 | tail -1
echo "== top 4096 rows"; python scripts/probe.py --config C2 --reps 2 --rows 258048:262144 | tail -1
for L in 148 296 592; do for S in 148 296; do echo "== light $L solo $S"; GSOFA_LIGHT_CTAS=$L GSOFA_SOLO_CTAS=$S python scripts/probe.py --config C2 --reps 2 | tail -1; done; done
echo "== C5 light 296 solo 296"; GSOFA_LIGHT_CTAS=296 python scripts/probe.py --config C5 --reps 2 | tail -1
