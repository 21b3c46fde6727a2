GW=paper_2007_00840_b200/libgsofa_gw.so
echo "== gw nosolo top rows only"; GSOFA_LIB=$GW GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/t1.bin timeout 120 python scripts/probe.py --config C2 --reps 1 --rows 258048:262144 | head -9
echo "== gw nosolo full C2"; GSOFA_LIB=$GW GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/t2.bin timeout 120 python scripts/probe.py --config C2 --reps 1 | head -9
echo "== gw nosolo 1 CTA/SM"; GSOFA_LIB=$GW GSOFA_SOLO_CTAS=0 GSOFA_LIGHT_CTAS=1184 GSOFA_GROUP_TRACE=/tmp/t3.bin timeout 120 python scripts/probe.py --config C2 --reps 1 | head -9
