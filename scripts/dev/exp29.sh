L=paper_2007_00840_b200
for v in ns "" ns ""; do echo "== C5top256 ${v:-base}"; GSOFA_LIB=$L/libgsofa${v:+_$v}.so timeout 200 python scripts/probe.py --config C5 --reps 2 --rows 2096896:2097152 | tail -1 | cut -c1-60; done
for v in ns ""; do echo "== C4hubs ${v:-base}"; GSOFA_LIB=$L/libgsofa${v:+_$v}.so timeout 200 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60; done
