python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
for a in 0.85 0.90 0.97; do echo "== alpha $a"; GSOFA_PART_ALPHA=$a timeout 600 python scripts/scaling_emulation.py --config C5 --gpus 8 --reps 1 2>&1 | tail -3; done
echo "== wide all ranks"; GSOFA_SOLO_WIDE=1 timeout 600 python scripts/scaling_emulation.py --config C5 --gpus 8 --reps 1 2>&1 | tail -3
echo "== src trace C5 full"; GSOFA_SRC_TRACE=/tmp/st.bin timeout 300 python scripts/probe.py --config C5 --reps 1 2>&1 | tail -16
echo "== src trace C5 top range"; GSOFA_SRC_TRACE=/tmp/st2.bin timeout 300 python scripts/probe.py --config C5 --reps 1 --rows 2092230:2097152 2>&1 | tail -16
