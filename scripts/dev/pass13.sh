python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
for c in C5 C4 C2 C3; do timeout 1200 python scripts/scaling_emulation.py --config $c --gpus 2 4 8 --out gpurun_out/p13_scal_$c.json 2>&1 | tail -7; done
bash scripts/measure.sh r2 C2 > gpurun_out/p13_measure_C2.log 2>&1; tail -3 gpurun_out/p13_measure_C2.log
cat profiles/traffic.json
