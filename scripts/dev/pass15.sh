python -c "from paper_2007_00840_b200.build import build; build()" > /dev/null 2>&1
timeout 1200 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode steal --blocks-per-rank 4 --out gpurun_out/p15_steal_C5_4.json 2>&1 | tail -4
timeout 1200 python scripts/scaling_emulation.py --config C5 --gpus 8 --mode steal --blocks-per-rank 2 --out gpurun_out/p15_steal_C5_2.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C4 --gpus 8 --mode steal --out gpurun_out/p15_steal_C4.json 2>&1 | tail -4
timeout 600 python scripts/scaling_emulation.py --config C2 --gpus 8 --mode steal --out gpurun_out/p15_steal_C2.json 2>&1 | tail -4
