"""Dev: run a config with the GSOFA_PROF build and print the solo kernel's cycle accounting."""
import os, subprocess, sys
import numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
rows = sys.argv[2] if len(sys.argv) > 2 else None
out = "/tmp/prof.bin"
if os.path.exists(out):
    os.remove(out)
env = dict(os.environ, GSOFA_LIB=os.path.join(root, "paper_2007_00840_b200", "libgsofa_prof.so"), GSOFA_PROF=out)
cmd = [sys.executable, os.path.join(root, "scripts", "probe.py"), "--config", cfg, "--reps", "1"]
if rows:
    cmd += ["--rows", rows]
print(subprocess.run(cmd, env=env, capture_output=True, text=True).stdout.strip().splitlines()[-1])
h = np.fromfile(out, dtype=np.uint64).reshape(-1, 16)[-1]
names = ["next-threshold", "window misses", "step start", "expand", "worklist", "levels", "steps", "ring levels"]
cyc = h[[0, 2, 3, 4]].astype(float)
tot = cyc.sum()
for i, nm in zip([0, 2, 3, 4], ["next-threshold", "step start", "expand", "worklist"]):
    print(f"  {nm:15s} {h[i]/tot*100:5.1f}%  {h[i]/max(1,h[5]):8.0f} cyc/level  {h[i]/max(1,h[6]):8.0f} cyc/step")
print(f"  levels {h[5]}  steps {h[6]}  window misses {h[1]} ({h[1]/max(1,h[6])*100:.1f}% of steps)  ring levels {h[7]}")
print(f"  total {tot/max(1,h[5]):.0f} cyc/level, {tot/max(1,h[6]):.0f} cyc/step")
