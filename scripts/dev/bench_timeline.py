"""Dev: the bench's call pattern (torch stream, device tensors, L2 flush,
free per step) with the library's GSOFA_TIMELINE dump."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

rp, ci = gen.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
d_rp, d_ci = torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()
ctx = g.Context(0)
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(4):
    if i == 3:
        os.environ["GSOFA_TIMELINE"] = "1"
    flush.zero_()
    r = g.symbolic(d_rp, d_ci, ctx=ctx, stream=stream, outputs_on_device=True)
    print(f"step {i}: ms_total {r.stats['ms_total']:.1f} traverse {r.stats['ms_traverse']:.1f}", flush=True)
    r.free()
