"""One cfg2-shaped sample_batch (states + FP4 operand) for ncu captures of sample_rows_kernel."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17066_b200 as P  # noqa: E402

torch.cuda.set_device(0)
m = int(os.environ.get("M", "2"))
probs = [0.1, 0.9] if m == 2 else [0.05, 0.15, 0.8]
d = P.ComponentDistribution.iid(295, probs)
S = 1 << 20
st = torch.empty((S, 295), dtype=torch.uint8, device="cuda")
rb = P._abi.fp4_row_bytes(295, m)
a4 = torch.empty((S, 2 * rb), dtype=torch.uint8, device="cuda")
for g in range(3):
    P.sample_batch(d, S, 0, g, out_states=st, out_fp4=a4)
torch.cuda.synchronize()
print("ok")
