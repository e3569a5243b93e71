"""Build one scale-mode level's block ILU and run a few forward sweeps (ncu driver).
    python tools/bilu_prof.py p n"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import structured as S  # noqa: E402

p, n = int(sys.argv[1]), int(sys.argv[2])
prob = S.helmholtz_box_problem((n, n, n), p, c=10.0)
sm = prob["M"].smoothers[0]
r = prob["b"].clone()
out = torch.empty_like(r)
for _ in range(3):
    sm.forward_into(r, out)
torch.cuda.synchronize()
print("ok")
