"""One fin_ppo_grad call at B = 65,536 on the C1 policy (after warm-up) -- for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_10709_b200 import fin  # noqa: E402
from synth import policy as spol  # noqa: E402

B = 65536
layers = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
g = torch.Generator(device="cuda").manual_seed(9)
x = torch.randn((B, 301), device="cuda", generator=g).to(torch.bfloat16).view(torch.int16)
z = torch.empty((B, 30), dtype=torch.float32, device="cuda")
hid = torch.empty((B, 2, 256), dtype=torch.int16, device="cuda")
a = torch.randn((B, 30), device="cuda", generator=g) * 0.1
lp = torch.zeros(B, device="cuda")
adv = torch.randn(B, device="cuda", generator=g)
ws = [torch.from_numpy((w.astype(np.uint32) << 16).view(np.float32)).cuda() for w, _ in layers]
grads = [(torch.empty_like(w), torch.empty(w.shape[0], device="cuda")) for w in ws]
st = torch.empty(4, dtype=torch.float64, device="cuda")
fin.fin_mlp_forward(pol, x, z, hid)
for _ in range(3):
    fin.fin_ppo_grad(x, hid, z, a, lp, adv, ws[1], ws[2], grads, st)
torch.cuda.synchronize()
print("ok")
