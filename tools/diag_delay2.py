"""Delay and reverb levels at short lengths (1,000-4,000 samples): device KERNELS vs the oracle."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import normrel
from golden_inputs import kernel_inputs
from oracle import mixgraph_oracle as O
from paper_2509_15948_b200.processors import KERNELS
for tag in "dr":
    for L in (1000, 1231, 1500, 2000, 2047, 2048, 2049, 2500, 2999, 3072, 4000):
        u, p, w = kernel_inputs(tag)
        if L > u.shape[-1]:
            rng = np.random.default_rng(L); u = 0.3 * rng.standard_normal((2, 2, L)); w = rng.standard_normal((2, 2, L))
        u = u[..., :L].copy(); w = w[..., :L].copy()
        ut = torch.tensor(u, dtype=torch.float32, device="cuda", requires_grad=True)
        pt = torch.tensor(p, dtype=torch.float64, device="cuda", requires_grad=True)
        yb, reg = KERNELS[tag](ut, pt)
        (torch.sum(yb.double() * torch.tensor(w, device="cuda")) + reg).backward()
        uo = torch.tensor(u.astype(np.float32).astype(np.float64), requires_grad=True); po = torch.tensor(p, requires_grad=True)
        yo, ro = O.KERNELS[tag](uo, po)
        (torch.sum(yo * torch.tensor(w)) + ro).backward()
        print(tag, L, "y %.1e gu %.1e gp %.1e" % (normrel(yb.detach().cpu().numpy(), yo.detach().numpy()),
              normrel(ut.grad.cpu().numpy(), uo.grad.numpy()), normrel(pt.grad.cpu().numpy(), po.grad.numpy(), floor=1e-6)), flush=True)
