import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd()+'/tests'); sys.path.insert(0, os.getcwd()+'/tests/golden')
import numpy as np, torch
from conftest import plaw8k_csr
from oracle import rowwin_oracle as orc
import paper_2412_08902_b200 as hc
from paper_2412_08902_b200.model import Gcn2
a_ref = plaw8k_csr(); n = a_ref.num_rows
a = hc.SparseCsr(n, n, a_ref.row_ptr, a_ref.col_idx, a_ref.values)
ws = hc.partition(a)
x = torch.from_numpy(orc.random_dense(n, 128, 3)).float().cuda()
labels = torch.from_numpy(np.random.default_rng(2).integers(0, 41, n)).cuda()
rows = np.repeat(np.arange(n), np.diff(a_ref.row_ptr))
ad = torch.zeros((n, n), dtype=torch.float64); ad[torch.from_numpy(rows), torch.from_numpy(a_ref.col_idx)] = torch.from_numpy(a_ref.values)
for prec_ref in ["f64"]:
    adr = ad.cuda()
    m = Gcn2(128, 64, 41, seed=0)
    rw1 = m.w1.detach().double().clone().requires_grad_(True); rw2 = m.w2.detach().double().clone().requires_grad_(True)
    h1 = adr @ x.double() @ rw1
    logits = adr @ torch.relu(h1) @ rw2
    loss_ref = torch.nn.functional.cross_entropy(logits, labels); loss_ref.backward()
    # also bf16-emulated reference: round X, A to bf16
    loss = m.epoch(x, labels, ws)
    for nm, g, r in [("w1", m.w1.grad, rw1.grad), ("w2", m.w2.grad, rw2.grad)]:
        d = (g.double() - r).abs()
        print(nm, "maxrel", float(d.max()/r.abs().max()), "relfro", float(d.norm()/r.norm()), "near-zero pre-acts", int((h1.abs() < 1e-3).sum()))
