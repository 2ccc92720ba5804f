"""Experiment (not product): the C3 epoch's three bf16-operand GEMMs (hcs_gemm_bf16) timed alone
(CUDA events, 50 launches each) and their outputs' checksums (to compare kernel variants bitwise)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_08902_b200.fused import dense_matmul_bf16

torch.cuda.set_device(0)
g = torch.Generator("cuda").manual_seed(0)
n = 232965
x = torch.rand(n, 128, device="cuda", generator=g) * 2 - 1
w1 = torch.rand(128, 64, device="cuda", generator=g) * 2 - 1
h = torch.relu(torch.rand(n, 64, device="cuda", generator=g) - 0.5)
w2 = torch.rand(64, 41, device="cuda", generator=g) * 2 - 1
s2 = (torch.rand(n, 44, device="cuda", generator=g) * 2 - 1)[:, :41]
cases = {"xw1": (x, w1, None), "hw2": (h, w2, None), "g1": (s2, w2.t().contiguous(), h)}
res = {}
for name, (a, b, m) in cases.items():
    for _ in range(3):
        op = dense_matmul_bf16(a, b, mask=m)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(50):
        op = dense_matmul_bf16(a, b, mask=m)
    e.record(); torch.cuda.synchronize()
    res[name] = {"us": round(s.elapsed_time(e) / 50 * 1e3, 1),
                 "checksum": float(op.t.float().double().sum().item())}
print(json.dumps(res))
