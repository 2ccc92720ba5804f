"""C1 (Cora-shaped, 170 windows: 1 TILE + 169 SCALAR) per-kernel latency: each part of one hybrid
SpMM replayed as its own CUDA graph (200 replays, CUDA events), so launch-bound costs are seen
kernel by kernel.  Variants: scalar K3 warp-per-window vs block-per-window; all-scalar; all-tile."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_08902_b200 as hc  # noqa: E402
from paper_2412_08902_b200 import _lib, graphgen  # noqa: E402
from paper_2412_08902_b200.executors import Assignment, Path, get_plan, stage_operand, _alloc_z, set_scalar_variant  # noqa: E402,E501


def graph_us(fn, reps=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(10):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    torch.cuda.set_device(0)
    adj = graphgen.gcn_normalize_device(graphgen.cora_shaped(seed=0))
    ws = hc.partition(adj)
    dim = int(os.environ.get("DIM", "128"))
    prec = os.environ.get("PREC", "bf16")
    x = graphgen.dense_features(adj.num_rows, dim, seed=1)
    for name, asg in (("classified", hc.classify_windows(hc.default_model(), ws)),
                      ("all-scalar", Assignment.uniform(len(ws), Path.SCALAR)),
                      ("all-tile", Assignment.uniform(len(ws), Path.TILE))):
        plan = get_plan(ws, asg, prec)
        xop, _ = stage_operand(x, prec, x.device, tf32_round=prec == "tf32")
        z, ldz = _alloc_z(ws.num_rows, dim, x.device)
        scr = plan.new_scratch() if plan.n_tile else None
        nt, ns = plan.n_tile, int(plan.scalar_list.numel())
        full = (0, len(ws), 0, nt, 0, ns)
        res = {"both": graph_us(lambda: plan.run(xop, z, ldz, scratch=scr))}
        if nt:
            res["tile only"] = graph_us(lambda: plan.run(xop, z, ldz, scratch=scr, part=(0, len(ws), 0, nt, 0, 0)))
        if ns:
            res["scalar only"] = graph_us(lambda: plan.run(xop, z, ldz, scratch=scr, part=(0, len(ws), 0, 0, 0, ns)))
            for var in ("warp", "rows", "block"):
                set_scalar_variant(var)
                res[f"scalar only ({var})"] = graph_us(
                    lambda: plan.run(xop, z, ldz, scratch=scr, part=(0, len(ws), 0, 0, 0, ns)))
                res[f"both ({var})"] = graph_us(lambda: plan.run(xop, z, ldz, scratch=scr))
            set_scalar_variant("auto")
        res["empty graph node (torch add)"] = graph_us(lambda: z.add_(0))
        print(f"{prec} dim {dim} {name}: tile windows {nt}, scalar windows {ns}, chunks {plan.nchunks}: " +
              ", ".join(f"{k} {v:.2f} us" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
