"""CPU: the torch.ops.hcspmm custom operators (ops.py)."""

import pytest


def test_custom_ops_registered_with_fake_kernels():
    """torch.ops.hcspmm.{spmm, gcn_layer} exist at import, infer output shapes without a GPU
    (fake tensors), and refuse CPU tensors (no CPU kernel)."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode

    import paper_2412_08902_b200  # noqa: F401

    with FakeTensorMode():
        rp = torch.empty(11, dtype=torch.int64)
        ci = torch.empty(30, dtype=torch.int32)
        v = torch.empty(30)
        x = torch.empty(12, 7, dtype=torch.bfloat16)
        w = torch.empty(7, 5)
        z = torch.ops.hcspmm.spmm(rp, ci, v, 12, x, "bf16")
        out, zz = torch.ops.hcspmm.gcn_layer(rp, ci, v, 12, x, w, "bf16")
    assert tuple(z.shape) == (10, 7) and z.dtype == torch.float32
    assert tuple(out.shape) == (10, 5) and tuple(zz.shape) == (10, 7)
    with pytest.raises(ValueError, match="no CPU kernel"):
        torch.ops.hcspmm.spmm(torch.zeros(3, dtype=torch.int64), torch.zeros(0, dtype=torch.int32), torch.zeros(0), 2,
                              torch.zeros(2, 4), "bf16")
