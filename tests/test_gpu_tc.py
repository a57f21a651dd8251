"""tcgen05 conventions (csrc/tc.cuh) the tensor-core voxelizer forward builds
on: TMEM layouts of A and D, the K-major B descriptor, the TF32 instruction
descriptor and commit -> mbarrier, through splatct_tc_selftest."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2411_04844_b200 import device as D  # noqa: E402


def _run(a, b, mode):
    dev = D.require_cuda()
    ta = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(b, np.float32)).to(dev)
    td = torch.full((128, 16), float("nan"), dtype=torch.float32, device=dev)
    D.call("splatct_tc_selftest", D.ptr(ta), D.ptr(tb), D.ptr(td), int(mode), D.stream_handle())
    torch.cuda.synchronize()
    return td.cpu().numpy()


def test_tf32_mma_layouts_exact():
    """Small dyadic operands are exact in TF32: D must equal A B^T bitwise,
    which pins every row / column / k position of A, B and D."""
    rng = np.random.default_rng(0)
    a = rng.integers(-8, 9, (128, 8)) / 4.0
    b = rng.integers(-8, 9, (16, 8)) / 8.0
    d = _run(a, b, 0)
    np.testing.assert_array_equal(d, (a @ b.T).astype(np.float32))


def test_3xtf32_split_is_fp32_accurate():
    rng = np.random.default_rng(1)
    a = rng.uniform(0, 1, (128, 8)).astype(np.float32)
    b = rng.uniform(0, 1, (16, 8)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64).T
    d1 = _run(a, b, 1)
    assert np.abs(d1 - want).max() / np.abs(want).max() < 2e-6
    d0 = _run(a, b, 0)   # one TF32 pass is ~1e-3 relative: the split is what buys fp32
    assert np.abs(d0 - want).max() / np.abs(want).max() > 1e-5
