"""The slab collectives on the NCCL backend (device buffers, no host staging).

Every multi-rank test runs gloo on one GPU (NCCL refuses two ranks on one
device), so this is the only place the NCCL code paths of
distributed.SlabComm execute: a one-rank NCCL group, where each collective
is the identity and a halo exchange has no neighbours.  It checks that every
call goes through NCCL with device tensors and leaves the data as the
multi-rank semantics say for one rank.
"""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import torch, torch.distributed as dist
    from paper_2411_04844_b200.distributed import SlabComm, row_bands
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    comm = SlabComm()
    assert comm.world == 1 and not comm.host_p2p and dist.get_backend() == "nccl"
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(0)
    t = torch.randn(1000, generator=g, dtype=torch.float64).to(dev)
    ref = t.clone()
    assert torch.equal(comm.allreduce_sum_(t), ref)
    assert torch.equal(comm.allreduce_max_(t), ref)
    grads = torch.randn((5, 777), generator=g, dtype=torch.float64).to(dev)
    want = grads.to(torch.float32).to(torch.float64)
    assert torch.equal(comm.allreduce_grads_(grads), want)
    vol = torch.randn((12, 10, 8), generator=g).to(dev)
    lo, hi = comm.halo(vol)
    assert lo is None and hi is None
    comm.halo_start(vol)
    assert comm.halo_wait() == (None, None)
    pred = torch.randn((3, 5, 13), generator=g).to(dev)
    bands = row_bands(13, 1)
    band = torch.empty((3, 5, 13), device=dev)
    comm.reduce_scatter_rows(pred, bands, band)
    assert torch.equal(band, pred)
    out = torch.full_like(pred, float("nan"))
    comm.all_gather_rows(band, bands, out)
    assert torch.equal(out, pred)
    torch.cuda.synchronize()
    dist.destroy_process_group()
    print("nccl ok")
""")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_slab_comm_on_nccl_one_rank():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "nccl ok" in r.stdout
