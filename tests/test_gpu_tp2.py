"""The product tensor-parallel stack (tp.TPDecodeStack) at world_size 2 on ONE GPU: two
processes on cuda:0, the row-parallel allreduces carried by gloo (NCCL refuses two ranks on
one device).  Every rank quantizes the full weights and keeps its shard (quantize before
sharding, incl. W8 per-channel row splits), runs the real kernels and the real allreduce
points of TPDecodeStack.step; the residual stream must match the unsharded (TP=1) stack."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SHAPE_ARGS = dict(name="tp2", hidden=1024, heads=8, kv_heads=4, head_dim=128, ffn=2048, layers=3)
TABLE = [[4, 4, 4, 8], [8, 8, 4, 4], [4, 8, 8, 4]]  # selective precision per (layer, module)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, rank, w8pc, batch):
    from paper_2505_15909_b200 import tp
    shape = tp.LlamaShape(**SHAPE_ARGS)
    table = np.array(TABLE, np.uint8)
    st = tp.TPDecodeStack(shape, table, world, rank, batch, max_len=40, pos=33, seed=9,
                          w8_per_channel=w8pc)
    x0 = (torch.randn(batch, shape.hidden, generator=torch.Generator().manual_seed(4)) * 0.5
          ).to(torch.bfloat16).cuda()
    x = st.step(x0).float().cpu()
    st.check()  # no non-finite activation flagged
    return x


def _worker(rank, world, port, w8pc, batch, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = _run(world, rank, w8pc, batch)
    dist.destroy_process_group()
    q.put((rank, x.numpy()))


@pytest.mark.parametrize("w8pc", [False, True])
@pytest.mark.parametrize("batch", [1, 5])
def test_tp_stack_world2_matches_unsharded(w8pc, batch):
    ctx = mp.get_context("spawn")
    port = _port()
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, w8pc, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _run(1, 0, w8pc, batch).numpy().astype(np.float64)
    for r in range(2):
        g = got[r].astype(np.float64)
        err = np.linalg.norm(g - ref) / np.linalg.norm(ref)
        assert err < 2e-2, (r, err)  # bf16 partial outputs, summed in another order
    assert np.array_equal(got[0], got[1])  # replicas of the residual stream agree exactly
