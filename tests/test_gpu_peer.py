"""Tensor-parallel partial sums over peer memory (peer.py, rtnq_dev_linear_peer /
rtnq_dev_add_rmsnorm_peer / rtnq_dev_peer_reduce).

The fused path must give the same bits as "row-split linear -> bf16 partial -> allreduce
(f32 sum in rank order, one bf16 rounding) -> consumer", on every rank, over many rounds (the
epoch / parity protocol).  All ranks run on cuda:0: one process driving the group
(PeerGroup.single_process), or two processes mapping each other's buffer through CUDA IPC."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rq():
    import paper_2505_15909_b200 as rq
    return rq


def _weights(world, n, k, bits, seed):
    rq = _rq()
    g = torch.Generator(device="cuda").manual_seed(seed)
    out = []
    for _ in range(world):
        w = ((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
        out.append(rq.quantize_pack(w, bits, 128 if bits == 4 else k))
    return out


def _allreduce_ref(parts):
    """bf16 partials -> f32 sum in rank order -> one bf16 rounding."""
    acc = torch.zeros_like(parts[0], dtype=torch.float32)
    for p in parts:
        acc += p.float()
    return acc.to(torch.bfloat16)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("m", [1, 5, 16])
def test_peer_linear_reduce_rounds(world, bits, m):
    rq = _rq()
    from paper_2505_15909_b200.peer import PeerGroup, slot_cap
    n, k = 1024, 2048
    qs = _weights(world, n, k, bits, seed=world * 10 + bits)
    groups = PeerGroup.single_process(world, slot_cap(64 * n))
    g = torch.Generator(device="cuda").manual_seed(m)
    for rnd in range(5):  # both slot parities, epochs 1..5
        a = [(torch.randn(m, k, device="cuda", generator=g)).to(torch.bfloat16) for _ in range(world)]
        parts = [rq.linear(a[r], qs[r], out=torch.empty(m, n, dtype=torch.bfloat16, device="cuda"))
                 for r in range(world)]
        for r in range(world):
            groups[r].linear(qs[r], a=a[r])
        acc = rnd % 2 == 1
        base = (torch.randn(m, n, device="cuda", generator=g)).to(torch.bfloat16)
        outs = [base.clone() if acc else torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
                for _ in range(world)]
        for r in range(world):
            groups[r].reduce(outs[r], accumulate=acc)
        want = _allreduce_ref(parts)
        if acc:
            want = (base.float() + want.float()).to(torch.bfloat16)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(outs[r], want), (rnd, r)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_add_rmsnorm_planes(world):
    """The fused consumer: x += sum, rmsnorm, activation planes -- identical to
    rtnq_dev_add_rmsnorm_planes with delta = the allreduced partial."""
    rq = _rq()
    from paper_2505_15909_b200.peer import PeerGroup, slot_cap
    m, h, k = 7, 4096, 1024
    qs = _weights(world, h, k, 4, seed=3)
    groups = PeerGroup.single_process(world, slot_cap(m * h))
    g = torch.Generator(device="cuda").manual_seed(1)
    wn = (1 + 0.1 * torch.rand(h, device="cuda", generator=g)).to(torch.bfloat16)
    for rnd in range(3):
        a = [torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16) for _ in range(world)]
        x0 = torch.randn(m, h, device="cuda", generator=g).to(torch.bfloat16)
        parts = [rq.linear(a[r], qs[r], out=torch.empty(m, h, dtype=torch.bfloat16, device="cuda"))
                 for r in range(world)]
        xr, yr, pr = x0.clone(), torch.empty(m, h, dtype=torch.bfloat16, device="cuda"), rq.Planes(m, h)
        rq.add_rmsnorm(xr, wn, yr, delta=_allreduce_ref(parts), planes=pr)
        for r in range(world):
            groups[r].linear(qs[r], a=a[r])
        for r in range(world):
            x, y, p = x0.clone(), torch.empty_like(yr), rq.Planes(m, h)
            groups[r].add_rmsnorm(x, wn, y, planes=p)
            torch.cuda.synchronize()
            assert torch.equal(x, xr) and torch.equal(y, yr), (rnd, r)
            assert torch.equal(p.planes, pr.planes) and torch.equal(p.texp, pr.texp)


def test_peer_rejects_bad_arguments():
    rq = _rq()
    from paper_2505_15909_b200.peer import PeerGroup, slot_cap
    (q,) = _weights(1, 256, 512, 4, seed=0)
    (grp,) = PeerGroup.single_process(1, slot_cap(256))
    a = torch.randn(2, 512, device="cuda").to(torch.bfloat16)
    with pytest.raises(rq.Error):  # 2 x 256 outputs > the slot's 256 elements
        grp.linear(q, a=a)
    with pytest.raises(rq.Error):  # 65 tokens: more than one launch (one round) can carry
        big = PeerGroup.single_process(1, slot_cap(65 * 256))[0]
        big.linear(q, a=torch.randn(65, 512, device="cuda").to(torch.bfloat16))


SHAPE_ARGS = dict(name="tp-peer", hidden=1024, heads=8, kv_heads=4, head_dim=128, ffn=2048, layers=3)
TABLE = [[4, 4, 4, 8], [8, 8, 4, 4], [4, 8, 8, 4]]


def _stacks(world, batch, w8pc, peer):
    from paper_2505_15909_b200 import tp
    from paper_2505_15909_b200.peer import PeerGroup, slot_cap
    shape = tp.LlamaShape(**SHAPE_ARGS)
    table = np.array(TABLE, np.uint8)
    stacks = [tp.TPDecodeStack(shape, table, world, r, batch, max_len=40, pos=33, seed=9,
                               w8_per_channel=w8pc, collectives=False) for r in range(world)]
    if peer:
        for st, grp in zip(stacks, PeerGroup.single_process(world, slot_cap(batch * shape.hidden))):
            st.peer = grp
    return shape, stacks


def _x0(batch, hidden):
    return (torch.randn(batch, hidden, generator=torch.Generator().manual_seed(4)) * 0.5
            ).to(torch.bfloat16).cuda()


def _simulated_step(stacks, x0):
    """The same ranks with the allreduce done by hand (f32 rank-order sum, bf16)."""
    for st in stacks:
        st.x.copy_(x0)
    delta = None
    for li in range(len(stacks[0].layers)):
        o = _allreduce_ref([st.layers[li].attn_half(st.x, delta, st.ws).clone() for st in stacks])
        delta = _allreduce_ref([st.layers[li].mlp_half(st.x, o, st.ws).clone() for st in stacks])
    for st in stacks:
        st.x.add_(delta)
    return [st.x.clone() for st in stacks]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("w8pc", [False, True])
@pytest.mark.parametrize("batch", [1, 5])
def test_tp_peer_stack_single_process(world, w8pc, batch):
    from paper_2505_15909_b200 import tp
    shape, stacks = _stacks(world, batch, w8pc, peer=True)
    x0 = _x0(batch, shape.hidden)
    want = _simulated_step(stacks, x0)
    for _ in range(3):  # repeated steps: the rounds keep counting
        got = [x.clone() for x in tp.step_peer(stacks, [x0] * world)]
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(got[r], want[r]), r
    for st in stacks:
        st.check()
    # and against the unsharded stack
    _, (ref,) = _stacks(1, batch, w8pc, peer=False)
    r1 = ref.step(x0).double()
    err = ((got[0].double() - r1).norm() / r1.norm()).item()
    assert err < 2e-2, err


def test_tp_peer_stack_cuda_graph():
    """The fused rounds replay from a CUDA graph (device-side epochs, no host state)."""
    from paper_2505_15909_b200 import tp
    world, batch = 2, 3
    shape, stacks = _stacks(world, batch, False, peer=True)
    x0 = _x0(batch, shape.hidden)
    want = [x.clone() for x in tp.step_peer(stacks, [x0] * world)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tp.step_peer(stacks, [x0] * world, [s] * world)  # warm the default workspaces on s
        s.synchronize()
        with torch.cuda.graph(graph, stream=s):
            outs = tp.step_peer(stacks, [x0] * world, [s] * world)
    for _ in range(4):
        with torch.cuda.stream(s):
            graph.replay()
        s.synchronize()
        for r in range(world):
            assert torch.equal(outs[r], want[r])


# ---- one process per rank, buffers exchanged as CUDA IPC handles ------------------------------
# Both processes share cuda:0 here, so a consumer spinning in one process's context would wait on
# a producer in the other context behind the GPU's time-slicing; the test therefore separates each
# round's produce and consume phases with a host barrier.  It checks what differs from the
# single-process group: the handle exchange, the P2P stores and flags through IPC mappings.

def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rq = _rq()
    from paper_2505_15909_b200.peer import PeerGroup, slot_cap
    m, n, k = 5, 1024, 2048
    qs = _weights(world, n, k, 4, seed=77)  # every rank draws all weights, keeps its own
    grp = PeerGroup.from_process_group(slot_cap(m * n))
    g = torch.Generator(device="cuda").manual_seed(5)
    outs, wants = [], []
    for rnd in range(4):
        a = [torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16) for _ in range(world)]
        wants.append(_allreduce_ref([rq.linear(a[r], qs[r]) for r in range(world)]).cpu())
        grp.linear(qs[rank], a=a[rank])
        torch.cuda.synchronize()
        dist.barrier()  # every rank's partial delivered
        out = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        grp.reduce(out)
        torch.cuda.synchronize()
        dist.barrier()  # every rank consumed the round
        outs.append(out.cpu())
    grp.close()  # collective
    dist.destroy_process_group()
    q.put((rank, [o.float().numpy() for o in outs], [w.float().numpy() for w in wants]))


@pytest.mark.timeout(400)
def test_peer_ipc_two_processes():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    port = _port()
    qu = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in procs:
            r, outs, wants = qu.get(timeout=300)
            got[r] = outs
            for o, w in zip(outs, wants):
                assert np.array_equal(o, w), r
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.exitcode is None:
                p.kill()
    assert all(np.array_equal(a, b) for a, b in zip(got[0], got[1]))


def _stack_worker(rank, world, port, batch, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_15909_b200 import tp
    shape = tp.LlamaShape(**SHAPE_ARGS)
    st = tp.TPDecodeStack(shape, np.array(TABLE, np.uint8), world, rank, batch, max_len=40, pos=33,
                          seed=9, collectives="peer")
    x0 = _x0(batch, shape.hidden)
    xs = [st.step(x0).float().cpu().numpy() for _ in range(2)]
    st.check()
    st.peer.close()
    dist.destroy_process_group()
    q.put((rank, xs))


@pytest.mark.timeout(400)
def test_tp_peer_stack_two_processes():
    """TPDecodeStack(collectives="peer") under one process per rank: the consumers spin on the
    device for the other process's producers (here both share cuda:0 and the GPU time-slices
    the two contexts); the result equals the single-process group's bits."""
    import torch.multiprocessing as mp
    world, batch = 2, 5
    ctx = mp.get_context("spawn")
    port = _port()
    qu = ctx.Queue()
    procs = [ctx.Process(target=_stack_worker, args=(r, world, port, batch, qu)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in procs:
            r, xs = qu.get(timeout=300)
            got[r] = xs
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.exitcode is None:
                p.kill()
    from paper_2505_15909_b200 import tp
    shape, stacks = _stacks(world, batch, False, peer=True)
    want = [x.float().cpu().numpy() for x in tp.step_peer(stacks, [_x0(batch, shape.hidden)] * world)]
    for r in range(world):
        for x in got[r]:
            assert np.array_equal(x, want[r]), r
