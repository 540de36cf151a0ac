"""Tensor-parallel partial sums over peer memory: the allreduce after a
row-split linear, fused into the linear's epilogue and the next add+RMSNorm.

The reference runs on one device (its GEMM, gemm.cpp:100-109, has no collective); the
tensor-parallel split of a Llama layer adds two allreduces per layer after the
row-split ``attn_out_proj`` / ``ffn_down``.  Here they are not separate collectives: the
int8 linear stores its bf16 output rows straight into this rank's slot of EVERY rank's
symmetric buffer over NVLink (P2P stores from the GEMM epilogue) and raises a release flag
when its last CTA finishes; the consumer (add+RMSNorm of the next half-layer, or
:meth:`PeerGroup.reduce`) waits for all flags on the device and sums the slots in rank
order.  No host synchronisation, no NCCL launch, capturable in a CUDA graph.  Protocol and
buffer layout: ``csrc/kernels/int8_mma.cuh`` ("partial sums over peer memory"); C-ABI:
``include/rtnq_capi.h`` (rtnq_dev_linear_peer / rtnq_dev_add_rmsnorm_peer /
rtnq_dev_peer_reduce).

Two ways to build the group:
  * :meth:`PeerGroup.single_process` -- one process drives ``world`` ranks (one device
    each, or all on one device for testing); rank q's buffer lives on its device and the
    others reach it through peer access.
  * :meth:`PeerGroup.from_process_group` -- one process per GPU (torchrun); buffers are
    exchanged as CUDA IPC handles over ``torch.distributed`` (any backend).
"""
import ctypes as C

import paper_2505_15909_b200 as rq


def slot_cap(elems: int) -> int:
    """Elements per slot for outputs of up to ``elems`` elements (a multiple of 8)."""
    return max(8, (int(elems) + 7) // 8 * 8)


class _Buffer:
    """A symmetric buffer of its own cudaMalloc allocation (rtnq_peer_alloc): an IPC handle
    maps a whole allocation, so it cannot be carved out of torch's caching allocator."""

    def __init__(self, cap, device):
        import torch
        self.device = torch.device(device)
        with torch.cuda.device(self.device):
            p = C.c_void_p()
            rq._check(rq.lib().rtnq_peer_alloc(cap, C.byref(p)))
        self.ptr = p.value

    def free(self):
        if self.ptr:
            import torch
            with torch.cuda.device(self.device):
                rq.lib().rtnq_peer_free(C.c_void_p(self.ptr))
            self.ptr = None


class PeerGroup:
    """One rank's handle on the group: its own buffer plus every rank's buffer address as
    seen from this rank's device."""

    def __init__(self, world: int, rank: int, cap: int, own, ptrs, opened=(), pg=None):
        assert 1 <= world <= 8 and 0 <= rank < world and len(ptrs) == world
        self.world, self.rank, self.cap = world, rank, cap
        self.own = own                       # this rank's buffer (_Buffer)
        self.device = own.device
        self._ptrs = (C.c_void_p * world)(*ptrs)
        self._opened = list(opened)          # IPC mappings to close
        self._pg = pg                        # process group of an IPC-mapped group

    # ---- construction -------------------------------------------------------------
    @classmethod
    def single_process(cls, world: int, cap: int, devices=None):
        """``world`` ranks driven by this process; ``devices[q]`` is rank q's device
        (default: all on the current device)."""
        import torch
        if devices is None:
            devices = [torch.cuda.current_device()] * world
        devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        for d in devices:
            for e in devices:
                rq._check(rq.lib().rtnq_peer_enable(d.index or 0, e.index or 0))
        bufs = [_Buffer(cap, d) for d in devices]
        ptrs = [b.ptr for b in bufs]
        return [cls(world, q, cap, bufs[q], ptrs) for q in range(world)]

    @classmethod
    def from_process_group(cls, cap: int, group=None, device=None):
        """One rank per process: allocate this rank's buffer, exchange CUDA IPC handles
        over ``group`` (all_gather_object) and map every peer's buffer."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        own = _Buffer(cap, device)
        h = (C.c_char * 64)()
        rq._check(rq.lib().rtnq_ipc_get_handle(C.c_void_p(own.ptr), h))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h), group=group)
        ptrs, opened = [], []
        for q, hq in enumerate(handles):
            if q == rank:
                ptrs.append(own.ptr)
                continue
            p = C.c_void_p()
            rq._check(rq.lib().rtnq_ipc_open((C.c_char * 64).from_buffer_copy(hq), C.byref(p)))
            ptrs.append(p.value)
            opened.append(p.value)
        torch.cuda.synchronize(device)
        dist.barrier(group)  # every rank mapped every buffer before any round starts
        return cls(world, rank, cap, own, ptrs, opened, pg=group if group is not None else True)

    def close(self):
        """Unmap the peers' buffers and free this rank's, once the last round completed
        (collective for an IPC-mapped group: every rank unmaps before any rank frees)."""
        import torch
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            rq.lib().rtnq_ipc_close(C.c_void_p(p))
        self._opened = []
        if self._pg is not None:
            import torch.distributed as dist
            dist.barrier(None if self._pg is True else self._pg)
        self.own.free()

    # ---- one round: produce (every rank), then consume (every rank) -------------------
    def linear(self, qw, a=None, planes=None, *, workspace=None, stream=None, pdl=False,
               err=None):
        """Row-split linear whose [m, qw.rows] bf16 output goes to every rank's slot
        (rtnq_dev_linear_peer); ``a`` is the bf16 activation or ``planes`` its int8 planes."""
        assert (a is None) != (planes is None)
        m, k = (a.shape if a is not None else (planes.m, planes.k))
        assert k == qw.cols and qw.layout in (rq.NATIVE_I4, rq.NATIVE_I8)
        wsb = rq.lib().rtnq_dev_linear_workspace_bytes(m, qw.rows, qw.cols, qw.bits, qw.group,
                                                       rq.PATH_FUSED, rq.layout(qw.layout))
        dev = self.device
        if workspace is None:
            workspace = rq._default_workspace(dev, stream, wsb)
        buf = workspace.ensure(wsb)
        rq._check(rq.lib().rtnq_dev_linear_peer(
            rq._ptr(a), None if planes is None else rq._ptr(planes.planes),
            None if planes is None else rq._ptr(planes.texp), m, k, rq._ptr(qw.codes),
            rq.layout(qw.layout), qw.bits, qw.rows, qw.group, int(qw.ragged), rq._ptr(qw.scales),
            rq.F16, rq.SCALES_NATIVE, self._ptrs, self.world, self.rank, self.cap, rq._ptr(err),
            rq._ptr(buf), buf.numel(), rq._stream(stream), rq.FLAG_PDL if pdl else 0))

    def add_rmsnorm(self, x, weight, out, eps=1e-5, stream=None, planes=None):
        """x += sum of the round's partials; out = rmsnorm(x) * weight (+ planes of out)."""
        m, h = x.shape
        rq._check(rq.lib().rtnq_dev_add_rmsnorm_peer(
            rq._ptr(x), C.c_void_p(self.own.ptr), self.world, self.cap, rq._ptr(weight),
            rq._ptr(out), m, h, eps, None if planes is None else rq._ptr(planes.planes),
            None if planes is None else rq._ptr(planes.texp), rq._stream(stream)))
        return out

    def reduce(self, out, accumulate=False, stream=None):
        """out (+)= sum of the round's partials (bf16, ``out.numel()`` elements)."""
        rq._check(rq.lib().rtnq_dev_peer_reduce(
            C.c_void_p(self.own.ptr), self.world, self.cap, rq._ptr(out), out.numel(),
            int(accumulate), rq._stream(stream)))
        return out
