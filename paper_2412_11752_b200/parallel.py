"""Multi-GPU host logic: view sharding (configs 3/4) and the gradient exchange (config 4).

One process per GPU (torch.distributed; NCCL on the B200 box, gloo in the CPU
tests).  Views are independent units of the forward pass:
primitives are replicated on every rank and each rank renders its own shard of
the views, so the forward has no data-path collective.  The training step has
one real exchange: the raw-parameter gradient buffer (n x scalar_count f32,
ABI layout) is summed across ranks and divided by the total number of views,
then every rank applies the same Adam update (replicas stay bit-identical
because NCCL's all-reduce returns the same sum on every rank).
"""
from __future__ import annotations

import numpy as np


def shard_views(n_views: int, world: int, rank: int, costs=None) -> list[int]:
    """Views rendered by `rank`.  With per-view cost estimates (e.g. tile-pair
    counts from a previous pass), greedy longest-processing-time assignment;
    otherwise contiguous equal blocks.  Every view is owned by exactly one rank."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    if costs is None:
        lo = n_views * rank // world
        hi = n_views * (rank + 1) // world
        return list(range(lo, hi))
    costs = np.asarray(costs, dtype=np.float64)
    if costs.shape != (n_views,):
        raise ValueError("one cost per view")
    load = np.zeros(world)
    owner = np.empty(n_views, dtype=np.int64)
    for v in np.argsort(-costs, kind="stable"):
        r = int(np.argmin(load))
        owner[v] = r
        load[r] += costs[v]
    return [int(v) for v in np.nonzero(owner == rank)[0]]


def allreduce_mean_(grad, total_views: int, group=None):
    """In-place sum of the per-rank accumulated gradients, divided by the
    total number of views (the multi-view gradient of SURVEY.md §8(d) is the
    mean over views of per-view backward_render)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    grad.mul_(1.0 / float(total_views))
    return grad


class NcclComm:
    """Native NCCL communicator of a Rasterizer's device (drk_comm_init; the
    unique id is created by rank 0 and broadcast over the torch.distributed
    process group, or passed in).  Used by the training step's gradient
    exchange (Rasterizer.allreduce_adam: reduce-scatter, sharded Adam,
    all-gather) and drk_allreduce_sum."""

    def __init__(self, rast, rank: int = 0, world: int = 1, uid: bytes | None = None, group=None):
        import ctypes as C

        from . import _lib
        if uid is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                _lib.check(_lib.lib().drk_comm_unique_id(buf))
            if world > 1:
                import torch.distributed as dist
                obj = [bytes(buf) if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                uid = obj[0]
            else:
                uid = bytes(buf)
        raw = (C.c_uint8 * 128).from_buffer_copy(uid)
        self.handle = C.c_void_p()
        self._rast = rast
        rast._check(_lib.lib().drk_comm_init(rast._h, raw, int(world), int(rank), C.byref(self.handle)))
        self.rank, self.world = rank, world

    def allreduce_sum_(self, buf):
        """In-place sum over the ranks (f32 device tensor)."""
        import ctypes as C

        from . import _lib
        self._rast._sync_stream()
        self._rast._check(_lib.lib().drk_allreduce_sum(self._rast._h, self.handle, C.c_void_p(buf.data_ptr()),
                                                       buf.numel()))
        return buf

    def close(self):
        from . import _lib
        if self.handle:
            _lib.lib().drk_comm_destroy(self.handle)
            self.handle = None


def params_checksum(params) -> float:
    """Order-independent fp64 checksum used to verify that replicas stay in sync."""
    import torch
    p = params.detach().to(torch.float64)
    return float((p * torch.arange(1, p.numel() + 1, dtype=torch.float64, device=p.device).reshape(p.shape)
                  .remainder(7.0).add(1.0)).sum())


class MultiViewRenderer:
    """Renders a batch of views on one GPU with ``inflight`` rasterizer contexts,
    each on its own CUDA stream driven by its own host thread (the C-ABI calls
    release the GIL).  A view's host-side sizing points (the scans that return
    row / pair counts) and its FP64-heavy binning then overlap another view's
    FP32 rasterization, instead of leaving the GPU idle between views.
    Views are handed out dynamically (next view to the first free context); each
    context activates the primitives once per batch (render, then render_again).
    Every view's framebuffers are identical to a single-context render.  Measured
    on config 3 (16 views): one context 1.42 s, two 1.43 s — with the host stalls
    removed the GPU is saturated by one context; more in flight guard against
    host-side gaps."""

    def __init__(self, device=None, inflight: int = 2):
        import torch

        from .api import Rasterizer
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.rasts = [Rasterizer(self.device.index) for _ in range(inflight)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(inflight)]

    def render(self, raw, cams, opt, k: int = 8):
        """Framebuffers of every camera (list, camera order); ordered after the
        caller's current stream and before it again on return."""
        import threading

        import torch
        start = torch.cuda.Event()
        start.record(torch.cuda.current_stream(self.device))
        results = [None] * len(cams)
        errors = []
        nxt = [0]
        lock = threading.Lock()

        def work(w):
            try:
                torch.cuda.set_device(self.device)
                s = self.streams[w]
                s.wait_event(start)
                first = True
                with torch.cuda.stream(s):
                    while True:
                        with lock:
                            i = nxt[0]
                            nxt[0] += 1
                        if i >= len(cams):
                            return
                        # each context activates the primitives once per batch
                        if first:
                            results[i] = self.rasts[w].render(raw, cams[i], opt, k=k)
                            first = False
                        else:
                            results[i] = self.rasts[w].render_again(cams[i], opt)
            except Exception as e:  # surfaced on the caller's thread
                errors.append(e)

        threads = [threading.Thread(target=work, args=(w,)) for w in range(len(self.rasts))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        main = torch.cuda.current_stream(self.device)
        for s in self.streams:
            main.wait_stream(s)
        return results

    def close(self):
        for r in self.rasts:
            r.close()
