"""Column-parallel FlashNorm linear across GPUs.

W* is column-sharded (rank p owns output rows [p*N/P, (p+1)*N/P) of W*t and the
matching slice of c*); activations are replicated.  Each rank computes the RMS of
its full local token rows (RMS is per token over K), so the path needs
NO collective to produce its shard of z.  The NCCL all-gather (through
torch.distributed, NVLink/NVSwitch on the box) runs only when the caller asks for
the gathered output; the [P][M][N/P] -> [M][N] permute is the library's
flashnorm_gather_columns kernel.

Host logic only (shard arithmetic, process-group plumbing); every arithmetic step
runs in libflashnorm's CUDA kernels.  The helpers take an explicit `compute_fn` /
`permute_fn` so the sharding and gather plumbing can be exercised with the gloo
backend on CPU in tests.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

ALIGN = 8  # bf16 rows of 16 bytes; also the decode kernel's 8-row tile


def shard_bounds(N: int, world: int, rank: int, align: int = ALIGN) -> Tuple[int, int]:
    """Contiguous, equal, `align`-multiple column shard [lo, hi) of N outputs for `rank`."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError(f"bad world/rank {world}/{rank}")
    if N % (world * align) != 0:
        raise ValueError(f"N = {N} must be a multiple of world*{align} = {world * align} for equal column shards")
    per = N // world
    return rank * per, (rank + 1) * per


def shard_columns(Wt_star, c_star, world: int, rank: int):
    """Views of this rank's rows of W*t [N, K] and of c* [N] (no copy: rows are contiguous)."""
    lo, hi = shard_bounds(Wt_star.shape[0], world, rank)
    return Wt_star[lo:hi], (None if c_star is None else c_star[lo:hi])


def gather_columns_reference(parts):
    """Layout contract of flashnorm_gather_columns: [P][M][Nl] -> [M][P*Nl] (torch ops; tests only)."""
    P, M, Nl = parts.shape
    return parts.permute(1, 0, 2).reshape(M, P * Nl)


class ColumnParallelFlashNorm:
    """One rank's shard of a FlashNorm linear layer z = (a W*) / RMSe(a) + c*.

    Parameters are folded ONCE (flashnorm_fold_weights on the local rows of the
    original W; the fold is row-local so sharding before or after folding is the
    same).
    """

    def __init__(self, Wt_star_local, c_star_local=None, group=None, world: Optional[int] = None,
                 rank: Optional[int] = None, compute_fn: Optional[Callable] = None,
                 permute_fn: Optional[Callable] = None):
        import torch.distributed as dist
        self.W = Wt_star_local
        self.c = c_star_local
        self.group = group
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if dist.is_initialized() else 0)
        if compute_fn is None:
            from . import linear as compute_fn
        if permute_fn is None:
            from . import gather_columns as permute_fn
        self._compute = compute_fn
        self._permute = permute_fn

    @classmethod
    def from_full(cls, Wt_star, c_star=None, **kw):
        """Build from the full folded weights: keep only this rank's contiguous rows."""
        import torch.distributed as dist
        world = kw.pop("world", dist.get_world_size(kw.get("group")) if dist.is_initialized() else 1)
        rank = kw.pop("rank", dist.get_rank(kw.get("group")) if dist.is_initialized() else 0)
        W, c = shard_columns(Wt_star, c_star, world, rank)
        return cls(W.contiguous(), None if c is None else c.contiguous(), world=world, rank=rank, **kw)

    def forward(self, a, eps: float = 1e-5, mode: str = "rmsnorm", alpha: float = 0.5, gather: bool = False):
        z_local = self._compute(a, self.W, self.c, eps=eps, mode=mode, alpha=alpha)
        if not gather or self.world == 1:
            return z_local
        import torch
        import torch.distributed as dist
        M, Nl = z_local.shape
        flat = torch.empty((self.world * M, Nl), dtype=z_local.dtype, device=z_local.device)
        dist.all_gather_into_tensor(flat, z_local.contiguous(), group=self.group)
        return self._permute(flat.view(self.world, M, Nl))  # [P][M][Nl] -> [M][P*Nl]

    def forward_fused_gather(self, a, eps: float = 1e-5, mode: str = "rmsnorm", alpha: float = 0.5,
                             copy: bool = False, multicast="auto"):
        """Gathered output with the all-gather FUSED into the GEMM epilogue (NEXT-3): every rank's
        epilogue stores its shard straight into every rank's gathered buffer over NVLink
        (flashnorm_linear_gather with the peers' symmetric-memory pointers), tile by tile while the
        next tiles compute; a device-side barrier then orders the peers' reads.  Replaces the
        NCCL all-gather + permute of `forward(gather=True)`.

        NVLS: when the symmetric buffer has a multicast mapping (torch symmetric memory's
        ``multicast_ptr`` is non-zero: NVSwitch with NVLink SHARP) and ``multicast`` is "auto" or True,
        the epilogue stores through it with multimem.st (flashnorm_linear_gather_multicast): each rank
        sends its shard once and the switch replicates it to every rank, instead of P - 1 peer stores.
        ``multicast=True`` without a multicast mapping raises; False forces the peer stores.

        Lifetime of the result: the gathered z lives in one of TWO persistent symmetric buffers
        that alternate between calls (peers write into them over NVLink).  The returned tensor is
        valid until the call after next; work that reads it on the current stream before that
        call is ordered by the entry barrier.  Pass ``copy=True`` for an owned tensor.  Needs CUDA,
        NCCL and torch symmetric memory; tests/test_gpu_dist.py runs it at world 1 and, on a box
        with >= 2 GPUs, at world N (tests/test_gpu_multi.py)."""
        import torch
        import torch.distributed._symmetric_memory as symm_mem
        from . import linear_gather
        M, Nl = a.shape[0], self.W.shape[0]
        N = Nl * self.world
        key = (M, N, a.dtype, a.device)
        if getattr(self, "_symm_key", None) != key:
            grp = self.group if self.group is not None else torch.distributed.group.WORLD
            bufs, hdls, peers = [], [], []
            for _ in range(2):
                buf = symm_mem.empty((M, N), dtype=a.dtype, device=a.device)
                hdl = symm_mem.rendezvous(buf, grp)
                bufs.append(buf)
                hdls.append(hdl)
                peers.append([hdl.get_buffer(p, (M, N), a.dtype) for p in range(self.world)])
            self._symm_key, self._symm_bufs, self._symm_hdls, self._symm_peers = key, bufs, hdls, peers
            self._symm_slot = 0
        i = self._symm_slot
        self._symm_slot ^= 1
        hdl = self._symm_hdls[i]
        mc_ptr = int(getattr(hdl, "multicast_ptr", 0) or 0)
        if multicast is True and not mc_ptr:
            raise RuntimeError("forward_fused_gather(multicast=True): no NVLS multicast mapping on this group")
        hdl.barrier(channel=0)  # every rank finished the work it ordered before this call on slot i
        if mc_ptr and multicast in ("auto", True):
            from . import linear_gather_multicast
            linear_gather_multicast(a, self.W, mc_ptr, N, self.rank * Nl, c_star=self.c, eps=eps, mode=mode,
                                    alpha=alpha)
            self.last_gather = "multicast"
        else:
            linear_gather(a, self.W, self._symm_peers[i], self.rank * Nl, c_star=self.c, eps=eps, mode=mode,
                          alpha=alpha)
            self.last_gather = "peer stores"
        hdl.barrier(channel=0)  # every shard has landed in every rank's buffer
        out = self._symm_bufs[i]
        return out.clone() if copy else out

    __call__ = forward
