"""Multi-GPU row-group sharding of one Shfl-BW layer.

Row groups are independent and write disjoint output rows
(/root/reference/proj/src/spmm.cpp:133-134), so a layer shards by groups
with no collective in the data path.  Rank p of P owns groups
[p*G//P, (p+1)*G//P) -- the reference's worker split
(src/spmm.cpp:137-142) -- and computes them with
``shflbw_cu_spmm_groups(compact=1)`` into contiguous rows.  Only when the
consumer needs the full output does an all-gather run (NCCL over NVLink on
the GPU box; ranks' chunks are padded to equal size), followed by
``shflbw_cu_unpermute_rows`` through a precomputed gathered-row -> output-row
map (-1 for padding rows).

``ShardPlan`` is pure host logic (tested with gloo on CPU);
``ShardedSpMM`` binds it to the CUDA kernels.

Multicast variant (``ShardedSpMM.full_multicast``, ``MulticastOutputs``):
the same epilogue stores go once through an NVLS multicast address bound to
every rank's output (torch symmetric memory), so each row chunk is one
multimem.st instead of P P2P stores.

Fused all-gather (``ShardedSpMM.full_fused``): every rank holds a full-size
output buffer; the buffers are shared through CUDA IPC once
(``PeerOutputs``), and ``shflbw_cu_spmm_groups_peers`` stores each finished
row at its final position into all ranks' buffers from the epilogue (P2P
stores over NVLink, overlapped with the remaining tiles' math) -- no NCCL
call, no padding, no unpermute pass.  A barrier orders the consumers after
every rank's kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class ShardPlan:
    groups: int
    v: int
    world: int

    def range(self, rank: int) -> tuple[int, int]:
        """The reference's static split: [G*w/W, G*(w+1)/W)."""
        return self.groups * rank // self.world, self.groups * (rank + 1) // self.world

    @property
    def chunk_groups(self) -> int:
        """Groups per rank after padding to equal all-gather counts."""
        return max(self.range(r)[1] - self.range(r)[0] for r in range(self.world))

    @property
    def chunk_rows(self) -> int:
        return self.chunk_groups * self.v

    def gathered_row_map(self, row_indices: torch.Tensor) -> torch.Tensor:
        """Row r' of the all-gathered (padded, group-ordered) buffer -> output
        row, or -1 for a padding row.  row_indices: the matrix's [M] map."""
        out = torch.full((self.world * self.chunk_rows,), -1, dtype=torch.int32, device=row_indices.device)
        for r in range(self.world):
            g0, g1 = self.range(r)
            n = (g1 - g0) * self.v
            out[r * self.chunk_rows: r * self.chunk_rows + n] = row_indices[g0 * self.v: g1 * self.v].to(torch.int32)
        return out


def gather_rows(plan: ShardPlan, local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather each rank's compact rows (padded to plan.chunk_rows) into
    the [world*chunk_rows, N] group-ordered buffer."""
    import torch.distributed as dist
    if local.shape[0] != plan.chunk_rows:
        pad = torch.zeros((plan.chunk_rows - local.shape[0], local.shape[1]), dtype=local.dtype,
                          device=local.device)
        local = torch.cat([local, pad])
    out = torch.empty((plan.world * plan.chunk_rows, local.shape[1]), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    else:
        dist.all_gather(list(out.chunk(plan.world)), local.contiguous(), group=group)
    return out


class ShardedSpMM:
    """One rank's share of C = decompress(A) @ B, optionally all-gathered."""

    def __init__(self, a, rank: int, world: int, group=None):
        from . import shflbw as sb
        self.sb = sb
        self.a = a
        self.plan = ShardPlan(a.group_count(), a.v, world)
        self.rank = rank
        self.group = group
        self.g0, self.g1 = self.plan.range(rank)
        ri, _, _, _ = a.to_host()
        self.row_map = self.plan.gathered_row_map(torch.from_numpy(ri.astype("int32")).cuda())

    def local(self, b: torch.Tensor, out_dtype=torch.bfloat16, out: torch.Tensor | None = None) -> torch.Tensor:
        """This rank's rows, group order (compact)."""
        if out is None:
            out = torch.empty((self.plan.chunk_rows, b.shape[1]), dtype=out_dtype, device=b.device)
        return self.sb.spmm_groups(self.a, self.g0, self.g1, b, out, compact=True)

    def full(self, b: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
        """All ranks' rows gathered and un-permuted into the full [M, N] output."""
        gathered = gather_rows(self.plan, self.local(b, out_dtype), self.group)
        c = torch.empty((self.a.rows, b.shape[1]), dtype=out_dtype, device=b.device)
        return self.sb.unpermute_rows(self.row_map.data_ptr(), gathered, c)


class PeerOutputs:
    """A full-size [M, N] output buffer on every rank, each rank holding P2P
    device pointers to all the others (CUDA IPC handles exchanged once over
    the process group).  ``ptrs`` lists this rank's buffer first."""

    def __init__(self, shape, dtype, world: int, rank: int, group=None, device=None):
        import torch.distributed as dist
        self.buf = torch.zeros(shape, dtype=dtype, device=device or torch.device("cuda", torch.cuda.current_device()))
        self.world, self.rank = world, rank
        self._opened = []
        peers = [None] * world
        if world > 1:
            from cuda.bindings import driver as drv
            from cuda.bindings import runtime as rt
            err, base, _ = drv.cuMemGetAddressRange(self.buf.data_ptr())
            if err != drv.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"cuMemGetAddressRange: {err}")
            offset = self.buf.data_ptr() - int(base)
            err, handle = rt.cudaIpcGetMemHandle(int(base))
            if err != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaIpcGetMemHandle: {err}")
            mine = (bytes(handle.reserved), offset)
            allh = [None] * world
            dist.all_gather_object(allh, mine, group=group)
            for r, (hb, off) in enumerate(allh):
                if r == rank:
                    continue
                h = rt.cudaIpcMemHandle_t()
                h.reserved = hb
                err, ptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
                if err != rt.cudaError_t.cudaSuccess:
                    raise RuntimeError(f"cudaIpcOpenMemHandle (rank {r}): {err}")
                self._opened.append(int(ptr))
                peers[r] = int(ptr) + off
        self.ptrs = [self.buf.data_ptr()] + [peers[(rank + i) % world] for i in range(1, world)]

    def close(self):
        if self._opened:
            from cuda.bindings import runtime as rt
            for p in self._opened:
                rt.cudaIpcCloseMemHandle(p)
            self._opened = []


def _full_fused(self, b: torch.Tensor, outputs: PeerOutputs) -> torch.Tensor:
    """This rank's groups, each row stored into every rank's full output
    buffer from the epilogue; returns this rank's buffer once all ranks'
    kernels are complete (barrier)."""
    import torch.distributed as dist
    if self.plan.world > 1:
        # every rank is done reading the previous result: its enqueued readers
        # must have finished on the device, not just been issued (a host
        # barrier alone lets a peer's epilogue overwrite rows still being read)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
    self.sb.spmm_groups_peers(self.a, self.g0, self.g1, b, outputs.ptrs, dtype=outputs.buf.dtype,
                              ldc=outputs.buf.stride(0))
    if self.plan.world > 1:
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)  # all ranks' rows have landed everywhere
    return outputs.buf


ShardedSpMM.full_fused = _full_fused


class MulticastOutputs:
    """A full-size [M, N] output on every rank in torch symmetric memory, with
    the NVLS multicast address bound to all ranks' buffers (``mc_ptr``; 0 when
    the GPUs / driver offer no multicast, e.g. without NVSwitch).  Stores
    through ``mc_ptr`` land in every rank's ``buf``."""

    def __init__(self, shape, dtype, group=None, device=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.buf = symm_mem.empty(*shape, dtype=dtype, device=dev)
        self.buf.zero_()
        self.handle = symm_mem.rendezvous(self.buf, group or dist.group.WORLD)
        self.mc_ptr = int(getattr(self.handle, "multicast_ptr", 0) or 0)
        # the multicast address maps the buffer's allocation; this tensor may
        # sit at an offset inside it
        self.mc_offset = int(getattr(self.handle, "buffer_offset", 0) or 0) if self.mc_ptr else 0


def _full_multicast(self, b: torch.Tensor, outputs: MulticastOutputs) -> torch.Tensor:
    """This rank's groups, each row stored ONCE through the NVLS multicast
    address into every rank's full output buffer (one multimem.st per 16
    bytes, replicated by the switch); returns this rank's buffer once all
    ranks' kernels are complete."""
    import torch.distributed as dist
    if not outputs.mc_ptr:
        raise RuntimeError("no NVLS multicast address (MulticastOutputs.mc_ptr == 0)")
    if self.plan.world > 1:
        torch.cuda.current_stream().synchronize()  # readers of the previous result are done
        dist.barrier(group=self.group)
    self.sb.spmm_groups_multicast(self.a, self.g0, self.g1, b, outputs.mc_ptr + outputs.mc_offset,
                                  outputs.buf.dtype, outputs.buf.stride(0))
    torch.cuda.current_stream().synchronize()
    if self.plan.world > 1:
        dist.barrier(group=self.group)  # all ranks' rows have landed everywhere
    return outputs.buf


ShardedSpMM.full_multicast = _full_multicast
