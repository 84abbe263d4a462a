"""Output-channel (tile-row) sharding of the FPx linear across GPUs.

North-star item (4): large weights are column-partitioned (reference rows M =
output channels) across ranks, one process per GPU; the full output is
assembled with an NCCL all-gather over NVLink only when it is required.

* Partition: rank r owns tile-rows [tr0, tr1) (fpx_shard_rows, balanced to
  one 64-row tile-row).  Tiles are stored in row-major tile order
  (reference prepack.cpp:190-191), so a rank's share of every packed stream
  is ONE contiguous byte range and its scales are one contiguous slice --
  sharding is zero-copy slicing of the packed buffers (PackedWeights.shard).
* Compute: each rank runs the fused kernel on its shard with the FULL
  problem's split_k, so the per-element K reduction (chunking, MMA order,
  fixed-order split-K fold) is identical to the unsharded launch and the
  rows a rank produces are bit-identical to the same rows of a 1-GPU run.
* Gather: each rank's fp32 col-major slice [n][m_local] is padded to the
  largest shard (m_slot rows), all-gathered into [world][n][m_slot] with
  torch.distributed (NCCL), and scattered into col-major C by the
  fpx_gather_permute kernel.  The weights never move.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .fpx import PackedWeights, _check, default_split, gemm_packed

__all__ = ["shard_tile_rows", "shard_layout", "local_shard", "sharded_linear", "gather_output", "cuda_permute"]


def shard_tile_rows(rows_p: int, rank: int, world: int) -> tuple[int, int]:
    """Tile-row range of `rank` (mirrors fpx_shard_rows in the C-ABI)."""
    trs = rows_p // 64
    world = max(world, 1)
    return trs * rank // world, trs * (rank + 1) // world


def shard_layout(rows_p: int, world: int):
    """Per-rank (first row, row count) and the padded slot height m_slot."""
    row0, nrows = [], []
    for r in range(world):
        a, b = shard_tile_rows(rows_p, r, world)
        row0.append(a * 64)
        nrows.append((b - a) * 64)
    return row0, nrows, max(nrows) if nrows else 0


def local_shard(p: PackedWeights, rank: int, world: int) -> PackedWeights:
    tr0, tr1 = shard_tile_rows(p.rows, rank, world)
    return p.shard(tr0, tr1)


def cuda_permute(gathered: torch.Tensor, row0, nrows, m_slot: int, n: int, out: torch.Tensor) -> torch.Tensor:
    """[world][n][m_slot] -> col-major out [n][ldc] on the GPU (fpx_gather_permute)."""
    L = _lib.load()
    dev = gathered.device
    r0 = torch.tensor(row0, dtype=torch.int32, device=dev)
    nr = torch.tensor(nrows, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _check(L.fpx_gather_permute(gathered.data_ptr(), r0.data_ptr(), nr.data_ptr(), len(row0), m_slot, n,
                                    out.data_ptr(), out.shape[1], torch.cuda.current_stream(dev).cuda_stream))
    return out


def gather_output(c_local: torch.Tensor, rows_p: int, rank: int, world: int, group=None,
                  permute=cuda_permute) -> torch.Tensor:
    """All-gather the ranks' [n, m_local] slices into the full [n, rows_p] C."""
    import torch.distributed as dist
    n = c_local.shape[0]
    row0, nrows, m_slot = shard_layout(rows_p, world)
    assert c_local.shape[1] == nrows[rank]
    padded = torch.zeros((n, m_slot), dtype=c_local.dtype, device=c_local.device)
    padded[:, :nrows[rank]] = c_local
    gathered = torch.empty((world * n, m_slot), dtype=c_local.dtype, device=c_local.device)
    if padded.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (CPU-side tests, several ranks sharing one GPU): stage through host memory
        host = torch.empty((world * n, m_slot), dtype=c_local.dtype)
        dist.all_gather_into_tensor(host, padded.cpu(), group=group)
        gathered.copy_(host)
    else:
        dist.all_gather_into_tensor(gathered, padded, group=group)  # rank-major concatenation (NCCL over NVLink)
    out = torch.empty((n, rows_p), dtype=c_local.dtype, device=c_local.device)
    return permute(gathered.view(world, n, m_slot), row0, nrows, m_slot, n, out)


def sharded_linear(p: PackedWeights, b: torch.Tensor, rank: int, world: int, group=None, *, gather: bool = True,
                   split_k: int = 0, compute=gemm_packed, permute=cuda_permute) -> torch.Tensor:
    """C = dequant(W) x B with W's tile-rows sharded over `world` ranks.

    `p` is the full packed matrix (or any object whose .shard() yields this
    rank's slice); only this rank's tile-rows are read.  split_k defaults to
    the unsharded problem's split so every rank's rows are bit-identical to a
    single-GPU launch.  Returns [n, rows_p] (gather=True) or this rank's
    [n, m_local] slice."""
    n = b.shape[0]
    sk = split_k or default_split(p.rows, p.cols, n)
    tr0, tr1 = shard_tile_rows(p.rows, rank, world)
    if tr1 > tr0:
        c_local = compute(p.shard(tr0, tr1), b, split_k=sk)
    else:
        # more ranks than tile-rows: this rank owns nothing but must still
        # join the collective, or the other ranks block in all_gather forever
        c_local = torch.empty((n, 0), dtype=torch.float32, device=b.device)
    if not gather or world == 1:
        return c_local
    return gather_output(c_local, p.rows, rank, world, group, permute=permute)
