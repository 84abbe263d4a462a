"""CPU (gloo, world_size 2/3) tests of the multi-GPU host logic in
paper_2401_14112_b200/shard.py: tile-row partition, zero-copy shard views of
the packed streams, the padded all-gather and the output permutation.  The
per-rank compute is the C oracle (test infrastructure) instead of the GPU
kernel, and the permutation is done with torch slicing on CPU tensors; the
GPU path (fpx_linear + fpx_gather_permute) is covered by tests/test_gpu_*.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_14112_b200 import shard
from paper_2401_14112_b200.fpx import FpxFormat, PackedWeights, SplitScheme


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torch_permute(gathered, row0, nrows, m_slot, n, out):
    for r in range(len(row0)):
        out[:, row0[r]:row0[r] + nrows[r]] = gathered[r, :, :nrows[r]]
    return out


def _make_problem(rows, cols, n, e, m, seed):
    from oracle.oracle import Oracle
    O = Oracle()
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    st, codes, scales, _ = O.quantize(w, e, m)
    assert st == 0
    st, streams = O.pack(codes, scales, e, m)
    b = rng.standard_normal((n, cols)).astype(np.float16)
    st, c_full = O.gemm_reference(codes, scales, e, m, b.view(np.uint16), orig_cols=cols)
    fmt = FpxFormat(e, m)
    p = PackedWeights(fmt, SplitScheme.for_format(fmt), codes.shape[0], codes.shape[1], rows, cols,
                      [torch.from_numpy(s) for s in streams], torch.from_numpy(scales.view(np.int16)))
    return p, b, c_full


def _oracle_compute(local: PackedWeights, b, split_k=0):
    from oracle.oracle import Oracle
    O = Oracle()
    e, m = local.format.exp_bits, local.format.man_bits
    streams = [s.numpy() for s in local.streams]
    st, codes = O.unpack(streams, local.rows, local.cols, e, m)
    assert st == 0
    scales = local.scales.numpy().view(np.uint16)
    st, c = O.gemm_reference(codes, scales, e, m, b.view(np.uint16), orig_cols=b.shape[1])
    assert st == 0
    return torch.from_numpy(c)


def _worker(rank, world, port, rows, cols, n, e, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, b, c_full = _make_problem(rows, cols, n, e, m, seed=rows + cols)
        c = shard.sharded_linear(p, b, rank, world, compute=_oracle_compute, permute=_torch_permute, split_k=1)
        ok = bool((c.numpy().view(np.uint32) == c_full.view(np.uint32)).all())
        local = shard.local_shard(p, rank, world)
        tr0, tr1 = shard.shard_tile_rows(p.rows, rank, world)
        # zero-copy: the shard's streams alias the full buffers at the tile-row offset
        gc = p.cols // 64
        alias = all(ls.data_ptr() == fs.data_ptr() + tr0 * gc * 512 * w
                    for ls, fs, w in zip(local.streams, p.streams, p.split.widths))
        q.put((rank, ok, alias, local.rows == (tr1 - tr0) * 64))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,n,fmt", [(2, 256, 192, 3, (3, 2)), (2, 2752 // 8, 128, 1, (2, 2)),
                                                    (3, 448, 128, 8, (2, 3))])
def test_sharded_linear_gloo(world, rows, cols, n, fmt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, n, fmt[0], fmt[1], q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=90) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok, alias, shape_ok in res:
        assert ok, f"rank {rank}: gathered C differs from the unsharded oracle"
        assert alias and shape_ok


def test_shard_layout_covers_all_rows():
    for rows_p in (64, 128, 2752, 8192, 22016, 28672):
        for world in (1, 2, 3, 4, 8):
            row0, nrows, m_slot = shard.shard_layout(rows_p, world)
            assert sum(nrows) == rows_p and m_slot == max(nrows)
            assert all(row0[i] + nrows[i] == row0[i + 1] for i in range(world - 1))


def test_concat_rows_is_shard_inverse():
    """PackedWeights.concat_rows (merged gate/up, Q/K/V) is the byte-level
    inverse of shard(): concatenating the tile-row shards of a packed weight
    gives back its streams and scales exactly, and mismatched parts are
    rejected (host logic; the GPU bit-identity of the merged linear is
    tests/test_gpu_parity.py::test_concat_rows_equals_separate_linears)."""
    from oracle.oracle import Oracle
    from paper_2401_14112_b200.fpx import FpxError
    O = Oracle()
    rng = np.random.default_rng(5)
    rows, cols = 320, 256
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    st, codes, scales, _ = O.quantize(w, 3, 2)
    st, streams = O.pack(codes, scales, 3, 2)
    p = PackedWeights(FpxFormat(3, 2), SplitScheme((2, 4)), rows, cols, rows, cols,
                      [torch.from_numpy(s) for s in streams], torch.from_numpy(scales.view(np.int16)))
    parts = [p.shard(0, 1), p.shard(1, 3), p.shard(3, 5)]
    q = PackedWeights.concat_rows(parts)
    assert q.rows == rows and q.cols == cols
    assert all(torch.equal(a, b) for a, b in zip(q.streams, p.streams))
    assert torch.equal(q.scales, p.scales)
    other = PackedWeights(FpxFormat(3, 2), SplitScheme((2, 4)), 64, 128, 64, 128,
                          [torch.zeros(64 * 128 * 2 // 8, dtype=torch.uint8),
                           torch.zeros(64 * 128 * 4 // 8, dtype=torch.uint8)], torch.zeros(64, dtype=torch.int16))
    with pytest.raises(FpxError):
        PackedWeights.concat_rows([parts[0], other])
