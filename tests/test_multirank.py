"""Multi-rank row partitioning on CPU (gloo, world_size 2): each rank takes
its nnz-balanced row block by the library's own boundary rule
(sfgx_row_bounds_host, the rule sfg_row_partition applies on the device),
computes its slice of y (the CPU oracle stands in for the device SpMV), and
the padded all-gather reassembles exactly the full product."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2403_05802_b200.rowpart import row_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_bounds_balance():
    rng = np.random.default_rng(0)
    # power-law rows: heavy rows first, like R-MAT
    lens = np.sort((rng.pareto(1.3, 1000) * 10).astype(int))[::-1]
    rows = np.repeat(np.arange(1000), lens)
    for parts in (1, 2, 4, 8):
        b = row_bounds(rows, 1000, parts)
        assert b[0] == 0 and b[-1] == 1000 and all(x <= y for x, y in zip(b, b[1:]))
        counts = [np.sum((rows >= b[p]) & (rows < b[p + 1])) for p in range(parts)]
        # rows are indivisible: each block is within two rows of nnz / P
        assert all(abs(cnt - len(rows) / parts) <= 2 * lens.max() for cnt in counts)
    assert row_bounds(np.zeros(0, int), 10, 4) == [0, 2, 5, 7, 10]


def test_library_host_rule_matches_restatement():
    """sfgx_row_bounds_host (C-ABI, no GPU) == rowpart.row_bounds."""
    import paper_2403_05802_b200 as sfg
    rng = np.random.default_rng(1)
    for m, nnz in ((1, 0), (10, 0), (1000, 5000), (4096, 70000)):
        rows = np.sort(rng.integers(0, m, nnz)).astype(np.int32)
        for parts in (1, 2, 3, 4, 8, 16):
            assert sfg.row_bounds_host(rows, m, parts) == row_bounds(rows, m, parts), (m, nnz, parts)


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    import oracle
    from matrices import power_law_coo
    import paper_2403_05802_b200 as sfg
    from paper_2403_05802_b200.rowpart import gather_rows, padded_chunk, row_bounds, unpad

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_lib = oracle.Port()
    m, n = 900, 700
    r, c, v = power_law_coo(3, m, n, avg=9)
    x = np.random.default_rng(1).random(n)
    b = sfg.row_bounds_host(r, m, world)
    assert b == row_bounds(r, m, world)
    sel = (r >= b[rank]) & (r < b[rank + 1])
    mloc = b[rank + 1] - b[rank]
    loc = port_lib.from_coo(max(mloc, 1), n, r[sel] - b[rank], c[sel], v[sel])
    y_loc = port_lib.spmv(port_lib.convert(loc, "CSR"), x)[:mloc]
    chunk = padded_chunk(mloc)
    pad = torch.zeros(chunk, dtype=torch.float64)
    pad[:mloc] = torch.from_numpy(y_loc)
    y = unpad(gather_rows(pad, chunk), b, chunk).numpy()
    if rank == 0:
        full = port_lib.spmv(port_lib.convert(port_lib.from_coo(m, n, r, c, v), "CSR"), x)
        np.save(result_path, np.stack([y, full]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_spmv_reassembly(tmp_path):
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    y, full = np.load(out)
    # same rows, same per-row f64 walk order => identical
    np.testing.assert_array_equal(y, full)
