"""Multi-rank host logic on CPU (gloo, world size 2): LPT patch ownership is
a disjoint cover and the MIN all-reduce gathers the owners' values."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from paper_1109_3577_b200 import dist


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w = dist.world()
        mine = dist.mine_mask(sizes, r, w, "cpu")
        # each rank "solves" its patches: node value = patch id + 0.5 for
        # owned patches, unreached (1.0 -> here 99) elsewhere; target 0
        color = np.repeat(np.arange(len(sizes)), sizes)
        v = torch.full((color.size,), 99.0, dtype=torch.float64)
        owned = torch.as_tensor(mine.numpy()[color].astype(bool))
        v[owned] = torch.as_tensor(color, dtype=torch.float64)[owned] + 0.5
        dist.gather_min(v)
        q.put((rank, mine.numpy().tolist(), v.numpy().tolist()))
    finally:
        td.destroy_process_group()


def test_lpt_ownership_and_min_gather_world2():
    sizes = [7, 3, 5, 11, 2, 2, 9, 4]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    m0, m1 = np.array(out[0][1]), np.array(out[1][1])
    assert np.all(m0 + m1 == 1)  # every patch owned by exactly one rank
    loads = [sum(s for s, m in zip(sizes, mm) if m) for mm in (m0, m1)]
    assert max(loads) <= sum(sizes) / 2 + max(sizes)
    color = np.repeat(np.arange(len(sizes)), sizes)
    want = color + 0.5
    for _, _, v in out:
        assert np.array_equal(np.array(v), want)  # identical gathered field on every rank


def _argmax_worker(rank, world, port, phi, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R, n = phi.shape
        mine = dist.my_colours(R, rank, world)
        # local running argmax over this rank's colours (strict >, from (0, 0))
        bv = torch.zeros(n, dtype=torch.float64)
        bi = torch.zeros(n, dtype=torch.int32)
        first = True
        for j in mine:
            x = torch.as_tensor(phi[j])
            take = x > bv
            if first:
                bi[:] = int(j)
                first = False
            bv = torch.where(take, x, bv)
            bi = torch.where(take, torch.full_like(bi, int(j)), bi)
        if len(mine) == 0:
            bi[:] = R - 1
        dist.merge_argmax(bv, bi, R)
        q.put((rank, bv.numpy().tolist(), bi.numpy().tolist()))
    finally:
        td.destroy_process_group()


def test_colour_split_argmax_merge_world2():
    """Colours split round-robin over 2 ranks; the merged argmax equals the
    single-device running argmax (lowest colour on ties, (0, 0) when all
    colours are 0) on every rank."""
    rng = np.random.default_rng(7)
    R, n = 5, 400
    phi = rng.choice([0.0, 0.25, 0.5, 1.0], size=(R, n)) * (rng.random((R, n)) < 0.6)
    phi[:, :20] = 0.0            # all-zero nodes
    phi[1:4, 20:40] = 0.75        # exact ties across ranks
    # reference: strict > scan over all colours
    want_v = np.zeros(n)
    want_i = np.zeros(n, dtype=np.int64)
    for j in range(R):
        t = phi[j] > want_v
        want_v = np.where(t, phi[j], want_v)
        want_i = np.where(t, j, want_i)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_argmax_worker, args=(r, 2, port, phi, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pos = want_v > 0
    for _, v, i in out:
        assert np.array_equal(np.array(v), want_v)
        assert np.array_equal(np.array(i)[pos], want_i[pos])  # index only matters where v > 0


def test_lpt_weights_change_the_assignment():
    # measured per-patch work (not node counts) decides the LPT bins when given
    from paper_1109_3577_b200 import dist

    sizes = [100, 90, 80, 10]
    work = [10.0, 90.0, 80.0, 100.0]
    by_nodes = dist.lpt_assign(sizes, 2)
    by_work = dist.lpt_assign(sizes, 2, work)
    assert by_nodes.tolist() == [0, 1, 1, 0]
    load = lambda owner: np.bincount(owner, weights=work, minlength=2).max()
    assert load(by_work) <= load(by_nodes)
    assert by_work[3] == 0  # the heaviest measured patch is placed first
    m0 = dist.mine_mask(sizes, 0, 2, "cpu", work).numpy()
    m1 = dist.mine_mask(sizes, 1, 2, "cpu", work).numpy()
    assert np.array_equal(m0 + m1, np.ones(4, dtype=np.uint8))


def _slab_worker(rank, world, port, n_rows, row_elems, n_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        calls = []

        def compute(b, e, field):
            # the slab's serials hold their own global index
            calls.append((b, e))
            field[b * row_elems:e * row_elems] = torch.arange(b * row_elems, e * row_elems,
                                                              dtype=torch.int32)

        out = dist.gather_slabs(compute, n_rows, row_elems, n_total, torch.int32, "cpu")
        q.put((rank, calls, out.numpy().tolist()))
    finally:
        td.destroy_process_group()


def test_slab_split_and_all_gather_world2():
    """The feedback stage split by slabs of block rows (dist.gather_slabs,
    solver.feedback_sharded): disjoint slabs covering every row, the
    all-gathered field complete on both ranks -- also when the rows do not
    divide evenly and the last block row is partial."""
    n_rows, row_elems, n_total = 7, 5, 33  # 7 block rows of 5 serials, the last one partial
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, n_rows, row_elems, n_total, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == [(0, 4)] and out[1][1] == [(4, 7)]
    for _, _, field in out:
        assert field == list(range(n_total))
    assert dist.slab_bounds(5, 8) == [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 5), (5, 5),
                                      (5, 5)]
