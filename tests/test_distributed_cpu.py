"""Multi-process (gloo, world_size 2) checks of the row-slab contract on CPU.

Each rank owns the slab of `slab_plan`; halo rows are exchanged exactly as the
library's Comm::exchange does (first rows to rank-1, last rows to rank+1); the
slab apply computed from the halo'd slab must equal the whole-grid apply bit
for bit (oracle operators), and distributed dots must match the global dot."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2412_04980_b200.distributed import slab_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, size, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        hier, b = oracle.mp1_problem(30.0, 129, 4, ("sommerfeld", "dirichlet", "sommerfeld", "dirichlet"))
        ny = hier.level(1).ny
        plan = slab_plan(ny, size, max_depth=7, min_rows=16)
        rng = np.random.default_rng(3)
        checks = {}
        for level in (1, 2, 3):
            depth = level - 1
            op = oracle.helmholtz_op(hier, level)
            u = rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)
            full = op.apply(u)
            if not plan.sharded(depth):
                checks[level] = "replicated"
                continue
            r0, n = plan.slab(depth, rank)
            R = op.r
            # halo exchange (Comm::exchange contract) over gloo
            mine = torch.from_numpy(u[r0:r0 + n].copy())
            up = torch.zeros((R, op.nx), dtype=torch.complex128)
            down = torch.zeros((R, op.nx), dtype=torch.complex128)
            ops = []
            if rank > 0:
                ops += [dist.P2POp(dist.isend, mine[:R].contiguous(), rank - 1),
                        dist.P2POp(dist.irecv, up, rank - 1)]
            if rank < size - 1:
                ops += [dist.P2POp(dist.isend, mine[n - R:].contiguous(), rank + 1),
                        dist.P2POp(dist.irecv, down, rank + 1)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            lo = r0 - R if rank > 0 else r0
            ext = np.concatenate(([up.numpy()] if rank > 0 else []) + [mine.numpy()] +
                                 ([down.numpy()] if rank < size - 1 else []), axis=0)
            kext = hier.ksq_at(level)[lo:lo + ext.shape[0]]
            bnd = list(hier.boundary)
            if rank > 0:
                bnd[2] = "sommerfeld"   # artificial edges: closure only touches discarded halo outputs
            if rank < size - 1:
                bnd[3] = "sommerfeld"
            lt, ld, mt, md, _ = oracle.level_kernels(level)
            eop = oracle.CpuLevelOp(op.nx, ext.shape[0], op.h, kext, bnd, lt, ld, mt, md, 1.0,
                                    oracle.mass_level_scale(level))
            got = eop.apply(ext)[r0 - lo:r0 - lo + n]
            checks[level] = bool(np.array_equal(got, full[r0:r0 + n]))
        # distributed dot: local partial + all-reduce
        u = rng.standard_normal((ny, hier.level(1).nx)) + 1j * rng.standard_normal((ny, hier.level(1).nx))
        v = rng.standard_normal(u.shape) + 1j * rng.standard_normal(u.shape)
        r0, n = plan.slab(0, rank)
        part = torch.tensor([np.vdot(u[r0:r0 + n], v[r0:r0 + n])], dtype=torch.complex128)
        dist.all_reduce(part)
        ref = np.vdot(u, v)
        checks["dot"] = abs(complex(part.item()) - ref) <= 1e-13 * abs(ref)
        checks["depths"] = plan.depths
        q.put((rank, checks))
    finally:
        dist.destroy_process_group()


def test_slab_apply_and_dot_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, checks in res.items():
        assert checks["depths"] >= 2
        for level in (1, 2, 3):
            assert checks[level] in (True, "replicated"), (rank, level, checks[level])
        assert checks[1] is True and checks[2] is True
        assert checks["dot"]


@pytest.mark.parametrize("ny,ranks", [(4097, 8), (4097, 2), (2001, 8), (129, 4), (9, 2)])
def test_slab_plan_nesting_and_balance(ny, ranks):
    max_depth = 1
    while (ny - 1) % 2 ** max_depth == 0 and (ny - 1) // 2 ** max_depth + 1 >= 3:
        max_depth += 1
    plan = slab_plan(ny, ranks, max_depth, min_rows=32)
    for d in range(plan.depths):
        rows = [plan.slab(d, r) for r in range(ranks)]
        assert rows[0][0] == 0 and sum(n for _, n in rows) == plan.rows_at(d)
        assert all(a[0] + a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert min(n for _, n in rows) >= 32
        if d > 0:
            assert all(plan.slab(d - 1, r)[0] == 2 * rows[r][0] for r in range(ranks))
    if ny == 4097 and ranks == 8:
        assert plan.depths == 5  # 4097..257 sharded, 129 and below replicated


def _gather_rank(rank, size, port, q, ny, min_rows):
    """Sharded -> replicated transition with the library's own row rule: each rank
    exchanges 2 halo rows of its last-sharded-depth slab (Comm::exchange
    contract), restricts the coarse rows hdb_plan_gather_rows assigns it (from
    its halo'd slab only; rows it does not hold are zeros, so a rule that reads
    beyond the exchanged halo shows up as a mismatch), and the all-gather of those
    rows must equal the whole-grid restriction bit for bit."""
    import torch
    import torch.distributed as dist
    from paper_2412_04980_b200.distributed import gather_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        max_depth = 1
        while (ny - 1) % 2 ** max_depth == 0 and (ny - 1) // 2 ** max_depth + 1 >= 3:
            max_depth += 1
        plan = slab_plan(ny, size, max_depth, min_rows=min_rows)
        d = plan.depths - 1  # last sharded depth
        nyf = plan.rows_at(d)
        nx = 33
        rng = np.random.default_rng(11)
        fine = rng.standard_normal((nyf, nx)) + 1j * rng.standard_normal((nyf, nx))  # same on every rank
        r0, n = plan.slab(d, rank)
        mine = torch.from_numpy(fine[r0:r0 + n].copy())
        H = 2
        up = torch.zeros((H, nx), dtype=torch.complex128)
        down = torch.zeros((H, nx), dtype=torch.complex128)
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, mine[:H].contiguous(), rank - 1), dist.P2POp(dist.irecv, up, rank - 1)]
        if rank < size - 1:
            ops += [dist.P2POp(dist.isend, mine[n - H:].contiguous(), rank + 1),
                    dist.P2POp(dist.irecv, down, rank + 1)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        local = np.zeros_like(fine)  # only what this rank holds after the exchange
        local[r0:r0 + n] = mine.numpy()
        if rank > 0:
            local[r0 - H:r0] = up.numpy()
        if rank < size - 1:
            local[r0 + n:r0 + n + H] = down.numpy()
        c0, cn = gather_rows(plan, d, rank)
        part = oracle.restrict(local)[c0:c0 + cn]
        # all-gather of variable-size row blocks (the library's allgatherv)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(size)]
        dist.all_gather(sizes, torch.tensor([cn], dtype=torch.int64))
        mx = int(max(s.item() for s in sizes))
        buf = torch.zeros((mx, part.shape[1]), dtype=torch.complex128)
        buf[:cn] = torch.from_numpy(part)
        outs = [torch.zeros_like(buf) for _ in range(size)]
        dist.all_gather(outs, buf)
        gathered = np.concatenate([o[:int(s.item())].numpy() for o, s in zip(outs, sizes)], axis=0)
        ref = oracle.restrict(fine)
        q.put((rank, {"equal": bool(np.array_equal(gathered, ref)), "starts": [plan.slab(d, r)[0] for r in range(size)],
                      "rows": (c0, cn)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ny,size,min_rows", [(129, 3, 8), (257, 3, 16), (129, 2, 16)])
def test_sharded_to_replicated_gather_rule_over_gloo(ny, size, min_rows):
    """P = 3 gives odd slab starts at the last sharded depth (a floor
    rule read a fine row outside the 2-row halo there)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_rank, args=(r, size, port, q, ny, min_rows)) for r in range(size)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, r in res.items():
        assert r["equal"], (rank, r)
    if size == 3:
        assert any(s % 2 for s in res[0]["starts"]), res[0]["starts"]  # the odd-start case is exercised
