"""Host-side logic of the multi-GPU path, CPU only.

* bmg_partition (C, host-only) gives contiguous slabs whose starts are
  multiples of 2^K and whose coarse-level ownership follows restriction
  (coarse row J is owned by the owner of fine row 2J);
* a world_size-2 gloo run performs the library's ghost-row exchange schedule
  (owned rows [ylo, ylo+HALO) to the lower neighbour, [yhi-HALO, yhi) to the
  upper one, local layout [max(ylo-HALO,0), min(yhi+HALO, ny+2))) with
  torch.distributed send/recv and checks every ghost row equals the global
  array's row -- the schedule the NCCL path runs on the GPU.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def bmg():
    import __graft_entry__ as ge

    ge.build_lib()
    from paper_2502_05279_b200 import bmg as b

    return b


def owned(yb, p, l, nyl):
    s = 1 << l
    return max((yb[p] + s - 1) // s, 1), min((yb[p + 1] + s - 1) // s, nyl + 1)


@pytest.mark.parametrize("n,P,agg", [(8191, 8, 128), (8191, 2, 128), (1023, 4, 16), (255, 3, 16), (4095, 5, 64)])
def test_partition_properties(bmg, n, P, agg):
    prm = bmg.bmg_params_default()
    prm.agglom_rows = agg
    yb, K = bmg.bmg_partition(n, n, P, prm)
    assert yb[0] == 1 and yb[-1] == n + 1 and K >= 1
    assert all(yb[p] < yb[p + 1] for p in range(P))
    assert all(yb[p] % (1 << K) == 0 for p in range(1, P))
    nyl = n
    for l in range(K):
        rows = [owned(yb, p, l, nyl) for p in range(P)]
        assert rows[0][0] == 1 and rows[-1][1] == nyl + 1
        assert all(rows[p][1] == rows[p + 1][0] for p in range(P - 1))  # contiguous cover
        assert min(b - a for a, b in rows) >= max(agg, 2 * bmg.BMG_HALO)
        # restriction ownership: coarse row J on level l+1 owned by the owner of fine row 2J on level l
        nyc = nyl // 2
        for p in range(P):
            a, b = owned(yb, p, l + 1, nyc)
            for J in (a, b - 1):
                if 1 <= J <= nyc:
                    assert rows[p][0] <= 2 * J < rows[p][1]
        nyl = nyc
    if K < 20:  # K is maximal: one more level would break the minimum slab height
        nyl = n
        for _ in range(K):
            nyl //= 2
        assert min(owned(yb, p, K, nyl)[1] - owned(yb, p, K, nyl)[0] for p in range(P)) < max(agg, 12) or \
            bmg.bmg_partition(n, n, P, prm)[1] == K


def test_partition_too_small(bmg):
    with pytest.raises(bmg.BmgError):
        bmg.bmg_partition(63, 63, 8, None)


def _exchange_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2502_05279_b200 import bmg

        G = bmg.BMG_HALO
        prm = bmg.bmg_params_default()
        prm.agglom_rows = 16
        yb, K = bmg.bmg_partition(n, n, world, prm)
        rng = np.random.default_rng(0)
        glob = rng.standard_normal((n + 2, n + 2))
        ok = True
        nyl = n
        for l in range(K):
            gl = glob[: nyl + 2, :]
            ylo, yhi = owned(yb, rank, l, nyl)
            roff, rend = max(ylo - G, 0), min(yhi + G, nyl + 2)
            loc = np.full((rend - roff, n + 2), np.nan)
            loc[ylo - roff: yhi - roff] = gl[ylo:yhi]  # owned rows only
            if ylo == 1:
                loc[0 - roff] = gl[0]
            if yhi == nyl + 1:
                loc[nyl + 1 - roff] = gl[nyl + 1]
            reqs, sends = [], []
            if rank > 0:
                g0 = max(ylo - G, 0)
                buf = torch.empty((ylo - g0, n + 2), dtype=torch.float64)
                reqs.append((dist.irecv(buf, rank - 1), buf, g0))
                t = torch.from_numpy(loc[ylo - roff: min(ylo + G, nyl + 2) - roff].copy())
                sends.append((dist.isend(t, rank - 1), t))
            if rank + 1 < world:
                g1 = min(yhi + G, nyl + 2)
                buf = torch.empty((g1 - yhi, n + 2), dtype=torch.float64)
                reqs.append((dist.irecv(buf, rank + 1), buf, yhi))
                t = torch.from_numpy(loc[max(yhi - G, 0) - roff: yhi - roff].copy())
                sends.append((dist.isend(t, rank + 1), t))
            for req, buf, r0 in reqs:
                req.wait()
                loc[r0 - roff: r0 - roff + buf.shape[0]] = buf.numpy()
            for req, _ in sends:
                req.wait()
            ok &= bool(np.array_equal(loc, gl[roff:rend]))
            nyl //= 2
        dist.barrier()
        q.put((rank, ok, K))
    finally:
        dist.destroy_process_group()


def test_gloo_ghost_exchange_world2(bmg):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, 511, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(K >= 2 for _, _, K in res)
