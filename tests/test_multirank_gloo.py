"""Multi-rank host logic on CPU (world size 2, gloo): each rank runs the host half of
pcg_setup (pcg_plan_build) on its own row block, the ranks exchange their results over
torch.distributed, and rank 0 checks them against the oracle's partitioned AINV (block-local,
w = 0) bit for bit.  The NCCL data path itself needs GPUs; its 1-rank instance is
covered by tests/test_gpu_parity.py::test_host_loop_and_comm_path_match_graph."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, halo, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1210_1878_b200 as pcg
        from paper_1210_1878_b200 import synth
        p = synth.config(name)
        rb = pcg.partition(p.ni, p.nj, p.mask, world)
        allrb = [None] * world
        dist.all_gather_object(allrb, rb.tolist())
        pl = pcg.Plan(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, j_begin=int(rb[rank]), j_end=int(rb[rank + 1]),
                      rank=rank, nranks=world, ainv_halo=halo)
        mine = dict(rank=rank, rows=(int(rb[rank]), int(rb[rank + 1])), n=pl.n_owned, first=pl.first_global,
                    zh=[a.tolist() for a in pl.export_zhat()])
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        # uid-style broadcast of an opaque 128-byte blob (the NCCL unique id path of Solver)
        blob = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        if rank == 0:
            q.put(dict(rb=allrb, parts=allp, blob_ok=blob[0] == bytes(range(128))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,halo", [("cfg1", 0), ("cfg2", 0), ("cfg2", 2), ("cfg2", 3), ("cfg2", 10 ** 6)])
def test_two_rank_setup_matches_oracle_partitioned(name, halo):
    """halo = 0: block-local AINV per rank; halo = w > 0: each rank's block starts w rows below its
    first row (halo-AINV across ranks), so its owned columns carry entries in those rows."""
    import oracle
    from paper_1210_1878_b200 import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, halo, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = synth.config(name)
    A = oracle.assemble(p)
    rb = oracle.partition(p.nj, p.ni, p.mask, world)
    assert res["rb"][0] == res["rb"][1] == rb.tolist()
    assert res["blob_ok"]
    ref = oracle.ainv(A, 0.1 + 1e-9, parts=world, halo=halo)
    if halo >= p.nj:    # NEXT-3 global Z: the ranks' columns stitch into the one-rank factor
        ref = oracle.ainv(A, 0.1 + 1e-9)
    parts = sorted(res["parts"], key=lambda d: d["rank"])
    assert sum(d["n"] for d in parts) == A.n
    assert parts[0]["first"] == 0 and parts[1]["first"] == parts[0]["n"]
    # stitch the owned columns of both ranks into the global CSC and compare bitwise
    colptr = [0]
    rows, zh, piv, sc = [], [], [], []
    for d in parts:
        cp, r, z, pv, s = (np.asarray(a) for a in d["zh"])
        rows.extend(r.tolist()); zh.extend(z.tolist()); piv.extend(pv.tolist()); sc.extend(s.tolist())
        colptr.extend((cp[1:] + colptr[-1]).tolist())
    assert np.array_equal(np.asarray(colptr), ref.colptr)
    assert np.array_equal(np.asarray(rows), ref.row)
    assert np.array_equal(np.asarray(zh), ref.zhat)
    assert np.array_equal(np.asarray(piv), ref.pivots)
    assert np.array_equal(np.asarray(sc), ref.scale)
    cols = np.repeat(np.arange(A.n), np.diff(ref.colptr))
    owner = np.searchsorted(np.cumsum([d["n"] for d in parts]), np.arange(A.n), side="right")
    if halo == 0:       # block-local: no entry of a rank's columns lies in the other rank's rows
        assert np.all(owner[ref.row] == owner[cols])
    else:               # halo-AINV: rank 1's columns reach into rank 0's top rows, never the reverse
        cross = owner[ref.row] != owner[cols]
        assert cross.any() and np.all(owner[cols[cross]] == 1) and np.all(owner[ref.row[cross]] == 0)


def test_multirank_canonical_sum_is_rank_tree():
    """The multi-rank canonical dot = 32-lane tree over the rank sums: with
    integer-valued inputs every order is exact, so the 2-part value equals the 1-part value."""
    import oracle
    from paper_1210_1878_b200 import synth
    p = synth.config("cfg2")
    A = oracle.assemble(p)
    rng = np.random.default_rng(3)
    a = rng.integers(-50, 50, A.n).astype(float)
    b = rng.integers(-50, 50, A.n).astype(float)
    exact = float(np.dot(a.astype(np.int64), b.astype(np.int64)))
    for parts in (1, 2, 4, 8):
        assert A.dot_canonical(a, b, pitch=192, parts=parts) == exact
