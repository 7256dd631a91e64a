"""NEXT-2 host logic on the CPU (no GPU): the row partition, each rank's local numbering / halo /
send lists (ajm_partition_rows, ajm_shard_plan of libajm.so -- host-only entry points), and a
world_size-2 gloo run of the sharded iteration built on exactly those plans: every rank
multiplies its rows by [its halo | own | halo] entries, the halo of x~^{t+1} travels over
torch.distributed (gloo), the five partials are all-gathered and summed in rank order, and every
rank takes the control decisions of Alg. 3 -- the same exchange the CUDA kernel does
over peer memory.  The result must be the oracle's (unsharded, literal two-SpMV) to 1e-10."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth


def _ajm():
    import paper_2407_03272_b200 as ajm
    ajm.lib()  # the host entry points need no CUDA device
    return ajm


@pytest.mark.parametrize("cfg,scale,R", [(1, 1.0, 1), (1, 1.0, 3), (2, 0.25, 8), (3, 0.02, 5), (4, 0.0125, 4)])
def test_partition_and_plan_consistency(cfg, scale, R):
    ajm = _ajm()
    p = synth.config_problem(cfg, scale)
    Q = p.Q
    st = ajm.ajm_partition_rows(Q.row_ptr, R)
    assert st[0] == 0 and st[-1] == Q.n and np.all(np.diff(st) >= 1)
    cost = 12.0 * np.diff(Q.row_ptr[st]) + 56.0 * np.diff(st)
    assert cost.max() <= cost.sum() / R + 12.0 * np.diff(Q.row_ptr).max() + 56.0 + 1e-9  # balanced to one row
    plans = []
    for r in range(R):
        rp, cg, vv = ajm.shard_rows(Q.row_ptr, Q.col, Q.val, st, r)
        pl = ajm.ajm_shard_plan(r, R, st, rp, cg)
        r0, r1 = st[r], st[r + 1]
        nl = r1 - r0
        halo = pl["halo_glob"]
        assert np.all(np.diff(halo) > 0) and np.all((halo < r0) | (halo >= r1))
        assert pl["h_lo"] == int(np.sum(halo < r0))
        # local column -> global index is the inverse of the plan's numbering
        ext = np.concatenate([halo[:pl["h_lo"]], np.arange(r0, r1), halo[pl["h_lo"]:]])
        np.testing.assert_array_equal(ext[pl["col_loc"].astype(np.int64) + pl["h_lo"]], cg)
        # the halo is exactly the set of referenced off-block columns
        off = np.unique(cg[(cg < r0) | (cg >= r1)])
        np.testing.assert_array_equal(off, halo)
        owners = np.searchsorted(st, halo, side="right") - 1
        np.testing.assert_array_equal(np.bincount(owners, minlength=R), pl["halo_cnt"])
        plans.append(pl)
    # rank s's send list to r (its rows, ascending) is r's halo entries owned by s, in order
    for r in range(R):
        hal = plans[r]["halo_glob"]
        owners = np.searchsorted(st, hal, side="right") - 1
        for s in range(R):
            if s == r:
                assert plans[s]["send_cnt"][r] == 0
                continue
            off = np.concatenate([[0], np.cumsum(plans[s]["send_cnt"])])
            rows = plans[s]["send_rows"][off[r]:off[r + 1]] + st[s]
            np.testing.assert_array_equal(rows, hal[owners == s])


def test_partition_errors():
    ajm = _ajm()
    rp = np.array([0, 1, 2, 3], dtype=np.int64)
    with pytest.raises(ajm.AjmError):
        ajm.ajm_partition_rows(rp, 4)  # more ranks than rows
    with pytest.raises(ajm.AjmError):
        ajm.ajm_partition_rows(rp, 0)
    with pytest.raises(ajm.AjmError):
        ajm.ajm_partition_rows(np.array([0, 2, 1, 3], dtype=np.int64), 2)
    with pytest.raises(ajm.AjmError):  # column outside [0, n)
        ajm.ajm_shard_plan(0, 2, [0, 1, 3], np.array([0, 1]), np.array([5], dtype=np.int32))


# ---------------- world_size-2 gloo run of the sharded iteration ----------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_alg3(rank, R, cfg, scale, maxit, restart, dist):
    """Alg. 3 with s = R row blocks, single-SpMV form (R22), driven by the
    library's host plan; the exchange goes through torch.distributed (gloo)."""
    ajm = _ajm()
    p = synth.config_problem(cfg, scale)
    Q = p.Q
    st = ajm.ajm_partition_rows(Q.row_ptr, R)
    rp, cg, vv = ajm.shard_rows(Q.row_ptr, Q.col, Q.val, st, rank)
    pl = ajm.ajm_shard_plan(rank, R, st, rp, cg)
    r0, r1 = int(st[rank]), int(st[rank + 1])
    nl, hlo, hhi = r1 - r0, pl["h_lo"], pl["h_hi"]
    cl = pl["col_loc"].astype(np.int64) + hlo  # index into ext = [lo halo | own | hi halo]
    rows = np.repeat(np.arange(nl), np.diff(rp))
    diagmask = cl == rows + hlo
    D = np.zeros(nl)
    np.add.at(D, rows, np.where(diagmask, vv, np.abs(vv)))  # eq-J-diag
    b = p.b[r0:r1]
    soff = np.concatenate([[0], np.cumsum(pl["send_cnt"])])
    # where each source rank's entries land in this rank's ext vector
    halo_owner = np.searchsorted(st, pl["halo_glob"], side="right") - 1
    hidx = np.arange(hlo + hhi)
    ext_of_halo = np.where(hidx < hlo, hidx, hidx + nl)  # halo entry k -> its index in ext
    recv_pos = [ext_of_halo[halo_owner == s] for s in range(R)]

    def exchange(x_own):
        ext = np.empty(hlo + nl + hhi)
        ext[hlo:hlo + nl] = x_own
        outs = [x_own[pl["send_rows"][soff[s]:soff[s + 1]]] for s in range(R)]  # per destination
        gathered = [None] * R
        dist.all_gather_object(gathered, outs)
        for s in range(R):
            if s != rank:
                ext[recv_pos[s]] = gathered[s][rank]
        return ext

    def allreduce5(v):
        parts = [None] * R
        dist.all_gather_object(parts, np.asarray(v, dtype=np.float64))
        tot = np.zeros(5)
        for s in range(R):  # rank order
            tot = tot + parts[s]
        return tot

    def spmv(ext):
        q = np.zeros(nl)
        np.add.at(q, rows, vv * ext[cl])
        return q

    nb = np.sqrt(allreduce5([float(np.dot(b, b)), 0, 0, 0, 0])[0])
    xt = np.zeros(nl)
    xp = np.zeros(nl)
    qxp = np.zeros(nl)
    alpha, beta, rst, K, Kre, t = 1.0, 0.0, False, 2, 0, 0
    restarts = []
    ext = exchange(xt)
    while True:
        q = spmv(ext)
        if not rst:
            y = xt + beta * (xt - xp)
            qy = q + beta * (q - qxp)
            xnow = xt
        else:
            y, qy, xnow = xp, qxp, xp
        xn = y + (b - qy) / D
        tot = allreduce5([np.sum((b - q) ** 2), np.dot(xt, q), np.dot(b, xt), np.sum((qy - b) * (xn - xnow)), 0])
        res = np.sqrt(tot[0]) / nb
        if t >= 1 and rst:
            restarts.append(t)
        if t == maxit:
            return (xp if rst else xt), t, restarts, st
        tn = t + 1
        rs = restart and tn > Kre + K and tot[3] >= 0.0
        an = (1.0 + np.sqrt(1.0 + 4.0 * alpha * alpha)) / 2.0
        if rs:
            Kre, K, alpha, beta_n = tn, 2 * K, 1.0, 0.0
        else:
            beta_n = (alpha - 1.0) / an
            alpha = an
        if not rst:
            qxp = q
            xp, xt = xt, xn
        else:
            xt = xn
        beta, rst, t = beta_n, rs, tn
        ext = exchange(xt)
        assert res > 0


def _worker(rank, world, port, cfg, scale, maxit, restart, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, t, restarts, st = _sharded_alg3(rank, world, cfg, scale, maxit, restart, dist)
        q.put((rank, x, t, restarts, st))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,scale,restart", [(1, 1.0, True), (3, 0.01, True), (2, 0.125, False)])
def test_sharded_iteration_gloo_world2_matches_oracle(cfg, scale, restart):
    import oracle
    maxit = 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, scale, maxit, restart, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted([q.get(timeout=300) for _ in procs], key=lambda v: v[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x = np.concatenate([o[1] for o in out])
    assert out[0][2] == out[1][2] == maxit and out[0][3] == out[1][3]  # identical decisions on both ranks
    p = synth.config_problem(cfg, scale)
    o = oracle.solve(p.Q, p.b, tol=0.0, maxit=maxit, restart=restart)
    assert o.restart_iters == out[0][3]
    assert np.abs(x - o.x).max() / np.abs(o.x).max() <= 1e-10


def _blob_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    import paper_2407_03272_b200 as ajm
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blob = bytes([rank]) * ajm.AJM_SHARD_BLOB_BYTES
        q.put((rank, ajm.allgather_bytes(blob)))
    finally:
        dist.destroy_process_group()


def test_connection_records_allgather_gloo_world2():
    """ShardSolver's default exchange of the connection records (torch.distributed all-gather, the
    plumbing of bench.py --gpus N) delivers every rank's record to every rank in rank order."""
    import paper_2407_03272_b200 as ajm
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blob_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, blobs in out:
        assert [b[0] for b in blobs] == [0, 1]
        assert all(len(b) == ajm.AJM_SHARD_BLOB_BYTES for b in blobs)
