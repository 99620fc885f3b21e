"""CPU, multi-process (torch.distributed gloo, world 2 and 3): the host-side
schedule of the column-sharded LDLT — boustrophedon ownership (ldlt.cpp:22-35),
per-step publication of the pivot column by its owner, every rank deriving
R_i / B_i from the broadcast panel, owner-only L store, gather to rank 0 —
restated over the float model (oracle/mpfloat.py) exactly in the order
csrc/hk_api.cu:dist_ldlt issues it, must reproduce the serial factorisation bit
for bit, with every (i, j, k) update applied exactly once (test_ldlt.cpp:135-145)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mpfloat as F
from oracle import restate as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pack(vals):
    return [(v.s, v.m, v.e) for v in vals]


def _unpack(t):
    return [F.MPF(*x) if x[0] else F.ZERO for x in t]


def _worker(rank, world, port, beta, n, p, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    owner = R.assign_columns(n, world)
    mu = [R.moment_integer(beta, j) for j in range(2 * n - 1)]
    cols = {j: [F.from_int(mu[k + j], p) for k in range(j, n)] for j in range(n) if owner[j] == rank}
    updates, sent = 0, 0

    def publish(col):
        nonlocal sent
        obj = [_pack(cols[col])] if owner[col] == rank else [None]
        if owner[col] == rank:
            sent += len(cols[col])
        dist.broadcast_object_list(obj, src=owner[col])
        return _unpack(obj[0])

    def derive(panel):
        r = F.recip(panel[0], p)
        return r, [F.mul(panel[t], r, p) for t in range(1, len(panel))]

    panel = publish(0)
    r, B = derive(panel)
    Rs = [r]
    for i in range(n):
        for j in sorted(cols):
            if j < i + 1:
                continue
            for k in range(j, n):
                cols[j][k - j] = F.fms(cols[j][k - j], panel[j - i], B[k - i - 1], p)
                updates += 1
        if owner[i] == rank:
            cols[i][1:] = B  # L(:, i) in place
        if i + 1 < n:
            panel = publish(i + 1)
            r, B = derive(panel)
            Rs.append(r)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object({j: _pack(v) for j, v in cols.items()}, gathered, dst=0)
    tot = [None] * world if rank == 0 else None
    dist.gather_object((updates, sent), tot, dst=0)
    if rank == 0:
        allcols = {}
        for g in gathered:
            allcols.update({j: _unpack(v) for j, v in g.items()})
        out_q.put(([allcols[j][0] for j in range(n)], [allcols[j][1:] for j in range(n)], Rs, tot))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,beta,n,p", [(2, (1, 2), 12, 128), (3, (1, 1), 14, 96), (2, (1, 3), 9, 256)])
def test_sharded_schedule_bit_identical_to_serial(world, beta, n, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, beta, n, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    D, L, Rs, tot = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    mu = [R.moment_integer(beta, j) for j in range(2 * n - 1)]
    D0, L0, R0 = F.ldlt(mu, n, p)
    assert D == D0 and L == L0 and Rs == R0
    assert sum(u for u, _ in tot) == n * (n * n - 1) // 6  # every update exactly once
    assert sum(s for _, s in tot) == sum(n - j for j in range(n))  # each column published once
