"""GPU: host-API behaviour around the path — graph-resident kernel timing,
re-use of one context across precisions (hk_set_limbs, as auto_precision /
scan do, pipeline.cpp:74-122), and the multi-GPU group with >= 2 real NCCL
ranks when the box has them (the reference's worker-count determinism,
acceptance.cpp:176-218)."""
import os
import socket

import pytest

from tests.mpf_helpers import from_arr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1810_01478_b200 import api as a

    return a


def run(ctx, mu, k):
    rec = ctx.compute(mu, k)
    return rec, from_arr(ctx.D()), from_arr(ctx.block())


def test_dataflow_ldlt_same_bits_as_step_graph(api, monkeypatch):
    """Small p: the one-kernel dataflow LDLT (k_ldlt_flow, the default below the tensor-core
    threshold) against the N-step look-ahead graph: every pivot, every column of L, the block
    and lambda bit for bit; it reports no per-step kernel times."""
    for beta, n, L, k, threads in [((1, 2), 64, 96, 8, None), ((1, 1), 97, 40, 8, "64"), ((1, 3), 33, 100, 12, "256"),
                                   ((1, 1), 120, 96, 16, None)]:
        if threads:
            monkeypatch.setenv("HK_LDLT_FLOW_THREADS", threads)
        else:
            monkeypatch.delenv("HK_LDLT_FLOW_THREADS", raising=False)
        mu, exact = api.build_hankel(beta, n, L)
        assert exact
        got = {}
        for flow in ("0", "1"):
            monkeypatch.setenv("HK_LDLT_FLOW", flow)
            with api.Context(L) as ctx:
                ctx.set_kernel_timing(True)
                rec, D, M = run(ctx, mu, k)
                cols = [from_arr(ctx.L_column(j)) for j in range(n - 1)]
                steps = ctx.kernel_times()["steps"]
                rec2, D2, M2 = run(ctx, mu, k)  # replay on the same context
                assert D2 == D and M2 == M
            got[flow] = (rec.lambda_hi, rec.lambda_lo, D, M, cols)
            assert steps == (0 if flow == "1" else n - 2)
        assert got["0"] == got["1"]


@pytest.mark.parametrize("beta,n,L,k,tc", [((1, 1), 70, 160, 8, "1"), ((1, 2), 90, 200, 16, "1"), ((1, 2), 48, 8, 8, "0"),
                                           ((1, 3), 40, 104, 12, "0"), ((1, 1), 3, 8, 3, "0"), ((1, 2), 1, 4, 1, "0")])
def test_inverse_steps_interleaved_with_ldlt_same_bits(api, beta, n, L, k, tc, monkeypatch):
    """hk_ldlt_invert: the L^-1 row-elimination steps riding in the LDLT graph (one GPU, small
    p) against the two separate passes (HK_INV_OVERLAP=0, and the plain decompose +
    invert_L_partial calls): pivots, L^-1, block and lambda bit for bit; replays; both stage
    times reported."""
    monkeypatch.setenv("HK_TC", tc)
    monkeypatch.setenv("HK_LDLT_FLOW", "0")  # the graph LDLT (the dataflow kernel has no steps to ride on)
    mu, _ = api.build_hankel(beta, n, L)
    kk = min(k, n)
    got = []
    for mode in ("overlap", "apart", "calls"):
        monkeypatch.setenv("HK_INV_OVERLAP", "0" if mode == "apart" else "1")
        with api.Context(L) as ctx:
            for rep in range(2):
                ctx.load_moments(mu)
                if mode == "calls":
                    ctx.decompose()
                    ctx.invert_L_partial(kk)
                else:
                    ctx.decompose_invert(kk)
                ctx.assemble_truncated_inverse(kk)
                lam = ctx.smallest_eigs_of_H(min(3, kk))
                cur = (from_arr(ctx.D()), from_arr(ctx.Linv()), from_arr(ctx.block()), repr(lam))  # (trunc_err may hold NaN)
                t = ctx.timings()
                assert t[1] > 0 and t[2] >= 0
                if rep:
                    assert cur == first
                first = cur
            rec = ctx.compute(mu, k)  # compute() goes through the same call
            assert rec.lambda_hi == list(lam[0])
        got.append(cur)
    assert got[0][0] == got[1][0] == got[2][0]
    # X entries (r, c >= min(r, m)) are zeros in every schedule; all must agree
    assert got[0][1] == got[1][1] == got[2][1]
    assert got[0][2] == got[1][2] == got[2][2]
    assert got[0][3] == got[1][3] == got[2][3]


@pytest.mark.parametrize("beta,n,L,k", [((1, 1), 150, 192, 8), ((1, 3), 96, 1152, 12), ((1, 2), 300, 392, 16)])
def test_tensor_core_inverse_steps_in_ldlt_graph_with_forced_redo(api, beta, n, L, k, monkeypatch):
    """The tensor-core L^-1 steps riding in the (fused, tensor-core) LDLT graph keep their own A
    operand, redo list and counters: with every 7th item of both stages forced to the exact
    redo (HK_TC_FORCE_FIX) the two lists are in use at the same time, and the bits must equal
    the two separate passes'."""
    monkeypatch.setenv("HK_TC", "1")
    monkeypatch.setenv("HK_LDLT_FLOW", "0")
    mu, _ = api.build_hankel(beta, n, L)
    got = {}
    for force in ("0", "1"):
        for overlap in ("1", "0"):
            monkeypatch.setenv("HK_TC_FORCE_FIX", force)
            monkeypatch.setenv("HK_INV_OVERLAP", overlap)
            with api.Context(L) as ctx:
                rec, D, M = run(ctx, mu, k)
                X = from_arr(ctx.Linv())
                rec2, D2, M2 = run(ctx, mu, k)
                assert D2 == D and M2 == M and from_arr(ctx.Linv()) == X
                assert ctx.fused_violations() == 0
            got[(force, overlap)] = (rec.lambda_hi, rec.lambda_lo, D, X, M)
    assert got[("0", "1")] == got[("0", "0")] == got[("1", "1")] == got[("1", "0")]


@pytest.mark.parametrize("beta,n,L,tc", [((1, 1), 60, 136, "1"), ((1, 2), 50, 16, "0")])
def test_one_context_many_k_and_n(api, beta, n, L, tc, monkeypatch):
    """One context, compute() with changing k and n (the cached graphs are keyed by (n, m); the
    buffers of the interleaved L^-1 steps grow): every result equals a fresh context's."""
    monkeypatch.setenv("HK_TC", tc)
    monkeypatch.setenv("HK_LDLT_FLOW", "0")
    cases = [(n, 4), (n, 9), (n - 7, 9), (n, 4), (n + 5, 12), (n, 9)]

    def result(ctx, mu, k):
        rec, D, M = run(ctx, mu, k)
        return repr((rec.lambda_hi, rec.lambda_lo, rec.trunc_err)), D, M, from_arr(ctx.Linv())

    want = {}
    for nn, k in set(cases):
        mu, _ = api.build_hankel(beta, nn, L)
        with api.Context(L) as ctx:
            want[(nn, k)] = result(ctx, mu, k)
    with api.Context(L) as ctx:
        for nn, k in cases:
            mu, _ = api.build_hankel(beta, nn, L)
            assert result(ctx, mu, k) == want[(nn, k)], (nn, k)


def test_interleaved_inverse_stops_on_a_failed_pivot(api, monkeypatch):
    monkeypatch.setenv("HK_LDLT_FLOW", "0")
    n, L = 16, 1
    mu, _ = api.build_hankel((1, 1), n, L)
    with api.Context(L) as ctx:
        ctx.load_moments(mu)
        with pytest.raises(api.PrecisionError):
            ctx.decompose_invert(4)
        col = ctx.bad_column
        with pytest.raises(ValueError):
            ctx.Linv()  # not inverted
        monkeypatch.setenv("HK_INV_OVERLAP", "0")
        ctx.load_moments(mu)
        with pytest.raises(api.PrecisionError):
            ctx.decompose_invert(4)
        assert ctx.bad_column == col


@pytest.mark.parametrize("beta,n,L,k,tc", [((1, 2), 48, 8, 8, "0"), ((1, 1), 40, 192, 8, "1")])
def test_kernel_timing_nodes_do_not_change_results(api, beta, n, L, k, tc, monkeypatch):
    monkeypatch.setenv("HK_TC", tc)
    monkeypatch.setenv("HK_LDLT_FLOW", "0")  # the timing nodes belong to the N-step graph
    mu, _ = api.build_hankel(beta, n, L)
    with api.Context(L) as ctx:
        r0, D0, M0 = run(ctx, mu, k)
        ctx.set_kernel_timing(True)
        r1, D1, M1 = run(ctx, mu, k)
        kt = ctx.kernel_times()
    assert D1 == D0 and M1 == M0 and r1.lambda_hi == r0.lambda_hi
    assert kt["steps"] == n - 2  # one timed bulk launch per step with columns >= i+2
    assert kt["products_ms"] > 0 and kt["round_ms"] >= 0
    assert kt["products_ms"] + kt["round_ms"] <= kt["ldlt_ms"] * 1.05


def test_set_limbs_reuses_context(api):
    beta, n, k = (1, 2), 40, 8
    mu1, _ = api.build_hankel(beta, n, 24)
    mu2, _ = api.build_hankel(beta, n, 40)
    with api.Context(40) as fresh:
        want = run(fresh, mu2, k)
    with api.Context(24) as ctx:
        run(ctx, mu1, k)
        ctx.set_limbs(40)
        got = run(ctx, mu2, k)
        ctx.set_limbs(40)  # no-op
        again = run(ctx, mu2, k)
    assert got[1] == want[1] and got[2] == want[2] and again[1] == want[1]


def test_set_limbs_sharded_keeps_communicator(api):
    """auto_precision on a sharded context: one ncclUniqueId, several precisions."""
    beta, n, k = (1, 2), 30, 8
    nid = api.nccl_unique_id()
    with api.Context(16, rank=0, world=1, nccl_id=nid) as ctx:
        for L in (16, 24, 16):
            mu, _ = api.build_hankel(beta, n, L)
            ctx.set_limbs(L)
            got = run(ctx, mu, k)
            with api.Context(L) as one:
                want = run(one, mu, k)
            assert got[1] == want[1] and got[2] == want[2] and got[0].lambda_hi == want[0].lambda_hi
        kt = ctx.kernel_times()
        assert kt["comm_steps"] == n and kt["comm_ms"] >= 0


def _rank_main(rank, world, port, beta, n, L, k, q):
    import torch
    import torch.distributed as dist

    from paper_1810_01478_b200 import api as a

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    obj = [a.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    mu, _ = a.build_hankel(beta, n, L)
    with a.Context(L, device=rank, rank=rank, world=world, nccl_id=obj[0]) as ctx:
        rec = ctx.compute(mu, k)
        out = (rec.lambda_hi, rec.lambda_lo)
        if rank == 0:
            out = out + (from_arr(ctx.D()), from_arr(ctx.block()))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_real_nccl_ranks_bit_identical(api, world):
    """>= 2 real NCCL ranks (one process per GPU) give the 1-GPU factors, block
    and lambdas bit for bit, and every rank returns rank 0's lambdas."""
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    beta, n, L, k = (1, 2), 96, 192, 16
    mu, _ = api.build_hankel(beta, n, L)
    with api.Context(L) as one:
        want = run(one, mu, k)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, beta, n, L, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert res[0][2] == want[1] and res[0][3] == want[2]
    for r in range(world):
        assert res[r][0] == want[0].lambda_hi and res[r][1] == want[0].lambda_lo


@pytest.mark.parametrize("beta,n,L,k", [((1, 1), 256, 192, 8), ((1, 3), 96, 1152, 12), ((1, 2), 48, 8, 8)])
def test_fused_rounding_bit_identical_to_rounding_pass(api, beta, n, L, k, monkeypatch):
    """The certified rounding fused into the product kernel (tc_fused.cuh) gives
    the same factors as the separate rounding pass, its exponent prediction
    never fails the normalisation check, and with every 7th item forced to the
    exact redo the bits do not change either."""
    monkeypatch.setenv("HK_TC", "1")
    mu, _ = api.build_hankel(beta, n, L)
    out = {}
    for fuse, force in (("0", "0"), ("1", "0"), ("1", "1")):
        monkeypatch.setenv("HK_TC_FUSE", fuse)
        monkeypatch.setenv("HK_TC_FORCE_FIX", force)
        with api.Context(L) as ctx:
            out[(fuse, force)] = run(ctx, mu, k)
            assert ctx.fused_violations() == 0
    base = out[("0", "0")]
    for key in (("1", "0"), ("1", "1")):
        assert out[key][1] == base[1] and out[key][2] == base[2], key
        assert out[key][0].lambda_hi == base[0].lambda_hi


def _same(a, b):
    import numpy as np

    return (np.array_equal(a.limbs, b.limbs) and np.array_equal(a.exps, b.exps) and np.array_equal(a.signs, b.signs))


# moments generated on the device (csrc/moments_dev.cuh) against the
# host generator (itself checked against the reference's integers, test_abi.py):
# every BASELINE weight, exact (p > bits) and rounded (p < bits, RNE incl. sticky
# and carry), one thread per limb and several limbs per thread
@pytest.mark.parametrize("beta,n,L", [
    ((1, 2), 64, 96),      # C1
    ((1, 1), 256, 192),    # C2
    ((1, 3), 512, 1152),   # C3
    ((1, 2), 1024, 1536),  # C4
    ((1, 2), 2048, 3584),  # C5 (several limbs per thread)
    ((1, 1), 1, 4), ((1, 2), 2, 1), ((1, 4), 9, 3),
    ((1, 2), 300, 8),      # rounded: 256 bits of a ~9000-bit integer
    ((1, 1), 700, 31),     # rounded
    ((1, 3), 150, 40),     # rounded, 3 factor pairs per moment
    ((1, 1), 33000, 1),    # factors past 65535 (multiplied one at a time), a ~1 Mbit integer in shared memory
])
def test_device_moments_bit_identical_to_host(api, beta, n, L):
    want, ex_h = api.build_hankel(beta, n, L)
    with api.Context(L) as ctx:
        ex_d = ctx.generate_moments(beta, n)
        got = ctx.moments()
    assert ex_d == ex_h
    assert _same(got, want)


def test_device_moments_compute_matches_host_path(api):
    beta, n, L, k = (1, 2), 48, 48, 8
    mu, exact = api.build_hankel(beta, n, L)
    with api.Context(L) as ctx:
        r0, D0, M0 = run(ctx, mu, k)
        r1 = ctx.compute_generated(beta, n, k)
        D1, M1 = from_arr(ctx.D()), from_arr(ctx.block())
        assert exact and ctx.moments_exact
    assert D1 == D0 and M1 == M0 and r1.lambda_hi == r0.lambda_hi and r1.lambda_lo == r0.lambda_lo


def test_device_moments_odd_q_is_host_only(api):
    with api.Context(8) as ctx:
        with pytest.raises(ValueError):
            ctx.generate_moments((2, 1), 8)  # beta = 2: half-integer Gamma needs sqrt(pi)
