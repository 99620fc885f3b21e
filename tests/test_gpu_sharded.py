"""GPU: the column-sharded (multi-GPU) LDLT path.  Only one GPU is available to
the tests, so (a) all ranks are emulated in one context on one device
(virtual mode: the broadcast / gather become device-to-device copies, the
sharded kernels and index maps are the real ones) and (b) a real NCCL
communicator of world size 1 exercises the ncclBroadcast / ncclSend / ncclRecv
calls.  Results must be bit-identical to the single-GPU path (every op is
correctly rounded), as the reference requires across worker counts
(ldlt.hpp:92-96, test_ldlt.cpp:147-154, acceptance.cpp:176-218)."""
import json
import os

import pytest

from tests.mpf_helpers import from_arr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def api():
    from paper_1810_01478_b200 import api as a

    return a


def results(ctx, mu, k):
    rec = ctx.compute(mu, k)
    return rec, from_arr(ctx.D()), from_arr(ctx.Linv()), from_arr(ctx.block())


@pytest.fixture(scope="module")
def single(api):
    out = {}
    for beta, n, L, k in [((1, 2), 40, 32, 8), ((1, 1), 50, 24, 8), ((1, 3), 24, 40, 12)]:
        mu, _ = api.build_hankel(beta, n, L)
        with api.Context(L) as ctx:
            out[(beta, n, L, k)] = (mu, results(ctx, mu, k))
    return out


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_virtual_sharded_bit_identical(api, single, world):
    for (beta, n, L, k), (mu, (r0, D0, X0, M0)) in single.items():
        with api.Context(L, world=world, virtual=True) as ctx:
            r1, D1, X1, M1 = results(ctx, mu, k)
        assert D1 == D0 and X1 == X0 and M1 == M0, (beta, n, world)
        assert r1.lambda_hi == r0.lambda_hi and r1.lambda_lo == r0.lambda_lo


def test_nccl_world1_bit_identical(api, single):
    nid = api.nccl_unique_id()
    (beta, n, L, k), (mu, (r0, D0, X0, M0)) = next(iter(single.items()))
    with api.Context(L, rank=0, world=1, nccl_id=nid) as ctx:
        r1, D1, X1, M1 = results(ctx, mu, k)
    assert D1 == D0 and X1 == X0 and M1 == M0


def test_virtual_sharded_c2_matches_model_digest(api):
    from tests.test_gpu_parity import digest

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "model_c2.json")))
    n, L, k = g["n"], g["p"] // 32, g["k"]
    mu, _ = api.build_hankel((1, 1), n, L)
    with api.Context(L, world=8, virtual=True) as ctx:
        ctx.compute(mu, k)
        assert digest(from_arr(ctx.D())) == g["D_sha256"]
        assert digest(from_arr(ctx.block())) == g["block_sha256"]


def test_virtual_sharded_precision_error(api):
    n, L = 16, 1
    mu, _ = api.build_hankel((1, 1), n, L)
    with api.Context(L) as ref:
        ref.load_moments(mu)
        with pytest.raises(api.PrecisionError):
            ref.decompose()
        want = ref.bad_column
    with api.Context(L, world=3, virtual=True) as ctx:
        ctx.load_moments(mu)
        with pytest.raises(api.PrecisionError):
            ctx.decompose()
        assert ctx.bad_column == want


@pytest.mark.parametrize("world,force_fix", [(1, "0"), (3, "0"), (3, "1")])
def test_virtual_sharded_tensor_core_path(api, single, world, force_fix, monkeypatch):
    """The sharded look-ahead schedule with the tensor-core bulk products forced
    (mode 2 of the product kernel + certified rounding; with force_fix every 7th
    item also through the exact fix-up), against the 1-GPU path."""
    monkeypatch.setenv("HK_TC", "1")
    monkeypatch.setenv("HK_TC_FORCE_FIX", force_fix)
    for (beta, n, L, k), (mu, (r0, D0, X0, M0)) in single.items():
        if L % 4:
            continue
        with api.Context(L, world=world, virtual=True) as ctx:
            r1, D1, X1, M1 = results(ctx, mu, k)
            # replay of the cached step graph gives the same factors
            r2, D2, _, _ = results(ctx, mu, k)
        assert D1 == D0 and X1 == X0 and M1 == M0, (beta, n, world)
        assert D2 == D0 and r2.lambda_hi == r0.lambda_hi


def test_nccl_world1_c2_digest(api):
    """Real NCCL communicator (world 1): the broadcasts are captured into the step graph."""
    from tests.test_gpu_parity import digest

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "model_c2.json")))
    n, L, k = g["n"], g["p"] // 32, g["k"]
    mu, _ = api.build_hankel((1, 1), n, L)
    with api.Context(L, rank=0, world=1, nccl_id=api.nccl_unique_id()) as ctx:
        for _ in range(2):
            ctx.compute(mu, k)
            assert digest(from_arr(ctx.D())) == g["D_sha256"]
            assert digest(from_arr(ctx.block())) == g["block_sha256"]


@pytest.mark.parametrize("world,kind", [(3, "blocks"), (4, "round_robin"), (2, "all_on_1")])
def test_virtual_sharded_any_owner_map(api, single, world, kind, monkeypatch):
    """decompose_parallel takes any ColumnAssignment (ldlt.cpp:355-395), on both
    product paths: bit-identical to the single-GPU factors."""
    for tc in ("0", "1"):
        monkeypatch.setenv("HK_TC", tc)
        for (beta, n, L, k), (mu, (r0, D0, X0, M0)) in single.items():
            if tc == "1" and L % 4:
                continue
            owner = {"blocks": [c * world // n for c in range(n)], "round_robin": [c % world for c in range(n)],
                     "all_on_1": [1] * n}[kind]
            with api.Context(L, world=world, virtual=True) as ctx:
                ctx.set_owner_map(owner)
                r1, D1, X1, M1 = results(ctx, mu, k)
            assert D1 == D0 and X1 == X0 and M1 == M0, (beta, n, world, kind, tc)


@pytest.mark.parametrize("beta,n,L,k,tc", [((1, 1), 300, 224, 8, "0"), ((1, 1), 300, 224, 12, "1"),
                                           ((1, 1), 290, 256, 16, "0")])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dist_inv", ["1", "0"])
def test_virtual_sharded_inverse_and_block_rows(api, beta, n, L, k, tc, world, dist_inv, monkeypatch):
    """L^-1 and the H^-1 block sharded by 128-row blocks (K5/K6: column and row
    broadcasts per step, per-rank subtrees of the pairwise tree finished on rank
    0) — with several row blocks per rank — give the single-GPU bits; so does
    the rank-0 schedule (HK_DIST_INV=0)."""
    monkeypatch.setenv("HK_TC", tc)
    monkeypatch.setenv("HK_DIST_INV", dist_inv)
    mu, _ = api.build_hankel(beta, n, L)
    with api.Context(L) as one:
        r0, D0, X0, M0 = results(one, mu, k)
    with api.Context(L, world=world, virtual=True) as ctx:
        r1, D1, X1, M1 = results(ctx, mu, k)
    assert D1 == D0 and X1 == X0 and M1 == M0, (beta, n, world, tc, dist_inv)
    assert r1.lambda_hi == r0.lambda_hi and r1.lambda_lo == r0.lambda_lo
