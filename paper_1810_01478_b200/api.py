"""ctypes binding of the C ABI (include/hankel_b200.h) — Python plumbing for the
tests and bench.py.  The product is libhankel_b200.so (CUDA sm_100a + C++ host
code); this module only marshals host arrays.  There is no CPU fallback: if the
library is missing or no CUDA device is visible, calls raise.

Mirrors the reference entry points (proj/include/hankel/*.hpp) by name:
``build_hankel`` (moments), ``decompose`` (LDLT), ``invert_L_partial``,
``assemble_truncated_inverse``, ``smallest_eigs_of_H`` and ``compute``.
Errors map like the reference's exceptions: HK_ERR_PRECISION ->
PrecisionError (hankel::precision_error), HK_ERR_INVALID -> ValueError
(std::invalid_argument), HK_ERR_RUNTIME -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HK_LIB_PATH") or os.path.join(_HERE, "libhankel_b200.so")  # override: dev A/B builds

HK_OK, HK_ERR_RUNTIME, HK_ERR_PRECISION, HK_ERR_INVALID = 0, 1, 2, 3
OP_FMS, OP_MUL, OP_ADD, OP_RECIP = 0, 1, 2, 3
OP_CTA = 16  # or-flag: CTA-cooperative kernels (critical-path variants)


class PrecisionError(RuntimeError):
    """hankel::precision_error (proj/include/hankel/errors.hpp:10-13)."""


_lib = None


def lib():
    """Load libhankel_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        u32p, i32p, f64p = C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_double)
        vp = C.c_void_p
        sig = {
            "hk_version": (C.c_int, []),
            "hk_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(vp)]),
            "hk_destroy": (None, [vp]),
            "hk_last_error": (C.c_char_p, [vp]),
            "hk_bad_column": (C.c_int, [vp]),
            "hk_limbs": (C.c_int, [vp]),
            "hk_moments": (C.c_int, [C.c_uint, C.c_uint, C.c_int, C.c_int, u32p, i32p, i32p, C.POINTER(C.c_int)]),
            "hk_load_moments": (C.c_int, [vp, C.c_int, u32p, i32p, i32p]),
            "hk_generate_moments": (C.c_int, [vp, C.c_uint, C.c_uint, C.c_int, C.POINTER(C.c_int)]),
            "hk_get_moments": (C.c_int, [vp, u32p, i32p, i32p]),
            "hk_compute_generated": (C.c_int, [vp, C.c_uint, C.c_uint, C.c_int, C.c_int, f64p, f64p, f64p,
                                               C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "hk_ldlt": (C.c_int, [vp]),
            "hk_ldlt_invert": (C.c_int, [vp, C.c_int]),
            "hk_get_D": (C.c_int, [vp, u32p, i32p, i32p]),
            "hk_get_L_column": (C.c_int, [vp, C.c_int, u32p, i32p, i32p]),
            "hk_invert_L_partial": (C.c_int, [vp, C.c_int]),
            "hk_get_Linv": (C.c_int, [vp, u32p, i32p, i32p]),
            "hk_assemble_block": (C.c_int, [vp, C.c_int]),
            "hk_get_block": (C.c_int, [vp, u32p, i32p, i32p]),
            "hk_smallest_eigs": (C.c_int, [vp, C.c_int, f64p, f64p, f64p]),
            "hk_compute": (C.c_int, [vp, C.c_int, u32p, i32p, i32p, C.c_int, f64p, f64p, f64p, C.POINTER(C.c_int)]),
            "hk_timings": (C.c_int, [vp, f64p]),
            "hk_launch_count": (C.c_longlong, [vp]),
            "hk_mp_batch": (C.c_int, [vp, C.c_int, C.c_longlong] + [u32p, i32p, i32p] * 4),
            "hk_assign_columns": (C.c_int, [C.c_int, C.c_int, i32p]),
            "hk_stream": (vp, [vp]),
            "hk_profile_ldlt": (C.c_int, [vp, f64p, C.POINTER(C.c_longlong)]),
            "hk_peak_imad": (C.c_int, [C.c_int, f64p]),
            "hk_peak_i8mma": (C.c_int, [C.c_int, f64p]),
            "hk_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "hk_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]),
            "hk_world": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "hk_set_limbs": (C.c_int, [vp, C.c_int]),
            "hk_set_owner_map": (C.c_int, [vp, C.c_int, i32p]),
            "hk_set_kernel_timing": (C.c_int, [vp, C.c_int]),
            "hk_kernel_times": (C.c_int, [vp, f64p]),
            "hk_fused_violations": (C.c_int, [vp, C.POINTER(C.c_longlong)]),
            "hk_fix_count": (C.c_int, [vp, C.POINTER(C.c_longlong)]),
            "hk_kernel_step_times": (C.c_int, [vp, f64p, C.c_int, C.POINTER(C.c_int)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _u32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class MPArray:
    """Host SoA array of p-bit floats (the ABI interchange format)."""

    limbs: np.ndarray  # uint32 [count, L]
    exps: np.ndarray  # int32 [count]
    signs: np.ndarray  # int32 [count]

    @staticmethod
    def empty(count: int, L: int) -> "MPArray":
        return MPArray(np.zeros((count, L), np.uint32), np.zeros(count, np.int32), np.zeros(count, np.int32))

    @property
    def L(self) -> int:
        return self.limbs.shape[1]

    def __len__(self):
        return self.limbs.shape[0]

    def entry(self, i: int):
        """(sign, mantissa int, exp) of entry i."""
        m = int.from_bytes(self.limbs[i].astype("<u4").tobytes(), "little")
        return int(self.signs[i]), m, int(self.exps[i])

    def set_entry(self, i: int, sign: int, m: int, e: int):
        self.limbs[i] = np.frombuffer(m.to_bytes(4 * self.L, "little"), dtype="<u4")
        self.exps[i] = e
        self.signs[i] = sign

    def to_fraction(self, i: int):
        from fractions import Fraction

        s, m, e = self.entry(i)
        if s == 0:
            return Fraction(0)
        sh = e - 32 * self.L
        v = Fraction(m << sh) if sh >= 0 else Fraction(m, 1 << (-sh))
        return v if s > 0 else -v

    def ptrs(self):
        return _u32(self.limbs), _i32(self.exps), _i32(self.signs)


def _check(rc: int, ctx=None):
    if rc == HK_OK:
        return
    msg = lib().hk_last_error(ctx).decode() if ctx else f"status {rc}"
    if rc == HK_ERR_PRECISION:
        raise PrecisionError(msg)
    if rc == HK_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg)


def build_hankel(beta: tuple[int, int], n: int, limbs: int, out: MPArray | None = None) -> tuple[MPArray, bool]:
    """The 2n-1 exact moments as p-bit floats (moments.cpp:102-133 / build_hankel),
    written into `out` when given (e.g. pinned host arrays)."""
    if out is None:
        out = MPArray.empty(2 * n - 1, limbs)
    elif len(out) != 2 * n - 1 or out.L != limbs:
        raise ValueError("build_hankel: `out` has the wrong shape")
    exact = C.c_int(0)
    _check(lib().hk_moments(beta[0], beta[1], 2 * n - 1, limbs, *out.ptrs(), C.byref(exact)))
    return out, bool(exact.value)


def peak_imad(device: int = 0) -> float:
    """Measured IMAD.WIDE limb-MAC/s of the device (roofline denominator)."""
    v = C.c_double()
    rc = lib().hk_peak_imad(device, C.byref(v))
    if rc != HK_OK:
        raise RuntimeError(f"hk_peak_imad failed ({rc})")
    return v.value


def peak_i8mma(device: int = 0) -> float:
    """Measured int8 tensor-core u8-MAC/s of the device (tcgen05 kind::i8; roofline denominator)."""
    v = C.c_double()
    rc = lib().hk_peak_i8mma(device, C.byref(v))
    if rc != HK_OK:
        raise RuntimeError(f"hk_peak_i8mma failed ({rc})")
    return v.value


def assign_columns(n: int, workers: int) -> list[int]:
    o = np.zeros(n, np.int32)
    rc = lib().hk_assign_columns(n, workers, _i32(o))
    if rc != HK_OK:
        raise ValueError("assign_columns: need n >= 1 and workers >= 1")
    return o.tolist()


@dataclass
class RunRecord:
    """pipeline.hpp:28-48 (numeric + timing fields)."""

    n: int
    k: int
    lambda_: list = field(default_factory=list)  # ~32-digit values (hi + lo as Fraction-free float pairs)
    lambda_hi: list = field(default_factory=list)
    lambda_lo: list = field(default_factory=list)
    trunc_err: list = field(default_factory=list)
    wall_s: float = 0.0
    ldlt_s: float = 0.0
    invL_s: float = 0.0
    invH_s: float = 0.0
    eigen_s: float = 0.0
    h2d_s: float = 0.0
    d2h_s: float = 0.0


def nccl_unique_id() -> bytes:
    """ncclUniqueId (128 bytes) for hk_create_sharded; make it on rank 0 and share it."""
    buf = C.create_string_buffer(128)
    if lib().hk_nccl_unique_id(buf) != HK_OK:
        raise RuntimeError("hk_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


class Context:
    """One device context at p = 32*limbs bits (hk_create / hk_destroy).

    world > 1 (or virtual=True) selects the column-sharded LDLT
    (hk_create_sharded): with `nccl_id` one process per GPU over NCCL, with
    virtual=True all `world` ranks emulated on this one device."""

    def __init__(self, limbs: int, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 virtual: bool = False):
        self.L = limbs
        h = C.c_void_p()
        if world > 1 or virtual or nccl_id is not None:
            if nccl_id is None and not virtual:
                raise ValueError("world > 1 needs an nccl_id (or virtual=True)")
            rc = lib().hk_create_sharded(device, limbs, rank, world, nccl_id, C.byref(h))
        else:
            rc = lib().hk_create(device, limbs, C.byref(h))
        if rc != HK_OK:
            raise RuntimeError(f"hk_create failed with status {rc} (CUDA device {device} unavailable?)")
        self.h = h
        self.n = 0
        self.rank, self.world = rank, world

    def close(self):
        if self.h:
            lib().hk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- stages
    def load_moments(self, mu: MPArray):
        n = (len(mu) + 1) // 2
        _check(lib().hk_load_moments(self.h, n, *mu.ptrs()), self.h)
        self.n = n

    def decompose(self):
        """decompose_parallel / decompose_serial (ldlt.hpp:90-99)."""
        rc = lib().hk_ldlt(self.h)
        if rc == HK_ERR_PRECISION:
            self.bad_column = lib().hk_bad_column(self.h)
        _check(rc, self.h)

    def D(self) -> MPArray:
        out = MPArray.empty(self.n, self.L)
        _check(lib().hk_get_D(self.h, *out.ptrs()), self.h)
        return out

    def L_column(self, col: int) -> MPArray:
        out = MPArray.empty(max(self.n - col - 1, 0), self.L)
        if len(out) == 0:
            _check(lib().hk_get_L_column(self.h, col, None, None, None), self.h)
            return out
        _check(lib().hk_get_L_column(self.h, col, *out.ptrs()), self.h)
        return out

    def invert_L_partial(self, m: int):
        _check(lib().hk_invert_L_partial(self.h, m), self.h)
        self.m = m

    def decompose_invert(self, m: int):
        """decompose + invert_L_partial(m) as compute() runs them (hk_ldlt_invert: L^-1 steps
        interleaved with the factorisation where both are latency-bound; same bits)."""
        self.m = m
        rc = lib().hk_ldlt_invert(self.h, m)
        if rc == HK_ERR_PRECISION:
            self.bad_column = lib().hk_bad_column(self.h)
        _check(rc, self.h)

    def Linv(self) -> MPArray:
        out = MPArray.empty(self.n * self.m, self.L)
        _check(lib().hk_get_Linv(self.h, *out.ptrs()), self.h)
        return out

    def assemble_truncated_inverse(self, k: int):
        _check(lib().hk_assemble_block(self.h, k), self.h)
        self.k = k

    def block(self) -> MPArray:
        out = MPArray.empty(self.k * self.k, self.L)
        _check(lib().hk_get_block(self.h, *out.ptrs()), self.h)
        return out

    def smallest_eigs_of_H(self, s: int):
        hi, lo, te = (np.zeros(s) for _ in range(3))
        f64 = C.POINTER(C.c_double)
        _check(lib().hk_smallest_eigs(self.h, s, hi.ctypes.data_as(f64), lo.ctypes.data_as(f64),
                                      te.ctypes.data_as(f64)), self.h)
        return hi.tolist(), lo.tolist(), te.tolist()

    def compute(self, mu: MPArray, k: int) -> RunRecord:
        """hankel::compute (pipeline.cpp:26-72) from host moments."""
        n = (len(mu) + 1) // 2
        hi, lo, te = (np.zeros(3) for _ in range(3))
        s = C.c_int(0)
        f64 = C.POINTER(C.c_double)
        rc = lib().hk_compute(self.h, n, *mu.ptrs(), k, hi.ctypes.data_as(f64), lo.ctypes.data_as(f64),
                              te.ctypes.data_as(f64), C.byref(s))
        if rc == HK_ERR_PRECISION:
            self.bad_column = lib().hk_bad_column(self.h)
        _check(rc, self.h)
        self.n, self.m, self.k = n, min(k, n), min(k, n)
        t = self.timings()
        ns = s.value
        return RunRecord(n=n, k=min(k, n), lambda_hi=hi[:ns].tolist(), lambda_lo=lo[:ns].tolist(),
                         trunc_err=te[:ns].tolist(), wall_s=t[0], ldlt_s=t[1], invL_s=t[2], invH_s=t[3],
                         eigen_s=t[4], h2d_s=t[5], d2h_s=t[6])

    def generate_moments(self, beta: tuple[int, int], n: int) -> bool:
        """build_hankel on the device (even 2/beta): the context's moments of order n; returns `exact`."""
        exact = C.c_int(0)
        _check(lib().hk_generate_moments(self.h, beta[0], beta[1], n, C.byref(exact)), self.h)
        self.n = n
        return bool(exact.value)

    def moments(self) -> MPArray:
        """The context's 2n-1 moments copied back (tests)."""
        out = MPArray.empty(2 * self.n - 1, self.L)
        _check(lib().hk_get_moments(self.h, *out.ptrs()), self.h)
        return out

    def compute_generated(self, beta: tuple[int, int], n: int, k: int) -> RunRecord:
        """hankel::compute (pipeline.cpp:26-72) with the moments generated on the device."""
        hi, lo, te = (np.zeros(3) for _ in range(3))
        s, ex = C.c_int(0), C.c_int(0)
        f64 = C.POINTER(C.c_double)
        rc = lib().hk_compute_generated(self.h, beta[0], beta[1], n, k, hi.ctypes.data_as(f64),
                                        lo.ctypes.data_as(f64), te.ctypes.data_as(f64), C.byref(s), C.byref(ex))
        if rc == HK_ERR_PRECISION:
            self.bad_column = lib().hk_bad_column(self.h)
        _check(rc, self.h)
        self.n, self.m, self.k = n, min(k, n), min(k, n)
        self.moments_exact = bool(ex.value)
        t = self.timings()
        ns = s.value
        return RunRecord(n=n, k=min(k, n), lambda_hi=hi[:ns].tolist(), lambda_lo=lo[:ns].tolist(),
                         trunc_err=te[:ns].tolist(), wall_s=t[0], ldlt_s=t[1], invL_s=t[2], invH_s=t[3],
                         eigen_s=t[4], h2d_s=t[5], d2h_s=t[6])

    def timings(self):
        t = np.zeros(7)
        lib().hk_timings(self.h, t.ctypes.data_as(C.POINTER(C.c_double)))
        return t.tolist()

    def stream_ptr(self) -> int:
        """cudaStream_t of the context (for torch.cuda.ExternalStream)."""
        return int(lib().hk_stream(self.h) or 0)

    def profile_ldlt(self):
        """Eager instrumented LDLT: ({stage: summed ms}, number of trailing steps).  On the
        tensor-core path `tc_products` + `tc_round` split `trailing`."""
        ms = np.zeros(7)
        n = C.c_longlong()
        _check(lib().hk_profile_ldlt(self.h, ms.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)), self.h)
        keys = ("trailing", "recip", "mulB", "storeL", "total", "tc_products", "tc_round")
        return dict(zip(keys, ms.tolist())), n.value

    def set_limbs(self, limbs: int):
        """New precision on the same device / communicator (hk_set_limbs)."""
        _check(lib().hk_set_limbs(self.h, limbs), self.h)
        self.L = limbs

    def set_owner_map(self, owner):
        """Column -> rank map of the sharded LDLT (any ColumnAssignment, ldlt.hpp:13-21)."""
        o = np.asarray(owner, dtype=np.int32)
        _check(lib().hk_set_owner_map(self.h, len(o), _i32(o)), self.h)

    def set_kernel_timing(self, on: bool = True):
        _check(lib().hk_set_kernel_timing(self.h, 1 if on else 0), self.h)

    def kernel_times(self) -> dict:
        """hk_kernel_times of the last LDLT: summed device ms of the product kernels, the rounding
        pass, timed steps, the pivot-column broadcasts (sharded) and their count, LDLT ms."""
        t = np.zeros(6)
        _check(lib().hk_kernel_times(self.h, t.ctypes.data_as(C.POINTER(C.c_double))), self.h)
        keys = ("products_ms", "round_ms", "steps", "comm_ms", "comm_steps", "ldlt_ms")
        return dict(zip(keys, t.tolist()))

    def kernel_step_times(self):
        """Per LDLT step (with kernel timing on): [(product ms, rounding ms), ...] of the last hk_ldlt."""
        cap = max(self.n, 1)
        buf = np.zeros(2 * cap)
        cnt = C.c_int(0)
        _check(lib().hk_kernel_step_times(self.h, buf.ctypes.data_as(C.POINTER(C.c_double)), cap, C.byref(cnt)),
               self.h)
        return [(buf[2 * s], buf[2 * s + 1]) for s in range(cnt.value)]

    def fix_count(self) -> int:
        """Items left to the exact redo by the certified roundings so far (hk_fix_count)."""
        v = C.c_longlong()
        _check(lib().hk_fix_count(self.h, C.byref(v)), self.h)
        return v.value

    def fused_violations(self) -> int:
        v = C.c_longlong()
        _check(lib().hk_fused_violations(self.h, C.byref(v)), self.h)
        return v.value

    def launch_count(self) -> int:
        return int(lib().hk_launch_count(self.h))

    def mp_batch(self, op: int, a: MPArray, b: MPArray | None = None, c: MPArray | None = None) -> MPArray:
        out = MPArray.empty(len(a), self.L)
        nul = (None, None, None)
        _check(lib().hk_mp_batch(self.h, op, len(a), *a.ptrs(), *(b.ptrs() if b is not None else nul),
                                 *(c.ptrs() if c is not None else nul), *out.ptrs()), self.h)
        return out
