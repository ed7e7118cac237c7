"""numpy/ctypes wrapper of liboracle.so — the plain-C restatement of the
reference CPU algorithm. TEST INFRASTRUCTURE ONLY: imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg, never by the product
package (paper_2310_03294_b200).

Also wraps the reference-built driver oracle/_ref/ref_driver (when present).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_DRIVER = HERE / "_ref" / "ref_driver"
# the same driver + unmodified reference sources compiled against the drop-in
# include/distattn/flashcore.hpp (the reference runtime on the B200 kernels)
DROPIN_DRIVER = HERE / "_ref" / "dropin_driver"

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_lib = None


def build() -> Path:
    """Compiles liboracle.so (gcc) when missing or stale."""
    src = HERE / "distattn_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < max(src.stat().st_mtime,
                                                      (HERE / "distattn_oracle.h").stat().st_mtime):
        subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.dao_make_inputs.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                      _d, _d, _d, _d]
        L.dao_schedule_build.argtypes = [C.c_int, C.c_int, _i32p, _i32p, _i64p, _i32p, _i64p]
        L.dao_block_attn_update.argtypes = [_d, C.c_int64, _d, _d, C.c_int64, C.c_int64, _d, _d, _d,
                                            C.c_int, C.c_double, C.c_int64, C.c_int64]
        L.dao_rescale.argtypes = [_d, _d, _d, _d, _d, _d, C.c_int64, C.c_int64, _d, _d, _d]
        L.dao_rescale.restype = None
        L.dao_finalize.argtypes = [_d, _d, _d, C.c_int64, C.c_int64, _d, _d]
        L.dao_backward_aux.argtypes = [_d, _d, C.c_int64, C.c_int64, _d]
        L.dao_backward_aux.restype = None
        L.dao_block_attn_backward.argtypes = [_d, C.c_int64, _d, _d, C.c_int64, C.c_int64, _d, _d,
                                              _d, C.c_int, C.c_double, C.c_int64, C.c_int64, _d, _d,
                                              _d]
        L.dao_dense_oracle.argtypes = [_d, _d, _d, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                       C.c_double, _d, _d]
        L.dao_dense_backward.argtypes = [_d, _d, _d, _d, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                         C.c_double, _d, _d, _d]
        L.dao_run_forward.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, _d, _d, _d, _d, _d,
                                      _i64p]
        L.dao_run_backward.argtypes = [C.c_int, C.c_int64, C.c_int64, _d, _d, _d, _d, _d, _d, _d,
                                       _d, _d, _i64p]
        L.dao_block_attn_backward_with_d.argtypes = [_d, C.c_int64, _d, _d, C.c_int64, C.c_int64,
                                                     _d, _d, _d, C.c_int, C.c_double, C.c_int64,
                                                     C.c_int64, _d, _d, _d]
        L.dao_run_backward_sched.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, _d, _d, _d,
                                             _d, _d, _d, _d, _d, _d, _i64p]
        L.dao_rng_next_u64.argtypes = [C.POINTER(C.c_uint64)]
        L.dao_rng_next_u64.restype = C.c_uint64
        L.dao_rng_next_unit.argtypes = [C.POINTER(C.c_uint64)]
        L.dao_rng_next_unit.restype = C.c_double
        L.dao_rng_fork.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.dao_rng_fork.restype = None
        L.dao_bf16_round.argtypes = [C.c_double]
        L.dao_bf16_round.restype = C.c_double
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _ok(rc, what):
    if rc != 0:
        raise OracleError(f"{what}: status {rc}")


# ---------------------------------------------------------------- RNG
class Rng:
    """numerics.hpp:140-174"""

    def __init__(self, seed: int):
        self._s = C.c_uint64(seed)

    def next_u64(self) -> int:
        return lib().dao_rng_next_u64(C.byref(self._s))

    def next_unit(self) -> float:
        return lib().dao_rng_next_unit(C.byref(self._s))

    def fork(self) -> "Rng":
        child = C.c_uint64(0)
        lib().dao_rng_fork(C.byref(self._s), C.byref(child))
        r = Rng(0)
        r._s = child
        return r


def make_inputs(seed: int, workers: int, n: int, d: int, heads: int, bf16: bool = True):
    """Parity inputs [H, N, D] float64 (see distattn_oracle.h)."""
    q, k, v, do = (np.empty((heads, n, d)) for _ in range(4))
    _ok(lib().dao_make_inputs(seed, workers, n, d, heads, 1 if bf16 else 0, q, k, v, do),
        "make_inputs")
    return q, k, v, do


_KINDS = {"ring": 0, "balanced": 1, "balanced_split": 4}


def schedule_flat(workers: int, kind: str):
    kind_i = _KINDS[kind]
    steps, nt, nm = C.c_int32(0), C.c_int64(0), C.c_int64(0)
    _ok(lib().dao_schedule_build(workers, kind_i, C.byref(steps), None, C.byref(nt), None,
                                 C.byref(nm)), "schedule")
    t = (C.c_int32 * (6 * nt.value))()
    m = (C.c_int32 * (4 * max(1, nm.value)))()
    _ok(lib().dao_schedule_build(workers, kind_i, C.byref(steps), t, C.byref(nt), m, C.byref(nm)),
        "schedule")
    return steps.value, [list(t[6 * i:6 * i + 6]) for i in range(nt.value)], \
        [list(m[4 * i:4 * i + 4]) for i in range(nm.value)]


# ---------------------------------------------------------------- flashcore
MASK = {"diagonal": 0, "full": 1, "empty": 2}


def block_attn_update(q, k, v, acc, mask: str, scale: float, blocks=(16, 16)):
    """flashcore.hpp:135-197; acc = (o, m, l) float64 or None (fresh). Returns a new acc."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    rq, d = q.shape
    if acc is None:
        o, m, l = np.zeros((rq, d)), np.full(rq, -np.inf), np.zeros(rq)
    else:
        o, m, l = (np.array(x, dtype=np.float64, copy=True) for x in acc)
    _ok(lib().dao_block_attn_update(q, rq, k, v, k.shape[0], d, o, m, l, MASK[mask], scale,
                                    blocks[0], blocks[1]), "block_attn_update")
    return o, m, l


def rescale(a, b):
    o, m, l = np.empty_like(a[0]), np.empty_like(a[1]), np.empty_like(a[2])
    lib().dao_rescale(*(np.ascontiguousarray(x) for x in (*a, *b)), a[0].shape[0], a[0].shape[1],
                      o, m, l)
    return o, m, l


def finalize(acc):
    o, m, l = (np.ascontiguousarray(x) for x in acc)
    out, lse = np.empty_like(o), np.empty_like(m)
    _ok(lib().dao_finalize(o, m, l, o.shape[0], o.shape[1], out, lse), "finalize")
    return out, lse


def block_attn_backward(q, k, v, out, lse, d_out, mask: str, scale: float, blocks=(16, 16)):
    q, k, v, out, lse, d_out = (np.ascontiguousarray(x, dtype=np.float64)
                                for x in (q, k, v, out, lse, d_out))
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _ok(lib().dao_block_attn_backward(q, q.shape[0], k, v, k.shape[0], q.shape[1], out, lse, d_out,
                                      MASK[mask], scale, blocks[0], blocks[1], dq, dk, dv),
        "block_attn_backward")
    return dq, dk, dv


def backward_aux(d_out, out):
    d_out, out = (np.ascontiguousarray(x, dtype=np.float64) for x in (d_out, out))
    dv = np.empty(out.shape[0])
    lib().dao_backward_aux(d_out, out, out.shape[0], out.shape[1], dv)
    return dv


def block_attn_backward_with_d(q, k, v, d_vec, lse, d_out, mask: str, scale: float,
                               blocks=(16, 16)):
    q, k, v, d_vec, lse, d_out = (np.ascontiguousarray(x, dtype=np.float64)
                                  for x in (q, k, v, d_vec, lse, d_out))
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _ok(lib().dao_block_attn_backward_with_d(q, q.shape[0], k, v, k.shape[0], q.shape[1], d_vec,
                                             lse, d_out, MASK[mask], scale, blocks[0], blocks[1],
                                             dq, dk, dv), "block_attn_backward_with_d")
    return dq, dk, dv


def dense_oracle(q, k, v, causal: bool, scale: float):
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    out, lse = np.empty((q.shape[0], v.shape[1])), np.empty(q.shape[0])
    _ok(lib().dao_dense_oracle(q, k, v, q.shape[0], k.shape[0], q.shape[1], int(causal), scale,
                               out, lse), "dense_oracle")
    return out, lse


def dense_backward(q, k, v, d_out, causal: bool, scale: float):
    q, k, v, d_out = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v, d_out))
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _ok(lib().dao_dense_backward(q, k, v, d_out, q.shape[0], k.shape[0], q.shape[1], int(causal),
                                 scale, dq, dk, dv), "dense_backward")
    return dq, dk, dv


# ---------------------------------------------------------------- runtime
def run_forward(q, k, v, workers: int, schedule: str):
    """Stepper run_forward over the whole sequence of ONE head ([N, D])."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    n, d = q.shape
    out, lse = np.empty((n, d)), np.empty(n)
    c = (C.c_int64 * 10)()
    _ok(lib().dao_run_forward(workers, _KINDS[schedule], n, d, q, k, v, out, lse, c),
        "run_forward")
    return out, lse, list(c)


def run_backward(q, k, v, out, lse, d_out, workers: int):
    q, k, v, out, lse, d_out = (np.ascontiguousarray(x, dtype=np.float64)
                                for x in (q, k, v, out, lse, d_out))
    n, d = q.shape
    dq, dk, dv = np.empty((n, d)), np.empty((n, d)), np.empty((n, d))
    c = (C.c_int64 * 10)()
    _ok(lib().dao_run_backward(workers, n, d, q, k, v, out, lse, d_out, dq, dk, dv, c),
        "run_backward")
    return dq, dk, dv, list(c)


def run_backward_sched(q, k, v, out, lse, d_out, workers: int, schedule: str):
    """Backward over the ring, balanced or balanced_split backward schedule
    (balanced / balanced_split: extensions; the task table of run_forward's
    schedule of that name plus a GradKV per direct task)."""
    q, k, v, out, lse, d_out = (np.ascontiguousarray(x, dtype=np.float64)
                                for x in (q, k, v, out, lse, d_out))
    n, d = q.shape
    dq, dk, dv = np.empty((n, d)), np.empty((n, d)), np.empty((n, d))
    c = (C.c_int64 * 10)()
    _ok(lib().dao_run_backward_sched(workers, _KINDS[schedule], n, d, q, k, v, out,
                                     lse, d_out, dq, dk, dv, c), "run_backward_sched")
    return dq, dk, dv, list(c)


# ---------------------------------------------------------------- reference build
def ref_available() -> bool:
    return REF_DRIVER.exists()


def ref_run(n: int, workers: int, heads: int, d: int, seed: int, schedule: str, bf16: bool,
            timeout: int = 600, driver: Path = REF_DRIVER, executor: str = "stepper"):
    """Runs the UNMODIFIED reference (oracle/_ref/ref_driver, or the drop-in
    build oracle/_ref/dropin_driver) and loads its outputs."""
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([str(driver), "run", str(n), str(workers), str(heads), str(d), str(seed),
                        schedule, td, "1" if bf16 else "0", executor], check=True, timeout=timeout)
        meta = json.loads(Path(td, "meta.json").read_text())
        arrs = {}
        for name in ("q", "k", "v", "d_out", "out", "lse", "dq", "dk", "dv"):
            a = np.fromfile(Path(td, f"{name}.bin"), dtype=np.float64)
            arrs[name] = a.reshape(heads, n) if name == "lse" else a.reshape(heads, n, d)
    return arrs, meta


def ref_time(n: int, workers: int, heads: int, d: int, schedule: str, threads: int,
             timeout: int = 900) -> dict:
    r = subprocess.run([str(REF_DRIVER), "time", str(n), str(workers), str(heads), str(d), schedule,
                        str(threads)], check=True, capture_output=True, text=True, timeout=timeout)
    return json.loads(r.stdout.strip().splitlines()[-1])


def ref_json(mode: str) -> dict:
    r = subprocess.run([str(REF_DRIVER), mode], check=True, capture_output=True, text=True,
                       timeout=120)
    return json.loads(r.stdout)
