"""ctypes wrapper of oracle/_ref/planner_oracle.so (plain-C restatement of the
reference planner path; TEST INFRASTRUCTURE ONLY - see planner_oracle.c)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "planner_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmimose_ref.so")
_lib = None

DISTS = {"uniform": 0, "normal": 1, "powerlaw": 2}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", HERE, "_ref/planner_oracle.so"], check=True,
                           capture_output=True)
        L = C.CDLL(LIB)
        i64p = C.POINTER(C.c_int64)
        L.orc_sample_workload.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                          C.c_double, C.c_int64, C.c_int64, C.c_uint64, i64p]
        L.orc_fit_layer.argtypes = [i64p, i64p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.orc_predict.restype = C.c_int64
        L.orc_predict.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int64]
        L.orc_generate_plan.argtypes = [i64p, C.POINTER(C.c_int), C.c_int, C.c_int64, C.c_int64,
                                        C.c_double, C.c_int64, C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]
        L.orc_simulate.argtypes = [i64p, i64p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int,
                                   C.c_int64, i64p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]
        _lib = L
    return _lib


def sample_workload(dist: str, batch_multiplier: int, iterations: int, seed: int):
    f = dist.split(":")
    kind = f[0]
    mu = sigma = 0.0
    alpha = 2.0
    if kind == "uniform":
        lo, hi = int(float(f[1])), int(float(f[2]))
    elif kind == "normal":
        mu, sigma = float(f[1]), float(f[2])
        lo, hi = int(float(f[3])), int(float(f[4]))
    else:
        alpha = float(f[1])
        lo, hi = int(float(f[2])), int(float(f[3]))
    out = (C.c_int64 * max(iterations, 1))()
    rc = lib().orc_sample_workload(DISTS[kind], lo, hi, mu, sigma, alpha, batch_multiplier,
                                   iterations, seed, out)
    assert rc == 0
    return list(out[:iterations])


def fit_layer(xs, ys, order=2):
    n = len(xs)
    xa = (C.c_int64 * n)(*xs)
    ya = (C.c_int64 * n)(*ys)
    co = (C.c_double * (order + 1))()
    rc = lib().orc_fit_layer(xa, ya, n, order, co)
    if rc:
        raise ValueError(f"orc_fit_layer rc={rc}")
    return list(co)


def predict(coeffs, x):
    arr = (C.c_double * len(coeffs))(*coeffs)
    return lib().orc_predict(arr, len(coeffs), x)


def generate_plan(est_bytes, positions, budget, reserve=-1, tol=0.10, constant=0,
                  excess_includes_constant=True):
    L = len(est_bytes)
    e = (C.c_int64 * L)(*est_bytes)
    p = (C.c_int * L)(*positions)
    d = (C.c_int * L)()
    ins = C.c_int()
    rc = lib().orc_generate_plan(e, p, L, budget, reserve, tol, constant,
                                 int(excess_includes_constant), d, C.byref(ins))
    assert rc == 0
    return [i for i in range(L) if d[i]], bool(ins.value)


def simulate(act, bnd, fwd, dropped_idx, constant):
    L = len(act)
    dm = [1 if i in set(dropped_idx) else 0 for i in range(L)]
    peak = C.c_int64()
    t = C.c_double()
    rc_ms = C.c_double()
    rc = lib().orc_simulate((C.c_int64 * L)(*act), (C.c_int64 * L)(*bnd), (C.c_double * L)(*fwd),
                            (C.c_int * L)(*dm), L, constant, C.byref(peak), C.byref(t),
                            C.byref(rc_ms))
    assert rc == 0
    return peak.value, t.value, rc_ms.value


def llround(v: float) -> int:
    """std::llround semantics (half away from zero)."""
    import math
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def layer_bytes(coeffs3, x):
    c0, c1, c2 = coeffs3
    xf = float(x)
    return llround(c0 + c1 * xf + c2 * xf * xf)
