"""ctypes facade of the host planner (libmimose_host.so, include/mimose_planner.h).

The planner itself is the C++ of include/mimose/*.hpp - the same code the B200
trainer links - so these calls produce the plans the GPU executor applies.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Sequence, Tuple

from ._lib import HOST_LIB_PATH, MimoseError

_host = None


class SchedCfg(C.Structure):
    _fields_ = [
        ("budget_bytes", C.c_int64),
        ("reserve_bytes", C.c_int64),
        ("bucket_tolerance", C.c_double),
        ("cache_tolerance", C.c_double),
        ("excess_includes_constant", C.c_int),
    ]

    def __init__(self, budget_bytes=0, reserve_bytes=-1, bucket_tolerance=0.10,
                 cache_tolerance=0.0, excess_includes_constant=True):
        super().__init__(budget_bytes, reserve_bytes, bucket_tolerance, cache_tolerance,
                         int(excess_includes_constant))


_P = C.c_void_p
SYMBOLS = [
    ("last_error", C.c_char_p, []),
    ("free", None, [_P]),
    ("fit", C.c_int, [C.c_char_p, C.c_int, C.POINTER(_P)]),
    ("plan_sequence", C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(SchedCfg),
                                C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_uint64), C.c_int,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("simulate", C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.c_int, C.c_int64,
                           C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("sample_workload", C.c_int, [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64,
                                  C.POINTER(C.c_int64)]),
    ("run_experiment", C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, C.c_int64, C.c_uint64,
                                 C.POINTER(SchedCfg), C.c_char_p, C.POINTER(_P), C.POINTER(_P)]),
]


class PlannerLib:
    """Binds one planner C ABI (product prefix `mimose_planner_`; the oracle's
    compiled reference exports the same functions under `ref_planner_`)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise MimoseError(f"{path} missing: run `make`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        for name, res, args in SYMBOLS:
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def _check(self, rc):
        if rc != 0:
            raise MimoseError(self.last_error().decode())

    def _take(self, p) -> str:
        try:
            return C.cast(p, C.c_char_p).value.decode()
        finally:
            self.free(p)

    # ------------------------------------------------------------- calls
    def fit_text(self, samples_csv: str, order: int = 2) -> str:
        out = _P()
        self._check(self.fit(samples_csv.encode(), order, C.byref(out)))
        return self._take(out)

    def plan_seq(self, estimator_text: str, model_text: str, cfg: SchedCfg,
                 xs: Sequence[int], layers: int) -> Tuple[List[int], List[int], List[int]]:
        n = len(xs)
        words = (layers + 63) // 64
        xa = (C.c_int64 * max(n, 1))(*xs)
        masks = (C.c_uint64 * max(n * words, 1))()
        ins = (C.c_int * max(n, 1))()
        hit = (C.c_int * max(n, 1))()
        self._check(self.plan_sequence(estimator_text.encode(), model_text.encode(),
                                       C.byref(cfg), xa, n, masks, words, ins, hit))
        m = [sum(masks[i * words + w] << (64 * w) for w in range(words)) for i in range(n)]
        return m, list(ins[:n]), list(hit[:n])

    def simulate_plan(self, model_text: str, dropped: Sequence[int], x: int):
        arr = (C.c_int * max(len(dropped), 1))(*dropped)
        peak, it, rc = C.c_int64(), C.c_double(), C.c_double()
        self._check(self.simulate(model_text.encode(), arr, len(dropped), x, C.byref(peak),
                                  C.byref(it), C.byref(rc)))
        return peak.value, it.value, rc.value

    def workload(self, dist: str, batch_multiplier: int, iterations: int, seed: int) -> List[int]:
        out = (C.c_int64 * max(iterations, 1))()
        self._check(self.sample_workload(dist.encode(), batch_multiplier, iterations, seed, out))
        return list(out[:iterations])

    def experiment(self, model_text: str, dist: str, batch_multiplier: int, iterations: int,
                   seed: int, cfg: SchedCfg, planner: str = "mimose") -> Tuple[str, str]:
        s, c = _P(), _P()
        self._check(self.run_experiment(model_text.encode(), dist.encode(), batch_multiplier,
                                        iterations, seed, C.byref(cfg), planner.encode(),
                                        C.byref(s), C.byref(c)))
        return self._take(s), self._take(c)


def host_lib() -> PlannerLib:
    global _host
    if _host is None:
        _host = PlannerLib(HOST_LIB_PATH, "mimose_planner_")
    return _host


def fit(samples_csv: str, order: int = 2) -> str:
    return host_lib().fit_text(samples_csv, order)


def plan_sequence(estimator_text, model_text, cfg, xs, layers):
    return host_lib().plan_seq(estimator_text, model_text, cfg, xs, layers)
