"""CPU-side checks of the C-ABI libraries (no GPU compute calls).

* both libraries load and export every symbol their header declares;
* nothing but the C ABI is exported (no C++ / libstdc++ symbol leakage that
  could interpose between the product and the oracle's compiled reference);
* the budget arena's book-keeping (the allocator core) enforces the cap,
  coalesces, and keeps byte-exact requested/reserved counters;
* host-side helpers (token tables) are deterministic and stable.
"""
import ctypes as C
import os
import random
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _declared(header, prefix):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z0-9_]+)\s*\(", text)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    return sorted({l.split()[-1] for l in out.splitlines() if " T " in l})


def test_cuda_lib_exports_exactly_the_header():
    from paper_2209_02478_b200 import _lib
    lib = _lib.cuda_lib()  # loads (no GPU needed) and binds every symbol
    decl = _declared("mimose_cuda.h", "mimose_")
    exp = _exported(_lib.CUDA_LIB_PATH)
    assert decl, "no declarations parsed"
    assert set(decl) <= set(exp), set(decl) - set(exp)
    assert all(s.startswith("mimose_") for s in exp), [s for s in exp if not s.startswith("mimose_")]
    bound = {name for name, _, _ in _lib.CUDA_SYMBOLS}
    assert set(decl) == bound, set(decl) ^ bound
    assert lib.mimose_abi_version() == _lib.ABI_VERSION == 7


def test_host_lib_exports_exactly_the_header():
    from paper_2209_02478_b200 import _lib, planner
    planner.host_lib()
    decl = _declared("mimose_planner.h", "mimose_planner_")
    exp = _exported(_lib.HOST_LIB_PATH)
    assert set(decl) == set(exp)


def _book():
    from paper_2209_02478_b200 import _lib
    lib = _lib.cuda_lib()
    h = C.c_void_p()
    assert lib.mimose_book_create(1 << 20, C.byref(h)) == 0
    return lib, h


def _stats(lib, h):
    from paper_2209_02478_b200 import _lib
    st = _lib.MemStats()
    lib.mimose_book_stats(h, C.byref(st))
    return st.as_dict()


def test_arena_book_enforces_budget_and_coalesces():
    lib, h = _book()
    a = lib.mimose_book_alloc(h, 300_000, 3)
    b = lib.mimose_book_alloc(h, 300_000, 3)
    c = lib.mimose_book_alloc(h, 300_000, 5)
    assert min(a, b, c) >= 0
    assert lib.mimose_book_alloc(h, 300_000, 3) == -1  # 1 MiB cap: 4th does not fit
    st = _stats(lib, h)
    assert st["requested"] == 900_000
    assert st["reserved"] == 3 * (300_000 + (-300_000) % 256)
    assert st["n_failures"] == 1
    assert st["tag_requested"]["act"] == 600_000 and st["tag_requested"]["transient"] == 300_000
    assert lib.mimose_book_free(h, b) == 0
    assert lib.mimose_book_free(h, a) == 0  # coalesces with b's hole
    d = lib.mimose_book_alloc(h, 600_000, 3)
    assert d == a  # best fit lands in the merged block
    assert lib.mimose_book_free(h, 12345) != 0  # foreign offset rejected
    assert lib.mimose_book_free(h, c) == 0 and lib.mimose_book_free(h, d) == 0
    st = _stats(lib, h)
    assert st["requested"] == 0 and st["reserved"] == 0 and st["largest_free"] == 1 << 20
    assert st["peak_requested"] == 900_000
    lib.mimose_book_destroy(h)


def test_arena_book_randomised_invariants():
    lib, h = _book()
    rng = random.Random(7)
    live = {}
    for _ in range(4000):
        if live and rng.random() < 0.45:
            off = rng.choice(list(live))
            assert lib.mimose_book_free(h, off) == 0
            del live[off]
        else:
            n = rng.randint(1, 60_000)
            off = lib.mimose_book_alloc(h, n, rng.randint(0, 7))
            if off >= 0:
                # no overlap with any live block
                for o, m in live.items():
                    assert off + n <= o or o + m <= off
                live[off] = n
        st = _stats(lib, h)
        assert st["requested"] == sum(live.values())
        assert st["reserved"] <= 1 << 20 and st["n_live"] == len(live)
    lib.mimose_book_destroy(h)


def test_token_tables_stable_counting_sort():
    from paper_2209_02478_b200.trainer import token_tables
    rng = np.random.default_rng(0)
    tok = rng.integers(0, 50, size=1000, dtype=np.int32)
    perm, seg, uid, nu = token_tables(tok, 50)
    assert nu == len(np.unique(tok))
    assert list(uid) == sorted(np.unique(tok).tolist())
    for u in range(nu):
        pos = perm[seg[u]:seg[u + 1]]
        assert np.all(tok[pos] == uid[u])
        assert np.all(np.diff(pos) > 0)  # ascending positions -> fixed summation order
    assert sorted(perm.tolist()) == list(range(1000))


def _plan(off, bucket):
    from paper_2209_02478_b200 import _lib
    lib = _lib.cuda_lib()
    arr = (C.c_int64 * len(off))(*off)
    out = (C.c_int64 * (3 * len(off)))()
    n = C.c_int()
    _lib.check(lib.mimose_dp_plan_buckets(arr, len(off) - 1, bucket, out, len(off), C.byref(n)))
    return [tuple(out[3 * i:3 * i + 3]) for i in range(n.value)]


def test_dp_bucket_schedule_covers_grads_back_to_front():
    """Buckets tile the flat gradient buffer exactly once, are issued in
    backward completion order (head, last block, ..., embeddings), each
    >= the bucket size except the final one, and only ever cover units that
    are already final when issued."""
    rng = random.Random(3)
    for _ in range(200):
        U = rng.randint(1, 30)
        sizes = [rng.choice([0, 64, 640, 7_000_000 // 64 * 64]) for _ in range(U)]
        off = [0]
        for s in sizes:
            off.append(off[-1] + s)
        bucket = rng.choice([1, 64, 1000, 5_000_000, 10 ** 9])
        b = _plan(off, bucket)
        covered = sorted((beg, end) for _, beg, end in b)
        pos = 0
        for beg, end in covered:
            assert beg == pos and end > beg
            pos = end
        assert pos == off[-1] or (pos == 0 and off[-1] == 0)
        units = [u for u, _, _ in b]
        assert units == sorted(units, reverse=True)
        for k, (u, beg, end) in enumerate(b):
            assert beg == off[u]  # the bucket starts at the unit just finished
            if k < len(b) - 1:
                assert end - beg >= bucket


def test_dp_bucket_schedule_examples():
    # 3 units of 100 elements, 150-element buckets: after unit 1 -> [100, 300), after unit 0
    assert _plan([0, 100, 200, 300], 150) == [(1, 100, 300), (0, 0, 100)]
    # one big bucket: only at the end
    assert _plan([0, 100, 200, 300], 10 ** 6) == [(0, 0, 300)]
    # per-unit buckets
    assert _plan([0, 100, 200, 300], 1) == [(2, 200, 300), (1, 100, 200), (0, 0, 100)]
