"""The C-ABI library loads without a GPU, exports every symbol include/*.h declares, and its
host-side planner is bit-exact with the reference plan_partition / recursion shape."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import blocktri_port as port
from paper_2509_03015_b200 import _native
import paper_2509_03015_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            syms |= set(re.findall(r"\b(btd_[a-z_]+)\s*\(", txt))
    return syms


def test_library_exports_declared_symbols():
    L = _native.lib()
    declared = _declared_symbols()
    assert declared == set(_native.EXPORTED_SYMBOLS)
    for s in declared:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.btd_version()


def test_native_plan_matches_golden(golden):
    seps, offs = golden["plans_seps"], golden["plans_offsets"]
    idx = 0
    for rho in range(1, 21):
        for N in range(3, 701):
            plan = pkg.plan_partition(N, pkg.RecursionConfig(segment_length=rho))
            assert list(plan.separators) == list(seps[offs[idx]:offs[idx + 1]])
            idx += 1


@pytest.mark.parametrize("rho", [1, 2, 3, 8, 17, 32])
def test_native_plan_matches_port_large(rho):
    for N in list(range(3, 3000, 7)) + [65536, 1048576, 1048575, 100003]:
        plan = pkg.plan_partition(N, pkg.RecursionConfig(segment_length=rho))
        assert list(plan.separators) == port.plan_separators(N, rho)


def _levels_native(N, cfg):
    L = _native.lib()
    h = ctypes.c_void_p()
    st = _native.BtdStatus()
    c = cfg._c()
    assert L.btd_create(N, 4, ctypes.byref(c), ctypes.byref(h), ctypes.byref(st)) == 0
    nl, nb, ov = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    L.btd_num_levels(h, ctypes.byref(nl), ctypes.byref(nb), ctypes.byref(ov))
    sizes = []
    for lvl in range(nl.value):
        a, p = ctypes.c_int64(), ctypes.c_int64()
        L.btd_level_info(h, lvl, ctypes.byref(a), ctypes.byref(p), None)
        sizes.append(a.value)
    L.btd_destroy(h)
    return sizes, nb.value, bool(ov.value)


def _levels_port(N, cross, rho, maxl, auto):
    sizes, cur = [], N
    while port.should_recurse(cur, cross, rho, auto):
        if len(sizes) >= maxl:
            return sizes, cur, True
        sizes.append(cur)
        cur = len(port.plan_separators(cur, rho))
    return sizes, cur, False


@pytest.mark.parametrize("cfg", [(64, 8, 32, False), (1, 1, 32, False), (5, 3, 2, False), (64, 8, 32, True),
                                 (10, 2, 3, True)])
def test_recursion_shape_matches_port(cfg):
    cross, rho, maxl, auto = cfg
    rc = pkg.RecursionConfig(crossover=cross, segment_length=rho, max_levels=maxl, auto_crossover=auto)
    for N in [1, 2, 3, 4, 9, 64, 65, 100, 1024, 4096, 65536, 1048576]:
        assert _levels_native(N, rc) == _levels_port(N, cross, rho, maxl, auto), (N, cfg)


def test_baseline_level_structure():
    # SURVEY.md §0 table (measured with the reference plan_partition)
    cfg = pkg.RecursionConfig()
    assert _levels_native(1024, cfg)[0:2] == ([1024, 115], 14)
    assert _levels_native(65536, cfg)[0:2] == ([65536, 7283, 810, 91], 11)
    assert _levels_native(1048576, cfg)[0:2] == ([1048576, 116510, 12947, 1440, 161], 19)
    assert _levels_native(4096, cfg)[0:2] == ([4096, 456], 52)


def test_config_validation():
    with pytest.raises(ValueError):
        pkg.RecursionConfig(crossover=0)
    with pytest.raises(ValueError):
        pkg.plan_partition(2, pkg.RecursionConfig())
