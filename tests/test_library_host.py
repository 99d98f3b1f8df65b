"""Host-only checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/irls_mincut.h declares, and its host helpers (status
strings, options defaults, the multi-GPU slab plan, the slot tree) behave."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1501_03105_b200 import build, irls
    build.build()
    return irls


def header_symbols():
    src = open(os.path.join(ROOT, "include", "irls_mincut.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(irls_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(L):
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(L.SYMBOLS) == syms


def test_options_default_and_status_strings(L):
    o = L.options()
    assert (o.eps, o.T, o.cg_rtol, o.cg_max_iter, o.cg_norm, o.warm_start) == (1e-6, 50, 1e-3, 50, 0, 1)
    for code, name in L.STATUS_NAMES.items():
        assert L.lib().irls_status_string(code).decode() == name


def test_plan_stencil_group_aligned(L):
    # config 4: 512x512x256, K = 16384 chunks, 32 planes per group
    for W in (1, 2, 4, 8):
        planes = []
        for r in range(W):
            z0, z1, g0, g1 = L.irls_plan_stencil(512, 512, 256, W, r)
            assert (g0, g1) == (r * 8 // W, (r + 1) * 8 // W)
            planes.append((z0, z1))
        assert planes[0][0] == 0 and planes[-1][1] == 256
        assert all(a[1] == b[0] for a, b in zip(planes, planes[1:]))
        assert all(z1 - z0 == 256 // W for z0, z1 in planes)
    # config 2: 128^3
    assert L.irls_plan_stencil(128, 128, 128, 8, 3)[:2] == (48, 64)
    with pytest.raises(L.IrlsError):
        L.irls_plan_stencil(128, 128, 128, 3, 0)      # world must divide 8
    with pytest.raises(L.IrlsError):
        L.irls_plan_stencil(100, 7, 9, 2, 0)          # group boundary inside a plane


def test_combine_slots_tree(L):
    import oracle
    rng = np.random.default_rng(5)
    for n in (5, 4097, 100003):
        v = rng.standard_normal(n)
        gs = oracle.c3_group_sums(v)
        assert L.irls_combine_slots(gs) == oracle.c3_sum(v)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_1501_03105_b200 import irls
    monkeypatch.setattr(irls, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(irls, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        irls.lib()
