"""The C-ABI library loads and exports every symbol include/qem.h declares (CPU; no kernel calls).

Also exercises the pure-host entry points (validation, shard ranges) and the
"fail loudly" contract of the product when the extension is missing.
"""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_08264_b200 import build
    build.build()
    from paper_2503_08264_b200 import _lib
    return _lib.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "qem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(qem_[a-z_]+)\s*\(", src)
    return sorted(set(names))


def test_every_declared_symbol_is_exported(lib):
    from paper_2503_08264_b200 import _lib
    decl = declared_functions()
    assert set(decl) == set(_lib.EXPORTS), set(decl) ^ set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a(lib):
    from paper_2503_08264_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validate_and_shard_range(lib):
    from paper_2503_08264_b200 import qem, synth
    for cid in (1, 2, 3, 4, 5):
        assert qem.model_validate(synth.config(cid)) is None
    bad = synth.config(4, K=2000)
    assert "K=2000" in qem.model_validate(bad)
    bad = synth.config(1)
    bad.d = 5
    assert "d=5" in qem.model_validate(bad) or "OBS_GAUSS" in qem.model_validate(bad)
    assert qem.model_validate(synth.config(2, d=5)) is None  # d = 5 is on the compiled menu
    bad = synth.config(2, d=11)
    assert "no compiled kernel" in qem.model_validate(bad) and "QEM_D_MENU" in qem.model_validate(bad)
    # shards tile [0, n) exactly, contiguous, balanced within 1
    for n in (1, 7, 100_000, 10_000):
        for world in (1, 2, 3, 8):
            prev = 0
            sizes = []
            for r in range(world):
                b, e = qem.shard_range(n, r, world)
                assert b == prev
                prev = e
                sizes.append(e - b)
            assert prev == n and max(sizes) - min(sizes) <= 1
    with pytest.raises(Exception):
        qem.shard_range(10, 3, 2)


def test_empty_and_out_of_range_group_blocks_are_rejected(lib):
    """Error behaviour of the boundary on degenerate shards (include/qem.h, qem_create): a context owns a
    non-empty block [group_begin, group_end) inside [0, n); an empty, reversed or out-of-range block --
    e.g. a rank of a world larger than n, whose qem_shard_range block is empty -- is
    QEM_INVALID_ARGUMENT before any device call (checked here on the CPU through qem_workspace_bytes,
    the host-only arithmetic of qem_create)."""
    from paper_2503_08264_b200 import _lib, qem, synth
    m = synth.config(1)  # n = 4 groups
    for gb, ge in ((0, 0), (2, 2), (3, 1), (-1, 2), (0, m.n + 1), (m.n, m.n)):
        with pytest.raises(_lib.QemError, match="QEM_INVALID_ARGUMENT"):
            qem.workspace_bytes(m, gb, ge)
    # world = 8 > n = 4: the blocks still tile [0, n) and half of them are empty (those ranks make no context)
    blocks = [qem.shard_range(m.n, r, 8) for r in range(8)]
    assert sum(e - b for b, e in blocks) == m.n and sum(1 for b, e in blocks if e == b) == 4
    m3 = synth.config(3)  # three-level: replicas only, a proper sub-block is QEM_UNSUPPORTED
    with pytest.raises(_lib.QemError, match="QEM_UNSUPPORTED"):
        qem.workspace_bytes(m3, 0, 3)


def test_product_fails_loudly_without_extension(tmp_path):
    """With libqem.so absent, the binding raises instead of falling back."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_2503_08264_b200 import _lib\n"
        "_lib.LIB_PATH = %r\n"
        "try:\n    _lib.lib()\nexcept _lib.QemError as e:\n    print('RAISED', e)\n" % (ROOT, str(tmp_path / "nope.so")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout
    assert "RAISED" in out


def test_product_does_not_import_oracle():
    """No module of the product package imports, links or executes anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2503_08264_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(^\s*(from|import)\s+oracle\b|liboracle|qem_oracle|orc_)", src, re.M), f


@pytest.mark.gpu
def test_caller_workspace_matches_own_workspace():
    """qem_create_in on a caller allocation (sized by qem_workspace_bytes) computes exactly what
    qem_create's own workspace does; a short or misaligned workspace is rejected."""
    import numpy as np
    import torch
    from paper_2503_08264_b200 import _lib, synth
    from paper_2503_08264_b200.qem import QEM, workspace_bytes
    m = synth.config(5, n=40, K=256)
    data = synth.make_data(m)
    outs = []
    for caller in (False, True):
        g = QEM(m, caller_workspace=caller)
        g.set_data(data)
        g.set_q(synth.initial_q(m))
        g.iterate(1, 2, seed=3)
        outs.append(g.result())
        if caller:
            assert g._ws.numel() == workspace_bytes(m)
        g.close()
    for l in range(2):
        np.testing.assert_array_equal(outs[0]["q_mean"][l], outs[1]["q_mean"][l])
        np.testing.assert_array_equal(outs[0]["w"][l], outs[1]["w"][l])
    L = _lib.lib()
    d = _lib_desc(m)
    o = _lib.Opts(0.3, 0.0, 1e-8, 0, 0)
    nb = workspace_bytes(m)
    buf = torch.empty(nb + 512, dtype=torch.uint8, device="cuda")
    ctx = ctypes.c_void_p()
    assert L.qem_create_in(ctypes.byref(d), ctypes.byref(o), 0, m.n, ctypes.c_void_p(buf.data_ptr()), nb - 256,
                           ctypes.byref(ctx)) == _lib.INVALID_ARGUMENT
    assert L.qem_create_in(ctypes.byref(d), ctypes.byref(o), 0, m.n, ctypes.c_void_p(buf.data_ptr() + 8), nb,
                           ctypes.byref(ctx)) == _lib.INVALID_ARGUMENT
    assert L.qem_create_in(ctypes.byref(d), ctypes.byref(o), 0, m.n, ctypes.c_void_p(buf.data_ptr()), nb,
                           ctypes.byref(ctx)) == _lib.OK
    L.qem_destroy(ctx)


def _lib_desc(m):
    from paper_2503_08264_b200.qem import _desc
    return _desc(m)


def test_history_weight_matches_the_oracle_schedule():
    """qem_history_weight (host arithmetic, no GPU): lambda = 1 - w, or 1 - t^-p with a schedule
    (R5; Theorem 1), equal to the oracle's."""
    from oracle import oracle as orc
    from paper_2503_08264_b200 import _lib
    L = _lib.lib()
    for t in (1, 2, 7, 100):
        for w, p in ((0.3, 0.0), (0.05, 0.0), (0.3, 0.5), (0.3, 0.75)):
            assert abs(L.qem_history_weight(t, w, p) - orc.lam(t, w, p)) <= 1e-15
