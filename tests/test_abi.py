"""CPU-side checks of the C-ABI boundary (no compute calls): libaca.so builds for sm_100a,
loads, exports every function include/aca.h declares, the ctypes structs match the C
layout, and the product and the oracle share no code."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "aca.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(aca_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libaca():
    from paper_cs_0502039_b200 import _build
    _build.build()
    import paper_cs_0502039_b200 as pkg
    return pkg


def test_header_declares_the_north_star_calls():
    fns = _header_functions()
    for name in ("aca_create", "aca_run_until", "aca_get_spins", "aca_get_times", "aca_get_counters",
                 "aca_get_stats", "aca_destroy", "aca_last_error"):
        assert name in fns


def test_library_exports_every_declared_symbol(libaca):
    fns = _header_functions()
    assert sorted(libaca.EXPORTS) == fns
    L = ctypes.CDLL(libaca.library_path())
    for name in fns:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libaca.library_path()], capture_output=True, text=True).stdout
    for name in fns:
        assert re.search(r"\bT %s$" % name, out, flags=re.M), name


def test_library_is_sm100a(libaca):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libaca.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_options_struct_layout(libaca):
    o = libaca.aca_default_options()
    assert o.struct_size == ctypes.sizeof(libaca.aca_options)
    assert o.init_q == 0.5 and o.world == 1 and o.shards == 1 and o.event_hash == 1 and o.device == -1


def test_no_cpu_fallback_without_gpu(libaca):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(libaca.AcaError) as ei:
        libaca.aca_create((8, 8))
    assert ei.value.code == -7   # ACA_ENODEV


def test_invalid_arguments_are_rejected_before_the_device(libaca):
    bad = [dict(dims=(1, 8)), dict(dims=(8,)), dict(dims=(8, 8), periodic=0), dict(dims=(8, 8), lam=0.0),
           dict(dims=(8, 8), beta=-1.0), dict(dims=(8, 8), rule=3), dict(dims=(4, 4, 4), rule=2),
           dict(dims=(8, 8), lam=float("nan"))]
    for kw in bad:
        dims = kw.pop("dims")
        with pytest.raises(libaca.AcaError) as ei:
            libaca.aca_create(dims, **kw)
        assert ei.value.code == -1, (dims, kw)


def test_product_and_oracle_share_no_code():
    """The oracle is independent of the CUDA path: neither imports, includes or loads the other."""
    pkg = os.path.join(ROOT, "paper_cs_0502039_b200")
    banned_in_product = ("import oracle", "from oracle", "aca_oracle", "liboracle", "nlog_tables.h\"")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                for b in banned_in_product:
                    assert b not in txt, (f, b)
    banned_in_oracle = ("import paper_cs_0502039_b200", "from paper_cs_0502039_b200", "libaca",
                        "aca_kernels", "aca_prim", "nlog_tables.cuh")
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            for b in banned_in_oracle:
                assert b not in txt, (f, b)
