"""The C-ABI library loads and exports every symbol include/tlp.h declares; host-side
validation works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tlp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tlp_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2211_03578_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2211_03578_b200 import build
        build.build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    from paper_2211_03578_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (tlp_\w+)", out))
    for s in syms:
        assert s in exported, s
        getattr(lib, s)
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a_and_links_pip_nccl():
    from paper_2211_03578_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    nccl = [l for l in ldd.splitlines() if "libnccl" in l]
    assert nccl and "nvidia/nccl" in nccl[0]


def test_default_config_is_the_papers(lib):
    from paper_2211_03578_b200 import _lib
    c = _lib.tlp_config()
    lib.tlp_default_config(C.byref(c))
    # P:273 / P:428: 25 x 22, 11-wide one-hot; 256 hidden, 8 heads, 1 layer, 2 res blocks
    assert (c.L, c.E, c.T, c.hidden, c.attn_heads, c.n_attn, c.n_res) == (25, 22, 11, 256, 8, 1, 2)
    assert list(c.up_dims[:c.n_up]) == [128, 256] and c.head_dim == 128
    assert abs(c.lr - 1e-3) < 1e-9 and abs(c.beta2 - 0.999) < 1e-7


def test_config_validation_is_host_side(lib):
    from paper_2211_03578_b200 import _lib
    c = _lib.tlp_config()
    lib.tlp_default_config(C.byref(c))
    c.hidden = 250  # not divisible by 8 heads / up_dims mismatch
    h = C.c_void_p()
    st = lib.tlp_create(C.byref(c), 0, C.byref(h))
    assert st == -2 and not h.value
    assert b"up_dims" in lib.tlp_last_error(None) or b"hidden" in lib.tlp_last_error(None)
    lib.tlp_default_config(C.byref(c))
    c.L = 40
    assert lib.tlp_create(C.byref(c), 0, C.byref(h)) == -2


def test_null_arguments_rejected(lib):
    assert lib.tlp_create(None, 0, None) == -1
    assert lib.tlp_sync(None) == -1
    assert lib.tlp_num_params(None) == -1


@pytest.mark.parametrize("kw", [dict(), dict(n_attn=2, n_tasks=4), dict(pos_enc=True, n_attn=2),
                                dict(backbone="lstm", n_attn=1, hidden=64, up_dims=(32, 64), head_dim=32)])
def test_product_param_layout_matches_r24(kw):
    """The binding's parameter layout (used to initialise weights without the
    oracle) equals the oracle's R24 order, names and shapes."""
    from paper_2211_03578_b200 import TLPConfig
    from oracle import model as OM
    pc = TLPConfig(**kw)
    oc = OM.Config(**{k: v for k, v in kw.items()})
    assert pc.param_shapes() == [(n, tuple(s)) for n, s in OM.param_shapes(oc)]
