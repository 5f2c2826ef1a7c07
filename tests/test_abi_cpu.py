"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol that
include/pca.h declares, and validates configurations before any device work."""
import ctypes
import os
import re

import pytest

import paper_2507_14869_b200 as P
from paper_2507_14869_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "pca.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pca_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return P.lib()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(P.EXPORTS) == names
    assert lib.pca_abi_version() == 1


def test_config_struct_layout_matches_header():
    # 6 int32, 5 double, 2 int32, double, uint64, 8 int32, 4 int32 reserved (natural alignment)
    assert ctypes.sizeof(P.pca_config) == 24 + 40 + 8 + 8 + 8 + 20 + 28
    assert P.pca_config.seed.offset == 80 and P.pca_config.inertia_p.offset == 112 and P.pca_config.packed_io.offset == 116 and P.pca_config.graphs.offset == 120 and P.pca_config.reserved.offset == 124


def test_workspace_and_validation(lib):
    c = P.make_config(64, 64, 2)
    assert P.pca_workspace_bytes(c) > 2 * 66 * 96
    bad = [
        dict(levels=1), dict(levels=256), dict(neighborhood=6), dict(periodic=True, height=2),
        dict(J=0.0), dict(q=-1.0), dict(sigma=0.0), dict(beta0=0.0), dict(beta_step=-0.1),
        dict(beta_period=0), dict(coef_scale=0.0), dict(rows=10, row0=60), dict(batch=0),
        dict(kernel=P.KERNEL_BINARY, levels=3), dict(rows_per_thread=-3), dict(batch=70000), dict(kernel=3), dict(inertia_p=3), dict(inertia_p=-1), dict(packed_io=2),
        dict(packed_io=1, levels=5),
    ]
    for kw in bad:
        args = dict(height=64, width=64, levels=2)
        args.update(kw)
        cfg = P.make_config(args.pop("height"), args.pop("width"), args.pop("levels"), **args)
        assert lib.pca_workspace_bytes(ctypes.byref(cfg)) == 0, kw
        assert lib.pca_last_error().decode(), kw
    c = P.make_config(64, 64, 2)
    c.sweeps_per_pass = 3
    assert lib.pca_workspace_bytes(ctypes.byref(c)) == 0
    c = P.make_config(64, 64, 2)
    c.reserved[2] = 1
    assert lib.pca_workspace_bytes(ctypes.byref(c)) == 0


def test_init_rejects_host_workspace_without_touching_a_device(lib):
    cfg = P.make_config(16, 16, 2)
    buf = ctypes.create_string_buffer(1 << 16)
    aligned = (ctypes.addressof(buf) + 255) // 256 * 256
    h = ctypes.c_void_p()
    g = (ctypes.c_uint8 * 256)()
    st = lib.pca_init(ctypes.byref(h), ctypes.byref(cfg), aligned, 1 << 15, ctypes.addressof(g),
                      None, None)
    assert st in (P.PCA_EINVAL, P.PCA_ENOSPACE) and not h.value
    st = lib.pca_init(ctypes.byref(h), ctypes.byref(cfg), aligned, 16, ctypes.addressof(g), None,
                      None)
    assert st == P.PCA_ENOSPACE
    assert lib.pca_sweep(None, 1) == P.PCA_EINVAL
    assert lib.pca_destroy(None) == P.PCA_OK
