"""The C-ABI library loads without a GPU and exports every symbol the header
declares; the ctypes binding covers the header one to one.  No compute calls."""

import ctypes
import re

import pytest

from conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "hmf.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(hmf_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_hot_path():
    names = header_functions()
    for must in ("hmf_sgd_range_f32", "hmf_sgd_range_f16", "hmf_sgd_range_f64",
                 "hmf_visit_order", "hmf_residual_sums_f32", "hmf_bucket_triples",
                 "hmf_memcpy_peer_async", "hmf_ipc_get_handle"):
        assert must in names


def test_library_exports_every_header_symbol():
    from paper_2006_15980_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2006_15980_b200 import _build
        _build.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in sorted(header_functions()):
        assert hasattr(lib, name), name


def test_binding_matches_header():
    from paper_2006_15980_b200 import _lib
    assert set(_lib.SIGNATURES) == header_functions()


def test_host_only_entry_points():
    from paper_2006_15980_b200 import _lib, kernels
    lib = _lib.load()
    assert lib.hmf_abi_version() == _lib.ABI_VERSION == 5
    for parts in [(0,), (7, 3, 1), (2 ** 63 - 1, 5), (123456789, 42, 17, 3)]:
        assert _lib.mix64_native(*parts) == kernels.mix64(*parts)
    # argument validation happens before any device work
    assert lib.hmf_visit_order(-1, 0, None, None) == _lib.HMF_ERR_ARG
    assert "out of range" in _lib.last_error()
    assert lib.hmf_set_tuning(99, 0) == _lib.HMF_ERR_ARG
    # per-launch options are validated before any device work (ABI 4)
    import ctypes
    args = (None, None, 128, None, None, None, None, None, 4, 1)
    tail = (0.01, 0.0, 0.0, 0, 0, 0, None)
    for bad in ({"pstore": 2}, {"impl": 1}, {"impl": 3}, {"impl": 7}, {"chain_cfg": 0},
                {"chain_cfg": 3},
                {"grid_share": 0}, {"grid_share": 65}, {"lockstep": 4}, {"qsync": -2},
                {"runs_wide": 2}, {"runs_wide": -2}):
        o = _lib.QbandOpts(**bad)
        assert lib.hmf_sgd_block_qband_f32(*args, ctypes.byref(o), *tail) == _lib.HMF_ERR_ARG, bad
    assert lib.hmf_qband_resolve_impl(128, 0) == 5
    assert [lib.hmf_qband_resolve_chain_cfg(k, f) for k in (32, 64, 128, 256) for f in (0, 1)] \
        == [2, 2, 2, 4, 5, 6, 5, 6]
    assert [lib.hmf_qband_chain_lanes(k, 0, -1) for k in (32, 64, 128, 256)] == [4, 8, 8, 16]
    assert lib.hmf_qband_max_items(128, 0, 0) == 8 and lib.hmf_qband_max_items(128, 0, 5) == 1 << 30
    assert lib.hmf_sgd_range_f32(None, None, 4, None, None, None, 0, 0, 0.1, 0, 0, 0, 0, 0, 0,
                                 None) == 0  # empty range: nothing to do, no error


def test_product_path_has_no_oracle_dependency():
    """The package never imports or loads the CPU oracle."""
    pkg = ROOT / "paper_2006_15980_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
        assert "hmf_oracle" not in src, p


def test_package_reexports_reference_names():
    """Every public name of the reference (hetmf/__init__.py:31-44) is
    importable from the package, except the two documented out-of-scope ones."""
    import paper_2006_15980_b200 as pkg
    from oracle import reference
    if reference.installed():
        ref_all = set(reference.hetmf().__all__)
        assert ref_all - set(pkg.REFERENCE_NAMES) == set(pkg.NOT_EXPORTED)
    for name in pkg.__all__:
        assert hasattr(pkg, name), name
