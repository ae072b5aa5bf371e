"""CPU-only checks of the boundary: libencoder.so loads, exports every entry point that
include/encoder.h declares, and rejects bad arguments on the host (no GPU needed for
these: argument validation happens before any device call)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "encoder.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(enc_\w+|encoder_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2007_00072_b200 import _abi
    return _abi.load()


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("encoder_layer_forward", "encoder_layer_backward", "enc_bsb_fwd", "enc_bsb_bwd",
              "enc_bdrln_fwd", "enc_bdrln_bwd", "enc_bad_fwd", "enc_bad_bwd", "enc_aib_fwd",
              "enc_aib_bwd", "enc_bei", "enc_dropout_mask"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2007_00072_b200 import _abi
    for n in _declared():
        assert hasattr(lib, n), n
        assert n in _abi.EXPORTED, f"{n} missing from the ctypes binding"


def test_host_side_validation(lib):
    from paper_2007_00072_b200 import _abi
    sb, cb = ctypes.c_size_t(), ctypes.c_size_t()
    ok = _abi.enc_dims(8, 512, 512, 16, 64, 64, 1024, 4096)
    assert lib.enc_layer_sizes(ctypes.byref(ok), 0, ctypes.byref(sb), ctypes.byref(cb)) == 0
    # saved set at config L: Q,K,V,C,X1,xhat1,xhat2 (7 x BJI) + P,A (2 x BHJK) + h,A1 (2 x BJU)
    BJI, BHJK, BJU = 4096 * 1024 * 2, 8 * 16 * 512 * 512 * 2, 4096 * 4096 * 2
    assert sb.value >= 7 * BJI + 2 * BHJK + 2 * BJU + 2 * 4096 * 4
    bad_k = _abi.enc_dims(8, 512, 256, 16, 64, 64, 1024, 4096)
    assert lib.enc_layer_sizes(ctypes.byref(bad_k), 0, None, None) == -1
    bad_i = _abi.enc_dims(8, 512, 512, 16, 64, 64, 1000, 4096)
    assert lib.enc_layer_sizes(ctypes.byref(bad_i), 0, None, None) == -1
    bad_al = _abi.enc_dims(8, 512, 512, 16, 60, 60, 960, 4096)
    assert lib.enc_layer_sizes(ctypes.byref(bad_al), 0, None, None) == -2
    assert lib.enc_layer_sizes(ctypes.byref(ok), 7, None, None) == -3
    # p outside [0, 1) is rejected before any launch
    assert lib.enc_dropout_mask(10, 0, 1.0, 1, 0, None, None) == -1
    assert lib.enc_strerror(-2).decode().startswith("misaligned")
    assert b"sm_100a" in lib.enc_version()


def test_binding_fails_loudly_without_library(tmp_path):
    from paper_2007_00072_b200 import _abi
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _abi.load(str(tmp_path / "missing.so"))


@pytest.mark.parametrize("script", ["bench.py", "bench_ops.py", "__graft_entry__.py",
                                    "tools/select_config.py", "tools/one_step.py",
                                    "tools/trace_fused.py"])
def test_driver_scripts_compile(script):
    """The driver runs bench.py and __graft_entry__.py on the GPU box only: catch syntax
    errors here."""
    import py_compile
    py_compile.compile(os.path.join(ROOT, script), doraise=True)


def test_bench_parses_its_flags():
    """bench.py's argument parser accepts every documented flag combination (no GPU)."""
    import sys
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    old = sys.argv
    try:
        for argv in (["bench.py"], ["bench.py", "--config", "Bb", "--causal", "--attn-overlap", "0"],
                     ["bench.py", "--layers", "24", "--optimizer", "--no-prefetch"],
                     ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"]):
            sys.argv = argv
            a = bench.parse()
            assert a.steps >= 1
    finally:
        sys.argv = old
