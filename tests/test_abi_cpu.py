"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
header declares, and rejects bad arguments host-side (no device work)."""

import ctypes
import os
import re

import pytest

from paper_2305_13925_b200 import _lib as L
from paper_2305_13925_b200.build_ext import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xlmimo_b200.h")


@pytest.fixture(scope="module")
def lib():
    build()
    return L.load_library()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("xl_gram", "xl_solve", "xl_rzf", "xl_sinr", "xl_apply_precoder",
              "xl_channel_generate", "xl_se_partials"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in L._SIGNATURES, f"{s} has no ctypes signature"


def test_abi_version(lib):
    assert lib.xl_abi_version() == 1


def test_host_side_validation_without_device(lib):
    # ConfigurationError-class checks return before any CUDA call.
    assert lib.xl_gram(0, None, 1, 4, 4, 0.0, None, None, None) == L.XL_ERR_CONFIG     # xi <= 0
    assert lib.xl_gram(7, None, 1, 4, 4, 1.0, None, None, None) == L.XL_ERR_CONFIG     # dtype
    assert b"dtype" in lib.xl_last_error()
    args = [0, L.XL_JACPCG, L.XL_TEXTBOOK, None, 1, 4, None, 4, None, None, 0, 0, -1.0,
            None, None, None, None, None, None, 0, None]
    assert lib.xl_solve(*args) == L.XL_ERR_CONFIG                                        # T = 0
    assert b"T must be >= 1" in lib.xl_last_error()
    args[2] = 5
    args[11] = 3
    assert lib.xl_solve(*args) == L.XL_ERR_CONFIG                                        # variant
    rz = [0, L.XL_JACPCG, L.XL_TEXTBOOK, None, 1, 8, 4, 1.0, None, 1.0, 4, 0.0]
    rz += [None] * 8 + [0, None]
    assert lib.xl_rzf(*rz) == L.XL_ERR_CONFIG                                            # sigma2 = 0
    assert b"noise power" in lib.xl_last_error()
    assert lib.xl_se_partials(None, 4, 0, None, None) == L.XL_ERR_CONFIG
    assert lib.xl_se_combine(None, 0, None, None) == L.XL_ERR_CONFIG
    # stationary solvers (linsolve.py:128-176): T < 1, omega <= 0, unknown method
    st = [0, L.XL_JOR, None, 1, 4, None, 4, None, 0.5, 0, -1.0] + [None] * 6 + [0, None]
    assert lib.xl_solve_stationary(*st) == L.XL_ERR_CONFIG                               # T = 0
    st[9] = 2
    st[8] = 0.0
    assert lib.xl_solve_stationary(*st) == L.XL_ERR_CONFIG                               # omega = 0
    assert b"omega" in lib.xl_last_error()
    st[1] = L.XL_JACPCG
    assert lib.xl_solve_stationary(*st) == L.XL_ERR_CONFIG                               # not JOR/GS
    # BER chain: bad sizes / dtype
    assert lib.xl_ber_errors(0, None, None, None, 1, 0, 8, None, None) == L.XL_ERR_CONFIG
    assert lib.xl_ber_errors(9, None, None, None, 1, 4, 8, None, None) == L.XL_ERR_CONFIG


def test_status_mapping_to_reference_exceptions():
    from paper_2305_13925_b200 import errors as E
    with pytest.raises(E.NotHpdError):
        L.raise_status([0, 1])
    with pytest.raises(E.SplittingError):
        L.raise_status([2])
    with pytest.raises(E.DegenerateChannelError):
        L.raise_status([0, 0, 3])
    with pytest.raises(E.NotHpdError):
        L.raise_status([4])
    L.raise_status([0, 0, 0])


def test_workspace_queries(lib):
    assert lib.xl_rzf_workspace_bytes(0, 0, 16, 1024, 64) > 0
    # K = 128 (streaming tcgen05 Gram / W): the K x K state (A, X, GX), no copy of H
    M, K, B = 4096, 128, 64
    w128 = lib.xl_rzf_workspace_bytes(0, 0, B, M, K)
    assert 2 * B * K * K * 8 <= w128 < B * M * K * 8
    # K = 256 (large_k.cu): the K x K state, flags / scales and the cluster solver's A slots
    # (64 x 512 KiB), no copy of H
    M, K = 2048, 256
    w256 = lib.xl_rzf_workspace_bytes(0, 0, B, M, K)
    assert 2 * B * K * K * 8 + 64 * 512 * 1024 <= w256 < B * M * K * 8  # 64 cluster slots
    # other large K (split-operand library GEMMs): also the split rows of H (2x its bytes)
    M, K = 2048, 320
    assert lib.xl_rzf_workspace_bytes(0, 0, B, M, K) >= 2 * B * M * K * 8
    # K = 128 with M not a multiple of 64 takes the split-operand path too
    assert lib.xl_rzf_workspace_bytes(0, 0, B, 4000, 128) >= 2 * B * 4000 * 128 * 8
    assert lib.xl_solve_workspace_bytes(1, 16, 64, 64) == 16 * 4 * 64 * 64 * 16
