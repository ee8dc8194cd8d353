"""The C-ABI library loads on a CPU-only host, exports every symbol that
include/neo_tbe.h declares, and rejects bad arguments on the host before
touching the device.  No compute calls (CPU only)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def capi():
    from paper_2104_05158_b200 import _build, _capi

    _build.build()
    return _capi


def declared_symbols():
    text = (ROOT / "include" / "neo_tbe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(neo_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("neo_tbe_forward", "neo_tbe_backward", "neo_bucketize_rowwise", "neo_permute_blocks",
                 "neo_copy_pieces", "neo_apply_row_updates"):
        assert name in syms


def test_every_declared_symbol_exported(capi):
    lib = C.CDLL(str(capi.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(capi.SIGNATURES), "ctypes table out of sync with the header"


def test_binding_loads_and_versions(capi):
    lib = capi.lib()
    assert lib.neo_version() == 10000


def test_host_side_argument_errors(capi):
    lib = capi.lib()
    rc = lib.neo_tbe_forward(-1, 4, None, None, 8, None, capi.NEO_F32, None, capi.NEO_I32, None,
                             capi.NEO_POOL_SUM, None, capi.NEO_F32, 8, None, None)
    assert rc == capi.NEO_E_ARG and "negative" in capi.last_error()
    rc = lib.neo_tbe_forward(1, 4, 1, 1, 8, 1, capi.NEO_F32, 1, 7, 1, capi.NEO_POOL_SUM, 1, capi.NEO_F32,
                             8, None, None)
    assert rc == capi.NEO_E_ARG and "index dtype" in capi.last_error()
    starts = (C.c_int64 * 3)(0, 5, 4)  # not tiling [0, H)
    rc = lib.neo_bucketize_rowwise(1, 1, 1, capi.NEO_I64, 2, starts, 1, 1, 1, -1, None, 1, 1 << 20, None)
    assert rc == capi.NEO_E_ARG and "tile" in capi.last_error()
    with pytest.raises(Exception) as e:
        capi.check(rc, "neo_bucketize_rowwise")
    assert type(e.value).__name__ == "InvalidValue"
    rc = lib.neo_tbe_backward(1, 4, 1, 10, 1, 8, 1, capi.NEO_F32, None, 1, capi.NEO_I32, 1, 4, 0, 1,
                              capi.NEO_F32, 8, capi.NEO_BWD_UPDATE, capi.NEO_OPT_ROWWISE_ADAGRAD,
                              -1.0, 0.0, None, None, None, None, 1, 1, None, None)
    assert rc == capi.NEO_E_ARG and "lr" in capi.last_error()


def test_workspace_queries_host_only(capi):
    lib = capi.lib()
    assert lib.neo_tbe_backward_workspace_bytes(1 << 20, 1 << 20, 128) > 5 * (1 << 22)
    assert lib.neo_tbe_backward_workspace_bytes(1 << 20, 1 << 33, 128) > \
        lib.neo_tbe_backward_workspace_bytes(1 << 20, 1 << 20, 128)
    assert lib.neo_permute_workspace_bytes(8, 64) >= 4 * 8 * 64 * 8
