"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/dvla_b200.h declares, and maps status codes onto the
reference's exception types."""

import ctypes

import pytest


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2605_13276_b200 import _lib
    syms = _lib.exported_symbols()
    assert len(syms) >= 8
    for name in syms:
        assert hasattr(_lib.lib, name), name
        assert ctypes.cast(getattr(_lib.lib, name), ctypes.c_void_p).value


def test_abi_version():
    from paper_2605_13276_b200 import _lib
    assert _lib.dvla_abi_version() == 1


def test_status_mapping_to_reference_exceptions():
    from paper_2605_13276_b200 import _lib
    from paper_2605_13276_b200.core import ConfigError, UsageError
    with pytest.raises(ConfigError):
        _lib.check(_lib.ERR_CONFIG, "x")
    with pytest.raises(UsageError):
        _lib.check(_lib.ERR_USAGE, "x")
    with pytest.raises(_lib.NativeError):
        _lib.check(_lib.ERR_CUDA, "x")


def test_config_errors_are_raised_before_any_device_work():
    """Argument validation happens host-side in the C-ABI (no CUDA calls)."""
    from paper_2605_13276_b200 import _lib
    st = _lib.dvla_token_loss_fwd_bwd(None, 1, None, None, None, None, None, 0, 8, 1, 1, 8,
                                      0.2, 1e-8, 0.0, 0, None, None, None, None, 0, None)
    assert st == _lib.ERR_CONFIG
    assert "at least one group" in _lib.last_error()
    st = _lib.dvla_token_loss_fwd_bwd(None, 1, None, None, None, None, None, 2, 1, 1, 1, 8,
                                      0.2, 1e-8, 0.0, 0, None, None, None, None, 0, None)
    assert st == _lib.ERR_CONFIG and "group_size" in _lib.last_error()


def test_workspace_size_is_monotone():
    from paper_2605_13276_b200 import _lib
    a = _lib.dvla_token_loss_workspace_bytes(64, 8, 1, 56)
    b = _lib.dvla_token_loss_workspace_bytes(128, 8, 1, 56)
    assert 0 < a < b
