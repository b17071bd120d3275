"""CPU-side checks of the C-ABI library: it loads, exports exactly what
include/ep/ep_attn.h declares, and fails cleanly (status + message, no
crash, no fallback) when no B200 is present."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from paper_2504_11729_b200 import _capi


def test_library_exports_every_header_symbol():
    lib = _capi.lib()
    declared = _capi.header_symbols()
    assert "ep_spliced_attention" in declared and "ep_partial_attention_f64" in declared
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T ep_" in l}
    assert set(declared) <= exported
    # nothing exported that the header does not declare
    assert exported <= set(declared), exported - set(declared)


def test_abi_version():
    assert _capi.lib().ep_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in l for l in out.splitlines() if "sm_" in l), out


def test_no_gpu_fails_cleanly_without_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = _capi.lib().ep_create(0, C.byref(h))
    assert rc in (_capi.EP_ECUDA, _capi.EP_EINVAL)
    assert _capi.lib().ep_last_error()
    from paper_2504_11729_b200 import partial_attention, EPError
    with pytest.raises(EPError):
        partial_attention(np.ones((1, 4)), np.ones((2, 4)), np.ones((2, 4)))


def test_shape_errors_are_invalid_argument_before_any_device_work():
    from paper_2504_11729_b200 import partial_attention, full_attention, merge_partials
    from paper_2504_11729_b200 import InvalidArgument, CausalSpan
    with pytest.raises(InvalidArgument):
        partial_attention(np.ones((1, 2)), np.ones((1, 3)), np.ones((1, 3)), CausalSpan(0, 0))
    with pytest.raises(InvalidArgument):
        full_attention(np.ones((1, 2)), np.ones((1, 2)), np.ones((2, 2)), CausalSpan(0, 0))
    with pytest.raises(InvalidArgument):
        partial_attention(np.ones((1, 0)), np.ones((1, 0)), np.ones((1, 0)))
    with pytest.raises(InvalidArgument):
        merge_partials([])
    with pytest.raises(ValueError):  # InvalidArgument is a ValueError like std::invalid_argument
        merge_partials([])
