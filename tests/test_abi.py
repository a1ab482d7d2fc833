"""C-ABI checks that need no GPU: the library loads and exports every entry point declared in
include/pcband.h; host-side argument validation that fails before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pcband.h")
LIB = os.path.join(ROOT, "paper_2511_17107_b200", "libpcband.so")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    d = declared()
    for name in ("pc_create", "pc_apply", "pc_precond", "pc_bands", "pc_gamma", "pc_info", "pc_destroy",
                 "pc_last_error"):
        assert name in d


@pytest.mark.skipif(not os.path.exists(LIB), reason="libpcband.so not built")
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(L, name), name


@pytest.mark.skipif(not os.path.exists(LIB), reason="libpcband.so not built")
def test_supported_sizes_and_invalid_create():
    from paper_2511_17107_b200 import api
    sizes = api.pc_supported_n()
    for n in (8, 32, 64, 128, 192):
        assert n in sizes
    # unsupported n and singular A fail on the host, before any CUDA call
    with pytest.raises(api.PcError) as e:
        api.pc_create(np.eye(3), 7, np.eye(3), np.zeros((4, 7, 7, 7), np.uint8))
    assert e.value.code == api.PC_EINVAL
    with pytest.raises(api.PcError) as e:
        api.pc_create(np.zeros((3, 3)), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
    assert e.value.code == api.PC_EINVAL
    bad = np.eye(3, dtype=complex)
    bad[0, 1] = 0.1j  # not Hermitian
    with pytest.raises(api.PcError) as e:
        api.pc_create(np.eye(3), 8, bad, np.zeros((4, 8, 8, 8), np.uint8))
    assert e.value.code == api.PC_EINVAL
    with pytest.raises(api.PcError) as e:
        api.pc_create(np.eye(3), 8, -np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
    assert e.value.code == api.PC_ENOTPD
    with pytest.raises(api.PcError) as e:  # diagonal mode with off-diagonal eps1
        import synth
        api.pc_create(np.eye(3), 8, synth.eps_pseudochiral(), np.zeros((4, 8, 8, 8), np.uint8), eps_mode="diagonal")
    assert e.value.code == api.PC_EINVAL
